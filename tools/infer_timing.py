"""configs[2] inference step split: CSR build vs forward (CUDA events, eager, as bench.py)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import Engine, Workspace, build_batch_csr, upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402

B = 4096
ds = make_dataset(2 * B, seed=3)
norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
model = gnn.create_model(hidden=512, seed=0, normalizer=norm)
batches = [upload_batch(*ds.collate(np.arange(i * B, (i + 1) * B)), device="cuda", build_csr=False) for i in range(2)]
eng = Engine(512, "bf16")
eng.set_params(model.param_items(), norm)
ws = Workspace(eng, max(b.N for b in batches), B, train=False)
for i in range(3):
    build_batch_csr(batches[i % 2])
    eng.forward(batches[i % 2], ws, predict=True)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
t_csr = t_fwd = 0.0
for i in range(10):
    b = batches[i % 2]
    ev[0].record()
    build_batch_csr(b)
    ev[1].record()
    eng.forward(b, ws, predict=True)
    ev[2].record()
    torch.cuda.synchronize()
    t_csr += ev[0].elapsed_time(ev[1])
    t_fwd += ev[1].elapsed_time(ev[2])
print(f"per batch: csr {t_csr / 10:.3f} ms, forward {t_fwd / 10:.3f} ms")
