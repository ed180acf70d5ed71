"""Share of K1 (CSR build) in a configs[2] inference batch (4096 graphs, hidden 512, bf16):
event-timed K1 alone, the forward alone, and both, on resident batches."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import Engine, Workspace, build_batch_csr, upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402

ds = make_dataset(8192, seed=3)
norm = gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float))
model = gnn.create_model(hidden=512, seed=0, normalizer=norm)
eng = Engine(512, "bf16")
eng.set_params(model.param_items(), model.normalizer)
bs = [upload_batch(*ds.collate(np.arange(i * 4096, (i + 1) * 4096)), device="cuda", build_csr=False) for i in range(2)]
ws = Workspace(eng, max(b.N for b in bs), 4096, train=False)


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


k1 = timed(lambda i=0: build_batch_csr(bs[i % 2]))
fw = timed(lambda i=0: eng.forward(bs[i % 2], ws, predict=True))
both = timed(lambda i=0: (build_batch_csr(bs[i % 2]), eng.forward(bs[i % 2], ws, predict=True)))
print(f"N = {bs[0].N}: K1 {k1:.1f} us, forward {fw:.1f} us, K1 + forward {both:.1f} us per 4096-graph batch")
