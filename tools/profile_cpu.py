"""Host-side cost of one training step (cProfile) and GPU-side time with syncs."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402

ds = make_dataset(4096, seed=2)
perm = np.random.default_rng(7).permutation(ds.num_graphs)
hb = [ds.collate(perm[i * 256:(i + 1) * 256]) for i in range(12)]
model = gnn.create_model(hidden=512, seed=0, normalizer=gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
tr = BatchTrainer(model, precision=sys.argv[1] if len(sys.argv) > 1 else "bf16")
res = [upload_batch(*b, device="cuda", build_csr=False) for b in hb]
tr.reserve(max(b.N for b in res), 256)
for i in range(4):
    tr.step_resident(res[i])
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(8):
    tr.step_resident(res[4 + i % 8])
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"enqueue {1e3 * (t1 - t0) / 8:.2f} ms/step, complete {1e3 * (t2 - t0) / 8:.2f} ms/step")
for i in range(3):
    torch.cuda.synchronize()
    a = time.perf_counter()
    tr.step_resident(res[i])
    torch.cuda.synchronize()
    print(f"synced step {1e3 * (time.perf_counter() - a):.2f} ms")
pr = cProfile.Profile()
pr.enable()
for i in range(8):
    tr.step_resident(res[i % 8])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
