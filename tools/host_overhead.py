"""CPU cost of submitting one eager training step (BatchTrainer.submit with pinned host
batches) vs its GPU time: is the end-to-end path host-bound?  Also a cProfile of the
submission loop (top functions by own time)."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import group_edges  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402

ds = make_dataset(2048, seed=2)
model = gnn.create_model(hidden=512, seed=0, normalizer=gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
tr = BatchTrainer(model, precision="bf16")
batches = []
for i in range(8):
    b = ds.collate(np.arange(i * 256, (i + 1) * 256))
    batches.append([torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (*b, group_edges(b[1], b[2], b[3]))])
for i in range(4):
    tr.step_host(*batches[i % 8])
torch.cuda.synchronize()
K = 40
t0 = time.perf_counter()
hs = [tr.submit(*batches[i % 8]) for i in range(K)]
t1 = time.perf_counter()
for h in hs:
    h.loss()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"submit: {1e3 * (t1 - t0) / K:.3f} ms CPU per step; wall incl. drain {1e3 * (t2 - t0) / K:.3f} ms per step")
pr = cProfile.Profile()
pr.enable()
hs = [tr.submit(*batches[i % 8]) for i in range(K)]
pr.disable()
for h in hs:
    h.loss()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
