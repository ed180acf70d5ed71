"""Where the end-to-end step's time goes: host time of each BatchTrainer.submit call, and the
device timeline (events on the compute and copy streams) of a short pipelined run."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import group_edges  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402

ds = make_dataset(2560, seed=2)
perm = np.random.default_rng(7).permutation(ds.num_graphs)
model = gnn.create_model(hidden=512, seed=0, normalizer=gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
tr = BatchTrainer(model, precision="bf16")
batches = []
for i in range(10):
    b = ds.collate(perm[i * 256:(i + 1) * 256])
    batches.append([torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                    for a in (*b[:4], b[4].astype(np.float64), b[5].astype(np.float64), group_edges(b[1], b[2], b[3]))])
for i in range(3):
    tr.step_host(*batches[i])
torch.cuda.synchronize()
K = 10
ev = []
host = []
t0 = time.perf_counter()
hs = []
for i in range(K):
    a = time.perf_counter()
    hs.append(tr.submit(*batches[i]))
    host.append(time.perf_counter() - a)
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    ev.append(e)
t_sub = time.perf_counter() - t0
for h in hs:
    h.loss()
torch.cuda.synchronize()
t_all = time.perf_counter() - t0
print(f"host per submit (us): {[round(1e6 * h) for h in host]}")
print(f"submit loop {1e3 * t_sub / K:.3f} ms/step, wall incl drain {1e3 * t_all / K:.3f} ms/step")
print("device step-end deltas (us):", [round(1e3 * ev[i - 1].elapsed_time(ev[i])) for i in range(1, K)])
