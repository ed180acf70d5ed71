"""Stress the global-path CSR build for run-to-run determinism (random multigraphs)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200.device import upload_batch  # noqa: E402
from oracle import dippm_oracle as O  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(1)
N, E = 5000, 40000
src = rng.integers(0, N, E)
dst = rng.integers(0, N, E)
x = np.zeros((N, 32), np.float32)
fs = np.zeros((1, 5), np.float32)
gp = np.array([0, N], np.int32)
rowptr, col, deg = O.csr_of_aggregation(N, list(zip(src.tolist(), dst.tolist())))
bad = 0
for r in range(reps):
    a = upload_batch(x, src, dst, gp, fs)
    ok = {"rowptr": np.array_equal(a.rowptr.cpu().numpy(), rowptr),
          "col": np.array_equal(a.col.cpu().numpy()[:len(col)], col),
          "deg": np.array_equal(a.deg.cpu().numpy(), deg)}
    if not all(ok.values()):
        bad += 1
        rp = a.rowptr.cpu().numpy()
        print("rep", r, ok, "first rowptr diff at", np.argmax(rp != rowptr) if not ok["rowptr"] else None, flush=True)
print(f"{bad} of {reps} builds differ from the oracle")
