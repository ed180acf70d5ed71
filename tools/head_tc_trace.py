"""Phase timeline of the tensor-core FC head (dippm_head_tc_trace) inside a configs[1] step."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, gnn  # noqa: E402
from paper_2303_11733_b200.device import upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402

lib = _lib.load()
lib.dippm_head_tc_enable(1)
ds = make_dataset(768, seed=2)
model = gnn.create_model(hidden=512, seed=0, normalizer=gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
tr = BatchTrainer(model, precision="bf16")
res = [upload_batch(*ds.collate(np.arange(i * 256, (i + 1) * 256)), build_csr=False) for i in range(3)]
tr.reserve(max(b.N for b in res), 256)
for b in res:
    tr.step_resident(b)
torch.cuda.synchronize()
buf = (C.c_uint64 * 16)()
lib.dippm_head_tc_trace(buf)
t = np.array(buf[:9], dtype=np.int64)
names = ["P1 fc1", "P2 fc2", "C fc3/loss", "D d2/db2", "P3 GATE+db1", "P4 dW2", "P5 du", "P6 dW1"]
for i, n in enumerate(names):
    print(f"{n:12s} {(t[i + 1] - t[i]) / 1e3:7.2f} us")
print(f"total {(t[8] - t[0]) / 1e3:.2f} us (after setup)")
