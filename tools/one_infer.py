"""Warm up, then run ONE configs[2] inference batch (G = 4096, hidden 512, bf16) between
cudaProfilerStart/Stop (for `ncu --profile-from-start off`)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import Engine, upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ds = make_dataset(G, seed=3)
model = gnn.create_model(hidden=512, seed=0, normalizer=gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
eng = gnn._engine(model, "bf16")
b = upload_batch(*ds.collate(np.arange(G)), device="cuda")
ws = gnn.infer_workspace(eng, b.N, b.G)
for _ in range(3):
    eng.forward(b, ws, predict=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.forward(b, ws, predict=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("one inference batch done")
