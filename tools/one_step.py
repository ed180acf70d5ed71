"""Warm up, then run ONE resident training step between cudaProfilerStart/Stop
(for `ncu --profile-from-start off`): the launch list of exactly one step."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
ds = make_dataset(1024, seed=2)
perm = np.random.default_rng(7).permutation(ds.num_graphs)
res = [upload_batch(*ds.collate(perm[i * 256:(i + 1) * 256]), build_csr=False) for i in range(4)]
model = gnn.create_model(hidden=512, seed=0, normalizer=gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
tr = BatchTrainer(model, precision=prec)
tr.reserve(max(b.N for b in res), 256)
for i in range(3):
    tr.step_resident(res[i])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tr.step_resident(res[3])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("one step done")
