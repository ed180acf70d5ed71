"""A few small training steps + predict through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): bf16 and fp32, sage and mlp, resident and host batches."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402

ds = make_dataset(40, seed=5, n_lo=20, n_hi=200)
norm = gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float))
for prec in ("bf16", "fp32"):
    model = gnn.create_model(hidden=256, seed=1, normalizer=norm)
    tr = BatchTrainer(model, precision=prec, dropout=True)
    b = upload_batch(*ds.collate(np.arange(0, 24)), device="cuda", build_csr=False)
    tr.step_resident(b)
    tr.step_host(*ds.collate(np.arange(10, 40)))
    recs = ds.records(range(8))
    gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs], precision=prec)
    gnn.backward(model, recs[:4], precision=prec)
mlp = gnn.create_mlp_model(hidden=128, seed=2, normalizer=norm)
gnn.backward(mlp, ds.records(range(6)))
torch.cuda.synchronize()
print("sanitize step done")
