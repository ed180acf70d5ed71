"""Break the configs[4] predict-from-JSON path into its parts (wall clock, best of 3):
featurise, collate (numpy) vs collate_pinned (native, pinned), upload + CSR, forward, read-back."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_11733_b200 import featurize as F  # noqa: E402
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_graph_documents  # noqa: E402


def best(fn, reps=3):
    out, ts = None, []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return out, min(ts) * 1e3


docs = [d.encode() for d in make_graph_documents(2048, seed=50)]
fb, t_feat = best(lambda: F.featurize_documents(docs))
norm = gnn.Normalizer(np.array([5.0, 74000.0, 2.0]), np.array([3.0, 150000.0, 1.0]),
                      fb.fs_vectors().mean(0), fb.fs_vectors().std(0) + 1e-3)
model = gnn.create_model(hidden=512, seed=0, normalizer=norm)
F.predict_featurized(model, fb, "bf16")
_, t_col = best(lambda: fb.collate())
arrs, t_colp = best(lambda: fb.collate_pinned())
eng = gnn._engine(model, "bf16")
b, t_up = best(lambda: upload_batch(*arrs[:5], None, device=eng.device, build_csr=True, edge_ptr=arrs[5]))
np_arrs = fb.collate()
_, t_up_np = best(lambda: upload_batch(*np_arrs[:5], None, device=eng.device, build_csr=True, edge_ptr=np_arrs[5]))
ws = gnn.infer_workspace(eng, b.N, b.G)
_, t_fwd = best(lambda: eng.forward(b, ws))
_, t_rb = best(lambda: (ws.y_pred[:b.G].cpu().numpy(), ws.mig[:b.G].cpu().numpy(), int(ws.nonfinite.item())))
_, t_pf = best(lambda: F.predict_featurized(model, fb, "bf16"))
_, t_all = best(lambda: F.predict_documents(model, docs, precision="bf16"))
print(f"G={len(docs)} N={b.N} E={b.E}  x32 {b.N * 128 / 1e6:.1f} MB")
for k, v in [("featurise", t_feat), ("collate numpy", t_col), ("collate_pinned", t_colp), ("upload+csr pinned", t_up),
             ("upload+csr numpy", t_up_np), ("forward", t_fwd), ("readback", t_rb), ("predict_featurized", t_pf),
             ("predict_documents", t_all)]:
    print(f"{k:22s} {v:8.2f} ms")
docs4 = [d.encode() for d in make_graph_documents(8192, seed=51)]
_, t_f4 = best(lambda: F.featurize_documents(docs4))
print(f"featurise 8192         {t_f4:8.2f} ms  ({8192 / t_f4 * 1e3:.0f} docs/s)")
for chunk in (0, 4096, 2048, 1024, 512):
    _, t = best(lambda: F.predict_documents(model, docs4, precision="bf16", chunk=chunk))
    print(f"predict 8192 chunk {chunk:5d} {t:8.2f} ms  ({8192 / t * 1e3:.0f} docs/s)")
