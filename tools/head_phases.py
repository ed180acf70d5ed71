"""Per-phase timing of the fused head kernel (globaltimer stamps of CTA 0) on a configs[1]
training step (G = 256, hidden 512, bf16), plus the kernel time from CUDA events."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, gnn  # noqa: E402
from paper_2303_11733_b200.device import Engine, Workspace, upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 256
ds = make_dataset(G, seed=2)
model = gnn.create_model(hidden=512, seed=0, normalizer=gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
b = upload_batch(*ds.collate(range(G)), device="cuda")
eng = Engine(512, "bf16")
eng.set_params(model.param_items(), model.normalizer)
ws = Workspace(eng, b.N, b.G, train=True)
eng.forward(b, ws, predict=False, defer_head=True)
eng.loss(b, ws, 1.0)
torch.cuda.synchronize()
pend = dict(ws.head_pending)
lib = _lib.load()
out = np.zeros(24, np.int64)
rows = []
for it in range(20):
    eng._head_fused(b, ws, pend["mask_mode"], pend["dropout_p"], pend["seed"], False,
                    loss=(pend["delta"], pend["grad_den"]), defer_wgrad="--defer" in sys.argv)
    torch.cuda.synchronize()
    lib.dippm_head_fused_trace(out.ctypes.data)
    rows.append(out.copy())
r = np.median(np.array(rows[5:]), 0) / 1.9e3  # cycles -> us at ~1.9 GHz
names = {1: "A landed", 2: "A unit0", 3: "A all", 4: "A sync", 5: "B landed", 6: "B unit0", 7: "B all", 8: "B sync",
         9: "C all", 10: "C sync", 11: "D landed", 12: "D unit0", 13: "D all", 14: "D sync", 15: "E landed",
         16: "E unit0", 17: "E all", 18: "E sync"}
print(f"G={G} (us since start, CTA 0):\n" + "\n".join(f"  {v:9s} {r[k]:7.2f}" for k, v in names.items()))
