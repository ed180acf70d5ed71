import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2303_11733_b200 import _lib, device as dev
rng = np.random.default_rng(3)
G = 37
n = rng.integers(1, 50, G)
gp = np.zeros(G + 1, np.int32); np.cumsum(n, out=gp[1:])
h = torch.from_numpy(rng.normal(size=(gp[-1], 64)).astype(np.float32)).cuda()
fs = torch.from_numpy(rng.normal(size=(G, 5)).astype(np.float32)).cuda()
norm = torch.from_numpy(np.concatenate([np.zeros(6), rng.normal(size=5), rng.uniform(0.5, 2, 5)])).cuda()
gpt = torch.from_numpy(gp).cuda()
u = torch.empty(G, 69, device="cuda")
try:
    _lib.call("dippm_pool_concat", dev.f32_act(h), gpt.data_ptr(), G, 64, fs.data_ptr(), norm.data_ptr(), u.data_ptr(), dev._stream())
    torch.cuda.synchronize(); print("ok", u[0, :4])
except Exception as e:
    print("ERR", repr(e))
