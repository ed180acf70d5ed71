"""Weight-gradient GEMM at the bench shapes, event-timed, with per-CTA phase stamps
(DIPPM_GEMM_TS): prologue, MMA done, partial written, reduce start.  Default: layer 1
(A1 = [X | agg X | 1 | 0] [R, 128] -> M = 65, dz1 [R, 512] in a [R, 1024] buffer, K = R = 76.8k
rows, fused split-K reduce); LAYER=2: layers 2-3 (A = [h | agg h] [R, 1024] -> M = 1024)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
TS = torch.zeros(1024 * 8, dtype=torch.int64, device="cuda")
os.environ["DIPPM_GEMM_TS"] = hex(TS.data_ptr())
from paper_2303_11733_b200 import _lib, device as dev  # noqa: E402
from paper_2303_11733_b200.device import ActBuf  # noqa: E402

lib = _lib.load()
R = int(os.environ.get("ROWS", 76800))
L23 = os.environ.get("LAYER", "1") != "1"
M, N = (1024, 512) if L23 else (65, 512)
A1 = ActBuf(R, 1024 if L23 else 128, dev.DT_BF16, "cuda"); A1.t.normal_()
DZ = ActBuf(R, 1024, dev.DT_BF16, "cuda"); DZ.t.normal_()
S = int(os.environ.get("SPLITS", 0)) or lib.dippm_wgrad_splits(M, N, R)
ws = torch.empty(S * max(M, 128) * N, device="cuda")
sync = torch.zeros(4096, dtype=torch.int32, device="cuda")
out = torch.empty(M * N, device="cuda")
args = _lib.GemmArgs(2, M, N, R, A1.view(), 1, _lib.Act(DZ.t.data_ptr(), 1024, 0, dev.DT_BF16), 1, None, 0,
                     _lib.Act(out.data_ptr(), N, 0, dev.DT_F32), ws.data_ptr(), N, S)
args.tile_sync, args.out_scale = sync.data_ptr(), 1.0
fn = lambda: _lib.check(lib.dippm_gemm(args, 0, dev._stream()))  # noqa: E731
for _ in range(3):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    fn()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
mb = (R * N * 2 + 2 * R * 64 * 2 + 2 * S * M * N * 4) / 1e6
print(f"WGRAD_1 R={R} S={S}: {us:.1f} us  (~{mb:.0f} MB -> {mb / us * 1e3:.0f} GB/s)")
ts = TS.cpu().numpy().reshape(1024, 8).astype(np.int64)
n = int((ts[:, 0] > 0).sum())
t0 = ts[:n, 0].min()
rel = (ts[:n] - t0) / 1e3
for k, name in [(1, "prologue done"), (4, "MMA done (1st tfull)"), (5, "partial written"), (6, "reduce start"),
                (2, "epilogue done"), (3, "end")]:
    print(f"  {name:22s} min {rel[:, k].min():6.2f}  mean {rel[:, k].mean():6.2f}  max {rel[:, k].max():6.2f} us")
