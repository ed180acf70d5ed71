"""Layer-1 WGRAD shapes (x = [N, 64], dz = [N, 512]) in both orientations, fused or not."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, device as dev  # noqa: E402
from paper_2303_11733_b200.device import ActBuf  # noqa: E402

lib = _lib.load()
R = 76800
dt = dev.DT_BF16
X = ActBuf(R, 64, dt, "cuda"); X.t.normal_()
DZ = ActBuf(R, 1024, dt, "cuda"); DZ.t.normal_()
ws = torch.empty(200 * 64 * 1024, device="cuda")
sync = torch.zeros(4096, dtype=torch.int32, device="cuda")
out = torch.empty(1024 * 1024, device="cuda")


def run(M, N, a, b, S, fused, pair):
    args = _lib.GemmArgs(2, M, N, R, a, 1, b, 1, None, 0, dev.Act(out.data_ptr(), N, 0, 0) if fused else dev.NULL_ACT,
                         ws.data_ptr(), N, S, dev.NULL_ACT, 1.0, 0, None, 0, 0.0, 0, None, None, None, 0, pair,
                         sync.data_ptr() if fused else None, 1.0)
    return lambda: _lib.check(lib.dippm_gemm(args, 0, dev._stream()))


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for S in (None, 8, 16, 37):
    s_new = S or lib.dippm_wgrad_splits(64, 512, R)
    s_old = S or lib.dippm_wgrad_splits(512, 64, R)
    for fused in (False, True):
        t_new = timeit(run(64, 512, X.view(), DZ.view(), s_new, fused, 1))
        t_old = timeit(run(512, 64, DZ.view(), X.view(), s_old, fused, 1))
        print(f"S={S} fused={fused}: new orientation (M=64,N=512,S={s_new}) {t_new:7.1f} us | "
              f"old (M=512,N=64,S={s_old}) {t_old:7.1f} us")
