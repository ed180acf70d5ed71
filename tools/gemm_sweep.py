"""FWD GEMM throughput vs shape (tcgen05 kernel, bf16) next to cuBLAS (torch.matmul) on the same shapes."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, device as dev  # noqa: E402
from paper_2303_11733_b200.device import ActBuf  # noqa: E402

lib = _lib.load()


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


SHAPES = [(76800, 512, 64), (76800, 512, 1024), (76800, 512, 4096), (76800, 1024, 1024), (76800, 2048, 1024),
          (8192, 8192, 8192)]
if len(sys.argv) > 1:
    SHAPES = SHAPES[:int(sys.argv[1])]
for M, N, K in SHAPES:
    A = ActBuf(M, K, dev.DT_BF16, "cuda"); A.t.normal_()
    W = ActBuf(N, K, dev.DT_BF16, "cuda"); W.t.normal_()
    out = ActBuf(M, N, dev.DT_BF16, "cuda")
    bias = torch.zeros(N, device="cuda")
    res = []
    bits = torch.empty(N // 32, M, dtype=torch.int32, device="cuda")
    out32 = ActBuf(M, N, dev.DT_F32, "cuda")
    for pair, ob, bp, tag in ((1, out, None, "pair1"), (2, out, None, "pair2"), (2, out, bits, "pair2+bits"),
                              (2, out32, None, "pair2 f32out")):
        args = _lib.GemmArgs(0, M, N, K, A.view(), 0, W.view(), 0, bias.data_ptr(), 1, ob.view(), None, 0, 1,
                             dev.NULL_ACT, 1.0, 0, None, 0, 0.0, 0, None, None if bp is None else bp.data_ptr(),
                             None, M, pair, None, 1.0)
        us = timeit(lambda: _lib.check(lib.dippm_gemm(args, 0, dev._stream())))
        res.append(f"{tag} {us:7.1f} us {2 * M * N * K / us / 1e6:7.1f} TF/s")
    a, w = A.t, W.t
    us = timeit(lambda: torch.matmul(a, w.t()))
    res.append(f"cuBLAS {us:7.1f} us {2 * M * N * K / us / 1e6:7.1f} TF/s")
    print(f"M={M} N={N} K={K}: " + " | ".join(res), flush=True)
    del A, W, out
