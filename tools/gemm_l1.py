"""Layer-1-shaped forward GEMM (K=64) in isolation, for ncu."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, device as dev  # noqa: E402
from paper_2303_11733_b200.device import ActBuf  # noqa: E402

M, N, K = 76800, 512, int(sys.argv[1]) if len(sys.argv) > 1 else 64
lib = _lib.load()
A = ActBuf(M, K, dev.DT_BF16, "cuda")
A.t.normal_()
W = ActBuf(K, N, dev.DT_BF16, "cuda")
W.t.normal_()
out = ActBuf(M, 2 * N, dev.DT_BF16, "cuda")
bias = torch.zeros(N, device="cuda")
args = _lib.GemmArgs(0, M, N, K, A.view(), 0, W.view(), 1, bias.data_ptr(), 1,
                     _lib.Act(out.t.data_ptr(), 2 * N, 0, dev.DT_BF16), None, 0, 1)
for _ in range(5):
    _lib.check(lib.dippm_gemm(args, 0, dev._stream()))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    _lib.check(lib.dippm_gemm(args, 0, dev._stream()))
e1.record()
torch.cuda.synchronize()
print(f"K={K}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
