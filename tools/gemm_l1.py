"""Layer-1/2-shaped forward GEMM (M 76.8k nodes, N 512) in isolation: K, with/without the 1-bit
masks, tile mode; event-timed.  DIPPM_GEMM_DEBUG bits switch parts of the epilogue off
(diagnostics).  Usage: python tools/gemm_l1.py K [bits 0/1] [cta_pair 0/1/2]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, device as dev  # noqa: E402
from paper_2303_11733_b200.device import ActBuf  # noqa: E402

import os
M, N = int(os.environ.get("GEMM_M", 76800)), 512
K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
use_bits = int(sys.argv[2]) if len(sys.argv) > 2 else 1
pair = int(sys.argv[3]) if len(sys.argv) > 3 else 0
TS = torch.zeros(148 * 4, dtype=torch.int64, device="cuda")
if os.environ.get("GEMM_TS_DUMP"):
    os.environ["DIPPM_GEMM_TS"] = hex(TS.data_ptr())
lib = _lib.load()
A = ActBuf(M, K, dev.DT_BF16, "cuda")
A.t.normal_()
W = ActBuf(K, N, dev.DT_BF16, "cuda")
W.t.normal_()
out = ActBuf(M, 2 * N, dev.DT_BF16, "cuda")
bias = torch.zeros(N, device="cuda")
bits = torch.empty(N // 32, M, dtype=torch.int32, device="cuda")
args = _lib.GemmArgs(0, M, N, K, A.view(), 0, W.view(), 1, bias.data_ptr(), 1,
                     _lib.Act(out.t.data_ptr(), 2 * N, 0, dev.DT_BF16), None, 0, 1)
if use_bits:
    args.relu_bits, args.bits_ld = bits.data_ptr(), M
args.cta_pair = pair
for _ in range(5):
    _lib.check(lib.dippm_gemm(args, 0, dev._stream()))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    _lib.check(lib.dippm_gemm(args, 0, dev._stream()))
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"K={K} bits={use_bits} pair={pair}: {us:.1f} us  ({2 * M * N * K / us / 1e6:.0f} TFLOP/s, "
      f"{(M * N * 2 + M * K * 2 + use_bits * M * N / 8) / us / 1e3:.0f} GB/s)")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            _lib.check(lib.dippm_gemm(args, 0, dev._stream()))
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"   in a CUDA graph: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per launch")
if os.environ.get("GEMM_TS_DUMP"):
    ts = TS.cpu().numpy().astype("int64").reshape(148, 4)
    n = int((ts[:, 0] > 0).sum())
    t0 = ts[:n, 0].min()
    rel = (ts[:n] - t0) / 1e3
    import numpy as np
    print(f"CTAs {n}: start spread {rel[:, 0].max():.2f} us; prologue mean {np.mean(rel[:, 1] - rel[:, 0]):.2f} "
          f"max {np.max(rel[:, 1] - rel[:, 0]):.2f}; epi-done min {rel[:, 2].min():.2f} max {rel[:, 2].max():.2f}; "
          f"end max {rel[:, 3].max():.2f} us")
