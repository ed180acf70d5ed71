"""Probe the layer-2/3 forward GEMM (bf16, CTA pair, bias+ReLU+bits) over M and K:
per-call time and TFLOP/s.  Run with DIPPM_GEMM_DEBUG=4 to skip the epilogue (mainloop only).
usage: python tools/gemm_probe.py [kind] ; kind = fwd | gate | wgrad"""
import os
import sys

import numpy as np

import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, device as dev  # noqa: E402
from paper_2303_11733_b200.device import ActBuf  # noqa: E402

lib = _lib.load()
kind = sys.argv[1] if len(sys.argv) > 1 else "fwd"


def act(rows, cols):
    a = ActBuf(rows, cols, dev.DT_BF16, "cuda")
    a.t.normal_()
    return a


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def g(k, a, amn, b, bmn, Mm, Nn, Kk, pool=(None, None, None, None), **kw):
    f = dict(bias=None, relu=0, out=dev.NULL_ACT, c=None, ldc=0, splits=1, gate=dev.NULL_ACT, gate_scale=1.0,
             drop_mode=0, mask=None, ldm=0, drop_p=0.0, seed=0, relu_bits=None, gate_bits=None, bits_ld=0,
             cta_pair=2, tile_sync=None, out_scale=1.0)
    f.update(kw)
    args = _lib.GemmArgs(k, Mm, Nn, Kk, a, amn, b, bmn, f["bias"], f["relu"], f["out"], f["c"], f["ldc"],
                         f["splits"], f["gate"], f["gate_scale"], f["drop_mode"], f["mask"], f["ldm"],
                         f["drop_p"], f["seed"], None, f["relu_bits"], f["gate_bits"], f["bits_ld"],
                         f["cta_pair"], f["tile_sync"], f["out_scale"], *pool)
    return lambda: _lib.check(lib.dippm_gemm(args, 0, dev._stream()))


N = 512
tag = os.environ.get("DIPPM_GEMM_DEBUG", "0")
for K in (1024, 4096):
    for M in (75776, 76800, 77568, 37888):
        A = act(M, K)
        Wmn = act(K, N)
        Wk = act(N, K)
        out = act(M, N)
        bias = torch.zeros(N, device="cuda")
        bits = torch.zeros(N // 32, M, dtype=torch.int32, device="cuda")
        if kind == "pool":  # layer-3 forward: fused readout epilogue (graphs of ~300 nodes), no stored output
            rng = np.random.default_rng(0)
            sizes = rng.integers(270, 331, M // 250)
            sizes = sizes[np.cumsum(sizes) <= M]
            gp = np.zeros(len(sizes) + 1, np.int32)
            np.cumsum(sizes, out=gp[1:])
            gp[-1] = M
            gp_t = torch.from_numpy(gp).cuda()
            ng = torch.from_numpy(np.repeat(np.arange(len(sizes), dtype=np.int32), np.diff(gp))).cuda()
            pp = torch.empty(lib.dippm_pool_partial_rows(M), N, device="cuda")
            pg = torch.empty(len(sizes), N, device="cuda")
            keep = (gp_t, ng, pp, pg)
            fn = g(0, A.view(), 0, Wmn.view(), 1, M, N, K, bias=bias.data_ptr(), relu=1, out=dev.NULL_ACT,
                   relu_bits=bits.data_ptr(), bits_ld=0, pool=(pp.data_ptr(), pg.data_ptr(), ng.data_ptr(), gp_t.data_ptr()))
        elif kind == "fwd":
            fn = g(0, A.view(), 0, Wmn.view(), 1, M, N, K, bias=bias.data_ptr(), relu=1, out=out.view(),
                   relu_bits=bits.data_ptr(), bits_ld=M)
        else:
            fn = g(3, A.view(), 0, Wk.view(), 0, M, N, K, out=out.view(), gate_bits=bits.data_ptr(), bits_ld=M)
        ms = timeit(fn)
        fl = 2.0 * M * N * K
        ref = timeit(lambda: torch.matmul(A.t, Wmn.t))
        print(f"dbg={tag} {kind} M={M:6d} K={K}: {ms*1e3:7.1f} us {fl/ms/1e9:7.1f} TF/s   cublas {ref*1e3:7.1f} us {fl/ref/1e9:7.1f}")
        del A, Wmn, Wk, out, bits
