"""Micro-benchmark of the tcgen05 GEMM variants at the training-step shapes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, device as dev  # noqa: E402
from paper_2303_11733_b200.device import ActBuf  # noqa: E402

N_NODES = int(sys.argv[1]) if len(sys.argv) > 1 else 76800
lib = _lib.load()


def act(rows, cols, dt):
    a = ActBuf(rows, cols, dt, "cuda")
    if dt == dev.DT_BF16:
        a.t.normal_()
    else:
        a.t[0].normal_()
        a.t[1].zero_()
    return a


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
    return e0.elapsed_time(e1) / reps


for prec in ("bf16", "fp32"):
    dt = dev.PRECISIONS[prec]
    M, K, N = N_NODES, 1024, 512
    A = act(M, K, dt)
    Wk = act(N, K, dt)       # K-major B [N, K]
    Wmn = act(K, N, dt)      # MN-major B [K, N]
    out = act(M, N, dt)
    gate = act(M, N, dt)
    bias = torch.zeros(N, device="cuda")
    c = torch.empty(M, 2 * N, device="cuda")
    dz = act(M, N, dt)
    S = lib.dippm_wgrad_splits(N, K, M)
    ws = torch.empty(S * N * K, device="cuda")
    fl = 2.0 * M * N * K

    def g(kind, a, amn, b, bmn, Mm, Nn, Kk, **kw):
        f = dict(bias=None, relu=0, out=dev.NULL_ACT, c=None, ldc=0, splits=1, gate=dev.NULL_ACT, gate_scale=1.0,
                 drop_mode=0, mask=None, ldm=0, drop_p=0.0, seed=0, relu_bits=None, gate_bits=None, bits_ld=0,
                 cta_pair=0, tile_sync=None, out_scale=1.0)
        f.update(kw)
        args = _lib.GemmArgs(kind, Mm, Nn, Kk, a, amn, b, bmn, f["bias"], f["relu"], f["out"], f["c"], f["ldc"],
                             f["splits"], f["gate"], f["gate_scale"], f["drop_mode"], f["mask"], f["ldm"],
                             f["drop_p"], f["seed"], None, f["relu_bits"], f["gate_bits"], f["bits_ld"],
                             f["cta_pair"], f["tile_sync"], f["out_scale"])
        return lambda: _lib.check(lib.dippm_gemm(args, 0, dev._stream()))

    bits = torch.zeros(N // 32, M, dtype=torch.int32, device="cuda")
    Sf = lib.dippm_wgrad_splits(K, N, M)
    sync = torch.zeros(lib.dippm_wgrad_sync_ints(K, N), dtype=torch.int32, device="cuda")
    wout = torch.empty(K, N, device="cuda")
    X1 = act(M, 64, dt)
    S1 = lib.dippm_wgrad_splits(64, N, M)
    wout1 = torch.empty(64, N, device="cuda")
    cases = {}
    for pair in (1, 2):
        cases.update({
            f"fwd  A:K B:K  pair{pair}": g(0, A.view(), 0, Wk.view(), 0, M, N, K, bias=bias.data_ptr(), relu=1,
                                           out=out.view(), cta_pair=pair),
            f"fwd  A:K B:MN pair{pair}": g(0, A.view(), 0, Wmn.view(), 1, M, N, K, bias=bias.data_ptr(), relu=1,
                                           out=out.view(), cta_pair=pair),
            f"fwd +bits     pair{pair}": g(0, A.view(), 0, Wmn.view(), 1, M, N, K, bias=bias.data_ptr(), relu=1,
                                           out=out.view(), relu_bits=bits.data_ptr(), bits_ld=M,
                                           cta_pair=pair),
            f"gate values   pair{pair}": g(3, A.view(), 0, Wk.view(), 0, M, N, K, out=out.view(), gate=gate.view(),
                                           cta_pair=pair),
            f"gate bits     pair{pair}": g(3, A.view(), 0, Wk.view(), 0, M, N, K, out=out.view(),
                                           gate_bits=bits.data_ptr(), bits_ld=M, cta_pair=pair),
            f"store(N=1024) pair{pair}": g(1, dz.view(), 0, Wmn.view(), 0, M, K, N, c=c.data_ptr(), ldc=K,
                                           cta_pair=pair),
            f"wgrad MN/MN   pair{pair}": g(2, dz.view(), 1, A.view(), 1, N, K, M, c=ws.data_ptr(), ldc=K, splits=S,
                                           cta_pair=pair),
            f"wgrad fused   pair{pair}": g(2, A.view(), 1, dz.view(), 1, K, N, M, c=ws.data_ptr(), ldc=N, splits=Sf,
                                           out=dev.f32_act(wout), tile_sync=sync.data_ptr(), cta_pair=pair),
            f"wgrad fused l1 (M=64)   ": g(2, X1.view(), 1, dz.view(), 1, 64, N, M, c=ws.data_ptr(), ldc=N, splits=S1,
                                           out=dev.f32_act(wout1), tile_sync=sync.data_ptr(), cta_pair=pair),
        })
    for name, fn in cases.items():
        ms = timeit(fn)
        print(f"{prec} {name} {ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TFLOP/s")
