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
                 drop_mode=0, mask=None, ldm=0, drop_p=0.0, seed=0)
        f.update(kw)
        args = _lib.GemmArgs(kind, Mm, Nn, Kk, a, amn, b, bmn, f["bias"], f["relu"], f["out"], f["c"], f["ldc"],
                             f["splits"], f["gate"], f["gate_scale"], f["drop_mode"], f["mask"], f["ldm"],
                             f["drop_p"], f["seed"])
        return lambda: _lib.check(lib.dippm_gemm(args, 0, dev._stream()))

    cases = {
        "fwd  A:K B:K  ": g(0, A.view(), 0, Wk.view(), 0, M, N, K, bias=bias.data_ptr(), relu=1, out=out.view()),
        "fwd  A:K B:MN ": g(0, A.view(), 0, Wmn.view(), 1, M, N, K, bias=bias.data_ptr(), relu=1, out=out.view()),
        "gate A:K B:K  ": g(3, A.view(), 0, Wk.view(), 0, M, N, K, out=out.view(), gate=gate.view()),
        "store(N=1024) ": g(1, dz.view(), 0, Wmn.view(), 0, M, K, N, c=c.data_ptr(), ldc=K),
        "wgrad MN/MN   ": g(2, dz.view(), 1, A.view(), 1, N, K, M, c=ws.data_ptr(), ldc=K, splits=S),
    }
    for name, fn in cases.items():
        ms = timeit(fn)
        print(f"{prec} {name} {ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TFLOP/s")
