"""Kernel-level parity on the B200: K1 CSR bit-exact vs the reference's dense
aggregation pattern, K2 aggregation, K3 tensor-core GEMMs vs the SIMT fp32
anchor and fp64 numpy, K4 pooling, MIG codes."""

import numpy as np
import pytest
import torch

from conftest import unpack_records
from oracle import dippm_oracle as O

pytestmark = pytest.mark.gpu

from paper_2303_11733_b200 import _lib, device as dev  # noqa: E402
from paper_2303_11733_b200.device import ActBuf, upload_batch  # noqa: E402
from paper_2303_11733_b200.errors import ShapeMismatch  # noqa: E402


def _batch_from(recs):
    n = np.array([r[0] for r in recs])
    gp = np.zeros(len(recs) + 1, np.int32)
    np.cumsum(n, out=gp[1:])
    src, dst = [], []
    for g, r in enumerate(recs):
        e = np.asarray(r[1], np.int64).reshape(-1, 2)
        src.append(e[:, 0] + gp[g])
        dst.append(e[:, 1] + gp[g])
    x = np.concatenate([r[2] for r in recs]).astype(np.float32)
    fs = np.stack([r[3] for r in recs]).astype(np.float32)
    return upload_batch(x, np.concatenate(src), np.concatenate(dst), gp, fs)


def test_csr_bit_exact_vs_reference_pattern(golden):
    recs = unpack_records(golden)
    b = _batch_from(recs)
    rowptr, col, deg = b.rowptr.cpu().numpy(), b.col.cpu().numpy(), b.deg.cpu().numpy()
    inv = b.inv_deg.cpu().numpy()
    assert int(b.bad.item()) == 0
    gp = b.graph_ptr.cpu().numpy()
    rp_off = col_off = 0
    for i, r in enumerate(recs):
        n = r[0]
        g_rp = golden["csr_rowptr"][rp_off:rp_off + n + 1]
        g_col = golden["csr_col"][col_off:col_off + golden["csr_ncol"][i]]
        lo = gp[i]
        mine_rp = rowptr[lo:lo + n + 1] - rowptr[lo]
        mine_col = col[rowptr[lo]:rowptr[lo + n]] - lo
        assert np.array_equal(mine_rp, g_rp), i
        assert np.array_equal(mine_col, g_col), i
        assert np.array_equal(deg[lo:lo + n], golden["csr_deg"][lo:lo + n]), i
        rp_off += n + 1
        col_off += len(g_col)
    nz = deg > 0
    assert np.array_equal(inv[nz], (1.0 / deg[nz]).astype(np.float32))
    assert np.all(inv[~nz] == 0)
    # transposed CSR is the exact transpose of the pattern, dst ascending per src row
    t_rowptr, t_col = b.t_rowptr.cpu().numpy(), b.t_col.cpu().numpy()
    pairs = sorted((int(c), int(v)) for v in range(b.N) for c in col[rowptr[v]:rowptr[v + 1]])
    mine = [(u, int(t_col[j])) for u in range(b.N) for j in range(t_rowptr[u], t_rowptr[u + 1])]
    assert mine == pairs


def test_csr_deterministic_and_bad_edges():
    rng = np.random.default_rng(1)
    N, E = 5000, 40000
    src = rng.integers(0, N, E)
    dst = rng.integers(0, N, E)
    x = np.zeros((N, 32), np.float32)
    fs = np.zeros((1, 5), np.float32)
    gp = np.array([0, N], np.int32)
    a = upload_batch(x, src, dst, gp, fs)
    b = upload_batch(x, src, dst, gp, fs)
    nnz = int(a.rowptr[-1])  # col / t_col are capacity-E buffers: only the first nnz entries are defined
    for k in ("rowptr", "deg", "t_rowptr"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    for k in ("col", "t_col"):
        assert torch.equal(getattr(a, k)[:nnz], getattr(b, k)[:nnz]), k
    rowptr, col, deg = O.csr_of_aggregation(N, list(zip(src.tolist(), dst.tolist())))
    assert np.array_equal(a.rowptr.cpu().numpy(), rowptr)
    assert np.array_equal(a.col.cpu().numpy()[:len(col)], col)
    assert np.array_equal(a.deg.cpu().numpy(), deg)
    bad = upload_batch(x, np.array([0, N + 3]), np.array([1, 2]), gp, fs, validate=False)
    assert int(bad.bad.item()) == 1
    with pytest.raises(ShapeMismatch):  # the host validation rejects it before upload
        upload_batch(x, np.array([0, N + 3]), np.array([1, 2]), gp, fs)


@pytest.mark.parametrize("width", [24, 32, 48, 64, 96, 192, 384, 512, 768, 1024])
def test_aggregate_matches_dense(width):
    rng = np.random.default_rng(width)
    N = 777
    src = rng.integers(0, N, 2000)
    dst = rng.integers(0, N, 2000)
    b = upload_batch(np.zeros((N, 32), np.float32), src, dst, np.array([0, N], np.int32), np.zeros((1, 5), np.float32))
    h = rng.normal(size=(N, width)).astype(np.float32)
    ht = torch.from_numpy(h).cuda()
    m = torch.empty(N, width, device="cuda")
    s = torch.empty(N, width, device="cuda")
    _lib.call("dippm_sage_aggregate", dev.f32_act(ht), dev.f32_act(m), dev.f32_act(s), N, width,
              b.rowptr.data_ptr(), b.col.data_ptr(), b.inv_deg.data_ptr(), dev._stream())
    ref = O.aggregation_matrix(N, list(zip(src.tolist(), dst.tolist()))) @ h.astype(np.float64)
    assert np.allclose(m.cpu().numpy(), ref, rtol=1e-5, atol=1e-5)
    assert torch.equal(s, ht)
    # with and without the self copy: the same m, bit for bit
    m2 = torch.empty(N, width, device="cuda")
    _lib.call("dippm_sage_aggregate", dev.f32_act(ht), dev.f32_act(m2), dev.NULL_ACT, N, width,
              b.rowptr.data_ptr(), b.col.data_ptr(), b.inv_deg.data_ptr(), dev._stream())
    assert torch.equal(m, m2)


@pytest.mark.parametrize("width", [64, 192, 384, 512, 768, 1024])
def test_aggregate_t_with_fused_bias_reduce(width):
    """agg^T + the in-kernel bias-gradient reduction agree with fp64 numpy; counters end at zero."""
    rng = np.random.default_rng(width + 1)
    N = 1500
    src = rng.integers(0, N, 4000)
    dst = rng.integers(0, N, 4000)
    b = upload_batch(np.zeros((N, 32), np.float32), src, dst, np.array([0, N], np.int32), np.zeros((1, 5), np.float32))
    dz = rng.normal(size=(N, width)).astype(np.float32)
    B = torch.zeros(N, 2 * width, device="cuda")
    B[:, :width] = torch.from_numpy(dz).cuda()
    lib = _lib.load()
    part = torch.empty(lib.dippm_colsum_rows(N), width, device="cuda")
    sync = torch.zeros(lib.dippm_colsum_sync_ints(N), dtype=torch.int32, device="cuda")
    bias = torch.empty(width, device="cuda")
    _lib.call("dippm_sage_aggregate_t", dev.f32_act(B), width, N, 1, b.t_rowptr.data_ptr(), b.t_col.data_ptr(),
              b.inv_deg.data_ptr(), part.data_ptr(), bias.data_ptr(), sync.data_ptr(), dev._stream())
    agg = O.aggregation_matrix(N, list(zip(src.tolist(), dst.tolist())))
    assert np.allclose(B[:, width:].cpu().numpy(), agg.T @ dz.astype(np.float64), rtol=1e-5, atol=1e-5)
    assert np.allclose(bias.cpu().numpy(), dz.astype(np.float64).sum(0), rtol=1e-5, atol=1e-3)
    assert int(sync.abs().sum()) == 0


def _rand_act(rows, cols, dt, rng, scale=1.0):
    a = ActBuf(rows, cols, dt, "cuda")
    v = (rng.normal(size=(rows, cols)) * scale).astype(np.float32)
    t = torch.from_numpy(v).cuda()
    v64 = torch.from_numpy(v.astype(np.float64)).cuda()
    _lib.call("dippm_pack", v64.data_ptr(), rows, cols, 0, a.view(), dev._stream())
    return a, a.to_float().double().cpu().numpy(), t


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("M,N,K", [(300, 512, 64), (1000, 512, 1024), (129, 64, 64), (5000, 256, 512)])
def test_tc_gemm_fwd(prec, M, N, K):
    rng = np.random.default_rng(M + N + K)
    dt = dev.PRECISIONS[prec]
    A, a64, _ = _rand_act(M, K, dt, rng)
    B, b64, _ = _rand_act(N, K, dt, rng, 0.05)
    bias = torch.from_numpy(rng.normal(size=N).astype(np.float32)).cuda()
    ref = np.maximum(a64 @ b64.T + bias.double().cpu().numpy(), 0)
    for backend in (0, 1):
        out = ActBuf(M, N, dev.DT_F32, "cuda")
        out.t.fill_(float("nan"))
        args = _lib.GemmArgs(_lib.GEMM_FWD, M, N, K, A.view(), 0, B.view(), 0, bias.data_ptr(), 1, out.view(),
                             None, 0, 1)
        _lib.check(_lib.load().dippm_gemm(args, backend, dev._stream()))
        got = out.t.double().cpu().numpy()
        tol = 1e-5 * np.abs(ref).max()
        assert np.max(np.abs(got - ref)) <= tol, (backend, np.max(np.abs(got - ref)), tol)


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("M,N,K", [(300, 1024, 512), (77, 128, 64)])
def test_tc_gemm_store(prec, M, N, K):
    rng = np.random.default_rng(7 + M)
    dt = dev.PRECISIONS[prec]
    A, a64, _ = _rand_act(M, K, dt, rng)
    B, b64, _ = _rand_act(N, K, dt, rng)
    ref = a64 @ b64.T
    c = torch.full((M, N), float("nan"), device="cuda")
    args = _lib.GemmArgs(_lib.GEMM_STORE, M, N, K, A.view(), 0, B.view(), 0, None, 0, dev.NULL_ACT, c.data_ptr(), N, 1)
    _lib.check(_lib.load().dippm_gemm(args, 0, dev._stream()))
    assert np.max(np.abs(c.double().cpu().numpy() - ref)) <= 1e-5 * np.abs(ref).max()


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("R,M,N", [(3000, 512, 1024), (777, 64, 64), (20000, 512, 64)])
def test_tc_gemm_wgrad(prec, R, M, N):
    """C = dz^T @ A over R node rows, both operands MN-major, split-K + fixed-order reduce."""
    rng = np.random.default_rng(R)
    dt = dev.PRECISIONS[prec]
    dz, dz64, _ = _rand_act(R, M, dt, rng)
    A, a64, _ = _rand_act(R, N, dt, rng)
    ref = (a64.T @ dz64)  # [N, M] = dW layout
    lib = _lib.load()
    S = lib.dippm_wgrad_splits(M, N, R)
    ws = torch.full((S, M, N), float("nan"), device="cuda")
    out = torch.full((N, M), float("nan"), device="cuda")
    for backend in (0, 1):
        args = _lib.GemmArgs(_lib.GEMM_WGRAD, M, N, R, dz.view(), 1, A.view(), 1, None, 0, dev.NULL_ACT,
                             ws.data_ptr(), N, S)
        _lib.check(lib.dippm_gemm(args, backend, dev._stream()))
        _lib.call("dippm_splitk_reduce_t", ws.data_ptr(), S, M, N, 1.0, out.data_ptr(), M, dev._stream())
        err = np.max(np.abs(out.double().cpu().numpy() - ref))
        assert err <= 1e-5 * np.abs(ref).max(), (backend, err)


def test_pool_concat_and_mig_codes(golden):
    rng = np.random.default_rng(3)
    G = 37
    n = rng.integers(1, 50, G)
    gp = np.zeros(G + 1, np.int32)
    np.cumsum(n, out=gp[1:])
    h = rng.normal(size=(gp[-1], 64)).astype(np.float32)
    fs = rng.normal(size=(G, 5))
    norm = np.concatenate([np.zeros(6), rng.normal(size=5), rng.uniform(0.5, 2, 5)])
    u = torch.full((G, 128), float("nan"), device="cuda")
    keep = [torch.from_numpy(a).cuda() for a in (h, gp, fs, norm)]  # hold the buffers across the launch
    _lib.call("dippm_pool_concat", dev.f32_act(keep[0]), keep[1].data_ptr(), G, 64, keep[2].data_ptr(),
              keep[3].data_ptr(), dev.f32_act(u), dev._stream())
    got = u.cpu().numpy()
    for g in range(G):
        assert np.allclose(got[g, :64], h[gp[g]:gp[g + 1]].astype(np.float64).mean(0), atol=1e-6)
        assert np.allclose(got[g, 64:69], (fs[g] - norm[6:11]) / norm[11:16], atol=1e-6)
        assert np.all(got[g, 69:] == 0)
    alphas = torch.from_numpy(golden["mig_alpha"]).cuda()
    codes = torch.empty(len(alphas), dtype=torch.int8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("dippm_mig_codes", alphas.data_ptr(), 1, len(alphas), codes.data_ptr(), flag.data_ptr(), dev._stream())
    assert codes.cpu().numpy().tolist() == golden["mig_code"].tolist()
    assert int(flag.item()) == 0


@pytest.mark.parametrize("width", [24, 96, 192, 384, 768, 1024])
def test_pool_concat_widths(width):
    """Mean readout + static-feature columns at the three-chunk widths and 1024 (more dynamic
    shared memory than launches without the opt-in attribute)."""
    rng = np.random.default_rng(width)
    G = 9
    gp = np.zeros(G + 1, np.int32)
    np.cumsum(rng.integers(1, 300, G), out=gp[1:])
    h = rng.normal(size=(gp[-1], width)).astype(np.float32)
    fs = rng.normal(size=(G, 5))
    norm = np.concatenate([np.zeros(6), rng.normal(size=5), rng.uniform(0.5, 2, 5)])
    u = torch.full((G, width + 64), float("nan"), device="cuda")
    keep = [torch.from_numpy(a).cuda() for a in (h, gp, fs, norm)]
    _lib.call("dippm_pool_concat", dev.f32_act(keep[0]), keep[1].data_ptr(), G, width, keep[2].data_ptr(),
              keep[3].data_ptr(), dev.f32_act(u), dev._stream())
    got = u.cpu().numpy()
    for g in range(G):
        assert np.allclose(got[g, :width], h[gp[g]:gp[g + 1]].astype(np.float64).mean(0), atol=1e-5)
        assert np.allclose(got[g, width:width + 5], (fs[g] - norm[6:11]) / norm[11:16], atol=1e-6)
        assert np.all(got[g, width + 5:] == 0)


def _gemm(kind, M, N, K, a, a_mn, b, b_mn, backend=0, **kw):
    f = dict(bias=None, relu=0, out=dev.NULL_ACT, c=None, ldc=0, splits=1, gate=dev.NULL_ACT, gate_scale=1.0,
             drop_mode=0, mask=None, ldm=0, drop_p=0.0, seed=0, seed_dev=None, relu_bits=None, gate_bits=None,
             bits_ld=0, cta_pair=0, tile_sync=None, out_scale=1.0)
    f.update(kw)
    args = _lib.GemmArgs(kind, M, N, K, a, a_mn, b, b_mn, f["bias"], f["relu"], f["out"], f["c"], f["ldc"],
                         f["splits"], f["gate"], f["gate_scale"], f["drop_mode"], f["mask"], f["ldm"], f["drop_p"],
                         f["seed"], f["seed_dev"], f["relu_bits"], f["gate_bits"], f["bits_ld"], f["cta_pair"],
                         f["tile_sync"], f["out_scale"])
    _lib.check(_lib.load().dippm_gemm(args, backend, dev._stream()))


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("M,N,K", [(1000, 512, 1024), (256, 512, 576), (3, 64, 64)])
def test_fwd_mn_major_b_with_dropout(prec, M, N, K):
    """Forward GEMM reading W in its natural [K, N] layout (MN-major B) with the
    bias + ReLU + inverted-dropout epilogue; mode 2 writes the mask it used, mode 1
    re-applies a given mask; tensor-core and SIMT backends agree."""
    rng = np.random.default_rng(K + M)
    dt = dev.PRECISIONS[prec]
    A, a64, _ = _rand_act(M, K, dt, rng)
    W, w64, _ = _rand_act(K, N, dt, rng, 0.05)
    bias = torch.from_numpy(rng.normal(size=N).astype(np.float32)).cuda()
    ref = np.maximum(a64 @ w64 + bias.double().cpu().numpy(), 0)
    p = 0.3
    outs = {}
    for backend in (0, 1):
        out = ActBuf(M, N, dev.DT_F32, "cuda")
        mask = torch.full((M, N), -1.0, device="cuda")
        _gemm(_lib.GEMM_FWD, M, N, K, A.view(), 0, W.view(), 1, backend, bias=bias.data_ptr(), relu=1,
              out=out.view(), drop_mode=2, mask=mask.data_ptr(), ldm=N, drop_p=p, seed=1234)
        mk = mask.cpu().numpy()
        assert set(np.unique(mk)) <= {0.0, np.float32(1 / (1 - p))}
        assert abs((mk == 0).mean() - p) < 0.05 or M * N < 1000
        got = out.t.double().cpu().numpy()
        assert np.max(np.abs(got - ref * mk)) <= 1e-5 * np.abs(ref).max() / (1 - p)
        outs[backend] = mk
        # mode 1 reproduces the same result from the stored mask
        out2 = ActBuf(M, N, dev.DT_F32, "cuda")
        _gemm(_lib.GEMM_FWD, M, N, K, A.view(), 0, W.view(), 1, backend, bias=bias.data_ptr(), relu=1,
              out=out2.view(), drop_mode=1, mask=mask.data_ptr(), ldm=N)
        assert torch.equal(out.t, out2.t)
    assert np.array_equal(outs[0], outs[1])  # same counter-hash stream on both backends


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_gate_gemm(prec):
    """dgrad GEMM with the ReLU/dropout gate epilogue: out = (gate>0) * s * (A @ B^T)."""
    rng = np.random.default_rng(5)
    dt = dev.PRECISIONS[prec]
    M, N, K = 2000, 512, 1024
    A, a64, _ = _rand_act(M, K, dt, rng)
    B, b64, _ = _rand_act(N, K, dt, rng, 0.05)
    gate, g64, _ = _rand_act(M, N, dt, rng)
    ref = np.where(g64 > 0, 1.25 * (a64 @ b64.T), 0.0)
    for backend in (0, 1):
        out = ActBuf(M, N, dev.DT_F32, "cuda")
        _gemm(_lib.GEMM_GATE, M, N, K, A.view(), 0, B.view(), 0, backend, out=out.view(), gate=gate.view(),
              gate_scale=1.25)
        assert np.max(np.abs(out.t.double().cpu().numpy() - ref)) <= 1e-5 * np.abs(ref).max()


def test_aggregate_t_and_reduce_rows():
    """agg^T dz into the right half + column partial sums; reduce_rows is exact in fixed order."""
    rng = np.random.default_rng(9)
    N, W = 3000, 64
    src = rng.integers(0, N, 5000)
    dst = rng.integers(0, N, 5000)
    b = upload_batch(np.zeros((N, 32), np.float32), src, dst, np.array([0, N], np.int32),
                     np.zeros((1, 5), np.float32))
    dz = rng.normal(size=(N, W)).astype(np.float32)
    B = torch.zeros(N, 2 * W, device="cuda")
    B[:, :W] = torch.from_numpy(dz).cuda()
    lib = _lib.load()
    nblk = lib.dippm_colsum_blocks(N)
    part = torch.empty(lib.dippm_colsum_rows(N), W, device="cuda")
    sync = torch.zeros(lib.dippm_colsum_sync_ints(N), dtype=torch.int32, device="cuda")
    # caller-reduced partials (bias_grad NULL): exactly dippm_colsum_blocks(N) rows
    _lib.call("dippm_sage_aggregate_t", dev.f32_act(B), W, N, 1, b.t_rowptr.data_ptr(), b.t_col.data_ptr(),
              b.inv_deg.data_ptr(), part.data_ptr(), None, None, dev._stream())
    agg = O.aggregation_matrix(N, list(zip(src.tolist(), dst.tolist())))
    assert np.allclose(B[:, W:].cpu().numpy(), agg.T @ dz.astype(np.float64), rtol=1e-5, atol=1e-5)
    out = torch.empty(W, device="cuda")
    _lib.call("dippm_reduce_rows", part.data_ptr(), nblk, W, W, 1.0, out.data_ptr(), dev._stream())
    assert np.allclose(out.cpu().numpy(), dz.astype(np.float64).sum(0), rtol=1e-5, atol=1e-4)
    out2 = torch.empty(W, device="cuda")
    _lib.call("dippm_reduce_rows", part.data_ptr(), nblk, W, W, 1.0, out2.data_ptr(), dev._stream())
    assert torch.equal(out, out2)
    fused = torch.empty(W, device="cuda")  # in-kernel reduction (its own block partition)
    _lib.call("dippm_sage_aggregate_t", dev.f32_act(B), W, N, 1, b.t_rowptr.data_ptr(), b.t_col.data_ptr(),
              b.inv_deg.data_ptr(), part.data_ptr(), fused.data_ptr(), sync.data_ptr(), dev._stream())
    assert int(sync.abs().sum()) == 0
    assert np.allclose(fused.cpu().numpy(), dz.astype(np.float64).sum(0), rtol=1e-5, atol=1e-4)
    fused2 = torch.empty(W, device="cuda")  # replay: same bits, counters back at zero
    _lib.call("dippm_sage_aggregate_t", dev.f32_act(B), W, N, 0, b.t_rowptr.data_ptr(), b.t_col.data_ptr(),
              b.inv_deg.data_ptr(), part.data_ptr(), fused2.data_ptr(), sync.data_ptr(), dev._stream())
    assert torch.equal(fused, fused2) and int(sync.abs().sum()) == 0


def test_fc3_forward_backward():
    rng = np.random.default_rng(2)
    G, W = 300, 128
    x3 = np.maximum(rng.normal(size=(G, W)), 0).astype(np.float32)
    w3 = rng.normal(size=(W, 3)).astype(np.float32)
    b3 = rng.normal(size=3).astype(np.float32)
    d3 = rng.normal(size=(G, 3)).astype(np.float32)
    t = {k: torch.from_numpy(v).cuda() for k, v in dict(x3=x3, w3=w3, b3=b3, d3=d3).items()}
    out = torch.empty(G, 3, device="cuda")
    norm = torch.tensor([1.0, 2.0, 3.0, 2.0, 3.0, 4.0] + [0.0] * 10, dtype=torch.float64, device="cuda")
    y = torch.empty(G, 3, dtype=torch.float64, device="cuda")
    mig = torch.empty(G, dtype=torch.int8, device="cuda")
    nf = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("dippm_fc3_forward", dev.f32_act(t["x3"]), G, W, t["w3"].data_ptr(), t["b3"].data_ptr(),
              out.data_ptr(), norm.data_ptr(), y.data_ptr(), mig.data_ptr(), nf.data_ptr(), dev._stream())
    ref = x3.astype(np.float64) @ w3 + b3
    assert np.allclose(out.cpu().numpy(), ref, atol=1e-4)
    assert np.allclose(y.cpu().numpy(), ref * [2, 3, 4] + [1, 2, 3], atol=1e-3)
    gw3 = torch.empty(W, 3, device="cuda")
    gb3 = torch.empty(3, device="cuda")
    gb2 = torch.empty(W, device="cuda")
    d2 = torch.empty(G, W, device="cuda")
    _lib.call("dippm_fc3_backward", dev.f32_act(t["x3"]), G, W, t["w3"].data_ptr(), t["d3"].data_ptr(), 2.0,
              gw3.data_ptr(), gb3.data_ptr(), dev.f32_act(d2), gb2.data_ptr(), dev._stream())
    d2_ref = np.where(x3 > 0, 2.0 * (d3.astype(np.float64) @ w3.T), 0)
    assert np.allclose(gw3.cpu().numpy(), x3.T.astype(np.float64) @ d3, atol=1e-3)
    assert np.allclose(gb3.cpu().numpy(), d3.sum(0), atol=1e-4)
    assert np.allclose(d2.cpu().numpy(), d2_ref, atol=1e-4)
    assert np.allclose(gb2.cpu().numpy(), d2_ref.sum(0), atol=1e-3)


def _csr_arrays(b):
    return [getattr(b, k).cpu().numpy() for k in ("rowptr", "deg", "inv_deg", "t_rowptr")] + \
           [b.col.cpu().numpy()[:int(b.rowptr[-1])], b.t_col.cpu().numpy()[:int(b.t_rowptr[-1])]]


@pytest.mark.parametrize("case", ["golden", "synth", "dups", "many"])
def test_grouped_csr_equals_global_path(golden, case):
    """The per-graph shared-memory CSR kernel is bit-identical to the global path ("many":
    8000 graphs, far more CTAs than fit on the GPU at once, so the offsets come through long
    decoupled look-back chains across CTAs that start at different times; repeated 5 times)."""
    from paper_2303_11733_b200.device import build_batch_csr, group_edges
    from paper_2303_11733_b200.synth import make_dataset
    if case == "golden":
        b = _batch_from(unpack_records(golden))
    elif case == "synth":
        ds = make_dataset(300, seed=9, n_lo=2, power_law=1.5, n_max=3000)
        b = upload_batch(*ds.collate(np.arange(300)), build_csr=False)
    else:  # random multigraphs with duplicates and self loops, grouped per graph
        rng = np.random.default_rng(4)
        G = 50 if case == "dups" else 8000
        n = rng.integers(1, 400 if case == "dups" else 120, G)
        gp = np.zeros(G + 1, np.int32)
        np.cumsum(n, out=gp[1:])
        src, dst = [], []
        for g in range(G):
            e = rng.integers(0, n[g], (int(rng.integers(0, 3 * n[g])), 2))
            src.append(e[:, 0] + gp[g])
            dst.append(e[:, 1] + gp[g])
        b = upload_batch(np.zeros((gp[-1], 32), np.float32), np.concatenate(src), np.concatenate(dst), gp,
                         np.zeros((G, 5), np.float32), build_csr=False)
    assert b.edge_ptr is not None
    build_batch_csr(b, grouped=False)
    slow = _csr_arrays(b)
    for _ in range(5 if case == "many" else 1):
        build_batch_csr(b, grouped=True)
        assert int(b.bad.item()) == 0
        fast = _csr_arrays(b)
        for f, s in zip(fast, slow):
            assert np.array_equal(f, s)
    # an edge crossing graphs is rejected by the host validation ...
    with pytest.raises(ShapeMismatch):
        group_edges(np.array([0, 5]), np.array([1, 1]), np.array([0, 3, 6]))
    # ... and flagged by the grouped kernel when it reaches the device
    x = upload_batch(np.zeros((6, 32), np.float32), np.array([0, 4]), np.array([1, 1]), np.array([0, 3, 6], np.int32),
                     np.zeros((2, 5), np.float32), build_csr=False, edge_ptr=np.array([0, 2, 2]))
    build_batch_csr(x, grouped=True)
    assert int(x.bad.item()) == 1


def _bits_of(x):
    """[M, N] bool -> chunk-major [N/32, M] int32 words: bit c%32 of word (c/32, r)."""
    b = x.reshape(x.shape[0], -1, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)
    return np.ascontiguousarray(b.sum(-1).astype(np.uint32).view(np.int32).T)


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("M", [612, 3001, 20000])
def test_cta_pair_tiles_equal_single_cta(prec, M):
    """cta_group::2 256x256 tiles (incl. a last pair whose second CTA is wholly past M)
    give the same results as 1-CTA tiles for every GEMM kind; FWD's 1-bit ReLU mask
    equals (out > 0) and GATE on those bits equals GATE on the activation values."""
    rng = np.random.default_rng(M)
    dt = dev.PRECISIONS[prec]
    N, K = 512, 1024
    A, a64, _ = _rand_act(M, K, dt, rng)
    Wn, wn64, _ = _rand_act(K, N, dt, rng, 0.05)   # natural [K, N] weights: MN-major B
    Wk, wk64, _ = _rand_act(N, K, dt, rng, 0.05)   # [N, K]: K-major B
    bias = torch.from_numpy(rng.normal(size=N).astype(np.float32)).cuda()
    ref_fwd = np.maximum(a64 @ wn64 + bias.double().cpu().numpy(), 0)
    tol = 1e-5 * np.abs(ref_fwd).max()
    res = {}
    for pair in (1, 2):
        out = ActBuf(M, N, dt, "cuda")
        bits = torch.full((N // 32, M), -1, dtype=torch.int32, device="cuda")
        _gemm(_lib.GEMM_FWD, M, N, K, A.view(), 0, Wn.view(), 1, bias=bias.data_ptr(), relu=1, out=out.view(),
              relu_bits=bits.data_ptr(), bits_ld=M, cta_pair=pair)
        h = out.to_float().double().cpu().numpy()
        assert np.max(np.abs(h - ref_fwd)) <= (2e-2 if prec == "bf16" else 1e-5) * np.abs(ref_fwd).max()
        assert np.array_equal(bits.cpu().numpy(), _bits_of(h > 0)), pair
        # GATE: values vs bits
        g_val = ActBuf(M, N, dev.DT_F32, "cuda")
        g_bit = ActBuf(M, N, dev.DT_F32, "cuda")
        _gemm(_lib.GEMM_GATE, M, N, K, A.view(), 0, Wk.view(), 0, out=g_val.view(), gate=out.view(),
              gate_scale=1.5, cta_pair=pair)
        _gemm(_lib.GEMM_GATE, M, N, K, A.view(), 0, Wk.view(), 0, out=g_bit.view(), gate=dev.NULL_ACT,
              gate_scale=1.5, gate_bits=bits.data_ptr(), bits_ld=M, cta_pair=pair)
        assert torch.equal(g_val.t, g_bit.t)
        ref_gate = np.where(h > 0, 1.5 * (a64 @ wk64.T), 0.0)
        assert np.max(np.abs(g_val.t.double().cpu().numpy() - ref_gate)) <= 1e-5 * np.abs(ref_gate).max()
        # STORE
        c = torch.full((M, N), float("nan"), device="cuda")
        _gemm(_lib.GEMM_STORE, M, N, K, A.view(), 0, Wk.view(), 0, c=c.data_ptr(), ldc=N, cta_pair=pair)
        # WGRAD (MN-major both): C[N=512 features, K=1024] over M rows
        S = _lib.load().dippm_wgrad_splits(N, K, M)
        ws = torch.full((S, N, K), float("nan"), device="cuda")
        dz, dz64, _ = (out, h, None)
        _gemm(_lib.GEMM_WGRAD, N, K, M, dz.view(), 1, A.view(), 1, c=ws.data_ptr(), ldc=K, splits=S, cta_pair=pair)
        wg = torch.empty(K, N, device="cuda")
        _lib.call("dippm_splitk_reduce_t", ws.data_ptr(), S, N, K, 1.0, wg.data_ptr(), N, dev._stream())
        ref_w = a64.T @ h
        assert np.max(np.abs(wg.double().cpu().numpy() - ref_w)) <= 1e-5 * (np.abs(a64).T @ np.abs(h)).max()
        res[pair] = (out.t.clone(), g_val.t.clone(), c.clone(), wg.clone())
    for x1, x2 in zip(res[1], res[2]):  # same per-element k order: expected bit-identical
        x1, x2 = x1.double(), x2.double()
        assert torch.allclose(x1, x2, rtol=0, atol=1e-6 * float(x1.abs().max())), float((x1 - x2).abs().max())


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("R,M,N,splits", [(76800, 1024, 512, 0), (76800, 64, 512, 0), (3000, 576, 512, 0),
                                          (5000, 1024, 512, 1), (20000, 1024, 512, 20), (300, 512, 512, 3)])
def test_wgrad_fused_reduce(prec, R, M, N, splits):
    """WGRAD with the in-kernel split-K reduction (tile_sync): every reduce mode
    (slice-parallel, last-arriver, single split) equals the separate fixed-order
    reduce of the same partials bit for bit, and matches fp64; the counters are
    left zero (the launch can be replayed)."""
    rng = np.random.default_rng(R + M)
    dt = dev.PRECISIONS[prec]
    X, x64, _ = _rand_act(R, M, dt, rng)
    dz, dz64, _ = _rand_act(R, N, dt, rng)
    lib = _lib.load()
    S = splits or lib.dippm_wgrad_splits(M, N, R)
    sync = torch.zeros(lib.dippm_wgrad_sync_ints(M, N), dtype=torch.int32, device="cuda")
    ref = x64.T @ dz64
    scale_ref = (np.abs(x64).T @ np.abs(dz64)).max()
    for backend in (0, 1):
        ws = torch.full((S, M, N), float("nan"), device="cuda")
        out = torch.full((M, N), float("nan"), device="cuda")
        for rep in range(2):
            _gemm(_lib.GEMM_WGRAD, M, N, R, X.view(), 1, dz.view(), 1, backend, out=dev.f32_act(out),
                  c=ws.data_ptr(), ldc=N, splits=S, tile_sync=sync.data_ptr(), out_scale=0.5)
            assert int(sync.abs().sum()) == 0
        got = out.double().cpu().numpy()
        assert np.max(np.abs(got - 0.5 * ref)) <= 1e-5 * scale_ref, (backend, np.max(np.abs(got - 0.5 * ref)))
        if S > 1:
            sep = ws[0].double()
            for k in range(1, S):  # fp64 sum of the same partials in split order
                sep += ws[k].double()
            assert torch.equal(out, (sep * 0.5).float()), backend


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("W", [64, 512])
def test_readout_aggregate_t_bits_equal_values(prec, W):
    """Layer-3 readout backward + agg^T + bias grad: gating on the forward's 1-bit masks
    (chunk-major, and row-major with bits_ld 0) gives exactly what gating on the h3 values
    gives, and all match fp64 numpy.  W = 512 takes the bits kernel's fast path."""
    rng = np.random.default_rng(21)
    G = 9
    n = rng.integers(3, 40, G)
    gp = np.zeros(G + 1, np.int32)
    np.cumsum(n, out=gp[1:])
    N = int(gp[-1])
    src, dst = [], []
    for g in range(G):
        for v in range(gp[g] + 1, gp[g + 1]):
            src.append(v - 1)
            dst.append(v)
            if v - gp[g] > 2:
                src.append(int(rng.integers(gp[g], v - 1)))
                dst.append(v)
    src, dst = np.array(src), np.array(dst)
    b = upload_batch(np.zeros((N, 32), np.float32), src, dst, gp, np.zeros((G, 5), np.float32))
    dt = dev.PRECISIONS[prec]
    h3, h64, _ = _rand_act(N, W, dt, rng)
    bits_np = _bits_of(h64 > 0)
    bits = torch.from_numpy(bits_np).cuda()
    bits_rm = torch.from_numpy(np.ascontiguousarray(bits_np.T)).cuda()  # [N, W/32] row-major
    du = torch.from_numpy(rng.normal(size=(G, W)).astype(np.float32)).cuda()
    lib = _lib.load()
    outs = []
    for use_bits in (0, 1, 2):  # values, chunk-major bits, row-major bits
        B = ActBuf(N, 2 * W, dt, "cuda")
        part = torch.empty(lib.dippm_colsum_rows(N), W, device="cuda")
        sync = torch.zeros(lib.dippm_colsum_sync_ints(N), dtype=torch.int32, device="cuda")
        bias = torch.empty(W, device="cuda")
        _lib.call("dippm_readout_aggregate_t", du.data_ptr(), W, b.graph_ptr.data_ptr(), b.node_graph.data_ptr(),
                  h3.view(), B.view(), W, N, b.t_rowptr.data_ptr(), b.t_col.data_ptr(), b.inv_deg.data_ptr(),
                  part.data_ptr(), bias.data_ptr(), sync.data_ptr(),
                  None if use_bits == 0 else (bits if use_bits == 1 else bits_rm).data_ptr(),
                  N if use_bits == 1 else 0, dev._stream())
        outs.append((B.to_float().clone(), bias.clone()))
    # the two bit layouts run the same arithmetic: identical
    assert torch.equal(outs[1][0], outs[2][0]) and torch.equal(outs[1][1], outs[2][1])
    if W < 256:  # generic kernel: bits and values gate the same terms in the same order
        assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    # (W = 512: the bits kernel factorises agg^T dz3 = dr * sum bit/deg -- checked against fp64 below)
    # fp64 reference: dz3[v] = du[g(v)] / N_g * (h3 > 0); agg^T dz3; bias = sum dz3
    gid = np.repeat(np.arange(G), n)
    dz = du.double().cpu().numpy()[gid] / n[gid][:, None] * (h64 > 0)
    agg = O.aggregation_matrix(N, list(zip(src.tolist(), dst.tolist())))
    tol = 2e-2 if prec == "bf16" else 1e-5
    for k in (0, 1):
        got = outs[k][0].double().cpu().numpy()
        assert np.allclose(got[:, :W], dz, atol=tol * np.abs(dz).max())
        assert np.allclose(got[:, W:], agg.T @ dz, atol=tol * np.abs(dz).max())
        assert np.allclose(outs[k][1].double().cpu().numpy(), dz.sum(0), atol=tol * np.abs(dz).sum(0).max())


@pytest.mark.parametrize("W", [256, 512, 1024])
def test_readout_bits_row_major_far_and_dense(W):
    """The training layout's readout kernel (bf16, row-major bits) on graphs that leave its fast
    paths: out-neighbours far beyond the staged halo (global bit reads), nodes with dozens of
    out-edges (blocks whose CSR slice exceeds the shared-memory stage), rows with zero, one and
    many out-edges -- dz3, agg^T dz3 and the bias gradient against fp64, and dz3 / agg^T dz3
    bit-identical to the layout-generic kernel on the chunk-major copy of the same masks."""
    rng = np.random.default_rng(W)
    n = np.array([5, 3000, 700, 1, 2500])
    G = len(n)
    gp = np.zeros(G + 1, np.int32)
    np.cumsum(n, out=gp[1:])
    N = int(gp[-1])
    src, dst = [], []
    for g in range(G):
        lo, hi = int(gp[g]), int(gp[g + 1])
        for v in range(lo + 1, hi):
            src.append(v - 1)
            dst.append(v)                                   # chain: one out-edge
            if v % 7 == 0:
                src.append(int(rng.integers(lo, v)))        # far back-reference (forward of u: far ahead)
                dst.append(v)
        if hi - lo > 100:
            for u in range(lo, lo + 120):                   # hub rows: ~40 out-edges each
                for v in rng.choice(np.arange(u + 1, hi), size=40, replace=False):
                    src.append(u)
                    dst.append(int(v))
    src, dst = np.array(src), np.array(dst)
    b = upload_batch(np.zeros((N, 32), np.float32), src, dst, gp, np.zeros((G, 5), np.float32))
    h3, h64, _ = _rand_act(N, W, dev.DT_BF16, rng)
    bits_np = _bits_of(h64 > 0)
    du = torch.from_numpy(rng.normal(size=(G, W)).astype(np.float32)).cuda()
    lib = _lib.load()
    outs = []
    for layout in ("chunk", "row"):
        bits = torch.from_numpy(bits_np if layout == "chunk" else np.ascontiguousarray(bits_np.T)).cuda()
        B = ActBuf(N, 2 * W, dev.DT_BF16, "cuda")
        part = torch.empty(lib.dippm_colsum_rows(N), W, device="cuda")
        sync = torch.zeros(lib.dippm_colsum_sync_ints(N), dtype=torch.int32, device="cuda")
        bias = torch.empty(W, device="cuda")
        _lib.call("dippm_readout_aggregate_t", du.data_ptr(), W, b.graph_ptr.data_ptr(), b.node_graph.data_ptr(),
                  h3.view(), B.view(), W, N, b.t_rowptr.data_ptr(), b.t_col.data_ptr(), b.inv_deg.data_ptr(),
                  part.data_ptr(), bias.data_ptr(), sync.data_ptr(), bits.data_ptr(), N if layout == "chunk" else 0,
                  dev._stream())
        outs.append((B.to_float().clone(), bias.clone()))
    assert torch.equal(outs[0][0], outs[1][0])
    # (the two kernels size their blocks differently, so the bias partial sums group differently)
    assert torch.allclose(outs[0][1], outs[1][1], rtol=1e-5, atol=1e-6)
    gid = np.repeat(np.arange(G), n)
    dz = du.double().cpu().numpy()[gid] / n[gid][:, None] * (h64 > 0)
    deg = np.zeros(N)
    pairs = np.unique(np.stack([dst, src], 1), axis=0)  # distinct (dst, src): the CSR pattern
    np.add.at(deg, dst, 1)                              # in-degree counts duplicates (gnn.py:136)
    aggt = np.zeros_like(dz)
    np.add.at(aggt, pairs[:, 1], dz[pairs[:, 0]] / deg[pairs[:, 0], None])
    got = outs[1][0].double().cpu().numpy()
    scale = np.abs(dz).max()
    assert np.allclose(got[:, :W], dz, atol=1e-2 * scale, rtol=1e-2)
    assert np.allclose(got[:, W:], aggt, atol=2e-2 * scale, rtol=2e-2)
    assert np.allclose(outs[1][1].double().cpu().numpy(), dz.sum(0), atol=1e-4 * np.abs(dz).sum(0).max())


@pytest.mark.parametrize("M,N", [(76800, 512), (3001, 256), (5, 512), (129, 512)])
def test_shortk_forward_equals_general_kernel(M, N):
    """The dedicated K = 64 forward (layer 1: 16 epilogue warps, resident W1) gives bit-identical
    activations and 1-bit masks to the general tcgen05 kernel (forced with cta_pair=1), and both
    match fp64 within the bf16 tolerance; rows past M are never written."""
    rng = np.random.default_rng(M + N)
    K = 64
    A, a64, _ = _rand_act(M, K, dev.DT_BF16, rng)
    W, w64, _ = _rand_act(K, N, dev.DT_BF16, rng, 0.1)
    bias = torch.from_numpy(rng.normal(scale=0.2, size=N).astype(np.float32)).cuda()
    ref = np.maximum(a64 @ w64 + bias.double().cpu().numpy(), 0)
    res = {}
    for pair in (0, 1):
        out = ActBuf(M + 3, 2 * N, dev.DT_BF16, "cuda")  # write the left half of a wider buffer, like A2
        out.t.fill_(7.0)
        bits = torch.full((N // 32, M + 3), -1, dtype=torch.int32, device="cuda")
        _gemm(_lib.GEMM_FWD, M, N, K, A.view(), 0, W.view(), 1, bias=bias.data_ptr(), relu=1,
              out=_lib.Act(out.t.data_ptr(), 2 * N, 0, dev.DT_BF16), relu_bits=bits.data_ptr(), bits_ld=M + 3,
              cta_pair=pair)
        h = out.t[:M, :N].double().cpu().numpy()
        assert np.max(np.abs(h - ref)) <= 2e-2 * np.abs(ref).max()
        assert np.array_equal(bits[:, :M].cpu().numpy(), _bits_of(h > 0))
        assert bool((out.t[M:, :] == 7.0).all()) and bool((out.t[:, N:] == 7.0).all())
        assert bool((bits[:, M:] == -1).all())
        res[pair] = (out.t.clone(), bits.clone())
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
