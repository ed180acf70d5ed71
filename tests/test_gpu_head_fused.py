"""The fused FC head (head_fused.cu: fc1 -> fc2 -> fc3 -> Huber -> head backward in one
cooperative launch) against the per-op path it replaces (tcgen05 GEMM launches + fc3 /
Huber / fc3-backward / colsum kernels), and against the fp64 oracle.

Both paths compute in bf16 with fp32 accumulation; they differ only in accumulation
order, so the comparison tolerance is a small multiple of bf16 rounding (stated per
check).  Dropout masks are drawn by the same counter hash, so train-mode steps compare
like for like."""

import numpy as np
import pytest
import torch

from oracle import dippm_oracle as O

pytestmark = pytest.mark.gpu

from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import Engine, Workspace, upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402

REL = 2e-2  # per-tensor ||a - b|| / ||b|| between the two bf16 paths


def _model(ds, hidden, seed=0, arch="sage"):
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    m = gnn.create_model(hidden=hidden, seed=seed, normalizer=norm) if arch == "sage" else \
        gnn.create_mlp_model(hidden=hidden, seed=seed, normalizer=norm)
    rng = np.random.default_rng(seed + 1)
    for _, arr in m.param_items():
        if arr.ndim == 1:
            arr[...] = rng.normal(0, 0.05, size=arr.shape)
    return m


def _step(model, b, fused, drop_p, arch="sage", seed=7):
    eng = Engine(model.hidden, "bf16", arch=arch)
    eng.fused_head = fused
    eng.set_params(model.param_items(), model.normalizer)
    ws = Workspace(eng, b.N, b.G, train=True)
    eng.grads.zero_()
    mode = 2 if drop_p > 0 else 0
    eng.forward(b, ws, mask_mode=mode, dropout_p=drop_p, seed=seed, predict=False, defer_head=True)
    eng.loss(b, ws, 1.0)
    eng.backward(b, ws, keep_scale=1.0 / (1.0 - drop_p))
    torch.cuda.synchronize()
    assert (ws.head_pending is None)
    return eng, ws


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("G,drop_p", [(256, 0.0), (200, 0.05), (37, 0.05)])
def test_fused_head_training_step_matches_per_op_path(G, drop_p):
    ds = make_dataset(G, seed=11)
    model = _model(ds, 512)
    b = upload_batch(*ds.collate(range(G)), device="cuda")
    e1, w1 = _step(model, b, True, drop_p)
    e0, w0 = _step(model, b, False, drop_p)
    assert e1.fused_head_ok(G) and not e0.fused_head_ok(G)
    l1, l0 = w1.loss.cpu().numpy(), w0.loss.cpu().numpy()
    assert abs(l1[0] - l0[0]) <= 1e-3 * abs(l0[0]) + 1e-6, (l1, l0)
    np.testing.assert_allclose(l1[1:], l0[1:], rtol=1e-2)
    # normalised outputs: bf16 head, same inputs
    np.testing.assert_allclose(w1.out[:G].cpu().numpy(), w0.out[:G].cpu().numpy(), rtol=0, atol=2e-2)
    g1, g0 = e1.get_grads(), e0.get_grads()
    for name in g0:
        assert _rel(g1[name], g0[name]) < REL, (name, _rel(g1[name], g0[name]))


def test_fused_head_deterministic_and_matches_oracle_gradients():
    """Two fused steps are bit-identical; the fused bf16 gradients agree with the fp64
    oracle (gnn.backward semantics) to bf16 accuracy."""
    G = 64
    ds = make_dataset(G, seed=5)
    model = _model(ds, 256, seed=3)
    b = upload_batch(*ds.collate(range(G)), device="cuda")
    ea, wa = _step(model, b, True, 0.0)
    eb, wb = _step(model, b, True, 0.0)
    for name, g in ea.get_grads().items():
        assert np.array_equal(g, eb.get_grads()[name]), name
    assert torch.equal(wa.loss, wb.loss)
    recs = ds.records(range(G))
    params = {k: np.array(v) for k, v in model.param_items()}
    n = model.normalizer
    norm = {"y_mean": n.y_mean, "y_std": n.y_std, "fs_mean": n.fs_mean, "fs_std": n.fs_std}
    orecs = [(r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector, r.target.as_array)
             for r in recs]
    ref_loss, ref = O.backward(params, norm, orecs)
    assert abs(float(wa.loss[0]) - ref_loss) <= 2e-2 * abs(ref_loss) + 1e-4
    got = ea.get_grads()
    for name in ("fc1.w", "fc1.b", "fc2.w", "fc2.b", "fc3.w", "fc3.b", "sage3.w_self", "sage1.w_neigh"):
        assert _rel(got[name], ref[name]) < 5e-2, (name, _rel(got[name], ref[name]))


def test_fused_head_forward_predict_and_mig():
    """predict path (no loss): y / MIG from the fused head vs the per-op head."""
    G = 300
    ds = make_dataset(G, seed=21)
    model = _model(ds, 512, seed=9)
    encs, fss = [r.encoding for r in ds.records(range(G))], [r.fs for r in ds.records(range(G))]
    eng = gnn._engine(model, "bf16")
    eng.fused_head = True
    y1, m1 = gnn.predict_batch(model, encs, fss, precision="bf16")
    eng.fused_head = False
    y0, m0 = gnn.predict_batch(model, encs, fss, precision="bf16")
    eng.fused_head = True
    np.testing.assert_allclose(y1, y0, rtol=2e-2, atol=1e-3 * np.abs(y0).max())
    assert (m1 == m0).mean() >= 0.98


def test_fused_head_mlp_arch_and_mixed_paths():
    """MLP baseline through the fused head (no readout below); and a non-deferred forward
    (fused forward) followed by the per-op loss/backward gives the same gradients."""
    G = 128
    ds = make_dataset(G, seed=4)
    mlp = _model(ds, 256, seed=2, arch="mlp")
    b = upload_batch(*ds.collate(range(G)), device="cuda", build_csr=False)
    e1, _ = _step(mlp, b, True, 0.05, arch="mlp")
    e0, _ = _step(mlp, b, False, 0.05, arch="mlp")
    g1, g0 = e1.get_grads(), e0.get_grads()
    for name in g0:
        assert _rel(g1[name], g0[name]) < REL, name
    # mixed: fused forward (not deferred) + per-op head backward
    model = _model(ds, 256, seed=6)
    bs = upload_batch(*ds.collate(range(G)), device="cuda")
    eng = Engine(256, "bf16")
    eng.set_params(model.param_items(), model.normalizer)
    ws = Workspace(eng, bs.N, bs.G, train=True)
    eng.grads.zero_()
    eng.forward(bs, ws, predict=False)          # fused forward only
    eng.loss(bs, ws, 1.0)                        # per-op Huber
    eng.backward(bs, ws)                         # per-op head backward
    gm = eng.get_grads()
    ed, _ = _step(model, bs, True, 0.0)
    gd = ed.get_grads()
    for name in gd:
        assert _rel(gm[name], gd[name]) < REL, name


def test_side_stream_weight_gradients_bit_identical():
    """The backward's weight-gradient GEMMs on a side stream (event fork/join) give exactly
    the gradients of the single-stream order (same kernels, no shared workspace races), eager
    and inside a captured CUDA graph."""
    G = 256
    ds = make_dataset(G, seed=17)
    model = _model(ds, 512, seed=8)
    b = upload_batch(*ds.collate(range(G)), device="cuda")
    grads = []
    for overlap in (False, True):
        eng = Engine(512, "bf16")
        eng.overlap_wgrad = overlap
        eng.set_params(model.param_items(), model.normalizer)
        ws = Workspace(eng, b.N, b.G, train=True)

        def step():
            eng.grads.zero_()
            eng.forward(b, ws, mask_mode=2, dropout_p=0.05, seed=5, predict=False, defer_head=True)
            eng.loss(b, ws, 1.0)
            eng.backward(b, ws, keep_scale=1 / 0.95)

        step()
        torch.cuda.synchronize()
        grads.append(eng.grads.clone())
        if overlap:  # the same step captured and replayed
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                step()  # warm the side stream inside a non-default stream first
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            g.replay()
            torch.cuda.synchronize()
            grads.append(eng.grads.clone())
    assert torch.equal(grads[0], grads[1])
    assert torch.equal(grads[0], grads[2])


def test_head_phase0_readout_combine_bit_identical(monkeypatch):
    """The optional phase 0 (u formed inside the fused head from the layer-3 block sums)
    reproduces dippm_pool_combine exactly: same u, same loss and gradients."""
    from paper_2303_11733_b200 import device as dev_mod
    G = 200
    ds = make_dataset(G, seed=19)
    model = _model(ds, 512, seed=12)
    b = upload_batch(*ds.collate(range(G)), device="cuda")
    res = []
    for flag in (False, True):
        monkeypatch.setattr(dev_mod, "HEAD_POOL", flag)
        eng, ws = _step(model, b, True, 0.05)
        res.append((ws.u.t[:G].clone(), ws.loss.clone(), eng.grads.clone()))
    for x, y in zip(res[0], res[1]):
        assert torch.equal(x, y)


@pytest.mark.parametrize("hidden,G", [(64, 5), (128, 33), (192, 70)])
def test_fused_head_small_shapes_match_per_op_path(hidden, G):
    """Narrow hidden widths (one or a few 32-column tiles, hp < 256 in the fc3 row pass) and
    tiny / ragged batches through the fused head."""
    ds = make_dataset(G, seed=29)
    model = _model(ds, hidden, seed=3)
    b = upload_batch(*ds.collate(range(G)), device="cuda")
    e1, w1 = _step(model, b, True, 0.05)
    e0, w0 = _step(model, b, False, 0.05)
    assert e1.fused_head_ok(G)
    np.testing.assert_allclose(w1.loss.cpu().numpy()[0], w0.loss.cpu().numpy()[0], rtol=2e-3)
    g1, g0 = e1.get_grads(), e0.get_grads()
    for name in g0:
        assert _rel(g1[name], g0[name]) < REL, (name, _rel(g1[name], g0[name]))


@pytest.mark.parametrize("G,drop_p", [(256, 0.05), (37, 0.0)])
def test_deferred_head_equals_in_kernel_head(monkeypatch, G, drop_p):
    """The training step's head (device.HEAD_WGRAD_DEFER): the column sums + loss in
    dippm_head_reduce, dW1 / dW2 as weight-gradient GEMMs on the side stream -- against the
    head doing all of it in-kernel.  The same device functions form the loss terms and the
    reductions, so the loss and every gradient except fc1.w / fc2.w are bit-identical; those
    two differ only in fp32 accumulation order."""
    from paper_2303_11733_b200 import device as dev_mod
    ds = make_dataset(G, seed=23)
    model = _model(ds, 512, seed=4)
    b = upload_batch(*ds.collate(range(G)), device="cuda")
    res = []
    for defer in (False, True):
        monkeypatch.setattr(dev_mod, "HEAD_WGRAD_DEFER", defer)
        eng, ws = _step(model, b, True, drop_p)
        res.append((ws.loss.clone(), eng.get_grads(), ws.du[:G].clone()))
    assert torch.equal(res[0][0], res[1][0])
    assert torch.equal(res[0][2], res[1][2])
    for name, g in res[0][1].items():
        if name in ("fc1.w", "fc2.w"):
            assert _rel(res[1][1][name], g) < 1e-5, name
        else:
            assert np.array_equal(res[1][1][name], g), name
