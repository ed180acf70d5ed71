"""The tensor-core FC head (head_tc.cu: one cluster of 8 CTAs, tcgen05 + TMA + TMEM) against the
mma.sync head (head_fused.cu) on the configs[1] head shape -- the same forward, Huber loss and
head backward to bf16 accuracy (different accumulation orders), bit-reproducible run to run,
dropout masks identical (same counter hash) -- and against the fp64 oracle via the headline
tests, whose bf16 step now runs it."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2303_11733_b200 import _lib, gnn  # noqa: E402
from paper_2303_11733_b200.device import Engine, Workspace, upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402


def _model(ds, hidden, seed):
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    m = gnn.create_model(hidden=hidden, seed=seed, normalizer=norm)
    rng = np.random.default_rng(seed + 1)
    for _, arr in m.param_items():
        if arr.ndim == 1:
            arr[...] = rng.normal(0, 0.05, size=arr.shape)
    return m


def _step(model, b, tc, drop_p):
    lib = _lib.load()
    was = lib.dippm_head_tc_enable(1 if tc else 0)
    try:
        eng = Engine(512, "bf16")
        eng.set_params(model.param_items(), model.normalizer)
        ws = Workspace(eng, b.N, b.G, train=True)
        eng.grads.zero_()
        eng.forward(b, ws, mask_mode=2 if drop_p else 0, dropout_p=drop_p, seed=11, predict=False, defer_head=True)
        eng.loss(b, ws, 1.0)
        eng.backward(b, ws, keep_scale=1.0 / (1.0 - drop_p))
        torch.cuda.synchronize()
        return eng, ws
    finally:
        lib.dippm_head_tc_enable(was)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("G,drop_p", [(256, 0.0), (256, 0.05), (200, 0.05), (7, 0.0), (129, 0.05)])
def test_tensor_core_head_matches_mma_sync_head(G, drop_p):
    ds = make_dataset(G, seed=40 + G)
    model = _model(ds, 512, seed=G)
    b = upload_batch(*ds.collate(range(G)), device="cuda")
    e1, w1 = _step(model, b, True, drop_p)
    e0, w0 = _step(model, b, False, drop_p)
    # the forward activations: bf16 operands, fp32 accumulation in a different order
    for name in ("x2", "x3"):
        x1, x0 = getattr(w1, name).t[:G].float(), getattr(w0, name).t[:G].float()
        assert torch.allclose(x1, x0, rtol=2e-2, atol=2e-2 * float(x0.abs().max())), name
        # dropout: the same counter-hash draws (a dropped unit is exactly zero in both)
        if drop_p:
            assert float(((x1 == 0) != (x0 == 0)).float().mean()) < 2e-3, name
    np.testing.assert_allclose(w1.out[:G].cpu().numpy(), w0.out[:G].cpu().numpy(), rtol=0, atol=2e-2)
    l1, l0 = w1.loss.cpu().numpy(), w0.loss.cpu().numpy()
    assert abs(l1[0] - l0[0]) <= 1e-3 * abs(l0[0]) + 1e-6, (l1, l0)
    np.testing.assert_allclose(l1[1:], l0[1:], rtol=1e-2)
    # (norm-relative: a pre-activation within rounding of 0 may take the other side of a ReLU in
    # the other accumulation order, which changes that row's d2 / d1 / du entries wholesale)
    assert _rel(w1.du[:G].cpu().numpy(), w0.du[:G].cpu().numpy()) < 3e-2
    g1, g0 = e1.get_grads(), e0.get_grads()
    for name in g0:
        assert _rel(g1[name], g0[name]) < 3e-2, (name, _rel(g1[name], g0[name]))
    assert int(e1.t_dev.item()) == int(e0.t_dev.item())


def test_tensor_core_head_deterministic():
    G = 256
    ds = make_dataset(G, seed=3)
    model = _model(ds, 512, seed=5)
    b = upload_batch(*ds.collate(range(G)), device="cuda")
    ea, wa = _step(model, b, True, 0.05)
    eb, wb = _step(model, b, True, 0.05)
    assert torch.equal(ea.grads, eb.grads) and torch.equal(wa.loss, wb.loss) and torch.equal(wa.du, wb.du)
