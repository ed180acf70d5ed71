"""Parity AT the headline configuration the bench times (BASELINE.json configs[1]):
hidden 512, 256-graph batches of ~300-node graphs, through the same BatchTrainer /
Engine code path `bench.py` runs (bf16 with the fused head; the fp32 mode beside it).

Stated tolerances:
  fp32 mode   every gradient tensor ||d|| <= 1e-4 ||g|| + 1e-6 sqrt(n); loss rel 1e-5;
              normalised outputs |d| <= 2e-5 max(1, |ref|) (measured 1.0e-5 relative here:
              the tensor cores' tf32 accumulation over K = 1024 at hidden 512)
  bf16 mode   every gradient tensor ||d|| <= 3e-2 ||g||; loss rel 1e-2;
              normalised outputs |d| <= 2e-2
against the fp64 oracle (oracle/dippm_oracle.py, pinned to the reference's goldens).
"""

import math

import numpy as np
import pytest

from oracle import dippm_oracle as O

pytestmark = pytest.mark.gpu

from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import Workspace, upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402

G, HIDDEN = 256, 512
BF16_GRAD_REL, BF16_LOSS_REL, BF16_OUT_ABS = 3e-2, 1e-2, 2e-2
FP32_GRAD_REL, FP32_GRAD_ABS, FP32_OUT_ABS = 1e-4, 1e-6, 2e-5


def _rel(got, ref):
    return np.linalg.norm(np.asarray(got) - ref) / max(np.linalg.norm(ref), 1e-30)


@pytest.fixture(scope="module")
def headline():
    """configs[1] batch: 256 graphs, N ~ U[270, 330], a model with random biases so every
    ReLU pattern is non-trivial, and the fp64 oracle's loss + 15 gradients over the batch."""
    ds = make_dataset(G, seed=1)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=HIDDEN, seed=0, normalizer=norm)
    rng = np.random.default_rng(1)
    for _, arr in model.param_items():
        if arr.ndim == 1:
            arr[...] = rng.normal(0, 0.05, size=arr.shape)
    recs = ds.records(range(G))
    params = {k: np.array(v) for k, v in model.param_items()}
    nd = {"y_mean": norm.y_mean, "y_std": norm.y_std, "fs_mean": norm.fs_mean, "fs_std": norm.fs_std}
    orecs = [(r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector, r.target.as_array)
             for r in recs]
    ref_loss, ref_grads = O.backward(params, nd, orecs)
    return ds, recs, model, params, nd, orecs, ref_loss, ref_grads


def _trainer_step(ds, model, precision):
    """One BatchTrainer step exactly as bench.py runs it (resident batch, CSR rebuilt in the
    step, deferred fused head in bf16), dropout off; returns (loss, grads, engine)."""
    tr = BatchTrainer(model, precision=precision, lr=1e-3, dropout=False)
    b = upload_batch(*ds.collate(np.arange(G)), device="cuda", build_csr=False)
    tr.step_resident(b)
    return float(tr.ws.loss[0]), tr.engine.get_grads(), tr.engine


def test_headline_bf16_step_all_gradients_vs_oracle(headline):
    ds, _, model, _, _, _, ref_loss, ref_grads = headline
    loss, grads, eng = _trainer_step(ds, model, "bf16")
    assert eng.fused_head_ok(G)  # the benched path: the whole FC head in one launch
    assert abs(loss - ref_loss) <= BF16_LOSS_REL * abs(ref_loss), (loss, ref_loss)
    assert sorted(grads) == sorted(ref_grads) and len(grads) == 15
    errs = {k: _rel(grads[k], g) for k, g in ref_grads.items()}
    print("bf16 headline gradient rel errors:", {k: f"{v:.2e}" for k, v in errs.items()})
    for k, e in errs.items():
        assert e <= BF16_GRAD_REL, (k, e)


def test_headline_fp32_step_all_gradients_vs_oracle(headline):
    ds, _, model, _, _, _, ref_loss, ref_grads = headline
    loss, grads, _ = _trainer_step(ds, model, "fp32")
    assert loss == pytest.approx(ref_loss, rel=1e-5)
    for k, g in ref_grads.items():
        d = np.linalg.norm(grads[k] - g)
        assert d <= FP32_GRAD_REL * np.linalg.norm(g) + FP32_GRAD_ABS * math.sqrt(g.size), (k, d)


def test_headline_bf16_dropout_step_vs_oracle(headline):
    """Train-mode dropout at the headline config: host masks (mask_mode 1, the reference's
    per-graph fc1/fc2 masks) through the fused head, against the oracle's train-mode
    forward + backward per graph with the same masks (the batch objective, gnn.py:383-405)."""
    ds, recs, model, params, nd, orecs, _, _ = headline
    p = 0.05
    eng = gnn._engine(model, "bf16")
    b = upload_batch(*ds.collate(np.arange(G)), device="cuda")
    ws = Workspace(eng, b.N, G, train=True)
    rng = np.random.default_rng(9)
    masks = (rng.random((2, G, HIDDEN)) >= p) / (1.0 - p)
    import torch
    ws.masks[:, :, :HIDDEN].copy_(torch.from_numpy(masks.astype(np.float32)))
    eng.forward(b, ws, mask_mode=1, predict=False, defer_head=True)
    eng.loss(b, ws)
    eng.backward(b, ws, keep_scale=1.0 / (1.0 - p))
    loss, grads = float(ws.loss[0]), eng.get_grads()
    ref = {k: np.zeros_like(v) for k, v in params.items()}
    ref_loss = 0.0
    for g, (n, edges, x, fs_raw, y_raw) in enumerate(orecs):
        agg = O.aggregation_matrix(n, edges)
        fs_norm = (fs_raw - nd["fs_mean"]) / nd["fs_std"]
        out, cache = O.forward_norm(params, x, agg, fs_norm, masks=(masks[0, g], masks[1, g]))
        lg, dout = O.huber_loss(out, (y_raw - nd["y_mean"]) / nd["y_std"])
        ref_loss += lg / G
        for k, v in O.backward_from(params, cache, dout, HIDDEN).items():
            ref[k] += v / G
    assert abs(loss - ref_loss) <= BF16_LOSS_REL * abs(ref_loss), (loss, ref_loss)
    for k, g in ref.items():
        assert _rel(grads[k], g) <= BF16_GRAD_REL, (k, _rel(grads[k], g))


def test_headline_all_256_graphs_predict_vs_oracle(headline):
    """Every graph of the configs[1] batch (not a sample): fp32 within 1e-5 normalised,
    bf16 within 2e-2 normalised, of the oracle's predictions."""
    _, recs, model, params, nd, orecs, _, _ = headline
    ref = np.stack([O.predict(params, nd, *r[:4]) for r in orecs])
    ys = nd["y_std"]
    y32, _ = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs], precision="fp32")
    d32 = np.abs((y32 - ref) / ys)
    assert np.all(d32 <= FP32_OUT_ABS * np.maximum(1.0, np.abs(ref / ys))), d32.max()
    y16, _ = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs], precision="bf16")
    d16 = np.abs((y16 - ref) / ys)
    print(f"all-256 normalised |d|: fp32 max {d32.max():.2e}, bf16 max {d16.max():.2e}")
    assert d16.max() <= BF16_OUT_ABS


def test_three_adam_steps_vs_oracle(headline):
    """Three fp32 BatchTrainer steps on different 64-graph batches.  At every step the
    device gradients equal the oracle's gradients AT THE DEVICE'S CURRENT PARAMETERS
    (gnn.backward), and the device's Adam update equals the reference adam_step chain
    (moments carried over three steps, so m / sqrt(v) depends on every gradient's
    magnitude) applied to those same gradients.  (Comparing against an independent oracle
    trajectory is ill-posed: the first Adam step moves each coordinate by ~lr sign(g), so
    coordinates with |g| ~ 0 may legitimately step in opposite directions.)"""
    ds, recs, model, _, nd, orecs, _, _ = headline
    lr = 1e-3
    tr = BatchTrainer(model, precision="fp32", lr=lr, dropout=False)
    m = v = None
    for t, sl in enumerate((slice(0, 64), slice(64, 128), slice(128, 192)), start=1):
        idx = np.arange(G)[sl]
        before = tr.engine.get_params()
        tr.step_resident(upload_batch(*ds.collate(idx), device="cuda", build_csr=False))
        _, grads = O.backward(before, nd, [orecs[i] for i in idx])
        got_g = tr.engine.get_grads()
        for k, g in grads.items():
            d = np.linalg.norm(got_g[k] - g)
            assert d <= FP32_GRAD_REL * np.linalg.norm(g) + FP32_GRAD_ABS * math.sqrt(g.size), (t, k, d)
        if m is None:
            m = {k: np.zeros_like(x) for k, x in before.items()}
            v = {k: np.zeros_like(x) for k, x in before.items()}
        after = tr.engine.get_params()
        for k in before:
            ref = O.adam_step(before[k], got_g[k], m[k], v[k], t, lr=lr)
            assert np.allclose(after[k], ref, rtol=1e-12, atol=1e-15), (t, k, np.abs(after[k] - ref).max())
