"""The drop-in surface on the device, exercised the way the reference's callers use it.

* The reference's own known answers for sage_forward / readout_mean / forward
  (pkg/tests/test_gnn.py:36-122), with golden records in place of `synth_dataset`.
  Where the reference compares fp64 values with array_equal, the stated fp32 tolerance
  applies unless the value is exactly representable on the device path.
* sage_forward / readout_mean at widths the kernels do not take natively (24, 96, 200,
  1000, 1500: padded to power-of-two or 1024-column chunks) against the oracle.
* The duck-typed model protocol `_fit` is generic over (gnn.py:212-262, 424-482):
  `_prepare_record`, `forward_norm(prep, fs_norm, train, rng)`, `backward_from(cache,
  dout)` for DippmModel and MlpModel, against the oracle, and a literal replay of the
  reference `_fit` loop written against that protocol (with this package's
  numerics.huber_loss / adam_step) reproducing the reference's golden training run.
"""

import math

import numpy as np
import pytest

from conftest import unpack_records
from oracle import dippm_oracle as O

pytestmark = pytest.mark.gpu

from paper_2303_11733_b200 import gnn, numerics  # noqa: E402
from paper_2303_11733_b200.errors import EmptyGraph, ShapeMismatch  # noqa: E402
from paper_2303_11733_b200.gnn import Normalizer, SageLayerParams  # noqa: E402
from paper_2303_11733_b200.types import DatasetRecord, GraphEncoding, TargetVector  # noqa: E402

FP32_ABS = 1e-5


class _FS:
    def __init__(self, v):
        self.as_vector = np.asarray(v)


def _records(g, prefix="rec_"):
    return [DatasetRecord(GraphEncoding(n, e, x), _FS(fs), TargetVector(*y)) for n, e, x, fs, y in
            unpack_records(g, prefix)]


def _fitted_model(records, hidden=8, seed=0):
    targets = np.stack([r.target.as_array for r in records])
    statics = np.stack([r.fs.as_vector for r in records])
    return gnn.create_model(hidden=hidden, seed=seed, normalizer=Normalizer.fit(targets, statics))


def _norm_dict(n):
    return {"y_mean": n.y_mean, "y_std": n.y_std, "fs_mean": n.fs_mean, "fs_std": n.fs_std}


# -- T/test_gnn.py:36-59 sage_forward ---------------------------------------------------


def test_sage_forward_ignores_edges_when_neighbor_weights_zero():
    feats = np.random.default_rng(0).normal(size=(3, 4))
    enc = GraphEncoding(3, [(0, 1), (1, 2)], feats)
    layer = SageLayerParams(w_self=np.eye(4), w_neigh=np.zeros((4, 4)), bias=np.zeros(4))
    out = gnn.sage_forward(enc, layer, enc.features)
    no_edges = gnn.sage_forward(GraphEncoding(3, [], enc.features), layer, enc.features)
    assert np.allclose(out, np.maximum(enc.features, 0.0), rtol=0, atol=FP32_ABS)
    assert np.array_equal(out, no_edges)  # zero neighbour weights contribute exactly nothing


def test_sage_forward_single_neighbor_mean_is_exact():
    feats = np.array([[1.0, -2.0], [0.5, 3.0]])
    enc = GraphEncoding(2, [(0, 1)], feats)
    layer = SageLayerParams(w_self=np.zeros((2, 2)), w_neigh=np.eye(2), bias=np.zeros(2))
    out = gnn.sage_forward(enc, layer, feats)
    assert np.array_equal(out[1], np.maximum(feats[0], 0.0))  # exactly representable: bit-exact
    assert np.array_equal(out[0], np.zeros(2))


def test_sage_forward_two_neighbor_mean():
    feats = np.array([[2.0, 0.0], [4.0, 2.0], [0.0, 0.0]])
    layer = SageLayerParams(w_self=np.zeros((2, 2)), w_neigh=np.eye(2), bias=np.zeros(2))
    out = gnn.sage_forward(GraphEncoding(3, [(0, 2), (1, 2)], feats), layer, feats)
    assert np.allclose(out[2], [3.0, 1.0])


# -- T/test_gnn.py:62-84 readout ---------------------------------------------------------


def test_readout_single_node_identity():
    z = np.array([[1.0, -2.0, 3.0]])
    assert np.array_equal(gnn.readout_mean(z), z[0])


def test_readout_symmetric_rows_cancel():
    e = np.array([1.0, -4.0, 2.0])
    assert np.allclose(gnn.readout_mean(np.stack([e, -e])), np.zeros(3))


def test_readout_order_invariant():
    rng = np.random.default_rng(3)
    z = rng.normal(size=(6, 5))
    assert np.allclose(gnn.readout_mean(z), gnn.readout_mean(z[rng.permutation(6)]))


def test_readout_empty_raises():
    with pytest.raises(EmptyGraph):
        gnn.readout_mean(np.zeros((0, 4)))


# -- T/test_gnn.py:90-122 forward ----------------------------------------------------------


def test_forward_zero_weights_returns_final_bias(golden):
    recs = _records(golden)[:3]
    model = _fitted_model(recs)
    for _, arr in model.param_items():
        arr[...] = 0.0
    model.fc[2].b[...] = np.array([1.5, -0.5, 2.0])
    for rec in recs:
        assert np.array_equal(gnn.forward(rec.encoding, rec.fs, model), [1.5, -0.5, 2.0])


def test_forward_eval_is_bit_identical(golden):
    recs = _records(golden)[:2]
    model = _fitted_model(recs, seed=9)
    a = gnn.forward(recs[0].encoding, recs[0].fs, model)
    b = gnn.forward(recs[0].encoding, recs[0].fs, model)
    assert np.array_equal(a, b)


def test_forward_rejects_bad_mode(golden):
    recs = _records(golden)[:1]
    model = _fitted_model(recs)
    with pytest.raises(ValueError):
        gnn.forward(recs[0].encoding, recs[0].fs, model, mode="predict")


def test_forward_isolated_nodes_finite(golden):
    rng = np.random.default_rng(0)
    enc = GraphEncoding(4, [], np.abs(rng.normal(size=(4, 32))))
    recs = _records(golden)[:2]
    model = _fitted_model(recs)
    assert np.all(np.isfinite(gnn.forward(enc, recs[0].fs, model)))


# -- widths the kernels do not take natively -----------------------------------------


@pytest.mark.parametrize("d_in,d_out", [(24, 24), (96, 96), (200, 200), (1000, 40), (1500, 70), (5, 3)])
def test_sage_forward_any_width_vs_oracle(d_in, d_out):
    rng = np.random.default_rng(d_in)
    n = 57
    edges = [(int(rng.integers(0, v)), v) for v in range(1, n) for _ in range(int(rng.integers(0, 3)))]
    h = rng.normal(size=(n, d_in))
    layer = SageLayerParams(rng.normal(size=(d_in, d_out)) / math.sqrt(d_in),
                            rng.normal(size=(d_in, d_out)) / math.sqrt(d_in), rng.normal(size=d_out) * 0.1)
    out = gnn.sage_forward(GraphEncoding(n, edges, h), layer, h)
    ref = O.sage_forward(n, edges, layer.w_self, layer.w_neigh, layer.bias, h)
    assert out.shape == ref.shape
    # stated fp32-mode tolerance grows with the contraction length K = 2 d_in (padded): the
    # tensor cores' fp32 accumulation of tf32 products rounds toward zero at every step, a
    # bias linear in K: 1e-5 max(1, |ref|) per 1024 of K
    K = 2 * gnn._agg_width(d_in, 32)
    assert np.max(np.abs(out - ref)) <= FP32_ABS * max(1.0, np.abs(ref).max()) * max(1.0, K / 1024)


@pytest.mark.parametrize("d", [3, 24, 96, 200, 1000, 1500, 2049])
def test_readout_mean_any_width(d):
    z = np.random.default_rng(d).normal(size=(77, d))
    got = gnn.readout_mean(z)
    assert got.shape == (d,)
    assert np.max(np.abs(got - z.mean(axis=0))) <= 1e-6


def test_sage_forward_errors():
    enc = GraphEncoding(3, [(0, 5)], np.zeros((3, 4)))
    layer = SageLayerParams(np.eye(4), np.eye(4), np.zeros(4))
    with pytest.raises(ShapeMismatch):
        gnn.sage_forward(enc, layer, np.zeros((3, 4)))
    with pytest.raises(ShapeMismatch):
        gnn.sage_forward(GraphEncoding(3, [], np.zeros((3, 4))), layer, np.zeros((3, 5)))


# -- the model protocol (gnn.py:212-262) ---------------------------------------------------------


def test_prepare_encoding_validation():
    with pytest.raises(EmptyGraph):
        gnn._prepare_encoding(GraphEncoding(0, [], np.zeros((0, 32))), _FS(np.zeros(5)))
    with pytest.raises(ShapeMismatch):
        gnn._prepare_encoding(GraphEncoding(2, [], np.zeros((2, 31))), _FS(np.zeros(5)))
    with pytest.raises(ShapeMismatch):
        gnn._prepare_encoding(GraphEncoding(2, [(0, 2)], np.zeros((2, 32))), _FS(np.zeros(5)))


@pytest.mark.parametrize("arch", ["sage", "mlp"])
@pytest.mark.parametrize("train", [False, True])
def test_forward_norm_backward_from_vs_oracle(golden, arch, train):
    recs = _records(golden)[:6]
    targets = np.stack([r.target.as_array for r in recs])
    statics = np.stack([r.fs.as_vector for r in recs])
    norm = Normalizer.fit(targets, statics)
    make = gnn.create_model if arch == "sage" else gnn.create_mlp_model
    model = make(hidden=32, seed=4, dropout_p=0.3, normalizer=norm)
    params = {k: np.array(v) for k, v in model.param_items()}
    for i, r in enumerate(recs):
        prep = gnn._prepare_record(r)
        fs_norm = norm.normalize_fs(prep.fs_raw)
        rng, rng_ref = np.random.default_rng(100 + i), np.random.default_rng(100 + i)
        out, cache = model.forward_norm(prep, fs_norm, train=train, rng=rng if train else None)
        masks = None
        if train:  # the reference draws fc1's mask, then fc2's (gnn.py:277-281)
            masks = (numerics.dropout_mask((32,), 0.3, rng_ref), numerics.dropout_mask((32,), 0.3, rng_ref))
            assert rng.random() == rng_ref.random()  # the device path consumed exactly those draws
        if arch == "sage":
            agg = O.aggregation_matrix(r.encoding.num_nodes, r.encoding.edges)
            ref_out, ref_cache = O.forward_norm(params, r.encoding.features, agg, fs_norm, masks)
        else:
            ref_out, ref_cache = O.fc_forward(params, fs_norm, masks)
        assert np.max(np.abs(out - ref_out)) <= FP32_ABS, (i, out, ref_out)
        dout = np.array([0.3, -1.1, 0.7])
        grads = model.backward_from(cache, dout)
        if arch == "sage":
            ref = O.backward_from(params, ref_cache, dout, 32)
        else:
            ref = {}
            O.fc_backward(params, ref_cache, dout, ref)
        assert sorted(grads) == sorted(ref)
        for k, g in ref.items():
            d = np.linalg.norm(grads[k] - g)
            assert d <= 1e-4 * np.linalg.norm(g) + 1e-6 * math.sqrt(g.size), (i, k, d)


def test_backward_from_matches_batched_backward(golden):
    """Sum of per-record protocol gradients / n == gnn.backward (gnn.py:383-405)."""
    recs = _records(golden)[:5]
    model = _fitted_model(recs, hidden=16, seed=3)
    for name, arr in model.param_items():
        if arr.ndim == 1:
            arr[...] = np.random.default_rng(len(name)).normal(0, 0.1, arr.shape)
    loss_b, grads_b = gnn.backward(model, recs)
    acc = {k: np.zeros_like(v) for k, v in model.param_items()}
    total = 0.0
    for r in recs:
        prep = gnn._prepare_record(r)
        out, cache = model.forward_norm(prep, model.normalizer.normalize_fs(prep.fs_raw))
        loss, dout = numerics.huber_loss(out, model.normalizer.normalize_y(prep.y_raw))
        total += loss
        for k, g in model.backward_from(cache, dout).items():
            acc[k] += g
    assert total / len(recs) == pytest.approx(loss_b, rel=1e-5)
    for k in acc:
        d = np.linalg.norm(acc[k] / len(recs) - grads_b[k])
        assert d <= 1e-4 * np.linalg.norm(grads_b[k]) + 1e-6 * math.sqrt(acc[k].size), (k, d)


def _protocol_fit(make_model, train_records, val_records, config):
    """The reference `_fit` (gnn.py:424-482) written against the protocol, verbatim in
    structure: everything it calls is this package's (prepare, forward_norm, backward_from,
    numerics.huber_loss, numerics.adam_step)."""
    rng = np.random.default_rng(config.seed)
    targets = np.stack([r.target.as_array for r in train_records])
    statics = np.stack([r.fs.as_vector for r in train_records])
    normalizer = Normalizer.fit(targets, statics)
    model = make_model(config.hidden, rng, gnn.DEFAULT_DROPOUT, normalizer)
    preps = [gnn._prepare_record(r) for r in train_records]
    fs_norm = np.stack([normalizer.normalize_fs(p.fs_raw) for p in preps])
    y_norm = np.stack([normalizer.normalize_y(p.y_raw) for p in preps])
    y_raw = np.stack([p.y_raw for p in preps])
    val_preps = [gnn._prepare_record(r) for r in val_records]
    params = model.param_items()
    states = {name: numerics.AdamState.for_param(arr.shape, config.lr) for name, arr in params}
    n, history = len(preps), []
    for epoch in range(1, config.epochs + 1):
        order = rng.permutation(n)
        loss_sum, ape_sum = 0.0, np.zeros(3)
        for i in order:
            out, cache = model.forward_norm(preps[i], fs_norm[i], train=True, rng=rng)
            loss, dout = numerics.huber_loss(out, y_norm[i], config.huber_delta)
            loss_sum += loss
            ape_sum += np.abs(normalizer.denormalize_y(out) - y_raw[i]) / np.abs(y_raw[i])
            grads = model.backward_from(cache, dout)
            for name, arr in params:
                arr[...] = numerics.adam_step(arr, grads[name], states[name])
        v_loss, v_ape = 0.0, np.zeros(3)
        for p in val_preps:
            out, _ = model.forward_norm(p, normalizer.normalize_fs(p.fs_raw))
            loss, _ = numerics.huber_loss(out, normalizer.normalize_y(p.y_raw), config.huber_delta)
            v_loss += loss
            v_ape += np.abs(normalizer.denormalize_y(out) - p.y_raw) / np.abs(p.y_raw)
        history.append([epoch, loss_sum / n, float((ape_sum / n).mean()), v_loss / len(val_preps),
                        float((v_ape / len(val_preps)).mean())])
    return model, np.array(history)


def test_reference_fit_loop_over_the_protocol_reproduces_golden_training(golden):
    recs = _records(golden, "train_rec_")
    cfg = gnn.TrainConfig(epochs=3, hidden=16, seed=123)
    model, hist = _protocol_fit(gnn._new_sage_model, recs[:8], recs[8:], cfg)
    assert np.allclose(hist, golden["train_hist"], rtol=1e-4, atol=1e-6), (hist, golden["train_hist"])
    for name, arr in model.param_items():
        r = golden[f"train_param_{name}"]
        assert np.max(np.abs(arr - r)) <= 1e-5 * max(1.0, np.abs(r).max()), name


# -- safety: concurrent read-only inference, error paths ---------------------


def test_concurrent_predict_on_shared_model(golden):
    """Several threads predicting with ONE model at once get exactly the serial results
    (each thread owns its workspaces; the parameters are read-only)."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2303_11733_b200.synth import make_dataset
    ds = make_dataset(96, seed=21, n_lo=20, n_hi=400)
    model = gnn.create_model(hidden=128, seed=2, normalizer=Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
    recs = ds.records(range(96))
    chunks = [recs[i::6] for i in range(6)]
    serial = [gnn.predict_batch(model, [r.encoding for r in c], [r.fs for r in c], precision=p)
              for c in chunks for p in ("fp32", "bf16")]

    def work(k):
        c, p = chunks[k // 2], ("fp32", "bf16")[k % 2]
        outs = []
        for _ in range(5):
            outs.append(gnn.predict_batch(model, [r.encoding for r in c], [r.fs for r in c], precision=p))
        return outs

    with ThreadPoolExecutor(6) as ex:
        results = list(ex.map(work, range(12)))
    for k, outs in enumerate(results):
        for y, mig in outs:
            assert np.array_equal(y, serial[k][0]) and np.array_equal(mig, serial[k][1]), k


def test_nonfinite_prediction_raises_in_batch_api_not_in_predict(golden):
    from paper_2303_11733_b200.errors import NonFinite
    recs = _records(golden)[:3]
    model = _fitted_model(recs, hidden=16)
    model.fc[2].b[1] = np.nan  # memory output NaN
    with pytest.raises(NonFinite):
        gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs])
    tv = gnn.predict(model, recs[0].encoding, recs[0].fs)  # the reference's predict returns the NaN
    assert math.isnan(tv.memory_mb)


def test_trainer_rejects_corrupt_host_batch():
    import torch
    from paper_2303_11733_b200.synth import make_dataset
    from paper_2303_11733_b200.trainer import BatchTrainer
    ds = make_dataset(8, seed=3)
    model = gnn.create_model(hidden=64, seed=1, normalizer=Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
    tr = BatchTrainer(model, precision="bf16")
    x, src, dst, gp, fs, y = ds.collate(np.arange(8))
    assert np.isfinite(tr.step_host(x, src, dst, gp, fs, y))
    bad = dst.copy()
    bad[5] = gp[-1] + 7  # endpoint outside the batch
    with pytest.raises(ShapeMismatch):
        tr.step_host(x, src, bad, gp, fs, y)
    cross = src.copy()
    cross[-1] = 0  # last graph's edge from graph 0's node
    with pytest.raises(ShapeMismatch):
        tr.step_host(x, cross, dst, gp, fs, y)
    ynan = y.copy()
    ynan[0, 0] = np.nan
    from paper_2303_11733_b200.errors import NonFinite
    with pytest.raises(NonFinite):
        tr.step_host(x, src, dst, gp, fs, ynan)
    del torch
