"""Pin the CPU oracle to the reference: every golden vector produced by running
the real `dippm` package (tests/golden/make_golden.py) must be reproduced."""

import numpy as np
import pytest

from conftest import unpack_records
from oracle import dippm_oracle as O


def _model(g, tag):
    hidden, seed = int(g[f"{tag}_hidden"]), int(g[f"{tag}_seed"])
    params = O.init_params(hidden, np.random.default_rng(seed))
    checksum = np.array([float(np.sum(params[k])) for k in O.SAGE_PARAM_NAMES])
    assert np.array_equal(checksum, g[f"{tag}_param_checksum"]), "numpy PCG64 stream changed"
    for k in O.SAGE_PARAM_NAMES:
        if params[k].ndim == 1:
            params[k] = g[f"{tag}_bias_{k}"].copy()
    return params


def _norm(g):
    return {"y_mean": g["norm_y_mean"], "y_std": g["norm_y_std"],
            "fs_mean": g["norm_fs_mean"], "fs_std": g["norm_fs_std"]}


def test_csr_pattern_and_degree_exact(golden):
    recs = unpack_records(golden)
    rp_off, col_off, deg_off = 0, 0, 0
    for i, (n, edges, *_rest) in enumerate(recs):
        rowptr, col, deg = O.csr_of_aggregation(n, edges)
        g_rp = golden["csr_rowptr"][rp_off:rp_off + n + 1]
        g_col = golden["csr_col"][col_off:col_off + golden["csr_ncol"][i]]
        g_deg = golden["csr_deg"][deg_off:deg_off + n]
        assert np.array_equal(rowptr, g_rp), i
        assert np.array_equal(col, g_col), i
        assert np.array_equal(deg, g_deg), i
        rp_off += n + 1
        col_off += len(g_col)
        deg_off += n


def test_duplicate_edge_semantics():
    # gnn.py:130-137: duplicates counted in deg, summed once
    agg = O.aggregation_matrix(3, [(0, 2), (0, 2), (1, 2)])
    h = np.array([1.0, 10.0, 100.0])
    assert (agg @ h)[2] == pytest.approx(11.0 / 3.0)


@pytest.mark.parametrize("tag", ["h32", "h512"])
def test_forward_and_predict_match_reference(golden, tag):
    params, norm = _model(golden, tag), _norm(golden)
    for i, (n, e, x, fs, _y) in enumerate(unpack_records(golden)):
        out = O.forward(params, norm, n, e, x, fs)
        assert np.allclose(out, golden[f"{tag}_forward"][i], rtol=0, atol=1e-12), i
        pred = O.predict(params, norm, n, e, x, fs)
        assert np.allclose(pred, golden[f"{tag}_predict"][i], rtol=1e-12, atol=1e-12), i


def test_backward_matches_reference(golden):
    params, norm = _model(golden, "h32"), _norm(golden)
    recs = unpack_records(golden)
    batch = [recs[i] for i in golden["h32_backward_idx"]]
    loss, grads = O.backward(params, norm, batch)
    assert loss == pytest.approx(float(golden["h32_backward_loss"]), rel=1e-12)
    assert O.batch_loss(params, norm, batch) == pytest.approx(float(golden["h32_batch_loss"]), rel=1e-12)
    for k in O.SAGE_PARAM_NAMES:
        assert np.allclose(grads[k], golden[f"h32_grad_{k}"], rtol=1e-9, atol=1e-12), k


def test_sage_forward_matches_reference(golden):
    params = _model(golden, "h32")
    n, e, x, _fs, _y = unpack_records(golden)[int(golden["sage_fwd_rec"])]
    out = O.sage_forward(n, e, params["sage1.w_self"], params["sage1.w_neigh"], params["sage1.bias"], x)
    assert np.allclose(out, golden["sage_fwd_out"], rtol=0, atol=1e-12)


def test_numerics_known_answers(golden):
    for p, t, l, gr in zip(golden["huber_pred"], golden["huber_tgt"], golden["huber_loss"], golden["huber_grad"]):
        loss, grad = O.huber_loss(p, t)
        assert loss == l
        assert np.array_equal(grad, gr)
    p = golden["adam_p0"].copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    for t, g in enumerate(golden["adam_grads"], start=1):
        p = O.adam_step(p, g, m, v, t)
    assert np.array_equal(p, golden["adam_p5"])
    assert np.array_equal(m, golden["adam_m5"]) and np.array_equal(v, golden["adam_v5"])
    assert np.array_equal(O.dropout_mask((512,), 0.05, np.random.default_rng(3)), golden["dropout_mask"])


def test_mig_sweep_matches_reference(golden):
    codes = [O.mig_code(float(a)) for a in golden["mig_alpha"]]
    assert codes == [int(c) for c in golden["mig_code"]]
    for bad in (float("nan"), float("inf"), -float("inf")):
        with pytest.raises(ValueError):
            O.mig_code(bad)


def test_reference_protocol_training_matches(golden):
    recs = unpack_records(golden, "train_rec_")
    params, _norm_, hist = O.train_reference_protocol(recs[:8], epochs=3, seed=123, hidden=16,
                                                      val_records=recs[8:])
    got = np.array([[h["epoch"], h["train_loss"], h["train_mape"], h["val_loss"], h["val_mape"]] for h in hist])
    assert np.allclose(got, golden["train_hist"], rtol=1e-10, atol=0)
    for k in O.SAGE_PARAM_NAMES:
        assert np.allclose(params[k], golden[f"train_param_{k}"], rtol=1e-10, atol=1e-14), k


# ---- §8f rows: MLP baseline, MAPE (tests/golden/make_golden_next.py) ----

MLP_TAGS = {"mlp32": (32, 11), "mlp512": (512, 0)}


def mlp_params(gn, tag):
    """Rebuild an MLP baseline from its seed (pins the reference draw order) + golden biases."""
    hidden, seed = MLP_TAGS[tag]
    params = O.init_mlp_params(hidden, np.random.default_rng(seed))
    checksum = np.array([float(np.sum(params[k])) for k in O.MLP_PARAM_NAMES])
    assert np.array_equal(checksum, gn[f"{tag}_param_checksum"]), "MLP init order / PCG64 stream changed"
    for k in O.MLP_PARAM_NAMES:
        if params[k].ndim == 1:
            params[k] = gn[f"{tag}_bias_{k}"].copy()
    return params


@pytest.mark.parametrize("tag", sorted(MLP_TAGS))
def test_mlp_forward_backward_match_reference(golden, golden_next, tag):
    recs, norm = unpack_records(golden), _norm(golden)
    params = mlp_params(golden_next, tag)
    fwd = np.stack([O.mlp_forward(params, norm, r[3]) for r in recs])
    assert np.allclose(fwd, golden_next[f"{tag}_forward"], rtol=1e-12, atol=1e-12)
    pred = np.stack([O.mlp_predict(params, norm, r[3]) for r in recs])
    assert np.allclose(pred, golden_next[f"{tag}_predict"], rtol=1e-12, atol=1e-9)
    loss, grads = O.mlp_backward(params, norm, recs[:20])
    assert abs(loss - float(golden_next[f"{tag}_backward_loss"])) <= 1e-12
    for k, g in grads.items():
        if f"{tag}_grad_{k}" in golden_next:
            assert np.allclose(g, golden_next[f"{tag}_grad_{k}"], rtol=1e-10, atol=1e-14), k
        else:
            st = golden_next[f"{tag}_gradstat_{k}"]
            assert np.isclose(np.linalg.norm(g), st[0], rtol=1e-10), k
            assert np.allclose(g.ravel()[::97], golden_next[f"{tag}_gradsample_{k}"], rtol=1e-9, atol=1e-14), k


def test_mape_matches_reference(golden, golden_next):
    recs, norm = unpack_records(golden), _norm(golden)
    params = mlp_params(golden_next, "mlp32")
    preds = [O.mlp_predict(params, norm, r[3]) for r in recs]
    m = O.mape(preds, [r[4] for r in recs])
    got = [m["latency"], m["memory"], m["energy"], m["overall"]]
    assert np.allclose(got, golden_next["mape_mlp32"], rtol=1e-12)


def test_mlp_reference_protocol_training_matches(golden, golden_next):
    recs = unpack_records(golden, "train_rec_")
    params, _n, hist = O.train_reference_protocol(recs[:8], epochs=3, seed=123, hidden=16, val_records=recs[8:],
                                                  arch="mlp")
    got = np.array([[h["epoch"], h["train_loss"], h["train_mape"], h["val_loss"], h["val_mape"]] for h in hist])
    assert np.allclose(got, golden_next["train_mlp_hist"], rtol=1e-10, atol=0)
    for k in O.MLP_PARAM_NAMES:
        assert np.allclose(params[k], golden_next[f"train_mlp_param_{k}"], rtol=1e-10, atol=1e-14), k
