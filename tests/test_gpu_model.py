"""Model-level parity on the B200 through the drop-in API, against the golden
vectors produced by the real reference and against the CPU oracle.

Tolerances: fp32 mode (3-pass TF32 tensor cores, fp32
elsewhere) normalised outputs |d| <= 1e-5 abs, de-normalised <= 1e-4 rel,
gradients ||d||/||g|| <= 1e-4 per tensor; bf16 mode normalised |d| <= 2e-2.
"""

import numpy as np
import pytest

from conftest import unpack_records
from oracle import dippm_oracle as O

pytestmark = pytest.mark.gpu

from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200 import mig as pmig  # noqa: E402
from paper_2303_11733_b200.errors import EmptyDataset, EmptyGraph, ShapeMismatch  # noqa: E402
from paper_2303_11733_b200.types import DatasetRecord, GraphEncoding, StaticFeatures, TargetVector  # noqa: E402

FP32_ABS = 1e-5
BF16_ABS = 2e-2


def grad_close(got, ref, rel=1e-4, abs_per_elem=1e-6):
    """Stated fp32 gradient tolerance: ||d|| <= 1e-4 ||g|| + 1e-6 sqrt(n).  The
    absolute floor covers reductions whose terms cancel (e.g. fc3.b = mean
    residual), where the ~1e-6 fp32 forward error dominates the tiny sum."""
    d = np.linalg.norm(np.asarray(got) - ref)
    return d <= rel * np.linalg.norm(ref) + abs_per_elem * np.sqrt(np.size(ref))


class _FS:
    def __init__(self, v):
        self.as_vector = np.asarray(v)


def _records(g, prefix="rec_"):
    out = []
    for n, e, x, fs, y in unpack_records(g, prefix):
        out.append(DatasetRecord(GraphEncoding(n, e, x), _FS(fs), TargetVector(*y)))
    return out


def _model(g, tag):
    hidden, seed = int(g[f"{tag}_hidden"]), int(g[f"{tag}_seed"])
    norm = gnn.Normalizer(g["norm_y_mean"], g["norm_y_std"], g["norm_fs_mean"], g["norm_fs_std"])
    m = gnn.create_model(hidden=hidden, seed=seed, normalizer=norm)
    for name, arr in m.param_items():
        if arr.ndim == 1:
            arr[...] = g[f"{tag}_bias_{name}"]
    return m


@pytest.mark.parametrize("tag", ["h32", "h512"])
def test_forward_matches_reference_fp32(golden, tag):
    model = _model(golden, tag)
    recs = _records(golden)
    for i, r in enumerate(recs):
        out = gnn.forward(r.encoding, r.fs, model)
        assert np.max(np.abs(out - golden[f"{tag}_forward"][i])) <= FP32_ABS, i
    y, mig = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs])
    ref = golden[f"{tag}_predict"]
    assert np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1e-3)) <= 1e-4
    assert np.max(np.abs((y - ref) / golden["norm_y_std"])) <= FP32_ABS
    assert [int(c) for c in mig] == [O.mig_code(float(v)) for v in ref[:, 1]]


@pytest.mark.parametrize("tag", ["h32", "h512"])
def test_forward_bf16_within_stated_tolerance(golden, tag):
    model = _model(golden, tag)
    recs = _records(golden)
    y, _ = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs], precision="bf16")
    ref = golden[f"{tag}_predict"]
    assert np.max(np.abs((y - ref) / golden["norm_y_std"])) <= BF16_ABS


def test_backward_matches_reference(golden):
    model = _model(golden, "h32")
    recs = _records(golden)
    batch = [recs[i] for i in golden["h32_backward_idx"]]
    loss, grads = gnn.backward(model, batch)
    assert loss == pytest.approx(float(golden["h32_backward_loss"]), rel=1e-5, abs=1e-7)
    assert gnn.batch_loss(model, batch) == pytest.approx(float(golden["h32_batch_loss"]), rel=1e-5, abs=1e-7)
    for name, _ in model.param_items():
        ref = golden[f"h32_grad_{name}"]
        assert grad_close(grads[name], ref), name


def test_backward_hidden512_vs_oracle(golden):
    model = _model(golden, "h512")
    recs = _records(golden)
    batch = recs[:24] + recs[34:39]
    loss, grads = gnn.backward(model, batch)
    params = {k: np.array(v) for k, v in model.param_items()}
    norm = {"y_mean": golden["norm_y_mean"], "y_std": golden["norm_y_std"],
            "fs_mean": golden["norm_fs_mean"], "fs_std": golden["norm_fs_std"]}
    orecs = [(r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector, r.target.as_array)
             for r in batch]
    ref_loss, ref_grads = O.backward(params, norm, orecs)
    assert loss == pytest.approx(ref_loss, rel=1e-5)
    for name in O.SAGE_PARAM_NAMES:
        assert grad_close(grads[name], ref_grads[name]), name


def test_sage_forward_reference_cases(golden):
    # T/test_gnn.py:36-59 known answers
    rng = np.random.default_rng(0)
    feats = rng.normal(size=(3, 4))
    enc = GraphEncoding(3, [(0, 1), (1, 2)], feats)
    layer = gnn.SageLayerParams(w_self=np.eye(4), w_neigh=np.zeros((4, 4)), bias=np.zeros(4))
    out = gnn.sage_forward(enc, layer, feats)
    assert np.allclose(out, np.maximum(feats, 0), atol=1e-6)
    feats = np.array([[1.0, -2.0], [0.5, 3.0]])
    out = gnn.sage_forward(GraphEncoding(2, [(0, 1)], feats),
                           gnn.SageLayerParams(np.zeros((2, 2)), np.eye(2), np.zeros(2)), feats)
    assert np.allclose(out[1], np.maximum(feats[0], 0)) and np.all(out[0] == 0)
    feats = np.array([[2.0, 0.0], [4.0, 2.0], [0.0, 0.0]])
    out = gnn.sage_forward(GraphEncoding(3, [(0, 2), (1, 2)], feats),
                           gnn.SageLayerParams(np.zeros((2, 2)), np.eye(2), np.zeros(2)), feats)
    assert np.allclose(out[2], [3.0, 1.0])
    # golden single layer
    model = _model(golden, "h32")
    r = _records(golden)[int(golden["sage_fwd_rec"])]
    out = gnn.sage_forward(r.encoding, model.sage[0], r.encoding.features)
    ref = golden["sage_fwd_out"]
    assert np.max(np.abs(out - ref)) <= 1e-5 * max(1.0, np.abs(ref).max())
    with pytest.raises(ShapeMismatch):
        gnn.sage_forward(r.encoding, model.sage[0], r.encoding.features[:, :5])


def test_readout_and_errors():
    z = np.array([[1.0, -2.0, 3.0]])
    assert np.allclose(gnn.readout_mean(z), z[0])
    e = np.array([1.0, -4.0, 2.0])
    assert np.allclose(gnn.readout_mean(np.stack([e, -e])), 0, atol=1e-7)
    with pytest.raises(EmptyGraph):
        gnn.readout_mean(np.zeros((0, 4)))
    model = gnn.create_model(hidden=8, seed=0)
    with pytest.raises(EmptyGraph):
        gnn.forward(GraphEncoding(0, [], np.zeros((0, 32))), _FS(np.zeros(5)), model)
    with pytest.raises(ShapeMismatch):
        gnn.forward(GraphEncoding(3, [], np.zeros((3, 31))), _FS(np.zeros(5)), model)
    with pytest.raises(ValueError):
        gnn.forward(GraphEncoding(3, [], np.zeros((3, 32))), _FS(np.zeros(5)), model, mode="predict")
    with pytest.raises(EmptyDataset):
        gnn.backward(model, [])


def test_zero_weights_give_final_bias(golden):
    model = _model(golden, "h32")
    for _, arr in model.param_items():
        arr[...] = 0.0
    model.fc[2].b[...] = np.array([1.5, -0.5, 2.0])
    for r in _records(golden)[:5]:
        assert np.array_equal(gnn.forward(r.encoding, r.fs, model), [1.5, -0.5, 2.0])


def test_mig_scalar_api_matches_reference_sweep(golden):
    codes = []
    for a in golden["mig_alpha"]:
        p = pmig.mig_profile(float(a))
        codes.append(-1 if p is None else list(pmig.MigProfile).index(p))
    assert codes == golden["mig_code"].tolist()


def test_reference_protocol_training_matches_golden(golden):
    recs = _records(golden, "train_rec_")
    cfg = gnn.TrainConfig(epochs=3, hidden=16, seed=123)
    model, hist = gnn.train(recs[:8], recs[8:], cfg)
    got = np.array([[h["epoch"], h["train_loss"], h["train_mape"], h["val_loss"], h["val_mape"]] for h in hist])
    ref = golden["train_hist"]
    assert np.allclose(got, ref, rtol=1e-4, atol=1e-6), (got, ref)
    for name, arr in model.param_items():
        r = golden[f"train_param_{name}"]
        assert np.max(np.abs(arr - r)) <= 1e-5 * max(1.0, np.abs(r).max()), name
    model2, hist2 = gnn.train(recs[:8], recs[8:], cfg)
    assert hist == hist2  # deterministic
    for (_, a), (_, b) in zip(model.param_items(), model2.param_items()):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("hidden", [40, 150, 200, 300, 700, 1000])
def test_odd_hidden_widths_match_oracle(hidden):
    """Hidden widths that are not powers of two are padded (64 / 192 / 256 / 384 / 768 / 1024
    wide on the device: three-chunk lanes for the 3 * 2^k widths) with zero weights:
    predictions equal the fp64 oracle's at fp32 tolerance."""
    from paper_2303_11733_b200.synth import make_dataset
    ds = make_dataset(6, seed=31, n_lo=20, n_hi=60)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=hidden, seed=2, normalizer=norm)
    recs = ds.records(range(6))
    y, _ = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs], precision="fp32")
    params = {k: np.array(v) for k, v in model.param_items()}
    nd = {"y_mean": norm.y_mean, "y_std": norm.y_std, "fs_mean": norm.fs_mean, "fs_std": norm.fs_std}
    for i, r in enumerate(recs):
        ref = O.predict(params, nd, r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector)
        assert np.allclose(y[i], ref, rtol=1e-4, atol=1e-3 * np.abs(ref).max()), (hidden, i, y[i], ref)


@pytest.mark.parametrize("hidden", [150, 300, 700])
def test_backward_three_chunk_widths_vs_oracle(hidden):
    """Gradients at hidden widths padded to 192 / 384 / 768 (the aggregation, transposed
    aggregation, readout and pooling kernels with three 8-column chunks per lane) against the
    fp64 oracle's backward."""
    from paper_2303_11733_b200.synth import make_dataset
    from paper_2303_11733_b200.device import Layout
    assert Layout(hidden).hp == {150: 192, 300: 384, 700: 768}[hidden]
    ds = make_dataset(12, seed=hidden, n_lo=20, n_hi=80)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=hidden, seed=4, normalizer=norm)
    batch = ds.records(range(12))
    loss, grads = gnn.backward(model, batch)
    params = {k: np.array(v) for k, v in model.param_items()}
    nd = {"y_mean": norm.y_mean, "y_std": norm.y_std, "fs_mean": norm.fs_mean, "fs_std": norm.fs_std}
    orecs = [(r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector, r.target.as_array)
             for r in batch]
    ref_loss, ref_grads = O.backward(params, nd, orecs)
    assert loss == pytest.approx(ref_loss, rel=1e-4)  # the forward's fp32 tolerance (3-pass tf32)
    # 768 wide: ReLU units within fp32 rounding of zero flip against the fp64 oracle; the oracle's
    # own SAGE gradients move by 2e-4..5e-4 (norm-relative) under a 1e-5 relative perturbation of
    # the weights at this width (tools/width_errors.py; 3e-3 at 1024), so the stated tolerance there is 1e-3
    rel = 1e-3 if hidden > 512 else 1e-4
    for name in O.SAGE_PARAM_NAMES:
        assert grad_close(grads[name], ref_grads[name], rel=rel), (hidden, name)
