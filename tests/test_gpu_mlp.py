"""MLP baseline (gnn.py:236-262, 418-421) on the B200 head kernels, against the
golden vectors of the real reference (tests/golden/make_golden_next.py).

Tolerances as for the graph model: fp32 mode normalised
|d| <= 1e-5, de-normalised rel <= 1e-4, gradients ||d|| <= 1e-4 ||g|| + 1e-6 sqrt(n)."""

import numpy as np
import pytest

from test_gpu_model import _records, grad_close

pytestmark = pytest.mark.gpu

from paper_2303_11733_b200 import gnn  # noqa: E402

MLP_TAGS = {"mlp32": (32, 11), "mlp512": (512, 0)}


def _mlp(golden, gn, tag):
    hidden, seed = MLP_TAGS[tag]
    norm = gnn.Normalizer(golden["norm_y_mean"], golden["norm_y_std"], golden["norm_fs_mean"], golden["norm_fs_std"])
    m = gnn.create_mlp_model(hidden=hidden, seed=seed, normalizer=norm)
    assert np.array_equal([float(np.sum(a)) for _, a in m.param_items()], gn[f"{tag}_param_checksum"])
    for name, arr in m.param_items():
        if arr.ndim == 1:
            arr[...] = gn[f"{tag}_bias_{name}"]
    return m


@pytest.mark.parametrize("tag", sorted(MLP_TAGS))
def test_mlp_forward_predict_backward(golden, golden_next, tag):
    model = _mlp(golden, golden_next, tag)
    recs = _records(golden)
    fwd = np.stack([gnn.forward(r.encoding, r.fs, model) for r in recs[:6]])
    assert np.max(np.abs(fwd - golden_next[f"{tag}_forward"][:6])) <= 1e-5
    y, mig = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs])
    ref = golden_next[f"{tag}_predict"]
    assert np.all(np.abs(y - ref) <= 1e-4 * np.abs(ref) + 1e-6)
    loss, grads = gnn.backward(model, recs[:20])
    assert abs(loss - float(golden_next[f"{tag}_backward_loss"])) <= 1e-5 * max(1.0, abs(loss))
    assert abs(gnn.batch_loss(model, recs[:20]) - float(golden_next[f"{tag}_batch_loss"])) <= 1e-5
    for k, g in grads.items():
        if f"{tag}_grad_{k}" in golden_next:
            assert grad_close(g, golden_next[f"{tag}_grad_{k}"]), k
        else:
            nrm = golden_next[f"{tag}_gradstat_{k}"][0]
            assert abs(np.linalg.norm(g) - nrm) <= 1e-4 * nrm + 1e-6 * np.sqrt(g.size), k


def test_mlp_reference_protocol_training(golden, golden_next):
    recs = _records(golden, "train_rec_")
    model, hist = gnn.train_mlp(recs[:8], recs[8:], gnn.TrainConfig(epochs=3, hidden=16, seed=123))
    assert model.arch == "mlp"
    got = np.array([[h["epoch"], h["train_loss"], h["train_mape"], h["val_loss"], h["val_mape"]] for h in hist])
    assert np.allclose(got, golden_next["train_mlp_hist"], rtol=1e-4, atol=1e-6)
    for name, arr in model.param_items():
        r = golden_next[f"train_mlp_param_{name}"]
        assert np.max(np.abs(arr - r)) <= 1e-5 * max(1.0, np.abs(r).max()), name


def test_mlp_save_load_round_trip(golden, golden_next, tmp_path):
    model = _mlp(golden, golden_next, "mlp32")
    path = tmp_path / "mlp.json"
    gnn.save_model(model, path)
    back = gnn.load_model(path)
    assert back.arch == "mlp"
    for (n1, a), (n2, b) in zip(model.param_items(), back.param_items()):
        assert n1 == n2 and np.array_equal(a, b)
    recs = _records(golden)[:4]
    y1, _ = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs])
    y2, _ = gnn.predict_batch(back, [r.encoding for r in recs], [r.fs for r in recs])
    assert np.array_equal(y1, y2)


def test_mlp_batched_training_bf16_reduces_loss(golden):
    recs = _records(golden, "train_rec_") * 8
    cfg = gnn.TrainConfig(epochs=20, hidden=64, seed=1, batch_size=16, precision="bf16", lr=3e-3)
    model, hist = gnn.train_mlp(recs, [], cfg)
    assert hist[-1]["train_loss"] < hist[0]["train_loss"]
