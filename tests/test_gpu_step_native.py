"""The native training-step executor (dippm_train_step, csrc/step.cu) against the Python
orchestration of the same step (device.Engine forward / loss / backward / adam_step):
same kernels, arguments and order, so after several steps -- dropout on, CSR rebuilt
every step, weight gradients on the side stream -- the fp64 masters, the Adam moments, the
gradients and every loss must be bit-identical, eager, captured in CUDA graphs, and
through the end-to-end submit() call.  The oracle parity of that path is
tests/test_gpu_headline.py (its bf16 trainer step now runs natively)."""

import copy

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2303_11733_b200 import gnn, trainer as trainer_mod  # noqa: E402
from paper_2303_11733_b200.device import group_edges, upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402


@pytest.fixture(scope="module")
def data():
    ds = make_dataset(640, seed=5)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=512, seed=3, normalizer=norm)
    rng = np.random.default_rng(4)
    for _, arr in model.param_items():
        if arr.ndim == 1:
            arr[...] = rng.normal(0, 0.05, size=arr.shape)
    perm = np.random.default_rng(9).permutation(ds.num_graphs)
    idx = [perm[0:256], perm[256:512], perm[512:640]]  # last batch smaller (ragged G)
    return ds, model, idx


def _run(model, ds, idx, native, monkeypatch, use_graphs=False, shuffle_edges=False, host=False, graphed=True,
         prep=True):
    monkeypatch.setattr(trainer_mod, "NATIVE_STEP", native)
    monkeypatch.setattr(trainer_mod, "NATIVE_GRAPHED", graphed)
    monkeypatch.setattr(trainer_mod, "NATIVE_PREP", prep)
    tr = BatchTrainer(copy.deepcopy(model), precision="bf16", lr=1e-3, seed=7, use_graphs=use_graphs)
    losses = []
    for rep in range(2 if use_graphs else 1):  # graphs: the second pass replays the captures
        for k, ix in enumerate(idx):
            x, src, dst, gp, fs, y = ds.collate(ix)
            if shuffle_edges:
                p = np.random.default_rng(k).permutation(len(src))
                src, dst = src[p], dst[p]
            if host:
                h = tr.submit(x, src, dst, gp, fs, y,
                              edge_ptr=None if shuffle_edges else group_edges(src, dst, gp))
                losses.append(h.loss())
                continue
            b = upload_batch(x, src, dst, gp, fs, y, device="cuda", build_csr=False,
                             edge_ptr=None if shuffle_edges else group_edges(src, dst, gp))
            if shuffle_edges:
                b.edge_ptr = None
            if use_graphs:
                tr._keep.append(b)  # one batch object per step, kept alive for its capture
            tr.step_resident(b)
            torch.cuda.synchronize()
            losses.append(float(tr.ws.loss[0]))
    torch.cuda.synchronize()
    e = tr.engine
    return losses, e.params.clone(), e.m.clone(), e.v.clone(), e.grads.clone(), int(e.t_dev.item()), tr


def _same(a, b):
    la, pa, ma, va, ga, ta, _ = a
    lb, pb, mb, vb, gb, tb, _ = b
    assert la == lb
    assert ta == tb
    for x, y in ((pa, pb), (ma, mb), (va, vb), (ga, gb)):
        assert torch.equal(x, y)


def test_native_step_bit_identical_to_python_orchestration(data, monkeypatch):
    ds, model, idx = data
    nat = _run(model, ds, idx, True, monkeypatch)
    assert nat[6]._native is not None  # the native executor ran
    py = _run(model, ds, idx, False, monkeypatch)
    assert py[6]._native is None
    _same(nat, py)
    assert all(np.isfinite(nat[0]))


def test_native_step_captured_in_cuda_graphs(data, monkeypatch):
    ds, model, idx = data
    nat = _run(model, ds, idx, True, monkeypatch, use_graphs=True)
    py = _run(model, ds, idx, False, monkeypatch, use_graphs=True)
    _same(nat, py)


def test_native_step_global_csr_path_and_submit(data, monkeypatch):
    """Edges not grouped by graph (edge_ptr None: the global K1 path inside the executor),
    and the end-to-end submit() call from host arrays."""
    ds, model, idx = data
    _same(_run(model, ds, idx, True, monkeypatch, shuffle_edges=True),
          _run(model, ds, idx, False, monkeypatch, shuffle_edges=True))
    py = _run(model, ds, idx, False, monkeypatch, host=True)
    _same(_run(model, ds, idx, True, monkeypatch, host=True), py)  # one updated CUDA graph per step
    _same(_run(model, ds, idx, True, monkeypatch, host=True, graphed=False), py)  # launch by launch


def test_native_graphed_steps_ragged_batches(data, monkeypatch):
    """submit() over many ragged batches (N, E, G change every step; the edge order switches
    between grouped and global K1 paths, which changes the captured topology and forces a
    re-instantiation): identical to the Python orchestration throughout."""
    ds, model, _ = data
    rng = np.random.default_rng(11)
    idx = [rng.choice(ds.num_graphs, size=int(s), replace=False) for s in (200, 256, 7, 256, 131, 256)]
    _same(_run(model, ds, idx, True, monkeypatch, host=True), _run(model, ds, idx, False, monkeypatch, host=True))


@pytest.mark.parametrize("mode", ["eager", "graphs", "host"])
def test_native_step_k1_inline_equals_prepared(data, monkeypatch, mode):
    """K1 at the head of the step (the plan's CSR buffers) and K1 ahead of it on another
    stream into per-batch / per-slot CSR sets (dippm_train_prep): identical results."""
    ds, model, idx = data
    kw = dict(use_graphs=mode == "graphs", host=mode == "host")
    _same(_run(model, ds, idx, True, monkeypatch, prep=False, **kw), _run(model, ds, idx, True, monkeypatch, **kw))
    if mode == "host":  # the global-CSR K1 path (edges not grouped by graph) prepared ahead too
        _same(_run(model, ds, idx, True, monkeypatch, prep=False, shuffle_edges=True),
              _run(model, ds, idx, True, monkeypatch, shuffle_edges=True))


def test_native_step_flags_bad_edges(data, monkeypatch):
    """A device-flagged edge (endpoint outside its graph) surfaces as ShapeMismatch at the
    loss read-back of the native step, as on the Python path."""
    from paper_2303_11733_b200.errors import ShapeMismatch
    ds, model, idx = data
    monkeypatch.setattr(trainer_mod, "NATIVE_STEP", True)
    tr = BatchTrainer(copy.deepcopy(model), precision="bf16", lr=1e-3)
    x, src, dst, gp, fs, y = ds.collate(idx[2])
    ep = group_edges(src, dst, gp)
    src = src.copy()
    src[3] = gp[5] + 1  # crosses into graph 5 (edge 3 belongs to graph 0)
    b = upload_batch(x, src, dst, gp, fs, y, device="cuda", build_csr=False, edge_ptr=ep, validate=False)
    tr.step_resident(b)
    torch.cuda.synchronize()
    assert int(b.bad[0]) == 1
    with pytest.raises(ShapeMismatch):
        tr.submit(x, src, dst, gp, fs, y, edge_ptr=ep).loss()


def test_native_step_follows_learning_rate_changes(data, monkeypatch):
    """A learning-rate schedule (trainer.lr changed between steps) reaches the native step."""
    ds, model, idx = data
    res = []
    for native in (True, False):
        monkeypatch.setattr(trainer_mod, "NATIVE_STEP", native)
        tr = BatchTrainer(copy.deepcopy(model), precision="bf16", lr=1e-3, seed=7)
        for k, ix in enumerate(idx):
            tr.lr = 1e-3 * (0.5 ** k)
            tr.step_resident(upload_batch(*ds.collate(ix), device="cuda", build_csr=False))
        torch.cuda.synchronize()
        res.append(tr.engine.params.clone())
    assert torch.equal(res[0], res[1])


@pytest.mark.parametrize("hidden", [40, 128, 300])
def test_native_step_other_widths(monkeypatch, hidden):
    """Other hidden widths (padded to 64 / 128 / 384: the layout-generic readout and
    aggregation kernels, three-chunk lanes, the fused head's small tiles) and tiny ragged
    batches: native == Python.  (Beyond 512 the fused head, and with it the native executor,
    is not used.)"""
    ds = make_dataset(96, seed=hidden)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=hidden, seed=1, normalizer=norm)
    idx = [np.arange(0, 64), np.arange(64, 65), np.arange(65, 96)]
    res = []
    for native in (True, False):
        monkeypatch.setattr(trainer_mod, "NATIVE_STEP", native)
        tr = BatchTrainer(copy.deepcopy(model), precision="bf16", lr=1e-3, seed=3)
        for ix in idx:
            tr.step_resident(upload_batch(*ds.collate(ix), device="cuda", build_csr=False))
        torch.cuda.synchronize()
        assert (tr._native is not None) == native
        res.append((tr.engine.params.clone(), float(tr.ws.loss[0])))
    assert torch.equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]


def test_native_prep_rejects_small_sets_and_plans(data, monkeypatch):
    """dippm_train_prep / dippm_train_step return DIPPM_ERR_ARG (nothing launched; raised as
    ShapeMismatch) for a CSR set smaller than the batch."""
    from paper_2303_11733_b200.errors import ShapeMismatch
    from paper_2303_11733_b200.trainer import CsrBuffers
    ds, model, idx = data
    monkeypatch.setattr(trainer_mod, "NATIVE_STEP", True)
    tr = BatchTrainer(copy.deepcopy(model), precision="bf16", lr=1e-3)
    b = upload_batch(*ds.collate(idx[0]), device="cuda", build_csr=False)
    tr.step_resident(b)  # builds the plan
    nat = tr._native
    small = CsrBuffers(b.N // 2, b.E // 2, b.G, b.x.device)
    with pytest.raises(ShapeMismatch, match="CSR set"):
        nat.prep(b, small, torch.cuda.current_stream())
    with pytest.raises(ShapeMismatch, match="prepared CSR set"):
        nat.step(b, cset=small)
    torch.cuda.synchronize()
