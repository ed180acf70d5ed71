"""Parity at BASELINE.json sizes (hidden 512, 256-graph batches of ~300-node
graphs, graphs up to 5k nodes, power-law batches) through properties that do
not need the CPU oracle on every graph: sampled oracle checks, bit-exact
determinism, permutation invariance, MIG agreement away from the ceilings,
and one batched training step against gnn.backward + adam_step."""

import numpy as np
import pytest
import torch

from oracle import dippm_oracle as O

pytestmark = pytest.mark.gpu

from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402
from paper_2303_11733_b200.device import upload_batch  # noqa: E402
from paper_2303_11733_b200.types import GraphEncoding  # noqa: E402

FP32_ABS = 1e-5


def fp32_close(got_norm, ref_norm):
    """Stated fp32 tolerance in normalised space: |d| <= 1e-5 * max(1, |ref|) (an
    absolute 1e-5 for O(1) outputs; relative once random-init outputs are large,
    where fp32 itself cannot do better than ~1e-7 x condition)."""
    return np.all(np.abs(got_norm - ref_norm) <= FP32_ABS * np.maximum(1.0, np.abs(ref_norm)))


def _oracle_inputs(model):
    params = {k: np.array(v) for k, v in model.param_items()}
    n = model.normalizer
    return params, {"y_mean": n.y_mean, "y_std": n.y_std, "fs_mean": n.fs_mean, "fs_std": n.fs_std}


def _trained_like(ds, hidden=512, seed=0, bias_scale=0.05):
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    m = gnn.create_model(hidden=hidden, seed=seed, normalizer=norm)
    rng = np.random.default_rng(seed + 1)
    for _, arr in m.param_items():
        if arr.ndim == 1:
            arr[...] = rng.normal(0, bias_scale, size=arr.shape)
    return m


@pytest.fixture(scope="module")
def cfg1():
    ds = make_dataset(256, seed=1)
    return ds, ds.records(range(256)), _trained_like(ds)


def test_cfg1_batch_sampled_oracle_and_determinism(cfg1):
    ds, recs, model = cfg1
    y1, mig1 = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs])
    y2, mig2 = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs])
    assert np.array_equal(y1, y2) and np.array_equal(mig1, mig2)  # bit-reproducible
    params, norm = _oracle_inputs(model)
    for i in (0, 17, 101, 255):
        r = recs[i]
        ref = O.predict(params, norm, r.encoding.num_nodes, r.encoding.edges, r.encoding.features,
                        r.fs.as_vector)
        assert fp32_close(y1[i] / norm["y_std"], ref / norm["y_std"]), (i, y1[i], ref)
    yb, _ = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs], precision="bf16")
    assert np.max(np.abs((yb - y1) / norm["y_std"])) <= 2e-2


def test_permutation_invariance_fp32(cfg1):
    _, recs, model = cfg1
    rng = np.random.default_rng(0)
    base = np.stack([gnn.forward(r.encoding, r.fs, model) for r in recs[:4]])
    for k, r in enumerate(recs[:4]):
        enc = r.encoding
        perm = rng.permutation(enc.num_nodes)
        feats = np.empty_like(enc.features)
        feats[perm] = enc.features
        edges = [(int(perm[s]), int(perm[d])) for s, d in enc.edges]
        out = gnn.forward(GraphEncoding(enc.num_nodes, edges, feats), r.fs, model)
        assert fp32_close(out, base[k])  # reference: <1e-9 in fp64 (T/test_gnn.py:283)


def test_large_graph_5k_nodes():
    ds = make_dataset(2, seed=4, n_lo=4900, n_hi=5000)
    model = _trained_like(ds, seed=3)
    recs = ds.records(range(2))
    y, _ = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs])
    params, norm = _oracle_inputs(model)
    r = recs[0]
    ref = O.predict(params, norm, r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector)
    assert fp32_close(y[0] / norm["y_std"], ref / norm["y_std"]), (y[0], ref)


def test_powerlaw_mig_picks_match_oracle():
    """cfg5-like: power-law node counts, normaliser spreading memory over all profiles."""
    ds = make_dataset(512, seed=5, n_lo=2, power_law=1.5, n_max=2000, memory_scale=40.0)
    model = _trained_like(ds, hidden=64, seed=5, bias_scale=0.5)
    # spread predicted memory across 0..45 GB: put the memory output on a wide scale
    model.normalizer.y_mean = np.array([model.normalizer.y_mean[0], 22000.0, model.normalizer.y_mean[2]])
    model.normalizer.y_std = np.array([model.normalizer.y_std[0], 13000.0, model.normalizer.y_std[2]])
    recs = ds.records(range(512))
    y, mig = gnn.predict_batch(model, [r.encoding for r in recs], [r.fs for r in recs])
    params, norm = _oracle_inputs(model)
    agree = band = 0
    for i in range(0, 512, 4):
        r = recs[i]
        ref = O.predict(params, norm, r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector)
        near = min(abs(ref[1] - c) for c in O.MIG_CEILINGS_MB) < 1.0
        band += near
        if not near:
            assert int(mig[i]) == O.mig_code(float(ref[1])), i
            agree += 1
    assert agree >= 120 and len(set(mig.tolist())) >= 3  # several profiles (and None) exercised


def test_batched_training_step_matches_backward_and_adam(cfg1):
    """One BatchTrainer step (dropout off, fp32) == gnn.backward over the batch + adam_step."""
    ds, recs, model = cfg1
    batch = list(range(64))
    params0, norm = _oracle_inputs(model)
    tr = BatchTrainer(model, precision="fp32", lr=1e-3, dropout=False)
    b = upload_batch(*ds.collate(np.array(batch)), device="cuda", build_csr=False)
    tr.step_resident(b)
    got = tr.engine.get_params()
    orecs = [(r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector, r.target.as_array)
             for r in (recs[i] for i in batch)]
    _, grads = O.backward(params0, norm, orecs)
    for k in O.SAGE_PARAM_NAMES:
        m, v = np.zeros_like(grads[k]), np.zeros_like(grads[k])
        ref = O.adam_step(params0[k], grads[k], m, v, 1, lr=1e-3)
        # first Adam step moves every coordinate by ~lr*sign(g): compare the update direction/size
        upd, ref_upd = got[k] - params0[k], ref - params0[k]
        big = np.abs(grads[k]) > 1e-3 * np.abs(grads[k]).max()
        assert np.mean(np.sign(upd[big]) == np.sign(ref_upd[big])) > 0.999, k
        assert np.allclose(upd[big], ref_upd[big], rtol=1e-3, atol=1e-7), k


def test_cuda_graph_replay_equals_eager_steps(cfg1):
    """Captured-and-replayed training steps (dropout on, bf16) are bit-identical to
    eager steps: Adam's t and the dropout stream advance on the device."""
    ds, _, model = cfg1
    finals = []
    for graphs in (False, True):
        tr = BatchTrainer(model, precision="bf16", lr=1e-3, dropout=True, use_graphs=graphs)
        b = upload_batch(*ds.collate(np.arange(64)), device="cuda", build_csr=False)
        losses = []
        for _ in range(4):
            tr.step_resident(b)
            losses.append(float(tr.ws.loss[0]))
        assert tr.engine.t == 4
        finals.append((tr.engine.params.cpu().numpy(), losses))
    assert np.array_equal(finals[0][0], finals[1][0])
    assert finals[0][1] == finals[1][1]
    assert len(set(finals[0][1])) == 4  # the steps really differ (masks and params move)


def test_pipelined_host_steps_equal_sequential_and_resident(cfg1):
    """BatchTrainer.submit (double-buffered H2D on a copy stream, loss read back per
    step) gives bit-identical parameters and losses to synchronous step_host and
    to step_resident on the same batches, including a batch larger than the
    staging slots (forces a re-reserve mid-pipeline)."""
    ds, _, model = cfg1
    idx = [np.arange(0, 48), np.arange(48, 96), np.arange(96, 256), np.arange(10, 40)]
    host = []
    for ii in idx:
        arrays = ds.collate(ii)
        host.append([torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in arrays])
    runs = []
    for mode in ("resident", "sync", "pipelined"):
        tr = BatchTrainer(model, precision="bf16", lr=1e-3, dropout=True)
        tr.reserve(int(host[0][3][-1]) + 1, 48)  # smaller than batch 2: re-reserve while steps are in flight
        losses = []
        if mode == "resident":
            for h in host:
                tr.step_resident(upload_batch(*[a.numpy() for a in h], device="cuda", build_csr=False))
                losses.append(float(tr.ws.loss[0]))
        elif mode == "sync":
            losses = [tr.step_host(*h) for h in host]
        else:
            losses = [hd.loss() for hd in [tr.submit(*h) for h in host]]
        runs.append((tr.engine.params.cpu().numpy(), losses))
    for p, l in runs[1:]:
        assert np.array_equal(p, runs[0][0])
        assert l == runs[0][1]


def test_fused_readout_matches_unfused_pool_and_simt_engine():
    """The readout fused into the layer-3 GEMM epilogue (segmented block sums + combine) gives
    the same pooled vectors as the unfused pool kernel of the SIMT anchor engine, for graph
    sizes around the 32-row block edges (1, 2, 31, 32, 33, 63, 64, 65, ...) and a 5k-node
    graph; training gradients of the two engines agree too (fp32)."""
    from paper_2303_11733_b200.device import Engine, Workspace
    sizes = [1, 2, 31, 32, 33, 63, 64, 65, 3, 127, 128, 129, 1, 300, 5000, 17, 1, 1, 40]
    rng = np.random.default_rng(12)
    gp = np.zeros(len(sizes) + 1, np.int32)
    np.cumsum(sizes, out=gp[1:])
    src, dst = [], []
    for g, n in enumerate(sizes):
        for v in range(1, n):
            src.append(gp[g] + v - 1)
            dst.append(gp[g] + v)
            if v > 2 and rng.random() < 0.3:
                src.append(gp[g] + int(rng.integers(0, v - 1)))
                dst.append(gp[g] + v)
    N = int(gp[-1])
    x = np.abs(rng.normal(size=(N, 32))).astype(np.float32)
    fs = rng.normal(size=(len(sizes), 5)).astype(np.float32)
    y = np.abs(rng.normal(size=(len(sizes), 3))).astype(np.float32) + 1
    b = upload_batch(x, np.array(src), np.array(dst), gp, fs, y, device="cuda")
    norm = gnn.Normalizer(np.zeros(3), np.ones(3), np.zeros(5), np.ones(5))
    model = _trained_like(make_dataset(64, seed=3), hidden=128, seed=5)
    model.normalizer = norm
    res = {}
    for backend in ("tc", "simt"):
        eng = Engine(128, "fp32", backend=backend)
        eng.set_params(model.param_items(), norm)
        ws = Workspace(eng, b.N, b.G, train=True)
        eng.forward(b, ws)
        eng.loss(b, ws)
        eng.backward(b, ws)
        res[backend] = (ws.u.to_float()[:, :128].double().cpu().numpy(), ws.out.double().cpu().numpy(),
                        eng.get_grads())
    u_tc, u_simt = res["tc"][0], res["simt"][0]
    assert np.max(np.abs(u_tc - u_simt)) <= 1e-5 * max(1.0, np.abs(u_simt).max())
    assert np.max(np.abs(res["tc"][1] - res["simt"][1])) <= 1e-4 * max(1.0, np.abs(res["simt"][1]).max())
    for k, g in res["simt"][2].items():
        d = np.linalg.norm(res["tc"][2][k] - g)
        assert d <= 1e-3 * np.linalg.norm(g) + 1e-6 * np.sqrt(g.size), (k, d, np.linalg.norm(g))
