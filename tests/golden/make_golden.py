"""Generate the golden fixtures by running the REAL reference `dippm` package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src (and its test helpers
from /root/reference/pkg/tests), runs it on seeded inputs and writes
tests/golden/golden_v1.npz.  The GPU box never runs this script; the tests
read only the .npz it produced.

What is pinned (reference file:line in brackets):
  * records: synth_dataset [dataset.py:164], random_graph [tests/helpers.py:55],
    a resnetish depth-60 graph (N=305) [graph_ir.py:577], hand-made encodings
    with duplicate edges, self loops, isolated nodes, unsorted edges
  * dense aggregation pattern + in-degree per record [gnn.py:130-137] as CSR
  * forward (normalised) / predict (denormalised) per record, hidden 32 and
    hidden 512 models [gnn.py:348-361]
  * sage_forward single layer [gnn.py:331-338]
  * backward loss + 15 grads over a batch [gnn.py:383-405], batch_loss [:368]
  * huber / adam / dropout known answers [numerics.py:45-114]
  * MIG picks on a boundary sweep [mig.py:32-45]
  * a short reference-protocol train() run (history + final params) [gnn.py:424-482]
"""

from __future__ import annotations

import random
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

from dippm import dataset, gnn, graph_ir, mig, numerics  # noqa: E402
from dippm.featurize import GraphEncoding, StaticFeatures  # noqa: E402
from dippm.dataset import DatasetRecord, TargetVector  # noqa: E402
from helpers import random_graph  # noqa: E402

OUT = Path(__file__).with_name("golden_v1.npz")


def _handmade():
    """Edge cases the featurizer never emits but the API accepts."""
    rng = np.random.default_rng(99)
    recs = []
    specs = [
        (3, [(0, 2), (0, 2), (1, 2)]),               # duplicate edge: deg 3, summed once
        (3, [(0, 2), (2, 2), (1, 0)]),               # self loop honoured
        (4, []),                                      # all isolated
        (1, []),                                      # single node
        (5, [(4, 0), (3, 0), (0, 1), (2, 1), (1, 3), (4, 3), (4, 3)]),  # unsorted, dup, src > dst
    ]
    for n, edges in specs:
        x = np.abs(rng.normal(size=(n, 32)))
        enc = GraphEncoding(num_nodes=n, edges=list(edges), features=x)
        fs = StaticFeatures(macs=int(rng.integers(1e5, 1e9)), batch=int(rng.integers(1, 9)),
                            t_conv=int(rng.integers(0, 5)), t_dense=int(rng.integers(0, 5)),
                            t_relu=int(rng.integers(0, 5)))
        tv = TargetVector(latency_ms=float(rng.uniform(1, 5)), memory_mb=float(rng.uniform(600, 700)),
                          energy_j=float(rng.uniform(0.5, 2)))
        recs.append(DatasetRecord(encoding=enc, fs=fs, target=tv, model_name=f"hand-{n}"))
    return recs


def _permuted(rec, rng):
    enc = rec.encoding
    perm = rng.permutation(enc.num_nodes)
    feats = np.empty_like(enc.features)
    feats[perm] = enc.features
    edges = [(int(perm[s]), int(perm[d])) for s, d in enc.edges]
    return DatasetRecord(GraphEncoding(enc.num_nodes, edges, feats), rec.fs, rec.target, rec.model_name + "-perm")


def _pack_records(recs):
    n = np.array([r.encoding.num_nodes for r in recs], dtype=np.int64)
    ne = np.array([len(r.encoding.edges) for r in recs], dtype=np.int64)
    edges = np.array([e for r in recs for e in r.encoding.edges], dtype=np.int64).reshape(-1, 2)
    x = np.concatenate([np.asarray(r.encoding.features, dtype=np.float64) for r in recs])
    fs = np.stack([r.fs.as_vector for r in recs])
    fs_int = np.array([[r.fs.macs, r.fs.batch, r.fs.t_conv, r.fs.t_dense, r.fs.t_relu] for r in recs], dtype=np.int64)
    y = np.stack([r.target.as_array for r in recs])
    return {"n": n, "ne": ne, "edges": edges, "x": x, "fs": fs, "fs_int": fs_int, "y": y}


def _csr_from_dense(agg):
    """Pattern and in-degree read back from the reference's dense matrix."""
    n = agg.shape[0]
    rowptr = [0]
    cols = []
    deg = np.zeros(n, dtype=np.int64)
    for v in range(n):
        nz = np.nonzero(agg[v])[0]
        cols.extend(int(c) for c in nz)
        rowptr.append(len(cols))
        if len(nz):
            deg[v] = int(round(1.0 / agg[v, nz[0]]))
    return np.array(rowptr, dtype=np.int64), np.array(cols, dtype=np.int64), deg


def main():
    out = {}
    # -- records ------------------------------------------------------------
    recs = dataset.synth_dataset(24, seed=3)
    prng = random.Random(2024)
    recs += [dataset.record_from_graph(random_graph(prng, small=(i % 2 == 0))) for i in range(10)]
    recs += [dataset.record_from_graph(graph_ir.build_zoo_model(
        graph_ir.ZooSpec(family="resnetish", depth=60, width=8, batch_size=2, input_hw=16, seed=7)))]
    recs += _handmade()
    prng_np = np.random.default_rng(5)
    recs += [_permuted(recs[i], prng_np) for i in (0, 5, 24)]
    for k, v in _pack_records(recs).items():
        out[f"rec_{k}"] = v

    # -- CSR pattern from the dense aggregation matrix -------------------------
    rp, cl, dg = [], [], []
    for r in recs:
        a, b, c = _csr_from_dense(gnn._aggregation_matrix(r.encoding.num_nodes, r.encoding.edges))
        rp.append(a)
        cl.append(b)
        dg.append(c)
    out["csr_rowptr"] = np.concatenate(rp)
    out["csr_col"] = np.concatenate(cl) if any(len(c) for c in cl) else np.zeros(0, np.int64)
    out["csr_ncol"] = np.array([len(c) for c in cl], dtype=np.int64)
    out["csr_deg"] = np.concatenate(dg)

    # -- models ---------------------------------------------------------------
    train_like = [r for r in recs[:24]]
    targets = np.stack([r.target.as_array for r in train_like])
    statics = np.stack([r.fs.as_vector for r in train_like])
    norm = gnn.Normalizer.fit(targets, statics)
    for tag, hidden, seed in (("h32", 32, 11), ("h512", 512, 0)):
        model = gnn.create_model(hidden=hidden, seed=seed, normalizer=norm)
        out[f"{tag}_seed"] = np.array(seed)
        out[f"{tag}_hidden"] = np.array(hidden)
        out[f"{tag}_param_checksum"] = np.array([float(np.sum(a)) for _, a in model.param_items()])
        # biases are zero at init: give them values so the bias path is pinned
        brng = np.random.default_rng(seed + 100)
        for name, arr in model.param_items():
            if arr.ndim == 1:
                arr[...] = brng.normal(0.0, 0.1, size=arr.shape)
                out[f"{tag}_bias_{name}"] = arr.copy()
        fwd = np.stack([gnn.forward(r.encoding, r.fs, model) for r in recs])
        pred = np.stack([gnn.predict(model, r.encoding, r.fs).as_array for r in recs])
        out[f"{tag}_forward"] = fwd
        out[f"{tag}_predict"] = pred
        if hidden == 32:
            batch = recs[:12] + recs[34:39]
            loss, grads = gnn.backward(model, batch)
            out["h32_backward_idx"] = np.array(list(range(12)) + list(range(34, 39)))
            out["h32_backward_loss"] = np.array(loss)
            for name, g in grads.items():
                out[f"h32_grad_{name}"] = g
            out["h32_batch_loss"] = np.array(gnn.batch_loss(model, batch))
            # one sage layer on record 30 (random_graph) with layer-1 weights
            r = recs[24]
            out["sage_fwd_rec"] = np.array(24)
            out["sage_fwd_out"] = gnn.sage_forward(r.encoding, model.sage[0], np.asarray(r.encoding.features))
    out["norm_y_mean"], out["norm_y_std"] = norm.y_mean, norm.y_std
    out["norm_fs_mean"], out["norm_fs_std"] = norm.fs_mean, norm.fs_std

    # -- numerics known answers --------------------------------------------------
    hr = np.random.default_rng(7)
    pred, tgt = hr.normal(size=(64, 3)) * 2, hr.normal(size=(64, 3))
    hl = [numerics.huber_loss(p, t, 1.0) for p, t in zip(pred, tgt)]
    out["huber_pred"], out["huber_tgt"] = pred, tgt
    out["huber_loss"] = np.array([a for a, _ in hl])
    out["huber_grad"] = np.stack([b for _, b in hl])
    p0 = hr.normal(size=(1000,))
    st = numerics.AdamState.for_param(p0.shape)
    p = p0.copy()
    gs = hr.normal(size=(5, 1000))
    for g in gs:
        p = numerics.adam_step(p, g, st)
    out["adam_p0"], out["adam_grads"], out["adam_p5"] = p0, gs, p
    out["adam_m5"], out["adam_v5"] = st.m.copy(), st.v.copy()
    drng = np.random.default_rng(3)
    out["dropout_mask"] = numerics.dropout_mask((512,), 0.05, drng)

    # -- MIG boundary sweep ---------------------------------------------------------
    alphas = [0.0, -5.0, 1e-6, 2865, 2873, 4771, 5952, 6736, 26439, 45000, 5120.000001, 99999.0]
    for cap in (5120.0, 10240.0, 20480.0, 40960.0):
        alphas += [cap, np.nextafter(cap, 0.0), np.nextafter(cap, 1e9),
                   float(np.float32(cap)), float(np.nextafter(np.float32(cap), np.float32(0))),
                   float(np.nextafter(np.float32(cap), np.float32(1e9)))]
    alphas += list(np.random.default_rng(1).uniform(-1000, 50000, size=200))
    alphas = np.array(alphas, dtype=np.float64)
    labels = ["1g.5gb", "2g.10gb", "3g.20gb", "7g.40gb"]
    codes = []
    for a in alphas:
        p_ = mig.mig_profile(float(a))
        codes.append(-1 if p_ is None else labels.index(p_.label))
    out["mig_alpha"], out["mig_code"] = alphas, np.array(codes, dtype=np.int64)

    # -- reference-protocol training run ------------------------------------------------
    tr = dataset.synth_dataset(10, seed=8)
    cfg = gnn.TrainConfig(epochs=3, hidden=16, seed=123)
    model, hist = gnn.train(tr[:8], tr[8:], cfg)
    for k, v in _pack_records(tr).items():
        out[f"train_rec_{k}"] = v
    out["train_hist"] = np.array([[h["epoch"], h["train_loss"], h["train_mape"], h["val_loss"], h["val_mape"]]
                                  for h in hist])
    for name, arr in model.param_items():
        out[f"train_param_{name}"] = arr.copy()

    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1024:.1f} KiB, {len(out)} arrays, {len(recs)} records)")


if __name__ == "__main__":
    main()
