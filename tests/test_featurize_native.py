"""§8f row 1 — the native front end (libdippm_host.so) against the reference's
Python front end: every golden document (tests/golden/make_golden_featurize.py:
zoo models, random graphs, non-canonical rewrites, batch overrides, malformed
documents) must give bit-identical features, edges and static features, or the
same exception class."""

import json

import numpy as np
import pytest

from pathlib import Path

from paper_2303_11733_b200 import errors as E
from paper_2303_11733_b200 import featurize as F

GOLD = Path(__file__).resolve().parent / "golden" / "golden_featurize_v1.npz"


@pytest.fixture(scope="module")
def gf():
    return dict(np.load(GOLD))


def _docs(g):
    blob, off = bytes(g["doc_bytes"]), g["doc_offsets"]
    return [blob[off[i]:off[i + 1]] for i in range(len(off) - 1)]


@pytest.mark.parametrize("threads", [1, 0])
def test_native_featuriser_bit_exact_vs_reference(gf, threads):
    docs = _docs(gf)
    bo = gf["batch_override"]
    fb = F.featurize_documents(docs, bo, threads=threads)
    xo = eo = 0
    for i in range(len(docs)):
        want = str(gf["error"][i])
        err = fb.error(i)
        if want:
            assert err is not None and type(err).__name__ == want, (i, want, err)
            continue
        assert err is None, (i, err)
        n, ne = int(gf["n"][i]), int(gf["ne"][i])
        enc = fb.encoding(i)
        assert enc.num_nodes == n, i
        assert np.array_equal(enc.features, gf["x"][xo:xo + n]), i  # float64, bit-exact
        assert [tuple(e) for e in enc.edges] == [tuple(e) for e in gf["edges"][eo:eo + ne].tolist()], i
        st = fb.static(i)
        assert [st.macs, st.batch, st.t_conv, st.t_dense, st.t_relu] == gf["fs_int"][i].tolist(), i
        assert np.array_equal(st.as_vector, fb.fs_vectors()[i])
        assert fb.names[i] == str(gf["name"][i])
        xo += n
        eo += ne


def test_collate_layout_matches_upload_contract(gf):
    docs = [d for d, e in zip(_docs(gf), gf["error"]) if not str(e)][:20]
    fb = F.featurize_documents(docs)
    x, src, dst, gp, fs, ep = fb.collate()
    assert x.dtype == np.float32 and x.shape == (int(fb.n.sum()), 32)
    assert gp[0] == 0 and gp[-1] == len(x) and len(gp) == len(docs) + 1
    for g in range(len(docs)):  # every edge stays inside its graph, edge_ptr groups them
        s, d = src[ep[g]:ep[g + 1]], dst[ep[g]:ep[g + 1]]
        assert np.all((s >= gp[g]) & (s < gp[g + 1]) & (d >= gp[g]) & (d < gp[g + 1]))
    assert np.array_equal(x, fb.x.astype(np.float32))
    # the native collated export (dippm_feat_collate) writes exactly these arrays
    G, N, E = len(docs), len(x), len(src)
    nx, ns, nd = np.empty((N, 32), np.float32), np.empty(E, np.int64), np.empty(E, np.int64)
    ngp, nep, nfs = np.empty(G + 1, np.int32), np.empty(G + 1, np.int64), np.empty((G, 5), np.float64)
    F._host().dippm_feat_collate(fb._h, nx.ctypes.data, ns.ctypes.data, nd.ctypes.data, ngp.ctypes.data,
                                 nep.ctypes.data, nfs.ctypes.data)
    for a, b in ((x, nx), (src, ns), (dst, nd), (gp, ngp), (ep, nep), (fs, nfs)):
        assert a.dtype == b.dtype and np.array_equal(a, b)


class _Node:
    def __init__(self, id, raw_name, inputs, attrs, out_shape):
        self.id, self.raw_name, self.inputs, self.attrs, self.out_shape = id, raw_name, inputs, attrs, out_shape


class _Graph:
    def __init__(self, nodes, outputs, batch_size, name):
        self.nodes, self.outputs, self.batch_size, self.name = nodes, outputs, batch_size, name


def test_drop_in_accepts_graph_objects_and_raises_reference_errors():
    g = _Graph([_Node(0, "input", [], {}, [2, 3, 8, 8]),
                _Node(1, "nn.conv2d", [0], {"kernel_h": 3, "kernel_w": 3, "pad_h": 1, "pad_w": 1, "out_features": 4},
                      None),
                _Node(2, "relu", [1], {}, None), _Node(3, "global_avgpool2d", [2], {}, None),
                _Node(4, "reshape", [3], {}, None), _Node(5, "dense", [4], {"out_features": 5}, None)],
               [5], 2, "tiny")
    enc = F.create_graph_encoding(g)
    assert enc.num_nodes == 5 and enc.edges == [(0, 1), (1, 2), (2, 3), (3, 4)]
    st = F.static_features(g)
    assert st.macs == 2 * 4 * 8 * 8 * 3 * 9 + 2 * 4 * 5 and st.t_conv == 1 and st.t_relu == 1 and st.t_dense == 1
    assert F.static_features(g, batch_size=4).macs == 2 * st.macs
    with pytest.raises(E.MalformedDocument):
        F.create_graph_encoding("{")
    with pytest.raises(E.EmptyGraph):
        F.create_graph_encoding(json.dumps({"batch": 1, "outputs": [0],
                                            "nodes": [{"id": 0, "op": "const", "out_shape": [1]}]}))


@pytest.mark.gpu
def test_predict_documents_end_to_end_vs_oracle(gf):
    """graph JSON -> native featuriser -> B200 forward + MIG, against the CPU oracle
    on the same documents (fp32 tolerance of DESIGN.md §4; MIG codes equal)."""
    from oracle import dippm_oracle as O
    from paper_2303_11733_b200 import gnn
    docs = [d for d, e, b in zip(_docs(gf), gf["error"], gf["batch_override"]) if not str(e) and b == 0][:24]
    fb = F.featurize_documents(docs)
    norm = gnn.Normalizer.fit(np.abs(np.random.default_rng(0).normal(size=(64, 3))) * [3, 9000, 2] + 1,
                              fb.fs_vectors())
    model = gnn.create_model(hidden=64, seed=4, normalizer=norm)
    y, mig, names = F.predict_documents(model, docs)
    assert names == fb.names
    params = {k: np.array(v) for k, v in model.param_items()}
    nd = {"y_mean": norm.y_mean, "y_std": norm.y_std, "fs_mean": norm.fs_mean, "fs_std": norm.fs_std}
    for i in range(len(docs)):
        enc = fb.encoding(i)
        ref = O.predict(params, nd, enc.num_nodes, enc.edges, enc.features, fb.fs_vectors()[i])
        assert np.all(np.abs(y[i] - ref) <= 1e-4 * np.abs(ref) + 1e-3), (i, y[i], ref)
        assert int(mig[i]) == O.mig_code(float(y[i, 1]))


@pytest.mark.gpu
def test_predict_documents_chunked_pipeline_identical():
    """predict_documents(chunk=k) overlaps featurisation with the device pass; every
    graph's prediction depends only on its own rows, so chunked and one-pass results agree
    to fp32 rounding (the readout's 32-row partial sums follow the global row alignment,
    which moves with the chunk: ulp-level differences), MIG codes equal, names in order."""
    from paper_2303_11733_b200 import gnn
    from paper_2303_11733_b200.synth import make_graph_documents
    docs = make_graph_documents(300, seed=77)
    fb = F.featurize_documents(docs)
    norm = gnn.Normalizer.fit(np.abs(np.random.default_rng(1).normal(size=(64, 3))) * [3, 9000, 2] + 1,
                              fb.fs_vectors())
    model = gnn.create_model(hidden=128, seed=2, normalizer=norm)
    for prec in ("bf16", "fp32"):
        y1, m1, n1 = F.predict_documents(model, docs, precision=prec)
        y2, m2, n2 = F.predict_documents(model, docs, precision=prec, chunk=64)
        assert n1 == n2 == fb.names
        np.testing.assert_allclose(y1, y2, rtol=2e-6, atol=0)
        np.testing.assert_array_equal(m1, m2)
