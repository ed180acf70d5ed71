"""Host collation of reference-style encodings (device.collate_host, gnn.py:140-154 validation):
list-of-pairs and ndarray edge lists give the same arrays, and the reference's errors are
raised (EmptyGraph for N < 1, ShapeMismatch for a non-(N, 32) feature matrix or an endpoint
outside [0, N)).  CPU only."""
import numpy as np
import pytest

from paper_2303_11733_b200.device import collate_host
from paper_2303_11733_b200.errors import EmptyGraph, ShapeMismatch
from paper_2303_11733_b200.types import GraphEncoding


def _enc(n, edges, rng):
    return GraphEncoding(num_nodes=n, edges=edges, features=rng.normal(size=(n, 32)))


def test_list_and_array_edges_collate_identically():
    rng = np.random.default_rng(0)
    encs, fss = [], []
    for g in range(9):
        n = int(rng.integers(1, 40))
        e = rng.integers(0, n, size=(int(rng.integers(0, 60)), 2))
        encs.append(_enc(n, [tuple(map(int, p)) for p in e], rng))
        fss.append(rng.normal(size=5))
    x, src, dst, gp, fs, y = collate_host(encs, fss, [np.arange(3.0)] * 9)
    encs2 = [GraphEncoding(num_nodes=e.num_nodes, edges=np.asarray(e.edges, np.int64).reshape(-1, 2),
                           features=e.features) for e in encs]
    x2, src2, dst2, gp2, fs2, y2 = collate_host(encs2, fss, [np.arange(3.0)] * 9)
    for a, b in ((x, x2), (src, src2), (dst, dst2), (gp, gp2), (fs, fs2), (y, y2)):
        assert np.array_equal(a, b)
    # reference layout: graph g's nodes at gp[g]..gp[g+1], endpoints offset by gp[g], f32 features
    assert x.dtype == np.float32 and src.dtype == np.int64 and gp.dtype == np.int32
    off = 0
    for g, e in enumerate(encs):
        ee = np.asarray(e.edges, np.int64).reshape(-1, 2)
        assert np.array_equal(src[off:off + len(ee)], ee[:, 0] + gp[g])
        assert np.allclose(x[gp[g]:gp[g + 1]], e.features.astype(np.float32))
        off += len(ee)


def test_collate_errors():
    rng = np.random.default_rng(1)
    ok = _enc(4, [(0, 1), (2, 3)], rng)
    with pytest.raises(EmptyGraph):
        collate_host([ok, GraphEncoding(num_nodes=0, edges=[], features=np.zeros((0, 32)))], [np.zeros(5)] * 2)
    with pytest.raises(ShapeMismatch):
        collate_host([GraphEncoding(num_nodes=3, edges=[], features=np.zeros((3, 31)))], [np.zeros(5)])
    for bad in ([(0, 4)], [(4, 0)], [(-1, 0)]):
        with pytest.raises(ShapeMismatch):
            collate_host([ok, _enc(4, bad, rng)], [np.zeros(5)] * 2)
