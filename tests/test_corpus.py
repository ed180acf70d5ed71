"""§8f row 2 — dataset storage: the JSONL interchange format against lines the
reference wrote (tests/golden/make_golden_next.py, dataset.py:255-343), and the
binary columnar sidecar (round trip, zero-copy collation equal to collating the
records, error behaviour).  The GPU test checks that a sidecar batch trains
exactly like the same records through the per-record API."""

import numpy as np
import pytest

from conftest import unpack_records
from paper_2303_11733_b200 import corpus
from paper_2303_11733_b200.device import collate_host, group_edges
from paper_2303_11733_b200.errors import IoFailure, MalformedRecord


def _ref_lines(gn):
    return bytes(gn["jsonl_bytes"]).decode("utf-8").splitlines()


def test_jsonl_reader_matches_reference_records(golden, golden_next):
    recs = [corpus.record_from_line(line, i + 1) for i, line in enumerate(_ref_lines(golden_next))]
    ref = unpack_records(golden)[:len(recs)]
    fs_int = golden["rec_fs_int"]
    for i, (r, (n, e, x, fs, y)) in enumerate(zip(recs, ref)):
        assert r.encoding.num_nodes == n and list(r.encoding.edges) == e
        assert np.array_equal(r.encoding.features, x)
        assert [r.fs.macs, r.fs.batch, r.fs.t_conv, r.fs.t_dense, r.fs.t_relu] == fs_int[i].tolist()
        assert np.array_equal(r.fs.as_vector, fs)
        assert np.array_equal(r.target.as_array, y)


def test_jsonl_writer_reproduces_reference_lines(golden_next):
    lines = _ref_lines(golden_next)
    recs = [corpus.record_from_line(line) for line in lines]
    assert [corpus.record_to_line(r) for r in recs] == lines  # byte-identical interchange


def test_jsonl_validation_errors(tmp_path):
    with pytest.raises(MalformedRecord):
        corpus.record_from_line("{not json")
    with pytest.raises(MalformedRecord):
        corpus.record_from_line('{"name": "a"}')
    good = '{"name": "a", "x": [[0.0] * 32], "edges": [], "n": 1, "fs": [0, 0, 0, 0, 0], ' \
           '"fs_raw": {"macs": 1, "batch": 1, "t_conv": 0, "t_dense": 0, "t_relu": 0}, ' \
           '"y": {"latency_ms": 1.0, "memory_mb": 2.0, "energy_j": 3.0}}'
    good = good.replace("[[0.0] * 32]", "[[" + ", ".join(["0.0"] * 32) + "]]")
    assert corpus.record_from_line(good).encoding.num_nodes == 1
    with pytest.raises(MalformedRecord):
        corpus.record_from_line(good.replace('"edges": []', '"edges": [[0, 3]]'))
    with pytest.raises(MalformedRecord):
        corpus.record_from_line(good.replace('"energy_j": 3.0', '"energy_j": -3.0'))
    with pytest.raises(IoFailure):
        corpus.read_jsonl(tmp_path / "missing.jsonl")


def test_corpus_round_trip_and_collate(tmp_path, golden_next):
    path = tmp_path / "d.jsonl"
    path.write_text("\n".join(_ref_lines(golden_next)) + "\n")
    recs = corpus.read_jsonl(path)
    bpath = tmp_path / "d.dippmbin"
    assert corpus.jsonl_to_corpus(path, bpath) == len(recs)
    c = corpus.Corpus(bpath)
    assert len(c) == len(recs) and c.num_nodes == sum(r.encoding.num_nodes for r in recs)
    back = c.records()
    for a, b in zip(recs, back):
        assert a.encoding.num_nodes == b.encoding.num_nodes and list(a.encoding.edges) == list(b.encoding.edges)
        assert np.array_equal(a.encoding.features.astype(np.float32), b.encoding.features.astype(np.float32))
        assert a.fs == b.fs and a.target == b.target and a.model_name == b.model_name
    ids = [5, 0, 7, 3]
    x, src, dst, gp, fs, y, ep = c.collate(ids)
    sel = [recs[i] for i in ids]
    rx, rsrc, rdst, rgp, rfs, ry = collate_host([r.encoding for r in sel], [r.fs.as_vector for r in sel],
                                                [r.target.as_array for r in sel])
    for a, b in ((x, rx), (src, rsrc), (dst, rdst), (gp, rgp), (fs, rfs), (y, ry)):
        assert np.array_equal(a, b)
    assert np.array_equal(ep, group_edges(rsrc, rdst, rgp))


def test_corpus_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.dippmbin"
    p.write_bytes(b"NOTDIPPM" + b"\0" * 100)
    with pytest.raises(IoFailure):
        corpus.Corpus(p)
    p.write_bytes(b"DIP")
    with pytest.raises(IoFailure):
        corpus.Corpus(p)


@pytest.mark.gpu
def test_corpus_batch_trains_like_records(tmp_path, golden_next):
    import torch
    from paper_2303_11733_b200 import gnn
    from paper_2303_11733_b200.trainer import BatchTrainer
    lines = _ref_lines(golden_next)
    recs = [corpus.record_from_line(line) for line in lines]
    corpus.write_corpus(recs, tmp_path / "c.dippmbin")
    c = corpus.Corpus(tmp_path / "c.dippmbin")
    norm = gnn.Normalizer.fit(c.y.astype(np.float64), c.fs.astype(np.float64))
    model = gnn.create_model(hidden=64, seed=2, normalizer=norm)
    ids = np.arange(len(c))
    a = BatchTrainer(model, precision="fp32", dropout=False)
    la = a.step_host(*[torch.from_numpy(np.ascontiguousarray(v)) for v in c.collate(ids)])
    b = BatchTrainer(model, precision="fp32", dropout=False)
    arrs = collate_host([r.encoding for r in recs], [r.fs.as_vector for r in recs], [r.target.as_array for r in recs])
    lb = b.step_host(*arrs)
    assert la == lb
    assert torch.equal(a.engine.params, b.engine.params)
