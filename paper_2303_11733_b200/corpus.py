"""Dataset storage for the B200 path — §8f row 2.

The reference keeps datasets as JSON Lines (dataset.py:255-343): one record
per line, ~81 KB per 300-node graph, parsed record by record into Python
objects.  This module keeps JSONL as the interchange format (reader/writer
with the reference's validation and error types) and adds a binary columnar
sidecar that maps straight onto the device batch layout:

  header   64 B   magic b"DIPPMBIN", version, G, N, E, metadata length
  meta     JSON   {"vocab_version", "names"}
  node_ptr int64  [G+1]     graph g owns node rows node_ptr[g]..node_ptr[g+1]
  edge_ptr int64  [G+1]     and edge rows edge_ptr[g]..edge_ptr[g+1]
  x        f32    [N, 32]   node features (the device computes in fp32; the
                            JSONL path casts the same way before upload)
  edges    int32  [E, 2]    (src, dst), graph-local ids, featurizer order
  fs_raw   int64  [G, 5]    macs, batch, t_conv, t_dense, t_relu
  fs       f64    [G, 5]    log1p(fs_raw) exactly as StaticFeatures.as_vector
  y        f64    [G, 3]    latency_ms, memory_mb, energy_j
  (every column 64-byte aligned; the file is read with np.memmap, zero copy)

`Corpus.collate(ids)` returns the arrays `device.upload_batch` takes (node ids
made batch-global, `edge_ptr` for the per-graph CSR kernel), so a batch goes
from disk to HBM with one gather on the host and no per-record objects.
"""

from __future__ import annotations

import json
import math
import struct
from pathlib import Path

import numpy as np

from .errors import IoFailure, MalformedRecord
from .types import (FEATURE_WIDTH, STATIC_WIDTH, VOCAB_VERSION, DatasetRecord, GraphEncoding, StaticFeatures,
                    TargetVector)

MAGIC = b"DIPPMBIN"
VERSION = 1
_HDR = struct.Struct("<8sIIQQQQ16x")  # magic, version, reserved, G, N, E, meta_len -> 64 bytes
_ALIGN = 64


# ---------------------------------------------------------------------------
# JSONL (dataset.py:255-343)

def record_to_line(record) -> str:
    """dataset.py:255-281 (same keys and value formatting via json.dumps)."""
    enc, fs, t = record.encoding, record.fs, record.target
    doc = {
        "name": getattr(record, "model_name", ""),
        "x": np.asarray(enc.features, dtype=np.float64).tolist(),
        "edges": [[int(s), int(d)] for s, d in enc.edges],
        "n": int(enc.num_nodes),
        "fs": np.asarray(fs.as_vector, dtype=np.float64).tolist(),
        "fs_raw": {"macs": fs.macs, "batch": fs.batch, "t_conv": fs.t_conv, "t_dense": fs.t_dense,
                   "t_relu": fs.t_relu},
        "y": {"latency_ms": t.latency_ms, "memory_mb": t.memory_mb, "energy_j": t.energy_j},
    }
    return json.dumps(doc)


def record_from_line(line: str, lineno: int = 0) -> DatasetRecord:
    """dataset.py:284-326: parse + validate one JSONL line (MalformedRecord on any defect)."""
    where = f"line {lineno}" if lineno else "record"
    try:
        doc = json.loads(line)
    except json.JSONDecodeError as exc:
        raise MalformedRecord(f"{where}: invalid JSON: {exc}") from exc
    if not isinstance(doc, dict):
        raise MalformedRecord(f"{where}: expected an object")
    for key in ("name", "x", "edges", "n", "fs", "fs_raw", "y"):
        if key not in doc:
            raise MalformedRecord(f'{where}: missing "{key}" field')
    try:
        features = np.asarray(doc["x"], dtype=np.float64)
        if features.ndim == 1 and features.size == 0:
            features = features.reshape(0, FEATURE_WIDTH)
        encoding = GraphEncoding(num_nodes=int(doc["n"]), edges=[(int(s), int(d)) for s, d in doc["edges"]],
                                 features=features)
        raw = doc["fs_raw"]
        fs = StaticFeatures(macs=int(raw["macs"]), batch=int(raw["batch"]), t_conv=int(raw["t_conv"]),
                            t_dense=int(raw["t_dense"]), t_relu=int(raw["t_relu"]))
        y = doc["y"]
        target = TargetVector(latency_ms=float(y["latency_ms"]), memory_mb=float(y["memory_mb"]),
                              energy_j=float(y["energy_j"]))
    except (KeyError, TypeError, ValueError) as exc:
        raise MalformedRecord(f"{where}: {exc}") from exc
    if encoding.num_nodes != encoding.features.shape[0] or (
            encoding.num_nodes and encoding.features.shape[1] != FEATURE_WIDTH):
        raise MalformedRecord(f"{where}: feature matrix does not match node count")
    for src, dst in encoding.edges:
        if not (0 <= src < encoding.num_nodes and 0 <= dst < encoding.num_nodes):
            raise MalformedRecord(f"{where}: edge ({src}, {dst}) out of range")
    if len(doc["fs"]) != STATIC_WIDTH:
        raise MalformedRecord(f"{where}: fs vector must have {STATIC_WIDTH} entries")
    for value in (target.latency_ms, target.memory_mb, target.energy_j):
        if not math.isfinite(value) or value <= 0:
            raise MalformedRecord(f"{where}: target values must be finite and positive")
    return DatasetRecord(encoding=encoding, fs=fs, target=target, model_name=str(doc["name"]))


def write_jsonl(records, path) -> None:
    """dataset.py:329-336."""
    try:
        with open(path, "w", encoding="utf-8") as fh:
            for record in records:
                fh.write(record_to_line(record))
                fh.write("\n")
    except OSError as exc:
        raise IoFailure(f"cannot write dataset to {path}: {exc}") from exc


def read_jsonl(path) -> list:
    """dataset.py:339-343."""
    try:
        text = Path(path).read_text(encoding="utf-8")
    except OSError as exc:
        raise IoFailure(f"cannot read dataset from {path}: {exc}") from exc
    return [record_from_line(line, i) for i, line in enumerate(text.splitlines(), start=1) if line.strip()]


# ---------------------------------------------------------------------------
# binary sidecar

def _columns(G: int, N: int, E: int):
    return [("node_ptr", np.int64, (G + 1,)), ("edge_ptr", np.int64, (G + 1,)), ("x", np.float32, (N, FEATURE_WIDTH)),
            ("edges", np.int32, (E, 2)), ("fs_raw", np.int64, (G, STATIC_WIDTH)),
            ("fs", np.float64, (G, STATIC_WIDTH)), ("y", np.float64, (G, 3))]


def _aligned(n: int) -> int:
    return -(-n // _ALIGN) * _ALIGN


def write_corpus(records, path) -> None:
    """Write DatasetRecord-like objects as a binary sidecar (see module docstring)."""
    recs = list(records)
    G = len(recs)
    n = np.array([int(r.encoding.num_nodes) for r in recs], dtype=np.int64)
    ne = np.array([len(r.encoding.edges) for r in recs], dtype=np.int64)
    node_ptr = np.zeros(G + 1, np.int64)
    edge_ptr = np.zeros(G + 1, np.int64)
    np.cumsum(n, out=node_ptr[1:])
    np.cumsum(ne, out=edge_ptr[1:])
    N, E = int(node_ptr[-1]), int(edge_ptr[-1])
    cols = {
        "node_ptr": node_ptr, "edge_ptr": edge_ptr,
        "x": (np.concatenate([np.asarray(r.encoding.features, np.float64).reshape(-1, FEATURE_WIDTH) for r in recs])
              if G else np.zeros((0, FEATURE_WIDTH))).astype(np.float32),
        "edges": (np.asarray([e for r in recs for e in r.encoding.edges], np.int64).reshape(-1, 2)).astype(np.int32),
        "fs_raw": np.array([[r.fs.macs, r.fs.batch, r.fs.t_conv, r.fs.t_dense, r.fs.t_relu] for r in recs],
                           dtype=np.int64).reshape(G, STATIC_WIDTH),
        "fs": np.array([np.asarray(r.fs.as_vector, np.float64) for r in recs]).reshape(G, STATIC_WIDTH),
        "y": np.array([[r.target.latency_ms, r.target.memory_mb, r.target.energy_j] for r in recs],
                      dtype=np.float64).reshape(G, 3),
    }
    meta = json.dumps({"vocab_version": VOCAB_VERSION,
                       "names": [str(getattr(r, "model_name", "")) for r in recs]}).encode("utf-8")
    try:
        with open(path, "wb") as fh:
            fh.write(_HDR.pack(MAGIC, VERSION, 0, G, N, E, len(meta)))
            fh.write(meta)
            fh.write(b"\0" * (_aligned(_HDR.size + len(meta)) - _HDR.size - len(meta)))
            for name, dt, shape in _columns(G, N, E):
                a = np.ascontiguousarray(cols[name], dtype=dt).reshape(shape)
                b = a.tobytes()
                fh.write(b)
                fh.write(b"\0" * (_aligned(len(b)) - len(b)))
    except OSError as exc:
        raise IoFailure(f"cannot write corpus to {path}: {exc}") from exc


def jsonl_to_corpus(jsonl_path, corpus_path) -> int:
    """Convert a reference JSONL dataset to the binary sidecar; returns the record count."""
    recs = read_jsonl(jsonl_path)
    write_corpus(recs, corpus_path)
    return len(recs)


class Corpus:
    """A memory-mapped binary sidecar: columns as zero-copy numpy views."""

    def __init__(self, path):
        self.path = Path(path)
        try:
            raw = np.memmap(self.path, dtype=np.uint8, mode="r")
        except (OSError, ValueError) as exc:
            raise IoFailure(f"cannot read corpus {path}: {exc}") from exc
        if raw.size < _HDR.size:
            raise IoFailure(f"corpus {path} is truncated (no header)")
        magic, version, _, G, N, E, meta_len = _HDR.unpack(bytes(raw[:_HDR.size]))
        if magic != MAGIC:
            raise IoFailure(f"{path} is not a DIPPM corpus (bad magic)")
        if version != VERSION:
            raise IoFailure(f"corpus {path} has format version {version}, expected {VERSION}")
        try:
            self.meta = json.loads(bytes(raw[_HDR.size:_HDR.size + meta_len]).decode("utf-8"))
        except ValueError as exc:
            raise IoFailure(f"corpus {path}: bad metadata: {exc}") from exc
        off = _aligned(_HDR.size + meta_len)
        for name, dt, shape in _columns(G, N, E):
            nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
            if off + nbytes > raw.size:
                raise IoFailure(f"corpus {path} is truncated (column {name})")
            setattr(self, name, raw[off:off + nbytes].view(dt).reshape(shape))
            off += _aligned(nbytes)
        self.num_graphs, self.num_nodes, self.num_edges = int(G), int(N), int(E)

    def __len__(self) -> int:
        return self.num_graphs

    @property
    def names(self) -> list:
        return self.meta.get("names", [])

    def collate(self, ids):
        """(x, src, dst, graph_ptr, fs, y, edge_ptr) for graphs `ids` — what device.upload_batch
        takes: node ids batch-global, edges grouped by graph (per-graph CSR kernel)."""
        ids = np.asarray(ids, dtype=np.int64)
        n = self.node_ptr[ids + 1] - self.node_ptr[ids]
        ne = self.edge_ptr[ids + 1] - self.edge_ptr[ids]
        gp = np.zeros(len(ids) + 1, np.int32)
        np.cumsum(n, out=gp[1:])
        ep = np.zeros(len(ids) + 1, np.int64)
        np.cumsum(ne, out=ep[1:])
        node_rows = np.concatenate([np.arange(self.node_ptr[g], self.node_ptr[g + 1]) for g in ids]) \
            if len(ids) else np.zeros(0, np.int64)
        edge_rows = np.concatenate([np.arange(self.edge_ptr[g], self.edge_ptr[g + 1]) for g in ids]) \
            if len(ids) else np.zeros(0, np.int64)
        x = self.x[node_rows]
        e = self.edges[edge_rows].astype(np.int64) + np.repeat(gp[:-1].astype(np.int64), ne)[:, None]
        return (x, e[:, 0].copy(), e[:, 1].copy(), gp, self.fs[ids].astype(np.float64), self.y[ids].astype(np.float64),
                ep)

    def records(self, ids=None) -> list:
        """DatasetRecord objects (for the drop-in per-record API)."""
        ids = range(self.num_graphs) if ids is None else ids
        out = []
        names = self.names
        for g in ids:
            g = int(g)
            a, b = int(self.node_ptr[g]), int(self.node_ptr[g + 1])
            ea, eb = int(self.edge_ptr[g]), int(self.edge_ptr[g + 1])
            enc = GraphEncoding(num_nodes=b - a, edges=[(int(s), int(d)) for s, d in self.edges[ea:eb]],
                                features=np.asarray(self.x[a:b], dtype=np.float64))
            fs = StaticFeatures(*[int(v) for v in self.fs_raw[g]])
            y = self.y[g]
            out.append(DatasetRecord(enc, fs, TargetVector(float(y[0]), float(y[1]), float(y[2])),
                                     model_name=names[g] if g < len(names) else ""))
        return out
