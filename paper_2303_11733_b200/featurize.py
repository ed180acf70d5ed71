"""Native front end in front of the B200 hot path — §8f row 1.

Turns graph JSON documents (the reference's graph schema, graph_ir.py:8-27)
into the GraphSAGE inputs: the operator-graph encoding (featurize.py:106-190)
and the static features (featurize.py:204-267).  The work runs in
libdippm_host.so (C++17, include/dippm_host.h) on all host cores, bit-identical
to the reference's Python front end (tests/test_featurize_native.py pins it to
reference outputs), and the batched call returns arrays already in the layout
`device.upload_batch` takes — graph JSON to HBM without per-node Python.

Drop-in names: `create_graph_encoding(graph)` and `static_features(graph)`
accept a JSON document (str/bytes) or a reference ComputationGraph object
(serialised to its canonical JSON first, graph_ir.serialize_graph
semantics); errors are the reference's exception classes.
"""

from __future__ import annotations

import ctypes as C
import json
import math
from pathlib import Path

import numpy as np

from . import errors as E
from .types import FEATURE_WIDTH, STATIC_WIDTH, GraphEncoding, StaticFeatures

HOST_LIB = Path(__file__).resolve().parent / "libdippm_host.so"
HOST_ABI_VERSION = 2

_STATUS = {1: E.MalformedDocument, 2: E.CyclicGraph, 3: E.DanglingReference, 4: E.BadShape, 5: E.ShapeMismatch,
           6: E.Underspecified, 7: E.EmptyGraph, 8: E.InvalidSpec, 9: ValueError, 10: OverflowError}
_lib = None


def _host():
    global _lib
    if _lib is None:
        if not HOST_LIB.exists():
            raise E.DippmError(f"{HOST_LIB.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(str(HOST_LIB))
        P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "dippm_host_abi_version": (I32, []),
            "dippm_featurize_docs": (P, [P, P, I64, P, I32]),
            "dippm_feat_count": (I64, [P]),
            "dippm_feat_status": (I32, [P, I64, C.c_char_p, I64]),
            "dippm_feat_name": (I64, [P, I64, C.c_char_p, I64]),
            "dippm_feat_sizes": (None, [P, P, P, P, P]),
            "dippm_feat_export": (None, [P, P, P, P, P]),
            "dippm_feat_free": (None, [P]),
            "dippm_feat_meta": (I64, [P, P, P, P, C.c_char_p, I64]),
            "dippm_feat_collate": (None, [P, P, P, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        if lib.dippm_host_abi_version() != HOST_ABI_VERSION:
            raise E.DippmError(f"{HOST_LIB.name} ABI mismatch; rebuild it")
        _lib = lib
    return _lib


def _as_bytes(doc) -> bytes:
    if isinstance(doc, bytes):
        return doc
    if isinstance(doc, str):
        return doc.encode("utf-8")
    return graph_to_json(doc).encode("utf-8")


def graph_to_json(graph) -> str:
    """A reference ComputationGraph (duck-typed) as its canonical JSON (graph_ir.py:326-350)."""
    doc = {"name": graph.name, "batch": graph.batch_size, "outputs": list(graph.outputs), "nodes": []}
    for node in graph.nodes:
        entry = {"id": node.id, "op": node.raw_name, "inputs": list(node.inputs),
                 "attrs": {k: node.attrs[k] for k in sorted(node.attrs)}}
        if node.out_shape is not None:
            entry["out_shape"] = list(node.out_shape)
        doc["nodes"].append(entry)
    return json.dumps(doc)


class FeaturizedBatch:
    """Result of featurising many documents in one native call.

    status[i] (0 = ok, else the reference exception, see `error(i)`), names[i],
    n[i] / ne[i] node and edge counts, x [sum n, 32] float64 feature rows,
    edges [sum ne, 2] graph-local (src, dst), fs_int [G, 5] (macs, batch,
    t_conv, t_dense, t_relu)."""

    def __init__(self, docs, batch_sizes=None, threads: int = 0, x32: bool = False):
        lib = _host()
        blobs = [_as_bytes(d) for d in docs]
        G = len(blobs)
        ptrs = (C.c_char_p * max(G, 1))(*blobs)
        lens = np.array([len(b) for b in blobs], dtype=np.int64)
        bo = None if batch_sizes is None else np.ascontiguousarray(batch_sizes, dtype=np.int64)
        if bo is not None and bo.shape != (G,):
            raise E.ShapeMismatch(f"{len(bo)} batch sizes for {G} documents")
        h = lib.dippm_featurize_docs(C.cast(ptrs, C.c_void_p), lens.ctypes.data if G else None, G,
                                     None if bo is None else bo.ctypes.data, int(threads))
        if not h:
            raise MemoryError("dippm_featurize_docs: allocation failed")
        self._h = h  # kept until the object dies: the float64 rows are exported on first use
        self.n = np.zeros(G, np.int64)
        self.ne = np.zeros(G, np.int64)
        tn, te = C.c_int64(0), C.c_int64(0)
        lib.dippm_feat_sizes(h, self.n.ctypes.data, self.ne.ctypes.data, C.byref(tn), C.byref(te))
        self._x = None
        self.x32 = np.empty((tn.value, FEATURE_WIDTH), np.float32) if x32 else None
        self.edges = np.empty((te.value, 2), np.int64)
        self.fs_int = np.zeros((G, STATIC_WIDTH), np.int64)
        lib.dippm_feat_export(h, None, self.edges.ctypes.data, self.fs_int.ctypes.data,
                              None if self.x32 is None else self.x32.ctypes.data)
        self.status = np.zeros(G, np.int32)
        self._fs_log = np.zeros((G, STATIC_WIDTH), np.float64)
        name_off = np.zeros(G + 1, np.int64)
        nbytes = lib.dippm_feat_meta(h, None, None, None, None, 0)
        buf = C.create_string_buffer(max(int(nbytes), 1))
        lib.dippm_feat_meta(h, self.status.ctypes.data, self._fs_log.ctypes.data, name_off.ctypes.data, buf,
                            int(nbytes))
        raw = buf.raw[:nbytes]
        self.names = [raw[name_off[i]:name_off[i + 1]].decode("utf-8") for i in range(G)]
        msg = C.create_string_buffer(512)
        self.messages = [""] * G
        for i in np.nonzero(self.status)[0]:  # messages only for the documents that failed
            lib.dippm_feat_status(h, int(i), msg, 512)
            self.messages[int(i)] = msg.value.decode("utf-8", "replace")
        self.node_ptr = np.zeros(G + 1, np.int64)
        np.cumsum(self.n, out=self.node_ptr[1:])
        self.edge_ptr = np.zeros(G + 1, np.int64)
        np.cumsum(self.ne, out=self.edge_ptr[1:])

    def __len__(self) -> int:
        return len(self.n)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.dippm_feat_free(h)

    @property
    def x(self) -> np.ndarray:
        """[sum n, 32] float64 feature rows (exported from the native batch on first use)."""
        if self._x is None:
            self._x = np.empty((int(self.n.sum()), FEATURE_WIDTH), np.float64)
            _host().dippm_feat_export(self._h, self._x.ctypes.data, None, None, None)
        return self._x

    def error(self, i: int):
        """The exception the reference raises for document i (None if it featurised)."""
        st = int(self.status[i])
        return None if st == 0 else _STATUS.get(st, E.DippmError)(self.messages[i])

    def raise_first_error(self) -> None:
        bad = np.nonzero(self.status)[0]
        if len(bad):
            raise self.error(int(bad[0]))

    def fs_vectors(self) -> np.ndarray:
        """StaticFeatures.as_vector for every document (libm log1p of the integers, float64)."""
        return self._fs_log

    def encoding(self, i: int) -> GraphEncoding:
        self.raise_if(i)
        a, b = self.node_ptr[i], self.node_ptr[i + 1]
        ea, eb = self.edge_ptr[i], self.edge_ptr[i + 1]
        return GraphEncoding(num_nodes=int(b - a), edges=[(int(s), int(d)) for s, d in self.edges[ea:eb]],
                             features=self.x[a:b].copy())

    def static(self, i: int) -> StaticFeatures:
        self.raise_if(i)
        return StaticFeatures(*[int(v) for v in self.fs_int[i]])

    def raise_if(self, i: int) -> None:
        err = self.error(i)
        if err is not None:
            raise err

    def collate(self):
        """(x f32, src, dst, graph_ptr, fs f64, edge_ptr) over all documents, node ids
        batch-global — the arrays device.upload_batch takes.  Raises the first error."""
        self.raise_first_error()
        x = self.x32 if self.x32 is not None else self.x.astype(np.float32)  # noqa: E501
        gp = self.node_ptr.astype(np.int32)
        off = np.repeat(self.node_ptr[:-1], self.ne)
        src = self.edges[:, 0] + off
        dst = self.edges[:, 1] + off
        return x, src, dst, gp, self.fs_vectors().astype(np.float64), self.edge_ptr

    def collate_pinned(self):
        """collate() written by the native library straight into pinned host tensors
        (dippm_feat_collate, multi-threaded): the same arrays, ready for asynchronous
        host->device copies.  The buffers come from torch's caching pinned allocator, so
        steady-state calls reuse them once their copies have completed."""
        import torch
        self.raise_first_error()
        G, N, E = len(self), int(self.node_ptr[-1]), int(self.edge_ptr[-1])

        def pinned(shape, dt):
            return torch.empty(shape, dtype=dt, pin_memory=True)
        x = pinned((N, FEATURE_WIDTH), torch.float32)
        src, dst = pinned((E,), torch.int64), pinned((E,), torch.int64)
        gp, ep = pinned((G + 1,), torch.int32), pinned((G + 1,), torch.int64)
        fs = pinned((G, STATIC_WIDTH), torch.float64)
        _host().dippm_feat_collate(self._h, x.data_ptr(), src.data_ptr(), dst.data_ptr(), gp.data_ptr(),
                                   ep.data_ptr(), fs.data_ptr())
        return x, src, dst, gp, fs, ep


def featurize_documents(docs, batch_sizes=None, threads: int = 0, x32: bool = True) -> FeaturizedBatch:
    """Featurise many graph documents in one native, multi-threaded call."""
    return FeaturizedBatch(docs, batch_sizes, threads, x32)


def create_graph_encoding(graph, batch_size: int | None = None) -> GraphEncoding:
    """featurize.create_graph_encoding (featurize.py:186-190) of a document or graph object."""
    fb = FeaturizedBatch([graph], None if batch_size is None else [batch_size], threads=1)
    return fb.encoding(0)


def static_features(graph, batch_size: int | None = None) -> StaticFeatures:
    """featurize.static_features (featurize.py:256-267) of a document or graph object."""
    fb = FeaturizedBatch([graph], None if batch_size is None else [batch_size], threads=1)
    return fb.static(0)


def predict_documents(model, docs, batch_sizes=None, precision: str = "fp32", threads: int = 0,
                      chunk: int = 0, info: dict | None = None):
    """The `dippm predict` path (cli.py:148-172) for many documents at once:
    native featurisation, one device pass (gnn.predict_batch semantics).
    Returns (y float64 [G, 3] latency_ms / memory_mb / energy_j, MIG codes int8 [G], names).

    chunk > 0 splits the documents into chunks of that many and pipelines them: the native
    featuriser (which runs outside the GIL) works on chunk k+1 while chunk k is collated,
    uploaded and run on the device.  Every graph's prediction is independent of the others
    in its batch, so the results are identical to the one-pass call; the first failing
    document raises the same exception."""
    if chunk <= 0 or len(docs) <= chunk:
        fb = featurize_documents(docs, batch_sizes, threads)
        y, mig = predict_featurized(model, fb, precision, info=info)
        return y, mig, fb.names
    from concurrent.futures import ThreadPoolExecutor
    spans = [(a, min(a + chunk, len(docs))) for a in range(0, len(docs), chunk)]

    def feat(span):
        a, b = span
        return featurize_documents(docs[a:b], None if batch_sizes is None else batch_sizes[a:b], threads)

    def feat_collate(span):
        fb = feat(span)
        return fb, fb.collate_pinned()

    from . import gnn
    eng = gnn._engine(model, precision)  # the model cannot change during the call: refresh once
    ys, migs, names = [], [], []
    with ThreadPoolExecutor(1) as ex:
        ahead = ex.submit(feat_collate, spans[0])
        for k in range(len(spans)):
            fb, arrays = ahead.result()
            if k + 1 < len(spans):
                ahead = ex.submit(feat_collate, spans[k + 1])
            y, mig = predict_featurized(model, fb, precision, arrays, eng, info=info)
            ys.append(y)
            migs.append(mig)
            names += fb.names
    return np.concatenate(ys), np.concatenate(migs), names


def predict_featurized(model, fb: FeaturizedBatch, precision: str = "fp32", arrays=None, eng=None,
                       info: dict | None = None):
    """Device half of predict_documents: one forward over an already featurised batch
    (`arrays` = its collate_pinned() output when already made; `eng` = the model's engine
    when the caller already refreshed it for this call)."""
    import torch

    from . import gnn
    from .device import upload_batch
    x, src, dst, gp, fs, ep = fb.collate_pinned() if arrays is None else arrays
    if eng is None:
        eng = gnn._engine(model, precision)
    b = upload_batch(x, src, dst, gp, fs, None, device=eng.device, build_csr=eng.arch == "sage", edge_ptr=ep)
    ws = gnn.infer_workspace(eng, b.N, b.G)
    eng.forward(b, ws)
    n_band = gnn.mig_rescore(model, eng, b, ws, precision)  # bf16: fp32 picks near the ceilings
    if info is not None:
        info["mig_rescored"] = info.get("mig_rescored", 0) + n_band
    y, mig, nf = gnn._readback(ws.y_pred[:b.G], ws.mig[:b.G], ws.nonfinite)
    if int(nf[0]):
        raise E.NonFinite("memory prediction is not finite")
    return y, mig
