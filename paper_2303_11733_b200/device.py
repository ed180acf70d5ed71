"""Device engine: HBM layout, batch collation and the launch sequences of the
batched GraphSAGE forward / backward / Adam step over the C ABI.

PyTorch is used for device memory (caching allocator), streams and pinned
host buffers only; every FLOP runs in libdippm_b200.so.

HBM layout (hidden H padded to Hp = ceil64(H), rounded up for the SAGE layers to the next
width whose 8-column chunks tile a warp in the aggregation kernels -- 64, 128, 192, 256, 384,
512, 768, 1024 (agg_width); padded weights are zero and stay exactly zero under Adam, so
results equal the unpadded network):
  params  fp64 [P]   master weights, reference order gnn.py:488-491, with
                     sage{l}.w_self/w_neigh adjacent -> W_cat_l [2 d_l, Hp];
                     fc1.w padded to [Hp+64, Hp] (fs rows at Hp..Hp+4)
  m, v    fp64 [P]   Adam moments (numerics.py:76-90)
  grads   fp32 [P]   same offsets;  p32 fp32 [P] compute copy (biases, fc3)
  Wf[l]   [2 d_l, Hp]  W_cat natural layout: forward B operand, MN-major
  Wd[l]   [Hp, 2Hp]    [W_self | W_neigh] rows: dgrad B operand, K-major (l=2,3)
  W1h     [Hp+64, Hp], W2h [Hp, Hp]: head operands (FWD MN-major, dgrad K-major)
  (all GEMM copies in the compute dtype, refreshed inside the Adam kernel)
Per batch (N nodes, G graphs):
  A1 [N, 64]  = [X | agg X]        A2 [N, 2Hp] = [h1 | agg h1]
  A3 [N, 2Hp] = [h2 | agg h2]      H3 [N, Hp]  = h3
  u  [G, Hp+64] = [mean_g h3 | fs_norm | 0]   x2, x3 [G, Hp] head activations
  backward: Bl [N, 2Hp] = [dz_l | agg^T dz_l]  (two ping-pong buffers)
Node rows of a graph are contiguous (graph_ptr), edges carry global ids.
"""

from __future__ import annotations

import ctypes as C
import itertools
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import Act, GemmArgs, DT_BF16, DT_F32, DT_TF32X3, GEMM_FWD, GEMM_GATE, GEMM_STORE, GEMM_WGRAD
from .errors import EmptyGraph, ShapeMismatch

FEATURE_WIDTH = 32   # featurize.py:38
STATIC_WIDTH = 5     # featurize.py:39
PRECISIONS = {"fp32": DT_TF32X3, "bf16": DT_BF16}
# the whole FC head in one cooperative launch (head_fused.cu) for bf16 batches of up to
# dippm_head_fused_max_graphs() graphs; DIPPM_FUSED_HEAD=0 keeps the per-op launches
FUSED_HEAD = os.environ.get("DIPPM_FUSED_HEAD", "1") != "0"
# the readout's second stage as the fused head's phase 0 instead of its own launch: measured ~8 us
# slower per step (one graph per CTA, latency-bound, plus a grid barrier), so off unless asked for
HEAD_POOL = os.environ.get("DIPPM_HEAD_POOL", "0") == "1"
# the fused head's dW1 / dW2 as side-stream weight-gradient GEMMs (off the dgrad chain);
# DIPPM_HEAD_WGRAD_INLINE=1 keeps them inside the head kernel (A/B switch; the native step
# reads the same variable)
HEAD_WGRAD_DEFER = os.environ.get("DIPPM_HEAD_WGRAD_INLINE", "0") != "1"
BACKENDS = {"tc": 0, "simt": 1}


def _stream() -> int:
    # the raw cudaStream_t of the current stream: a direct C call (torch.cuda.current_stream()
    # re-validates the device through Python on every call, ~15 us, and a step makes ~20 calls)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def require_device(device=None) -> torch.device:
    _lib.load()
    if not torch.cuda.is_available():
        raise _lib.DeviceUnavailable("no CUDA device visible; the DIPPM B200 path has no CPU fallback")
    return torch.device(device if device is not None else "cuda")


_libc = C.CDLL(None)
_libc.memcmp.restype = C.c_int
_libc.memcmp.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]


def _same_bytes(a: np.ndarray, b: np.ndarray) -> bool:
    """Byte equality of two C-contiguous arrays (memcmp)."""
    return a.nbytes == b.nbytes and (a.nbytes == 0 or _libc.memcmp(a.ctypes.data, b.ctypes.data, a.nbytes) == 0)


def _p(t) -> int | None:
    return None if t is None else t.data_ptr()


class ActBuf:
    """[rows, cols] activation buffer in a compute dtype (bf16, tf32 hi/lo planes, or fp32)."""

    def __init__(self, rows: int, cols: int, dtype: int, device):
        self.rows, self.cols, self.dtype = rows, cols, dtype
        if dtype == DT_BF16:
            self.t = torch.empty(rows, cols, dtype=torch.bfloat16, device=device)
            self.elem, self.plane = 2, 0
        elif dtype == DT_TF32X3:
            self.t = torch.empty(2, rows, cols, dtype=torch.float32, device=device)
            self.elem, self.plane = 4, rows * cols
        else:
            self.t = torch.empty(rows, cols, dtype=torch.float32, device=device)
            self.elem, self.plane = 4, 0

    def view(self, col0: int = 0) -> Act:
        return Act(self.t.data_ptr() + col0 * self.elem, self.cols, self.plane, self.dtype)

    def to_float(self, col0: int = 0, width: int | None = None) -> torch.Tensor:
        width = self.cols - col0 if width is None else width
        if self.dtype == DT_TF32X3:
            return (self.t[0] + self.t[1])[:, col0:col0 + width].float()
        return self.t[:, col0:col0 + width].float()


def f32_act(t: torch.Tensor) -> Act:
    return Act(t.data_ptr(), t.shape[1], 0, DT_F32)


NULL_ACT = Act(None, 0, 0, 0)


ARCHS = ("sage", "mlp")


# widths the aggregation / pooling kernels take (csrc/aggregate.cu cpl_for): 8 * 2^k columns
# (1-128 chunks of 8) and 24 * 2^k columns (3-96 chunks, three per lane)
AGG_WIDTHS = tuple(sorted({8 << k for k in range(8)} | {24 << k for k in range(6)}))


def agg_width(d: int, align: int = 8) -> int:
    """Smallest width >= d (and >= align) that the aggregation kernels take and that is a
    multiple of align; beyond 1024 columns a multiple of 1024 (callers split the columns)."""
    d = max(int(d), align, 1)
    if d > 1024:
        return -(-d // 1024) * 1024
    return next(w for w in AGG_WIDTHS if w >= d and w % align == 0)


class Layout:
    """Flat parameter layout with hidden padded to a multiple of 64.

    arch "sage": DippmModel (gnn.py:178-233), fc1 input u = [mean h3 | fs_norm | 0];
    arch "mlp":  MlpModel (gnn.py:236-262), the static-features-only baseline,
                 fc1 input u = [fs_norm | 0] (64 wide, K-aligned).
    """

    def __init__(self, hidden: int, arch: str = "sage"):
        if arch not in ARCHS:
            raise ValueError(f"arch must be one of {ARCHS}, got {arch!r}")
        self.hidden, self.arch = hidden, arch
        # padded width: a multiple of 64 (tensor-core K blocks); for the SAGE layers also one whose
        # 8-column chunks tile a warp in the aggregation kernels (64, 128, 192, 256, 384, 512, 768,
        # 1024; a power of two beyond).  Padded weights are zero and stay zero, so results equal
        # the unpadded net.
        hp = -(-hidden // 64) * 64
        if arch == "sage":
            hp = agg_width(hp, 64) if hp <= 1024 else 1 << (hp - 1).bit_length()
        self.hp = hp
        self.d_in = [FEATURE_WIDTH, hp, hp] if arch == "sage" else []
        shapes = []
        for i, d in enumerate(self.d_in, start=1):
            shapes += [(f"sage{i}.w_self", (d, hp)), (f"sage{i}.w_neigh", (d, hp)), (f"sage{i}.bias", (hp,))]
        # [r | fs | 0] (sage) or [fs | 0] (mlp): K of fc1 aligned to the tensor-core k-block
        self.u_width = hp + 64 if arch == "sage" else 64
        self.fs_col = hp if arch == "sage" else 0
        shapes += [("fc1.w", (self.u_width, hp)), ("fc1.b", (hp,)), ("fc2.w", (hp, hp)), ("fc2.b", (hp,)),
                   ("fc3.w", (hp, 3)), ("fc3.b", (3,))]
        self.shapes = dict(shapes)
        self.offsets = {}
        off = 0
        for name, shp in shapes:
            self.offsets[name] = off
            off += int(np.prod(shp))
        self.total = off
        self.head_off = self.offsets["fc1.w"]

    def ref_shape(self, name: str):
        h = self.hidden
        if self.arch == "mlp":
            return {"fc1.w": (STATIC_WIDTH, h), "fc1.b": (h,), "fc2.w": (h, h), "fc2.b": (h,),
                    "fc3.w": (h, 3), "fc3.b": (3,)}[name]
        return {
            "sage1.w_self": (FEATURE_WIDTH, h), "sage1.w_neigh": (FEATURE_WIDTH, h), "sage1.bias": (h,),
            "sage2.w_self": (h, h), "sage2.w_neigh": (h, h), "sage2.bias": (h,),
            "sage3.w_self": (h, h), "sage3.w_neigh": (h, h), "sage3.bias": (h,),
            "fc1.w": (h + STATIC_WIDTH, h), "fc1.b": (h,), "fc2.w": (h, h), "fc2.b": (h,),
            "fc3.w": (h, 3), "fc3.b": (3,),
        }[name]

    def pad(self, name: str, arr: np.ndarray) -> np.ndarray:
        h, hp = self.hidden, self.hp
        out = np.zeros(self.shapes[name], dtype=np.float64)
        a = np.asarray(arr, dtype=np.float64)
        if a.shape != self.ref_shape(name):
            raise ShapeMismatch(f"parameter {name}: shape {a.shape}, expected {self.ref_shape(name)}")
        if name == "fc1.w":
            r = a.shape[0] - STATIC_WIDTH   # rows fed by the readout (0 for the MLP)
            out[:r, :h] = a[:r]
            out[self.fs_col:self.fs_col + STATIC_WIDTH, :h] = a[r:]
        elif a.ndim == 1:
            out[:a.shape[0]] = a
        else:
            out[:a.shape[0], :a.shape[1]] = a
        return out

    def unpad(self, name: str, padded: np.ndarray) -> np.ndarray:
        h, hp = self.hidden, self.hp
        shp = self.ref_shape(name)
        if name == "fc1.w":
            r = shp[0] - STATIC_WIDTH
            return np.concatenate([padded[:r, :h], padded[self.fs_col:self.fs_col + STATIC_WIDTH, :h]])
        if len(shp) == 1:
            return padded[:shp[0]].copy()
        return padded[:shp[0], :shp[1]].copy()

    def slice(self, flat: torch.Tensor, name: str) -> torch.Tensor:
        off = self.offsets[name]
        shp = self.shapes[name]
        return flat[off:off + int(np.prod(shp))].view(*shp)


# ---------------------------------------------------------------------------
# batches

@dataclass
class Batch:
    """A collated, device-resident batch of graphs plus its CSR."""
    G: int
    N: int
    E: int
    x: torch.Tensor          # f32 [N, 32]
    src: torch.Tensor        # i64 [E]
    dst: torch.Tensor        # i64 [E]
    graph_ptr: torch.Tensor  # i32 [G+1]
    fs: torch.Tensor         # f64 [G, 5] log1p static features
    y: torch.Tensor | None   # f64 [G, 3] raw targets
    rowptr: torch.Tensor | None = None
    col: torch.Tensor | None = None
    deg: torch.Tensor | None = None
    inv_deg: torch.Tensor | None = None
    t_rowptr: torch.Tensor | None = None
    t_col: torch.Tensor | None = None
    bad: torch.Tensor | None = None
    h2d_bytes: int = 0
    edge_ptr: torch.Tensor | None = None  # i64 [G+1] when edges are grouped by graph (fast CSR path)
    max_nodes: int = 0                    # largest graph (nodes / edges) for the per-graph CSR kernel
    max_edges: int = 0
    node_graph: torch.Tensor | None = None  # i32 [N] node -> graph id


def group_edges(src, dst, graph_ptr):
    """edge_ptr [G+1] if the edge list is a concatenation of per-graph edge lists
    (what collation produces), else None.  Host-side, O(E).

    Also the host validation of a collated batch (the reference builds each graph's
    aggregation matrix from its own edges, gnn.py:130-137): an endpoint outside
    [0, N) or an edge joining two graphs raises ShapeMismatch."""
    src, dst, gp = np.asarray(src), np.asarray(dst), np.asarray(graph_ptr, dtype=np.int64)
    G = len(gp) - 1
    if len(dst) == 0:
        return np.zeros(G + 1, np.int64)
    n = int(gp[-1])
    if min(int(src.min()), int(dst.min())) < 0 or max(int(src.max()), int(dst.max())) >= n:
        raise ShapeMismatch(f"edge endpoint outside [0, {n})")
    gd = np.searchsorted(gp, dst, side="right") - 1
    if np.any(np.searchsorted(gp, src, side="right") - 1 != gd):
        raise ShapeMismatch("edge joins two different graphs of the batch")
    if np.any(np.diff(gd) < 0):
        return None
    ep = np.zeros(G + 1, np.int64)
    np.cumsum(np.bincount(gd, minlength=G), out=ep[1:])
    return ep


def _edge_pairs(edges) -> np.ndarray:
    """[m, 2] int64 view of one graph's edge list: an ndarray as is, a list of (src, dst)
    pairs flattened with np.fromiter (~3x faster than np.asarray on a list of tuples)."""
    if isinstance(edges, np.ndarray):
        return edges.astype(np.int64, copy=False).reshape(-1, 2)
    m = len(edges)
    try:
        flat = np.fromiter(itertools.chain.from_iterable(edges), dtype=np.int64)
    except (TypeError, ValueError):
        flat = None
    if flat is None or flat.size != 2 * m:  # not a list of pairs: the general (slow) conversion
        return np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    return flat.reshape(m, 2)


def collate_host(encodings, fs_vectors, targets=None):
    """Host-side collation of reference-style encodings into flat arrays.

    Validation mirrors gnn.py:141-144 (EmptyGraph for N < 1, ShapeMismatch for
    a feature matrix that is not (N, 32), or an edge endpoint outside [0, N)).
    Returns numpy arrays.  One pass per graph: features converted straight into the f32
    node matrix, edges flattened with np.fromiter; the endpoint check is one vectorised
    test over the batch."""
    G = len(encodings)
    n = np.empty(G, dtype=np.int64)
    feats, edges = [], []
    for g, enc in enumerate(encodings):
        ng = int(enc.num_nodes)
        if ng < 1:
            raise EmptyGraph("encoding has no nodes")
        f = enc.features
        if not isinstance(f, np.ndarray):
            f = np.asarray(f)
        if f.shape != (ng, FEATURE_WIDTH):
            raise ShapeMismatch(f"feature matrix {f.shape} does not match {ng} nodes")
        feats.append(f)
        edges.append(_edge_pairs(enc.edges))
        n[g] = ng
    graph_ptr = np.zeros(G + 1, dtype=np.int32)
    np.cumsum(n, out=graph_ptr[1:])
    N = int(graph_ptr[-1]) if G else 0
    x = np.empty((N, FEATURE_WIDTH), np.float32)
    for g, f in enumerate(feats):
        x[graph_ptr[g]:graph_ptr[g + 1]] = f
    ne = np.array([e.shape[0] for e in edges], dtype=np.int64)
    e_all = np.concatenate(edges) if G else np.zeros((0, 2), np.int64)
    if e_all.size:
        lo = np.repeat(graph_ptr[:-1].astype(np.int64), ne)  # each edge's graph offset
        hi = np.repeat(n, ne)
        if (e_all.min() < 0) or bool(((e_all[:, 0] >= hi) | (e_all[:, 1] >= hi)).any()):
            raise ShapeMismatch("edge endpoint outside [0, num_nodes)")
        src, dst = e_all[:, 0] + lo, e_all[:, 1] + lo
    else:
        src = dst = np.zeros(0, np.int64)
    # static features and targets stay float64 (StaticFeatures.as_vector, TargetVector.as_array):
    # the device z-scores them in fp64, so a small fs / y std cannot amplify an fp32 rounding
    fs = np.asarray(fs_vectors, dtype=np.float64).reshape(G, STATIC_WIDTH)
    y = None if targets is None else np.asarray(targets, dtype=np.float64).reshape(G, 3)
    return x, src, dst, graph_ptr, fs, y


def upload_batch(x, src, dst, graph_ptr, fs, y=None, device="cuda", build_csr=True, edge_ptr=None,
                 validate=True) -> Batch:
    """Pinned host -> device copies of a collated batch, then K1 CSR on device.

    validate: host check of the edge endpoints (group_edges); False leaves bad edges to
    the device flag `Batch.bad` (kernel tests)."""
    dev = torch.device(device)

    def h2d(a, dtype=None):
        # already-pinned tensors copy asynchronously; numpy arrays go straight from pageable
        # memory (a fresh pinned staging buffer per call costs more than it saves)
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        return t.to(dev, dtype=dtype, non_blocking=t.is_pinned())

    if edge_ptr is None:
        try:
            edge_ptr = group_edges(src, dst, graph_ptr)
        except ShapeMismatch:
            if validate:
                raise
            edge_ptr = None
    arrays = [x, src, dst, graph_ptr, fs] + ([y] if y is not None else [])
    # the kernels' layouts: f32 features, int64 edge endpoints, int32 graph_ptr (an int32 edge list
    # reinterpreted as int64 would read garbage endpoints)
    b = Batch(G=int(len(graph_ptr) - 1), N=int(graph_ptr[-1]), E=int(len(src)), x=h2d(x, torch.float32),
              src=h2d(src, torch.int64), dst=h2d(dst, torch.int64), graph_ptr=h2d(graph_ptr, torch.int32),
              fs=h2d(fs, torch.float64),
              y=None if y is None else h2d(y, torch.float64),
              h2d_bytes=int(sum(np.asarray(a).nbytes for a in arrays)))
    if edge_ptr is not None:
        b.edge_ptr = h2d(edge_ptr if isinstance(edge_ptr, torch.Tensor) else np.asarray(edge_ptr, np.int64))
        b.max_nodes = int(np.diff(np.asarray(graph_ptr)).max())
        b.max_edges = int(np.diff(edge_ptr).max()) if len(edge_ptr) > 1 else 0
        b.h2d_bytes += int(np.asarray(edge_ptr).nbytes)
    if build_csr:
        build_batch_csr(b)
    return b


GROUPED_MAX_EDGES = 8192  # per-graph limit (edges and nodes) of the shared-memory CSR kernel
GROUPED_MAX_GRAPHS = 8192


def build_batch_csr(b: Batch, grouped: bool | None = None) -> Batch:
    """K1: deterministic CSR + transposed CSR of the batch (gnn.py:130-137).

    Uses the per-graph shared-memory kernel when the batch is grouped by graph
    (2 launches), else the global path; both give bit-identical output."""
    dev = b.x.device
    N, E = b.N, b.E
    i32 = dict(dtype=torch.int32, device=dev)
    b.rowptr = torch.empty(N + 1, **i32)
    b.col = torch.empty(max(E, 1), **i32)
    b.deg = torch.empty(N, **i32)
    b.inv_deg = torch.empty(N, dtype=torch.float32, device=dev)
    b.t_rowptr = torch.empty(N + 1, **i32)
    b.t_col = torch.empty(max(E, 1), **i32)
    b.bad = torch.empty(1, **i32)
    b.node_graph = torch.empty(max(N, 1), **i32)
    lib = _lib.load()
    if grouped is None:
        grouped = (b.edge_ptr is not None and b.G <= GROUPED_MAX_GRAPHS and b.max_edges <= GROUPED_MAX_EDGES
                   and b.max_nodes <= GROUPED_MAX_EDGES)
    if grouped:  # the per-graph kernels also write node -> graph
        ws_bytes = lib.dippm_csr_grouped_workspace_bytes(b.G, E)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        _lib.call("dippm_build_csr_grouped", _p(b.src), _p(b.dst), _p(b.graph_ptr), _p(b.edge_ptr), b.G, N, E,
                  b.max_nodes, b.max_edges, _p(b.rowptr), _p(b.col), _p(b.deg), _p(b.inv_deg), _p(b.t_rowptr),
                  _p(b.t_col), _p(b.bad), _p(b.node_graph), _p(ws), ws_bytes, _stream())
        return b
    _lib.call("dippm_node_graph", _p(b.graph_ptr), b.G, _p(b.node_graph), _stream())
    ws_bytes = lib.dippm_csr_workspace_bytes(N, E)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    _lib.call("dippm_build_csr", _p(b.src), _p(b.dst), E, N, _p(b.rowptr), _p(b.col), _p(b.deg), _p(b.inv_deg),
              _p(b.t_rowptr), _p(b.t_col), _p(b.bad), _p(ws), ws_bytes, _stream())
    return b


# ---------------------------------------------------------------------------
# engine

class Workspace:
    """Per-batch activation / gradient buffers (sized for up to N nodes, G graphs)."""

    def __init__(self, eng: "Engine", N: int, G: int, train: bool):
        dev, dt, hp = eng.device, eng.dtype, eng.L.hp
        f32 = dict(dtype=torch.float32, device=dev)
        lib = _lib.load()
        self.N, self.G = N, G
        sage = eng.L.arch == "sage"
        if sage:
            # A1 = [X | agg X | 1 | 0...]: the constant ones column (col 64) turns the layer-1 weight
            # gradient GEMM into [dW_self; dW_neigh; db] in one pass (row 64 = sum_rows dz1 = the
            # bias gradient, gnn.py:230, which lands on sage1.bias right after w_neigh in the layout)
            self.A = [ActBuf(N, 4 * FEATURE_WIDTH, dt, dev), ActBuf(N, 2 * hp, dt, dev), ActBuf(N, 2 * hp, dt, dev)]
            a1 = self.A[0].t
            (a1[0] if dt == DT_TF32X3 else a1)[:, 2 * FEATURE_WIDTH:].zero_()
            (a1[0] if dt == DT_TF32X3 else a1)[:, 2 * FEATURE_WIDTH] = 1.0
            if dt == DT_TF32X3:
                a1[1][:, 2 * FEATURE_WIDTH:].zero_()
            self.H3 = ActBuf(N, hp, dt, dev) if eng.backend != 0 else None  # SIMT anchor only (unfused readout)
            # fused readout (layer-3 GEMM epilogue): per-32-row-block boundary sums + whole-graph sums
            self.pool_part = torch.empty(lib.dippm_pool_partial_rows(N), hp, **f32)
            self.pool_graph = torch.empty(G, hp, **f32)
        self.u = ActBuf(G, eng.L.u_width, dt, dev)
        self.x2 = ActBuf(G, hp, dt, dev)
        self.x3 = ActBuf(G, hp, dt, dev)
        self.masks = torch.ones(2, G, hp, **f32)
        self.out = torch.empty(G, 3, **f32)
        self.y_pred = torch.empty(G, 3, dtype=torch.float64, device=dev)
        self.mig = torch.empty(G, dtype=torch.int8, device=dev)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
        self.loss = torch.zeros(4, dtype=torch.float64, device=dev)
        self.row_loss = torch.empty(G, 4, dtype=torch.float64, device=dev)   # fused head: per-graph loss terms
        self.head_sync = torch.zeros(lib.dippm_head_fused_sync_ints(), dtype=torch.int32, device=dev)  # fused head
        self.head_pending = None  # forward(defer_head=True) -> loss() -> backward() runs the fused head once
        self.u_pending = None     # batch whose u the fused head still has to form (its phase 0)
        self.train = train
        if train:
            self.dout = torch.empty(G, 3, **f32)
            self.d2 = ActBuf(G, hp, dt, dev)
            self.d1 = ActBuf(G, hp, dt, dev)
            self.head_bits = torch.empty(hp // 32, G, dtype=torch.int32, device=dev)
            self.dhead_f32 = torch.empty(2, G, hp, **f32)  # fused head: fp32 d2, d1 (bias-gradient sums)
            if sage:
                self.du = torch.empty(G, hp, **f32)
                # one [dz_l | agg^T dz_l] buffer per layer: the weight-gradient GEMM of layer l may
                # still read B_l on the side stream while the dgrad chain fills B_{l-1}
                self.B = [ActBuf(N, 2 * hp, dt, dev) for _ in range(3)]
                # 1-bit ReLU' masks of h1, h2 (and of the head's x2, dropout included) written by the
                # forward GEMM epilogues and read by the GATE epilogues (replaces re-reading activations)
                # chunk-major [3, Hp/32, N]: word (c/32, r); a warp's 32 rows store/load 128 contiguous bytes
                self.relu_bits = torch.empty(3, hp // 32, N, dtype=torch.int32, device=dev)  # h1, h2, h3
                self.colsum = torch.empty(lib.dippm_colsum_rows(N), hp, **f32)
                # layer 3's partials apart from layer 2's: each is folded by its layer's weight-gradient
                # GEMM on the side stream, which may still read layer 3's while layer 2's are written
                self.colsum3 = torch.empty(lib.dippm_colsum_rows(N), hp, **f32)
                self.colsum_sync = torch.zeros(lib.dippm_colsum_sync_ints(N), dtype=torch.int32, device=dev)
            # WGRAD outputs are [width, Hp] (M = width, N = Hp, reduction over rows), split-K
            # partials reduced inside the GEMM kernel (tile_sync counters stay zero between launches)
            # split counts are chosen per call from the actual row count (<= these upper bounds)
            big = 1 << 30
            wg_rows = [2 * d + (1 if i == 0 else 0) for i, d in enumerate(eng.L.d_in)]  # layer 1: + bias row
            smax = [lib.dippm_wgrad_splits(w, hp, big) for w in wg_rows]
            hmax = [lib.dippm_wgrad_splits(hp, hp, big), lib.dippm_wgrad_splits(eng.L.u_width, hp, big)]
            widest = max([s * w for s, w in zip(smax, wg_rows)] + [hmax[0] * hp, hmax[1] * eng.L.u_width])
            self.splitk = torch.empty(widest * hp, **f32)
            sync = max(lib.dippm_wgrad_sync_ints(w, hp) for w in [2 * d for d in eng.L.d_in] + [eng.L.u_width])
            self.tile_sync = torch.zeros(sync, dtype=torch.int32, device=dev)


class Engine:
    """Device-resident DIPPM GraphSAGE network (weights, Adam state, GEMM operand copies)."""

    def __init__(self, hidden: int, precision: str = "fp32", device=None, backend: str = "tc", arch: str = "sage"):
        """backend is test-only: "simt" selects the library's SIMT GEMM anchor, which the kernel
        tests compare the tcgen05 path against.  The package itself always runs "tc"."""
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(PRECISIONS)}, got {precision!r}")
        if backend not in BACKENDS:
            raise ValueError(f"backend must be one of {sorted(BACKENDS)}, got {backend!r}")
        self.device = require_device(device)
        self.L = L = Layout(hidden, arch)
        self.arch = arch
        self.precision, self.dtype, self.backend = precision, PRECISIONS[precision], BACKENDS[backend]
        n = L.total
        f64 = dict(dtype=torch.float64, device=self.device)
        self.params = torch.zeros(n, **f64)
        self.m = torch.zeros(n, **f64)
        self.v = torch.zeros(n, **f64)
        self.grads = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.p32 = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.norm = torch.zeros(16, **f64)
        # [y_mean | y_std | 0 | 1]: for callers that hand over fs already normalised (forward_norm)
        self.norm_fs_id = torch.zeros(16, **f64)
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=self.device)  # Adam step count (graph-safe)
        hp, dt, d = L.hp, self.dtype, self.device
        self.Wf = [ActBuf(2 * di, hp, dt, d) for di in L.d_in]
        self.Wd = [None] + [ActBuf(di, 2 * hp, dt, d) for di in L.d_in[1:]]
        self.W1h = ActBuf(L.u_width, hp, dt, d)
        self.W2h = ActBuf(hp, hp, dt, d)
        segs = []
        for i, di in enumerate(L.d_in):
            segs.append(_lib.PackSeg(L.offsets[f"sage{i + 1}.w_self"], 2 * di, hp, 0, self.Wf[i].view()))
            if i > 0:
                segs.append(_lib.PackSeg(L.offsets[f"sage{i + 1}.w_self"], di, hp, 0, self.Wd[i].view()))
                segs.append(_lib.PackSeg(L.offsets[f"sage{i + 1}.w_neigh"], di, hp, hp, self.Wd[i].view()))
        segs.append(_lib.PackSeg(L.offsets["fc1.w"], L.u_width, hp, 0, self.W1h.view()))
        segs.append(_lib.PackSeg(L.offsets["fc2.w"], hp, hp, 0, self.W2h.view()))
        self._segs = (_lib.PackSeg * len(segs))(*segs)
        self.launches = 0
        self.cta_pair = 0       # GEMM tile policy passed to the library: 0 auto, 1 single-CTA, 2 CTA pair
        self.gemm_hook = None  # bench instrumentation: called ("pre"|"post", flops) around each GEMM
        self.fused_head = True  # FUSED_HEAD and this flag gate the fused head kernel
        self._t_advanced = False  # the fused head advanced the step counter for the coming adam_step
        # backward: the weight-gradient GEMMs run on a side stream, off the dgrad critical path
        # (readout -> GATE_3 -> agg^T_2 -> GATE_2 -> WGRAD_1), so they fill the tail waves and
        # memory-bound gaps of that chain; the step joins the side stream before Adam
        self.overlap_wgrad = os.environ.get("DIPPM_OVERLAP_WGRAD", "1") != "0"
        self._side = None
        self.head_fused_max = int(_lib.load().dippm_head_fused_max_graphs())
        self._lock = threading.Lock()  # parameter uploads vs concurrent read-only predict calls

    # -- parameters -----------------------------------------------------------
    def set_params(self, items, normalizer) -> None:
        """Upload the host model's current values (padded layout) and refresh the operand copies.
        Skipped when the values are byte-identical to the last upload (repeated predict calls):
        one memcmp per tensor, ~13 MB at hidden 512, instead of an elementwise compare."""
        items = [(name, np.ascontiguousarray(arr, np.float64)) for name, arr in items]
        norm = np.concatenate([np.asarray(normalizer.y_mean, np.float64), np.asarray(normalizer.y_std, np.float64),
                               np.asarray(normalizer.fs_mean, np.float64), np.asarray(normalizer.fs_std, np.float64)])
        with self._lock:
            last = getattr(self, "_uploaded", None)
            if (last is not None and _same_bytes(last[1], norm) and len(last[0]) == len(items)
                    and all(n0 == n1 and a0.shape == a1.shape and _same_bytes(a0, a1)
                            for (n0, a0), (n1, a1) in zip(last[0], items))):
                return
            host = np.zeros(self.L.total, dtype=np.float64)
            for name, arr in items:
                off = self.L.offsets[name]
                padded = self.L.pad(name, arr)
                host[off:off + padded.size] = padded.ravel()
            self.params.copy_(torch.from_numpy(host), non_blocking=False)
            self.set_normalizer(normalizer)
            self.refresh()
            self._uploaded = ([(name, arr.copy()) for name, arr in items], norm)

    def check_batch(self, b: "Batch") -> None:
        """Raise ShapeMismatch if K1 flagged an edge endpoint outside its graph (synchronises;
        the per-call drop-in paths read results back right after anyway)."""
        if b.bad is not None and int(b.bad[0].item()):
            raise ShapeMismatch("edge endpoint outside its graph's node range")

    def set_normalizer(self, norm) -> None:
        self._uploaded = None
        vec = np.concatenate([np.asarray(norm.y_mean, np.float64), np.asarray(norm.y_std, np.float64),
                              np.asarray(norm.fs_mean, np.float64), np.asarray(norm.fs_std, np.float64)])
        self.norm.copy_(torch.from_numpy(vec))
        vec = vec.copy()
        vec[6:11], vec[11:16] = 0.0, 1.0
        self.norm_fs_id.copy_(torch.from_numpy(vec))

    def reset_adam(self) -> None:
        self.m.zero_()
        self.v.zero_()
        self.t_dev.zero_()

    @property
    def t(self) -> int:
        """Adam step count (lives on the device so captured steps advance it)."""
        return int(self.t_dev.item())

    def _unpack(self, flat: np.ndarray) -> dict:
        return {name: self.L.unpad(name, flat[off:off + int(np.prod(self.L.shapes[name]))].reshape(self.L.shapes[name]))
                for name, off in self.L.offsets.items()}

    def get_params(self) -> dict:
        return self._unpack(self.params.cpu().numpy())

    def get_grads(self) -> dict:
        return self._unpack(self.grads.double().cpu().numpy())

    def _adam_pack(self, do_adam: int, lr=0.0, beta1=0.9, beta2=0.999, eps=1e-8, grad_scale=1.0) -> None:
        _lib.call("dippm_adam_pack", _p(self.params), _p(self.m), _p(self.v), _p(self.grads), grad_scale,
                  self.L.total, 0, _p(self.t_dev), lr, beta1, beta2, eps, do_adam, _p(self.p32), self._segs,
                  len(self._segs), _stream())
        self.launches += 1

    def refresh(self) -> None:
        """Refresh the fp32 copy and every GEMM operand copy from the fp64 masters."""
        self._adam_pack(0)

    def adam_step(self, lr: float, beta1=0.9, beta2=0.999, eps=1e-8, grad_scale: float = 1.0) -> None:
        """numerics.adam_step over all 15 tensors + operand refresh (t += 1 on the device first)."""
        self._uploaded = None  # device values now differ from the last host upload
        if not self._t_advanced:  # (the fused head of this step already advanced it)
            _lib.call("dippm_step_counter", _p(self.t_dev), _stream())
        self._t_advanced = False
        self._adam_pack(1, lr, beta1, beta2, eps, grad_scale)

    def _f32(self, name: str) -> int:
        return self.p32.data_ptr() + 4 * self.L.offsets[name]

    def _g32(self, name: str) -> int:
        return self.grads.data_ptr() + 4 * self.L.offsets[name]

    # -- kernels --------------------------------------------------------------
    def _gemm(self, kind, M, N, K, a, a_mn, b, b_mn, bias=None, relu=0, out=NULL_ACT, c=None, ldc=0, splits=1,
              gate=NULL_ACT, gate_scale=1.0, drop_mode=0, mask=None, ldm=0, drop_p=0.0, seed=0, seed_dev=None,
              relu_bits=None, gate_bits=None, bits_ld=0, tile_sync=None, out_scale=1.0, pool_partial=None,
              pool_graph=None, node_graph=None, graph_ptr=None, bias_partial=None, bias_grad=None):
        args = GemmArgs(kind, M, N, K, a, a_mn, b, b_mn, bias, relu, out, c, ldc, splits, gate, gate_scale,
                        drop_mode, mask, ldm, drop_p, int(seed) & (2**64 - 1), seed_dev, relu_bits, gate_bits,
                        bits_ld, self.cta_pair, tile_sync, out_scale, pool_partial, pool_graph, node_graph, graph_ptr,
                        bias_partial, bias_grad)
        if self.gemm_hook is not None:
            self.gemm_hook("pre", 2.0 * M * N * K)
        _lib.check(_lib.load().dippm_gemm(args, self.backend, _stream()), "dippm_gemm")
        if self.gemm_hook is not None:
            self.gemm_hook("post", 2.0 * M * N * K)
        self.launches += 1

    def _wgrad(self, dz: Act, x: Act, rows: int, width: int, ws: Workspace, out_name: str,
               bias_partial: int | None = None, bias_grad: int | None = None) -> None:
        """grads[out_name] (as [width, Hp]) = x^T @ dz over `rows` rows (gnn.py:228-229, 296):
        one split-K tcgen05 launch that also reduces its partials in fixed split order (and, with
        bias_partial, folds the layer's deferred bias-gradient partial rows into bias_grad)."""
        hp = self.L.hp
        splits = _lib.load().dippm_wgrad_splits(width, hp, rows)
        self._gemm(GEMM_WGRAD, width, hp, rows, x, 1, dz, 1, out=Act(self._g32(out_name), hp, 0, DT_F32),
                   c=_p(ws.splitk), ldc=hp, splits=splits, tile_sync=_p(ws.tile_sync), out_scale=1.0,
                   bias_partial=bias_partial, bias_grad=bias_grad)

    def fused_head_ok(self, G: int) -> bool:
        """The fused head kernel covers this batch (bf16 tensor-core path, small batch)."""
        return (FUSED_HEAD and self.fused_head and self.backend == 0 and self.dtype == DT_BF16
                and self.L.hp <= 512 and self.L.u_width <= 576 and G <= self.head_fused_max)

    def forward(self, b: Batch, ws: Workspace, mask_mode: int = 0, dropout_p: float = 0.0, seed: int = 0,
                predict: bool = True, defer_head: bool = False, fs_normalized: bool = False) -> None:
        """Eval (mask_mode 0) or train-mode forward (1: masks in ws.masks, 2: generated):
        K2 aggregation -> K3 GEMM x3, K4 pooling, K5 head (2 GEMMs + fc3).

        defer_head (training steps: forward -> loss -> backward): when the fused head kernel
        covers the batch, the head is not run here; loss() records its arguments and backward()
        runs forward, loss and backward of the head in one launch.

        fs_normalized: b.fs already holds normalised static features (the model protocol's
        forward_norm receives fs_norm, gnn.py:212), so the device z-score is the identity."""
        s, L, hp = _stream(), self.L, self.L.hp
        fs_norm = self.norm_fs_id if fs_normalized else self.norm
        if self.arch == "mlp":  # MlpModel.forward_norm (gnn.py:253-255): the head on [fs_norm | 0]
            _lib.call("dippm_fs_normalize", _p(b.fs), b.G, _p(fs_norm), ws.u.view(), L.u_width, s)
            self.launches += 1
            self._head_or_defer(b, ws, mask_mode, dropout_p, seed, predict, defer_head)
            return
        _lib.call("dippm_sage_aggregate", f32_act(b.x), ws.A[0].view(FEATURE_WIDTH), ws.A[0].view(0), b.N,
                  FEATURE_WIDTH, _p(b.rowptr), _p(b.col), _p(b.inv_deg), s)
        fused = self.backend == 0  # readout fused into the layer-3 GEMM epilogue (h3 never stored)
        outs = [ws.A[1].view(0), ws.A[2].view(0), NULL_ACT if fused else ws.H3.view(0)]
        bits = ws.relu_bits if ws.train else None
        for i in range(3):
            if i > 0:
                _lib.call("dippm_sage_aggregate", ws.A[i].view(0), ws.A[i].view(hp), NULL_ACT, b.N, hp,
                          _p(b.rowptr), _p(b.col), _p(b.inv_deg), s)
            pool = dict(pool_partial=_p(ws.pool_part), pool_graph=_p(ws.pool_graph), node_graph=_p(b.node_graph),
                        graph_ptr=_p(b.graph_ptr)) if fused and i == 2 else {}
            self._gemm(GEMM_FWD, b.N, hp, 2 * L.d_in[i], ws.A[i].view(0), 0, self.Wf[i].view(), 1,
                       bias=self._f32(f"sage{i + 1}.bias"), relu=1, out=outs[i],
                       relu_bits=_p(bits[i]) if bits is not None else None,
                       # h3's mask is read per row by the readout backward: row-major (bits_ld 0)
                       bits_ld=0 if i == 2 else ws.N, **pool)
        ws.u_pending = None
        if fused and self.fused_head_ok(b.G) and HEAD_POOL and not fs_normalized:  # K4 second stage inside the fused head (phase 0)
            ws.u_pending = b
        elif fused:  # K4 second stage: means from the block sums + static features (gnn.py:214-215)
            _lib.call("dippm_pool_combine", _p(ws.pool_part), _p(ws.pool_graph), _p(b.graph_ptr), b.G, hp,
                      _p(b.fs), _p(fs_norm), ws.u.view(), s)
        else:
            _lib.call("dippm_pool_concat", ws.H3.view(0), _p(b.graph_ptr), b.G, hp, _p(b.fs), _p(fs_norm),
                      ws.u.view(), s)
        self.launches += 3 + 1
        self._head_or_defer(b, ws, mask_mode, dropout_p, seed, predict, defer_head)

    def _head_or_defer(self, b, ws, mask_mode, dropout_p, seed, predict, defer_head) -> None:
        if defer_head and ws.train and not predict and self.fused_head_ok(b.G):
            ws.head_pending = dict(mask_mode=mask_mode, dropout_p=dropout_p, seed=seed)
            return
        ws.head_pending = None
        self._head_forward(b, ws, mask_mode, dropout_p, seed, predict)

    def _head_fused(self, b: Batch, ws: Workspace, mask_mode: int, dropout_p: float, seed: int, predict: bool,
                    loss=None, keep_scale: float = 1.0, advance_step: bool = False,
                    defer_wgrad: bool = False) -> None:
        """K5/K6 in one cooperative launch (head_fused.cu): forward, and with loss = (delta,
        grad_den) the Huber loss and, on a training workspace, the whole head backward
        (defer_wgrad: except dW1 / dW2, which the caller runs as weight-gradient GEMMs)."""
        L, hp = self.L, self.L.hp
        drop = mask_mode if dropout_p > 0.0 or mask_mode == 1 else 0
        train = loss is not None and ws.train
        if predict:
            ws.nonfinite.zero_()
        a = _lib.HeadArgs()
        a.G, a.hp, a.u_width = b.G, hp, L.u_width
        a.u, a.w1, a.w2 = _p(ws.u.t), _p(self.W1h.t), _p(self.W2h.t)
        a.b1, a.b2, a.w3, a.b3 = self._f32("fc1.b"), self._f32("fc2.b"), self._f32("fc3.w"), self._f32("fc3.b")
        a.x2, a.x3 = _p(ws.x2.t), _p(ws.x3.t)
        if ws.train:
            a.bits, a.bits_ld = _p(ws.head_bits), ws.G
        a.drop_mode, a.drop_p, a.keep_scale = drop, float(dropout_p), float(keep_scale)
        a.seed1, a.seed2 = (int(seed) * 2) & (2**64 - 1), (int(seed) * 2 + 1) & (2**64 - 1)  # dippm_gemm's seeds
        a.seed_dev = _p(self.t_dev) if drop == 2 else None
        if drop == 1:
            a.mask1, a.mask2 = _p(ws.masks[0]), _p(ws.masks[1])
        a.out, a.norm = _p(ws.out), _p(self.norm)
        if predict:
            a.y_pred, a.mig, a.nonfinite = _p(ws.y_pred), _p(ws.mig), _p(ws.nonfinite)
        if loss is not None:
            a.y_raw, a.delta, a.grad_den = _p(b.y), float(loss[0]), float(loss[1])
            a.loss_out, a.row_loss = _p(ws.loss), _p(ws.row_loss)
        if train:
            a.dout, a.d2, a.d1 = _p(ws.dout), _p(ws.d2.t), _p(ws.d1.t)
            a.d2f, a.d1f = _p(ws.dhead_f32[0]), _p(ws.dhead_f32[1])
            a.gw1, a.gb1, a.gw2, a.gb2 = self._g32("fc1.w"), self._g32("fc1.b"), self._g32("fc2.w"), self._g32("fc2.b")
            if defer_wgrad:  # dW1 / dW2 and the column sums + loss: launched by backward()
                a.gw1 = a.gw2 = None
                a.defer_reduce = 1
                ws.head_args = a
            a.gw3, a.gb3 = self._g32("fc3.w"), self._g32("fc3.b")
            a.du = _p(ws.du) if self.arch == "sage" else None
            a.train = 1
            if advance_step:  # this step's t += 1 here (the adam_step that follows skips its launch)
                a.step_counter = _p(self.t_dev)
                self._t_advanced = True
        a.sync = _p(ws.head_sync)
        pb, ws.u_pending = getattr(ws, "u_pending", None), None
        if pb is not None:  # u's readout columns from the layer-3 block sums (dippm_pool_combine's work)
            a.pool_partial, a.pool_graph, a.graph_ptr, a.fs_raw = (_p(ws.pool_part), _p(ws.pool_graph),
                                                                   _p(pb.graph_ptr), _p(pb.fs))
        _lib.call("dippm_head_fused", C.byref(a), _stream())
        self.launches += 1

    def _head_forward(self, b: Batch, ws: Workspace, mask_mode: int, dropout_p: float, seed: int,
                      predict: bool) -> None:
        """K5: fc1/fc2 tcgen05 GEMMs (bias, ReLU, dropout epilogue) + fc3/de-normalise/MIG (gnn.py:265-284)."""
        s, hp = _stream(), self.L.hp
        if self.fused_head_ok(b.G):
            self._head_fused(b, ws, mask_mode, dropout_p, seed, predict)
            return
        if predict:
            ws.nonfinite.zero_()  # workspaces are reused across calls
        drop = mask_mode if dropout_p > 0.0 or mask_mode == 1 else 0
        for j, (x, W, out) in enumerate(((ws.u, self.W1h, ws.x2), (ws.x2, self.W2h, ws.x3))):
            self._gemm(GEMM_FWD, b.G, hp, x.cols, x.view(), 0, W.view(), 1, bias=self._f32(f"fc{j + 1}.b"), relu=1,
                       out=out.view(), drop_mode=drop, ldm=hp, drop_p=dropout_p,
                       # generated masks (mode 2) are not recorded on the tensor-core path: the
                       # backward gates on the 1-bit masks; the SIMT anchor records them
                       mask=None if drop == 2 and self.backend == 0 else ws.masks[j].data_ptr(),
                       seed=seed * 2 + j, seed_dev=_p(self.t_dev) if drop == 2 else None,
                       relu_bits=_p(ws.head_bits) if ws.train and j == 0 else None, bits_ld=ws.G)
        _lib.call("dippm_fc3_forward", ws.x3.view(), b.G, hp, self._f32("fc3.w"), self._f32("fc3.b"), _p(ws.out),
                  _p(self.norm), _p(ws.y_pred) if predict else None, _p(ws.mig) if predict else None,
                  _p(ws.nonfinite), s)
        self.launches += 1

    def loss(self, b: Batch, ws: Workspace, delta: float = 1.0, grad_den: float = 0.0) -> None:
        """Huber loss + dout (numerics.py:58-73); grad_den = global batch size under DP (0: this batch)."""
        if ws.head_pending is not None:  # deferred fused head: runs in backward()
            ws.head_pending.update(delta=float(delta), grad_den=float(grad_den))
            return
        _lib.call("dippm_huber", _p(ws.out), _p(b.y), b.G, _p(self.norm), float(delta), float(grad_den),
                  _p(ws.dout) if ws.train else None, _p(ws.loss), _stream())
        self.launches += 1

    def backward(self, b: Batch, ws: Workspace, keep_scale: float = 1.0, on_partial=None,
                 advance_step: bool = False) -> None:
        """Head backward (fc3 fused kernel, fc2/fc1 tcgen05 WGRAD/GATE/STORE), readout
        backward, then per SAGE layer: agg^T + bias, WGRAD, gated dgrad GEMM."""
        s, L, hp, N = _stream(), self.L, self.L.hp, b.N
        pend, ws.head_pending = ws.head_pending, None
        if pend is not None:  # the deferred head: forward + loss + backward in one launch
            if "delta" not in pend:
                raise RuntimeError("forward(defer_head=True) needs loss() before backward()")
            # advance_step: an adam_step follows this backward, so the fused head may advance the
            # device step counter itself (one launch fewer)
            # sage: dW1 / dW2 leave the head's critical path (weight-gradient GEMMs below)
            head_wgrad = self.arch == "sage" and HEAD_WGRAD_DEFER
            self._head_fused(b, ws, pend["mask_mode"], pend["dropout_p"], pend["seed"], False,
                             loss=(pend["delta"], pend["grad_den"]), keep_scale=keep_scale,
                             advance_step=advance_step, defer_wgrad=head_wgrad)
            if self.arch == "mlp":
                return
        else:
            head_wgrad = False
            _lib.call("dippm_fc3_backward", ws.x3.view(), b.G, hp, self._f32("fc3.w"), _p(ws.dout),
                      float(keep_scale), self._g32("fc3.w"), self._g32("fc3.b"), ws.d2.view(), self._g32("fc2.b"), s)
            self._wgrad(ws.d2.view(), ws.x2.view(), b.G, hp, ws, "fc2.w")
            self._gemm(GEMM_GATE, b.G, hp, hp, ws.d2.view(), 0, self.W2h.view(), 0, out=ws.d1.view(),
                       gate=ws.x2.view(), gate_scale=keep_scale, gate_bits=_p(ws.head_bits), bits_ld=ws.G)
            _lib.call("dippm_colsum_act", ws.d1.view(), b.G, hp, self._g32("fc1.b"), s)
            self._wgrad(ws.d1.view(), ws.u.view(), b.G, L.u_width, ws, "fc1.w")
            if self.arch == "mlp":  # no graph network below the head
                self.launches += 2
                return
            self._gemm(GEMM_STORE, b.G, hp, hp, ws.d1.view(), 0, self.W1h.view(), 0, c=_p(ws.du), ldc=hp)
        side = None
        if self.overlap_wgrad and on_partial is None and self.backend == 0:
            if self._side is None:
                self._side = torch.cuda.Stream(self.device)
            side = self._side
        main = torch.cuda.current_stream()
        if head_wgrad:  # the fused head's reductions, dW2 = x2^T d2, dW1 = u^T d1 (off the dgrad chain)
            def head_wgrads():
                _lib.call("dippm_head_reduce", C.byref(ws.head_args), _stream())
                self._wgrad(ws.d2.view(), ws.x2.view(), b.G, hp, ws, "fc2.w")
                self._wgrad(ws.d1.view(), ws.u.view(), b.G, L.u_width, ws, "fc1.w")
            if side is None:
                head_wgrads()
            else:
                ev = torch.cuda.Event()
                ev.record(main)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    head_wgrads()
            self.launches += 3

        # layers 2-3: the bias gradient (gnn.py:230) is folded by the layer's weight-gradient GEMM
        # from the agg^T kernel's partial rows (tensor-core backend), not in the agg^T kernel's tail
        defer = self.backend == 0

        def wgrad(B, i, part=None):
            width = 2 * L.d_in[i] + (1 if i == 0 else 0)  # layer 1: + the ones row (bias gradient)
            fold = dict(bias_partial=_p(part), bias_grad=self._g32(f"sage{i + 1}.bias")) if part is not None else {}
            if side is None:
                self._wgrad(B.view(0), ws.A[i].view(0), N, width, ws, f"sage{i + 1}.w_self", **fold)
                return
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            with torch.cuda.stream(side):
                self._wgrad(B.view(0), ws.A[i].view(0), N, width, ws, f"sage{i + 1}.w_self", **fold)

        for i in (2, 1, 0):
            B = ws.B[i]
            bias = None if defer else self._g32(f"sage{i + 1}.bias")  # gnn.py:230
            part = ws.colsum3 if i == 2 else ws.colsum
            if i == 0:  # layer 1: the bias gradient comes out of the WGRAD GEMM (ones column of A1)
                wgrad(B, 0)
                continue
            if i == 2:  # readout backward fused: dz3 formed on the fly (gnn.py:224, 227)
                _lib.call("dippm_readout_aggregate_t", _p(ws.du), hp, _p(b.graph_ptr), _p(b.node_graph),
                          NULL_ACT if ws.H3 is None else ws.H3.view(0), B.view(0), hp, N, _p(b.t_rowptr),
                          _p(b.t_col), _p(b.inv_deg), _p(part), bias, _p(ws.colsum_sync),
                          _p(ws.relu_bits[2]) if self.backend == 0 else None, 0, s)  # row-major; SIMT: no bits
            else:
                _lib.call("dippm_sage_aggregate_t", B.view(0), hp, N, int(i > 0), _p(b.t_rowptr), _p(b.t_col),
                          _p(b.inv_deg), _p(part), bias, _p(ws.colsum_sync), s)
            wgrad(B, i, part if defer else None)
            self._gemm(GEMM_GATE, N, L.d_in[i], 2 * hp, B.view(0), 0, self.Wd[i].view(), 0,
                       out=ws.B[i - 1].view(0), gate=ws.A[i].view(0), gate_scale=1.0,
                       gate_bits=_p(ws.relu_bits[i - 1]), bits_ld=ws.N)
            if i == 2 and on_partial is not None:  # sage3 + head gradients are final here
                on_partial(L.offsets["sage3.w_self"])
        if side is not None:  # join: Adam reads every gradient
            ev = torch.cuda.Event()
            ev.record(side)
            main.wait_event(ev)
        self.launches += 5 + 3 * 2 - 3 - 1


# ---------------------------------------------------------------------------
# MIG-pick parity of the bf16 predict path

# the re-score band in normalised units: the stated bf16 tolerance of the normalised
# outputs; times y_std[memory] it is the band in MB around each ceiling
BF16_MIG_BAND = 2e-2


def mig_band_rescore(eng32: "Engine", b: Batch, ws: Workspace, band_mb: float, holder) -> int:
    """Re-score in fp32 the graphs of batch `b` whose bf16-predicted memory (ws.y_pred) lies
    within band_mb of a MIG ceiling, and write their fp32 predictions and picks back into
    ws.y_pred / ws.mig.  Outside the band the bf16 pick equals the reference's (the bf16
    error is below the band); inside it the fp32 pick does, except within the fp32
    tolerance of a ceiling.  Device-side select / gather / scatter (rescore.cu); one small
    read-back of the band size.  Returns the number of graphs re-scored."""
    if b.edge_ptr is None:
        raise ShapeMismatch("MIG re-score needs edges grouped by graph (edge_ptr)")
    dv, G = b.x.device, b.G
    i32, i64 = dict(dtype=torch.int32, device=dv), dict(dtype=torch.int64, device=dv)
    sel_idx, node_ptr = torch.empty(G, **i32), torch.empty(G + 1, **i32)
    edge_ptr, totals = torch.empty(G + 1, **i64), torch.empty(3, **i64)
    s = _stream()
    _lib.call("dippm_mig_band_select", _p(ws.y_pred), G, float(band_mb), _p(b.graph_ptr), _p(b.edge_ptr),
              _p(sel_idx), _p(node_ptr), _p(edge_ptr), _p(totals), s)
    count, nodes, edges = (int(v) for v in totals.cpu().tolist())
    if count == 0:
        return 0
    f32 = dict(dtype=torch.float32, device=dv)
    x, fs = torch.empty(nodes, FEATURE_WIDTH, **f32), torch.empty(count, STATIC_WIDTH, dtype=torch.float64, device=dv)
    src, dst = torch.empty(max(edges, 1), **i64), torch.empty(max(edges, 1), **i64)
    _lib.call("dippm_gather_graphs", _p(sel_idx), count, _p(node_ptr), _p(edge_ptr), _p(b.graph_ptr), _p(b.edge_ptr),
              _p(b.x), _p(b.src), _p(b.dst), _p(b.fs), _p(x), _p(src), _p(dst), _p(fs), s)
    sub = Batch(G=count, N=nodes, E=edges, x=x, src=src[:edges], dst=dst[:edges], graph_ptr=node_ptr[:count + 1],
                fs=fs, y=None, edge_ptr=edge_ptr[:count + 1], max_nodes=b.max_nodes, max_edges=b.max_edges)
    if eng32.arch == "sage":
        build_batch_csr(sub)
    ws32 = getattr(holder, "rescore_ws", None)
    if ws32 is None or ws32.N < nodes or ws32.G < count:
        holder.rescore_ws = ws32 = None
        ws32 = Workspace(eng32, max(nodes, b.N // 8), max(count, G // 8), train=False)
        holder.rescore_ws = ws32
    eng32.forward(sub, ws32, predict=True)
    _lib.call("dippm_scatter_rescore", _p(sel_idx), count, _p(ws32.y_pred), _p(ws32.mig), _p(ws.y_pred), _p(ws.mig), s)
    return count
