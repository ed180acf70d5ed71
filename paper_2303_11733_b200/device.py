"""Device engine: HBM layout, batch collation and the launch sequences of the
batched GraphSAGE forward / backward / Adam step over the C ABI.

PyTorch is used for device memory (caching allocator), streams and pinned
host buffers only; every FLOP runs in libdippm_b200.so.

HBM layout (hidden H padded to Hp = ceil64(H); padded weights are zero and
stay exactly zero under Adam, so results equal the unpadded network):
  params  fp64 [P]   master weights, reference order gnn.py:488-491, with
                     sage{l}.w_self/w_neigh adjacent -> W_cat_l [2 d_l, Hp]
  m, v    fp64 [P]   Adam moments (numerics.py:76-90)
  grads   fp32 [P]   same offsets
  p32     fp32 [P]   compute copy (biases, FC head)
  wt[l]   [Hp, 2 d_l]   K-major W_cat^T, forward B operand (bf16 / tf32 hi|lo)
  wb[l]   [2 d_l, Hp]   K-major W_cat, dgrad B operand (layers 2, 3)
Per batch (N nodes, G graphs):
  A1 [N, 64]  = [X | agg X]         A2 [N, 2Hp] = [h1 | agg h1]
  A3 [N, 2Hp] = [h2 | agg h2]       H3 [N, Hp]  = h3
  u  [G, Hp+5] = [mean_g h3 | fs_norm]
Node rows of a graph are contiguous (graph_ptr), edges carry global ids.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import Act, GemmArgs, DT_BF16, DT_F32, DT_TF32X3, GEMM_FWD, GEMM_STORE, GEMM_WGRAD
from .errors import EmptyGraph, ShapeMismatch

FEATURE_WIDTH = 32   # featurize.py:38
STATIC_WIDTH = 5     # featurize.py:39
PRECISIONS = {"fp32": DT_TF32X3, "bf16": DT_BF16}
BACKENDS = {"tc": 0, "simt": 1}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def require_device(device=None) -> torch.device:
    _lib.load()
    if not torch.cuda.is_available():
        raise _lib.DeviceUnavailable("no CUDA device visible; the DIPPM B200 path has no CPU fallback")
    return torch.device(device if device is not None else "cuda")


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


class Layout:
    """Flat parameter layout with hidden padded to a multiple of 64."""

    def __init__(self, hidden: int):
        self.hidden = hidden
        self.hp = hp = -(-hidden // 64) * 64
        self.d_in = [FEATURE_WIDTH, hp, hp]
        shapes = []
        for i, d in enumerate(self.d_in, start=1):
            shapes += [(f"sage{i}.w_self", (d, hp)), (f"sage{i}.w_neigh", (d, hp)), (f"sage{i}.bias", (hp,))]
        shapes += [("fc1.w", (hp + STATIC_WIDTH, hp)), ("fc1.b", (hp,)), ("fc2.w", (hp, hp)), ("fc2.b", (hp,)),
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
            out[:h, :h] = a[:h]
            out[hp:hp + STATIC_WIDTH, :h] = a[h:]
        elif a.ndim == 1:
            out[:a.shape[0]] = a
        else:
            out[:a.shape[0], :a.shape[1]] = a
        return out

    def unpad(self, name: str, padded: np.ndarray) -> np.ndarray:
        h, hp = self.hidden, self.hp
        shp = self.ref_shape(name)
        if name == "fc1.w":
            return np.concatenate([padded[:h, :h], padded[hp:hp + STATIC_WIDTH, :h]])
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
    fs: torch.Tensor         # f32 [G, 5] log1p static features
    y: torch.Tensor | None   # f32 [G, 3] raw targets
    rowptr: torch.Tensor | None = None
    col: torch.Tensor | None = None
    deg: torch.Tensor | None = None
    inv_deg: torch.Tensor | None = None
    t_rowptr: torch.Tensor | None = None
    t_col: torch.Tensor | None = None
    bad: torch.Tensor | None = None
    h2d_bytes: int = 0


def collate_host(encodings, fs_vectors, targets=None):
    """Host-side collation of reference-style encodings into flat arrays.

    Validation mirrors gnn.py:141-144 (EmptyGraph for N < 1, ShapeMismatch for
    a feature matrix that is not (N, 32)).  Returns numpy arrays.
    """
    G = len(encodings)
    n = np.empty(G, dtype=np.int64)
    xs, srcs, dsts = [], [], []
    off = 0
    for g, enc in enumerate(encodings):
        ng = int(enc.num_nodes)
        if ng < 1:
            raise EmptyGraph("encoding has no nodes")
        feats = np.asarray(enc.features)
        if feats.shape != (ng, FEATURE_WIDTH):
            raise ShapeMismatch(f"feature matrix {feats.shape} does not match {ng} nodes")
        e = np.asarray(enc.edges, dtype=np.int64).reshape(-1, 2)
        if e.size and (e.min() < 0 or e.max() >= ng):
            raise ShapeMismatch(f"edge endpoint outside [0, {ng})")
        xs.append(feats)
        srcs.append(e[:, 0] + off)
        dsts.append(e[:, 1] + off)
        n[g] = ng
        off += ng
    graph_ptr = np.zeros(G + 1, dtype=np.int32)
    np.cumsum(n, out=graph_ptr[1:])
    x = np.concatenate(xs).astype(np.float32) if G else np.zeros((0, FEATURE_WIDTH), np.float32)
    src = np.concatenate(srcs) if G else np.zeros(0, np.int64)
    dst = np.concatenate(dsts) if G else np.zeros(0, np.int64)
    fs = np.asarray(fs_vectors, dtype=np.float32).reshape(G, STATIC_WIDTH)
    y = None if targets is None else np.asarray(targets, dtype=np.float32).reshape(G, 3)
    return x, src, dst, graph_ptr, fs, y


def upload_batch(x, src, dst, graph_ptr, fs, y=None, device="cuda", build_csr=True) -> Batch:
    """Pinned host -> device copies of a collated batch, then K1 CSR on device."""
    dev = torch.device(device)

    def h2d(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.pin_memory().to(dev, non_blocking=True) if t.numel() else t.to(dev)

    arrays = [x, src, dst, graph_ptr, fs] + ([y] if y is not None else [])
    b = Batch(G=int(len(graph_ptr) - 1), N=int(graph_ptr[-1]), E=int(len(src)), x=h2d(x), src=h2d(src),
              dst=h2d(dst), graph_ptr=h2d(graph_ptr), fs=h2d(fs), y=None if y is None else h2d(y),
              h2d_bytes=int(sum(np.asarray(a).nbytes for a in arrays)))
    if build_csr:
        build_batch_csr(b)
    return b


def build_batch_csr(b: Batch) -> Batch:
    """K1: deterministic CSR + transposed CSR of the batch (gnn.py:130-137)."""
    dev = b.x.device
    N, E = b.N, b.E
    i32 = dict(dtype=torch.int32, device=dev)
    b.rowptr = torch.empty(N + 1, **i32)
    b.col = torch.empty(max(E, 1), **i32)
    b.deg = torch.empty(N, **i32)
    b.inv_deg = torch.empty(N, dtype=torch.float32, device=dev)
    b.t_rowptr = torch.empty(N + 1, **i32)
    b.t_col = torch.empty(max(E, 1), **i32)
    b.bad = torch.zeros(1, **i32)
    lib = _lib.load()
    ws_bytes = lib.dippm_csr_workspace_bytes(N, E)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    _lib.call("dippm_build_csr", _p(b.src), _p(b.dst), E, N, _p(b.rowptr), _p(b.col), _p(b.deg), _p(b.inv_deg),
              _p(b.t_rowptr), _p(b.t_col), _p(b.bad), _p(ws), ws_bytes, _stream())
    return b


# ---------------------------------------------------------------------------
# engine

class Workspace:
    """Per-batch activation / gradient buffers (sized for N nodes, G graphs)."""

    def __init__(self, eng: "Engine", N: int, G: int, train: bool):
        dev, dt, hp = eng.device, eng.dtype, eng.L.hp
        f32 = dict(dtype=torch.float32, device=dev)
        self.N, self.G = N, G
        self.A = [ActBuf(N, 2 * FEATURE_WIDTH, dt, dev), ActBuf(N, 2 * hp, dt, dev), ActBuf(N, 2 * hp, dt, dev)]
        self.H3 = ActBuf(N, hp, dt, dev)
        self.u = torch.empty(G, hp + STATIC_WIDTH, **f32)
        self.cache = torch.empty(4, G, hp, **f32)
        self.masks = torch.ones(2, G, hp, **f32)
        self.out = torch.empty(G, 3, **f32)
        self.y_pred = torch.empty(G, 3, dtype=torch.float64, device=dev)
        self.mig = torch.empty(G, dtype=torch.int8, device=dev)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
        self.loss = torch.zeros(4, dtype=torch.float64, device=dev)
        if train:
            self.dout = torch.empty(G, 3, **f32)
            self.du = torch.empty(G, hp + STATIC_WIDTH, **f32)
            self.head_scratch = torch.empty(_lib.load().dippm_head_scratch_floats(G, hp), **f32)
            self.dA = torch.empty(N, 2 * hp, **f32)
            self.dz = [ActBuf(N, hp, dt, dev), ActBuf(N, hp, dt, dev)]
            self.colsum = torch.empty(_lib.load().dippm_colsum_blocks(N), hp, **f32)
            lib = _lib.load()
            s_max = max(lib.dippm_wgrad_splits(hp, 2 * d, N) for d in eng.L.d_in)
            self.splits = [lib.dippm_wgrad_splits(hp, 2 * d, N) for d in eng.L.d_in]
            self.splitk = torch.empty(s_max * hp * 2 * hp, **f32)


class Engine:
    """Device-resident DIPPM GraphSAGE network (weights, Adam state, packs)."""

    def __init__(self, hidden: int, precision: str = "fp32", device=None, backend: str = "tc"):
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(PRECISIONS)}, got {precision!r}")
        if backend not in BACKENDS:
            raise ValueError(f"backend must be one of {sorted(BACKENDS)}, got {backend!r}")
        self.device = require_device(device)
        self.L = Layout(hidden)
        self.precision, self.dtype, self.backend = precision, PRECISIONS[precision], BACKENDS[backend]
        n = self.L.total
        f64 = dict(dtype=torch.float64, device=self.device)
        self.params = torch.zeros(n, **f64)
        self.m = torch.zeros(n, **f64)
        self.v = torch.zeros(n, **f64)
        self.grads = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.p32 = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.norm = torch.zeros(16, **f64)
        self.t = 0
        hp = self.L.hp
        self.wt = [ActBuf(hp, 2 * d, self.dtype, self.device) for d in self.L.d_in]
        self.wb = [None] + [ActBuf(2 * d, hp, self.dtype, self.device) for d in self.L.d_in[1:]]
        self.launches = 0
        self.gemm_hook = None  # bench instrumentation: called ("pre"|"post", flops) around each GEMM

    # -- parameters -----------------------------------------------------------
    def set_params(self, items, normalizer) -> None:
        host = np.zeros(self.L.total, dtype=np.float64)
        for name, arr in items:
            off = self.L.offsets[name]
            padded = self.L.pad(name, arr)
            host[off:off + padded.size] = padded.ravel()
        self.params.copy_(torch.from_numpy(host), non_blocking=False)
        self.set_normalizer(normalizer)
        self.refresh()

    def set_normalizer(self, norm) -> None:
        vec = np.concatenate([np.asarray(norm.y_mean, np.float64), np.asarray(norm.y_std, np.float64),
                              np.asarray(norm.fs_mean, np.float64), np.asarray(norm.fs_std, np.float64)])
        self.norm.copy_(torch.from_numpy(vec))

    def reset_adam(self) -> None:
        self.m.zero_()
        self.v.zero_()
        self.t = 0

    def get_params(self) -> dict:
        host = self.params.cpu().numpy()
        return {name: self.L.unpad(name, host[off:off + int(np.prod(self.L.shapes[name]))].reshape(self.L.shapes[name]))
                for name, off in self.L.offsets.items()}

    def get_grads(self) -> dict:
        host = self.grads.double().cpu().numpy()
        return {name: self.L.unpad(name, host[off:off + int(np.prod(self.L.shapes[name]))].reshape(self.L.shapes[name]))
                for name, off in self.L.offsets.items()}

    def refresh(self) -> None:
        """Pack fp64 masters into the fp32 copy and the GEMM operand layouts."""
        s = _stream()
        L = self.L
        n = L.total
        _lib.call("dippm_pack", _p(self.params), 1, n, 0, Act(self.p32.data_ptr(), n, 0, DT_F32), s)
        for i, d in enumerate(L.d_in):
            w = self.params[L.offsets[f"sage{i + 1}.w_self"]:]
            _lib.call("dippm_pack", _p(w), 2 * d, L.hp, 1, self.wt[i].view(), s)
            if i > 0:
                _lib.call("dippm_pack", _p(w), 2 * d, L.hp, 0, self.wb[i].view(), s)
        self.launches += 1 + len(L.d_in) + len(L.d_in) - 1

    def adam_step(self, lr: float, beta1=0.9, beta2=0.999, eps=1e-8, grad_scale: float = 1.0) -> None:
        """numerics.adam_step over all 15 tensors (one launch), then repack."""
        self.t += 1
        _lib.call("dippm_adam", _p(self.params), _p(self.m), _p(self.v), _p(self.grads), grad_scale, self.L.total, self.t,
                  lr, beta1, beta2, eps, _stream())
        self.launches += 1
        self.refresh()

    # -- kernels --------------------------------------------------------------
    def _gemm(self, kind, M, N, K, a, a_mn, b, b_mn, bias=None, relu=0, out=NULL_ACT, c=None, ldc=0, splits=1):
        args = GemmArgs(kind, M, N, K, a, a_mn, b, b_mn, bias, relu, out, c, ldc, splits)
        if self.gemm_hook is not None:
            self.gemm_hook("pre", 2.0 * M * N * K)
        _lib.check(_lib.load().dippm_gemm(args, self.backend, _stream()), "dippm_gemm")
        if self.gemm_hook is not None:
            self.gemm_hook("post", 2.0 * M * N * K)
        self.launches += 1

    def forward(self, b: Batch, ws: Workspace, mask_mode: int = 0, dropout_p: float = 0.0, seed: int = 0,
                predict: bool = True) -> None:
        """Eval (mask_mode 0) or train-mode forward: K2 -> K3 x3, K4, K5."""
        s, L, hp = _stream(), self.L, self.L.hp
        P32 = self.p32
        bias = lambda i: P32.data_ptr() + 4 * L.offsets[f"sage{i}.bias"]  # noqa: E731
        # layer 1: A1 = [X | agg X]
        _lib.call("dippm_sage_aggregate", f32_act(b.x), ws.A[0].view(FEATURE_WIDTH), ws.A[0].view(0), b.N,
                  FEATURE_WIDTH, _p(b.rowptr), _p(b.col), _p(b.inv_deg), s)
        outs = [ws.A[1].view(0), ws.A[2].view(0), ws.H3.view(0)]
        for i in range(3):
            if i > 0:
                _lib.call("dippm_sage_aggregate", ws.A[i].view(0), ws.A[i].view(hp), NULL_ACT, b.N, hp,
                          _p(b.rowptr), _p(b.col), _p(b.inv_deg), s)
            self._gemm(GEMM_FWD, b.N, hp, 2 * L.d_in[i], ws.A[i].view(0), 0, self.wt[i].view(), 0,
                       bias=bias(i + 1), relu=1, out=outs[i])
        _lib.call("dippm_pool_concat", ws.H3.view(0), _p(b.graph_ptr), b.G, hp, _p(b.fs), _p(self.norm),
                  _p(ws.u), s)
        _lib.call("dippm_head_forward", _p(ws.u), b.G, hp, P32.data_ptr() + 4 * L.head_off, _p(ws.cache),
                  _p(ws.masks), mask_mode, float(dropout_p), int(seed) & (2**64 - 1), _p(ws.out), _p(self.norm),
                  _p(ws.y_pred) if predict else None, _p(ws.mig) if predict else None, _p(ws.nonfinite), s)
        self.launches += 3 + 2 + 5

    def loss(self, b: Batch, ws: Workspace, delta: float = 1.0) -> None:
        _lib.call("dippm_huber", _p(ws.out), _p(b.y), b.G, _p(self.norm), float(delta), _p(ws.dout), _p(ws.loss),
                  _stream())
        self.launches += 1

    def backward(self, b: Batch, ws: Workspace, use_masks: bool) -> None:
        """Head backward, readout backward, 3 x (WGRAD, DGRAD, transposed gather)."""
        s, L, hp, N = _stream(), self.L, self.L.hp, b.N
        G32 = self.grads.data_ptr()
        off = lambda name: G32 + 4 * L.offsets[name]  # noqa: E731
        lib = _lib.load()
        nblk = lib.dippm_colsum_blocks(N)
        _lib.call("dippm_head_backward", _p(ws.u), b.G, hp, self.p32.data_ptr() + 4 * L.head_off, _p(ws.cache),
                  _p(ws.masks), int(use_masks), _p(ws.dout), off("fc1.w"), _p(ws.du), _p(ws.head_scratch), s)
        _lib.call("dippm_readout_backward", _p(ws.du), hp + STATIC_WIDTH, _p(b.graph_ptr), b.G, hp, ws.H3.view(0),
                  ws.dz[0].view(), N, _p(ws.colsum), s)
        _lib.call("dippm_reduce_rows", _p(ws.colsum), nblk, hp, hp, 1.0, off("sage3.bias"), s)
        cur = 0
        for i in (2, 1, 0):
            width = 2 * L.d_in[i]
            dz = ws.dz[cur]
            S = ws.splits[i]
            self._gemm(GEMM_WGRAD, hp, width, N, dz.view(), 1, ws.A[i].view(0), 1, c=_p(ws.splitk), ldc=width,
                       splits=S)
            _lib.call("dippm_splitk_reduce_t", _p(ws.splitk), S, hp, width, 1.0, off(f"sage{i + 1}.w_self"), hp, s)
            if i == 0:
                break
            self._gemm(GEMM_STORE, N, width, hp, dz.view(), 0, self.wb[i].view(), 0, c=_p(ws.dA), ldc=width)
            nxt = ws.dz[1 - cur]
            _lib.call("dippm_sage_backward_gather", _p(ws.dA), width, hp, ws.A[i].view(0), nxt.view(), N,
                      _p(b.t_rowptr), _p(b.t_col), _p(b.inv_deg), _p(ws.colsum), s)
            _lib.call("dippm_reduce_rows", _p(ws.colsum), nblk, hp, hp, 1.0, off(f"sage{i}.bias"), s)
            cur = 1 - cur
        self.launches += 3 + 11 + 3 * 2 - 1
