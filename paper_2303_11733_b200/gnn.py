"""DIPPM GraphSAGE predictor — drop-in for the reference `dippm.gnn` (gnn.py:1-578).

Same public names, argument meanings, return types and error behaviour; the
arithmetic runs on the B200 through libdippm_b200.so (see device.py).  The
host model object keeps the fp64 "truth" exactly like the reference
(`param_items()` returns live numpy arrays that callers may mutate); each call
uploads the current values, so in-place edits between calls are honoured.

Additions (batched surface): `predict_batch`, `predict_records`,
`TrainConfig.batch_size / precision / device`.

Numerics: `precision="fp32"` (default) runs the SAGE GEMMs as 3-pass TF32 on
the tensor cores (fp32-grade), everything else in fp32 with fp64 Adam
masters; `precision="bf16"` uses bf16 GEMM operands with fp32 accumulation.
Stated tolerances vs the fp64 reference: see DESIGN.md §Parity.
"""

from __future__ import annotations

import json
import math
import threading
from dataclasses import dataclass
from pathlib import Path
from types import SimpleNamespace
from typing import ClassVar

import numpy as np
import torch

from . import _lib, device as dev
from ._lib import Act
from .device import ActBuf, Batch, Engine, Workspace, collate_host, f32_act, upload_batch
from .errors import EmptyDataset, EmptyGraph, IoFailure, NonFinite, ShapeMismatch, VersionMismatch
from .mig import profile_from_code
from .types import FEATURE_WIDTH, STATIC_WIDTH, VOCAB_VERSION, TargetVector, fs_vector, target_vector

DEFAULT_HIDDEN = 512          # gnn.py:42
DEFAULT_DROPOUT = 0.05        # gnn.py:43
DEFAULT_LEARNING_RATE = 2.754e-5  # numerics.py:17


@dataclass
class SageLayerParams:
    w_self: np.ndarray   # (d_in, d_out)
    w_neigh: np.ndarray  # (d_in, d_out)
    bias: np.ndarray     # (d_out,)


@dataclass
class AffineParams:
    w: np.ndarray  # (d_in, d_out)
    b: np.ndarray  # (d_out,)


@dataclass
class Normalizer:
    """Z-score statistics for targets and static features (gnn.py:59-97)."""

    y_mean: np.ndarray
    y_std: np.ndarray
    fs_mean: np.ndarray
    fs_std: np.ndarray

    @classmethod
    def identity(cls) -> "Normalizer":
        return cls(np.zeros(3), np.ones(3), np.zeros(STATIC_WIDTH), np.ones(STATIC_WIDTH))

    @classmethod
    def fit(cls, targets: np.ndarray, statics: np.ndarray) -> "Normalizer":
        def clamp(std):
            std = std.copy()
            std[std < 1e-9] = 1.0
            return std

        return cls(y_mean=targets.mean(axis=0), y_std=clamp(targets.std(axis=0)),
                   fs_mean=statics.mean(axis=0), fs_std=clamp(statics.std(axis=0)))

    def normalize_y(self, y: np.ndarray) -> np.ndarray:
        return (y - self.y_mean) / self.y_std

    def denormalize_y(self, y: np.ndarray) -> np.ndarray:
        return y * self.y_std + self.y_mean

    def normalize_fs(self, fs: np.ndarray) -> np.ndarray:
        return (fs - self.fs_mean) / self.fs_std


@dataclass
class TrainConfig:
    """gnn.py:100-117 plus the batched-training knobs.

    batch_size=1 reproduces the reference protocol (one Adam step per record,
    host-drawn PCG64 dropout masks in the reference draw order); batch_size>1
    takes one Adam step per batch on the batch-mean gradient (gnn.backward's
    objective) with device-generated dropout masks.
    """

    epochs: int
    lr: float = DEFAULT_LEARNING_RATE
    seed: int = 0
    hidden: int = DEFAULT_HIDDEN
    huber_delta: float = 1.0
    shuffle: bool = True
    batch_size: int = 1
    precision: str = "fp32"
    device: str | None = None

    def __post_init__(self):
        if self.epochs < 1:
            raise ValueError(f"epochs must be >= 1, got {self.epochs}")
        if self.lr <= 0:
            raise ValueError(f"learning rate must be positive, got {self.lr}")
        if self.hidden < 1:
            raise ValueError(f"hidden width must be >= 1, got {self.hidden}")
        if self.huber_delta <= 0:
            raise ValueError(f"huber delta must be positive, got {self.huber_delta}")
        if self.batch_size < 1:
            raise ValueError(f"batch size must be >= 1, got {self.batch_size}")
        if self.precision not in dev.PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(dev.PRECISIONS)}, got {self.precision!r}")


def _glorot(rng: np.random.Generator, fan_in: int, fan_out: int) -> np.ndarray:
    return rng.normal(0.0, math.sqrt(2.0 / (fan_in + fan_out)), size=(fan_in, fan_out))


def _fc_stack(rng, dims):
    return [AffineParams(w=_glorot(rng, di, do), b=np.zeros(do)) for di, do in dims]


@dataclass
class DippmModel:
    """Trained weights of the graph network plus its normalizers (gnn.py:178-200)."""

    sage: list
    fc: list
    dropout_p: float
    normalizer: Normalizer
    hidden: int
    vocab_version: str = VOCAB_VERSION

    arch: ClassVar[str] = "sage"

    def param_items(self) -> list:
        items = []
        for i, layer in enumerate(self.sage, start=1):
            items.append((f"sage{i}.w_self", layer.w_self))
            items.append((f"sage{i}.w_neigh", layer.w_neigh))
            items.append((f"sage{i}.bias", layer.bias))
        for i, layer in enumerate(self.fc, start=1):
            items.append((f"fc{i}.w", layer.w))
            items.append((f"fc{i}.b", layer.b))
        return items

    def forward_norm(self, prep, fs_norm, train: bool = False, rng=None, precision: str = "fp32"):
        """gnn.py:212-217 on the device: embed -> mean readout -> [r | fs_norm] -> FC head.
        Returns (out (3,) normalised, cache); the cache keeps the activations in HBM."""
        return _device_forward_norm(self, prep, fs_norm, train, rng, precision)

    def backward_from(self, cache, dout) -> dict:
        """gnn.py:219-233 on the device: every parameter's gradient of <out, dout>."""
        return _device_backward_from(self, cache, dout)


@dataclass
class MlpModel:
    """Baseline that regresses from the static features alone (gnn.py:236-262).

    Same head as DippmModel but fc1 reads only the 5 normalised static
    features; runs on the same tcgen05 head kernels (device arch "mlp")."""

    fc: list
    dropout_p: float
    normalizer: Normalizer
    hidden: int
    vocab_version: str = VOCAB_VERSION

    arch: ClassVar[str] = "mlp"

    def param_items(self) -> list:
        items = []
        for i, layer in enumerate(self.fc, start=1):
            items.append((f"fc{i}.w", layer.w))
            items.append((f"fc{i}.b", layer.b))
        return items

    def forward_norm(self, prep, fs_norm, train: bool = False, rng=None, precision: str = "fp32"):
        """gnn.py:255-257 on the device: the FC head on fs_norm alone."""
        return _device_forward_norm(self, prep, fs_norm, train, rng, precision)

    def backward_from(self, cache, dout) -> dict:
        """gnn.py:259-262 on the device."""
        return _device_backward_from(self, cache, dout)


def create_model(hidden: int = DEFAULT_HIDDEN, seed: int = 0, dropout_p: float = DEFAULT_DROPOUT,
                 normalizer: Normalizer | None = None) -> DippmModel:
    """Glorot-normal init in the reference draw order (gnn.py:302-319)."""
    return _new_sage_model(hidden, np.random.default_rng(seed), dropout_p, normalizer or Normalizer.identity())


def create_mlp_model(hidden: int = DEFAULT_HIDDEN, seed: int = 0, dropout_p: float = DEFAULT_DROPOUT,
                     normalizer: Normalizer | None = None) -> MlpModel:
    """gnn.py:307-309: Glorot-normal fc1..fc3 in the reference draw order."""
    return _new_mlp_model(hidden, np.random.default_rng(seed), dropout_p, normalizer or Normalizer.identity())


def _new_mlp_model(hidden, rng, dropout_p, normalizer) -> MlpModel:
    fc = _fc_stack(rng, [(STATIC_WIDTH, hidden), (hidden, hidden), (hidden, 3)])  # gnn.py:322-324
    return MlpModel(fc=fc, dropout_p=dropout_p, normalizer=normalizer, hidden=hidden)


def _new_sage_model(hidden, rng, dropout_p, normalizer) -> DippmModel:
    dims = [(FEATURE_WIDTH, hidden), (hidden, hidden), (hidden, hidden)]
    sage = [SageLayerParams(w_self=_glorot(rng, di, do), w_neigh=_glorot(rng, di, do), bias=np.zeros(do))
            for di, do in dims]
    fc = _fc_stack(rng, [(hidden + STATIC_WIDTH, hidden), (hidden, hidden), (hidden, 3)])
    return DippmModel(sage=sage, fc=fc, dropout_p=dropout_p, normalizer=normalizer, hidden=hidden)


# ---------------------------------------------------------------------------
# per-record preparation and the duck-typed model protocol (gnn.py:120-154, 212-262)

@dataclass
class _Prepared:
    """Per-record arrays (gnn.py:120-127).  The reference's dense aggregation matrix is
    replaced by the edge list: the device builds the CSR (K1) from it at forward time."""

    num_nodes: int
    features: np.ndarray      # (N, 32) float64
    edges: np.ndarray         # (E, 2) int64, (src, dst) producer -> consumer
    fs_raw: np.ndarray        # (5,) log1p static features
    y_raw: np.ndarray | None  # (3,) original-unit targets, None at predict time


def _prepare_encoding(encoding, fs, target=None) -> _Prepared:
    """gnn.py:140-150: validation (EmptyGraph, ShapeMismatch) + the arrays the forward needs."""
    n = int(encoding.num_nodes)
    if n < 1:
        raise EmptyGraph("encoding has no nodes")
    feats = np.asarray(encoding.features)
    if feats.shape != (n, FEATURE_WIDTH):
        raise ShapeMismatch(f"feature matrix {feats.shape} does not match {n} nodes")
    e = np.asarray(encoding.edges, dtype=np.int64).reshape(-1, 2)
    if e.size and (e.min() < 0 or e.max() >= n):
        raise ShapeMismatch(f"edge endpoint outside [0, {n})")
    return _Prepared(num_nodes=n, features=np.asarray(feats, dtype=np.float64), edges=e, fs_raw=fs_vector(fs),
                     y_raw=None if target is None else target_vector(target))


def _prepare_record(record) -> _Prepared:
    """gnn.py:153-154."""
    return _prepare_encoding(record.encoding, record.fs, record.target)


class _DeviceCache:
    """What forward_norm hands to backward_from: the device batch and the training workspace
    holding the layer activations and ReLU masks (the reference caches (h, m, z) per layer
    and the head inputs on the host, gnn.py:217)."""

    __slots__ = ("precision", "batch", "ws", "keep")

    def __init__(self, precision, batch, ws, keep):
        self.precision, self.batch, self.ws, self.keep = precision, batch, ws, keep


def _device_forward_norm(model, prep, fs_norm, train, rng, precision):
    masks = _draw_masks(model, rng) if train else None  # gnn.py:277-281 draw order (fc1, fc2)
    eng = _engine(model, precision)
    n = prep.num_nodes
    fsn = np.asarray(fs_norm, dtype=np.float64).reshape(1, STATIC_WIDTH)
    e = prep.edges
    b = upload_batch(prep.features.astype(np.float32), e[:, 0].copy(), e[:, 1].copy(), np.array([0, n], np.int32),
                     fsn, device=eng.device, build_csr=model.arch == "sage")
    ws = Workspace(eng, b.N, 1, train=True)
    if masks is not None:
        ws.masks[:, :, :masks.shape[-1]].copy_(torch.from_numpy(masks.astype(np.float32)))
    # fs_norm comes from the caller already normalised (gnn.py:353): the device skips its z-score
    eng.forward(b, ws, mask_mode=1 if masks is not None else 0, predict=False, fs_normalized=True)
    eng.check_batch(b)
    keep = 1.0 / (1.0 - model.dropout_p) if masks is not None else 1.0
    return ws.out[0].double().cpu().numpy(), _DeviceCache(precision, b, ws, keep)


def _device_backward_from(model, cache, dout) -> dict:
    if not isinstance(cache, _DeviceCache):
        raise TypeError("backward_from needs the cache returned by this package's forward_norm")
    dout = np.asarray(dout, dtype=np.float64)
    if dout.shape != (3,):
        raise ShapeMismatch(f"dout must have shape (3,), got {dout.shape}")
    # the reference's backward reads the model's CURRENT weights with the cached activations
    eng = _engine(model, cache.precision)
    ws = cache.ws
    ws.dout[0].copy_(torch.from_numpy(dout.astype(np.float32)))
    eng.backward(cache.batch, ws, keep_scale=cache.keep)
    return eng.get_grads()


# ---------------------------------------------------------------------------
# engine binding

_ENGINE_LOCK = threading.Lock()


def _engine(model, precision: str = "fp32", device=None) -> Engine:
    """Device engine for `model`, refreshed from the model's current host values."""
    arch = getattr(model, "arch", "sage")
    if device is not None and torch.device(device) == torch.device("cuda", torch.cuda.current_device()):
        device = None
    key = (precision, str(device), int(model.hidden), arch)
    with _ENGINE_LOCK:
        cache = model.__dict__.setdefault("_b200_engines", {})
        eng = cache.get(key)
        if eng is None:
            eng = Engine(model.hidden, precision, device, arch=arch)
            cache[key] = eng
    eng.set_params(model.param_items(), model.normalizer)
    return eng


def _records_arrays(encodings, fss, targets=None):
    return collate_host(encodings, [fs_vector(f) for f in fss],
                        None if targets is None else [target_vector(t) for t in targets])


def _grow(holder, key, eng: Engine, N: int, G: int, train: bool) -> Workspace:
    """A grow-only workspace kept in `holder` under `key`: reused for every batch that fits
    (workspaces accept batches smaller than their capacity), regrown x1.25 otherwise, so
    batches of ever-different node counts cost one allocation, not one each."""
    ws = getattr(holder, key, None)
    if ws is None or ws.N < N or ws.G < G:
        if ws is not None:  # drop the old buffers before allocating the larger set
            setattr(holder, key, None)
            del ws
        old = getattr(holder, key + "_cap", (0, 0))
        ws = Workspace(eng, max(N, int(1.25 * old[0])), max(G, int(1.25 * old[1])), train=train)
        setattr(holder, key, ws)
        setattr(holder, key + "_cap", (ws.N, ws.G))
    return ws


def _thread_slots(eng: Engine):
    """Per-thread workspace slots of an engine: concurrent read-only predict calls on one
    shared model never share activation buffers (the reference guarantees concurrent
    inference on a trained model)."""
    tls = eng.__dict__.get("_tls")
    if tls is None:
        tls = eng.__dict__.setdefault("_tls", threading.local())
    return tls


def infer_workspace(eng: Engine, N: int, G: int) -> Workspace:
    """This thread's reusable inference workspace for the engine (grow-only)."""
    return _grow(_thread_slots(eng), "infer", eng, N, G, train=False)


def train_workspace(eng: Engine, N: int, G: int) -> Workspace:
    """This thread's reusable training workspace for the engine (grow-only)."""
    return _grow(_thread_slots(eng), "train", eng, N, G, train=True)


def _run_forward(eng: Engine, encodings, fss, targets=None, mask_mode=0, masks=None, train_buffers=False):
    x, src, dst, gp, fs, y = _records_arrays(encodings, fss, targets)
    b = upload_batch(x, src, dst, gp, fs, y, device=eng.device, build_csr=eng.arch == "sage")
    ws = train_workspace(eng, b.N, b.G) if train_buffers else infer_workspace(eng, b.N, b.G)
    if masks is not None:
        ws.masks[:, :, :masks.shape[-1]].copy_(torch.from_numpy(masks.astype(np.float32)))
    eng.forward(b, ws, mask_mode=mask_mode)
    return b, ws


def _readback(*tensors):
    """Device -> pinned host copies of several results, then ONE wait for all of them."""
    outs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in tensors]
    for o, t in zip(outs, tensors):
        o.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return [o.numpy() for o in outs]


def _check_flags(b, ws, bad_flag, nonfinite_flag):
    if b is not None and b.bad is not None and int(bad_flag[0]):
        raise ShapeMismatch("edge endpoint outside its graph's node range")
    if nonfinite_flag is not None and int(nonfinite_flag[0]):
        raise NonFinite("predicted memory is NaN or infinite")


def _check_mode(mode):
    if mode not in ("train", "eval"):
        raise ValueError(f'mode must be "train" or "eval", got {mode!r}')


def _draw_masks(model, rng, G=1):
    """Host PCG64 dropout masks in the reference draw order (gnn.py:277-281 -> numerics.py:45-55)."""
    from .numerics import dropout_mask
    if model.dropout_p <= 0.0:
        return None
    if rng is None:
        raise ValueError("training-mode forward needs an rng for dropout")
    out = np.ones((2, G, model.hidden))
    for g in range(G):
        out[0, g] = dropout_mask((model.hidden,), model.dropout_p, rng)
        out[1, g] = dropout_mask((model.hidden,), model.dropout_p, rng)
    return out


# ---------------------------------------------------------------------------
# public forward / backward surface (gnn.py:331-405)

def sage_forward(encoding, layer: SageLayerParams, h_in: np.ndarray, precision: str = "fp32") -> np.ndarray:
    """One message-passing block over the encoding's predecessor edges (gnn.py:331-338)."""
    h_in = np.asarray(h_in)
    if h_in.ndim != 2 or h_in.shape[0] != encoding.num_nodes:
        raise ShapeMismatch(f"h_in {h_in.shape} does not cover {encoding.num_nodes} nodes")
    w_self, w_neigh, bias = (np.asarray(layer.w_self), np.asarray(layer.w_neigh), np.asarray(layer.bias))
    if h_in.shape[1] != w_self.shape[0]:
        raise ShapeMismatch(f"h_in width {h_in.shape[1]} vs layer input {w_self.shape[0]}")
    device = dev.require_device()
    n, d_in, d_out = h_in.shape[0], h_in.shape[1], w_self.shape[1]
    if n < 1:
        raise EmptyGraph("encoding has no nodes")
    dip, dop = _agg_width(d_in, 32), -(-d_out // 64) * 64
    e = np.asarray(encoding.edges, dtype=np.int64).reshape(-1, 2)
    if e.size and (e.min() < 0 or e.max() >= n):
        raise ShapeMismatch(f"edge endpoint outside [0, {n})")
    xp = np.zeros((n, dip), np.float32)
    xp[:, :d_in] = h_in
    b = upload_batch(np.zeros((n, FEATURE_WIDTH), np.float32), e[:, 0].copy(), e[:, 1].copy(),
                     np.array([0, n], np.int32), np.zeros((1, STATIC_WIDTH)), device=device)
    dt = dev.PRECISIONS[precision]
    w_cat = np.zeros((2 * dip, dop))
    w_cat[:d_in, :d_out] = w_self
    w_cat[dip:dip + d_in, :d_out] = w_neigh
    bp = np.zeros(dop, np.float32)
    bp[:d_out] = bias
    xt = torch.from_numpy(xp).to(device)
    wt64 = torch.from_numpy(w_cat).to(device)
    bt = torch.from_numpy(bp).to(device)
    A = ActBuf(n, 2 * dip, dt, device)
    Wt = ActBuf(dop, 2 * dip, dt, device)
    out = ActBuf(n, dop, dev.DT_F32, device)
    s = dev._stream()
    for c0 in range(0, dip, 1024):  # the aggregation kernel takes widths up to 1024
        w = min(dip - c0, 1024)
        _lib.call("dippm_sage_aggregate", Act(xt.data_ptr() + 4 * c0, dip, 0, dev.DT_F32), A.view(dip + c0),
                  A.view(c0), n, w, b.rowptr.data_ptr(), b.col.data_ptr(), b.inv_deg.data_ptr(), s)
    _lib.call("dippm_pack", wt64.data_ptr(), 2 * dip, dop, 1, Wt.view(), s)
    args = _lib.GemmArgs(_lib.GEMM_FWD, n, dop, 2 * dip, A.view(0), 0, Wt.view(), 0, bt.data_ptr(), 1, out.view(),
                         None, 0, 1)
    _lib.check(_lib.load().dippm_gemm(args, 0, s), "dippm_gemm")
    return out.t[:, :d_out].double().cpu().numpy()


def _agg_width(d: int, lo: int) -> int:
    """Padded width for the aggregation / pooling kernels (device.agg_width): the next width
    whose 8-column chunks tile a warp, a multiple of lo; beyond 1024 a multiple of 1024."""
    return dev.agg_width(d, lo)


def readout_mean(z: np.ndarray) -> np.ndarray:
    """Arithmetic mean over node embeddings (gnn.py:341-345), on device (K4), any width."""
    z = np.asarray(z)
    if z.ndim != 2 or z.shape[0] < 1:
        raise EmptyGraph("readout needs at least one node embedding")
    device = dev.require_device()
    n, d = z.shape
    dp = _agg_width(d, 8)
    zp = torch.zeros(n, dp, dtype=torch.float32)
    zp[:, :d] = torch.from_numpy(np.asarray(z, dtype=np.float32))
    zt = zp.to(device)
    gp = torch.tensor([0, n], dtype=torch.int32, device=device)
    fs = torch.zeros(1, STATIC_WIDTH, dtype=torch.float64, device=device)
    norm = torch.tensor([0.0] * 6 + [0.0] * 5 + [1.0] * 5, dtype=torch.float64, device=device)
    # two rows: a column chunk also writes its [fs | 0] tail past its own columns; chunks run in
    # ascending order, so the tail lands on the next chunk's columns (rewritten next) or row 1
    u = torch.empty(2, dp + 8, dtype=torch.float32, device=device)
    for c0 in range(0, dp, 1024):
        w = min(dp - c0, 1024)
        _lib.call("dippm_pool_concat", Act(zt.data_ptr() + 4 * c0, dp, 0, dev.DT_F32), gp.data_ptr(), 1, w,
                  fs.data_ptr(), norm.data_ptr(), Act(u.data_ptr() + 4 * c0, dp + 8, 0, dev.DT_F32), dev._stream())
    return u[0, :d].double().cpu().numpy()


def forward(encoding, fs, model, mode: str = "eval", rng=None, precision: str = "fp32") -> np.ndarray:
    """Normalised-space prediction for one graph (gnn.py:348-355)."""
    _check_mode(mode)
    masks = _draw_masks(model, rng) if mode == "train" else None
    eng = _engine(model, precision)
    b, ws = _run_forward(eng, [encoding], [fs], mask_mode=1 if masks is not None else 0, masks=masks)
    out, bad = _readback(ws.out[0], b.bad if b.bad is not None else ws.nonfinite)
    _check_flags(b, ws, bad, None)
    return out.astype(np.float64)


def mig_rescore(model, eng: Engine, b, ws, precision: str) -> int:
    """bf16 predictions: re-score the graphs near a MIG ceiling in fp32 so the picks are the
    reference's (see device.mig_band_rescore).  Returns the number re-scored (0 in fp32)."""
    if precision != "bf16":
        return 0
    band = dev.BF16_MIG_BAND * float(np.asarray(model.normalizer.y_std)[1])
    return dev.mig_band_rescore(_engine(model, "fp32", eng.device), b, ws, band, _thread_slots(eng))


def predict_batch(model, encodings, fss, precision: str = "fp32", check_nonfinite: bool = True,
                  info: dict | None = None):
    """Batched eval prediction: (y float64 [G, 3] in original units, MIG codes int8 [G]).

    MIG codes: 0=1g.5gb, 1=2g.10gb, 2=3g.20gb, 3=7g.40gb, -1=None; computed on
    the device from y[:, 1] with the same rule as mig.mig_profile.  A NaN/Inf predicted
    memory raises NonFinite like mig_profile (mig.py:38-39) unless check_nonfinite=False
    (then its code is -1 and y carries the NaN, as the reference's predict returns it).
    precision="bf16": graphs whose bf16 memory prediction is within the stated bf16
    tolerance of a profile ceiling are re-scored in fp32 (their y and pick are the fp32
    ones), so picks match the reference's wherever fp32 does; info["mig_rescored"] counts them.
    """
    if len(encodings) != len(fss):
        raise ShapeMismatch(f"{len(encodings)} encodings vs {len(fss)} static-feature vectors")
    if not encodings:
        raise EmptyDataset("batch is empty")
    eng = _engine(model, precision)
    b, ws = _run_forward(eng, encodings, fss)
    G = len(encodings)
    n_band = mig_rescore(model, eng, b, ws, precision)
    if info is not None:
        info["mig_rescored"] = n_band
    y, mig, bad, nf = _readback(ws.y_pred[:G], ws.mig[:G], b.bad if b.bad is not None else ws.nonfinite,
                                ws.nonfinite)
    _check_flags(b, ws, bad, nf if check_nonfinite else None)
    return y, mig


def predict(model, encoding, fs, precision: str = "fp32") -> TargetVector:
    """Original-unit eval-mode prediction (gnn.py:358-361)."""
    y, _ = predict_batch(model, [encoding], [fs], precision, check_nonfinite=False)
    return TargetVector(latency_ms=float(y[0, 0]), memory_mb=float(y[0, 1]), energy_j=float(y[0, 2]))


def predict_record(model, record, precision: str = "fp32") -> TargetVector:
    return predict(model, record.encoding, record.fs, precision)


def predict_records(model, records, precision: str = "fp32", with_mig: bool = False):
    """Batched `predict_record` over many records (one device pass)."""
    y, mig = predict_batch(model, [r.encoding for r in records], [r.fs for r in records], precision,
                           check_nonfinite=with_mig)
    preds = [TargetVector(latency_ms=float(a), memory_mb=float(b), energy_j=float(c)) for a, b, c in y]
    if with_mig:
        return preds, [profile_from_code(int(c)) for c in mig]
    return preds


def batch_loss(model, records, huber_delta: float = 1.0, precision: str = "fp32") -> float:
    """Mean eval-mode Huber loss over a batch, in normalised space (gnn.py:368-380)."""
    if not records:
        raise EmptyDataset("batch is empty")
    eng = _engine(model, precision)
    b, ws = _run_forward(eng, [r.encoding for r in records], [r.fs for r in records],
                         [r.target for r in records], train_buffers=True)
    eng.loss(b, ws, huber_delta)
    loss, bad = _readback(ws.loss[:1], b.bad if b.bad is not None else ws.nonfinite)
    _check_flags(b, ws, bad, None)
    return float(loss[0])


def backward(model, records, huber_delta: float = 1.0, precision: str = "fp32"):
    """Mean batch Huber loss plus exact gradients for every parameter (gnn.py:383-405).

    Dropout is off (eval-mode forward).  Returns (loss, {name: fp64 ndarray}).
    """
    if not records:
        raise EmptyDataset("batch is empty")
    eng = _engine(model, precision)
    b, ws = _run_forward(eng, [r.encoding for r in records], [r.fs for r in records],
                         [r.target for r in records], train_buffers=True)
    eng.loss(b, ws, huber_delta)
    eng.backward(b, ws)
    loss, bad = _readback(ws.loss[:1], b.bad if b.bad is not None else ws.nonfinite)
    _check_flags(b, ws, bad, None)
    return float(loss[0]), eng.get_grads()


# ---------------------------------------------------------------------------
# training (gnn.py:412-482)

def train(train_records, val_records, config: TrainConfig):
    """Fit the graph network; returns the final-epoch model and history."""
    return _fit(_new_sage_model, train_records, val_records, config)


def train_mlp(train_records, val_records, config: TrainConfig):
    """Fit the static-features-only baseline with the identical protocol (gnn.py:418-421)."""
    return _fit(_new_mlp_model, train_records, val_records, config)


def _fit(make_model, train_records, val_records, config: TrainConfig):
    if not train_records:
        raise EmptyDataset("training split is empty")
    rng = np.random.default_rng(config.seed)
    targets = np.stack([target_vector(r.target) for r in train_records])
    statics = np.stack([fs_vector(r.fs) for r in train_records])
    normalizer = Normalizer.fit(targets, statics)
    model = make_model(config.hidden, rng, DEFAULT_DROPOUT, normalizer)
    eng = Engine(config.hidden, config.precision, config.device, arch=model.arch)
    eng.set_params(model.param_items(), normalizer)
    sage = model.arch == "sage"
    n = len(train_records)
    B = config.batch_size
    dropout = model.dropout_p > 0.0
    keep = 1.0 / (1.0 - model.dropout_p) if dropout else 1.0

    if B == 1:
        batches = [upload_batch(*_records_arrays([r.encoding], [r.fs], [r.target]), device=eng.device,
                                build_csr=sage) for r in train_records]
    n_max = max(b.N for b in batches) if B == 1 else None
    ws1 = Workspace(eng, n_max, 1, train=True) if B == 1 else None
    slots = SimpleNamespace()  # grow-only training / evaluation workspaces
    acc = torch.zeros(4, dtype=torch.float64, device=eng.device)
    history = []
    step = 0
    for epoch in range(1, config.epochs + 1):
        order = rng.permutation(n) if config.shuffle else np.arange(n)
        acc.zero_()
        if B == 1:
            for i in order:
                b = batches[i]
                if dropout:
                    m = _draw_masks(model, rng)
                    ws1.masks[:, :, :model.hidden].copy_(torch.from_numpy(m.astype(np.float32)), non_blocking=True)
                eng.forward(b, ws1, mask_mode=1 if dropout else 0, predict=False, defer_head=True)
                eng.loss(b, ws1, config.huber_delta)
                eng.backward(b, ws1, keep_scale=keep, advance_step=True)
                acc.add_(ws1.loss)  # after backward: a deferred fused head computes the loss there
                eng.adam_step(config.lr)
        else:
            for s0 in range(0, n, B):
                idx = order[s0:s0 + B]
                recs = [train_records[i] for i in idx]
                b = upload_batch(*_records_arrays([r.encoding for r in recs], [r.fs for r in recs],
                                                  [r.target for r in recs]), device=eng.device, build_csr=sage)
                ws = _grow(slots, "train", eng, b.N, b.G, train=True)
                step += 1
                eng.forward(b, ws, mask_mode=2 if dropout else 0, dropout_p=model.dropout_p,
                            seed=config.seed * 1000003 + step, predict=False, defer_head=True)
                eng.loss(b, ws, config.huber_delta)
                eng.backward(b, ws, keep_scale=keep, advance_step=True)
                acc[:1].add_(ws.loss[:1], alpha=float(b.G))  # loss is the batch mean; APE terms are sums
                acc[1:].add_(ws.loss[1:])
                eng.adam_step(config.lr)
        a = acc.cpu().numpy()
        if not np.all(np.isfinite(a)):
            raise NonFinite(f"training loss diverged at epoch {epoch}")
        entry = {"epoch": epoch, "train_loss": float(a[0] / n), "train_mape": float((a[1:] / n).mean()),
                 "val_loss": None, "val_mape": None}
        if val_records:
            v_loss, v_ape = _evaluate(eng, val_records, config.huber_delta, slots)
            entry["val_loss"] = v_loss
            entry["val_mape"] = v_ape
        history.append(entry)
    final = eng.get_params()
    for name, arr in model.param_items():
        arr[...] = final[name]
    return model, history


def _evaluate(eng, records, delta, slots, chunk=256):
    """Eval-mode loss and MAPE over `records` (gnn.py:466-475), one read-back per chunk."""
    loss_sum, ape = 0.0, np.zeros(3)
    for s0 in range(0, len(records), chunk):
        recs = records[s0:s0 + chunk]
        b = upload_batch(*_records_arrays([r.encoding for r in recs], [r.fs for r in recs],
                                          [r.target for r in recs]), device=eng.device, build_csr=eng.arch == "sage")
        ws = _grow(slots, "eval", eng, b.N, b.G, train=False)
        eng.forward(b, ws, predict=False)
        eng.loss(b, ws, delta)
        out = ws.loss.cpu().numpy()
        loss_sum += out[0] * b.G
        ape += out[1:]
    return float(loss_sum / len(records)), float((ape / len(records)).mean())


# ---------------------------------------------------------------------------
# persistence (gnn.py:488-578) — identical JSON format

_SAGE_PARAM_NAMES = tuple(
    [f"sage{i}.{part}" for i in (1, 2, 3) for part in ("w_self", "w_neigh", "bias")]
    + [f"fc{i}.{part}" for i in (1, 2, 3) for part in ("w", "b")]
)
_MLP_PARAM_NAMES = tuple(f"fc{i}.{part}" for i in (1, 2, 3) for part in ("w", "b"))
_VECTOR_SUFFIXES = (".bias", ".b")


def save_model(model, path) -> None:
    """Write the model as one JSON document; round-trips bit-exactly."""
    params = {}
    for name, arr in model.param_items():
        arr = np.asarray(arr)
        if arr.ndim == 1:
            params[name] = {"rows": 1, "cols": int(arr.shape[0]), "data": arr.tolist()}
        else:
            params[name] = {"rows": int(arr.shape[0]), "cols": int(arr.shape[1]), "data": arr.ravel().tolist()}
    doc = {
        "vocab_version": model.vocab_version,
        "arch": model.arch,
        "hidden": model.hidden,
        "dropout_p": model.dropout_p,
        "normalizer": {
            "y_mean": np.asarray(model.normalizer.y_mean).tolist(),
            "y_std": np.asarray(model.normalizer.y_std).tolist(),
            "fs_mean": np.asarray(model.normalizer.fs_mean).tolist(),
            "fs_std": np.asarray(model.normalizer.fs_std).tolist(),
        },
        "params": params,
    }
    try:
        Path(path).write_text(json.dumps(doc), encoding="utf-8")
    except OSError as exc:
        raise IoFailure(f"cannot write model to {path}: {exc}") from exc


def load_model(path):
    """Read a model file back; refuses files from another vocabulary."""
    try:
        text = Path(path).read_text(encoding="utf-8")
    except OSError as exc:
        raise IoFailure(f"cannot read model from {path}: {exc}") from exc
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise IoFailure(f"model file {path} is not valid JSON: {exc}") from exc
    if not isinstance(doc, dict):
        raise IoFailure(f"model file {path} must contain an object")
    version = doc.get("vocab_version")
    if version != VOCAB_VERSION:
        raise VersionMismatch(f"model was built for vocabulary {version!r}, this build uses {VOCAB_VERSION!r}")
    arch = doc.get("arch")
    if arch not in ("sage", "mlp"):
        raise IoFailure(f"unknown model arch {arch!r}")
    try:
        hidden = int(doc["hidden"])
        dropout_p = float(doc["dropout_p"])
        nd = doc["normalizer"]
        normalizer = Normalizer(y_mean=np.asarray(nd["y_mean"], dtype=np.float64),
                                y_std=np.asarray(nd["y_std"], dtype=np.float64),
                                fs_mean=np.asarray(nd["fs_mean"], dtype=np.float64),
                                fs_std=np.asarray(nd["fs_std"], dtype=np.float64))
        arrays = {}
        for name in (_SAGE_PARAM_NAMES if arch == "sage" else _MLP_PARAM_NAMES):
            entry = doc["params"][name]
            rows, cols = int(entry["rows"]), int(entry["cols"])
            data = np.asarray(entry["data"], dtype=np.float64)
            if data.size != rows * cols:
                raise IoFailure(f"parameter {name}: {data.size} values for a {rows}x{cols} matrix")
            arrays[name] = data if name.endswith(_VECTOR_SUFFIXES) else data.reshape(rows, cols)
    except (KeyError, TypeError, ValueError) as exc:
        raise IoFailure(f"model file {path} is incomplete: {exc}") from exc
    fc = [AffineParams(w=arrays[f"fc{i}.w"], b=arrays[f"fc{i}.b"]) for i in (1, 2, 3)]
    if arch == "mlp":
        return MlpModel(fc=fc, dropout_p=dropout_p, normalizer=normalizer, hidden=hidden, vocab_version=version)
    sage = [SageLayerParams(w_self=arrays[f"sage{i}.w_self"], w_neigh=arrays[f"sage{i}.w_neigh"],
                            bias=arrays[f"sage{i}.bias"]) for i in (1, 2, 3)]
    return DippmModel(sage=sage, fc=fc, dropout_p=dropout_p, normalizer=normalizer, hidden=hidden,
                      vocab_version=version)
