"""DIPPM GraphSAGE predictor — drop-in for the reference `dippm.gnn` (gnn.py:1-578).

Same public names, argument meanings, return types and error behaviour; the
arithmetic runs on the B200 through libdippm_b200.so (see device.py).  The
host model object keeps the fp64 "truth" exactly like the reference
(`param_items()` returns live numpy arrays that callers may mutate); each call
uploads the current values, so in-place edits between calls are honoured.

Additions (batched surface): `predict_batch`, `predict_records`,
`TrainConfig.batch_size / precision / device / backend`.

Numerics: `precision="fp32"` (default) runs the SAGE GEMMs as 3-pass TF32 on
the tensor cores (fp32-grade), everything else in fp32 with fp64 Adam
masters; `precision="bf16"` uses bf16 GEMM operands with fp32 accumulation.
Stated tolerances vs the fp64 reference: see DESIGN.md §Parity.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path
from typing import ClassVar

import numpy as np
import torch

from . import _lib, device as dev
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
    backend: str = "tc"

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
# engine binding

def _engine(model, precision: str = "fp32", device=None, backend: str = "tc") -> Engine:
    """Device engine for `model`, refreshed from the model's current host values."""
    arch = getattr(model, "arch", "sage")
    key = (precision, str(device), backend, int(model.hidden), arch)
    cache = model.__dict__.setdefault("_b200_engines", {})
    eng = cache.get(key)
    if eng is None:
        eng = Engine(model.hidden, precision, device, backend, arch=arch)
        cache[key] = eng
    eng.set_params(model.param_items(), model.normalizer)
    return eng


def _records_arrays(encodings, fss, targets=None):
    return collate_host(encodings, [fs_vector(f) for f in fss],
                        None if targets is None else [target_vector(t) for t in targets])


def infer_workspace(eng: Engine, N: int, G: int) -> Workspace:
    """The engine's reusable inference workspace, grown (x1.25) when a batch needs more rows/graphs."""
    ws = getattr(eng, "_infer_ws", None)
    if ws is None or ws.N < N or ws.G < G:
        ws = Workspace(eng, max(N, int(1.25 * (ws.N if ws else 0))), max(G, int(1.25 * (ws.G if ws else 0))),
                       train=False)
        eng._infer_ws = ws
    return ws


def _run_forward(eng: Engine, encodings, fss, targets=None, mask_mode=0, masks=None, train_buffers=False):
    x, src, dst, gp, fs, y = _records_arrays(encodings, fss, targets)
    b = upload_batch(x, src, dst, gp, fs, y, device=eng.device, build_csr=eng.arch == "sage")
    ws = Workspace(eng, b.N, b.G, train=True) if train_buffers else infer_workspace(eng, b.N, b.G)
    if masks is not None:
        ws.masks[:, :, :masks.shape[-1]].copy_(torch.from_numpy(masks.astype(np.float32)))
    eng.forward(b, ws, mask_mode=mask_mode)
    return b, ws


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
    dip, dop = -(-d_in // 32) * 32, -(-d_out // 64) * 64
    e = np.asarray(encoding.edges, dtype=np.int64).reshape(-1, 2)
    if e.size and (e.min() < 0 or e.max() >= n):
        raise ShapeMismatch(f"edge endpoint outside [0, {n})")
    xp = np.zeros((n, dip), np.float32)
    xp[:, :d_in] = h_in
    b = upload_batch(np.zeros((n, FEATURE_WIDTH), np.float32), e[:, 0].copy(), e[:, 1].copy(),
                     np.array([0, n], np.int32), np.zeros((1, STATIC_WIDTH), np.float32), device=device)
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
    _lib.call("dippm_sage_aggregate", f32_act(xt), A.view(dip), A.view(0), n, dip, b.rowptr.data_ptr(),
              b.col.data_ptr(), b.inv_deg.data_ptr(), s)
    _lib.call("dippm_pack", wt64.data_ptr(), 2 * dip, dop, 1, Wt.view(), s)
    args = _lib.GemmArgs(_lib.GEMM_FWD, n, dop, 2 * dip, A.view(0), 0, Wt.view(), 0, bt.data_ptr(), 1, out.view(),
                         None, 0, 1)
    _lib.check(_lib.load().dippm_gemm(args, 0, s), "dippm_gemm")
    return out.t[:, :d_out].double().cpu().numpy()


def readout_mean(z: np.ndarray) -> np.ndarray:
    """Arithmetic mean over node embeddings (gnn.py:341-345), on device (K4)."""
    z = np.asarray(z)
    if z.ndim != 2 or z.shape[0] < 1:
        raise EmptyGraph("readout needs at least one node embedding")
    device = dev.require_device()
    n, d = z.shape
    dp = -(-d // 8) * 8
    zp = torch.zeros(n, dp, dtype=torch.float32)
    zp[:, :d] = torch.from_numpy(np.asarray(z, dtype=np.float32))
    zt = zp.to(device)
    gp = torch.tensor([0, n], dtype=torch.int32, device=device)
    fs = torch.zeros(1, STATIC_WIDTH, dtype=torch.float32, device=device)
    norm = torch.tensor([0.0] * 6 + [0.0] * 5 + [1.0] * 5, dtype=torch.float64, device=device)
    u = torch.empty(1, dp + 8, dtype=torch.float32, device=device)
    _lib.call("dippm_pool_concat", f32_act(zt), gp.data_ptr(), 1, dp, fs.data_ptr(), norm.data_ptr(), f32_act(u),
              dev._stream())
    return u[0, :d].double().cpu().numpy()


def forward(encoding, fs, model, mode: str = "eval", rng=None, precision: str = "fp32") -> np.ndarray:
    """Normalised-space prediction for one graph (gnn.py:348-355)."""
    _check_mode(mode)
    masks = _draw_masks(model, rng) if mode == "train" else None
    eng = _engine(model, precision)
    _, ws = _run_forward(eng, [encoding], [fs], mask_mode=1 if masks is not None else 0, masks=masks)
    return ws.out[0].double().cpu().numpy()


def predict_batch(model, encodings, fss, precision: str = "fp32"):
    """Batched eval prediction: (y float64 [G, 3] in original units, MIG codes int8 [G]).

    MIG codes: 0=1g.5gb, 1=2g.10gb, 2=3g.20gb, 3=7g.40gb, -1=None; computed on
    the device from y[:, 1] with the same rule as mig.mig_profile.
    """
    if len(encodings) != len(fss):
        raise ShapeMismatch(f"{len(encodings)} encodings vs {len(fss)} static-feature vectors")
    if not encodings:
        raise EmptyDataset("batch is empty")
    eng = _engine(model, precision)
    _, ws = _run_forward(eng, encodings, fss)
    G = len(encodings)
    return ws.y_pred[:G].cpu().numpy(), ws.mig[:G].cpu().numpy()


def predict(model, encoding, fs, precision: str = "fp32") -> TargetVector:
    """Original-unit eval-mode prediction (gnn.py:358-361)."""
    y, _ = predict_batch(model, [encoding], [fs], precision)
    return TargetVector(latency_ms=float(y[0, 0]), memory_mb=float(y[0, 1]), energy_j=float(y[0, 2]))


def predict_record(model, record, precision: str = "fp32") -> TargetVector:
    return predict(model, record.encoding, record.fs, precision)


def predict_records(model, records, precision: str = "fp32", with_mig: bool = False):
    """Batched `predict_record` over many records (one device pass)."""
    y, mig = predict_batch(model, [r.encoding for r in records], [r.fs for r in records], precision)
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
    return float(ws.loss[0].item())


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
    return float(ws.loss[0].item()), eng.get_grads()


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
    eng = Engine(config.hidden, config.precision, config.device, config.backend, arch=model.arch)
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
    ws_cache = {}
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
                ws = _workspace(ws_cache, eng, b, train=True)
                step += 1
                eng.forward(b, ws, mask_mode=2 if dropout else 0, dropout_p=model.dropout_p,
                            seed=config.seed * 1000003 + step, predict=False, defer_head=True)
                eng.loss(b, ws, config.huber_delta)
                eng.backward(b, ws, keep_scale=keep, advance_step=True)
                acc.add_(ws.loss * torch.tensor([b.G, 1, 1, 1], dtype=torch.float64, device=eng.device))
                eng.adam_step(config.lr)
        a = acc.cpu().numpy()
        if not np.all(np.isfinite(a)):
            raise NonFinite(f"training loss diverged at epoch {epoch}")
        entry = {"epoch": epoch, "train_loss": float(a[0] / n), "train_mape": float((a[1:] / n).mean()),
                 "val_loss": None, "val_mape": None}
        if val_records:
            v_loss, v_ape = _evaluate(eng, val_records, config.huber_delta, ws_cache)
            entry["val_loss"] = v_loss
            entry["val_mape"] = v_ape
        history.append(entry)
    final = eng.get_params()
    for name, arr in model.param_items():
        arr[...] = final[name]
    return model, history


def _workspace(cache, eng, b, train):
    key = (b.N, b.G, train)
    ws = cache.get(key)
    if ws is None:
        ws = Workspace(eng, b.N, b.G, train=train)
        cache[key] = ws
    return ws


def _evaluate(eng, records, delta, ws_cache, chunk=256):
    loss_sum, ape = 0.0, np.zeros(3)
    for s0 in range(0, len(records), chunk):
        recs = records[s0:s0 + chunk]
        b = upload_batch(*_records_arrays([r.encoding for r in recs], [r.fs for r in recs],
                                          [r.target for r in recs]), device=eng.device, build_csr=eng.arch == "sage")
        ws = _workspace(ws_cache, eng, b, train=True)
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
