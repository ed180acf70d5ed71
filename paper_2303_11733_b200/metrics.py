"""Evaluation on the device — the `dippm eval` path (cli.py:175-192) and
`dataset.mape` (dataset.py:229-248), §8f row 4.

`mape(preds, actuals)` is the reference's host-side function (same errors,
same arithmetic).  `evaluate(model, records)` produces the same MapeResult
without a per-record round trip: records are collated into batches, each
batch runs the eval-mode forward on the B200 and the Huber/APE kernel
(dippm_huber, gnn.py:458-459 semantics) accumulates the absolute percentage
errors of the de-normalised predictions on the device; the sums are read
back once at the end.  Works for DippmModel and MlpModel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import gnn
from .device import upload_batch
from .errors import LengthMismatch, ZeroActual
from .types import target_vector


@dataclass
class MapeResult:
    """dataset.py:86-91."""
    latency: float
    memory: float
    energy: float
    overall: float

    def as_dict(self) -> dict:
        return {"latency": self.latency, "memory": self.memory, "energy": self.energy, "overall": self.overall}


def mape(preds, actuals) -> MapeResult:
    """Per-target mean absolute percentage error plus the mean of the three (dataset.py:229-248)."""
    if len(preds) != len(actuals):
        raise LengthMismatch(f"{len(preds)} predictions vs {len(actuals)} actuals")
    if not preds:
        raise LengthMismatch("need at least one prediction")
    sums = np.zeros(3, dtype=np.float64)
    for pred, actual in zip(preds, actuals):
        p = target_vector(pred)
        a = target_vector(actual)
        if np.any(a == 0.0):
            raise ZeroActual("actual target contains a zero component")
        sums += np.abs(p - a) / np.abs(a)
    per_target = sums / len(preds)
    return MapeResult(latency=float(per_target[0]), memory=float(per_target[1]), energy=float(per_target[2]),
                      overall=float(per_target.mean()))


def evaluate(model, records, precision: str = "fp32", batch_size: int = 4096, with_loss: bool = False):
    """MAPE of `model` over `records`, computed on the device (one read-back).

    Equals mape([predict_record(model, r) for r in records], [r.target ...])
    within the stated fp32 tolerance.  with_loss=True also returns the mean
    eval-mode Huber loss (gnn.batch_loss over all records)."""
    if not records:
        raise LengthMismatch("need at least one prediction")
    targets = np.stack([target_vector(r.target) for r in records])
    if np.any(targets == 0.0):
        raise ZeroActual("actual target contains a zero component")
    eng = gnn._engine(model, precision)
    acc = torch.zeros(4, dtype=torch.float64, device=eng.device)
    slots = gnn.SimpleNamespace()
    for s0 in range(0, len(records), batch_size):
        recs = records[s0:s0 + batch_size]
        arrays = gnn._records_arrays([r.encoding for r in recs], [r.fs for r in recs], [r.target for r in recs])
        b = upload_batch(*arrays, device=eng.device, build_csr=eng.arch == "sage")
        ws = gnn._grow(slots, "eval", eng, b.N, b.G, train=False)
        eng.forward(b, ws, predict=False)
        eng.loss(b, ws, 1.0)
        acc[:1].add_(ws.loss[:1], alpha=float(b.G))
        acc[1:].add_(ws.loss[1:])
    a = acc.cpu().numpy() / len(records)
    res = MapeResult(latency=float(a[1]), memory=float(a[2]), energy=float(a[3]), overall=float(a[1:].mean()))
    return (res, float(a[0])) if with_loss else res


def eval_report(model, records, precision: str = "fp32") -> dict:
    """The JSON document `dippm eval` prints (cli.py:183-191)."""
    res = evaluate(model, records, precision)
    return {"mape": res.as_dict(), "n": len(records)}
