"""CPU oracle for the DIPPM GraphSAGE hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy, float64 restatement of the reference
``dippm.gnn`` / ``dippm.numerics`` / ``dippm.mig`` algorithms (reference tree
``/root/reference/pkg/src/dippm``; every function cites the file:line it
follows).  It exists so the tests, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` have a checker
and a CPU timing arm on the GPU box, where ``/root/reference`` is absent.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its CPU
baseline leg) may import it.  The product package
``paper_2303_11733_b200`` never imports, calls or links anything here.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference in
the build container, runs it on seeded inputs and stores the results in
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this oracle
against those vectors (CSR pattern/in-degree exact, floats to 1e-12).

Data model: a "record" is a tuple ``(num_nodes, edges, X, fs_raw, y_raw)``
with ``edges`` a list/array of (src, dst) pairs, ``X`` (N, 32) float64,
``fs_raw`` (5,) log1p static features, ``y_raw`` (3,) targets or None.
Parameters are a dict keyed by the reference names (gnn.py:488-491).
"""

from __future__ import annotations

import math

import numpy as np

FEATURE_WIDTH = 32          # featurize.py:38
STATIC_WIDTH = 5            # featurize.py:39
DEFAULT_HIDDEN = 512        # gnn.py:42
DEFAULT_DROPOUT = 0.05      # gnn.py:43
DEFAULT_LEARNING_RATE = 2.754e-5  # numerics.py:17
ADAM_BETA1, ADAM_BETA2, ADAM_EPS = 0.9, 0.999, 1e-8  # numerics.py:18-20
MIG_CEILINGS_MB = (5 * 1024, 10 * 1024, 20 * 1024, 40 * 1024)  # mig.py:19-22
MIG_LABELS = ("1g.5gb", "2g.10gb", "3g.20gb", "7g.40gb")

SAGE_PARAM_NAMES = tuple(
    [f"sage{i}.{p}" for i in (1, 2, 3) for p in ("w_self", "w_neigh", "bias")]
    + [f"fc{i}.{p}" for i in (1, 2, 3) for p in ("w", "b")]
)  # gnn.py:488-491


# ---------------------------------------------------------------------------
# aggregation (gnn.py:130-137, 157-162)

def aggregation_matrix(num_nodes: int, edges) -> np.ndarray:
    """Dense agg[dst, src] = 1/indeg(dst); assignment, so duplicates count
    twice in deg but are summed once (gnn.py:130-137)."""
    agg = np.zeros((num_nodes, num_nodes), dtype=np.float64)
    deg = np.zeros(num_nodes, dtype=np.float64)
    for _, dst in edges:
        deg[dst] += 1.0
    for src, dst in edges:
        agg[dst, src] = 1.0 / deg[dst]
    return agg


def csr_of_aggregation(num_nodes: int, edges):
    """CSR view of the dense matrix above: (rowptr, col, deg) with rows = dst,
    columns = the distinct src of each row in ascending order, deg = in-degree
    counting duplicates (the denominator gnn.py:133-136 uses)."""
    deg = np.zeros(num_nodes, dtype=np.int64)
    pairs = set()
    for src, dst in edges:
        deg[int(dst)] += 1
        pairs.add((int(dst), int(src)))
    ordered = sorted(pairs)
    rowptr = np.zeros(num_nodes + 1, dtype=np.int64)
    for dst, _ in ordered:
        rowptr[dst + 1] += 1
    rowptr = np.cumsum(rowptr)
    col = np.array([s for _, s in ordered], dtype=np.int64)
    return rowptr, col, deg


# ---------------------------------------------------------------------------
# normaliser (gnn.py:59-97)

def normalizer_fit(targets: np.ndarray, statics: np.ndarray) -> dict:
    def clamp(std):
        std = std.copy()
        std[std < 1e-9] = 1.0
        return std
    return {
        "y_mean": targets.mean(axis=0), "y_std": clamp(targets.std(axis=0)),
        "fs_mean": statics.mean(axis=0), "fs_std": clamp(statics.std(axis=0)),
    }


def normalizer_identity() -> dict:
    return {"y_mean": np.zeros(3), "y_std": np.ones(3),
            "fs_mean": np.zeros(STATIC_WIDTH), "fs_std": np.ones(STATIC_WIDTH)}


# ---------------------------------------------------------------------------
# init (gnn.py:169-175, 302-319)

def glorot(rng: np.random.Generator, fan_in: int, fan_out: int) -> np.ndarray:
    return rng.normal(0.0, math.sqrt(2.0 / (fan_in + fan_out)), size=(fan_in, fan_out))


def init_params(hidden: int, rng: np.random.Generator) -> dict:
    """Draw order sage1..3 (w_self, w_neigh), then fc1..3 w (gnn.py:312-319)."""
    p = {}
    dims = [(FEATURE_WIDTH, hidden), (hidden, hidden), (hidden, hidden)]
    for i, (di, do) in enumerate(dims, start=1):
        p[f"sage{i}.w_self"] = glorot(rng, di, do)
        p[f"sage{i}.w_neigh"] = glorot(rng, di, do)
        p[f"sage{i}.bias"] = np.zeros(do)
    for i, (di, do) in enumerate([(hidden + STATIC_WIDTH, hidden), (hidden, hidden), (hidden, 3)], start=1):
        p[f"fc{i}.w"] = glorot(rng, di, do)
        p[f"fc{i}.b"] = np.zeros(do)
    return {k: p[k] for k in SAGE_PARAM_NAMES}


# ---------------------------------------------------------------------------
# numerics (numerics.py:45-114)

def dropout_mask(shape, p: float, rng) -> np.ndarray:
    """numerics.py:45-55."""
    if p == 0.0:
        return np.ones(shape, dtype=np.float64)
    keep = rng.random(shape) >= p
    return keep.astype(np.float64) / (1.0 - p)


def huber_loss(pred, target, delta=1.0):
    """numerics.py:58-73: mean elementwise Huber and its gradient."""
    r = pred - target
    a = np.abs(r)
    quad = a <= delta
    elems = np.where(quad, 0.5 * r * r, delta * (a - 0.5 * delta))
    grad = np.where(quad, r, delta * np.sign(r)) / r.size
    return float(elems.mean()), grad


def adam_step(param, grad, m, v, t, lr=DEFAULT_LEARNING_RATE,
              beta1=ADAM_BETA1, beta2=ADAM_BETA2, eps=ADAM_EPS):
    """numerics.py:93-114, same op order; m, v updated in place; t is the
    step count AFTER the increment.  Returns the new parameter."""
    m *= beta1
    m += (1.0 - beta1) * grad
    tmp = grad * grad
    tmp *= 1.0 - beta2
    v *= beta2
    v += tmp
    denom = v / (1.0 - beta2 ** t)
    np.sqrt(denom, out=denom)
    denom += eps
    step = m / (1.0 - beta1 ** t)
    step /= denom
    step *= -lr
    step += param
    return step


# ---------------------------------------------------------------------------
# forward / backward (gnn.py:202-233, 265-299)

def embed(params, X, agg):
    """gnn.py:202-210."""
    h = np.asarray(X, dtype=np.float64)
    caches = []
    for i in (1, 2, 3):
        m = agg @ h
        z = h @ params[f"sage{i}.w_self"] + m @ params[f"sage{i}.w_neigh"] + params[f"sage{i}.bias"]
        caches.append((h, m, z))
        h = np.maximum(z, 0.0)
    return h, caches


def fc_forward(params, u, masks=None):
    """gnn.py:265-284; ``masks`` = (mask1, mask2) for train mode or None."""
    cache = []
    x = u
    for i in (1, 2, 3):
        a = x @ params[f"fc{i}.w"] + params[f"fc{i}.b"]
        if i == 3:
            cache.append((x, a, None))
            x = a
            continue
        h = np.maximum(a, 0.0)
        mask = None if masks is None else masks[i - 1]
        if mask is not None:
            h = h * mask
        cache.append((x, a, mask))
        x = h
    return x, cache


def forward_norm(params, X, agg, fs_norm, masks=None):
    """gnn.py:212-217."""
    h, sage_cache = embed(params, X, agg)
    r = h.mean(axis=0)
    u = np.concatenate([r, fs_norm])
    out, fc_cache = fc_forward(params, u, masks)
    return out, (agg, sage_cache, h.shape[0], fc_cache)


def fc_backward(params, cache, dout, grads):
    """gnn.py:287-299."""
    d = dout
    for i in (3, 2, 1):
        x, a, mask = cache[i - 1]
        if i != 3:
            if mask is not None:
                d = d * mask
            d = d * (a > 0.0)
        grads[f"fc{i}.w"] = np.outer(x, d)
        grads[f"fc{i}.b"] = d.copy()
        d = params[f"fc{i}.w"] @ d
    return d


def backward_from(params, cache, dout, hidden):
    """gnn.py:219-233."""
    agg, sage_cache, n_nodes, fc_cache = cache
    grads = {}
    du = fc_backward(params, fc_cache, dout, grads)
    dr = du[:hidden]
    dh = np.tile(dr / n_nodes, (n_nodes, 1))
    for i in (3, 2, 1):
        h_in, m, z = sage_cache[i - 1]
        dz = dh * (z > 0.0)
        grads[f"sage{i}.w_self"] = h_in.T @ dz
        grads[f"sage{i}.w_neigh"] = m.T @ dz
        grads[f"sage{i}.bias"] = dz.sum(axis=0)
        dh = dz @ params[f"sage{i}.w_self"].T + agg.T @ (dz @ params[f"sage{i}.w_neigh"].T)
    return grads


# ---------------------------------------------------------------------------
# public-level restatements (gnn.py:331-405, mig.py:32-45)

def sage_forward(num_nodes, edges, w_self, w_neigh, bias, h_in):
    """gnn.py:331-338."""
    m = aggregation_matrix(num_nodes, edges) @ h_in
    return np.maximum(h_in @ w_self + m @ w_neigh + bias, 0.0)


def forward(params, norm, num_nodes, edges, X, fs_raw, masks=None):
    """gnn.py:348-355 (eval when masks is None)."""
    fs_norm = (fs_raw - norm["fs_mean"]) / norm["fs_std"]
    out, _ = forward_norm(params, X, aggregation_matrix(num_nodes, edges), fs_norm, masks)
    return out


def predict(params, norm, num_nodes, edges, X, fs_raw):
    """gnn.py:358-361: de-normalised (latency_ms, memory_mb, energy_j)."""
    return forward(params, norm, num_nodes, edges, X, fs_raw) * norm["y_std"] + norm["y_mean"]


def batch_loss(params, norm, records, delta=1.0):
    """gnn.py:368-380."""
    total = 0.0
    for n, edges, X, fs_raw, y_raw in records:
        out = forward(params, norm, n, edges, X, fs_raw)
        loss, _ = huber_loss(out, (y_raw - norm["y_mean"]) / norm["y_std"], delta)
        total += loss
    return total / len(records)


def backward(params, norm, records, delta=1.0, hidden=None):
    """gnn.py:383-405: mean loss and mean per-record gradients (eval mode)."""
    hidden = params["sage1.w_self"].shape[1] if hidden is None else hidden
    grads = {k: np.zeros_like(v) for k, v in params.items()}
    total = 0.0
    for n, edges, X, fs_raw, y_raw in records:
        fs_norm = (fs_raw - norm["fs_mean"]) / norm["fs_std"]
        y_norm = (y_raw - norm["y_mean"]) / norm["y_std"]
        out, cache = forward_norm(params, X, aggregation_matrix(n, edges), fs_norm)
        loss, dout = huber_loss(out, y_norm, delta)
        total += loss
        for k, g in backward_from(params, cache, dout, hidden).items():
            grads[k] += g
    scale = 1.0 / len(records)
    for k in grads:
        grads[k] *= scale
    return total * scale, grads


def mig_code(alpha_mb: float) -> int:
    """mig.py:32-45 as an integer code: index into MIG_LABELS, -1 for None.
    Raises ValueError for NaN/Inf (the reference raises NonFinite)."""
    if not math.isfinite(alpha_mb):
        raise ValueError(f"memory prediction is not finite: {alpha_mb}")
    if alpha_mb <= 0:
        return -1
    for i, cap in enumerate(MIG_CEILINGS_MB):
        if alpha_mb <= cap:
            return i
    return -1


def train_reference_protocol(records, epochs, seed=0, hidden=DEFAULT_HIDDEN, lr=DEFAULT_LEARNING_RATE,
                             delta=1.0, shuffle=True, dropout_p=DEFAULT_DROPOUT, val_records=(), arch="sage"):
    """gnn.py:424-482: batch-size-1 Adam over records with PCG64 dropout masks
    drawn in the reference order.  arch "mlp" = train_mlp (gnn.py:418-421).
    Returns (params, normaliser, history)."""
    rng = np.random.default_rng(seed)
    targets = np.stack([r[4] for r in records])
    statics = np.stack([r[3] for r in records])
    norm = normalizer_fit(targets, statics)
    mlp = arch == "mlp"
    params = init_mlp_params(hidden, rng) if mlp else init_params(hidden, rng)
    preps = [(aggregation_matrix(n, e), np.asarray(X, dtype=np.float64)) for n, e, X, _, _ in records]
    fs_norm = [(r[3] - norm["fs_mean"]) / norm["fs_std"] for r in records]
    y_norm = [(r[4] - norm["y_mean"]) / norm["y_std"] for r in records]
    state = {k: (np.zeros_like(v), np.zeros_like(v)) for k, v in params.items()}
    t = 0
    history = []
    n = len(records)
    for epoch in range(1, epochs + 1):
        order = rng.permutation(n) if shuffle else np.arange(n)
        loss_sum, ape = 0.0, np.zeros(3)
        for i in order:
            masks = None
            if dropout_p > 0.0:
                m1 = dropout_mask((hidden,), dropout_p, rng)
                m2 = dropout_mask((hidden,), dropout_p, rng)
                masks = (m1, m2)
            agg, X = preps[i]
            if mlp:
                out, cache = fc_forward(params, fs_norm[i], masks)
            else:
                out, cache = forward_norm(params, X, agg, fs_norm[i], masks)
            loss, dout = huber_loss(out, y_norm[i], delta)
            loss_sum += loss
            pred = out * norm["y_std"] + norm["y_mean"]
            ape += np.abs(pred - records[i][4]) / np.abs(records[i][4])
            if mlp:
                grads = {}
                fc_backward(params, cache, dout, grads)
            else:
                grads = backward_from(params, cache, dout, hidden)
            t += 1
            for k in params:
                m, v = state[k]
                params[k][...] = adam_step(params[k], grads[k], m, v, t, lr)
        entry = {"epoch": epoch, "train_loss": loss_sum / n, "train_mape": float((ape / n).mean()),
                 "val_loss": None, "val_mape": None}
        if val_records:
            vl, va = 0.0, np.zeros(3)
            for vn, ve, vX, vfs, vy in val_records:
                out = mlp_forward(params, norm, vfs) if mlp else forward(params, norm, vn, ve, vX, vfs)
                loss, _ = huber_loss(out, (vy - norm["y_mean"]) / norm["y_std"], delta)
                vl += loss
                va += np.abs(out * norm["y_std"] + norm["y_mean"] - vy) / np.abs(vy)
            entry["val_loss"] = vl / len(val_records)
            entry["val_mape"] = float((va / len(val_records)).mean())
        history.append(entry)
    return params, norm, history


# ---------------------------------------------------------------------------
# MLP baseline (gnn.py:236-262, 322-324, 418-421) — static features only

MLP_PARAM_NAMES = tuple(f"fc{i}.{p}" for i in (1, 2, 3) for p in ("w", "b"))


def init_mlp_params(hidden: int, rng: np.random.Generator) -> dict:
    """gnn.py:322-324 via _fc_stack gnn.py:174-175: fc1..3 w in draw order."""
    p = {}
    for i, (di, do) in enumerate([(STATIC_WIDTH, hidden), (hidden, hidden), (hidden, 3)], start=1):
        p[f"fc{i}.w"] = glorot(rng, di, do)
        p[f"fc{i}.b"] = np.zeros(do)
    return p


def mlp_forward(params, norm, fs_raw, masks=None):
    """MlpModel.forward_norm gnn.py:253-255 after normalize_fs gnn.py:96-97."""
    out, _ = fc_forward(params, (np.asarray(fs_raw, np.float64) - norm["fs_mean"]) / norm["fs_std"], masks)
    return out


def mlp_predict(params, norm, fs_raw):
    return mlp_forward(params, norm, fs_raw) * norm["y_std"] + norm["y_mean"]


def mlp_backward(params, norm, records, delta=1.0):
    """gnn.backward (gnn.py:383-405) for an MlpModel: mean loss, mean grads (eval mode)."""
    grads = {k: np.zeros_like(v) for k, v in params.items()}
    total = 0.0
    for _, _, _, fs_raw, y_raw in records:
        fs_norm = (fs_raw - norm["fs_mean"]) / norm["fs_std"]
        out, cache = fc_forward(params, fs_norm)
        loss, dout = huber_loss(out, (y_raw - norm["y_mean"]) / norm["y_std"], delta)
        total += loss
        g = {}
        fc_backward(params, cache, dout, g)
        for k, v in g.items():
            grads[k] += v
    scale = 1.0 / len(records)
    return total * scale, {k: v * scale for k, v in grads.items()}


def mape(preds, actuals):
    """dataset.mape (dataset.py:229-248): per-target mean |p - a| / |a| and their mean."""
    p, a = np.asarray(preds, np.float64), np.asarray(actuals, np.float64)
    if p.shape != a.shape or len(p) == 0:
        raise ValueError("need matching, non-empty prediction / actual lists")
    if np.any(a == 0.0):
        raise ValueError("actual target contains a zero component")
    per = (np.abs(p - a) / np.abs(a)).sum(axis=0) / len(p)
    return {"latency": float(per[0]), "memory": float(per[1]), "energy": float(per[2]),
            "overall": float(per.mean())}
