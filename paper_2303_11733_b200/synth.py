"""Seeded synthetic DIPPM-shaped datasets (SURVEY.md §8(d) "generator B").

Vectorised numpy; emits collated arrays directly (no per-graph Python
objects), shaped like the reference featuriser's output:
  * DAG per graph: chain edge v-1 -> v plus skip edges u -> v (u < v - 1) until
    E/N ~ 1.33, producer -> consumer like featurize.py:154-162;
  * node rows follow the 32-slot layout of featurize.py:10-16 / 166-183:
    one-hot over 16 kinds, log1p attribute slots 16-27 (has_bias 0/1 in 26,
    epsilon raw in 27), log1p output-shape slots 28-31;
  * fs = log1p(macs, batch, #conv, #dense, #relu) (featurize.py:66-87);
  * targets from a closed-form cost of (N, E, depth proxy, fs), positive,
    in the range of dataset.py:98-119 labels (memory spans 0.6-45 GB when
    `memory_scale` is raised, so every MIG profile occurs).
Node counts: uniform N in [n_lo, n_hi] or a truncated power law.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

FEATURE_WIDTH = 32
STATIC_WIDTH = 5


@dataclass
class SynthDataset:
    n: np.ndarray          # int64 [G] nodes per graph
    node_ptr: np.ndarray   # int64 [G+1]
    x: np.ndarray          # f32 [sum N, 32]
    edge_ptr: np.ndarray   # int64 [G+1]
    src: np.ndarray        # int64 [sum E] graph-local ids
    dst: np.ndarray        # int64 [sum E]
    fs: np.ndarray         # f32 [G, 5]
    y: np.ndarray          # f32 [G, 3]

    @property
    def num_graphs(self) -> int:
        return len(self.n)

    def collate(self, ids) -> tuple:
        """Arrays for the graphs `ids`, node ids offset to be batch-global."""
        ids = np.asarray(ids)
        n = self.n[ids]
        gp = np.zeros(len(ids) + 1, np.int32)
        np.cumsum(n, out=gp[1:])
        rows = np.concatenate([np.arange(self.node_ptr[i], self.node_ptr[i + 1]) for i in ids])
        erows = [np.arange(self.edge_ptr[i], self.edge_ptr[i + 1]) for i in ids]
        off = np.concatenate([np.full(len(e), gp[k], np.int64) for k, e in enumerate(erows)])
        erows = np.concatenate(erows)
        return (self.x[rows], self.src[erows] + off, self.dst[erows] + off, gp, self.fs[ids], self.y[ids])

    def records(self, ids):
        """Reference-style record objects (for parity subsets / the CPU oracle)."""
        from .types import DatasetRecord, GraphEncoding, TargetVector
        out = []
        for i in ids:
            a, b = self.node_ptr[i], self.node_ptr[i + 1]
            ea, eb = self.edge_ptr[i], self.edge_ptr[i + 1]
            edges = list(zip(self.src[ea:eb].tolist(), self.dst[ea:eb].tolist()))
            enc = GraphEncoding(int(self.n[i]), edges, self.x[a:b].astype(np.float64))
            out.append(DatasetRecord(enc, _FsVec(self.fs[i].astype(np.float64)), TargetVector(*map(float, self.y[i]))))
        return out


class _FsVec:
    def __init__(self, v):
        self.as_vector = v


def node_counts(num_graphs: int, rng, n_lo=270, n_hi=330, power_law: float | None = None, n_max=5000):
    if power_law is None:
        return rng.integers(n_lo, n_hi + 1, num_graphs).astype(np.int64)
    # truncated power law p(N) ~ N^-alpha on [n_lo, n_max] by inverse CDF
    a = 1.0 - power_law
    u = rng.random(num_graphs)
    lo, hi = float(n_lo) ** a, float(n_max) ** a
    return np.clip(np.floor((lo + u * (hi - lo)) ** (1.0 / a)), n_lo, n_max).astype(np.int64)


def make_dataset(num_graphs: int, seed: int = 0, n_lo: int = 270, n_hi: int = 330, edge_ratio: float = 1.33,
                 power_law: float | None = None, n_max: int = 5000, memory_scale: float = 1.0,
                 nodes=None) -> SynthDataset:
    """`nodes` (optional int array [num_graphs]) fixes the node counts explicitly."""
    rng = np.random.default_rng(seed)
    n = node_counts(num_graphs, rng, n_lo, n_hi, power_law, n_max) if nodes is None else \
        np.asarray(nodes, dtype=np.int64).reshape(num_graphs)
    node_ptr = np.zeros(num_graphs + 1, np.int64)
    np.cumsum(n, out=node_ptr[1:])
    total = int(node_ptr[-1])
    gid = np.repeat(np.arange(num_graphs), n)
    local = np.arange(total) - node_ptr[gid]

    # node features (featurize.py slot layout)
    x = np.zeros((total, FEATURE_WIDTH), np.float32)
    kind = rng.integers(0, 16, total)
    x[np.arange(total), kind] = 1.0
    attrs = np.log1p(rng.integers(0, 4, (total, 9))).astype(np.float32)        # kernel/stride/pad/dil/groups
    attrs *= (rng.random((total, 1)) < 0.4)                                       # only conv/pool rows carry them
    x[:, 16:25] = attrs
    x[:, 25] = np.log1p(rng.integers(0, 135, total)) * (rng.random(total) < 0.3)  # out_features
    x[:, 26] = rng.integers(0, 2, total) * (rng.random(total) < 0.3)              # has_bias
    x[:, 27] = 1e-5 * (rng.random(total) < 0.1)                                   # epsilon (raw)
    x[:, 28:32] = np.log1p(rng.integers(1, 4096, (total, 4))) * (rng.random((total, 4)) < 0.8)

    # edges: chain + skip edges (u < v - 1), E/N ~ edge_ratio
    chain_dst = local >= 1
    c_dst = np.nonzero(chain_dst)[0]
    c_src = c_dst - 1
    n_skip = np.maximum(0, np.round(n * (edge_ratio - 1.0)).astype(np.int64))
    sk_g = np.repeat(np.arange(num_graphs), n_skip)
    sk_v = 2 + np.floor(rng.random(len(sk_g)) * np.maximum(n[sk_g] - 2, 1)).astype(np.int64)
    sk_v = np.minimum(sk_v, n[sk_g] - 1)
    sk_u = np.floor(rng.random(len(sk_g)) * np.maximum(sk_v - 1, 1)).astype(np.int64)
    ok = sk_v >= 2
    sk_g, sk_v, sk_u = sk_g[ok], sk_v[ok], sk_u[ok]
    src_g = np.concatenate([c_src - node_ptr[gid[c_dst]], sk_u])
    dst_g = np.concatenate([local[c_dst], sk_v])
    eg = np.concatenate([gid[c_dst], sk_g])
    order = np.lexsort((src_g, dst_g, eg))            # per graph, dst ascending (featurizer order)
    src_g, dst_g, eg = src_g[order], dst_g[order], eg[order]
    keep = np.ones(len(eg), bool)
    keep[1:] = (eg[1:] != eg[:-1]) | (src_g[1:] != src_g[:-1]) | (dst_g[1:] != dst_g[:-1])  # no duplicates
    src_g, dst_g, eg = src_g[keep], dst_g[keep], eg[keep]
    ecount = np.bincount(eg, minlength=num_graphs)
    edge_ptr = np.zeros(num_graphs + 1, np.int64)
    np.cumsum(ecount, out=edge_ptr[1:])

    # static features and closed-form targets
    macs = np.exp(rng.uniform(np.log(1e5), np.log(1e11), num_graphs))
    batch = rng.integers(1, 129, num_graphs)
    t_conv = rng.integers(0, np.maximum(n // 3, 1))
    t_dense = rng.integers(0, np.maximum(n // 10, 1))
    t_relu = rng.integers(0, np.maximum(n // 3, 1))
    fs = np.stack([np.log1p(macs), np.log1p(batch), np.log1p(t_conv), np.log1p(t_dense), np.log1p(t_relu)],
                  1).astype(np.float32)
    depth = n * 0.6 + ecount * 0.1
    latency = 0.05 * n + macs / 1e8 + 0.2 * depth * 0.05 + 0.01 * batch
    memory = 600.0 + memory_scale * (4.0 * macs / 2**20 / 1e2 + 2.0 * n)
    energy = 0.25 * latency * (1.0 + macs / 1e9)
    y = np.stack([latency, memory, energy], 1).astype(np.float32)
    return SynthDataset(n=n, node_ptr=node_ptr, x=x, edge_ptr=edge_ptr, src=src_g.astype(np.int64),
                        dst=dst_g.astype(np.int64), fs=fs, y=y)


# ---------------------------------------------------------------------------
# graph JSON documents (reference schema, graph_ir.py:8-27) for the end-to-end
# predict path: native featuriser -> device forward -> MIG (configs[4])

def _resnet_doc(n_ops: int, rng: np.random.Generator, name: str) -> str:
    """A resnet-like model with about n_ops operator nodes: stem conv/bn/relu,
    residual blocks (conv, batchnorm, relu, conv, batchnorm, add, relu) with an
    occasional maxpool, a few constant inputs, then global pool, reshape, dense.
    Non-source shapes are left out, so parsing runs shape inference."""
    import json
    batch = int(rng.choice([1, 2, 4, 8, 16, 32, 64]))
    c = int(rng.choice([8, 16, 32, 64]))
    hw = int(rng.choice([32, 64, 128, 224]))
    nodes = [{"id": 0, "op": "input", "inputs": [], "attrs": {}, "out_shape": [batch, 3, hw, hw]}]

    def add(op, inputs, attrs=None):
        nodes.append({"id": len(nodes), "op": op, "inputs": inputs, "attrs": attrs or {}})
        return len(nodes) - 1

    conv = {"kernel_h": 3, "kernel_w": 3, "stride_h": 1, "stride_w": 1, "pad_h": 1, "pad_w": 1,
            "dilation_h": 1, "dilation_w": 1, "groups": 1, "out_features": c, "has_bias": 0}
    cur = add("nn.conv2d", [0], dict(conv))
    cur = add("nn.batch_norm" if rng.random() < 0.5 else "batchnorm", [cur], {"epsilon": 1e-5})
    cur = add("nn.relu", [cur])
    ops = 3
    size = hw
    while ops + 10 < n_ops:
        skip = cur
        a = add("nn.conv2d", [cur], dict(conv))
        a = add("batchnorm", [a], {"epsilon": 1e-5})
        a = add("nn.relu", [a])
        a = add("nn.conv2d", [a], dict(conv))
        a = add("batchnorm", [a], {"epsilon": 1e-5})
        if rng.random() < 0.2:  # a constant scale through dropped plumbing (edge contraction)
            k = add("const", [])
            nodes[k]["out_shape"] = [batch, c, size, size]
            a = add("multiply", [a, k])
            ops += 1
        a = add("add", [a, skip])
        cur = add("nn.relu", [a])
        ops += 7
        if size >= 4 and rng.random() < 0.1:
            cur = add("nn.maxpool2d" if rng.random() < 0.5 else "maxpool2d", [cur],
                      {"kernel_h": 2, "kernel_w": 2, "stride_h": 2, "stride_w": 2})
            size //= 2
            ops += 1
    cur = add("global_avgpool2d", [cur])
    cur = add("reshape", [cur])
    cur = add("nn.dense", [cur], {"out_features": int(rng.integers(10, 1000)), "has_bias": 1})
    return json.dumps({"name": name, "batch": batch, "outputs": [cur], "nodes": nodes})


def make_graph_documents(count: int, seed: int = 5, n_lo: int = 12, n_hi: int = 5000, alpha: float = 1.5) -> list:
    """`count` graph JSON documents with operator-node counts from a truncated
    power law (N in [n_lo, n_hi], alpha 1.5)."""
    rng = np.random.default_rng(seed)
    u = rng.random(count)
    a1 = 1.0 - alpha
    n = ((n_hi ** a1 - n_lo ** a1) * u + n_lo ** a1) ** (1.0 / a1)
    return [_resnet_doc(int(k), rng, f"synth-{seed}-{i}") for i, k in enumerate(n.astype(np.int64))]
