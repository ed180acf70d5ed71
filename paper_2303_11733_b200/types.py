"""Boundary data types, field-for-field the reference's (featurize.py:48-87,
dataset.py:54-70).  The API is duck-typed: objects of the reference package
itself are accepted wherever these are."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

FEATURE_WIDTH = 32   # featurize.py:38
STATIC_WIDTH = 5     # featurize.py:39
VOCAB_VERSION = "v1"  # featurize.py:45


@dataclass(eq=False)
class GraphEncoding:
    """Adjacency edge list (producer -> consumer) plus node-feature matrix."""

    num_nodes: int
    edges: list
    features: np.ndarray  # (num_nodes, 32)

    def __eq__(self, other) -> bool:
        if not isinstance(other, GraphEncoding):
            return NotImplemented
        return (self.num_nodes == other.num_nodes and list(self.edges) == list(other.edges)
                and np.array_equal(self.features, other.features))


@dataclass
class StaticFeatures:
    """Graph-level summary: MACs, batch size, and three operator counts."""

    macs: int
    batch: int
    t_conv: int
    t_dense: int
    t_relu: int

    @property
    def as_vector(self) -> np.ndarray:
        return np.array([math.log1p(self.macs), math.log1p(self.batch), math.log1p(self.t_conv),
                         math.log1p(self.t_dense), math.log1p(self.t_relu)], dtype=np.float64)


@dataclass
class TargetVector:
    latency_ms: float
    memory_mb: float
    energy_j: float

    @property
    def as_array(self) -> np.ndarray:
        return np.array([self.latency_ms, self.memory_mb, self.energy_j], dtype=np.float64)


@dataclass
class DatasetRecord:
    encoding: GraphEncoding
    fs: StaticFeatures
    target: TargetVector
    model_name: str = ""


def fs_vector(fs) -> np.ndarray:
    """F_s as the 5-vector the network consumes (StaticFeatures.as_vector or a raw array)."""
    if hasattr(fs, "as_vector"):
        return np.asarray(fs.as_vector, dtype=np.float64)
    return np.asarray(fs, dtype=np.float64).reshape(STATIC_WIDTH)


def target_vector(t) -> np.ndarray:
    if hasattr(t, "as_array"):
        return np.asarray(t.as_array, dtype=np.float64)
    return np.asarray(t, dtype=np.float64).reshape(3)
