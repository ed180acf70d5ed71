"""B200-native DIPPM GraphSAGE predictor (arXiv 2303.11733) — hot-path drop-in.

Mirrors the reference package's model / predict / train / MIG API
(`dippm.gnn`, `dippm.mig`, the training-step parts of `dippm.numerics`);
compute runs in hand-written sm_100a kernels behind the C ABI of
include/dippm_b200.h (libdippm_b200.so).  Featurisation, dataset I/O, the
graph IR and the CLI are out of scope.
"""

from .errors import (DippmError, EmptyDataset, EmptyGraph, IoFailure, NonFinite, ShapeMismatch,  # noqa: F401
                     VersionMismatch)
from .gnn import (DEFAULT_DROPOUT, DEFAULT_HIDDEN, AffineParams, DippmModel, MlpModel, Normalizer,  # noqa: F401
                  SageLayerParams, TrainConfig, backward, batch_loss, create_mlp_model, create_model, forward,
                  load_model, predict, predict_batch, predict_record, predict_records, readout_mean, sage_forward,
                  save_model, train, train_mlp)
from .mig import MigProfile, mig_profile  # noqa: F401
from .types import (FEATURE_WIDTH, STATIC_WIDTH, VOCAB_VERSION, DatasetRecord, GraphEncoding,  # noqa: F401
                    StaticFeatures, TargetVector)

__version__ = "0.1.0"
