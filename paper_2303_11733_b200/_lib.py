"""ctypes binding of libdippm_b200.so (the C ABI declared in include/dippm_b200.h).

This is the only way the package reaches compute: there is no CPU or
PyTorch-eager fallback.  If the library is missing, or no CUDA device is
visible when a compute entry point is used, a DeviceUnavailable error is
raised.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import DippmError, NonFinite, ShapeMismatch

LIB_PATH = Path(__file__).resolve().parent / "libdippm_b200.so"

OK, ERR_ARG, ERR_CUDA, ERR_NONFINITE, ERR_UNSUPPORTED = 0, 1, 2, 3, 4
DT_F32, DT_BF16, DT_TF32X3 = 0, 1, 2
GEMM_FWD, GEMM_STORE, GEMM_WGRAD, GEMM_GATE = 0, 1, 2, 3


class DeviceUnavailable(DippmError):
    """The CUDA library or a CUDA device is not available (no fallback exists)."""


class KernelError(DippmError):
    """A CUDA launch or runtime error reported by the native library."""


class Act(C.Structure):
    """dippm_act_t: activation matrix view."""
    _fields_ = [("data", C.c_void_p), ("ld", C.c_int64), ("plane_stride", C.c_int64), ("dtype", C.c_int64)]


ABI_VERSION = 15  # DIPPM_ABI_VERSION in include/dippm_b200.h


class GemmArgs(C.Structure):
    """dippm_gemm_args_t."""
    _fields_ = [
        ("kind", C.c_int64), ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64),
        ("a", Act), ("a_mn_major", C.c_int64), ("b", Act), ("b_mn_major", C.c_int64),
        ("bias", C.c_void_p), ("relu", C.c_int64), ("out", Act),
        ("c", C.c_void_p), ("ldc", C.c_int64), ("splits", C.c_int64),
        ("gate", Act), ("gate_scale", C.c_double), ("drop_mode", C.c_int64), ("mask", C.c_void_p),
        ("ldm", C.c_int64), ("drop_p", C.c_double), ("seed", C.c_uint64), ("seed_dev", C.c_void_p),
        ("relu_bits", C.c_void_p), ("gate_bits", C.c_void_p), ("bits_ld", C.c_int64), ("cta_pair", C.c_int64),
        ("tile_sync", C.c_void_p), ("out_scale", C.c_double),
        ("pool_partial", C.c_void_p), ("pool_graph", C.c_void_p), ("node_graph", C.c_void_p),
        ("graph_ptr", C.c_void_p), ("bias_partial", C.c_void_p), ("bias_grad", C.c_void_p),
    ]


P, I32, I64, U64, F32, F64, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_size_t


class HeadArgs(C.Structure):
    """dippm_head_args_t (the fused FC head, dippm_head_fused)."""
    _fields_ = [
        ("G", C.c_int64), ("hp", C.c_int32), ("u_width", C.c_int32),
        ("u", P), ("w1", P), ("w2", P), ("b1", P), ("b2", P), ("w3", P), ("b3", P),
        ("x2", P), ("x3", P), ("bits", P), ("bits_ld", C.c_int64),
        ("drop_mode", C.c_int32), ("drop_p", C.c_double), ("keep_scale", C.c_float),
        ("seed1", C.c_uint64), ("seed2", C.c_uint64), ("seed_dev", P), ("mask1", P), ("mask2", P),
        ("out", P), ("norm", P), ("y_pred", P), ("mig", P), ("nonfinite", P),
        ("y_raw", P), ("delta", C.c_double), ("grad_den", C.c_double), ("loss_out", P), ("row_loss", P),
        ("dout", P), ("d2", P), ("d1", P), ("d2f", P), ("d1f", P),
        ("gw1", P), ("gb1", P), ("gw2", P), ("gb2", P), ("gw3", P), ("gb3", P), ("du", P),
        ("sync", P), ("train", C.c_int32),
        ("pool_partial", P), ("pool_graph", P), ("graph_ptr", P), ("fs_raw", P), ("step_counter", P),
        ("defer_reduce", C.c_int32),
    ]


class PackSeg(C.Structure):
    """dippm_pack_seg_t: one fp64-master -> compute-copy segment refreshed by dippm_adam_pack."""
    _fields_ = [("src_off", C.c_int64), ("rows", C.c_int64), ("cols", C.c_int64), ("dst_col_off", C.c_int64),
                ("dst", Act)]


MAX_PACK_SEGS = 12


class TrainPlan(C.Structure):
    """dippm_train_plan_t: the fixed device pointers of the native training step."""
    _fields_ = [
        ("hp", C.c_int32), ("u_width", C.c_int32),
        ("params", P), ("m", P), ("v", P), ("grads", P), ("p32", P), ("n_params", C.c_int64), ("t_dev", P),
        ("norm", P), ("Wf", Act * 3), ("Wd", Act * 3), ("W1h", Act), ("W2h", Act), ("segs", P), ("n_segs", C.c_int32),
        ("off_w", C.c_int64 * 3), ("off_b", C.c_int64 * 3),
        ("off_fc1w", C.c_int64), ("off_fc1b", C.c_int64), ("off_fc2w", C.c_int64), ("off_fc2b", C.c_int64),
        ("off_fc3w", C.c_int64), ("off_fc3b", C.c_int64),
        ("ws_N", C.c_int64), ("ws_G", C.c_int64), ("ws_E", C.c_int64),
        ("A", Act * 3), ("B", Act * 3), ("relu_bits", P), ("pool_part", P), ("pool_graph", P),
        ("u", Act), ("x2", Act), ("x3", Act), ("d2", Act), ("d1", Act), ("dhead_f32", P), ("head_bits", P),
        ("out", P), ("dout", P), ("du", P), ("loss", P), ("row_loss", P), ("head_sync", P),
        ("colsum", P), ("colsum3", P), ("colsum_sync", P), ("splitk", P), ("tile_sync", P),
        ("rowptr", P), ("col", P), ("deg", P), ("t_rowptr", P), ("t_col", P), ("bad", P), ("node_graph", P),
        ("inv_deg", P), ("csr_ws", P), ("csr_ws_bytes", C.c_size_t),
        ("dropout_p", C.c_double), ("keep_scale", C.c_double), ("delta", C.c_double), ("grad_den", C.c_double),
        ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("seed", C.c_uint64),
        ("side_stream", P), ("ev", P * 4), ("graph_exec", P), ("capture_stream", P), ("head_done", P),
    ]


class CsrSet(C.Structure):
    """dippm_csr_set_t: one batch's K1 outputs (CSR, transposed CSR, node->graph, A1)."""
    _fields_ = [("rowptr", P), ("col", P), ("deg", P), ("t_rowptr", P), ("t_col", P), ("node_graph", P),
                ("inv_deg", P), ("csr_ws", P), ("csr_ws_bytes", SZ), ("a1", Act), ("cap_N", C.c_int64),
                ("cap_E", C.c_int64)]


class TrainBatch(C.Structure):
    """dippm_train_batch_t: one device-resident batch for dippm_train_step."""
    _fields_ = [("x", P), ("src", P), ("dst", P), ("graph_ptr", P), ("edge_ptr", P), ("fs", P), ("y", P),
                ("N", C.c_int64), ("E", C.c_int64), ("G", C.c_int64), ("max_nodes", C.c_int32),
                ("max_edges", C.c_int32), ("loss_out", P), ("bad_out", P), ("csr", C.POINTER(CsrSet)),
                ("no_adam", C.c_int32)]


# name -> (restype, argtypes); must match include/dippm_b200.h
SIGNATURES = {
    "dippm_last_error": (C.c_char_p, []),
    "dippm_abi_version": (I32, []),
    "dippm_launch_count": (C.c_uint64, []),
    "dippm_device_sm_count": (I32, []),
    "dippm_mig_code": (I32, [F64, C.POINTER(I32)]),
    "dippm_mig_codes": (I32, [P, I64, I64, P, P, P]),
    "dippm_csr_workspace_bytes": (SZ, [I64, I64]),
    "dippm_build_csr": (I32, [P, P, I64, I64, P, P, P, P, P, P, P, P, SZ, P]),
    "dippm_csr_grouped_workspace_bytes": (SZ, [I64, I64]),
    "dippm_build_csr_grouped": (I32, [P, P, P, P, I64, I64, I64, I32, I32, P, P, P, P, P, P, P, P, P, SZ, P]),
    "dippm_build_csr_grouped_l1": (I32, [P, P, P, P, I64, I64, I64, I32, I32, P, P, P, P, P, P, P, P, P, SZ, P, Act, P]),
    "dippm_sage_aggregate": (I32, [Act, Act, Act, I64, I32, P, P, P, P]),
    "dippm_colsum_blocks": (I32, [I64]),
    "dippm_colsum_count_slot": (P, [P, I64, I32]),
    "dippm_colsum_rows": (I32, [I64]),
    "dippm_colsum_sync_ints": (I32, [I64]),
    "dippm_sage_aggregate_t": (I32, [Act, I32, I64, I32, P, P, P, P, P, P, P]),
    "dippm_readout_backward": (I32, [P, I64, P, I64, I32, Act, Act, I64, P]),
    "dippm_readout_aggregate_t": (I32, [P, I64, P, P, Act, Act, I32, I64, P, P, P, P, P, P, P, I64, P]),
    "dippm_node_graph": (I32, [P, I64, P, P]),
    "dippm_fs_normalize": (I32, [P, I64, P, Act, I32, P]),
    "dippm_reduce_rows": (I32, [P, I64, I64, I32, F64, P, P]),
    "dippm_wgrad_splits": (I32, [I64, I64, I64]),
    "dippm_wgrad_sync_ints": (I64, [I64, I64]),
    "dippm_gemm": (I32, [C.POINTER(GemmArgs), I32, P]),
    "dippm_splitk_reduce_t": (I32, [P, I32, I64, I64, F64, P, I64, P]),
    "dippm_pool_concat": (I32, [Act, P, I64, I32, P, P, Act, P]),
    "dippm_pool_partial_rows": (I64, [I64]),
    "dippm_pool_combine": (I32, [P, P, P, I64, I32, P, P, Act, P]),
    "dippm_fc3_forward": (I32, [Act, I64, I32, P, P, P, P, P, P, P, P]),
    "dippm_fc3_backward": (I32, [Act, I64, I32, P, P, F32, P, P, Act, P, P]),
    "dippm_head_fused_max_graphs": (I32, []),
    "dippm_head_fused_sync_ints": (I32, []),
    "dippm_head_tc_enable": (I32, [I32]),
    "dippm_head_tc_trace": (I32, [P]),
    "dippm_head_fused": (I32, [C.POINTER(HeadArgs), P]),
    "dippm_head_reduce": (I32, [C.POINTER(HeadArgs), P]),
    "dippm_head_fused_trace": (I32, [P]),
    "dippm_colsum_act": (I32, [Act, I64, I32, P, P]),
    "dippm_huber": (I32, [P, P, I64, P, F64, F64, P, P, P]),
    "dippm_adam_pack": (I32, [P, P, P, P, F64, I64, I64, P, F64, F64, F64, F64, I32, P, C.POINTER(PackSeg), I32, P]),
    "dippm_step_counter": (I32, [P, P]),
    "dippm_pack": (I32, [P, I64, I64, I32, Act, P]),
    "dippm_huber_f64": (I32, [P, P, I64, F64, P, P, P, P]),
    "dippm_adam": (I32, [P, P, P, P, P, I64, F64, F64, F64, F64, F64, F64, F64, F64, P]),
    "dippm_elementwise_f64": (I32, [I32, P, P, F64, P, I64, P]),
    "dippm_dgemm": (I32, [P, P, P, I64, I64, I64, P]),
    "dippm_mig_band_select": (I32, [P, I64, F64, P, P, P, P, P, P, P]),
    "dippm_gather_graphs": (I32, [P, I64, P, P, P, P, P, P, P, P, P, P, P, P, P]),
    "dippm_scatter_rescore": (I32, [P, I64, P, P, P, P, P]),
    "dippm_train_plan_init": (I32, [C.POINTER(TrainPlan)]),
    "dippm_train_plan_destroy": (I32, [C.POINTER(TrainPlan)]),
    "dippm_train_step": (I32, [C.POINTER(TrainPlan), C.POINTER(TrainBatch), P]),
    "dippm_train_step_graphed": (I32, [C.POINTER(TrainPlan), C.POINTER(TrainBatch), P]),
    "dippm_train_prep": (I32, [C.POINTER(TrainPlan), C.POINTER(TrainBatch), C.POINTER(CsrSet), P]),
}

_lib = None


def load():
    """Load the native library (once) and bind every exported symbol."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise DeviceUnavailable(
            f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.dippm_abi_version() != ABI_VERSION:
        raise DeviceUnavailable(f"{LIB_PATH.name} has ABI {lib.dippm_abi_version()}, expected {ABI_VERSION}; rebuild it")
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status == OK:
        return
    msg = load().dippm_last_error().decode(errors="replace")
    if status == ERR_NONFINITE:
        raise NonFinite(msg)
    if status in (ERR_ARG, ERR_UNSUPPORTED):
        raise ShapeMismatch(f"{what}: {msg}" if what else msg)
    raise KernelError(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
