"""ctypes binding of the C ABI in include/gridcast_b200.h (libgridcast_b200.so).

The library is built in-tree (``python -m paper_2603_01122_b200.build`` or
``__graft_entry__.build()``) into ``paper_2603_01122_b200/_lib/``.  There is no CPU
fallback: every product entry point calls :func:`lib` and fails loudly when the
shared library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GC_LIB_PATH: load another build of the same ABI (A/B timing of kernel variants)
LIB_PATH = os.environ.get("GC_LIB_PATH") or os.path.join(_HERE, "_lib", "libgridcast_b200.so")

GC_OK = 0
GC_BAD_ARG = 1
GC_EMPTY_CONTROL_SET = 2
GC_SNAP_MISMATCH = 3
GC_UNSUPPORTED_Q = 4
GC_CUDA_ERROR = 5
GC_WINDOW_OVERFLOW = 6
# bits of gc_predict's d_error word (include/gridcast_b200.h)
GC_ERRBIT_WINDOW_OVERFLOW = 1 << 6
GC_ERRBIT_HYPOTHESES = 1 << 8
GC_ERRBIT_WINDOW_CAPACITY = 1 << 9
GC_ERRBIT_TABLE_ID = 1 << 10
GC_ERRBIT_ASSUME_QG = 1 << 11
GC_MAX_HYPOTHESES = 256
GC_MAX_SMOOTH_RADIUS = 56  # include/gridcast_b200.h
GC_MAX_ACTIONS = 512

GC_Q_GOAL_PROGRESS = 0
GC_Q_GOAL_PROGRESS_FULL = 1
GC_Q_DEFAULT = 2
GC_Q_TABLE = 3
GC_UNION_MAX, GC_UNION_INDEPENDENT, GC_UNION_MISS, GC_UNION_COMPLEMENT = 0, 1, 2, 3

GC_HIST_GLOBAL, GC_HIST_SMEM = 0, 1

GC_RNG_REFERENCE = 0
GC_RNG_UNIFORMS = 1
GC_RNG_PRODUCTION = 2

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U64 = ctypes.c_uint64
F32 = ctypes.c_float
F64 = ctypes.c_double


class ActionTable(ctypes.Structure):
    _fields_ = [
        ("m", I32), ("m_keep", I32), ("q_kind", I32), ("ref_grid_rows", I32),
        ("d_sx", P), ("d_sy", P), ("d_at", P), ("d_pen", P), ("d_dispx", P), ("d_dispy", P),
        ("d_keep", P),
        ("n_speeds", I32), ("n_headings", I32),
        ("dv", F32), ("tau", F32), ("w_v", F32), ("w_th", F32),
        ("d_cos_h", P), ("d_sin_h", P), ("d_theta_h", P), ("d_a_index", P),
        ("h_cos_h", P), ("h_sin_h", P), ("h_theta_h", P),
    ]


class PredictArgs(ctypes.Structure):
    _fields_ = [
        ("n_humans", I32), ("n", I32), ("steps", I32), ("rng_mode", I32),
        ("grid_w", I32), ("grid_h", I32),
        ("origin_x32", F32), ("origin_y32", F32), ("res32", F32),
        ("d_start_xy", P), ("d_hyp_off", P), ("d_beta32", P), ("d_goal32", P),
        ("d_cdf", P), ("d_log_w", P),
        ("d_seed", P), ("d_prefix", P), ("d_prefix_len", P), ("d_stream_id", P),
        ("d_uniforms", P), ("d_hyp_u", P), ("d_hyp_in", P),
        ("h_tables", ctypes.POINTER(ActionTable)), ("n_tables", I32), ("d_table_id", P),
        ("d_step_r", P), ("d_step_off", P), ("human_stride", I64),
        ("max_win_cells", I32), ("_pad2", I32), ("d_counts", P),
        ("d_hyp_out", P), ("d_xy_out", P), ("d_error", P),
        ("t_begin", I32), ("t_end", I32), ("d_state_xy", P), ("d_state_hyp", P),
        ("p_offset", I32), ("hist_path", I32),
        ("ref_exact_only", I32), ("d_ref_fallbacks", P),
        ("assume_qg", I32), ("_pad3", I32),
    ]


class EpilogueArgs(ctypes.Structure):
    _fields_ = [
        ("n_humans", I32), ("n", I32), ("steps", I32),
        ("grid_w", I32), ("grid_h", I32), ("radius", I32),
        ("d_kernel", P), ("d_zx", P), ("d_zy", P),
        ("origin_x32", F32), ("origin_y32", F32), ("res32", F32), ("n_tiles", I32),
        ("d_start_xy", P), ("d_step_r", P), ("d_step_off", P), ("human_stride", I64),
        ("d_tiles", P), ("d_counts", P),
        ("d_layers64", P), ("d_union32", P), ("d_union64", P), ("time_union", I32),
        ("tile_begin", I32), ("tile_end", I32), ("t_begin", I32), ("t_end", I32),
        ("_pad_e", I32), ("d_union_tile_flags", P),
    ]


class PublishArgs(ctypes.Structure):
    _fields_ = [
        ("steps", I32), ("grid_w", I32), ("grid_h", I32), ("t_begin", I32), ("t_end", I32),
        ("dtype_bytes", I32), ("time_or", I32), ("_pad", I32),
        ("d_union", P), ("d_tile_flags", P), ("d_host_flags", P), ("h_dst", P),
    ]


class BeliefArgs(ctypes.Structure):
    _fields_ = [
        ("n_humans", I32), ("m", I32),
        ("d_v", P), ("d_theta", P), ("d_sx", P), ("d_sy", P), ("d_at", P), ("d_pen", P),
        ("d_masked", P), ("q_kind", I32), ("d_qtable", P), ("d_hyp_off", P),
        ("d_beta", P), ("d_goal", P), ("d_obs", P), ("d_fallback_theta", P),
        ("dt", F64), ("snap_tol", F64), ("clamp_on_mismatch", I32),
        ("d_prior", P), ("d_post", P), ("d_status", P), ("d_action", P),
    ]


class ExactArgs(ctypes.Structure):
    _fields_ = [
        ("n_hyp", I32), ("m", I32), ("grid_w", I32), ("grid_h", I32), ("steps", I32), ("q_kind", I32),
        ("origin_x", F64), ("origin_y", F64), ("res", F64), ("z0x", F64), ("z0y", F64),
        ("d_beta", P), ("d_goal", P), ("d_belief", P),
        ("d_sx", P), ("d_sy", P), ("d_at", P), ("d_pen", P),
        ("d_dispx", P), ("d_dispy", P), ("d_masked", P), ("d_qtable", P), ("d_qtable0", P),
        ("d_pi", P), ("d_p", P), ("d_nxt", P), ("d_pi0", P), ("d_landing", P), ("d_layers", P),
    ]


class NaiveArgs(ctypes.Structure):
    _fields_ = [
        ("n", I32), ("steps", I32), ("n_hyp", I32), ("m_keep", I32),
        ("q_kind", I32), ("grid_w", I32), ("grid_h", I32), ("prefix_len", I32),
        ("seed", U64), ("prefix", ctypes.c_uint32 * 4),
        ("start_x", F64), ("start_y", F64), ("origin_x", F64), ("origin_y", F64), ("res", F64),
        ("d_hyp", P), ("d_beta", P), ("d_goal", P), ("d_keep", P),
        ("d_sx", P), ("d_sy", P), ("d_at", P), ("d_pen", P), ("d_dispx", P), ("d_dispy", P),
        ("d_counts", P), ("d_xy_out", P),
    ]


class MppiArgs(ctypes.Structure):
    _fields_ = [
        ("n_rollouts", I32), ("horizon", I32),
        ("dt", F64), ("temperature", F64), ("std_a", F64), ("std_w", F64),
        ("q", F64 * 4), ("qf", F64 * 4), ("r", F64 * 2), ("collision_penalty", F64),
        ("quadratic_control_cost", I32),
        ("a_max", F64), ("omega_max", F64), ("v_max", F64),
        ("z", F64 * 4), ("goal", F64 * 4),
        ("d_nominal", P), ("d_noise", P), ("seed", U64), ("d_blocked", P),
        ("n_layers", I32), ("grid_w", I32), ("grid_h", I32),
        ("origin_x", F64), ("origin_y", F64), ("res", F64),
        ("d_layer_of", P), ("d_noise_out", P),
        ("d_costs", P), ("d_controls", P), ("d_weights", P), ("d_diag", P),
    ]


EXPORTS = (
    "gc_predict", "gc_grid_epilogue", "gc_belief_update", "gc_propagate_step",
    "gc_sample_hypotheses", "gc_derive_seed", "gc_stream_f32", "gc_last_error",
    "gc_abi_version", "gc_launch_count", "gc_emplace_counts", "gc_smooth_layers",
    "gc_collision_field", "gc_exact_predict", "gc_mppi_step", "gc_predict_naive",
    "gc_union_layers", "gc_time_union", "gc_publish_tiles", "gc_fill_zero", "gc_union_tiles",
    "gc_peer_alloc", "gc_peer_free", "gc_peer_export", "gc_peer_import", "gc_peer_close",
)

_lib = None


class GridcastLibraryMissing(RuntimeError):
    """The sm_100a shared library has not been built (no CPU fallback exists)."""


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise GridcastLibraryMissing(
            f"{LIB_PATH} not found; build it with `python -m paper_2603_01122_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.gc_predict.argtypes = [ctypes.POINTER(PredictArgs), P]
    L.gc_grid_epilogue.argtypes = [ctypes.POINTER(EpilogueArgs), P]
    L.gc_belief_update.argtypes = [ctypes.POINTER(BeliefArgs), P]
    L.gc_propagate_step.argtypes = [P, P, I32, P, P, I32, ctypes.POINTER(ActionTable), P, U64, P,
                                    I32, I32, P]
    L.gc_sample_hypotheses.argtypes = [P, I32, I32, U64, P, I32, P, P]
    L.gc_emplace_counts.argtypes = [P, I64, I32, I32, F32, F32, F32, P, P]
    L.gc_smooth_layers.argtypes = [P, P, I32, I32, I32, I32, P, P, P, P]
    L.gc_collision_field.argtypes = [P, I32, I32, I32, I32, P, I32, F64, P, P, P]
    L.gc_exact_predict.argtypes = [ctypes.POINTER(ExactArgs), P]
    L.gc_mppi_step.argtypes = [ctypes.POINTER(MppiArgs), P]
    L.gc_predict_naive.argtypes = [ctypes.POINTER(NaiveArgs), P]
    L.gc_union_layers.argtypes = [P, I32, I32, I64, I64, I32, P, I32, P]
    L.gc_time_union.argtypes = [P, I32, I32, I32, I64, P]
    L.gc_publish_tiles.argtypes = [ctypes.POINTER(PublishArgs), P]
    L.gc_fill_zero.argtypes = [P, I64, P]
    L.gc_union_tiles.argtypes = [P, I32, I32, I32, I32, P, I32, P, I32, P]
    L.gc_peer_alloc.argtypes = [I64, ctypes.POINTER(P)]
    L.gc_peer_free.argtypes = [P]
    L.gc_peer_export.argtypes = [P, P]
    L.gc_peer_import.argtypes = [P, ctypes.POINTER(P)]
    L.gc_peer_close.argtypes = [P]
    for fn in ("gc_predict", "gc_grid_epilogue", "gc_belief_update", "gc_propagate_step",
               "gc_sample_hypotheses", "gc_emplace_counts", "gc_smooth_layers", "gc_collision_field",
               "gc_exact_predict", "gc_mppi_step", "gc_predict_naive", "gc_union_layers",
               "gc_time_union", "gc_publish_tiles", "gc_fill_zero", "gc_union_tiles", "gc_peer_alloc", "gc_peer_free", "gc_peer_export", "gc_peer_import",
               "gc_peer_close"):
        getattr(L, fn).restype = ctypes.c_int
    L.gc_derive_seed.argtypes = [U64, P, I32]
    L.gc_derive_seed.restype = U64
    L.gc_stream_f32.argtypes = [U64, P, I32, P, I64]
    L.gc_stream_f32.restype = None
    L.gc_last_error.restype = ctypes.c_char_p
    L.gc_abi_version.restype = I32
    L.gc_launch_count.restype = U64
    _lib = L
    return L


def last_error() -> str:
    return lib().gc_last_error().decode(errors="replace")


def check_error_word(word: int, what: str = "gc_predict"):
    """Raise for the GC_ERRBIT_* bits of a gc_predict device status word."""
    word = int(word) & 0xFFFFFFFF
    if word == 0:
        return
    if word & GC_ERRBIT_HYPOTHESES:
        raise ValueError(f"{what}: every human needs 1..{GC_MAX_HYPOTHESES} hypotheses")
    if word & GC_ERRBIT_WINDOW_CAPACITY:
        raise ValueError(f"{what}: max_win_cells is smaller than the launch's reachable-cell windows")
    if word & GC_ERRBIT_TABLE_ID:
        raise ValueError(f"{what}: a human's action-table id is outside the launch's tables")
    if word & GC_ERRBIT_ASSUME_QG:
        raise ValueError(f"{what}: assume_qg was set but a hypothesis needs the general speed-weight form")
    if word & GC_ERRBIT_WINDOW_OVERFLOW:
        raise RuntimeError(f"{what}: a particle left its reachable-cell window (internal error)")
    raise RuntimeError(f"{what}: device status word {word:#x}")


def check(status: int, what: str = ""):
    """Map a gc_status onto the reference's exception classes."""
    if status == GC_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == GC_EMPTY_CONTROL_SET:
        from .agents import EmptyControlSetError
        raise EmptyControlSetError(msg)
    if status == GC_SNAP_MISMATCH:
        from .belief import ControlSnapMismatch
        raise ControlSnapMismatch(msg)
    if status == GC_UNSUPPORTED_Q:
        raise NotImplementedError(msg)
    if status == GC_BAD_ARG:
        raise ValueError(msg)
    raise RuntimeError(msg)
