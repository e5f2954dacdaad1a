"""ctypes binding of libdynscreen.so (the C ABI declared in include/dynscreen.h).

The library is loaded lazily and loudly: if it is missing or no CUDA device is
present, the first call raises.  There is no CPU fallback anywhere in the
package.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libdynscreen.so")
CHECKED_PATH = os.path.join(HERE, "_lib", "libdynscreen_checked.so")   # DSCR_LIB=checked: bounds-checked build

DSCR_OK, DSCR_EINVAL, DSCR_ENONFINITE, DSCR_ERADIUS, DSCR_ECUDA, DSCR_ENOCOMM = 0, -1, -2, -3, -4, -5
F64, F32, BF16 = 0, 1, 2
ALGO_CODES = {"ista": 0, "fista": 1, "twist": 2, "sparsa": 3, "cp": 4}
STRATEGY_CODES = {"none": 0, "static": 1, "dynamic": 2}
TEST_CODES = {None: -1, "safe": 0, "dst3": 1, "dome": 2, "gsafe": 3, "gst3": 4}
STOP_RUNNING, STOP_RELTOL, STOP_GAP, STOP_MAXITER, STOP_EMPTY, STOP_TRIVIAL, STOP_ERROR = range(7)
TRACE_FIELDS = 10
TR_T, TR_KEPT, TR_NNZ, TR_OBJ, TR_GAP, TR_RADIUS, TR_L, TR_NS, TR_UNITS, TR_SUPPORT = range(10)
(PH_SETUP_LOCAL, PH_SETUP_ADOPT, PH_SETUP_VEC, PH_SETUP_FINISH, PH_STATIC_LOCAL, PH_STATIC_FINISH) = range(6)
PH_K1, PH_K1R, PH_K2, PH_K3A, PH_K3S, PH_K3B = range(10, 16)
PH_K2S, PH_K1R1, PH_K2C = 16, 17, 18
PH_K3X_PUSH, PH_K3X_REDUCE = 19, 20   # native exchange over peer memory
OC_SLOT, OC_MAX_WORLD = 8, 64   # one-collective rank slots: 8 doubles per rank after the SUM vector
CM_MAX, CM_SETUP, CM_SUM, CM_VEC = 0, 8, 16, 32

ABI_FUNCTIONS = (
    "dscr_last_error", "dscr_abi_version", "dscr_correlate", "dscr_column_norms", "dscr_corr_prox",
    "dscr_group_corr_prox", "dscr_residual", "dscr_compact_work_size", "dscr_compact", "dscr_apply_work_size", "dscr_apply", "dscr_prox_l1",
    "dscr_prox_group", "dscr_test_sphere", "dscr_test_dome", "dscr_test_group",
    "dscr_operator_norm_work_size", "dscr_operator_norm", "dscr_solver_workspace_size",
    "dscr_solver_create", "dscr_solver_setup", "dscr_solver_run", "dscr_solver_scalars",
    "dscr_solver_get_buffers", "dscr_solver_profile", "dscr_solver_phase", "dscr_solver_set_collectives", "dscr_solver_set_peers", "dscr_peer_buffer_bytes",
    "dscr_peer_alloc", "dscr_peer_open", "dscr_peer_close", "dscr_peer_free", "dscr_solver_destroy",
    "dscr_batched_gemm_bf16", "dscr_batched_workspace_size", "dscr_batched_create", "dscr_batched_setup",
    "dscr_batched_run", "dscr_batched_get_buffers", "dscr_batched_profile", "dscr_batched_destroy",
    "dscr_corr_exact_work_size", "dscr_corr_exact_bf16", "dscr_group_spectral_norms", "dscr_ingest_rows_f64",
)


class ProblemDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("n_rows", C.c_int32), ("n_cols", C.c_int32), ("ldd", C.c_int32),
        ("D", C.c_void_p), ("y", C.c_void_p), ("lam", C.c_double),
        ("n_groups", C.c_int32), ("norm_aware", C.c_int32),
        ("group_ptr", C.c_void_p), ("group_w", C.c_void_p), ("group_snorm", C.c_void_p),
        ("col_offset", C.c_int32), ("n_cols_total", C.c_int32),
        ("group_offset", C.c_int32), ("n_groups_total", C.c_int32),
        ("col_norms", C.c_void_p),
    ]


class Config(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int32), ("strategy", C.c_int32), ("test", C.c_int32), ("max_iters", C.c_int32),
        ("rel_tol", C.c_double), ("gap_tol", C.c_double), ("L0", C.c_double),
        ("backtrack_factor", C.c_double), ("twist_alpha", C.c_double), ("twist_beta", C.c_double),
        ("twist_step", C.c_double), ("cp_gamma", C.c_double), ("cp_step_safety", C.c_double),
        ("bb_L_min", C.c_double), ("bb_L_max", C.c_double), ("op_norm", C.c_double),
    ]


_SCALAR_INTS = ("t run_limit max_iters mode stop status parity xi moved have_fprev n_units n_units_new "
                "n_support p_eff kept_atoms nnz dropped_nz nonfinite trivial lmax_index lmax_unit any_group "
                "static_done trips").split()
_SCALAR_DBLS = ("L l_acc l_new beta tau sigma phi sigma_new theta_sq theta_y yy lmax lmax_sign shift_sq "
                "corr_inf mu rsafe_sq radius dome_rs dome_cut dome_slope dome_flat maj_cs maj_ss pen ss_red "
                "f_prev F gap t0_ns gst3_coef gst3_nsq ds_sq fc tw_step spare astar_nsq gstar_w oc_empty oc_spare").split()


class Scalars(C.Structure):
    _fields_ = [(n, C.c_int32) for n in _SCALAR_INTS] + [(n, C.c_double) for n in _SCALAR_DBLS]


class Buffers(C.Structure):
    _fields_ = [
        ("scalars", C.c_void_p), ("theta", C.c_void_p * 2), ("resid", C.c_void_p), ("corr", C.c_void_p),
        ("x", C.c_void_p * 3), ("u", C.c_void_p * 2), ("y_corr", C.c_void_p), ("star_corr", C.c_void_p),
        ("cc", C.c_void_p), ("cnorm", C.c_void_p), ("act", C.c_void_p * 2), ("act_cnt", C.c_void_p * 2),
        ("act_off", C.c_void_p * 2), ("mask", C.c_void_p), ("trace", C.c_void_p),
        ("kts", C.c_void_p), ("max_kts", C.c_int32), ("G", C.c_int32), ("cap", C.c_int32), ("comm_len", C.c_int32),
        ("comm", C.c_void_p), ("vec", C.c_void_p),
    ]


class BatchedDesc(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int32), ("n_atoms", C.c_int32), ("n_obs", C.c_int32), ("ldd", C.c_int32),
        ("Dt", C.c_void_p), ("Y", C.c_void_p), ("ldy", C.c_int32), ("splits", C.c_int32),
        ("lam", C.c_void_p), ("L", C.c_double), ("test", C.c_int32), ("cap", C.c_int32),
        ("max_iters", C.c_int32), ("fused", C.c_int32), ("beta", C.c_void_p),
    ]


class BatchedBuffers(C.Structure):
    _fields_ = [
        ("s_idx", C.c_void_p * 2), ("s_x", C.c_void_p * 2), ("s_u", C.c_void_p * 2), ("s_cnt", C.c_void_p * 2),
        ("F", C.c_void_p), ("gap", C.c_void_p), ("nnz", C.c_void_p), ("kept", C.c_void_p),
        ("status", C.c_void_p), ("lmax", C.c_void_p), ("radius", C.c_void_p), ("trace", C.c_void_p),
        ("iterations", C.c_void_p), ("C", C.c_void_p), ("mask", C.c_void_p),
    ]


_lib = None
_lock = threading.Lock()


def _declare(lib):
    vp, i32, i64, dbl, sz = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_size_t
    sig = {
        "dscr_last_error": (C.c_char_p, []),
        "dscr_abi_version": (i32, []),
        "dscr_correlate": (i32, [i32, vp, i32, i32, i32, vp, vp, vp]),
        "dscr_column_norms": (i32, [i32, vp, i32, i32, i32, vp, vp]),
        "dscr_corr_prox": (i32, [i32, vp, i32, i32, vp, i32, vp, vp, vp, dbl, i32, dbl, dbl, vp, vp, vp, vp, vp]),
        "dscr_group_corr_prox": (i32, [i32, vp, i32, i32, vp, vp, i32, vp, i32, vp, vp, vp, vp, dbl, i32, dbl, dbl,
                                       vp, vp, vp, vp, vp, vp]),
        "dscr_residual": (i32, [i32, vp, i32, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp]),
        "dscr_compact_work_size": (sz, [i32]),
        "dscr_compact": (i32, [vp, i32, vp, vp, vp, vp, sz, vp]),
        "dscr_apply_work_size": (sz, [i32, i32, i32]),
        "dscr_apply": (i32, [i32, vp, i32, i32, i32, vp, vp, vp, sz, vp]),
        "dscr_prox_l1": (i32, [vp, i64, dbl, vp, vp]),
        "dscr_prox_group": (i32, [vp, vp, i32, vp, dbl, vp, vp]),
        "dscr_test_sphere": (i32, [vp, vp, i32, dbl, vp, vp]),
        "dscr_test_dome": (i32, [vp, vp, vp, i32, dbl, dbl, dbl, vp, vp]),
        "dscr_test_group": (i32, [vp, vp, vp, vp, i32, dbl, vp, vp]),
        "dscr_operator_norm_work_size": (sz, [i32, i32]),
        "dscr_operator_norm": (i32, [i32, vp, i32, i32, i32, dbl, i32, vp, C.POINTER(dbl), vp]),
        "dscr_solver_workspace_size": (sz, [C.POINTER(ProblemDesc), C.POINTER(Config)]),
        "dscr_solver_create": (i32, [C.POINTER(ProblemDesc), C.POINTER(Config), vp, sz, vp, C.POINTER(vp)]),
        "dscr_solver_setup": (i32, [vp, vp]),
        "dscr_solver_run": (i32, [vp, i32, vp]),
        "dscr_solver_scalars": (i32, [vp, vp, C.POINTER(Scalars)]),
        "dscr_solver_get_buffers": (i32, [vp, C.POINTER(Buffers)]),
        "dscr_solver_destroy": (i32, [vp]),
        "dscr_solver_profile": (i32, [vp, i32, vp, C.POINTER(C.c_float)]),
        "dscr_solver_phase": (i32, [vp, i32, vp]),
        "dscr_solver_set_collectives": (i32, [vp, i32, i32, i32]),
        "dscr_solver_set_peers": (i32, [vp, i32, i32, vp, vp]),
        "dscr_peer_buffer_bytes": (sz, [i32, i32]),
        "dscr_peer_alloc": (i32, [sz, C.POINTER(vp), vp]),
        "dscr_peer_open": (i32, [vp, C.POINTER(vp)]),
        "dscr_peer_close": (i32, [vp]),
        "dscr_peer_free": (i32, [vp]),
        "dscr_batched_gemm_bf16": (i32, [vp, i32, i32, vp, i32, i32, i32, i32, vp, i32, vp]),
        "dscr_batched_workspace_size": (sz, [C.POINTER(BatchedDesc)]),
        "dscr_batched_create": (i32, [C.POINTER(BatchedDesc), vp, sz, vp, C.POINTER(vp)]),
        "dscr_batched_setup": (i32, [vp, vp]),
        "dscr_batched_run": (i32, [vp, i32, vp]),
        "dscr_batched_get_buffers": (i32, [vp, C.POINTER(BatchedBuffers)]),
        "dscr_batched_destroy": (i32, [vp]),
        "dscr_batched_profile": (i32, [vp, i32, vp, C.POINTER(C.c_float)]),
        "dscr_corr_exact_work_size": (sz, [i32, i32, i32]),
        "dscr_corr_exact_bf16": (i32, [vp, i32, i32, i32, vp, i32, i32, vp, i32, vp, sz, vp]),
        "dscr_group_spectral_norms": (i32, [i32, vp, i32, i32, i32, vp, vp, dbl, i32, vp, vp]),
        "dscr_ingest_rows_f64": (i32, [vp, i32, i32, i32, i32, vp, i32, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load_library(path=LIB_PATH):
    """dlopen the library without touching the GPU (used by the CPU symbol tests)."""
    lib = C.CDLL(path)
    _declare(lib)
    return lib


def lib():
    """The loaded library; raises if it is missing or no CUDA device exists."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            sel = os.environ.get("DSCR_LIB", "")
            path = CHECKED_PATH if sel == "checked" else (sel if sel.endswith(".so") else LIB_PATH)
            if not os.path.exists(path):
                raise RuntimeError(
                    f"{os.path.basename(path)} not built ({path}); run `python -m paper_1412_4080_b200.build`")
            import torch
            if not torch.cuda.is_available():
                raise RuntimeError("paper_1412_4080_b200 needs a CUDA device (sm_100a); none is available")
            _lib = load_library(path)
    return _lib


def check(rc, what="dynscreen"):
    """Map a C return code onto the reference's exception types."""
    if rc == DSCR_OK:
        return
    msg = lib().dscr_last_error().decode(errors="replace") or what
    if rc == DSCR_EINVAL:
        raise ValueError(msg)
    if rc == DSCR_ENONFINITE:
        raise FloatingPointError(msg)
    raise RuntimeError(msg)


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
