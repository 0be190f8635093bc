"""ctypes mirror of ``include/mixedstep_b200.h`` and the loader of the in-tree
``libmixedstep_b200.so``.

The product path has no CPU fallback: if the library is missing the import of
the compute API raises, and every compute call on a machine without a B200
returns MS_ECUDA, surfaced here as :class:`CudaError`.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
# MS_LIB_PATH: an alternative build of the same sources (kernel-geometry tuning runs)
LIB_PATH = Path(os.environ["MS_LIB_PATH"]) if os.environ.get("MS_LIB_PATH") else PKG / "libmixedstep_b200.so"

MS_OK, MS_EINVAL, MS_ECUDA = 0, 1, 2
MS_BINARY32, MS_BINARY64 = 0, 1
MS_SINGLE, MS_MIXED1, MS_MIXED2, MS_DOUBLE, MS_CUSTOM = 0, 1, 2, 3, 4
(MS_COMPLETED, MS_MAX_ITERATIONS, MS_MAX_FAILED_STEPS, MS_WALL_CLOCK, MS_SLOW_SOLVER,
 MS_STEP_TOO_SMALL, MS_NON_FINITE) = range(7)
MS_MODEL_LCO, MS_MODEL_KURAMOTO, MS_MODEL_CC = 0, 1, 2
MS_MODEL_SCALAR_EXP, MS_MODEL_SCALAR_ZERO, MS_MODEL_SCALAR_NAN = 16, 17, 18
MS_K_SCALAR, MS_K_F32, MS_K_F16, MS_K_BF16 = 0, 1, 2, 3
MS_HOST_F64, MS_HOST_F32 = 0, 1
MS_RHS_FAST, MS_RHS_FAITHFUL, MS_RHS_ORDERED = 0, 1, 2


class StagePrec(C.Structure):
    _fields_ = [("f_prec", C.c_uint8), ("sum_prec", C.c_uint8), ("g_prec", C.c_uint8), ("_pad", C.c_uint8)]


class Policy(C.Structure):
    _fields_ = [("per_stage", StagePrec * 3), ("first_step_k1", StagePrec), ("storage", C.c_uint8),
                ("variant", C.c_uint8), ("_pad", C.c_uint8 * 2)]


class SolverConfigC(C.Structure):
    _fields_ = [
        ("rel_tol", C.c_double), ("abs_tol", C.c_double), ("h_min_factor", C.c_double),
        ("max_iterations", C.c_int64), ("max_failed_steps", C.c_int64),
        ("time_limits_enabled", C.c_int32), ("record_step_log", C.c_int32),
        ("wall_clock_limit", C.c_double), ("slow_solver_elapsed", C.c_double),
        ("slow_solver_progress", C.c_double), ("safety", C.c_double), ("fac_min", C.c_double),
        ("fac_max", C.c_double), ("controller_exponent", C.c_double),
        ("record_snapshots", C.c_int32), ("_pad", C.c_int32),
    ]


class StepRecordC(C.Structure):
    _fields_ = [("t", C.c_double), ("h", C.c_double), ("err", C.c_double), ("accepted", C.c_int32),
                ("_pad", C.c_int32)]


_DP = C.POINTER(C.c_double)


class SystemDesc(C.Structure):
    _fields_ = [
        ("model", C.c_int32), ("n_agents", C.c_int32), ("coupled_slot", C.c_int32),
        ("k_storage", C.c_int32), ("rhs_mode", C.c_int32), ("device", C.c_int32),
        ("row_begin", C.c_int32), ("row_end", C.c_int32),
        ("coupling_k", C.c_double), ("stimulus_i0", C.c_double),
        ("m", _DP), ("omega", _DP), ("w2", _DP), ("cc_k1", _DP), ("cc_theta_h", _DP),
        ("cc_k0", _DP), ("cc_k2", _DP), ("cc_a", _DP), ("cc_b", _DP), ("cc_c", _DP), ("cc_eps", _DP),
        ("K", C.c_void_p), ("k_host_dtype", C.c_int32), ("_pad", C.c_int32),
    ]


class SolveResultC(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("_pad", C.c_int32), ("t_reached", C.c_double),
        ("n_accepted", C.c_int64), ("n_failed", C.c_int64), ("rhs_evals", C.c_int64),
        ("flops_low", C.c_int64), ("flops_high", C.c_int64),
        ("final_state", _DP), ("step_log", C.POINTER(StepRecordC)),
        ("step_log_capacity", C.c_int64), ("step_log_count", C.c_int64), ("device_ms", C.c_double),
        ("snapshots", _DP), ("snapshot_h", _DP), ("snapshot_capacity", C.c_int64), ("snapshot_count", C.c_int64),
        ("t_eval", _DP), ("n_eval", C.c_int64), ("y_eval", _DP), ("n_eval_done", C.c_int64),
    ]


class StepOutcomeC(C.Structure):
    _fields_ = [
        ("x_next", _DP), ("x_tilde", _DP), ("k4", _DP), ("x_store", _DP),
        ("err", C.c_double), ("accepted", C.c_int32), ("_pad", C.c_int32),
        ("h_used", C.c_double), ("h_next", C.c_double),
        ("rhs_evals", C.c_int64), ("flops_low", C.c_int64), ("flops_high", C.c_int64),
    ]


class BatchResultC(C.Structure):
    _fields_ = [("status", C.POINTER(C.c_int32)), ("t_reached", _DP), ("n_accepted", C.POINTER(C.c_int64)),
                ("n_failed", C.POINTER(C.c_int64)), ("rhs_evals", C.POINTER(C.c_int64)), ("final_state", _DP),
                ("attempts", C.c_int64), ("device_ms", C.c_double)]


class ExchangeC(C.Structure):
    _fields_ = [("needed", C.c_int32), ("_pad", C.c_int32), ("buf", C.c_void_p), ("offset", C.c_int64),
                ("count", C.c_int64), ("total", C.c_int64)]


# (name, restype, argtypes) of every symbol include/mixedstep_b200.h declares
SIGNATURES = [
    ("ms_abi_version", C.c_int, []),
    ("ms_last_error", C.c_char_p, []),
    ("ms_abi_sizes", C.c_int, [C.POINTER(C.c_int64)]),
    ("ms_device_count", C.c_int, []),
    ("ms_launch_count", C.c_int64, []),
    ("ms_default_config", None, [C.POINTER(SolverConfigC)]),
    ("ms_policy_for", C.c_int, [C.c_int, C.POINTER(Policy)]),
    ("ms_policy_lowest_format", C.c_int, [C.POINTER(Policy)]),
    ("ms_rng_uniform", C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, C.c_double, C.c_double, _DP]),
    ("ms_rng_normal", C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, _DP]),
    ("ms_system_create", C.c_int, [C.POINTER(SystemDesc), C.POINTER(C.c_void_p)]),
    ("ms_system_destroy", C.c_int, [C.c_void_p]),
    ("ms_system_fill_k_uniform", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_double, C.c_double]),
    ("ms_system_get_k", C.c_int, [C.c_void_p, _DP]),
    ("ms_system_dim", C.c_int, [C.c_void_p]),
    ("ms_system_agents", C.c_int, [C.c_void_p]),
    ("ms_system_flop_profile", C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    ("ms_eval_rhs", C.c_int, [C.c_void_p, C.c_double, _DP, StagePrec, _DP]),
    ("ms_estimate_error", C.c_int, [C.c_int64, _DP, _DP, _DP, C.c_double, C.c_double, _DP]),
    ("ms_adjust_step", C.c_int, [C.c_double, C.c_double, C.c_double, C.POINTER(SolverConfigC), _DP]),
    ("ms_initial_step", C.c_int, [C.c_void_p, C.c_double, C.c_double, _DP, C.POINTER(SolverConfigC), C.c_int,
                                  _DP, C.POINTER(C.c_int64)]),
    ("ms_bs32_step", C.c_int, [C.c_void_p, C.c_double, _DP, C.c_double, _DP, C.POINTER(Policy),
                               C.POINTER(SolverConfigC), C.POINTER(StepOutcomeC)]),
    ("ms_solve", C.c_int, [C.c_void_p, _DP, C.c_double, C.c_double, C.POINTER(Policy), C.POINTER(SolverConfigC),
                           C.POINTER(SolveResultC)]),
    ("ms_solve_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.POINTER(Policy),
                                  C.POINTER(SolverConfigC), C.POINTER(SolveResultC), C.c_void_p]),
    ("ms_loop_begin", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double, C.POINTER(Policy),
                                C.POINTER(SolverConfigC), C.c_int64, C.c_void_p]),
    ("ms_loop_segment_count", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int)]),
    ("ms_loop_run_segment", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.POINTER(ExchangeC)]),
    ("ms_loop_done", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]),
    ("ms_loop_end", C.c_int, [C.c_void_p, C.POINTER(SolveResultC), C.c_int, C.c_void_p]),
    ("ms_loop_push_info", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                    C.POINTER(C.c_void_p)]),
    ("ms_loop_push_setup", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    ("ms_loop_push_wait", C.c_int, [C.c_void_p, C.c_void_p]),
    ("ms_ipc_export", C.c_int, [C.c_void_p, C.POINTER(C.c_ubyte)]),
    ("ms_ipc_import", C.c_int, [C.POINTER(C.c_ubyte), C.POINTER(C.c_void_p)]),
    ("ms_ipc_close", C.c_int, [C.c_void_p]),
    ("ms_variants_create", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("ms_variants_destroy", C.c_int, [C.c_void_p]),
    ("ms_variants_solve", C.c_int, [C.c_void_p, _DP, C.c_double, C.c_double, C.POINTER(Policy),
                                    C.POINTER(SolverConfigC), C.POINTER(SolveResultC)]),
    ("ms_batch_create", C.c_int, [C.c_void_p, C.c_int32, _DP, C.c_int32, C.POINTER(C.c_void_p)]),
    ("ms_batch_destroy", C.c_int, [C.c_void_p]),
    ("ms_batch_eval_rhs", C.c_int, [C.c_void_p, _DP, StagePrec, _DP]),
    ("ms_batch_solve", C.c_int, [C.c_void_p, _DP, C.c_double, C.c_double, C.POINTER(Policy),
                                 C.POINTER(SolverConfigC), C.POINTER(BatchResultC)]),
    ("ms_batch_profile_rhs", C.c_int, [C.c_void_p, _DP, StagePrec, C.c_int, _DP, _DP]),
    ("ms_profile_rhs", C.c_int, [C.c_void_p, _DP, StagePrec, C.c_int, _DP, _DP]),
    ("ms_dp54_reference", C.c_int, [C.c_void_p, _DP, C.c_double, C.c_double, C.POINTER(SolverConfigC),
                                    C.POINTER(SolveResultC)]),
]


class MixedstepError(RuntimeError):
    pass


class CudaError(MixedstepError):
    """MS_ECUDA: CUDA failure or no B200 present (there is no CPU fallback)."""


_lib = None


ABI_VERSION = 3  # MS_ABI_VERSION of include/mixedstep_b200.h


def lib() -> C.CDLL:
    """Load the in-tree sm_100a library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, res, args in SIGNATURES:
            if os.environ.get("MS_LIB_PATH") and not hasattr(L, name):
                continue  # an older build used for an A/B timing run
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.ms_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH}: ABI version {L.ms_abi_version()} != {ABI_VERSION}: rebuild it")
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == MS_OK:
        return
    msg = (lib().ms_last_error() or b"").decode(errors="replace")
    if rc == MS_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise CudaError(f"{what}: {msg}")


def dptr(a) -> "C._Pointer":
    """double* of a C-contiguous float64 numpy array (None -> NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(_DP)


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0")
