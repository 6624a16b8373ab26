"""Loads the in-tree CUDA library (libsmpc_b200.so) and declares the C ABI.

There is no fallback: if the library is missing or no CUDA device is usable,
``load()`` raises. The product path never routes through the CPU oracle.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .scenario import (SmpcLoopResult, SmpcPlantConfig, SmpcProblem, SmpcSolution, SmpcTubeSolution,
                       SmpcWeightSummary)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsmpc_b200.so")

# Every symbol include/smpc_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "smpc_create", "smpc_create_with_ops", "smpc_destroy", "smpc_last_error", "smpc_error_location", "smpc_get_dims",
    "smpc_set_mean", "smpc_get_mean", "smpc_compute_control", "smpc_tube_compute_control",
    "smpc_shift_control_sequence", "smpc_get_solve_count", "smpc_set_solve_count",
    "smpc_generate_samples", "smpc_rollout", "smpc_compute_weights", "smpc_sorted_samples", "smpc_export_sample_trajectories", "smpc_run_control_loop", "smpc_run_control_loops", "smpc_set_x0",
    "smpc_launch_iteration", "smpc_synchronize", "smpc_stream", "smpc_kernels_per_solve",
    "smpc_rollout_kernel_ms", "smpc_icdf_domain", "smpc_icdf_table", "smpc_comm_unique_id", "smpc_comm_init", "smpc_comm_set_mode", "smpc_set_injected_noise", "smpc_group_init",
    "smpc_group_compute_control", "smpc_host_libm_uses_fma",
    "smpc_measure_fp32_peak", "smpc_sqrt_check", "smpc_libm_hash", "smpc_fast_math_check", "smpc_select_noise_strategy", "smpc_noise_strategy_rule",
    "smpc_version",
]

_lib = None


# smpc_model_ops (include/smpc_b200.h): a user model's launcher table
_OPS_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class SmpcModelOps(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("args_bytes", ctypes.c_int32),
        ("n_x", ctypes.c_int32),
        ("n_u", ctypes.c_int32),
        ("n_y", ctypes.c_int32),
        ("name", ctypes.c_char_p),
        ("user", ctypes.c_void_p),
        ("user_bytes", ctypes.c_int64),
        ("rollout", ctypes.c_void_p),
        ("update", ctypes.c_void_p),
        ("combine", ctypes.c_void_p),
        ("generate", ctypes.c_void_p),
        ("plant_step", ctypes.c_void_p),
        ("rmppi_select", ctypes.c_void_p),
    ]


class SmpcError(RuntimeError):
    """smpc::Error — message text matches the reference's exception."""

    def __init__(self, status: int, message: str, sample=-1, timestep=-1, channel=-1):
        super().__init__(message)
        self.status = status
        self.sample, self.timestep, self.channel = sample, timestep, channel


class SmpcConfigError(SmpcError):
    """smpc::ConfigError."""


NOISE_AUTO, NOISE_SPLIT, NOISE_FUSED = 0, 1, 2


class SmpcNoiseChoice(ctypes.Structure):
    """smpc_noise_choice (include/smpc_b200.h)."""
    _fields_ = [("kind", ctypes.c_int32), ("split_median_ms", ctypes.c_double),
                ("fused_median_ms", ctypes.c_double), ("timed", ctypes.c_int32)]


def load(path: str = None) -> ctypes.CDLL:
    """Load the library (SMPC_B200_LIB overrides the in-tree path, for A/B runs)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("SMPC_B200_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = ctypes.CDLL(path)
    P = ctypes.POINTER
    c_ctx = ctypes.c_void_p
    f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
    u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
    L.smpc_create.argtypes = [P(SmpcProblem), P(c_ctx)]
    L.smpc_create_with_ops.argtypes = [P(SmpcProblem), P(SmpcModelOps), P(c_ctx)]
    L.smpc_create_with_ops.restype = ctypes.c_int
    L.smpc_destroy.argtypes = [c_ctx]
    L.smpc_destroy.restype = None
    L.smpc_last_error.argtypes = [c_ctx]
    L.smpc_last_error.restype = ctypes.c_char_p
    L.smpc_error_location.argtypes = [c_ctx, P(ctypes.c_int64), P(ctypes.c_int32), P(ctypes.c_int32)]
    L.smpc_get_dims.argtypes = [c_ctx, P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32)]
    L.smpc_set_mean.argtypes = [c_ctx, ctypes.c_int32, f32p]
    L.smpc_get_mean.argtypes = [c_ctx, ctypes.c_int32, f32p]
    L.smpc_compute_control.argtypes = [c_ctx, f32p, P(SmpcSolution)]
    L.smpc_tube_compute_control.argtypes = [c_ctx, f32p, P(SmpcTubeSolution)]
    L.smpc_shift_control_sequence.argtypes = [c_ctx, ctypes.c_double, ctypes.c_double]
    L.smpc_get_solve_count.argtypes = [c_ctx, P(ctypes.c_uint64)]
    L.smpc_set_solve_count.argtypes = [c_ctx, ctypes.c_uint64]
    L.smpc_generate_samples.argtypes = [c_ctx, f32p, ctypes.c_uint32, f32p, ctypes.c_void_p]
    L.smpc_rollout.argtypes = [c_ctx, ctypes.c_int32, f32p, f32p, ctypes.c_void_p, ctypes.c_uint32, f64p,
                               ctypes.c_void_p]
    L.smpc_compute_weights.argtypes = [c_ctx, f64p, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p,
                                       P(SmpcWeightSummary)]
    L.smpc_sorted_samples.argtypes = [c_ctx, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    L.smpc_run_control_loop.argtypes = [c_ctx, P(SmpcPlantConfig), f32p, ctypes.c_double, P(SmpcLoopResult),
                                         ctypes.c_void_p]
    L.smpc_run_control_loops.argtypes = [P(c_ctx), ctypes.c_int32, P(SmpcPlantConfig), f32p, ctypes.c_double,
                                          P(SmpcLoopResult)]
    L.smpc_export_sample_trajectories.argtypes = [c_ctx, f32p, f32p, ctypes.c_void_p, ctypes.c_uint32,
                                                  ctypes.c_double, P(ctypes.c_int64), ctypes.c_void_p,
                                                  ctypes.c_void_p]
    L.smpc_set_x0.argtypes = [c_ctx, f32p]
    L.smpc_launch_iteration.argtypes = [c_ctx]
    L.smpc_synchronize.argtypes = [c_ctx]
    L.smpc_stream.argtypes = [c_ctx]
    L.smpc_stream.restype = ctypes.c_void_p
    L.smpc_kernels_per_solve.argtypes = [c_ctx]
    L.smpc_kernels_per_solve.restype = ctypes.c_int32
    L.smpc_rollout_kernel_ms.argtypes = [c_ctx, ctypes.c_int32, P(ctypes.c_double), P(ctypes.c_int64)]
    L.smpc_icdf_domain.argtypes = [c_ctx, f32p]
    L.smpc_icdf_table.argtypes = [c_ctx, f32p]
    L.smpc_comm_unique_id.argtypes = [ctypes.c_char_p]
    L.smpc_comm_init.argtypes = [c_ctx, ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32]
    L.smpc_set_injected_noise.argtypes = [c_ctx, ctypes.c_void_p]
    L.smpc_set_injected_noise.restype = ctypes.c_int
    L.smpc_comm_set_mode.argtypes = [c_ctx, ctypes.c_int32]
    L.smpc_comm_set_mode.restype = ctypes.c_int
    L.smpc_group_init.argtypes = [P(c_ctx), ctypes.c_int32]
    L.smpc_group_compute_control.argtypes = [P(c_ctx), ctypes.c_int32, f32p, P(SmpcSolution)]
    L.smpc_host_libm_uses_fma.argtypes = []
    L.smpc_host_libm_uses_fma.restype = ctypes.c_int32
    L.smpc_measure_fp32_peak.argtypes = [ctypes.c_int32, P(ctypes.c_double)]
    L.smpc_measure_fp32_peak.restype = ctypes.c_int
    L.smpc_sqrt_check.argtypes = [ctypes.c_int32, P(ctypes.c_uint64)]
    L.smpc_sqrt_check.restype = ctypes.c_int
    L.smpc_libm_hash.argtypes = [ctypes.c_int32, ctypes.c_int32, P(ctypes.c_uint64)]
    L.smpc_libm_hash.restype = ctypes.c_int
    L.smpc_fast_math_check.argtypes = [ctypes.c_int32, ctypes.c_int32, P(ctypes.c_uint64)]
    L.smpc_fast_math_check.restype = ctypes.c_int
    L.smpc_select_noise_strategy.argtypes = [c_ctx, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, f32p,
                                             P(SmpcNoiseChoice)]
    L.smpc_select_noise_strategy.restype = ctypes.c_int
    L.smpc_noise_strategy_rule.argtypes = [ctypes.c_double] * 4
    L.smpc_noise_strategy_rule.restype = ctypes.c_int32
    L.smpc_version.argtypes = []
    L.smpc_version.restype = ctypes.c_char_p
    for name in ["smpc_create", "smpc_error_location", "smpc_get_dims", "smpc_set_mean", "smpc_get_mean",
                 "smpc_compute_control", "smpc_tube_compute_control", "smpc_shift_control_sequence",
                 "smpc_get_solve_count", "smpc_set_solve_count", "smpc_generate_samples", "smpc_rollout",
                 "smpc_compute_weights", "smpc_sorted_samples", "smpc_export_sample_trajectories", "smpc_run_control_loop", "smpc_run_control_loops", "smpc_set_x0", "smpc_launch_iteration", "smpc_synchronize",
                 "smpc_rollout_kernel_ms", "smpc_icdf_domain", "smpc_icdf_table", "smpc_comm_unique_id", "smpc_comm_init", "smpc_group_init",
                 "smpc_group_compute_control"]:
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def check(status: int, ctx=None) -> None:
    if status == 0:
        return
    L = load()
    msg = (L.smpc_last_error(ctx) or b"").decode()
    sample, t, ch = ctypes.c_int64(-1), ctypes.c_int32(-1), ctypes.c_int32(-1)
    if ctx:
        L.smpc_error_location(ctx, ctypes.byref(sample), ctypes.byref(t), ctypes.byref(ch))
    cls = SmpcConfigError if status == 2 else SmpcError
    raise cls(status, msg, sample.value, t.value, ch.value)
