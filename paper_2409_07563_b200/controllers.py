"""Python mirror of the reference's controller / engine / sampler interface,
running on the B200 through the C ABI (include/smpc_b200.h).

Names, argument meaning and error behaviour follow the reference:
  make_controller            controllers.cpp:294-344
  MppiController             controllers.hpp:89-97   (compute_control, set_mean,
                                                      shift_control_sequence)
  TubeMppiController         controllers.hpp:134-160 (tube_compute_control)
  RolloutEngine              engine.hpp:98-151       (rollout, compute_weights)
  GaussianSampler            sampling.hpp:50-84      (generate_samples)
Errors raise SmpcError / SmpcConfigError carrying the reference's exception
text (smpc::Error / smpc::ConfigError).
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Optional

import numpy as np

from . import _lib
from ._lib import SmpcConfigError, SmpcError, check
from .scenario import Scenario, SmpcSolution, SmpcTubeSolution, SmpcWeightSummary, shard_range

__all__ = ["make_controller", "MppiController", "TubeMppiController", "RolloutEngine", "GaussianSampler",
           "ControllerSolution", "TubeSolution", "WeightResult", "SmpcError", "SmpcConfigError"]


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


@dataclasses.dataclass
class WeightResult:
    """engine.hpp:87-91 plus the argmin the north star pins."""

    baseline: float
    normalizer: float
    weights: Optional[np.ndarray]
    argmin: int = -1
    nonzero: int = -1


@dataclasses.dataclass
class ControllerSolution:
    """controllers.hpp:17-27."""

    controls: np.ndarray  # [T, n_u]
    states: np.ndarray    # [T+1, n_x]
    outputs: np.ndarray   # [T, n_y]
    weights: WeightResult
    solve_time_ms: float


@dataclasses.dataclass
class TubeSolution:
    """controllers.hpp:120-127 (applied = nominal u0; PID stays host-side)."""

    nominal: ControllerSolution
    real: ControllerSolution
    nominal_state: np.ndarray


class _Context:
    """Owns one smpc_ctx (device buffers + captured CUDA graph)."""

    def __init__(self, scenario: Scenario, shard: Optional[tuple] = None, ops=None):
        """ops: a user model's smpc_model_ops (SmpcModelOps, from a plugin
        compiled against include/smpc_b200_plugin.cuh) for dynamics="plugin"."""
        self.lib = _lib.load()
        self.scenario = scenario
        self._problem = scenario.to_problem(shard)
        self.ctx = ctypes.c_void_p()
        if ops is not None:
            self._ops = ops
            check(self.lib.smpc_create_with_ops(ctypes.byref(self._problem), ctypes.byref(ops), ctypes.byref(self.ctx)))
        else:
            check(self.lib.smpc_create(ctypes.byref(self._problem), ctypes.byref(self.ctx)))
        nx, nu, ny = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        self.lib.smpc_get_dims(self.ctx, ctypes.byref(nx), ctypes.byref(nu), ctypes.byref(ny))
        self.n_x, self.n_u, self.n_y = nx.value, nu.value, ny.value
        self.T = scenario.horizon
        self.M = scenario.num_samples
        self.shard = shard if shard is not None else (0, self.M)
        self.M_local = self.shard[1] - self.shard[0]

    def close(self) -> None:
        if getattr(self, "ctx", None) and self.ctx.value:
            self.lib.smpc_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, status: int) -> None:
        check(status, self.ctx)


class RolloutEngine(_Context):
    """RolloutEngine::rollout / compute_weights on the device."""

    def rollout(self, x0s, means, eps=None, stream: int = 0, outputs: bool = False):
        """costs [S, M_shard] (importance term included when enabled) [, outputs [S, M, T, n_y]].

        eps=None regenerates the Philox batch for `stream` inside the kernel;
        otherwise eps is an injected batch [M_shard, T, n_u] (reference layout).
        """
        x0s = _f32(x0s).reshape(-1)
        S = x0s.size // self.n_x
        means = _f32(means).reshape(-1)
        costs = np.zeros(S * self.M_local, np.float64)
        outs = np.zeros(S * self.M_local * self.T * self.n_y, np.float32) if outputs else None
        e = _f32(eps).reshape(-1) if eps is not None else None
        self._check(self.lib.smpc_rollout(self.ctx, S, x0s, means, e.ctypes.data if e is not None else None,
                                          stream, costs, outs.ctypes.data if outs is not None else None))
        costs = costs.reshape(S, self.M_local)
        if outputs:
            return costs, outs.reshape(S, self.M_local, self.T, self.n_y)
        return costs

    def export_sample_trajectories(self, x0, mean, fraction: float, eps=None, stream: int = 0):
        """RolloutEngine::export_sample_trajectories (engine.cpp:411-455): the
        ceil(fraction*M) lowest-cost samples (cost, index order) of the rollout
        of (x0, mean, eps | Philox stream) and their [k, T, n_y] outputs."""
        k_max = int(np.ceil(fraction * self.M)) if 0.0 <= fraction <= 1.0 else 0
        order = np.zeros(max(k_max, 1), np.int64)
        outs = np.zeros(max(k_max, 1) * self.T * self.n_y, np.float32)
        k = ctypes.c_int64()
        e = _f32(eps).reshape(-1) if eps is not None else None
        self._check(self.lib.smpc_export_sample_trajectories(
            self.ctx, _f32(x0).ravel(), _f32(mean).ravel(), e.ctypes.data if e is not None else None, stream,
            float(fraction), ctypes.byref(k), order.ctypes.data, outs.ctypes.data))
        return order[:k.value], outs[:k.value * self.T * self.n_y].reshape(k.value, self.T, self.n_y)

    def select_noise_strategy(self, kind: str = "auto", trials: int = 0, split_budget_bytes: float = 256 << 20,
                              x0=None) -> dict:
        """RolloutEngine::auto_select / set_strategy (engine.cpp:281-335) for the
        device's noise evaluation orders: "split" (normals materialised by one
        parallel pass) or "fused" (regenerated in registers); "auto" applies
        the scratch budget, then times both from x0 (median of max(3, trials)
        after 2 warm-ups) and keeps fused only if strictly faster."""
        from ._lib import SmpcNoiseChoice, NOISE_AUTO, NOISE_SPLIT, NOISE_FUSED
        k = {"auto": NOISE_AUTO, "split": NOISE_SPLIT, "fused": NOISE_FUSED}[kind]
        ch = SmpcNoiseChoice()
        x = _f32(x0 if x0 is not None else self.scenario.x0()).ravel()
        if x.size == self.n_x:  # the same state for both systems of a Tube controller
            x = np.tile(x, 2)
        self._check(self.lib.smpc_select_noise_strategy(self.ctx, k, int(trials), float(split_budget_bytes), x,
                                                        ctypes.byref(ch)))
        return {"kind": {NOISE_SPLIT: "split", NOISE_FUSED: "fused"}[ch.kind],
                "split_median_ms": ch.split_median_ms, "fused_median_ms": ch.fused_median_ms,
                "timed": bool(ch.timed)}

    def compute_weights(self, costs, lam: float) -> WeightResult:
        costs = np.ascontiguousarray(costs, np.float64).ravel()
        w = np.zeros_like(costs)
        sm = SmpcWeightSummary()
        self._check(self.lib.smpc_compute_weights(self.ctx, costs, costs.size, float(lam), w.ctypes.data,
                                                  ctypes.byref(sm)))
        return WeightResult(sm.baseline, sm.normalizer, w, sm.argmin, sm.nonzero)


class GaussianSampler(_Context):
    """GaussianSampler::generate_samples on the device (reference layout out)."""

    def generate_samples(self, mean, stream: int):
        eps = np.zeros(self.M_local * self.T * self.n_u, np.float32)
        flags = np.zeros(self.M_local, np.uint8)
        self._check(self.lib.smpc_generate_samples(self.ctx, _f32(mean).ravel(), stream, eps, flags.ctypes.data))
        return eps.reshape(self.M_local, self.T, self.n_u), flags


class MppiController(RolloutEngine):
    """MppiController (also DMD: step sizes via the scenario; CemController:
    elite selection via controller="cem", controllers.cpp:149-203)."""

    def set_mean(self, mean, system: int = 0) -> None:
        self._check(self.lib.smpc_set_mean(self.ctx, system, _f32(mean).ravel()))

    def mean(self, system: int = 0) -> np.ndarray:
        out = np.zeros(self.T * self.n_u, np.float32)
        self._check(self.lib.smpc_get_mean(self.ctx, system, out))
        return out.reshape(self.T, self.n_u)

    def reset_mean(self) -> None:
        self.set_mean(np.zeros((self.T, self.n_u), np.float32))

    @property
    def solve_count(self) -> int:
        n = ctypes.c_uint64()
        self._check(self.lib.smpc_get_solve_count(self.ctx, ctypes.byref(n)))
        return n.value

    @solve_count.setter
    def solve_count(self, n: int) -> None:
        self._check(self.lib.smpc_set_solve_count(self.ctx, int(n)))

    def shift_control_sequence(self, elapsed_s: float, dt_min: float) -> None:
        self._check(self.lib.smpc_shift_control_sequence(self.ctx, float(elapsed_s), float(dt_min)))

    def _solution_struct(self, want_weights: bool):
        bufs = dict(controls=np.zeros(self.T * self.n_u, np.float32),
                    states=np.zeros((self.T + 1) * self.n_x, np.float32),
                    outputs=np.zeros(self.T * self.n_y, np.float32),
                    weights=np.zeros(self.M_local, np.float64) if want_weights else None)
        sol = SmpcSolution()
        sol.controls = bufs["controls"].ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        sol.states = bufs["states"].ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        sol.outputs = bufs["outputs"].ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        if want_weights:
            sol.weights = bufs["weights"].ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        return sol, bufs

    def _wrap(self, sol, bufs) -> ControllerSolution:
        s = sol.summary
        return ControllerSolution(
            controls=bufs["controls"].reshape(self.T, self.n_u),
            states=bufs["states"].reshape(self.T + 1, self.n_x),
            outputs=bufs["outputs"].reshape(self.T, self.n_y),
            weights=WeightResult(s.baseline, s.normalizer, bufs["weights"], s.argmin, s.nonzero),
            solve_time_ms=sol.solve_time_ms)

    def compute_control(self, x0, want_weights: bool = False) -> ControllerSolution:
        sol, bufs = self._solution_struct(want_weights)
        self._check(self.lib.smpc_compute_control(self.ctx, _f32(x0).ravel(), ctypes.byref(sol)))
        return self._wrap(sol, bufs)

    def sorted_samples(self, count: int, system: int = 0):
        """(order, costs) of the first `count` samples of the last rollout in
        (cost, index) order — std::partial_sort with CemController's
        comparator (controllers.cpp:165-171), on the device."""
        order = np.zeros(count, np.int64)
        costs = np.zeros(count, np.float64)
        self._check(self.lib.smpc_sorted_samples(self.ctx, system, int(count), order.ctypes.data, costs.ctypes.data))
        return order, costs

    # --- device-resident replay (bench) -----------------------------------
    def set_x0(self, x0) -> None:
        self._check(self.lib.smpc_set_x0(self.ctx, _f32(x0).ravel()))

    def launch_iteration(self) -> None:
        self._check(self.lib.smpc_launch_iteration(self.ctx))

    def synchronize(self) -> None:
        self._check(self.lib.smpc_synchronize(self.ctx))

    @property
    def stream(self) -> int:
        return self.lib.smpc_stream(self.ctx) or 0

    @property
    def kernels_per_solve(self) -> int:
        return self.lib.smpc_kernels_per_solve(self.ctx)

    def rollout_timing(self, enable: Optional[bool] = None):
        """(total rollout-kernel ms, launches) since the last (re)enable."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        flag = -1 if enable is None else int(bool(enable))
        self._check(self.lib.smpc_rollout_kernel_ms(self.ctx, flag, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def comm_init(self, unique_id: bytes, rank: int, world: int) -> None:
        self._check(self.lib.smpc_comm_init(self.ctx, unique_id, rank, world))

    def set_injected_noise(self, device_ptr: int) -> None:
        """Injected-noise mode: later solves read the shard's [M_local, T, n_u]
        fp32 noise from this DEVICE pointer (e.g. a CUDA tensor's data_ptr());
        0 returns to the Philox sampler. The caller keeps the buffer alive."""
        self._check(self.lib.smpc_set_injected_noise(self.ctx, ctypes.c_void_p(int(device_ptr)) if device_ptr else None))

    def comm_set_mode(self, mode: str) -> None:
        """"single" (default): one all-gather per iteration; "exact": three."""
        self._check(self.lib.smpc_comm_set_mode(self.ctx, COMM_MODES[mode]))


class TubeMppiController(MppiController):
    """TubeMppiController: nominal + real systems share one noise batch."""

    def tube_compute_control(self, x_real, want_weights: bool = False) -> TubeSolution:
        ns, nb = self._solution_struct(want_weights)
        rs, rb = self._solution_struct(want_weights)
        nominal_state = np.zeros(self.n_x, np.float32)
        t = SmpcTubeSolution()
        t.nominal, t.real = ns, rs
        t.nominal_state = nominal_state.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        self._check(self.lib.smpc_tube_compute_control(self.ctx, _f32(x_real).ravel(), ctypes.byref(t)))
        return TubeSolution(self._wrap(t.nominal, nb), self._wrap(t.real, rb), nominal_state)

    def compute_control(self, x0, want_weights: bool = False) -> ControllerSolution:
        return self.tube_compute_control(x0, want_weights).nominal


COMM_MODES = {"exact": 0, "single": 1}


def make_controller(scenario: Scenario, shard: Optional[tuple] = None, ops=None) -> MppiController:
    """make_controller (controllers.cpp:294-344): mppi | dmd | cem | tube (+ rmppi, builder-defined).
    ops: a user model's smpc_model_ops for scenario.dynamics == "plugin"."""
    if scenario.controller in ("tube", "rmppi"):
        return TubeMppiController(scenario, shard, ops)
    if scenario.controller in ("mppi", "dmd", "cem"):
        return MppiController(scenario, shard, ops)
    raise SmpcConfigError(2, f"controller.kind '{scenario.controller}' is not recognized")


def host_libm_uses_fma() -> bool:
    return bool(_lib.load().smpc_host_libm_uses_fma())


class ShardGroup:
    """n sample shards of one problem in this process (smpc_group_*): the
    multi-GPU iteration (rank-indexed gathers, fixed-rank-order combine) with
    device-to-device copies standing in for NCCL. devices: one ordinal per
    shard (default: all on the scenario's device)."""

    def __init__(self, scenario: Scenario, n: int, devices=None, mode: str = "single"):
        self.n = n
        self.members = []
        for r in range(n):
            sc = dataclasses.replace(scenario)
            if devices is not None:
                sc.device = devices[r]
            self.members.append(MppiController(sc, shard_range(scenario.num_samples, r, n)))
            self.members[-1].comm_set_mode(mode)
        self.lib = self.members[0].lib
        self._arr = (ctypes.c_void_p * n)(*[m.ctx.value for m in self.members])
        check(self.lib.smpc_group_init(self._arr, n), self.members[0].ctx)

    def compute_control(self, x0):
        m0 = self.members[0]
        sols, bufs = [], []
        for m in self.members:
            s, b = m._solution_struct(False)
            sols.append(s)
            bufs.append(b)
        arr = (SmpcSolution * self.n)(*sols)
        check(self.lib.smpc_group_compute_control(self._arr, self.n, _f32(x0).ravel(), arr), m0.ctx)
        return [m._wrap(arr[i], bufs[i]) for i, m in enumerate(self.members)]
