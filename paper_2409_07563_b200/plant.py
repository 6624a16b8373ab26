"""Closed-loop driver on the device: the reference's Plant::run_control_loop
(plant.cpp:133-181) and the step-size sweep bench_dmd_sweep (bench.cpp:86-133)
through the C ABI (smpc_run_control_loop / smpc_run_control_loops).

The simulated system, the shifts, every compute_control and the applied
control / cost / disturbed Euler step stay on the GPU; independent runs (the
sweep's trials) advance in lockstep on their own streams.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .controllers import MppiController, make_controller
from .scenario import Scenario, SmpcLoopResult, SmpcPlantConfig


@dataclasses.dataclass
class LoopResult:
    """plant.hpp LoopResult; rows = ControlLogRow {t, x, u, running_cost} as arrays."""

    accumulated_cost: float
    solve_count: int
    mean_solve_ms: float
    t: Optional[np.ndarray] = None
    x: Optional[np.ndarray] = None
    u: Optional[np.ndarray] = None
    running_cost: Optional[np.ndarray] = None


@dataclasses.dataclass
class SweepRecord:
    """bench.hpp SweepRecord."""

    samples: int
    gamma: float
    mean_cost: float
    std_cost: float
    mean_ms: float
    trials: int


def plant_config(sc: Scenario) -> SmpcPlantConfig:
    return SmpcPlantConfig(float(sc.replan_rate), float(sc.dt_min), float(sc.disturbance_std),
                           int(sc.rng_seed) & 0xFFFFFFFFFFFFFFFF)


def run_control_loop(ctl: MppiController, duration_s: float, x0=None, log: bool = False) -> LoopResult:
    """Plant::run_control_loop(sim, duration_s) with make_plant / make_simulated_system
    of the controller's scenario (plant.cpp:208-230)."""
    sc = ctl.scenario
    x0 = np.ascontiguousarray(sc.x0() if x0 is None else x0, np.float32)
    steps = int(round(duration_s / sc.dt))
    width = 2 + ctl.n_x + ctl.n_u
    rows = np.zeros(max(steps, 1) * width, np.float64) if log else None
    res = SmpcLoopResult()
    pc = plant_config(sc)
    ctl._check(ctl.lib.smpc_run_control_loop(ctl.ctx, ctypes.byref(pc), x0, float(duration_s), ctypes.byref(res),
                                             rows.ctypes.data if rows is not None else None))
    out = LoopResult(res.accumulated_cost, res.solve_count, res.mean_solve_ms)
    if log:
        r = rows.reshape(-1, width)[:steps]
        out.t, out.x = r[:, 0], r[:, 1:1 + ctl.n_x]
        out.u, out.running_cost = r[:, 1 + ctl.n_x:1 + ctl.n_x + ctl.n_u], r[:, -1]
    return out


def run_control_loops(ctls: Sequence[MppiController], duration_s: float) -> List[LoopResult]:
    """Independent closed loops advanced in lockstep (one stream per controller)."""
    n = len(ctls)
    lib = ctls[0].lib
    arr = (ctypes.c_void_p * n)(*[c.ctx.value for c in ctls])
    pcs = (SmpcPlantConfig * n)(*[plant_config(c.scenario) for c in ctls])
    x0s = np.ascontiguousarray(np.concatenate([c.scenario.x0() for c in ctls]), np.float32)
    outs = (SmpcLoopResult * n)()
    _lib.check(lib.smpc_run_control_loops(arr, n, pcs, x0s, float(duration_s), outs), ctls[0].ctx)
    return [LoopResult(o.accumulated_cost, o.solve_count, o.mean_solve_ms) for o in outs]


def _stats(values):
    v = np.asarray(values, np.float64)
    mean = float(v.sum() / v.size) if v.size else 0.0
    std = float(math.sqrt(((v - mean) ** 2).sum() / (v.size - 1))) if v.size > 1 else 0.0
    return mean, std


def bench_dmd_sweep(scenario: Scenario, sample_counts=(64, 256, 1024, 4096), gammas=(0.2, 0.4, 0.6, 0.8, 1.0),
                    trials: int = 50, steps: int = 1000, base_seed: int = 0) -> List[SweepRecord]:
    """bench.cpp:86-133 on the device: per (samples, gamma) cell, `trials`
    closed loops of `steps` steps (dmd controller, step size gamma, seed
    base_seed + trial), all trials of a cell run concurrently."""
    if trials < 1:
        raise ValueError("bench_dmd_sweep: need at least 1 trial")
    if steps < 1:
        raise ValueError("bench_dmd_sweep: need at least 1 step")
    if not sample_counts or not gammas:
        raise ValueError("bench_dmd_sweep: sample counts and gammas must be non-empty")
    for g in gammas:
        if not (0.0 < g <= 1.0):
            raise ValueError("bench_dmd_sweep: gammas must be in (0, 1]")
    records = []
    for samples in sample_counts:
        if samples < 1:
            raise ValueError("bench_dmd_sweep: sample counts must be >= 1")
        for gamma in gammas:
            ctls = []
            for trial in range(trials):
                run = dataclasses.replace(scenario, num_samples=int(samples), controller="dmd", step_size=float(gamma),
                                          step_size_per_step=None, rng_seed=base_seed + trial)
                ctls.append(make_controller(run))
            res = run_control_loops(ctls, steps * scenario.dt)
            for c in ctls:
                c.close()
            cost_mean, cost_std = _stats([r.accumulated_cost for r in res])
            ms_mean, _ = _stats([r.mean_solve_ms for r in res])
            records.append(SweepRecord(int(samples), float(gamma), cost_mean, cost_std, ms_mean, trials))
    return records


def best_gamma_per_samples(records: Sequence[SweepRecord]):
    """bench.cpp:135-154: lowest mean cost per sample count, ties to the smaller gamma."""
    best, order = {}, []
    for r in records:
        if r.samples not in best:
            best[r.samples] = r
            order.append(r.samples)
        elif r.mean_cost < best[r.samples].mean_cost or (
                r.mean_cost == best[r.samples].mean_cost and r.gamma < best[r.samples].gamma):
            best[r.samples] = r
    return [(s, best[s].gamma) for s in order]


def write_sweep_csv(path: str, records: Sequence[SweepRecord]) -> None:
    """bench.cpp:170-181 (same header and %.9g formatting)."""
    with open(path, "w") as f:
        f.write("samples,gamma,mean_cost,std_cost,mean_ms,trials\n")
        for r in records:
            f.write("%d,%.9g,%.9g,%.9g,%.9g,%d\n" % (r.samples, r.gamma, r.mean_cost, r.std_cost, r.mean_ms, r.trials))
