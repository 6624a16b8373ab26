"""GPU closed loop (smpc_run_control_loop): the device-resident
Plant::run_control_loop (plant.cpp:133-181) against the reference's own loop
(tests/golden/loop_*.npz, from oracle/_ref via oracle/gen_golden.py) and the
Python checker loop around the C oracle (oracle.bindings.control_loop).

Bars: the replan schedule, shifts and disturbance noise are integer/bit work
and exact; applied controls inherit the 1e-4 FP32 tolerance of U* and the
states/costs are compared with the same |a-b| <= 1e-4 * max(1, |a|, |b|).
"""
import glob
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def close(a, b, tol=TOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))


def relerr(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))))


@pytest.fixture(scope="module")
def mods(oracle_built):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import bindings
    from paper_2409_07563_b200 import controllers, plant, scenario
    return dict(B=bindings, C=controllers, P=plant, S=scenario)


LOOPS = sorted(glob.glob(os.path.join(GOLDEN, "loop_*.npz")))


@pytest.mark.parametrize("path", LOOPS, ids=[os.path.basename(p)[:-4] for p in LOOPS])
def test_device_loop_matches_reference_loop(mods, path):
    S = mods["S"]
    name = os.path.basename(path)[:-4]
    rec = dict(np.load(path))
    d = json.load(open(os.path.join(GOLDEN, "index.json")))["scenarios"][name]
    sc = S.Scenario(**{k: (tuple(v) if k == "control_std" else v) for k, v in d.items()})
    if sc.cost == "diff_drive_nav":
        sc.costmap = S.synthetic_costmap()
    steps = int(rec["steps"])
    ctl = mods["C"].make_controller(sc)
    r = mods["P"].run_control_loop(ctl, steps * sc.dt, log=True)
    ref = rec["rows"]
    n_x = sc.dims[0]
    print(name, "acc", r.accumulated_cost, rec["accumulated_cost"], "x rel", relerr(r.x, ref[:, 1:1 + n_x]))
    assert np.array_equal(r.t, ref[:, 0])
    assert close(r.x, ref[:, 1:1 + n_x]) and close(r.u, ref[:, 1 + n_x:-1]) and close(r.running_cost, ref[:, -1])
    assert close(r.accumulated_cost, rec["accumulated_cost"])
    assert r.solve_count == ctl.solve_count


def test_lockstep_loops_equal_single_loops(mods):
    """smpc_run_control_loops (the sweep's concurrent trials) == one loop at a time."""
    S, C, P = mods["S"], mods["C"], mods["P"]
    scs = []
    for seed in range(4):
        sc = S.default_sweep_scenario()
        sc.num_samples, sc.step_size, sc.rng_seed, sc.disturbance_std = 128, 0.8, seed, 0.2
        scs.append(sc)
    batch = P.run_control_loops([C.make_controller(sc) for sc in scs], 80 * 0.02)
    for sc, b in zip(scs, batch):
        single = P.run_control_loop(C.make_controller(sc), 80 * 0.02)
        assert single.accumulated_cost == b.accumulated_cost and single.solve_count == b.solve_count == 80


def test_device_loop_matches_checker_cartpole_replan(mods):
    """cartpole (glibc sinf/cosf path) at 25 Hz replanning with disturbance, vs
    the Python checker loop around the C oracle."""
    S = mods["S"]
    sc = S.cartpole_scenario(num_samples=512, horizon=40, seed=6)
    sc.replan_rate, sc.disturbance_std = 25.0, 0.1
    r = mods["P"].run_control_loop(mods["C"].make_controller(sc), 120 * sc.dt, log=True)
    acc, rows = mods["B"].control_loop(sc, 120 * sc.dt)
    assert close(r.x, rows[:, 1:5]) and close(r.accumulated_cost, acc)


def test_loop_errors(mods):
    S, C, P = mods["S"], mods["C"], mods["P"]
    sc = S.default_sweep_scenario()
    sc.num_samples = 16
    ctl = C.make_controller(sc)
    sc.replan_rate = 0.0
    with pytest.raises(C.SmpcError, match="^plant: replan_rate must be > 0$"):
        P.run_control_loop(ctl, 0.1)
    sc.replan_rate = 50.0
    with pytest.raises(C.SmpcError, match="^plant: loop duration must be > 0$"):
        P.run_control_loop(ctl, 0.0)


def test_small_dmd_sweep(mods):
    """bench_dmd_sweep on the device: records per (samples, gamma) cell, each
    the statistics of `trials` independent loops (checked against single runs)."""
    S, C, P = mods["S"], mods["C"], mods["P"]
    base = S.default_sweep_scenario()
    recs = P.bench_dmd_sweep(base, sample_counts=(64, 256), gammas=(0.5, 1.0), trials=3, steps=50, base_seed=0)
    assert [(r.samples, r.gamma) for r in recs] == [(64, 0.5), (64, 1.0), (256, 0.5), (256, 1.0)]
    import dataclasses
    costs = []
    for t in range(3):
        run = dataclasses.replace(base, num_samples=256, controller="dmd", step_size=1.0, rng_seed=t)
        costs.append(P.run_control_loop(C.make_controller(run), 50 * base.dt).accumulated_cost)
    assert abs(recs[3].mean_cost - float(np.mean(costs))) <= 1e-9 * max(1.0, abs(recs[3].mean_cost))
    assert len(P.best_gamma_per_samples(recs)) == 2
