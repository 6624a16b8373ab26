"""The reference's own acceptance criteria (tests/acceptance_main.cpp), run
on the device path. Each test cites the check it mirrors; thresholds are the
reference's.
"""
import dataclasses
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods(oracle_built):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import bindings
    from paper_2409_07563_b200 import controllers, plant, scenario
    return dict(B=bindings, C=controllers, P=plant, S=scenario)


def test_weight_transform_oracle(mods):
    """check_weight_transform_oracle (acceptance_main.cpp:49-100): softmin
    weights vs a long-double reference, per-weight error <= 1e-6, sums within
    1e-5 of one, across random cost vectors."""
    eng = mods["C"].RolloutEngine(mods["S"].cartpole_scenario(num_samples=16, horizon=4))
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(1, 5000))
        lam = float(rng.uniform(0.01, 100.0))
        costs = rng.uniform(0, float(rng.choice([1.0, 100.0, 1e4])), n) + float(rng.uniform(0, 1e6))
        r = eng.compute_weights(costs, lam)
        c = costs.astype(np.longdouble)
        e = np.exp(-(c - c.min()) / np.longdouble(lam))
        w = e / e.sum()
        assert np.max(np.abs(r.weights.astype(np.longdouble) - w)) <= 1e-6
        assert abs(r.weights.sum() - 1.0) <= 1e-5


def test_baseline_invariance(mods):
    """check_baseline_invariance (:380-433): adding a large constant to every
    cost leaves the weights unchanged to tight absolute tolerance."""
    eng = mods["C"].RolloutEngine(mods["S"].cartpole_scenario(num_samples=16, horizon=4))
    rng = np.random.default_rng(3)
    costs = rng.uniform(0, 20, 4096)
    a = eng.compute_weights(costs, 1.0)
    b = eng.compute_weights(costs + 1e6, 1.0)
    assert np.max(np.abs(a.weights - b.weights)) <= 1e-6 and a.argmin == b.argmin


def test_tube_nominal_insulation(mods):
    """check_tube_nominal_insulation (:435-484): with zero feedback gains the
    nominal line of the tube controller is bit-identical whether or not the
    executing system is disturbed (50 steps, shifting the sequence)."""
    S, C, B = mods["S"], mods["C"], mods["B"]
    O = B.Oracle("port")

    def run(disturbance_std):
        sc = S.Scenario(num_samples=256, horizon=16, dt=0.02, control_std=(1.0, 1.0), rng_seed=3,
                        dynamics="double_integrator", cost="circle_track", controller="tube",
                        initial_state={"X": 2.0, "V_Y": 2.0})
        tube = C.make_controller(sc)
        x = sc.x0()
        sim_seed = 11
        states, controls = [], []
        for step in range(50):
            sol = tube.tube_compute_control(x)
            states.append(sol.nominal_state.copy())
            controls.append(sol.nominal.controls[0].copy())
            u = sol.nominal.controls[0]  # zero gains: applied = nominal u0
            xn, _ = O.step(sc, x, u, np.float32(0.02))
            if disturbance_std > 0:  # SimulatedSystem::step disturbance (plant.cpp:36-43)
                scale = np.float32(disturbance_std * math.sqrt(0.02))
                z = O.quad(sim_seed, step, 0, 0)
                xn = (xn + scale * z[:4]).astype(np.float32)
            x = xn
            tube.shift_control_sequence(0.02, 0.02)
        return np.array(states), np.array(controls)

    ds, dc = run(0.1)
    cs, cc = run(0.0)
    assert np.array_equal(ds, cs) and np.array_equal(dc, cc)


def test_sampler_statistics(mods):
    """check_sampler_statistics (:541-613): device noise passes a KS test
    against N(0, 0.2) at the 1% level; the zero-mean quota is exactly
    ceil(f M) (capped at M-1 with the mean sample) filled from the tail."""
    S, C = mods["S"], mods["C"]
    sc = S.Scenario(num_samples=4000, horizon=25, dynamics="cartpole", cost="road", control_std=(0.2,),
                    include_mean_sample=False, rng_seed=2024)
    mean = (0.01 * np.arange(25, dtype=np.float32)).reshape(25, 1)
    eps, _ = C.GaussianSampler(sc).generate_samples(mean, 0)
    pooled = np.sort(eps.ravel().astype(np.float64))
    n = pooled.size
    f = 0.5 * (1.0 + np.array([math.erf(v / (0.2 * math.sqrt(2.0))) for v in pooled]))
    i = np.arange(n)
    d = max(np.max(f - i / n), np.max((i + 1) / n - f))
    assert d < 1.62762 / math.sqrt(n)
    for frac, with_mean, M, expected in [(0.3, True, 10, 3), (0.25, False, 16, 4), (1.0, True, 10, 9),
                                          (1.0, False, 10, 10)]:
        q = S.Scenario(num_samples=M, horizon=4, dynamics="cartpole", cost="road", control_std=(0.2,),
                       zero_mean_fraction=frac, include_mean_sample=with_mean)
        _, flags = C.GaussianSampler(q).generate_samples(np.zeros((4, 1), np.float32), 0)
        zero = (flags & 2) != 0
        assert zero.sum() == expected and not zero[:M - expected].any()


def test_closed_loop_improvement(mods):
    """check_closed_loop_improvement (:341-378): the mean accumulated cost of
    20 seeded 500-step closed loops (device) is below the zero-control cost."""
    S, C, P, B = mods["S"], mods["C"], mods["P"], mods["B"]
    base = S.default_sweep_scenario()
    base.controller, base.num_samples = "mppi", 1024
    O = B.Oracle("port")
    x = base.x0()
    zero_cost = 0.0
    for t in range(500):
        zero_cost += O.running_cost(base, x)
        x, _ = O.step(base, x, np.zeros(2, np.float32), np.float32(base.dt))
    ctls = [C.make_controller(dataclasses.replace(base, rng_seed=s)) for s in range(20)]
    res = P.run_control_loops(ctls, 500 * base.dt)
    mean_cost = float(np.mean([r.accumulated_cost for r in res]))
    print("mean closed-loop cost", mean_cost, "vs zero-control", zero_cost)
    assert mean_cost < zero_cost


def test_fused_timing_scaling(mods):
    """check_fused_timing_scaling (:313-339): solve time grows sublinearly from
    128 to 1024 samples and within 1.3x of linear from 4096 to 16384."""
    import time
    S, C = mods["S"], mods["C"]

    def solve_ms(n):
        sc = S.diff_drive_nav_scenario(num_samples=n, horizon=56, seed=1)
        ctl = C.make_controller(sc)
        x0 = sc.x0()
        for _ in range(3):
            ctl.compute_control(x0)
        t0 = time.perf_counter()
        for _ in range(30):
            ctl.compute_control(x0)
        return (time.perf_counter() - t0) / 30

    t = {n: solve_ms(n) for n in (128, 1024, 4096, 16384)}
    assert t[1024] / t[128] < 8.0 and t[16384] / t[4096] <= 4.0 * 1.3
