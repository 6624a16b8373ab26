"""GPU: controllers on out-of-tree user models (include/smpc_b200_plugin.cuh,
tests/native/user_model.cu) — the device plugin API standing in for the
reference's DynamicsModel / CostFunction subclassing (dynamics.hpp:17-74,
costs.hpp:16-37).

* A double integrator + quadratic cost written in the plugin from the
  reference's equations gives solves bit-identical to the built-in pair.
* A new model (damped spring-mass with a control-dependent cost) rolls out
  bit-exactly against a numpy float32 / float64 restatement on injected
  noise, and its compute_control runs the whole MPPI iteration (update,
  nominal rollout, RMPPI, closed loop) through the plugin's launchers.
"""
import ctypes
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from test_plugin import load_user_model
    from paper_2409_07563_b200 import controllers, scenario
    return dict(C=controllers, S=scenario, P=load_user_model())


def test_user_double_integrator_equals_builtin(mods):
    C, S, P = mods["C"], mods["S"], mods["P"]
    target, weights = [1.0, -1.0, 0.0, 0.0], [1.0, 1.0, 0.1, 0.1]
    builtin = S.Scenario(num_samples=20000, horizon=60, dynamics="double_integrator", cost="quadratic",
                         target=target, weights=weights, rng_seed=3, control_std=(0.7, 0.4), lambda_=2.0,
                         zero_mean_fraction=0.1)
    plug = S.Scenario(**{**vars(builtin), "dynamics": "plugin", "plugin_dims": (4, 2, 4)})
    # the reference's QuadraticCost holds float parameters (make_cost's static_cast<float>)
    f = [float(np.float32(v)) for v in weights]
    ops = P.user_di_ops((ctypes.c_double * 4)(*target), (ctypes.c_double * 4)(*f))
    a, b = C.make_controller(builtin), C.make_controller(plug, ops=ops)
    x0 = builtin.x0()
    for _ in range(3):
        ra, rb = a.compute_control(x0, want_weights=True), b.compute_control(x0, want_weights=True)
        assert ra.weights.baseline == rb.weights.baseline and ra.weights.argmin == rb.weights.argmin
        assert np.array_equal(ra.controls, rb.controls)
        assert np.array_equal(ra.weights.weights, rb.weights.weights)
        assert np.array_equal(ra.states, rb.states)


def spring_reference(x0, mean, eps, dt, k, c, f_max):
    """numpy restatement of SpringMass + SpringCost (user_model.cu), the
    reference's run_sample_fused order (engine.cpp:211-239)."""
    f32 = np.float32
    M, T, _ = eps.shape
    J = np.zeros(M)
    for m in range(M):
        p, v = f32(x0[0]), f32(x0[1])
        total = 0.0
        for t in range(T):
            u = f32(mean[t, 0]) + f32(eps[m, t, 0])
            uc = min(max(u, f32(-f_max)), f32(f_max))
            dv = (uc - f32(k) * p - f32(c) * v) * f32(0.5)
            p, v = p + f32(dt) * v, v + f32(dt) * dv
            dp = float(p) - 1.0
            # the cost sees the clamped sampled control (sampled_control, engine.cpp:40-48)
            total += dp * dp + 0.1 * (float(v) * float(v)) + 0.01 * (float(uc) * float(uc))
        dp = float(p) - 1.0
        J[m] = total + 10.0 * (dp * dp)
    return J


def test_spring_mass_rollout_matches_numpy(mods):
    C, S, P = mods["C"], mods["S"], mods["P"]
    sc = S.Scenario(num_samples=300, horizon=40, dynamics="plugin", plugin_dims=(2, 1, 2), control_std=(1.0,),
                    rng_seed=5, importance_sampling=False, initial_state={"X0": -0.5})
    eng = C.RolloutEngine(sc, ops=P.spring_ops(2.0, 0.5, 3.0))
    rng = np.random.default_rng(0)
    eps = (rng.standard_normal((300, 40, 1)) * 1.5).astype(np.float32)
    mean = (rng.standard_normal((40, 1)) * 0.3).astype(np.float32)
    costs = eng.rollout(sc.x0()[None], mean[None], eps=eps)[0]
    ref = spring_reference(sc.x0(), mean, eps, sc.dt, 2.0, 0.5, 3.0)
    assert np.array_equal(costs.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("controller", ["mppi", "tube", "rmppi"])
def test_spring_mass_controllers_run_on_plugin(mods, controller):
    C, S, P = mods["C"], mods["S"], mods["P"]
    sc = S.Scenario(num_samples=4096, horizon=50, dynamics="plugin", plugin_dims=(2, 1, 2), control_std=(1.0,),
                    rng_seed=5, controller=controller, initial_state={"X0": -0.5})
    if controller == "rmppi":
        sc.feedback_gain, sc.cost_threshold = [[-1.0, -0.5]], 1e9
    ctl = C.make_controller(sc, ops=P.spring_ops(2.0, 0.5, 3.0))
    x = sc.x0()
    for _ in range(5):
        r = ctl.tube_compute_control(x).nominal if controller != "mppi" else ctl.compute_control(x)
        assert np.all(np.isfinite(r.controls)) and np.all(np.isfinite(r.states))
    # the plan drives p from -0.5 towards the cost's target 1
    assert r.states[-1, 0] > x[0] + 0.1


def test_spring_mass_closed_loop_on_plugin(mods):
    C, S, P = mods["C"], mods["S"], mods["P"]
    from paper_2409_07563_b200 import plant
    sc = S.Scenario(num_samples=2048, horizon=40, dynamics="plugin", plugin_dims=(2, 1, 2), control_std=(1.0,),
                    rng_seed=9, initial_state={"X0": -0.5})
    ctl = C.make_controller(sc, ops=P.spring_ops(2.0, 0.5, 3.0))
    res = plant.run_control_loop(ctl, duration_s=1.0, log=True)
    assert np.isfinite(res.accumulated_cost) and res.solve_count == 50
    assert abs(res.x[-1, 0] - 1.0) < abs(res.x[0, 0] - 1.0)  # the loop drives p towards the target
