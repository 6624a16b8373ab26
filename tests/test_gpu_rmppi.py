"""GPU parity for the builder-defined RMPPI controller (
no reference implementation — the oracle twin is
oracle/smpc_oracle.c:oracle_rmppi_compute_control): ancillary feedback
u_real = u + K (x_real - x_nominal) inside every sample, one control sequence
updated from the real system's weights, and the nominal state chosen on the
segment previous-nominal -> real under the cost threshold.

Bars: the candidate choice and the chosen nominal state are exact, the
baseline (min real cost) and argmin exact (the coupled rollout reproduces the
twin's IEEE op sequence), U* / states within the north-star 1e-4.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def close(a, b, tol=TOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))


@pytest.fixture(scope="module")
def mods(oracle_built):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.bindings import OracleController
    from paper_2409_07563_b200 import controllers, scenario
    return dict(OracleController=OracleController, C=controllers, S=scenario)


def rmppi_scenarios(S):
    di = S.di_swarm_scenario(num_samples=4096, horizon=50, seed=7)
    di.controller = "rmppi"
    di.feedback_gain = [[-2.0, 0.0, -1.0, 0.0], [0.0, -2.0, 0.0, -1.0]]
    di.cost_threshold = 12000.0
    cp = S.cartpole_scenario(num_samples=2048, horizon=60, seed=3)
    cp.controller = "rmppi"
    cp.feedback_gain = [[0.5, 0.3, 3.0, 0.5]]
    cp.cost_threshold = 20000.0
    cp.num_candidates = 5
    nav = S.diff_drive_nav_scenario(num_samples=1000, horizon=40, seed=9)
    nav.controller = "rmppi"
    nav.feedback_gain = [[-0.5, -0.5, 0.0], [0.0, 0.0, -1.0]]
    nav.cost_threshold = 1e9
    return {"di_circle": di, "cartpole": cp, "diff_drive_nav": nav}


@pytest.mark.parametrize("name", ["di_circle", "cartpole", "diff_drive_nav"])
def test_rmppi_matches_oracle(mods, name):
    sc = rmppi_scenarios(mods["S"])[name]
    gpu = mods["C"].make_controller(sc)
    ref = mods["OracleController"](sc, "port")
    x = sc.x0()
    rng = np.random.default_rng(1)
    choices = []
    for solve in range(4):
        a = gpu.tube_compute_control(x)
        b = ref.rmppi_compute_control(x)
        choices.append(b["choice"])
        assert np.array_equal(a.nominal_state, b["nominal_state"]), solve
        assert a.real.weights.baseline == b["baseline"] and a.real.weights.argmin == b["argmin"], solve
        assert a.nominal.weights.baseline == b["baseline"]
        assert close(a.nominal.controls, b["controls"]), np.abs(a.nominal.controls - b["controls"]).max()
        assert np.array_equal(a.nominal.controls, a.real.controls)  # one control sequence
        assert close(a.nominal.states, b["nominal_states"]) and close(a.real.states, b["real_states"])
        gpu.set_mean(b["controls"])
        # the measured state drifts away from the nominal prediction
        x = (b["nominal_states"][1] + rng.standard_normal(x.size).astype(np.float32) * 0.05).astype(np.float32)
    print(name, "candidate choices", choices)


def test_rmppi_zero_gain_infinite_threshold_is_tube_like(mods):
    """K = 0 and alpha = inf: the nominal state is the real state every solve
    (largest candidate always admissible) and both systems see identical
    samples, so nominal and real costs coincide."""
    S = mods["S"]
    sc = S.cartpole_scenario(num_samples=512, horizon=30, seed=2)
    sc.controller = "rmppi"
    gpu = mods["C"].make_controller(sc)
    x = sc.x0()
    for _ in range(2):
        a = gpu.tube_compute_control(x)
        assert np.array_equal(a.nominal_state, x)
        assert a.nominal.weights.baseline == a.real.weights.baseline
        x = a.nominal.states[1] + np.float32(0.01)
