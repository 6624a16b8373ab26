"""Regression tests for defects found in review."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods(oracle_built):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.bindings import Oracle
    from paper_2409_07563_b200 import controllers, scenario, _lib
    return dict(Oracle=Oracle, C=controllers, S=scenario, L=_lib)


def test_compute_weights_on_cem_context_is_softmin(mods):
    """RolloutEngine::compute_weights (engine.cpp:342-363) is the softmin even
    when called on a CEM controller: w = e/eta, not e/k."""
    S, C = mods["S"], mods["C"]
    sc = S.cartpole_scenario(num_samples=300, horizon=20, seed=2)
    sc.controller, sc.elite_fraction = "cem", 0.1
    ctl = C.make_controller(sc)
    costs = np.random.default_rng(3).uniform(0, 4, 1000) + 10.0
    w, rho, eta, am = mods["Oracle"]("port").compute_weights(costs, 1.5)
    r = ctl.compute_weights(costs, 1.5)
    assert r.baseline == rho and r.argmin == am
    assert np.allclose(r.weights, w, rtol=1e-12, atol=0)
    assert abs(r.weights.sum() - 1.0) < 1e-12


@pytest.mark.parametrize("kind", ["tube", "rmppi"])
def test_group_rejects_tube_and_rmppi(mods, kind):
    S, C = mods["S"], mods["C"]
    sc = S.cartpole_scenario(num_samples=256, horizon=20, seed=2)
    sc.controller = kind
    with pytest.raises(mods["L"].SmpcError, match="not supported by the in-process group"):
        C.ShardGroup(sc, 2)


def test_shift_is_ordered_after_a_launched_iteration(mods):
    """smpc_shift_control_sequence runs on the context stream, so it sees the
    mean written by a graph launched with smpc_launch_iteration (no explicit
    synchronize in between)."""
    S, C = mods["S"], mods["C"]
    sc = S.di_swarm_scenario(num_samples=1 << 18, horizon=100, seed=7)
    a, b = C.make_controller(sc), C.make_controller(sc)
    x0 = sc.x0()
    a.compute_control(x0)
    want = np.concatenate([a.mean()[3:], np.repeat(a.mean()[-1:], 3, axis=0)])
    b.set_x0(x0)
    b.launch_iteration()
    b.shift_control_sequence(3 * sc.dt, sc.dt)
    assert np.array_equal(b.mean(), want)


def test_first_solve_after_create_sees_initialised_state(mods):
    """Creation-time uploads (result header with its no-error key, sigma,
    gamma, costmap, model tensors) are ordered on the context's non-blocking
    stream and complete before the first solve: a pageable cudaMemcpy could
    return before its DMA landed, and a solve launched right away read the
    zeroed header as error key 0 ("non-finite state channel 0 at sample 0
    timestep 0"; seen once in a bench sweep). Contexts are created and solved
    back to back, with the previous context's memory freed just before."""
    S, C = mods["S"], mods["C"]
    builders = [lambda: S.cartpole_scenario(num_samples=2048, horizon=100, seed=1),
                lambda: S.di_swarm_scenario(num_samples=65536, horizon=100, seed=7)]
    for k in range(40):
        sc = builders[k % 2]()
        ctl = C.make_controller(sc)
        ctl.set_x0(sc.x0())
        ctl.launch_iteration()
        ctl.synchronize()  # raises on a spurious error key
        ctl.close()
