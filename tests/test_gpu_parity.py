"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bars (north_star): Philox noise, per-sample costs, rho and argmin bit-exact
(integer/byte-exact where the reference arithmetic is reproduced op for op);
weights, eta and the updated control sequence within FP32 relative 1e-4
(SURVEY.md Appendix C rule 6: |a-b| <= 1e-4 * max(1, |a|, |b|)) because the
device reduces sums in a tree instead of the reference's sequential order.
"""
import math

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
    from oracle.bindings import Oracle, OracleController
    from paper_2409_07563_b200 import controllers, scenario
    return dict(Oracle=Oracle, OracleController=OracleController, C=controllers, S=scenario)


def scenarios(S):
    sp = S.Scenario
    return {
        "cartpole": S.cartpole_scenario(num_samples=512, horizon=100, seed=1),
        "double_integrator": S.di_swarm_scenario(num_samples=1024, horizon=60, seed=7),
        "diff_drive_nav": S.diff_drive_nav_scenario(num_samples=500, horizon=56, seed=42),
        "unicycle_road": sp(num_samples=300, horizon=40, dynamics="unicycle", cost="road", rng_seed=11,
                            control_std=(0.5, 0.3), zero_mean_fraction=0.25),
        "cartpole_road_perstep": sp(num_samples=256, horizon=30, dynamics="cartpole", cost="road", rng_seed=5,
                                    control_std=(1.0,), std_per_step=[[0.5 + 0.02 * t] for t in range(30)],
                                    zero_mean_fraction=0.1, include_mean_sample=False),
        "di_quadratic_dmd": sp(num_samples=384, horizon=25, dynamics="double_integrator", cost="quadratic",
                               target=[1.0, -1.0, 0.0, 0.0], weights=[1.0, 1.0, 0.1, 0.1], rng_seed=3,
                               control_std=(0.7, 0.4), controller="dmd", step_size=0.6, lambda_=2.0),
        # BASELINE.json configs[1]: builder-defined 13-state quadrotor (restated oracle only)
        "quadrotor": S.quadrotor_scenario(num_samples=1024, horizon=100, seed=13),
        # BASELINE.json configs[2]: builder-defined kinematic bicycle on the synthetic costmap
        "bicycle_nav": S.bicycle_nav_scenario(num_samples=2000, horizon=56, seed=42),
    }


def test_tail_table_and_icdf_exhaustive(mods):
    """Every one of the 2^23 uniforms the sampler can produce maps to the
    reference's Phi^-1 value bit for bit (noise generated on the device)."""
    O = mods["Oracle"]("port")
    ref = O.icdf_domain()
    S = mods["S"]
    # One sample, T*n_u = 2^23 would be too long; instead draw many samples and
    # compare the device sampler with the oracle sampler (same Philox words).
    sc = S.Scenario(num_samples=4096, horizon=64, dynamics="cartpole", cost="road", control_std=(1.0,),
                    rng_seed=123, include_mean_sample=False)
    gs = mods["C"].GaussianSampler(sc)
    mean = np.zeros((64, 1), np.float32)
    eps_d, _ = gs.generate_samples(mean, 9)
    eps_o, _ = O.generate_samples(sc, mean, 9)
    assert np.array_equal(eps_d.view(np.uint32), eps_o.view(np.uint32))
    # every produced value is one of the domain values
    assert np.isin(eps_d.ravel(), ref).all()


def test_icdf_whole_domain_bit_exact(mods):
    """normal_icdf(to_open_unit(w)) on the device — packed Acklam central
    branch, packed Markstein division, tail table — equals the reference for
    ALL 2^23 possible uniforms."""
    ref = mods["Oracle"]("port").icdf_domain()
    eng = mods["C"].RolloutEngine(mods["S"].cartpole_scenario(num_samples=16, horizon=4))
    out = np.zeros(1 << 23, np.float32)
    eng._check(eng.lib.smpc_icdf_domain(eng.ctx, out))
    bad = np.nonzero(out.view(np.uint32) != ref.view(np.uint32))[0]
    assert bad.size == 0, (bad[:10], out[bad[:10]], ref[bad[:10]])


def test_full_domain_icdf_table_bit_exact(mods):
    """The resident full-domain normal_icdf table the steady-state rollout
    reads for part of its draws equals the in-register evaluation (and so the
    oracle) on all 2^23 uniforms."""
    O = mods["Oracle"]("port")
    ref = O.icdf_domain()
    eng = mods["C"].RolloutEngine(mods["S"].cartpole_scenario(num_samples=16, horizon=4))
    out = np.zeros(1 << 23, np.float32)
    eng._check(eng.lib.smpc_icdf_table(eng.ctx, out))
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))


def test_branch_free_sqrt_exhaustive(mods):
    """The cost / dynamics functors' branch-free sqrt (std::sqrt of
    costs.cpp:59, the quaternion norm) equals sqrt.rn.f32 on all 2^32 floats."""
    import ctypes
    from paper_2409_07563_b200 import _lib
    n = ctypes.c_uint64(123)
    assert _lib.load().smpc_sqrt_check(0, ctypes.byref(n)) == 0
    assert n.value == 0, n.value


@pytest.mark.parametrize("name", ["cartpole", "double_integrator", "diff_drive_nav", "unicycle_road",
                                  "cartpole_road_perstep", "di_quadratic_dmd", "quadrotor", "bicycle_nav"])
def test_generate_samples_bit_exact(mods, name):
    sc = scenarios(mods["S"])[name]
    n_x, n_u, n_y = sc.dims
    mean = (np.sin(np.arange(sc.horizon * n_u, dtype=np.float32)) * 0.3).reshape(sc.horizon, n_u)
    gs = mods["C"].GaussianSampler(sc)
    eps_d, flags_d = gs.generate_samples(mean, 77)
    eps_o, flags_o = mods["Oracle"]("port").generate_samples(sc, mean, 77)
    assert np.array_equal(flags_d, flags_o)
    assert np.array_equal(eps_d.view(np.uint32), eps_o.view(np.uint32))


@pytest.mark.parametrize("name", ["cartpole", "double_integrator", "diff_drive_nav", "unicycle_road",
                                  "cartpole_road_perstep", "di_quadratic_dmd", "quadrotor", "bicycle_nav"])
@pytest.mark.parametrize("systems", [1, 2])
def test_rollout_costs_bit_exact(mods, name, systems):
    """Fused rollout (Philox regenerated in-kernel and injected noise) vs oracle:
    per-sample costs and stored trajectories bit-identical."""
    sc = scenarios(mods["S"])[name]
    n_x, n_u, n_y = sc.dims
    T = sc.horizon
    rng = np.random.default_rng(0)
    means = (rng.standard_normal((systems, T, n_u)) * 0.2).astype(np.float32)
    x0s = np.stack([sc.x0() + 0.05 * s for s in range(systems)]).astype(np.float32)
    eng = mods["C"].RolloutEngine(sc)
    O = mods["Oracle"]("port")
    eps, _ = O.generate_samples(sc, means[0], 31)
    c_ref, o_ref = O.rollout(sc, x0s, means, eps, outputs=True)
    c_inj, o_inj = eng.rollout(x0s, means, eps=eps, outputs=True)
    c_gen, o_gen = eng.rollout(x0s, means, stream=31, outputs=True)
    assert np.array_equal(c_inj.view(np.uint64), c_ref.view(np.uint64))
    assert np.array_equal(c_gen.view(np.uint64), c_ref.view(np.uint64))
    assert np.array_equal(o_inj.view(np.uint32), o_ref.view(np.uint32))
    assert np.array_equal(o_gen.view(np.uint32), o_ref.view(np.uint32))


@pytest.mark.parametrize("name", ["cartpole", "double_integrator", "diff_drive_nav", "unicycle_road",
                                  "cartpole_road_perstep", "di_quadratic_dmd", "quadrotor", "bicycle_nav",
                                  "di_circle_at_rest"])
@pytest.mark.parametrize("systems", [1, 2])
def test_rollout_costs_fast_path_bit_exact(mods, name, systems):
    """The unchecked fast loop (no stored outputs: sticky flags, fast sqrt,
    branch-free two-quad steady state) gives the oracle's costs bit for bit.
    di_circle_at_rest: zero velocity and zero mean, so the mean sample's
    speed is exactly 0 every step (sqrt edge case -> exact replay)."""
    S = mods["S"]
    if name == "di_circle_at_rest":
        sc = S.Scenario(num_samples=777, horizon=50, dt=0.02, lambda_=1.0, control_std=(1.0, 1.0), rng_seed=5,
                        importance_sampling=False, dynamics="double_integrator", cost="circle_track",
                        initial_state={"X": 2.0})
    else:
        sc = scenarios(S)[name]
    n_x, n_u, n_y = sc.dims
    T = sc.horizon
    rng = np.random.default_rng(2)
    means = (rng.standard_normal((systems, T, n_u)) * 0.2).astype(np.float32)
    if name == "di_circle_at_rest":
        means[:] = 0.0
    x0s = np.stack([sc.x0() + (0.05 * s if name != "di_circle_at_rest" else 0.0) for s in range(systems)])
    x0s = x0s.astype(np.float32)
    eng = mods["C"].RolloutEngine(sc)
    O = mods["Oracle"]("port")
    eps, _ = O.generate_samples(sc, means[0], 17)
    c_ref, _ = O.rollout(sc, x0s, means, eps, outputs=True)
    c_gen = eng.rollout(x0s, means, stream=17)
    assert np.array_equal(c_gen.view(np.uint64), c_ref.view(np.uint64))


def test_compute_weights_matches_oracle(mods):
    rng = np.random.default_rng(1)
    eng = mods["C"].RolloutEngine(mods["S"].cartpole_scenario(num_samples=64, horizon=10))
    O = mods["Oracle"]("port")
    for n, lam, spread in [(1, 1.0, 1.0), (7, 0.5, 3.0), (4096, 1.0, 5.0), (100000, 10.0, 100.0), (3, 1.0, 1e6)]:
        costs = rng.uniform(0, spread, n) + 1e3
        costs[n // 2] = costs.min()  # a tie: lowest index must win
        w, rho, eta, am = O.compute_weights(costs, lam)
        r = eng.compute_weights(costs, lam)
        assert r.baseline == rho and r.argmin == am
        assert close(r.normalizer, eta, 1e-12)
        assert close(r.weights, w, 1e-12)
    # frozen reference value: J = [1, 3, 2], lambda = 1 (test_engine.cpp:187-197)
    r = eng.compute_weights(np.array([1.0, 3.0, 2.0]), 1.0)
    e = np.exp(-np.array([0.0, 2.0, 1.0]))
    assert np.allclose(r.weights, e / e.sum(), rtol=0, atol=1e-15)


@pytest.mark.parametrize("name", ["cartpole", "double_integrator", "diff_drive_nav", "unicycle_road",
                                  "cartpole_road_perstep", "di_quadratic_dmd", "quadrotor", "bicycle_nav"])
def test_compute_control_matches_oracle(mods, name):
    """Three warm-started solves: rho and argmin exact, U*/states/weights within 1e-4."""
    sc = scenarios(mods["S"])[name]
    gpu = mods["C"].make_controller(sc)
    ref = mods["OracleController"](sc, "port")
    x0 = sc.x0()
    for solve in range(3):
        a = gpu.compute_control(x0, want_weights=True)
        b = ref.compute_control(x0, want_weights=True)
        assert a.weights.baseline == b["baseline"], (solve, a.weights.baseline, b["baseline"])
        assert a.weights.argmin == b["argmin"], (solve, a.weights.argmin, b["argmin"])
        assert close(a.weights.normalizer, b["normalizer"])
        assert close(a.weights.weights, b["weights"])
        assert close(a.controls, b["controls"]), np.abs(a.controls - b["controls"]).max()
        assert close(a.states, b["states"])
        assert close(a.outputs, b["outputs"])
        # keep both controllers on the identical warm start so errors do not compound
        gpu.set_mean(b["controls"])
    assert gpu.solve_count == 3


def test_tube_matches_oracle(mods):
    S = mods["S"]
    sc = S.cartpole_scenario(num_samples=512, horizon=50, seed=4)
    sc.controller = "tube"
    gpu = mods["C"].make_controller(sc)
    ref = mods["OracleController"](sc, "port")
    x = sc.x0()
    for k in range(3):
        a = gpu.tube_compute_control(x)
        b = ref.tube_compute_control(x)
        for side, bb in (("nominal", b["nominal"]), ("real", b["real"])):
            aa = getattr(a, side)
            assert aa.weights.baseline == bb["baseline"] and aa.weights.argmin == bb["argmin"], side
        assert close(a.nominal.controls, b["nominal_controls"])
        assert close(a.real.controls, b["real_controls"])
        assert np.array_equal(a.nominal_state, b["nominal_state"])
        gpu.set_mean(b["nominal_controls"], 0)
        gpu.set_mean(b["real_controls"], 1)
        x = x + np.float32(0.01)  # the measured state drifts from the nominal


def test_step_size_one_is_plain_mppi(mods):
    """gamma = 1 (dmd) is bit-identical to mppi (test_controllers.cpp:46-66)."""
    S = mods["S"]
    a_sc = S.di_swarm_scenario(num_samples=2048, horizon=40, seed=9)
    b_sc = S.di_swarm_scenario(num_samples=2048, horizon=40, seed=9)
    b_sc.controller, b_sc.step_size = "dmd", 1.0
    a, b = mods["C"].make_controller(a_sc), mods["C"].make_controller(b_sc)
    for _ in range(3):
        ra, rb = a.compute_control(a_sc.x0()), b.compute_control(b_sc.x0())
        assert np.array_equal(ra.controls, rb.controls)


def test_non_finite_state_error_message(mods):
    """engine.cpp:51-57: the first non-finite state names channel/sample/timestep."""
    S = mods["S"]
    sc = S.Scenario(num_samples=64, horizon=20, dynamics="double_integrator", cost="road", control_std=(1.0, 1.0))
    eng = mods["C"].RolloutEngine(sc)
    eps = np.zeros((64, 20, 2), np.float32)
    eps[5, 3, 1] = np.inf
    eps[9, 1, 0] = np.inf
    with pytest.raises(mods["C"].SmpcError) as ei:
        eng.rollout(sc.x0()[None], np.zeros((1, 20, 2), np.float32), eps=eps)
    O = mods["Oracle"]("port")
    with pytest.raises(Exception) as eo:
        O.rollout(sc, sc.x0()[None], np.zeros((1, 20, 2), np.float32), eps)
    assert str(ei.value) == str(eo.value) == "rollout produced non-finite state channel 3 at sample 5 timestep 3"


def test_invalid_config_messages(mods):
    S, C = mods["S"], mods["C"]
    with pytest.raises(C.SmpcError, match="^mppi: lambda must be > 0$"):
        C.make_controller(S.Scenario(num_samples=16, horizon=5, dynamics="cartpole", cost="road",
                                     control_std=(1.0,), lambda_=0.0))
    with pytest.raises(C.SmpcConfigError, match="expects 4 output channels"):
        C.make_controller(S.Scenario(num_samples=16, horizon=5, dynamics="unicycle", cost="circle_track"))


@pytest.mark.parametrize("M", [1, 2, 127, 129, 4097])
def test_ragged_sample_counts(mods, M):
    sc = mods["S"].cartpole_scenario(num_samples=M, horizon=12, seed=2)
    sc.zero_mean_fraction = 0.5
    gpu = mods["C"].make_controller(sc)
    ref = mods["OracleController"](sc, "port")
    a = gpu.compute_control(sc.x0(), True)
    b = ref.compute_control(sc.x0(), True)
    assert a.weights.baseline == b["baseline"] and a.weights.argmin == b["argmin"]
    assert close(a.controls, b["controls"])


def test_full_size_di_swarm_properties(mods):
    """BASELINE C5 at full size (N = 2^20, T = 100): costs of a strided subset
    bit-exact vs the oracle rolled out on the same samples; argmin consistent
    with the full cost vector; weights sum to 1; U* = mean + gamma * sum w eps
    reproduced from the oracle's own eps for the non-zero-weight samples."""
    S, C = mods["S"], mods["C"]
    sc = S.di_swarm_scenario(num_samples=1 << 20, horizon=100, seed=7)
    gpu = C.make_controller(sc)
    x0 = sc.x0()
    sol = gpu.compute_control(x0, want_weights=True)
    w = sol.weights.weights
    assert abs(w.sum() - 1.0) < 1e-9
    assert sol.weights.argmin == int(np.argmax(w))
    # costs: regenerate the same Philox batch (stream 0) on the device
    eng = C.RolloutEngine(sc)
    costs = eng.rollout(x0[None], np.zeros((1, 100, 2), np.float32), stream=0)[0]
    assert costs.min() == sol.weights.baseline and int(np.argmin(costs)) == sol.weights.argmin
    O = mods["Oracle"]("port")
    idx = np.arange(0, 1 << 20, 4099)
    sub = S.di_swarm_scenario(num_samples=1 << 20, horizon=100, seed=7)
    for m in list(idx[:64]) + [sol.weights.argmin]:
        e, _ = O.generate_samples(sub, np.zeros((100, 2), np.float32), 0, m_begin=int(m), m_end=int(m) + 1)
        c = O.rollout(sub, x0[None], np.zeros((1, 100, 2), np.float32), e)[0, 0]
        assert c == costs[m], m
    nz = np.nonzero(w)[0]
    acc = np.zeros((100, 2), np.float64)
    for m in nz:
        e, _ = O.generate_samples(sub, np.zeros((100, 2), np.float32), 0, m_begin=int(m), m_end=int(m) + 1)
        acc += w[m] * e[0].astype(np.float64)
    assert close(sol.controls, acc.astype(np.float32))


@pytest.mark.parametrize("mode", ["single", "exact"])
@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("name", ["cartpole", "double_integrator", "unicycle_road"])
def test_shard_group_matches_single(mods, name, n, mode):
    """World > 1 device path (gathers + rank-ordered combine) on one GPU, in
    both exchange modes (one all-gathered record per iteration with the
    rescaled combine, or the three exact collectives): rho/argmin exact, U*
    within tolerance, every rank bitwise identical."""
    sc = scenarios(mods["S"])[name]
    grp = mods["C"].ShardGroup(sc, n, mode=mode)
    ref = mods["OracleController"](sc, "port")
    x0 = sc.x0()
    for solve in range(2):
        sols = grp.compute_control(x0)
        b = ref.compute_control(x0)
        for s in sols[1:]:
            assert np.array_equal(s.controls, sols[0].controls)
            assert np.array_equal(s.states, sols[0].states)
        a = sols[0]
        assert a.weights.baseline == b["baseline"] and a.weights.argmin == b["argmin"]
        assert close(a.weights.normalizer, b["normalizer"])
        assert close(a.controls, b["controls"])
        assert close(a.states, b["states"])
        for m in grp.members:
            m.set_mean(b["controls"])


@pytest.mark.parametrize("name", ["cartpole", "double_integrator", "quadrotor"])
def test_noise_strategies_bit_identical(mods, name):
    """split (materialised normals) and fused (in-register) noise give the
    same solves bit for bit (the reference's split == fused contract,
    test_engine.cpp:86-99); auto times both and follows the decision rule."""
    from paper_2409_07563_b200 import _lib
    sc = scenarios(mods["S"])[name]
    a = mods["C"].make_controller(sc)
    b = mods["C"].make_controller(sc)
    assert a.select_noise_strategy("split")["kind"] == "split"
    assert b.select_noise_strategy("fused")["kind"] == "fused"
    x = sc.x0()
    for _ in range(3):
        sa, sb = a.compute_control(x), b.compute_control(x)
        assert sa.weights.baseline == sb.weights.baseline and sa.weights.argmin == sb.weights.argmin
        assert np.array_equal(sa.controls.view(np.uint32), sb.controls.view(np.uint32))
        assert np.array_equal(sa.states.view(np.uint32), sb.states.view(np.uint32))
    ch = a.select_noise_strategy("auto", trials=3)
    assert ch["timed"] and ch["split_median_ms"] > 0 and ch["fused_median_ms"] > 0
    rule = _lib.load().smpc_noise_strategy_rule(0.0, 1.0, ch["split_median_ms"], ch["fused_median_ms"])
    assert ch["kind"] == {_lib.NOISE_SPLIT: "split", _lib.NOISE_FUSED: "fused"}[rule]
    # auto must not disturb the controller: the next solve continues the sequence
    sa, sb = a.compute_control(x), b.compute_control(x)
    assert np.array_equal(sa.controls.view(np.uint32), sb.controls.view(np.uint32))
    # over the scratch budget -> fused without timing
    ch = a.select_noise_strategy("auto", split_budget_bytes=0.0)
    assert ch["kind"] == "fused" and not ch["timed"]
    a.close()
    b.close()
