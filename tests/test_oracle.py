"""CPU: pin the oracle restatement before trusting it.

* Random123 Philox4x32-10 known-answer vectors (published KATs).
* Reference-derived normals and iteration-level goldens quoted in SURVEY.md §8(c).
* Frozen values from the reference's own unit tests (test_costs.cpp,
  test_engine.cpp).
* Every committed golden fixture (tests/golden/*.npz, generated from the
  unmodified reference by oracle/gen_golden.py): noise, costs, trajectories,
  weights and three warm-started compute_control solves, bit for bit.
* When oracle/_ref exists here, a randomized cross-check port vs reference.
"""
import glob
import json
import math
import os

import numpy as np
import pytest

from paper_2409_07563_b200 import scenario as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def port(oracle_built):
    return oracle_built.Oracle("port")


def test_philox_random123_kats(port):
    kats = [
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ]
    for ctr, key, want in kats:
        assert list(port.philox(ctr, key)) == want


def test_reference_normals(port):
    """NormalStream(0).quad(0, m, 0) values quoted from the reference."""
    want = {
        0: ["-0x1.05f49ep-2", "0x1.2d7676p+0", "0x1.42a772p-1", "0x1.11fbcep-2"],
        1: ["-0x1.abe806p-3", "0x1.5ea166p+0", "-0x1.f0d8d4p-4", "-0x1.e75df8p+0"],
        4: ["-0x1.0bca66p-1", "-0x1.266446p-1", "-0x1.a0b29ap+0", "0x1.33b902p+1"],  # lane 3: tail draw
    }
    for m, hx in want.items():
        got = port.quad(0, 0, m, 0)
        assert [float(v) for v in got] == [float.fromhex(h) for h in hx]
    got = port.quad(42, 0, 1, 0)
    assert np.allclose(got, [-0.639522672, -0.0220570546, -0.88855195, -0.210258484], rtol=0, atol=5e-9)


def test_golden_kats_file(port):
    with open(os.path.join(GOLDEN, "index.json")) as f:
        kat = json.load(f)["kat"]
    for ctr, key, want in kat["philox"]:
        assert [int(v) for v in port.philox(ctr, key)] == want
    for seed, a, b, c, hx in kat["quad"]:
        assert [float(v) for v in port.quad(seed, a, b, c)] == [float.fromhex(h) for h in hx]


def test_iteration_goldens_from_survey(oracle_built):
    """SURVEY §8(c) iteration-level goldens measured on the reference (8 workers)."""
    C = oracle_built.OracleController
    sc = S.cartpole_scenario(num_samples=2048, horizon=100, seed=1)
    r = C(sc, "port").compute_control(sc.x0(), want_weights=True)
    assert r["baseline"] == 9834.4165807109839
    assert r["normalizer"] == 1.247186023295634
    assert int(np.argmax(r["weights"])) == 1900
    assert float(r["controls"][0, 0]) == float.fromhex("-0x1.08bac6p-1")
    sc = S.di_swarm_scenario(num_samples=8192, horizon=100, seed=7)
    r = C(sc, "port").compute_control(sc.x0())
    assert r["baseline"] == 76047.396015882492
    assert r["normalizer"] == 1.0 and r["argmin"] == 5221
    assert float(r["controls"][0, 0]) == float.fromhex("-0x1.d0ab1cp-1")


def test_frozen_cost_values(port):
    """test_costs.cpp:101-114 (circle 0 / 1012), :148-167 (nav 40 / 30), :169-175 (quadratic 4)."""
    circle = S.Scenario(dynamics="double_integrator", cost="circle_track")
    assert port.running_cost(circle, [2, 0, 0, 2]) == 0.0
    assert port.running_cost(circle, [0, 0, 0, 0]) == 1012.0
    cm = S.Costmap.empty(4.0, 4.0, 0.5, -2.0, -2.0)
    cm.fill_rect(0.9, 0.9, 1.4, 1.4, True)
    nav = S.Scenario(dynamics="diff_drive", cost="diff_drive_nav", costmap=cm)
    assert port.running_cost(nav, [0.0, 0.0, 0.0]) == 40.0   # 5*(4+4), free cell
    assert port.running_cost(nav, [1.0, 1.0, 0.0]) == 30.0   # 5*(1+1) + 20, occupied
    assert abs(port.running_cost(nav, [0.0, 0.0, 6.2831853]) - 40.0) < 40.0 * 1e-5  # yaw wraps
    quad = S.Scenario(dynamics="double_integrator", cost="quadratic", target=[1, -1], weights=[2, 0.5])
    assert port.running_cost(quad, [2, 1]) == 4.0             # 2*1 + 0.5*4
    assert port.terminal_cost(quad, [2, 1]) == 4.0


def test_frozen_weights(port):
    """test_engine.cpp:187-197: J = [1, 3, 2], lambda = 1."""
    w, rho, eta, am = port.compute_weights(np.array([1.0, 3.0, 2.0]), 1.0)
    e = np.exp(-np.array([0.0, 2.0, 1.0]))
    assert rho == 1.0 and am == 0
    assert np.allclose(w, e / e.sum(), rtol=0, atol=1e-15)
    w, rho, eta, am = port.compute_weights(np.full(4, 7.0), 1.0)
    assert np.all(w == 0.25) and am == 0


def test_di_exact_step(port):
    """test_dynamics.cpp:107-116: x' = x + dt * (v, u)."""
    sc = S.Scenario(dynamics="double_integrator", cost="road")
    xn, y = port.step(sc, [1, 2, 3, 4], [0.5, -0.5], 0.1)
    assert np.allclose(xn, [1.3, 2.4, 3.05, 3.95], atol=1e-6)
    assert np.array_equal(xn, y)


def _scenario_from_index(name, rec):
    d = json.load(open(os.path.join(GOLDEN, "index.json")))["scenarios"][name]
    sc = S.Scenario(**{k: (tuple(v) if k == "control_std" else v) for k, v in d.items()})
    if "costmap" in rec:
        res, ox, oy = rec["costmap_geom"]
        sc.costmap = S.Costmap(rec["costmap"].astype(np.uint8), float(res), float(ox), float(oy))
    return sc


GOLDEN_FILES = sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz")) if not os.path.basename(p).startswith("loop_"))
LOOP_FILES = sorted(glob.glob(os.path.join(GOLDEN, "loop_*.npz")))


@pytest.mark.parametrize("path", GOLDEN_FILES, ids=[os.path.basename(p)[:-4] for p in GOLDEN_FILES])
def test_oracle_matches_reference_goldens(oracle_built, port, path):
    name = os.path.basename(path)[:-4]
    rec = dict(np.load(path))
    sc = _scenario_from_index(name, rec)
    eps, flags = port.generate_samples(sc, rec["mean"], int(rec["stream"]))
    assert np.array_equal(eps.view(np.uint32), rec["eps"].view(np.uint32))
    assert np.array_equal(flags, rec["flags"])
    costs, outputs = port.rollout(sc, rec["x0s"], rec["means"], rec["eps"], outputs=True)
    assert np.array_equal(costs.view(np.uint64), rec["costs"].view(np.uint64))
    assert np.array_equal(outputs.view(np.uint32), rec["outputs"].view(np.uint32))
    w, rho, eta, am = port.compute_weights(rec["costs"][0], sc.lambda_)
    assert rho == rec["rho"] and eta == rec["eta"] and am == rec["argmin"]
    assert np.array_equal(w, rec["weights"])
    ctl = oracle_built.OracleController(sc, "port")
    x = sc.x0()
    for k in range(3):
        if sc.controller == "tube":
            r = ctl.tube_compute_control(x)
            assert np.array_equal(r["nominal_controls"], rec[f"solve{k}_nominal_controls"])
            assert np.array_equal(r["real_controls"], rec[f"solve{k}_real_controls"])
            assert np.array_equal(r["nominal_states"], rec[f"solve{k}_nominal_states"])
            assert np.array_equal(r["real_states"], rec[f"solve{k}_real_states"])
            assert np.array_equal(r["nominal_state"], rec[f"solve{k}_nominal_state"])
            for side in ("nominal", "real"):
                assert r[side]["baseline"] == rec[f"solve{k}_{side}_rho"]
                assert r[side]["argmin"] == rec[f"solve{k}_{side}_argmin"]
            x = x + np.float32(0.01)
        else:
            r = ctl.compute_control(x, want_weights=True)
            assert np.array_equal(r["controls"], rec[f"solve{k}_controls"])
            assert np.array_equal(r["states"], rec[f"solve{k}_states"])
            assert np.array_equal(r["outputs"], rec[f"solve{k}_outputs"])
            assert np.array_equal(r["weights"], rec[f"solve{k}_weights"])
            assert r["baseline"] == rec[f"solve{k}_rho"]
            if rec[f"solve{k}_argmin"] >= 0:  # -1: CEM (the shim cannot recover argmin from flat 1/k weights)
                assert r["argmin"] == rec[f"solve{k}_argmin"]
            if sc.controller == "cem":
                assert r["normalizer"] == rec[f"solve{k}_eta"] == max(1, math.ceil(sc.elite_fraction * sc.num_samples))


def test_cem_partial_sort_ties(port):
    """The CEM comparator: cost, then lower index (controllers.cpp:165-171)."""
    costs = np.array([3.0, 1.0, 2.0, 1.0, 0.5, 1.0, 3.0])
    assert list(port.partial_sort(costs, 7)) == [4, 1, 3, 5, 2, 0, 6]
    assert list(port.partial_sort(costs, 3)) == [4, 1, 3]


def test_port_vs_reference_randomized(oracle_built):
    """Randomized cross-check against oracle/_ref (skipped where it was not built)."""
    if not oracle_built.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    P, R = oracle_built.Oracle("port"), oracle_built.Oracle("reference")
    rng = np.random.default_rng(2024)
    pairs = [("double_integrator", "circle_track"), ("double_integrator", "road"), ("cartpole", "quadratic"),
             ("cartpole", "road"), ("diff_drive", "diff_drive_nav"), ("unicycle", "road"), ("unicycle", "diff_drive_nav"),
             ("diff_drive", "quadratic")]
    for trial in range(16):
        dyn, cost = pairs[trial % len(pairs)]
        n_x, n_u, n_y = S.MODEL_DIMS[dyn]
        sc = S.Scenario(num_samples=int(rng.integers(1, 200)), horizon=int(rng.integers(1, 40)), dynamics=dyn,
                        cost=cost, rng_seed=int(rng.integers(0, 2 ** 63)), control_std=tuple(rng.uniform(0.1, 2, n_u)),
                        zero_mean_fraction=float(rng.choice([0.0, 0.3, 1.0])),
                        include_mean_sample=bool(rng.integers(0, 2)), importance_sampling=bool(trial % 3 != 0),
                        lambda_=float(rng.uniform(0.1, 10)))
        if cost == "quadratic":
            sc.weights = list(rng.uniform(0, 2, n_y))
            sc.target = list(rng.standard_normal(n_y))
        if cost == "diff_drive_nav":
            sc.costmap = S.synthetic_costmap(int(rng.integers(0, 100)))
        mean = (rng.standard_normal((sc.horizon, n_u)) * 0.3).astype(np.float32)
        e1, f1 = P.generate_samples(sc, mean, trial)
        e2, f2 = R.generate_samples(sc, mean, trial, workers=int(rng.integers(1, 5)))
        assert np.array_equal(e1.view(np.uint32), e2.view(np.uint32)) and np.array_equal(f1, f2)
        x0 = (rng.standard_normal((1, n_x)) * 0.5).astype(np.float32)
        c1 = P.rollout(sc, x0, mean[None], e1)
        c2 = R.rollout(sc, x0, mean[None], e1, strategy=int(rng.integers(0, 2)), workers=3)
        assert np.array_equal(c1.view(np.uint64), c2.view(np.uint64))


def test_quadrotor_hover_is_an_equilibrium(port):
    """Builder-defined quadrotor (no reference model): zero control from hover
    keeps the state exactly (thrust m g cancels gravity, unit quaternion)."""
    sc = S.quadrotor_scenario(num_samples=4, horizon=5)
    x = sc.x0()
    assert x[6] == 1.0
    xn, y = port.step(sc, x, np.zeros(4, np.float32), np.float32(0.02))
    assert np.array_equal(xn, x) and np.array_equal(y, x)
    # a pure yaw-rate command rotates about z, keeps |q| = 1 and does not lift
    xr = x.copy()
    for _ in range(50):
        xr, _ = port.step(sc, xr, np.array([0, 0, 1.0, 0], np.float32), np.float32(0.02))
    assert abs(float(np.linalg.norm(xr[6:10])) - 1.0) < 1e-6
    assert abs(xr[2]) < 1e-5 and xr[12] > 0.9
    # thrust is clamped to [0, T_max]
    xc, _ = port.step(sc, x, np.array([0, 0, 0, 1e6], np.float32), np.float32(0.02))
    assert abs(xc[5] - 0.02 * (39.24 - 9.81)) < 1e-5


def test_mlp_oracle_zero_network_is_pure_kinematics(port):
    """With an all-zero network the MLP model is the AutoRally kinematics only."""
    sc = S.autorally_scenario(num_samples=4, horizon=5)
    sc.mlp_weights = np.zeros(1412, np.float32)
    x = np.array([0, 0, 0.5, 0, 2.0, 0.5, 0.3], np.float32)
    xn, _ = port.step(sc, x, np.array([0.2, 0.4], np.float32), np.float32(0.1))
    c, s = np.cos(np.float32(0.5)), np.sin(np.float32(0.5))
    assert abs(xn[0] - 0.1 * (2.0 * c - 0.5 * s)) < 1e-6 and abs(xn[1] - 0.1 * (2.0 * s + 0.5 * c)) < 1e-6
    assert abs(xn[2] - 0.53) < 1e-6 and np.array_equal(xn[3:], x[3:])



@pytest.mark.parametrize("path", LOOP_FILES, ids=[os.path.basename(p)[:-4] for p in LOOP_FILES])
def test_closed_loop_checker_matches_reference_goldens(oracle_built, path):
    """The Python Plant::run_control_loop around the C oracle (oracle.bindings.
    control_loop) reproduces the reference's own closed loop bit for bit:
    replan schedule, shifts, applied controls, running costs, disturbances."""
    name = os.path.basename(path)[:-4]
    rec = dict(np.load(path))
    sc = _scenario_from_index(name, rec)
    if sc.cost == "diff_drive_nav" and sc.costmap is None:
        sc.costmap = S.synthetic_costmap()
    acc, rows = oracle_built.control_loop(sc, int(rec["steps"]) * sc.dt)
    assert acc == rec["accumulated_cost"]
    assert np.array_equal(rows, rec["rows"])


def test_bicycle_oracle_kinematics(port):
    """Builder-defined kinematic bicycle: straight line at zero steering, yaw
    rate v tan(delta) / L, controls clamped to the configured bounds."""
    sc = S.bicycle_nav_scenario(num_samples=4, horizon=5)
    x = np.array([0.0, 0.0, 0.0], np.float32)
    xn, _ = port.step(sc, x, np.array([0.4, 0.0], np.float32), np.float32(0.1))
    assert np.allclose(xn, [0.04, 0.0, 0.0], atol=1e-7)
    xn, _ = port.step(sc, x, np.array([0.4, 0.3], np.float32), np.float32(0.1))
    assert abs(xn[2] - 0.1 * 0.4 * np.tan(0.3) / 0.5) < 1e-6
    xn, _ = port.step(sc, x, np.array([9.0, 9.0], np.float32), np.float32(0.1))  # clamped to (0.5, 0.6)
    assert abs(xn[0] - 0.05) < 1e-7 and abs(xn[2] - 0.1 * 0.5 * np.tan(0.6) / 0.5) < 1e-6
