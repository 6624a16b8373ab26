"""GPU path against the UNMODIFIED reference's own outputs (tests/golden,
generated from oracle/_ref by oracle/gen_golden.py) — every fixture, not just
the restated oracle.

Per fixture: the device noise batch and flags, the rollout costs (injected and
regenerated noise) and stored outputs are compared bit for bit; the weights
(rho/argmin exact, eta and w within 1e-12); then three warm-started solves of
the reference controller (compute_control, or tube_compute_control) with
rho/argmin exact and U*/states within the north-star FP32 tolerance 1e-4.
The *_iter3 / *_iter2 fixtures run iterations > 1 inside each solve, which
exercises Controller::stream_for(iter) (controllers.cpp:63-66) and the mean
updated between in-solve iterations (controllers.cpp:115-131);
di_dmd_perstep_iter3 has one step size per timestep (engine.cpp:397-401).
"""
import glob
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
FILES = sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz")) if not os.path.basename(p).startswith("loop_"))


def close(a, b, tol=TOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))


@pytest.fixture(scope="module")
def mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_07563_b200 import controllers, scenario
    return dict(C=controllers, S=scenario)


def load(S, path):
    name = os.path.basename(path)[:-4]
    rec = dict(np.load(path))
    d = json.load(open(os.path.join(GOLDEN, "index.json")))["scenarios"][name]
    sc = S.Scenario(**{k: (tuple(v) if k == "control_std" else v) for k, v in d.items()})
    if "costmap" in rec:
        res, ox, oy = rec["costmap_geom"]
        sc.costmap = S.Costmap(rec["costmap"].astype(np.uint8), float(res), float(ox), float(oy))
    return sc, rec


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(p)[:-4] for p in FILES])
def test_device_noise_and_rollout_match_reference(mods, path):
    C, S = mods["C"], mods["S"]
    sc, rec = load(S, path)
    smp = C.GaussianSampler(sc)
    eps, flags = smp.generate_samples(rec["mean"], int(rec["stream"]))
    assert np.array_equal(eps.view(np.uint32), rec["eps"].view(np.uint32))
    assert np.array_equal(flags, rec["flags"])
    eng = C.RolloutEngine(sc)
    costs, outputs = eng.rollout(rec["x0s"], rec["means"], eps=rec["eps"], outputs=True)
    assert np.array_equal(costs.view(np.uint64), rec["costs"].view(np.uint64))
    assert np.array_equal(outputs.view(np.uint32), rec["outputs"].view(np.uint32))
    regen = eng.rollout(rec["x0s"], rec["means"], stream=int(rec["stream"]))
    assert np.array_equal(regen.view(np.uint64), rec["costs"].view(np.uint64))
    r = eng.compute_weights(rec["costs"][0], sc.lambda_)
    assert r.baseline == rec["rho"] and r.argmin == rec["argmin"]
    assert close(r.normalizer, rec["eta"], 1e-12)
    assert close(r.weights, rec["weights"], 1e-12)


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(p)[:-4] for p in FILES])
def test_device_solves_match_reference(mods, path):
    C, S = mods["C"], mods["S"]
    sc, rec = load(S, path)
    gpu = C.make_controller(sc)
    x = sc.x0()
    for k in range(3):
        if sc.controller == "tube":
            a = gpu.tube_compute_control(x)
            for side in ("nominal", "real"):
                w = getattr(a, side).weights
                assert w.baseline == rec[f"solve{k}_{side}_rho"], (k, side)
                assert w.argmin == rec[f"solve{k}_{side}_argmin"], (k, side)
                assert close(w.normalizer, rec[f"solve{k}_{side}_eta"])
            assert close(a.nominal.controls, rec[f"solve{k}_nominal_controls"])
            assert close(a.real.controls, rec[f"solve{k}_real_controls"])
            assert close(a.nominal.states, rec[f"solve{k}_nominal_states"])
            assert close(a.real.states, rec[f"solve{k}_real_states"])
            assert np.array_equal(a.nominal_state, rec[f"solve{k}_nominal_state"])
            gpu.set_mean(rec[f"solve{k}_nominal_controls"], 0)
            gpu.set_mean(rec[f"solve{k}_real_controls"], 1)
            x = x + np.float32(0.01)
        else:
            a = gpu.compute_control(x, want_weights=True)
            assert a.weights.baseline == rec[f"solve{k}_rho"], k
            if rec[f"solve{k}_argmin"] >= 0:  # -1: CEM golden (argmin not recoverable from 1/k weights)
                assert a.weights.argmin == rec[f"solve{k}_argmin"], k
            if sc.controller == "cem":
                assert np.array_equal(a.weights.weights, rec[f"solve{k}_weights"])
                assert a.weights.normalizer == rec[f"solve{k}_eta"]
            else:
                assert close(a.weights.normalizer, rec[f"solve{k}_eta"])
                assert close(a.weights.weights, rec[f"solve{k}_weights"])
            assert close(a.controls, rec[f"solve{k}_controls"]), np.abs(a.controls - rec[f"solve{k}_controls"]).max()
            assert close(a.states, rec[f"solve{k}_states"])
            assert close(a.outputs, rec[f"solve{k}_outputs"])
            gpu.set_mean(rec[f"solve{k}_controls"])
    assert gpu.solve_count == 3
