"""BASELINE C5 (double integrator + circle track, N = 2^20, T = 100) at full
size against the reference, not a subset:

* every one of the 2^20 device costs equals the oracle's bit for bit (the
  oracle regenerates the same Philox batch chunk by chunk);
* two warm-started solves of the UNMODIFIED reference MppiController
  (oracle/_ref, all host threads) against smpc_compute_control: rho and
  argmin exact, weights and U* within the north-star tolerance.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4
N = 1 << 20
T = 100


def close(a, b, tol=TOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))


@pytest.fixture(scope="module")
def mods(oracle_built):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.bindings import Oracle, OracleController, ref_available
    from paper_2409_07563_b200 import controllers, scenario
    return dict(Oracle=Oracle, OracleController=OracleController, C=controllers, S=scenario,
                ref_available=ref_available)


def test_all_full_size_costs_bit_exact(mods):
    S, C = mods["S"], mods["C"]
    sc = S.di_swarm_scenario(num_samples=N, horizon=T, seed=7)
    x0 = sc.x0()
    rng = np.random.default_rng(5)
    mean = (rng.standard_normal((T, 2)) * 0.3).astype(np.float32)
    costs = C.RolloutEngine(sc).rollout(x0[None], mean[None], stream=3)[0]
    O = mods["Oracle"]("port")
    chunk = 1 << 16
    for b in range(0, N, chunk):
        e, _ = O.generate_samples(sc, mean, 3, m_begin=b, m_end=b + chunk)
        c = O.rollout(sc, x0[None], mean[None], e)[0]
        bad = np.nonzero(c.view(np.uint64) != costs[b:b + chunk].view(np.uint64))[0]
        assert bad.size == 0, (b + bad[:5], c[bad[:5]], costs[b + bad[:5]])


def test_full_size_solves_match_reference_controller(mods):
    if not mods["ref_available"]():
        pytest.skip("oracle/_ref not built")
    S, C = mods["S"], mods["C"]
    sc = S.di_swarm_scenario(num_samples=N, horizon=T, seed=7)
    gpu = C.make_controller(sc)
    ref = mods["OracleController"](sc, "reference", workers=os.cpu_count() or 1)
    x0 = sc.x0()
    for solve in range(2):
        a = gpu.compute_control(x0, want_weights=True)
        b = ref.compute_control(x0, want_weights=True)
        assert a.weights.baseline == b["baseline"], solve
        assert a.weights.argmin == b["argmin"], solve
        assert close(a.weights.normalizer, b["normalizer"])
        assert close(a.weights.weights, b["weights"])
        assert close(a.controls, b["controls"]), np.abs(a.controls - b["controls"]).max()
        assert close(a.states, b["states"])
        gpu.set_mean(b["controls"])
