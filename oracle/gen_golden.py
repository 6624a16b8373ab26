"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

TEST INFRASTRUCTURE ONLY. Run here (where /root/reference exists):
    python oracle/gen_golden.py
Each fixture records, for one scenario: the reference's noise batch, rollout
costs (fused and split strategies, 3 workers), stored trajectories, the
compute_weights result, and three warm-started compute_control solves (or
tube solves). The C restatement (oracle/smpc_oracle.c) and the GPU path are
checked against these files; /root/reference is not needed at test time.
"""
import json
import os
import sys
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.bindings import Oracle, OracleController, build  # noqa: E402
from paper_2409_07563_b200 import scenario as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
OBSTACLES = "/root/reference/proj/configs/obstacles.costmap"


def fixture_scenarios():
    sc = {}
    sc["cartpole_c1"] = S.cartpole_scenario(num_samples=256, horizon=100, seed=1)
    sc["di_swarm_c5"] = S.di_swarm_scenario(num_samples=512, horizon=100, seed=7)
    nav = S.diff_drive_nav_scenario(num_samples=200, horizon=56, seed=42,
                                    costmap=S.Costmap.load(OBSTACLES))
    nav.control_std = (1.0, 1.0)  # proj/configs/diff_drive_nav.json uses sigma = 1
    sc["diffdrive_nav_obstacles"] = nav
    sc["diffdrive_nav_synthetic"] = S.diff_drive_nav_scenario(num_samples=200, horizon=56, seed=3)
    sc["unicycle_road_zero_mean"] = S.Scenario(num_samples=160, horizon=40, dynamics="unicycle", cost="road",
                                               rng_seed=11, control_std=(0.5, 0.3), zero_mean_fraction=0.25)
    sc["cartpole_perstep_nomean"] = S.Scenario(num_samples=128, horizon=30, dynamics="cartpole", cost="road",
                                               rng_seed=5, control_std=(1.0,),
                                               std_per_step=[[0.5 + 0.02 * t] for t in range(30)],
                                               zero_mean_fraction=0.1, include_mean_sample=False)
    sc["di_quadratic_dmd"] = S.Scenario(num_samples=192, horizon=25, dynamics="double_integrator", cost="quadratic",
                                        target=[1.0, -1.0, 0.0, 0.0], weights=[1.0, 1.0, 0.1, 0.1], rng_seed=3,
                                        control_std=(0.7, 0.4), controller="dmd", step_size=0.6, lambda_=2.0)
    circle = S.di_swarm_scenario(num_samples=256, horizon=32, seed=7)
    circle.controller, circle.step_size = "dmd", 0.8  # proj/configs/circle_track_dmd.json
    sc["circle_track_dmd_config"] = circle
    # CemController (controllers.cpp:149-203); importance on in the config to
    # pin that CEM ranks the raw costs
    sc["di_quadratic_cem"] = S.Scenario(num_samples=192, horizon=25, dynamics="double_integrator", cost="quadratic",
                                        target=[1.0, -1.0, 0.0, 0.0], weights=[1.0, 1.0, 0.1, 0.1], rng_seed=9,
                                        control_std=(0.7, 0.4), controller="cem", elite_fraction=0.25,
                                        zero_mean_fraction=0.1)
    cem_c1 = S.cartpole_scenario(num_samples=300, horizon=60, seed=2)
    cem_c1.controller, cem_c1.elite_fraction = "cem", 0.07
    sc["cartpole_cem"] = cem_c1
    tube = S.cartpole_scenario(num_samples=256, horizon=50, seed=4)
    tube.controller = "tube"
    sc["cartpole_tube"] = tube
    # iterations > 1 (controllers.cpp:115-131): stream_for(iter) and the mean
    # updated between the in-solve iterations
    it3 = S.cartpole_scenario(num_samples=256, horizon=60, seed=21)
    it3.iterations = 3
    sc["cartpole_iter3"] = it3
    # DMD with per-step gamma (engine.cpp:397-401) and I = 3
    sc["di_dmd_perstep_iter3"] = S.Scenario(num_samples=192, horizon=25, dynamics="double_integrator",
                                            cost="quadratic", target=[1.0, -1.0, 0.0, 0.0],
                                            weights=[1.0, 1.0, 0.1, 0.1], rng_seed=31, control_std=(0.7, 0.4),
                                            controller="dmd", iterations=3, lambda_=0.7,
                                            step_size_per_step=[0.3 + 0.025 * t for t in range(25)])
    tube3 = S.cartpole_scenario(num_samples=256, horizon=40, seed=23)
    tube3.controller, tube3.iterations = "tube", 3
    sc["cartpole_tube_iter3"] = tube3
    cem3 = S.di_swarm_scenario(num_samples=200, horizon=30, seed=25)
    cem3.controller, cem3.elite_fraction, cem3.iterations = "cem", 0.1, 3
    sc["di_cem_iter3"] = cem3
    # C3 with sigma = 0.2 (non-power-of-two sigma^2: the importance term divides)
    # and I = 2, over the reference's own obstacles.costmap
    nav2 = S.diff_drive_nav_scenario(num_samples=200, horizon=56, seed=44, costmap=S.Costmap.load(OBSTACLES))
    nav2.iterations, nav2.lambda_ = 2, 0.3
    sc["diffdrive_nav_sigma02_iter2"] = nav2
    return sc


def closed_loop_scenarios():
    sweep = S.default_sweep_scenario()  # bench.cpp:186-202
    sweep.num_samples, sweep.step_size, sweep.rng_seed, sweep.disturbance_std = 256, 0.6, 3, 0.3
    nav = S.diff_drive_nav_scenario(num_samples=200, horizon=20, seed=8)
    nav.replan_rate, nav.disturbance_std = 20.0, 0.2  # replans every 2.5 steps: shifts + idx > 0
    return {"loop_sweep_dmd": (sweep, 200), "loop_nav_replan20": (nav, 100)}


def scenario_record(sc: S.Scenario) -> dict:
    d = {k: v for k, v in vars(sc).items() if k not in ("costmap", "mlp_weights")}
    d["control_std"] = list(sc.control_std)
    return d


def main(only=None):
    """Regenerate every fixture, or only the named ones (index.json is merged)."""
    build()
    R = Oracle("reference")
    os.makedirs(OUT, exist_ok=True)
    index = {}
    old = None
    if only:
        old = json.load(open(os.path.join(OUT, "index.json")))
        index = old["scenarios"]
    for name, sc in fixture_scenarios().items():
        if only and name not in only:
            continue
        n_x, n_u, n_y = sc.dims
        T = sc.horizon
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        mean = (rng.standard_normal((T, n_u)) * 0.2).astype(np.float32)
        stream = 5
        eps, flags = R.generate_samples(sc, mean, stream, workers=3)
        S_ = 2 if sc.controller == "tube" else 1
        means = np.stack([mean] + [mean * 0.5] * (S_ - 1)).astype(np.float32)
        x0s = np.stack([sc.x0() + np.float32(0.05 * s) for s in range(S_)]).astype(np.float32)
        costs_split, outputs = R.rollout(sc, x0s, means, eps, outputs=True, workers=3)
        costs_fused = R.rollout(sc, x0s, means, eps, strategy=1, workers=3)
        assert np.array_equal(costs_split, costs_fused)
        w, rho, eta, am = R.compute_weights(costs_fused[0], sc.lambda_)
        rec = dict(mean=mean, stream=np.int64(stream), eps=eps, flags=flags, x0s=x0s, means=means,
                   costs=costs_fused, outputs=outputs, weights=w, rho=np.float64(rho), eta=np.float64(eta),
                   argmin=np.int64(am))
        ctl = OracleController(sc, "reference", workers=3)
        x = sc.x0()
        for k in range(3):
            if sc.controller == "tube":
                r = ctl.tube_compute_control(x)
                rec[f"solve{k}_x"] = x.copy()
                rec[f"solve{k}_nominal_controls"] = r["nominal_controls"]
                rec[f"solve{k}_real_controls"] = r["real_controls"]
                rec[f"solve{k}_nominal_states"] = r["nominal_states"]
                rec[f"solve{k}_real_states"] = r["real_states"]
                rec[f"solve{k}_nominal_state"] = r["nominal_state"]
                for side in ("nominal", "real"):
                    rec[f"solve{k}_{side}_rho"] = np.float64(r[side]["baseline"])
                    rec[f"solve{k}_{side}_eta"] = np.float64(r[side]["normalizer"])
                    rec[f"solve{k}_{side}_argmin"] = np.int64(r[side]["argmin"])
                x = x + np.float32(0.01)
            else:
                r = ctl.compute_control(x, want_weights=True)
                rec[f"solve{k}_controls"] = r["controls"]
                rec[f"solve{k}_states"] = r["states"]
                rec[f"solve{k}_outputs"] = r["outputs"]
                rec[f"solve{k}_weights"] = r["weights"]
                rec[f"solve{k}_rho"] = np.float64(r["baseline"])
                rec[f"solve{k}_eta"] = np.float64(r["normalizer"])
                rec[f"solve{k}_argmin"] = np.int64(r["argmin"])
        cm = sc.effective_costmap()
        if cm is not None:
            rec["costmap"] = cm.grid
            rec["costmap_geom"] = np.array([cm.resolution, cm.origin_x, cm.origin_y])
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        index[name] = scenario_record(sc)
        print(name, "rho", rho, "argmin", am, "bytes", os.path.getsize(os.path.join(OUT, f"{name}.npz")))
    # Closed loops: the reference's own Plant::run_control_loop (plant.cpp:133-181).
    from oracle.bindings import reference_control_loop
    for name, (sc, steps) in closed_loop_scenarios().items():
        if only and name not in only:
            continue
        acc, rows = reference_control_loop(sc, steps * sc.dt)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), accumulated_cost=np.float64(acc), rows=rows,
                            steps=np.int64(steps))
        index[name] = scenario_record(sc)
        print(name, "accumulated cost", acc)
    # Random123 Philox4x32-10 known-answer vectors and reference normals.
    kat = old["kat"] if old else {
        "philox": [
            [[0, 0, 0, 0], [0, 0], [int(v) for v in R.philox([0, 0, 0, 0], [0, 0])]],
            [[0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [int(v) for v in R.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)]],
            [[0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
             [int(v) for v in R.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0])]],
        ],
        "quad": [[seed, a, b, c, [float(v).hex() for v in R.quad(seed, a, b, c)]]
                 for seed, a, b, c in [(0, 0, 0, 0), (0, 0, 1, 0), (0, 0, 4, 0), (42, 0, 1, 0), (7, 256, 5221, 3)]],
    }
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump({"scenarios": index, "kat": kat,
                   "generator": "oracle/gen_golden.py via oracle/_ref/libsmpc_ref.so (reference compiled from "
                                "/root/reference/proj/core/src with the Eigen-subset shim)"}, f, indent=1,
                  default=lambda o: list(o) if isinstance(o, tuple) else o)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)
