"""CPU: Scenario -> smpc_problem flattening mirrors the reference schema."""
import ctypes
import math

import numpy as np

from paper_2409_07563_b200 import scenario as S


def test_struct_layout_matches_header():
    # offsets the C compiler uses for smpc_problem (include/smpc_b200.h)
    import subprocess
    import tempfile
    import os
    src = r'''
#include <stddef.h>
#include <stdio.h>
#include "smpc_b200.h"
int main(){printf("%zu %zu %zu %zu %zu %zu\n", sizeof(smpc_problem), offsetof(smpc_problem, costmap),
 offsetof(smpc_problem, device), offsetof(smpc_problem, update_skip_mass), sizeof(smpc_solution),
 sizeof(smpc_tube_solution)); return 0;}
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "t.c"), "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(root, "include"), os.path.join(d, "t.c"), "-o", os.path.join(d, "t")],
                       check=True)
        out = subprocess.run([os.path.join(d, "t")], capture_output=True, text=True).stdout.split()
    want = [ctypes.sizeof(S.SmpcProblem), S.SmpcProblem.costmap.offset, S.SmpcProblem.device.offset,
            S.SmpcProblem.update_skip_mass.offset, ctypes.sizeof(S.SmpcSolution), ctypes.sizeof(S.SmpcTubeSolution)]
    assert [int(v) for v in out] == want


def test_defaults_follow_scenario_hpp():
    sc = S.Scenario()
    assert (sc.dt, sc.horizon, sc.num_samples, sc.iterations, sc.lambda_) == (0.02, 100, 1024, 1, 1.0)
    assert tuple(sc.control_std) == (0.2,) and sc.rng_seed == 0
    assert sc.include_mean_sample and sc.importance_sampling and sc.zero_mean_fraction == 0.0
    assert sc.dynamics == "diff_drive" and sc.cost == "diff_drive_nav" and sc.controller == "mppi"
    assert math.isinf(sc.nominal_reset_bound)
    cm = sc.effective_costmap()  # make_cost default: all-free 11 m x 11 m @ 0.1 m
    assert cm.grid.shape == (110, 110) and cm.grid.sum() == 0


def test_problem_fields():
    sc = S.Scenario(dynamics="cartpole", cost="quadratic", weights=[1, 2, 3, 4], control_std=(0.5,), rng_seed=2 ** 40 + 3,
                    controller="dmd", step_size_per_step=[0.5] * 100)
    p = sc.to_problem(shard=(10, 20))
    assert p.dynamics_kind == 1 and p.cost_kind == 3 and p.n_quad == 4 and p.controller_kind == 1
    assert p.seed == 2 ** 40 + 3 and p.n_step_sizes == 100 and p.step_sizes[99] == np.float32(0.5)
    assert (p.shard_begin, p.shard_end) == (10, 20)
    assert list(p.quad_target)[:4] == [0, 0, 0, 0]
    assert p.update_skip_mass == 2.0 ** -64


def test_initial_state_by_name():
    sc = S.di_swarm_scenario(num_samples=4)
    assert list(sc.x0()) == [2.0, 0.0, 0.0, 2.0]


def test_costmap_text_roundtrip(tmp_path):
    cm = S.synthetic_costmap(5)
    path = str(tmp_path / "m.costmap")
    cm.save(path)
    back = S.Costmap.load(path)
    assert np.array_equal(back.grid, cm.grid) and back.resolution == cm.resolution


def test_costmap_empty_rounds_halves_away_from_zero():
    """Costmap2D ctor uses std::lround (costmap.cpp:22-23): 0.25 m at 0.1 m is
    2.5 cells -> 3 (Python's round() would give 2)."""
    cm = S.Costmap.empty(0.25, 0.45, 0.1, 0.0, 0.0)  # 2.5 x 4.5 cells
    assert cm.grid.shape == (5, 3)
    assert S._lround(2.5) == 3 and S._lround(-2.5) == -3 and S._lround(2.49) == 2
