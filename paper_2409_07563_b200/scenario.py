"""Scenario description shared by the product, the oracle and the reference.

`Scenario` mirrors the reference's ``ScenarioConfig`` JSON schema
(/root/reference/proj/core/include/smpc/scenario.hpp:13-140) with the same
field names and defaults, restricted to what the MPPI iteration consumes.
``Scenario.to_problem()`` flattens it into the C-ABI ``smpc_problem`` struct
(include/smpc_b200.h) that the CUDA library, the C oracle and the reference
shim all accept, so one description drives all three.
"""
from __future__ import annotations

import ctypes
import dataclasses
import json
import math
from typing import Dict, List, Optional, Sequence

import numpy as np

SMPC_MAX_DIM = 16
SMPC_MAX_PARAMS = 32
ABI_VERSION = 4

DYNAMICS_KINDS = {"unicycle": 0, "cartpole": 1, "diff_drive": 2, "double_integrator": 3,
                  # builder-defined (no reference counterpart): BASELINE.json configs[1] / configs[3]
                  "quadrotor": 4, "mlp": 5, "bicycle": 6,
                  # a user model compiled against include/smpc_b200_plugin.cuh (smpc_create_with_ops)
                  "plugin": 100}
COST_KINDS = {"road": 0, "circle_track": 1, "diff_drive_nav": 2, "quadratic": 3}
CONTROLLER_KINDS = {"mppi": 0, "dmd": 1, "cem": 2, "tube": 3, "rmppi": 4}

# ModelDims per dynamics kind (dynamics.cpp:122-181) and state names
# (used by initial_state, scenario.hpp:136-137 / state_from_named_values).
MODEL_DIMS = {
    "unicycle": (3, 2, 3),
    "cartpole": (4, 1, 4),
    "diff_drive": (3, 2, 3),
    "double_integrator": (4, 2, 4),
    "quadrotor": (13, 4, 13),
    "mlp": (7, 2, 7),
    "bicycle": (3, 2, 3),
}
STATE_NAMES = {
    "unicycle": ["X", "Y", "YAW"],
    "cartpole": ["X", "X_DOT", "THETA", "THETA_DOT"],
    "diff_drive": ["X", "Y", "YAW"],
    "double_integrator": ["X", "Y", "V_X", "V_Y"],
    "quadrotor": ["X", "Y", "Z", "V_X", "V_Y", "V_Z", "QW", "QX", "QY", "QZ", "W_X", "W_Y", "W_Z"],
    # AutoRally state convention (MPPI-Generic AutoRallyDynamics): pose, then the
    # body-frame dynamic state the network predicts
    "mlp": ["X", "Y", "YAW", "ROLL", "V_X", "V_Y", "YAW_RATE"],
    "bicycle": ["X", "Y", "YAW"],
}


class SmpcProblem(ctypes.Structure):
    """ctypes mirror of ``smpc_problem`` (include/smpc_b200.h)."""

    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("num_samples", ctypes.c_int32),
        ("horizon", ctypes.c_int32),
        ("iterations", ctypes.c_int32),
        ("dt", ctypes.c_double),
        ("lambda_", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("n_control_std", ctypes.c_int32),
        ("control_std", ctypes.c_float * SMPC_MAX_DIM),
        ("std_per_step", ctypes.POINTER(ctypes.c_float)),
        ("zero_mean_fraction", ctypes.c_double),
        ("include_mean_sample", ctypes.c_int32),
        ("importance_sampling", ctypes.c_int32),
        ("controller_kind", ctypes.c_int32),
        ("n_step_sizes", ctypes.c_int32),
        ("step_sizes", ctypes.POINTER(ctypes.c_float)),
        ("nominal_reset_bound", ctypes.c_double),
        ("elite_fraction", ctypes.c_double),
        ("feedback_gain", ctypes.POINTER(ctypes.c_float)),
        ("cost_threshold", ctypes.c_double),
        ("num_candidates", ctypes.c_int32),
        ("dynamics_kind", ctypes.c_int32),
        ("n_dyn_params", ctypes.c_int32),
        ("dyn_params", ctypes.c_double * SMPC_MAX_PARAMS),
        ("dyn_tensor", ctypes.POINTER(ctypes.c_float)),
        ("dyn_tensor_len", ctypes.c_int64),
        ("cost_kind", ctypes.c_int32),
        ("n_cost_params", ctypes.c_int32),
        ("cost_params", ctypes.c_double * SMPC_MAX_PARAMS),
        ("n_quad", ctypes.c_int32),
        ("quad_target", ctypes.c_float * SMPC_MAX_DIM),
        ("quad_weights", ctypes.c_float * SMPC_MAX_DIM),
        ("costmap", ctypes.POINTER(ctypes.c_uint8)),
        ("costmap_cells_x", ctypes.c_int32),
        ("costmap_cells_y", ctypes.c_int32),
        ("costmap_resolution", ctypes.c_double),
        ("costmap_origin_x", ctypes.c_double),
        ("costmap_origin_y", ctypes.c_double),
        ("device", ctypes.c_int32),
        ("shard_begin", ctypes.c_int64),
        ("shard_end", ctypes.c_int64),
        ("update_skip_mass", ctypes.c_double),
    ]


class SmpcWeightSummary(ctypes.Structure):
    _fields_ = [
        ("baseline", ctypes.c_double),
        ("normalizer", ctypes.c_double),
        ("argmin", ctypes.c_int64),
        ("nonzero", ctypes.c_int64),
    ]


class SmpcSolution(ctypes.Structure):
    _fields_ = [
        ("controls", ctypes.POINTER(ctypes.c_float)),
        ("states", ctypes.POINTER(ctypes.c_float)),
        ("outputs", ctypes.POINTER(ctypes.c_float)),
        ("weights", ctypes.POINTER(ctypes.c_double)),
        ("summary", SmpcWeightSummary),
        ("solve_time_ms", ctypes.c_double),
    ]


class SmpcTubeSolution(ctypes.Structure):
    _fields_ = [
        ("nominal", SmpcSolution),
        ("real", SmpcSolution),
        ("nominal_state", ctypes.POINTER(ctypes.c_float)),
    ]


class SmpcPlantConfig(ctypes.Structure):
    """smpc_plant_config (include/smpc_b200.h)."""

    _fields_ = [("replan_rate", ctypes.c_double), ("dt_min", ctypes.c_double),
                ("disturbance_std", ctypes.c_double), ("rng_seed", ctypes.c_uint64)]


class SmpcLoopResult(ctypes.Structure):
    """smpc_loop_result (include/smpc_b200.h)."""

    _fields_ = [("accumulated_cost", ctypes.c_double), ("solve_count", ctypes.c_int64),
                ("mean_solve_ms", ctypes.c_double), ("steps", ctypes.c_int64)]


def _lround(x: float) -> int:
    """std::lround: halves round away from zero (Python's round() is half-even)."""
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


@dataclasses.dataclass
class Costmap:
    """Costmap2D (costmap.hpp:17-63): binary grid, row 0 at the lowest y."""

    grid: np.ndarray  # uint8 [cells_y, cells_x]
    resolution: float
    origin_x: float
    origin_y: float

    @staticmethod
    def empty(width_m: float, height_m: float, resolution: float, origin_x: float, origin_y: float) -> "Costmap":
        cx = _lround(width_m / resolution)
        cy = _lround(height_m / resolution)
        return Costmap(np.zeros((cy, cx), np.uint8), resolution, origin_x, origin_y)

    def fill_rect(self, x0: float, y0: float, x1: float, y1: float, occupied: bool = True) -> None:
        """Costmap2D::fill_rect (costmap.cpp:42-52): cells whose centre is inside."""
        cy, cx = self.grid.shape
        for iy in range(cy):
            yc = self.origin_y + (iy + 0.5) * self.resolution
            if yc < y0 or yc > y1:
                continue
            for ix in range(cx):
                xc = self.origin_x + (ix + 0.5) * self.resolution
                if xc < x0 or xc > x1:
                    continue
                self.grid[iy, ix] = 1 if occupied else 0

    @staticmethod
    def load(path: str) -> "Costmap":
        """Costmap2D::load text format (costmap.cpp:54-108)."""
        with open(path) as f:
            lines = f.read().splitlines()
        width = float(lines[0].split()[1])
        height = float(lines[1].split()[1])
        res = float(lines[2].split()[1])
        ox, oy = (float(v) for v in lines[3].split()[1:3])
        cm = Costmap.empty(width, height, res, ox, oy)
        cy, cx = cm.grid.shape
        for iy in range(cy):
            cm.grid[iy] = np.array([int(v) for v in lines[4 + iy].split()[:cx]], np.uint8)
        return cm

    def save(self, path: str) -> None:
        cy, cx = self.grid.shape
        with open(path, "w") as f:
            f.write(f"width_m {cx * self.resolution:g}\nheight_m {cy * self.resolution:g}\n")
            f.write(f"resolution {self.resolution:g}\norigin {self.origin_x:g} {self.origin_y:g}\n")
            for iy in range(cy):
                f.write(" ".join(str(int(v)) for v in self.grid[iy]) + "\n")


@dataclasses.dataclass
class Scenario:
    """ScenarioConfig subset (scenario.hpp:118-140), same names and defaults."""

    dt: float = 0.02
    horizon: int = 100
    num_samples: int = 1024
    iterations: int = 1
    lambda_: float = 1.0
    control_std: Sequence[float] = (0.2,)
    rng_seed: int = 0
    # sampler (scenario.hpp:14-23)
    std_per_step: Optional[Sequence[Sequence[float]]] = None
    zero_mean_fraction: float = 0.0
    include_mean_sample: bool = True
    importance_sampling: bool = True
    # dynamics (scenario.hpp:25-43)
    dynamics: str = "diff_drive"
    dynamics_params: Dict[str, float] = dataclasses.field(default_factory=dict)
    # cost (scenario.hpp:45-81)
    cost: str = "diff_drive_nav"
    cost_params: Dict[str, float] = dataclasses.field(default_factory=dict)
    target: Optional[Sequence[float]] = None
    weights: Optional[Sequence[float]] = None
    costmap: Optional[Costmap] = None
    # SMPC_DYN_MLP parameter blob (1412 floats, see autorally_mlp_weights)
    mlp_weights: Optional[np.ndarray] = None
    # controller (scenario.hpp:83-94)
    controller: str = "mppi"
    step_size: float = 1.0
    step_size_per_step: Optional[Sequence[float]] = None
    nominal_reset_bound: float = math.inf
    elite_fraction: float = 0.125
    # RMPPI (builder-defined, see include/smpc_b200.h SMPC_CTRL_RMPPI)
    feedback_gain: Optional[Sequence[Sequence[float]]] = None  # K [n_u][n_x]
    cost_threshold: float = math.inf
    num_candidates: int = 9
    initial_state: Dict[str, float] = dataclasses.field(default_factory=dict)
    # plant (PlantSection, scenario.hpp:107-114)
    replan_rate: float = 50.0
    dt_min: float = 0.02
    disturbance_std: float = 0.0
    device: int = 0
    # user model (dynamics="plugin"): (n_x, n_u, n_y) of the plugin's functors
    plugin_dims: Optional[Sequence[int]] = None
    # B200 deployment knob (not in the reference schema): weighted-update
    # samples with w_m < update_skip_mass / M are skipped (0 = exact).
    update_skip_mass: float = 2.0 ** -64

    # --- derived -----------------------------------------------------------
    @property
    def dims(self):
        if self.dynamics == "plugin":
            return tuple(int(v) for v in self.plugin_dims)
        return MODEL_DIMS[self.dynamics]

    def x0(self) -> np.ndarray:
        names = STATE_NAMES.get(self.dynamics) or [f"X{i}" for i in range(self.dims[0])]
        x = np.zeros(len(names), np.float32)
        for k, v in self.initial_state.items():
            x[names.index(k)] = np.float32(v)
        return x

    def step_sizes(self) -> List[float]:
        """make_controller (controllers.cpp:315-321): dmd only."""
        if self.controller != "dmd":
            return []
        if self.step_size_per_step:
            return [float(v) for v in self.step_size_per_step]
        return [float(self.step_size)]

    def _dyn_params(self) -> List[float]:
        d = self.dynamics_params
        if self.dynamics == "cartpole":
            return [d.get("cart_mass", 1.0), d.get("pole_mass", 1.0), d.get("pole_length", 1.0), d.get("gravity", 9.81)]
        if self.dynamics == "diff_drive":
            return [d.get("wheel_radius", 1.0), d.get("wheel_length", 1.0), d.get("v_min", -0.35),
                    d.get("v_max", 0.5), d.get("w_min", -0.5), d.get("w_max", 0.5)]
        if self.dynamics == "bicycle":
            return [d.get("wheelbase", 0.5), d.get("v_min", -0.35), d.get("v_max", 0.5),
                    d.get("steer_min", -0.6), d.get("steer_max", 0.6)]
        if self.dynamics == "quadrotor":
            return [d.get("mass", 1.0), d.get("gravity", 9.81), d.get("rate_time_constant", 0.05),
                    d.get("thrust_max", 39.24), d.get("rate_max", 5.0)]
        return []

    def _cost_params(self) -> List[float]:
        c = self.cost_params
        if self.cost == "road":
            return [c.get("road_half_width", 1.0), c.get("road_linear_coeff", 1.0), c.get("road_quadratic_coeff", 10.0)]
        if self.cost == "circle_track":
            return [c.get("inner_radius", 1.875), c.get("outer_radius", 2.125), c.get("crash_cost", 1000.0),
                    c.get("speed_target", 2.0), c.get("speed_coeff", 2.0), c.get("angular_momentum_target", 4.0),
                    c.get("angular_momentum_coeff", 2.0)]
        if self.cost == "diff_drive_nav":
            return [c.get("goal_x", 2.0), c.get("goal_y", 2.0), c.get("goal_yaw", 0.0), c.get("dist_coeff", 5.0),
                    c.get("yaw_coeff", 5.0), c.get("obstacle_cost", 20.0)]
        return []

    def effective_costmap(self) -> Optional[Costmap]:
        if self.cost != "diff_drive_nav":
            return None
        if self.costmap is not None:
            return self.costmap
        c = self.cost_params  # make_cost all-free map (costs.cpp:137-140)
        return Costmap.empty(c.get("map_width", 11.0), c.get("map_height", 11.0), c.get("map_resolution", 0.1),
                             c.get("map_origin_x", -5.5), c.get("map_origin_y", -5.5))

    def to_problem(self, shard: Optional[tuple] = None) -> SmpcProblem:
        n_x, n_u, n_y = self.dims
        p = SmpcProblem()
        p.abi_version = ABI_VERSION
        p.num_samples = int(self.num_samples)
        p.horizon = int(self.horizon)
        p.iterations = int(self.iterations)
        p.dt = float(self.dt)
        p.lambda_ = float(self.lambda_)
        p.seed = int(self.rng_seed) & 0xFFFFFFFFFFFFFFFF
        std = list(self.control_std)
        p.n_control_std = len(std)
        for i, v in enumerate(std):
            p.control_std[i] = float(v)
        keep = []
        if self.std_per_step:
            arr = np.ascontiguousarray(np.asarray(self.std_per_step, np.float32).reshape(self.horizon, n_u))
            keep.append(arr)
            p.std_per_step = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        p.zero_mean_fraction = float(self.zero_mean_fraction)
        p.include_mean_sample = int(bool(self.include_mean_sample))
        p.importance_sampling = int(bool(self.importance_sampling))
        p.controller_kind = CONTROLLER_KINDS[self.controller]
        steps = self.step_sizes()
        if steps:
            sarr = np.ascontiguousarray(np.asarray(steps, np.float32))
            keep.append(sarr)
            p.n_step_sizes = len(steps)
            p.step_sizes = sarr.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        p.nominal_reset_bound = float(self.nominal_reset_bound)
        p.elite_fraction = float(self.elite_fraction)
        if self.feedback_gain is not None:
            kg = np.ascontiguousarray(np.asarray(self.feedback_gain, np.float32).reshape(n_u, n_x))
            keep.append(kg)
            p.feedback_gain = kg.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        p.cost_threshold = float(self.cost_threshold)
        p.num_candidates = int(self.num_candidates)
        p.dynamics_kind = DYNAMICS_KINDS[self.dynamics]
        if self.dynamics == "mlp":
            wb = np.ascontiguousarray(self.mlp_weights if self.mlp_weights is not None else autorally_mlp_weights(),
                                      np.float32).ravel()
            keep.append(wb)
            p.dyn_tensor = wb.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
            p.dyn_tensor_len = wb.size
        dp = self._dyn_params()
        p.n_dyn_params = len(dp)
        for i, v in enumerate(dp):
            p.dyn_params[i] = float(v)
        p.cost_kind = COST_KINDS.get(self.cost, 0)
        cp = self._cost_params()
        p.n_cost_params = len(cp)
        for i, v in enumerate(cp):
            p.cost_params[i] = float(v)
        if self.cost == "quadratic":
            w = list(self.weights or [])
            t = list(self.target or [0.0] * len(w))
            p.n_quad = len(w)
            for i in range(len(w)):
                p.quad_weights[i] = float(w[i])
                p.quad_target[i] = float(t[i])
        cm = self.effective_costmap()
        if cm is not None:
            g = np.ascontiguousarray(cm.grid.astype(np.uint8))
            keep.append(g)
            p.costmap = g.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
            p.costmap_cells_y, p.costmap_cells_x = g.shape
            p.costmap_resolution = float(cm.resolution)
            p.costmap_origin_x = float(cm.origin_x)
            p.costmap_origin_y = float(cm.origin_y)
        p.device = int(self.device)
        if shard is not None:
            p.shard_begin, p.shard_end = int(shard[0]), int(shard[1])
        p.update_skip_mass = float(self.update_skip_mass)
        p._keepalive = keep  # arrays must outlive the struct
        return p

    def to_json(self) -> str:
        """The reference's scenario JSON (scenario.cpp:305-387 field names)."""
        d = {
            "dt": self.dt, "horizon": self.horizon, "num_samples": self.num_samples,
            "iterations": self.iterations, "lambda": self.lambda_, "control_std": list(self.control_std),
            "rng_seed": self.rng_seed,
            "sampler": {"zero_mean_fraction": self.zero_mean_fraction,
                        "include_mean_sample": self.include_mean_sample,
                        "importance_sampling": self.importance_sampling},
            "dynamics": {"kind": self.dynamics, **self.dynamics_params},
            "cost": {"kind": self.cost, **self.cost_params},
            "controller": {"kind": self.controller, "step_size": self.step_size,
                           "elite_fraction": self.elite_fraction},
            "initial_state": self.initial_state,
        }
        if self.std_per_step:
            d["sampler"]["std_per_step"] = [list(r) for r in self.std_per_step]
        if self.cost == "quadratic":
            d["cost"]["weights"] = list(self.weights or [])
            d["cost"]["target"] = list(self.target or [])
        if self.step_size_per_step:
            d["controller"]["step_size_per_step"] = list(self.step_size_per_step)
        return json.dumps(d)


def shard_range(num_samples: int, rank: int, world: int) -> tuple:
    """WorkerPool chunk rule (worker_pool.hpp:28-29): [i*n/W, (i+1)*n/W)."""
    return (rank * num_samples // world, (rank + 1) * num_samples // world)


# ---- the BASELINE.json configs as scenarios ---------------------------------

def cartpole_scenario(num_samples: int = 2048, horizon: int = 100, seed: int = 1) -> Scenario:
    """C1: cartpole + quadratic swing-up target."""
    return Scenario(num_samples=num_samples, horizon=horizon, dt=0.02, lambda_=1.0, control_std=(1.0,),
                    rng_seed=seed, dynamics="cartpole", cost="quadratic",
                    target=[0.0, 0.0, math.pi, 0.0], weights=[1.0, 0.1, 10.0, 0.1])


def di_swarm_scenario(num_samples: int = 1 << 20, horizon: int = 100, seed: int = 7) -> Scenario:
    """C5: double integrator + circle track, importance off."""
    return Scenario(num_samples=num_samples, horizon=horizon, dt=0.02, lambda_=1.0, control_std=(1.0, 1.0),
                    rng_seed=seed, importance_sampling=False, dynamics="double_integrator",
                    cost="circle_track", initial_state={"X": 2.0, "V_Y": 2.0})


def bicycle_nav_scenario(num_samples: int = 2000, horizon: int = 56, seed: int = 42,
                         costmap: Optional[Costmap] = None) -> Scenario:
    """C3: kinematic bicycle / Ackermann vehicle on the synthetic 11 m x 11 m
    costmap with the diff_drive_nav cost (BASELINE.json configs[2], the Nav2
    comparison workload; builder-defined model, see models.cuh:BicycleDyn)."""
    return Scenario(num_samples=num_samples, horizon=horizon, dt=0.02, lambda_=1.0, control_std=(0.2, 0.3),
                    rng_seed=seed, dynamics="bicycle", cost="diff_drive_nav",
                    costmap=costmap if costmap is not None else synthetic_costmap(),
                    initial_state={"X": -2.0, "Y": -2.0})


def quadrotor_scenario(num_samples: int = 8192, horizon: int = 100, seed: int = 13) -> Scenario:
    """C2: 13-state quadrotor, quadratic tracking of the hover point (1, 1, 1)
    from hover at the origin (BASELINE.json configs[1]; builder-defined model,
    see models.cuh:QuadrotorDyn). Control = (body-rate commands, thrust offset
    from hover), so the zero mean is hover."""
    target = [1.0, 1.0, 1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0]
    weights = [10.0, 10.0, 10.0, 1.0, 1.0, 1.0, 5.0, 5.0, 5.0, 5.0, 0.1, 0.1, 0.1]
    return Scenario(num_samples=num_samples, horizon=horizon, dt=0.02, lambda_=1.0,
                    control_std=(0.5, 0.5, 0.5, 2.0), rng_seed=seed, dynamics="quadrotor", cost="quadratic",
                    target=target, weights=weights, initial_state={"QW": 1.0})


MLP_LAYOUT = dict(W1=(32, 6), b1=(32,), W2=(32, 32), b2=(32,), W3=(4, 32), b3=(4,))


def autorally_mlp_weights(seed: int = 0) -> np.ndarray:
    """Random-init AutoRally-style dynamics network 6-32-32-4 (tanh), flattened
    in the SMPC_DYN_MLP blob order W1 b1 W2 b2 W3 b3 (1412 floats). Synthetic
    (no checkpoint is available offline): fan-in scaled Gaussian weights, the
    output layer scaled so accelerations stay O(1) over a 2 s horizon."""
    rng = np.random.default_rng(seed)
    parts = []
    for name, shape in MLP_LAYOUT.items():
        fan_in = shape[1] if len(shape) == 2 else 1
        if name.startswith("W"):
            scale = (0.5 if name == "W3" else 1.0) / math.sqrt(fan_in)
            parts.append(rng.standard_normal(shape) * scale)
        else:
            parts.append(rng.standard_normal(shape) * 0.1)
    return np.concatenate([q.ravel() for q in parts]).astype(np.float32)


def autorally_scenario(num_samples: int = 8192, horizon: int = 100, seed: int = 21, controller: str = "mppi",
                       weights_seed: int = 0) -> Scenario:
    """C4: AutoRally-style neural dynamics (tcgen05 rollout), quadratic cost on
    lateral offset / heading / a 4 m/s forward-speed target (BASELINE.json
    configs[3]; builder-defined model). controller="tube" gives the dual
    nominal/real rollout."""
    return Scenario(num_samples=num_samples, horizon=horizon, dt=0.02, lambda_=1.0, control_std=(0.3, 0.3),
                    rng_seed=seed, dynamics="mlp", cost="quadratic",
                    target=[0.0, 0.0, 0.0, 0.0, 4.0, 0.0, 0.0], weights=[0.0, 0.5, 1.0, 0.1, 1.0, 0.1, 0.1],
                    mlp_weights=autorally_mlp_weights(weights_seed), controller=controller,
                    initial_state={"V_X": 2.0})


def default_timing_scenario(num_samples: int = 1024, seed: int = 0) -> Scenario:
    """bench.cpp:178-185, the reference's own timing subject (the paper's
    protocol): diff-drive + diff_drive_nav on the default
    all-free 11 m x 11 m map at 0.1 m, ScenarioConfig defaults otherwise
    (T = 100, dt = 0.02, lambda = 1, sigma = 0.2), starting at (-2, -2)."""
    return Scenario(num_samples=num_samples, rng_seed=seed, dynamics="diff_drive", cost="diff_drive_nav",
                    controller="mppi", initial_state={"X": -2.0, "Y": -2.0})


def default_sweep_scenario() -> Scenario:
    """bench.cpp:186-202: the point mass holding an annular orbit, the stock
    subject of the closed-loop step-size sweep (dmd controller)."""
    return Scenario(dt=0.02, horizon=32, lambda_=1.0, control_std=(1.0, 1.0), importance_sampling=False,
                    dynamics="double_integrator", cost="circle_track", controller="dmd", step_size=1.0,
                    replan_rate=50.0, dt_min=0.02, initial_state={"X": 2.0, "V_Y": 2.0})


def synthetic_costmap(seed: int = 3) -> Costmap:
    """11 m x 11 m @ 0.1 m map with seed-derived boxes (paper protocol)."""
    rng = np.random.default_rng(seed)
    cm = Costmap.empty(11.0, 11.0, 0.1, -5.5, -5.5)
    for _ in range(12):
        cx, cy = rng.uniform(-4.5, 4.5, 2)
        hw, hh = rng.uniform(0.2, 0.6, 2)
        if math.hypot(cx + 2, cy + 2) < 1.0 or math.hypot(cx - 2, cy - 2) < 1.0:
            continue  # keep start and goal free
        cm.fill_rect(cx - hw, cy - hh, cx + hw, cy + hh)
    return cm


def diff_drive_nav_scenario(num_samples: int = 2000, horizon: int = 56, seed: int = 42,
                            costmap: Optional[Costmap] = None) -> Scenario:
    """C3 stand-in: diff-drive + nav costmap, sigma 0.2."""
    return Scenario(num_samples=num_samples, horizon=horizon, dt=0.02, lambda_=1.0, control_std=(0.2, 0.2),
                    rng_seed=seed, dynamics="diff_drive", cost="diff_drive_nav",
                    costmap=costmap if costmap is not None else synthetic_costmap(),
                    initial_state={"X": -2.0, "Y": -2.0})
