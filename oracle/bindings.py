"""ctypes bindings for the parity checkers. TEST INFRASTRUCTURE ONLY.

Two checkers with one Python surface:
  * ``Oracle("port")``      — oracle/liboracle.so, the plain-C restatement;
  * ``Oracle("reference")`` — oracle/_ref/libsmpc_ref.so, the unmodified
    reference library (+ ref_capi.cpp shim), when it was built here.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arms import this module; the product path never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

from paper_2409_07563_b200.scenario import (Scenario, SmpcProblem, SmpcWeightSummary)

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libsmpc_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    pass


class _OracleErr(ctypes.Structure):
    _fields_ = [("message", ctypes.c_char * 256), ("sample", ctypes.c_int64),
                ("timestep", ctypes.c_int32), ("channel", ctypes.c_int32)]


def build(quiet: bool = True) -> None:
    """make -C oracle (liboracle.so always; _ref only with /root/reference)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/core/src"):
        targets.append("ref")
    out = subprocess.run(["make", "-C", HERE, "-j8", *targets], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-2000:] + out.stderr[-4000:])


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


class Oracle:
    """Uniform numpy API over the C restatement ("port") or the reference ("reference")."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise OracleError(f"{path} not built (run oracle.bindings.build())")
        self.lib = ctypes.CDLL(path)
        L = self.lib
        if kind == "port":
            L.oracle_philox.argtypes = [_u32p, _u32p, _u32p]
            L.oracle_quad.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _f32p]
            L.oracle_icdf_domain.argtypes = [_f32p]
            L.oracle_generate_samples.argtypes = [ctypes.POINTER(SmpcProblem), _f32p, ctypes.c_int64, ctypes.c_int64,
                                                  ctypes.c_uint32, _f32p, ctypes.c_void_p, ctypes.POINTER(_OracleErr)]
            L.oracle_importance.argtypes = [ctypes.POINTER(SmpcProblem), _f32p, ctypes.c_int64, _f32p, _f64p]
            L.oracle_rollout.argtypes = [ctypes.POINTER(SmpcProblem), ctypes.c_int32, _f32p, _f32p, _f32p,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, _f64p, ctypes.c_void_p,
                                         ctypes.POINTER(_OracleErr)]
            L.oracle_compute_weights.argtypes = [_f64p, ctypes.c_int64, ctypes.c_double, _f64p,
                                                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                                 ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_OracleErr)]
            L.oracle_weighted_update.argtypes = [_f32p, ctypes.c_int32, ctypes.c_int32, _f32p, ctypes.c_int64, _f64p,
                                                 ctypes.c_void_p, ctypes.c_int32, _f32p, ctypes.POINTER(_OracleErr)]
            L.oracle_compute_control.argtypes = [ctypes.POINTER(SmpcProblem), _f32p, ctypes.POINTER(ctypes.c_uint64),
                                                 _f32p, _f32p, _f32p, _f32p, ctypes.c_void_p,
                                                 ctypes.POINTER(SmpcWeightSummary), ctypes.POINTER(_OracleErr)]
            L.oracle_partial_sort.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64,
                                              np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")]
            L.oracle_clamp_control.argtypes = [ctypes.POINTER(SmpcProblem), _f32p, _f32p]
            L.oracle_rmppi_compute_control.argtypes = [
                ctypes.POINTER(SmpcProblem), _f32p, _f32p, ctypes.POINTER(ctypes.c_int32),
                ctypes.POINTER(ctypes.c_uint64), _f32p, _f32p, _f32p, _f32p, _f32p, ctypes.POINTER(ctypes.c_int32),
                ctypes.POINTER(SmpcWeightSummary), ctypes.POINTER(_OracleErr)]
            L.oracle_wrap_angle.argtypes = [ctypes.c_float]
            L.oracle_wrap_angle.restype = ctypes.c_float
            L.oracle_angular_channel.argtypes = [ctypes.POINTER(SmpcProblem)]
            L.oracle_running_cost.argtypes = [ctypes.POINTER(SmpcProblem), _f32p]
            L.oracle_running_cost.restype = ctypes.c_double
            L.oracle_terminal_cost.argtypes = [ctypes.POINTER(SmpcProblem), _f32p]
            L.oracle_terminal_cost.restype = ctypes.c_double
            L.oracle_step.argtypes = [ctypes.POINTER(SmpcProblem), _f32p, _f32p, ctypes.c_float, _f32p, _f32p,
                                      ctypes.POINTER(_OracleErr)]
            L.oracle_tube_compute_control.argtypes = [
                ctypes.POINTER(SmpcProblem), _f32p, _f32p, _f32p, ctypes.POINTER(ctypes.c_int32),
                ctypes.POINTER(ctypes.c_uint64), _f32p, _f32p, _f32p, _f32p, _f32p,
                ctypes.POINTER(SmpcWeightSummary), ctypes.POINTER(SmpcWeightSummary), ctypes.POINTER(_OracleErr)]
        else:
            E = [ctypes.c_char_p, ctypes.c_size_t]
            L.ref_philox.argtypes = [_u32p, _u32p, _u32p]
            L.ref_quad.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _f32p]
            L.ref_generate_samples.argtypes = [ctypes.POINTER(SmpcProblem), _f32p, ctypes.c_uint32, ctypes.c_int,
                                               _f32p, ctypes.c_void_p, *E]
            L.ref_rollout.argtypes = [ctypes.POINTER(SmpcProblem), ctypes.c_int, _f32p, _f32p, _f32p, ctypes.c_int,
                                      ctypes.c_int, _f64p, ctypes.c_void_p, *E]
            L.ref_compute_weights.argtypes = [_f64p, ctypes.c_int64, ctypes.c_double, _f64p,
                                              ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), *E]
            L.ref_controller_create.argtypes = [ctypes.POINTER(SmpcProblem), ctypes.c_int, ctypes.c_int, *E]
            L.ref_controller_create.restype = ctypes.c_void_p
            L.ref_controller_destroy.argtypes = [ctypes.c_void_p]
            L.ref_set_mean.argtypes = [ctypes.c_void_p, _f32p]
            L.ref_get_mean.argtypes = [ctypes.c_void_p, _f32p]
            L.ref_shift_control_sequence.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, *E]
            L.ref_compute_control.argtypes = [ctypes.c_void_p, _f32p, _f32p, _f32p, _f32p, ctypes.c_void_p, _f64p, *E]
            L.ref_run_control_loop.argtypes = [ctypes.POINTER(SmpcProblem), ctypes.c_double, ctypes.c_double,
                                               ctypes.c_double, _f32p, ctypes.c_double, ctypes.c_int,
                                               ctypes.POINTER(ctypes.c_double), ctypes.c_void_p,
                                               ctypes.POINTER(ctypes.c_int64), *E]
            L.ref_tube_compute_control.argtypes = [ctypes.c_void_p, _f32p, _f32p, _f32p, _f64p, _f32p, _f32p, _f64p,
                                                   _f32p, *E]

    # ---- rng -----------------------------------------------------------------
    def philox(self, ctr, key) -> np.ndarray:
        out = np.zeros(4, np.uint32)
        fn = self.lib.oracle_philox if self.kind == "port" else self.lib.ref_philox
        fn(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
        return out

    def quad(self, seed: int, a: int, b: int, c: int) -> np.ndarray:
        out = np.zeros(4, np.float32)
        fn = self.lib.oracle_quad if self.kind == "port" else self.lib.ref_quad
        fn(seed, a, b, c, out)
        return out

    def icdf_domain(self) -> np.ndarray:
        out = np.zeros(1 << 23, np.float32)
        self.lib.oracle_icdf_domain(out)
        return out

    # ---- plugins ----------------------------------------------------------------
    def running_cost(self, sc: Scenario, y) -> float:
        p = sc.to_problem()
        return self.lib.oracle_running_cost(ctypes.byref(p), np.ascontiguousarray(y, np.float32))

    def terminal_cost(self, sc: Scenario, y) -> float:
        p = sc.to_problem()
        return self.lib.oracle_terminal_cost(ctypes.byref(p), np.ascontiguousarray(y, np.float32))

    def step(self, sc: Scenario, x, u, dt: float):
        n_x, n_u, n_y = sc.dims
        p = sc.to_problem()
        xn = np.zeros(n_x, np.float32)
        y = np.zeros(n_y, np.float32)
        err = _OracleErr()
        rc = self.lib.oracle_step(ctypes.byref(p), np.ascontiguousarray(x, np.float32),
                                  np.ascontiguousarray(u, np.float32), dt, xn, y, ctypes.byref(err))
        self._check(rc, err.message)
        return xn, y

    # ---- sampler / engine ----------------------------------------------------
    def generate_samples(self, sc: Scenario, mean: np.ndarray, stream: int, m_begin: int = 0,
                         m_end: Optional[int] = None, workers: int = 1):
        n_x, n_u, n_y = sc.dims
        M, T = sc.num_samples, sc.horizon
        m_end = M if m_end is None else m_end
        mean = np.ascontiguousarray(mean, np.float32).reshape(T * n_u)
        p = sc.to_problem()
        if self.kind == "port":
            eps = np.zeros((m_end - m_begin) * T * n_u, np.float32)
            flags = np.zeros(m_end - m_begin, np.uint8)
            err = _OracleErr()
            rc = self.lib.oracle_generate_samples(ctypes.byref(p), mean, m_begin, m_end, stream, eps,
                                                  flags.ctypes.data, ctypes.byref(err))
            self._check(rc, err.message)
        else:
            eps = np.zeros(M * T * n_u, np.float32)
            flags = np.zeros(M, np.uint8)
            buf = ctypes.create_string_buffer(512)
            rc = self.lib.ref_generate_samples(ctypes.byref(p), mean, stream, workers, eps, flags.ctypes.data, buf, 512)
            self._check(rc, buf.value)
            eps = eps.reshape(M, T * n_u)[m_begin:m_end].ravel().copy()
            flags = flags[m_begin:m_end].copy()
        return eps.reshape(m_end - m_begin, T, n_u), flags

    def rollout(self, sc: Scenario, x0s: np.ndarray, means: np.ndarray, eps: np.ndarray,
                outputs: bool = False, strategy: int = 1, workers: int = 1):
        """costs [S, M] (importance term included when enabled) [, outputs [S, M, T, n_y]]."""
        n_x, n_u, n_y = sc.dims
        T = sc.horizon
        x0s = np.ascontiguousarray(x0s, np.float32).reshape(-1)
        S = x0s.size // n_x
        means = np.ascontiguousarray(means, np.float32).reshape(S * T * n_u)
        eps = np.ascontiguousarray(eps, np.float32).reshape(-1)
        M = eps.size // (T * n_u)
        costs = np.zeros(S * M, np.float64)
        outs = np.zeros(S * M * T * n_y, np.float32) if outputs else None
        p = sc.to_problem()
        if self.kind == "port":
            adj = None
            if sc.importance_sampling:
                adj = np.zeros(S * M, np.float64)
                for s in range(S):
                    a = np.zeros(M, np.float64)
                    self.lib.oracle_importance(ctypes.byref(p), eps, M, np.ascontiguousarray(means[s * T * n_u:(s + 1) * T * n_u]), a)
                    adj[s * M:(s + 1) * M] = a
            err = _OracleErr()
            rc = self.lib.oracle_rollout(ctypes.byref(p), S, x0s, means, eps, 0, M,
                                         adj.ctypes.data if adj is not None else None, costs,
                                         outs.ctypes.data if outs is not None else None, ctypes.byref(err))
            self._check(rc, err.message, err)
        else:
            p.num_samples = M
            buf = ctypes.create_string_buffer(512)
            rc = self.lib.ref_rollout(ctypes.byref(p), S, x0s, means, eps, 0 if outputs else strategy, workers, costs,
                                      outs.ctypes.data if outs is not None else None, buf, 512)
            self._check(rc, buf.value)
        costs = costs.reshape(S, M)
        if outputs:
            return costs, outs.reshape(S, M, T, n_y)
        return costs

    def compute_weights(self, costs: np.ndarray, lam: float):
        costs = np.ascontiguousarray(costs, np.float64)
        w = np.zeros_like(costs)
        rho, eta = ctypes.c_double(), ctypes.c_double()
        if self.kind == "port":
            am = ctypes.c_int64()
            err = _OracleErr()
            rc = self.lib.oracle_compute_weights(costs, costs.size, lam, w, ctypes.byref(rho), ctypes.byref(eta),
                                                 ctypes.byref(am), ctypes.byref(err))
            self._check(rc, err.message)
            return w, rho.value, eta.value, am.value
        buf = ctypes.create_string_buffer(512)
        rc = self.lib.ref_compute_weights(costs, costs.size, lam, w, ctypes.byref(rho), ctypes.byref(eta), buf, 512)
        self._check(rc, buf.value)
        return w, rho.value, eta.value, int(np.argmin(costs))

    def partial_sort(self, costs, k: int) -> np.ndarray:
        """First k of std::partial_sort with CemController's comparator (controllers.cpp:165-171)."""
        costs = np.ascontiguousarray(costs, np.float64)
        out = np.zeros(k, np.int64)
        self.lib.oracle_partial_sort(costs, costs.size, k, out)
        return out

    def weighted_update(self, mean, eps, weights, step_sizes=()):
        T, n_u = mean.shape
        out = np.zeros(T * n_u, np.float32)
        steps = np.ascontiguousarray(step_sizes, np.float32)
        err = _OracleErr()
        rc = self.lib.oracle_weighted_update(np.ascontiguousarray(mean, np.float32).ravel(), T, n_u,
                                             np.ascontiguousarray(eps, np.float32).ravel(), len(weights),
                                             np.ascontiguousarray(weights, np.float64),
                                             steps.ctypes.data if steps.size else None, steps.size, out,
                                             ctypes.byref(err))
        self._check(rc, err.message)
        return out.reshape(T, n_u)

    @staticmethod
    def _check(rc, msg, err=None):
        if rc != 0:
            m = msg.decode() if isinstance(msg, bytes) else str(msg)
            raise OracleError(m)


class OracleController:
    """MppiController / TubeMppiController on a checker (stateful warm start)."""

    def __init__(self, sc: Scenario, kind: str = "port", workers: int = 1, strategy: int = 1):
        self.sc = sc
        self.o = Oracle(kind)
        self.kind = kind
        n_x, n_u, n_y = sc.dims
        self.mean = np.zeros(sc.horizon * n_u, np.float32)
        self.real_mean = np.zeros(sc.horizon * n_u, np.float32)
        self.nominal_state = np.zeros(n_x, np.float32)
        self.nominal_started = ctypes.c_int32(0)
        self.solve_count = ctypes.c_uint64(0)
        self.problem = sc.to_problem()
        self.handle = None
        if kind == "reference":
            buf = ctypes.create_string_buffer(512)
            self.handle = self.o.lib.ref_controller_create(ctypes.byref(self.problem), workers, strategy, buf, 512)
            if not self.handle:
                raise OracleError(buf.value.decode())

    def __del__(self):
        if getattr(self, "handle", None):
            self.o.lib.ref_controller_destroy(self.handle)
            self.handle = None

    def set_mean(self, mean):
        self.mean[:] = np.asarray(mean, np.float32).ravel()
        if self.handle:
            self.o.lib.ref_set_mean(self.handle, self.mean)

    def compute_control(self, x0, want_weights: bool = False):
        sc = self.sc
        n_x, n_u, n_y = sc.dims
        T, M = sc.horizon, sc.num_samples
        x0 = np.ascontiguousarray(x0, np.float32)
        controls = np.zeros(T * n_u, np.float32)
        states = np.zeros((T + 1) * n_x, np.float32)
        outputs = np.zeros(T * n_y, np.float32)
        weights = np.zeros(M, np.float64) if want_weights else None
        if self.kind == "port":
            sm = SmpcWeightSummary()
            err = _OracleErr()
            rc = self.o.lib.oracle_compute_control(ctypes.byref(self.problem), self.mean, ctypes.byref(self.solve_count),
                                                   x0, controls, states, outputs,
                                                   weights.ctypes.data if weights is not None else None,
                                                   ctypes.byref(sm), ctypes.byref(err))
            Oracle._check(rc, err.message)
            summary = dict(baseline=sm.baseline, normalizer=sm.normalizer, argmin=sm.argmin, nonzero=sm.nonzero)
        else:
            s4 = np.zeros(4, np.float64)
            buf = ctypes.create_string_buffer(512)
            w = weights if weights is not None else np.zeros(M, np.float64)
            rc = self.o.lib.ref_compute_control(self.handle, x0, controls, states, outputs, w.ctypes.data, s4, buf, 512)
            Oracle._check(rc, buf.value)
            self.o.lib.ref_get_mean(self.handle, self.mean)
            # the shim derives argmin from the first maximum weight: not the argmin for CEM's flat 1/k weights
            argmin = -1 if sc.controller == "cem" else int(s4[2])
            summary = dict(baseline=s4[0], normalizer=s4[1], argmin=argmin, nonzero=int(np.count_nonzero(w)),
                           solve_time_ms=s4[3])
        return dict(controls=controls.reshape(T, n_u), states=states.reshape(T + 1, n_x),
                    outputs=outputs.reshape(T, n_y), weights=weights, **summary)

    def rmppi_compute_control(self, x_real):
        """Builder-defined RMPPI solve on the C oracle (port only)."""
        sc = self.sc
        n_x, n_u, n_y = sc.dims
        T = sc.horizon
        x_real = np.ascontiguousarray(x_real, np.float32)
        ctl = np.zeros(T * n_u, np.float32)
        ns = np.zeros((T + 1) * n_x, np.float32)
        rs = np.zeros((T + 1) * n_x, np.float32)
        chosen = np.zeros(n_x, np.float32)
        choice = ctypes.c_int32()
        sm = SmpcWeightSummary()
        err = _OracleErr()
        rc = self.o.lib.oracle_rmppi_compute_control(
            ctypes.byref(self.problem), self.mean, self.nominal_state, ctypes.byref(self.nominal_started),
            ctypes.byref(self.solve_count), x_real, ctl, ns, rs, chosen, ctypes.byref(choice), ctypes.byref(sm),
            ctypes.byref(err))
        Oracle._check(rc, err.message)
        return dict(controls=ctl.reshape(T, n_u), nominal_states=ns.reshape(T + 1, n_x),
                    real_states=rs.reshape(T + 1, n_x), nominal_state=chosen, choice=choice.value,
                    baseline=sm.baseline, normalizer=sm.normalizer, argmin=sm.argmin)

    def tube_compute_control(self, x_real):
        sc = self.sc
        n_x, n_u, n_y = sc.dims
        T = sc.horizon
        x_real = np.ascontiguousarray(x_real, np.float32)
        nc = np.zeros(T * n_u, np.float32)
        ns = np.zeros((T + 1) * n_x, np.float32)
        rcn = np.zeros(T * n_u, np.float32)
        rs = np.zeros((T + 1) * n_x, np.float32)
        nominal_state_used = np.zeros(n_x, np.float32)
        if self.kind == "port":
            smn, smr = SmpcWeightSummary(), SmpcWeightSummary()
            err = _OracleErr()
            rc = self.o.lib.oracle_tube_compute_control(
                ctypes.byref(self.problem), self.mean, self.real_mean, self.nominal_state,
                ctypes.byref(self.nominal_started), ctypes.byref(self.solve_count), x_real, nc, ns, rcn, rs,
                ctypes.byref(smn), ctypes.byref(smr), ctypes.byref(err))
            Oracle._check(rc, err.message)
            nominal_state_used = ns[:n_x].copy()
            sn = dict(baseline=smn.baseline, normalizer=smn.normalizer, argmin=smn.argmin)
            sr = dict(baseline=smr.baseline, normalizer=smr.normalizer, argmin=smr.argmin)
        else:
            s4n, s4r = np.zeros(4), np.zeros(4)
            buf = ctypes.create_string_buffer(512)
            rc = self.o.lib.ref_tube_compute_control(self.handle, x_real, nc, ns, s4n, rcn, rs, s4r,
                                                     nominal_state_used, buf, 512)
            Oracle._check(rc, buf.value)
            sn = dict(baseline=s4n[0], normalizer=s4n[1], argmin=int(s4n[2]))
            sr = dict(baseline=s4r[0], normalizer=s4r[1], argmin=int(s4r[2]))
        return dict(nominal_controls=nc.reshape(T, n_u), nominal_states=ns.reshape(T + 1, n_x),
                    real_controls=rcn.reshape(T, n_u), real_states=rs.reshape(T + 1, n_x),
                    nominal_state=nominal_state_used, nominal=sn, real=sr)


def shift_mean(mean: np.ndarray, T: int, n_u: int, dt: float, elapsed_s: float, dt_min: float) -> np.ndarray:
    """Controller::shift_control_sequence (controllers.cpp:68-84) on a flat mean."""
    if elapsed_s <= 0.0:
        return mean
    quantized = float(np.rint(elapsed_s / dt_min)) * dt_min
    steps = int(np.rint(quantized / dt))
    if steps <= 0:
        return mean
    m = mean.reshape(T, n_u)
    if steps >= T:
        return np.zeros_like(mean)
    out = np.concatenate([m[steps:], np.repeat(m[T - 1:T], steps, axis=0)])
    return np.ascontiguousarray(out.ravel(), np.float32)


def control_loop(sc: Scenario, duration_s: float, kind: str = "port", workers: int = 1):
    """Plant::run_control_loop (plant.cpp:133-181) with SimulatedSystem::step
    (plant.cpp:31-48) on a checker controller, in Python around the C oracle
    (kind "port") or the reference controller (kind "reference"). Returns
    (accumulated_cost, rows[steps, 2 + n_x + n_u] = {t, x, u_applied, c})."""
    port = Oracle("port")
    ctl = OracleController(sc, kind, workers=workers)
    n_x, n_u, n_y = sc.dims
    T, dt = sc.horizon, sc.dt
    p = sc.to_problem()
    steps = int(round(duration_s / dt))
    interval = 1.0 / sc.replan_rate
    sim_seed = (int(sc.rng_seed) ^ 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    scale = np.float32(sc.disturbance_std * np.sqrt(dt))
    ang = port.lib.oracle_angular_channel(ctypes.byref(p))
    x = np.ascontiguousarray(sc.x0(), np.float32)
    next_replan_t, solution_t, solved_once = 0.0, 0.0, False
    sol = None
    rows = np.zeros((steps, 2 + n_x + n_u))
    acc = 0.0
    for step in range(steps):
        t = step * dt
        if not solved_once or t >= next_replan_t - 1e-9:
            if solved_once:
                if kind == "reference":
                    buf = ctypes.create_string_buffer(512)
                    ctl.o.lib.ref_shift_control_sequence(ctl.handle, t - solution_t, sc.dt_min, buf, 512)
                else:
                    ctl.set_mean(shift_mean(ctl.mean, T, n_u, dt, t - solution_t, sc.dt_min))
            sol = ctl.compute_control(x)
            solution_t, solved_once = t, True
            while next_replan_t <= t + 1e-9:
                next_replan_t += interval
        idx = min(max(int(np.floor((t - solution_t) / dt)), 0), T - 1)
        u = np.ascontiguousarray(sol["controls"][idx], np.float32)
        uc = np.zeros(n_u, np.float32)
        port.lib.oracle_clamp_control(ctypes.byref(p), u, uc)
        c = port.running_cost(sc, x)
        rows[step] = np.concatenate([[t], x, uc, [c]])
        acc += c
        xn, _ = port.step(sc, x, uc, np.float32(dt))
        if scale > 0:
            for ch in range(n_x):
                z = port.quad(sim_seed, step & 0xFFFFFFFF, ch // 4, 0)[ch % 4]
                xn[ch] = np.float32(xn[ch] + np.float32(scale * z))
            if ang >= 0:
                xn[ang] = port.lib.oracle_wrap_angle(float(xn[ang]))
        x = xn
    return acc, rows


def reference_control_loop(sc: Scenario, duration_s: float, workers: int = 1):
    """The reference's own Plant::run_control_loop (oracle/_ref). Same return as control_loop."""
    o = Oracle("reference")
    n_x, n_u, _ = sc.dims
    steps = int(round(duration_s / sc.dt))
    rows = np.zeros((steps, 2 + n_x + n_u))
    acc, n = ctypes.c_double(), ctypes.c_int64()
    buf = ctypes.create_string_buffer(512)
    p = sc.to_problem()
    rc = o.lib.ref_run_control_loop(ctypes.byref(p), sc.replan_rate, sc.dt_min, sc.disturbance_std,
                                    np.ascontiguousarray(sc.x0(), np.float32), duration_s, workers, ctypes.byref(acc),
                                    rows.ctypes.data, ctypes.byref(n), buf, 512)
    Oracle._check(rc, buf.value)
    return acc.value, rows[:n.value]
