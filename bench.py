#!/usr/bin/env python3
"""MPPI iteration benchmark (BASELINE.json metric: ms per MPPI iteration and
rollout samples/s vs N at T=100, 1/2/4/8 B200).

A step = one MppiController::compute_control with I = 1 (controllers.cpp:
113-135): Philox noise -> fused rollout -> softmin weights -> weighted update
-> nominal rollout, on synthetic initial states. Default workload: BASELINE
config C5, the double-integrator swarm + circle-track cost at N = 2^20
samples, T = 100 (the large-sample sweep config the metric is quoted on for
1/2/4/8 GPUs; strong scaling: the 2^20 samples are sharded over the ranks
with the WorkerPool chunk rule).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload di|cartpole|diffdrive|quadrotor|autorally|bicycle] [--samples N]
                  [--scaling strong|weak]

Rank 0 prints ONE JSON line. `value` = samples/s of the whole job from
device-resident graph replays (CUDA events on the context stream, L2 flushed
between steps, max over ranks); `e2e` = the same metric through the public
C-ABI call `smpc_compute_control` with host x0 in and the host solution out.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2409_07563_b200 import scenario as S  # noqa: E402

# Algorithmic work per sample-step (reference-semantic
# op counts; FP32 add/sub/mul/div/compare, noise generated in-kernel).
# quadrotor (builder-defined): noise 4x29, control 4, clamp 8,
# derivative 49, Euler 26, quaternion normalisation 11 (+1 sqrt); FP64:
# quadratic cost 13x4 + total 1 + importance 4x3.
# autorally (C4, Tube S=2; per system-sample-step): SIMT layers 1 and 3 =
# (6x32 + 32x4) MACs = 640 FP32 ops + 64 tanh, noise 2x29, kinematics 6,
# Euler 14; tensor layer 2 = 32x32 MACs = 2048 flops (3xTF32 issues 3x that).
# bicycle (C3, Ackermann): noise 58, control+clamp 6, derivative 5 (+4 sin/cos),
# Euler 6, wrap 2, nav cost 16.
FP32_OPS_PER_SAMPLE_STEP = {"di": 83, "cartpole": 56, "diffdrive": 90, "quadrotor": 214, "autorally": 718,
                            "bicycle": 93}
FP64_OPS_PER_SAMPLE_STEP = {"di": 9, "cartpole": 23, "diffdrive": 19, "quadrotor": 65, "autorally": 41,
                            "bicycle": 19}
TENSOR_FLOPS_PER_SAMPLE_STEP = {"autorally": 2048}
# workloads whose model exists in the reference (oracle/_ref can time them)
REFERENCE_WORKLOADS = ("di", "cartpole", "diffdrive")


def make_scenario(workload: str, n: int) -> S.Scenario:
    if workload == "di":
        return S.di_swarm_scenario(num_samples=n, horizon=100, seed=7)
    if workload == "cartpole":
        return S.cartpole_scenario(num_samples=n, horizon=100, seed=1)
    if workload == "diffdrive":
        return S.diff_drive_nav_scenario(num_samples=n, horizon=56, seed=42)
    if workload == "quadrotor":
        return S.quadrotor_scenario(num_samples=n, horizon=100, seed=13)
    if workload == "bicycle":
        return S.bicycle_nav_scenario(num_samples=n, horizon=56, seed=42)
    if workload == "autorally":
        return S.autorally_scenario(num_samples=n, horizon=100, seed=21, controller="tube")
    raise SystemExit(f"unknown workload {workload}")


def workload_name(workload: str, n: int) -> str:
    return {"di": f"C5 double_integrator+circle_track MPPI N={n} T=100",
            "cartpole": f"C1 cartpole+quadratic MPPI N={n} T=100",
            "diffdrive": f"C3 diff_drive+diff_drive_nav(costmap 110x110) MPPI N={n} T=56",
            "quadrotor": f"C2 quadrotor(13-state)+quadratic tracking MPPI N={n} T=100",
            "autorally": f"C4 AutoRally MLP dynamics (tcgen05) Tube-MPPI N={n} T=100",
            "bicycle": f"C3 Ackermann/bicycle+diff_drive_nav(costmap 110x110) MPPI N={n} T=56"}[workload]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return rank, world, local, dist
    return 0, 1, 0, None


def barrier(dist, local):
    if dist is not None:
        import torch
        dist.barrier(device_ids=[local])
        torch.cuda.synchronize()


def max_over_ranks(dist, value: float) -> float:
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_reference_run(sc, steps: int, warmup: int, budget_s: float, prefer_ref: bool = True):
    """Time the reference's own compute_control on the host cores.

    oracle/_ref (the unmodified reference, compiled here) with all host
    threads when present; else the C restatement (single thread)."""
    from oracle import bindings
    ncores = os.cpu_count() or 1
    if prefer_ref and bindings.ref_available():
        ctl = bindings.OracleController(sc, "reference", workers=ncores, strategy=1)
        kind, cores = "reference", ncores
    else:
        ctl = bindings.OracleController(sc, "port")
        kind, cores = "port", 1
    x0 = sc.x0()
    for _ in range(warmup):
        ctl.compute_control(x0)
    times = []
    t_start = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        ctl.compute_control(x0)
        times.append((time.perf_counter() - t0) * 1e3)
        if time.perf_counter() - t_start > budget_s and len(times) >= 3:
            break
    ms = statistics.mean(times)
    return {"kind": kind, "cores": cores, "ms": ms, "n": len(times),
            "value": sc.num_samples * 1000.0 / ms}


def run_reference_arm(args):
    rank, world, local, dist = init_dist()
    if rank != 0:
        return
    sc = make_scenario(args.workload, args.samples)
    r = cpu_reference_run(sc, args.steps, args.warmup, budget_s=args.ref_budget,
                          prefer_ref=args.workload in REFERENCE_WORKLOADS)
    line = {
        "metric": "rollout samples/s per MPPI iteration (compute_control, I=1)",
        "value": r["value"], "unit": "samples/s", "n_gpus": world, "steps": r["n"], "warmup": args.warmup,
        "ms_per_step": r["ms"], "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32+f64", "data": "synthetic (seeded Philox noise, fixed x0)",
        "config": {"workload": workload_name(args.workload, args.samples), "samples": args.samples,
                   "horizon": sc.horizon, "iterations": 1},
        "impl": "reference",
        "cpu_baseline": {"value": r["value"], "unit": "samples/s", "cores": r["cores"], "kind": r["kind"],
                         "sample": f"{r['n']} compute_control solves after {args.warmup} warm-ups, full N"},
        "e2e": {"value": r["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def load_traffic(workload: str, samples: int):
    """dram bytes per rollout launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{workload}:{samples}")
    except (OSError, ValueError):
        return None


def run_ours(args):
    import torch
    rank, world, local, dist = init_dist()
    from paper_2409_07563_b200 import _lib
    from paper_2409_07563_b200.controllers import make_controller

    device = local
    torch.cuda.set_device(device)
    n_global = args.samples * (world if args.scaling == "weak" else 1)
    sc = make_scenario(args.workload, n_global)
    sc.device = device
    shard = S.shard_range(n_global, rank, world)
    ctl = make_controller(sc, shard=shard)
    if world > 1:
        uid = bytes(128)
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            _lib.check(_lib.load().smpc_comm_unique_id(buf))
            uid = buf.raw
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ctl.comm_init(obj[0], rank, world)
    x0 = sc.x0()
    stream = torch.cuda.ExternalStream(ctl.stream, device=torch.device("cuda", device))
    # L2 flush buffer (> 126 MB L2): written between timed steps, outside the events.
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{device}")

    ctl.set_x0(x0)
    for _ in range(args.warmup):
        ctl.launch_iteration()
    ctl.synchronize()
    barrier(dist, local)

    # ---- timed region: device-resident graph replays --------------------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(device) as clocks:
        torch.cuda.synchronize()
        barrier(dist, local)
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(k & 0xFF)
                starts[k].record(stream)
            ctl.launch_iteration()
            ends[k].record(stream)
        ctl.synchronize()
        torch.cuda.synchronize()
        barrier(dist, local)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = max_over_ranks(dist, float(sum(step_ms)))
    ms_per_step = total_ms / args.steps
    value = n_global * 1000.0 / ms_per_step
    launches = ctl.kernels_per_solve * args.steps

    # ---- roofline: rollout kernel alone (CUDA events around each launch) -----
    ctl.rollout_timing(True)
    for k in range(args.roofline_steps):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        ctl.launch_iteration()
        ctl.synchronize()
    roll_ms_total, roll_n = ctl.rollout_timing(False)
    roll_ms = roll_ms_total / max(roll_n, 1)
    systems = 2 if sc.controller == "tube" else 1
    ops_per_launch = (shard[1] - shard[0]) * sc.horizon * systems * FP32_OPS_PER_SAMPLE_STEP[args.workload]
    peak = ctypes.c_double()
    _lib.load().smpc_measure_fp32_peak(device, ctypes.byref(peak))
    achieved = ops_per_launch / (roll_ms * 1e-3) / 1e12
    roofline = {"bound": "fp32", "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                "frac": achieved / peak.value if peak.value else None,
                "traffic": load_traffic(args.workload, n_global),
                "kernel": "rollout_kernel", "kernel_ms": roll_ms,
                "kernel_share_of_step": roll_ms / ms_per_step,
                "peak_source": "measured in-run: FADD/FMUL issue-rate probe (no FMA: reference semantics)",
                "algorithmic": f"{FP32_OPS_PER_SAMPLE_STEP[args.workload]} FP32 ops + "
                               f"{FP64_OPS_PER_SAMPLE_STEP[args.workload]} FP64 ops per sample-step "
                               f"x {shard[1] - shard[0]} samples x {sc.horizon} steps per launch",
                "hbm_peak_gbs_measured": None}
    if args.workload in TENSOR_FLOPS_PER_SAMPLE_STEP:
        # tcgen05 layer: algorithmic TF32 flops / rollout time vs the dense TF32 peak
        # (half the measured bf16 peak in MEASURED_PEAKS.json; B200_PROFILING.md fallback 1125 TF/s)
        tf = (shard[1] - shard[0]) * sc.horizon * systems * TENSOR_FLOPS_PER_SAMPLE_STEP[args.workload]
        bf16 = None
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                bf16 = json.load(f).get("bf16_tflops")
        except (OSError, ValueError):
            pass
        tpeak = bf16 / 2 if bf16 else 1125.0
        roofline["tensor"] = {"achieved": tf / (roll_ms * 1e-3) / 1e12, "peak": tpeak, "unit": "TFLOP/s (tf32)",
                              "frac": tf / (roll_ms * 1e-3) / 1e12 / tpeak,
                              "algorithmic": f"{TENSOR_FLOPS_PER_SAMPLE_STEP[args.workload]} flops per sample-step "
                                             "(32x32 layer; 3xTF32 issues 3 MMAs per product)"}

    # ---- e2e: public C-ABI call with host buffers (H2D x0, D2H solution) -----
    barrier(dist, local)
    e2e_steps = max(3, min(args.steps, args.e2e_steps))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ctl.compute_control(x0)
    e2e_s = max_over_ranks(dist, time.perf_counter() - t0)
    e2e_ms = e2e_s * 1e3 / e2e_steps
    n_x, n_u, n_y = sc.dims
    d2h = systems * 4 * (sc.horizon * n_u + (sc.horizon + 1) * n_x + sc.horizon * n_y) + 128
    e2e = {"value": n_global * 1000.0 / e2e_ms, "unit": "samples/s", "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": 4 * n_x, "d2h_bytes_per_step": d2h,
           "api": "smpc_compute_control (MppiController::compute_control)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference_run(sc, steps=args.cpu_steps, warmup=1, budget_s=args.cpu_budget,
                              prefer_ref=args.workload in REFERENCE_WORKLOADS)
        cpu = {"value": r["value"], "unit": "samples/s", "cores": r["cores"], "kind": r["kind"],
               "ms_per_step": r["ms"],
               "sample": f"{r['n']} full-size compute_control solves (N={n_global}) after 1 warm-up"}

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": "rollout samples/s per MPPI iteration (compute_control, I=1)",
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32+f64",
            "data": "synthetic (seeded Philox noise regenerated in-kernel, fixed x0)",
            "config": {"workload": workload_name(args.workload, n_global), "samples": n_global,
                       "samples_per_gpu": shard[1] - shard[0], "horizon": sc.horizon, "iterations": 1,
                       "parallelism": f"sample-shard dp{world}",
                       "l2": "flushed between timed steps (256 MiB write, outside the events)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": {"sm_mhz": clk["sm_mhz"], "sm_max_mhz": clk["sm_max_mhz"], "reasons": clk["reasons"]},
            "p50_ms": statistics.median(step_ms), "p99_ms": float(np.percentile(step_ms, 99)),
        }
        print(json.dumps(line), flush=True)
    ctl.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="di", choices=["di", "cartpole", "diffdrive", "quadrotor", "autorally",
                                                           "bicycle"])
    ap.add_argument("--samples", type=int, default=1 << 20)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--roofline-steps", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--cpu-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=120.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
