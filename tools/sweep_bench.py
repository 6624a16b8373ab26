#!/usr/bin/env python3
"""Closed-loop step-size sweep (bench_dmd_sweep, bench.cpp:86-133) on the GPU:
the reference acceptance grid (samples 64..4096 x gamma 0.2..1.0 x 50 trials
x 1000 steps) by default. Prints one JSON line: wall time, per-cell records,
best gamma per sample count, and the acceptance predicate of
check_step_size_sweep (acceptance_main.cpp:277-311). --cpu-cells times the
reference's own closed loop (oracle/_ref Plant) on a few trials for scale."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2409_07563_b200 import plant as P  # noqa: E402
from paper_2409_07563_b200 import scenario as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", default="64,256,1024,4096")
    ap.add_argument("--gammas", default="0.2,0.4,0.6,0.8,1.0")
    ap.add_argument("--trials", type=int, default=50)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--cpu-trials", type=int, default=0, help="reference loops to time (M=max samples, gamma=1)")
    args = ap.parse_args()
    samples = [int(v) for v in args.samples.split(",")]
    gammas = [float(v) for v in args.gammas.split(",")]
    base = S.default_sweep_scenario()
    t0 = time.perf_counter()
    recs = P.bench_dmd_sweep(base, samples, gammas, trials=args.trials, steps=args.steps)
    wall = time.perf_counter() - t0
    best = dict(P.best_gamma_per_samples(recs))
    mean_at = {(r.samples, r.gamma): r.mean_cost for r in recs}
    ok = (best.get(max(samples)) == 1.0 and best.get(min(samples), 1.0) < 1.0
          and mean_at[(max(samples), 1.0)] < mean_at[(min(samples), 1.0)]) if 1.0 in gammas else None
    line = {"gpu_wall_s": wall, "cells": len(recs), "loops": len(recs) * args.trials,
            "solves": len(recs) * args.trials * args.steps, "best_gamma": best, "acceptance_step_size_sweep": ok,
            "records": [vars(r) for r in recs]}
    if args.cpu_trials:
        from oracle import bindings as B
        import dataclasses
        run = dataclasses.replace(base, num_samples=max(samples), controller="dmd", step_size=1.0)
        t1 = time.perf_counter()
        for t in range(args.cpu_trials):
            B.reference_control_loop(dataclasses.replace(run, rng_seed=t), args.steps * base.dt, workers=os.cpu_count())
        cpu = (time.perf_counter() - t1) / args.cpu_trials
        line["cpu_reference_s_per_loop"] = {"samples": max(samples), "steps": args.steps, "s": cpu,
                                            "workers": os.cpu_count()}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
