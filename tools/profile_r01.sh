#!/bin/bash
# Round-1 profiling recipe (run under gpurun on one B200):
#  1) per-launch device times of one short bench run (cold, serialised by ncu)
#  2) one `ncu --set full` capture of the rollout / weights / update kernels.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --roofline-steps 2 --e2e-steps 3"
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"rollout_kernel|weights_kernel|update_kernel" -s 9 -c 3 -o gpurun_out/prof_r01 $B > gpurun_out/prof_r01.log 2>&1
ls -la gpurun_out
