#!/bin/bash
# Steady-state evidence for the C5 iteration (run under gpurun, one B200):
# the per-launch device times of 160 solves (ncu launch list, cold and
# serialised) and one `ncu --set full` capture of a converged update /
# weights launch (>= 150 solves in) plus one rollout launch.
TAG=${1:-steady}
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 150 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 3"
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_$TAG.csv $B > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt
ncu --set full --clock-control none --import-source on -k regex:"update_kernel|weights_kernel|rollout_kernel" -s 480 -c 3 \
  -o gpurun_out/prof_$TAG $B > gpurun_out/prof_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass -k regex:update_kernel > gpurun_out/src_upd_$TAG.csv 2>/dev/null
tail -30 gpurun_out/launches_$TAG.txt
