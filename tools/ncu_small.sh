#!/bin/bash
# ncu --set full of the small-N (cartpole N=2048) rollout and update kernels.
mkdir -p gpurun_out
TAG=${1:-small}
B="python bench.py --workload cartpole --samples 2048 --steps 3 --warmup 20 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 3"
ncu --set full --clock-control none --import-source on -k regex:"update_kernel|rollout_kernel|weights_kernel|gen_zq" -s 80 -c 4 \
  -o gpurun_out/prof_$TAG $B > gpurun_out/prof_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass -k regex:update_kernel > gpurun_out/src_upd_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass -k regex:rollout_kernel > gpurun_out/src_roll_$TAG.csv 2>/dev/null
