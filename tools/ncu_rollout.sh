#!/bin/bash
# ncu --set full of the DI rollout + update kernels (one launch each) + SASS source page.
mkdir -p gpurun_out
TAG=${1:-cur}
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --roofline-steps 1 --e2e-steps 3"
ncu --set full --clock-control none --import-source on -k regex:"rollout_kernel|update_kernel" -s 2 -c 2 -o gpurun_out/prof_$TAG $B > gpurun_out/prof_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass -k regex:rollout_kernel > gpurun_out/src_$TAG.csv 2>/dev/null
ls -la gpurun_out | tail -5
