#!/bin/bash
# ncu --set full of one steady-state (dense-weight) update kernel launch.
mkdir -p gpurun_out
TAG=${1:-upd}
B="python bench.py --steps 3 --warmup 14 --no-cpu-baseline --roofline-steps 1 --e2e-steps 3"
ncu --set full --clock-control none --import-source on -k regex:"update_kernel|weights_kernel" -s 24 -c 2 -o gpurun_out/prof_$TAG $B > gpurun_out/prof_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ls -la gpurun_out | tail -4
