#!/bin/bash
# ncu --set full (with source) of one steady-state update kernel launch
# (160 solves in: the converged weight distribution), plus the SASS mix and
# per-line stall attribution.
mkdir -p gpurun_out
TAG=${1:-upd}
B="python bench.py --steps 10 --warmup 170 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 3"
ncu --set full --clock-control none --import-source on -k regex:"update_kernel" -s 160 -c 1 -o gpurun_out/prof_$TAG $B > gpurun_out/prof_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
python tools/sass_hot.py gpurun_out/src_$TAG.csv > gpurun_out/sass_$TAG.txt 2>/dev/null
python tools/ncu_summary.py gpurun_out/raw_$TAG.csv > gpurun_out/ncu_$TAG.json
rm -f gpurun_out/prof_$TAG.ncu-rep
