#!/bin/bash
# ncu --set full (with source) of the quadrotor N=8192 rollout (small-N serial-chain regime).
mkdir -p gpurun_out
B="python bench.py --workload quadrotor --samples 8192 --steps 3 --warmup 20 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"rollout_kernel" -s 20 -c 1 -o gpurun_out/prof_quad $B > gpurun_out/prof_quad.log 2>&1
ncu -i gpurun_out/prof_quad.ncu-rep --page source --csv --print-source sass > gpurun_out/src_quad.csv 2>/dev/null
ncu -i gpurun_out/prof_quad.ncu-rep --page raw --csv > gpurun_out/raw_quad.csv 2>/dev/null
python tools/sass_hot.py gpurun_out/src_quad.csv > gpurun_out/sass_quad.txt 2>/dev/null
python tools/ncu_summary.py gpurun_out/raw_quad.csv > gpurun_out/ncu_quad.json
gzip -f gpurun_out/src_quad.csv
rm -f gpurun_out/prof_quad.ncu-rep
