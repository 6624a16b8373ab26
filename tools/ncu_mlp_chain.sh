#!/bin/bash
# ncu --set full (with source) of the RMPPI+MLP update kernel (its tail runs the
# warp-cooperative nominal MLP chain) and the candidate-scoring kernel.
mkdir -p gpurun_out
B="python bench.py --workload autorally_rmppi --samples 8192 --steps 3 --warmup 10 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"update_kernel|rmppi_select" -s 10 -c 2 -o gpurun_out/prof_mc $B > gpurun_out/prof_mc.log 2>&1
ncu -i gpurun_out/prof_mc.ncu-rep --page source --csv --print-source sass -k regex:update_kernel > gpurun_out/src_mc_upd.csv 2>/dev/null
ncu -i gpurun_out/prof_mc.ncu-rep --page source --csv --print-source sass -k regex:rmppi_select > gpurun_out/src_mc_sel.csv 2>/dev/null
python tools/sass_hot.py gpurun_out/src_mc_upd.csv > gpurun_out/sass_mc_upd.txt 2>/dev/null
python tools/sass_hot.py gpurun_out/src_mc_sel.csv > gpurun_out/sass_mc_sel.txt 2>/dev/null
gzip -f gpurun_out/src_mc_upd.csv gpurun_out/src_mc_sel.csv
rm -f gpurun_out/prof_mc.ncu-rep
