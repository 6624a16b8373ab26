#!/bin/bash
# C4 bench lines (Tube + MLP on tcgen05) at two sizes, and an ncu capture of the MLP rollout.
mkdir -p gpurun_out
for n in 8192 65536 262144; do
  timeout 300 python bench.py --workload autorally --samples $n --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_autorally_$n.json
  python -c "
import json; d=json.load(open('gpurun_out/bench_autorally_$n.json')); r=d['roofline']
print('autorally N=$n ms/iter %.4f rollout %.4f ms fp32 frac %.3f tensor %.1f TF/s frac %.4f' % (d['ms_per_step'], r['kernel_ms'], r['frac'], r['tensor']['achieved'], r['tensor']['frac']))"
done
ncu --set full --clock-control none --import-source on -k regex:"mlp_rollout_kernel" -s 2 -c 1 -o gpurun_out/prof_mlp \
  python bench.py --workload autorally --samples 65536 --steps 3 --warmup 2 --no-cpu-baseline --roofline-steps 1 --e2e-steps 3 > gpurun_out/prof_mlp.log 2>&1
ncu -i gpurun_out/prof_mlp.ncu-rep --page source --csv --print-source sass > gpurun_out/src_mlp.csv 2>/dev/null
ncu -i gpurun_out/prof_mlp.ncu-rep --page raw --csv > gpurun_out/raw_mlp.csv 2>/dev/null
python tools/sass_hot.py gpurun_out/src_mlp.csv | head -45
