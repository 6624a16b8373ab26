#!/bin/bash
# Per-round evidence (run under gpurun on one B200): the default bench line,
# the per-launch device times of a short bench run (ncu launch list, cold and
# serialised) and one `ncu --set full` capture of the C5 rollout / weights /
# update kernels, plus the SASS opcode mix of the rollout.
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; tail -1 gpurun_out/bench_$TAG.log > gpurun_out/bench_$TAG.json
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --roofline-steps 2 --e2e-steps 3"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv $B > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt
ncu --set full --clock-control none --import-source on -k regex:"rollout_kernel|weights_kernel|update_kernel" -s 14 -c 3 \
  -o gpurun_out/prof_$TAG $B > gpurun_out/prof_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass -k regex:rollout_kernel > gpurun_out/src_$TAG.csv 2>/dev/null
python tools/sass_hot.py gpurun_out/src_$TAG.csv > gpurun_out/mix_$TAG.txt 2>/dev/null
cat gpurun_out/bench_$TAG.json; tail -12 gpurun_out/launches_$TAG.txt
