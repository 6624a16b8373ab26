#!/bin/bash
# Parity tests + short benches of the secondary workloads (one line each).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
for w in "quadrotor 8192" "cartpole 8192" "cartpole 2048" "diffdrive 2000" "bicycle 2000" "autorally 8192" "di 65536"; do
  set -- $w
  timeout 300 python bench.py --workload $1 --samples $2 --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
r=d['roofline']
print('%-10s N=%-8s ms/iter %.4f  e2e %.4f  rollout %.4f ms  frac %.3f' % ('$1', '$2', d['ms_per_step'], d['e2e']['ms_per_step'], r['kernel_ms'], r['frac']))"
done
