#!/bin/bash
# Parity tests + one bench line per workload (no CPU baseline).
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for w in "di" "cartpole --samples 8192" "cartpole --samples 2048" "diffdrive --samples 2000" "di --samples 65536"; do
  timeout 300 python bench.py --workload $w --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['config']['workload'], 'ms/iter %.4f'%d['ms_per_step'], 'samples/s %.3g'%d['value'], 'e2e ms %.4f'%d['e2e']['ms_per_step'], 'rollout ms %.4f'%d['roofline']['kernel_ms'], 'frac %.3f'%d['roofline']['frac'])"
done
