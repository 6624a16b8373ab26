#!/bin/bash
# A/B: bench the in-tree library and each build/libsmpc_b200_*.so variant.
for lib in paper_2409_07563_b200/libsmpc_b200.so $(ls build/libsmpc_b200_*.so 2>/dev/null); do
  SMPC_B200_LIB=$lib timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-sweep ${BENCH_ARGS} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$lib', 'ms/iter %.4f'%d['ms_per_step'], 'e2e ms %.4f'%d['e2e']['ms_per_step'], 'rollout ms %.4f'%d['roofline']['kernel_ms'], 'frac %.3f'%d['roofline']['frac'])"
done
