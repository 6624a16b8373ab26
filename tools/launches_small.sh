#!/bin/bash
# Per-kernel device times (ncu launch list) of the small-N workloads.
mkdir -p gpurun_out
for w in "cartpole 2048" "quadrotor 8192" "paper 2048" "autorally_rmppi 8192"; do
  set -- $w
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$1_$2.csv \
    python bench.py --workload $1 --samples $2 --steps 20 --warmup 10 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 3 > /dev/null 2>&1
  echo "== $1 $2"; python tools/launch_table.py gpurun_out/launches_$1_$2.csv | tail -12
done
