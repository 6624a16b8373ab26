#!/bin/bash
# A/B of the library variants on the small-N workloads.
for w in "cartpole 2048" "quadrotor 8192" "paper 2048" "diffdrive 2000" "bicycle 2000"; do
  set -- $w
  BENCH_ARGS="--workload $1 --samples $2" bash tools/ab_bench.sh 2>/dev/null | sed "s/^/$1 $2 /"
done
