#!/bin/bash
# Phase timing of the update kernel (main loop / last-CTA commit / finish) per
# workload. Requires an instrumented build in build/timing/ (globaltimer
# printf in the update kernel's tail; not part of the product build).
for w in "cartpole 2048" "quadrotor 8192" "paper 2048" "di 1048576" "autorally_rmppi 8192"; do
  set -- $w
  echo "== $1 $2"
  SMPC_B200_LIB=build/timing/libsmpc_b200.so timeout 300 python bench.py --workload $1 --samples $2 --steps 5 --warmup 40 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 1 2>&1 | grep UPDT | tail -3
done
