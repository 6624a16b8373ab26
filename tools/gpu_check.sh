#!/bin/bash
# Quick GPU loop: parity tests, one bench line, per-launch times.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 300 python bench.py --steps 100 --warmup 5 --cpu-steps 2 --cpu-budget 5 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --roofline-steps 2 --e2e-steps 3 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches.csv | tail -25
