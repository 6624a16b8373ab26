#!/bin/bash
# Per-round evidence (one B200, under gpurun):
#  1. the default bench line (C5 headline + sweep + CPU reference)
#  2. ncu launch list of the C5 bench at steady state (160 solves in)
#  3. ncu --set full of a converged C5 rollout / weights / update launch,
#     the SASS opcode mix of the rollout
#  4. ncu --set full of the small-N (cartpole 2048) rollout / update, the
#     injected-noise (TMA) rollout and the tcgen05 MLP rollout
TAG=${1:-r2}
mkdir -p gpurun_out/$TAG
O=gpurun_out/$TAG
timeout 900 python bench.py > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
B="python bench.py --steps 10 --warmup 150 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 3"
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file $O/launches.csv $B > /dev/null 2>&1
python tools/launch_table.py $O/launches.csv > $O/launches.txt
ncu --set full --clock-control none --import-source on -k regex:"update_kernel|weights_kernel|rollout_kernel" -s 480 -c 3 \
  -o $O/prof_c5 $B > $O/prof_c5.log 2>&1
ncu -i $O/prof_c5.ncu-rep --page raw --csv > $O/raw_c5.csv 2>/dev/null
python tools/ncu_summary.py $O/raw_c5.csv > $O/ncu_c5_summary.json
ncu -i $O/prof_c5.ncu-rep --page source --csv --print-source sass -k regex:rollout_kernel > $O/src_roll_c5.csv 2>/dev/null
python tools/sass_hot.py $O/src_roll_c5.csv > $O/rollout_c5_sass_mix.txt 2>/dev/null
S="python bench.py --workload cartpole --samples 2048 --steps 3 --warmup 20 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 3"
ncu --set full --clock-control none -k regex:"update_kernel|rollout_kernel|gen_zq|weights_kernel" -s 80 -c 4 -o $O/prof_small $S > $O/prof_small.log 2>&1
ncu -i $O/prof_small.ncu-rep --page raw --csv > $O/raw_small.csv 2>/dev/null
python tools/ncu_summary.py $O/raw_small.csv > $O/ncu_small_summary.json
cat > $O/inj.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from bench import make_scenario
from paper_2409_07563_b200.controllers import make_controller
sc = make_scenario("di", 1 << 20); ctl = make_controller(sc)
eps = torch.randn(1 << 20, 100, 2, device="cuda"); ctl.set_injected_noise(eps.data_ptr())
for _ in range(4): ctl.compute_control(sc.x0())
PY
ncu --set full --clock-control none -k regex:"rollout_kernel|update_kernel" -s 4 -c 2 -o $O/prof_inj python $O/inj.py > $O/prof_inj.log 2>&1
ncu -i $O/prof_inj.ncu-rep --page raw --csv > $O/raw_inj.csv 2>/dev/null
python tools/ncu_summary.py $O/raw_inj.csv > $O/ncu_injected_summary.json
M="python bench.py --workload autorally --samples 262144 --steps 3 --warmup 5 --no-cpu-baseline --no-sweep --roofline-steps 1 --e2e-steps 3"
ncu --set full --clock-control none -k regex:"mlp_rollout" -s 3 -c 1 -o $O/prof_mlp $M > $O/prof_mlp.log 2>&1
ncu -i $O/prof_mlp.ncu-rep --page raw --csv > $O/raw_mlp.csv 2>/dev/null
python tools/ncu_summary.py $O/raw_mlp.csv > $O/ncu_mlp_summary.json
rm -f $O/*.ncu-rep.tmp
tail -12 $O/launches.txt
# keep the pull-back under gpurun's 64 MiB: reports and per-line exports stay on the box
rm -f $O/*.ncu-rep $O/src_*.csv $O/launches.csv
du -sh $O
