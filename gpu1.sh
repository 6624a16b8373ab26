set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30
timeout 300 python bench.py --steps 50 --warmup 5 --cpu-steps 3 --cpu-budget 10 2>&1 | tail -3
