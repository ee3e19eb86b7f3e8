set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -30
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 600 python bench.py --grid 128 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -5
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -5
