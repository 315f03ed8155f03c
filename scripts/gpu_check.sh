set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_apply.py -x -q 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_eigs.py -x -q 2>&1 | tail -30
