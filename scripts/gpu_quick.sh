export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
python scripts/profile_breakdown.py --config 4 --eigs 2>&1 | tail -2
