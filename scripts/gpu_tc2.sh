export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
timeout 600 python -m pytest tests/test_gpu_apply.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python scripts/profile_breakdown.py --config 4 --eigs 2>&1 | tail -1
for b in 8 16 32 64; do timeout 120 python scripts/profile_breakdown.py --config 5 --k5 16 --b $b --applies 10 2>&1 | tail -1; done
