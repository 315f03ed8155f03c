export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
timeout 900 python -m pytest tests/test_gpu_eigs.py tests/test_gpu_apply.py -x -q 2>&1 | tail -1
timeout 600 python scripts/sp8_tail.py 4 2>&1 | tail -3
timeout 600 python scripts/fuse_modes.py 4 3 2>&1 | tail -1
