export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eigs.py -x -q 2>&1 | tail -6
timeout 600 python scripts/fuse_modes.py 4 3 2>&1 | tail -4
