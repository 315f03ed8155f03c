export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_eigs.py -x -q 2>&1 | tail -2
for b in 3 4 3 4; do echo "bps $b"; SBMDS_FOLD_BPS=$b timeout 600 python scripts/fuse_modes.py 4 3 2>&1 | tail -1; done
