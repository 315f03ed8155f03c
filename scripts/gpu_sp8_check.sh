export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_eigs.py -x -q -k "tensor_core_sparse_step and 2" 2>&1 | tail -15
timeout 600 python scripts/fuse_modes.py 2 1 3 2>&1 | tail -5
timeout 900 python scripts/fuse_modes.py 4 1 3 2>&1 | tail -5
