export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sbha.py -q -x -s > gpurun_out/r02f_full.log 2>&1; tail -60 gpurun_out/r02f_full.log
