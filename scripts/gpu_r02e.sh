export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bmds.py tests/test_gpu_shard.py -q -x -s > gpurun_out/r02e_full.log 2>&1; tail -60 gpurun_out/r02e_full.log
