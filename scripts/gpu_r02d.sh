# Round 2: BMDS + sharded apply + precision tests, then the whole GPU suite.
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bmds.py tests/test_gpu_shard.py -q -s 2>&1 | tail -40
timeout 2400 python -m pytest tests/ -q -m gpu 2>&1 | tail -15
