# Round 2: precision contract + sharded apply tests, then the whole GPU suite.
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precision.py tests/test_gpu_shard.py -q -x -s 2>&1 | tail -30
timeout 2400 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
