# Round 2: new parity tests (configs 3/4/5 vs oracle, precision contract, error statuses), then
# the whole GPU suite.
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_precision.py -q -x 2>&1 | tail -25
timeout 2400 python -m pytest tests/test_gpu_configs.py -q 2>&1 | tail -25
timeout 1500 python -m pytest tests/ -q -m gpu --deselect tests/test_gpu_configs.py --deselect tests/test_gpu_precision.py 2>&1 | tail -15
