# sparse-step iteration: eigs tests, mode timings, a normal-step timeline
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eigs.py tests/test_gpu_configs.py -q -x > gpurun_out/sp8_iter_tests.log 2>&1; grep -E "passed|failed|Error" gpurun_out/sp8_iter_tests.log | tail -3
timeout 300 python scripts/sp8_modes.py 4 2>&1 | grep sp8_dbg
timeout 300 python scripts/sp8_timeline.py 26 2>&1 | tail -50 > gpurun_out/tl26.txt; sed -n '1,4p;20,24p;48,50p' gpurun_out/tl26.txt
