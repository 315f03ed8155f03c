# variable-size blocks (split where a dictionary exceeds an image): parity, config-3 lines
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02y
O=gpurun_out/r02y
(timeout 1800 python -m pytest tests/test_gpu_apply.py tests/test_gpu_configs.py tests/test_gpu_eigs.py -q -m gpu -x -k "tensor_core or config3 or config4 or int8_gram or deferred or split") > $O/tests.log 2>&1; tail -12 $O/tests.log
python scripts/cfg3_sp8_state.py 3 2>&1 | tail -9
timeout 600 python bench.py --mode apply --config 3 --b 32 --no-cpu-baseline > $O/apply3.json 2> $O/apply3.err; echo rc=$?; head -c 900 $O/apply3.json; echo
timeout 600 python bench.py --mode apply --config 4 --no-cpu-baseline > $O/apply4.json 2> $O/apply4.err; echo rc=$?; head -c 300 $O/apply4.json; echo
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo rc=$?; head -c 300 $O/bench.json; echo
