# b = 32 halves on the tensor-core sparse kernels: parity, config-3 apply line
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02x
O=gpurun_out/r02x
(timeout 1500 python -m pytest tests/test_gpu_apply.py tests/test_gpu_configs.py -q -m gpu -x -k "tensor_core or config3 or config4") > $O/tests.log 2>&1; tail -12 $O/tests.log
timeout 600 python bench.py --mode apply --config 3 --b 32 --no-cpu-baseline > $O/apply3.json 2> $O/apply3.err; echo rc=$?; head -c 700 $O/apply3.json; echo
timeout 600 python bench.py --mode apply --config 4 --no-cpu-baseline > $O/apply4.json 2> $O/apply4.err; echo rc=$?; head -c 400 $O/apply4.json; echo
timeout 600 python scripts/family_times.py 3 > $O/family3.json 2>&1; tail -c 700 $O/family3.json
