# standalone apply on the tensor-core sparse kernels: parity tests, apply bench lines
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02w
O=gpurun_out/r02w
(timeout 1500 python -m pytest tests/test_gpu_apply.py tests/test_gpu_precision.py -q -m gpu -x) > $O/tests.log 2>&1; tail -12 $O/tests.log
timeout 600 python bench.py --mode apply --config 4 --no-cpu-baseline > $O/apply4.json 2> $O/apply4.err; echo rc=$?; head -c 1500 $O/apply4.json; echo
timeout 600 python scripts/family_times.py 4 > $O/family4.json 2>&1; tail -c 1200 $O/family4.json
