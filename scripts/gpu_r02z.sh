# eigs at b = 32 through two 16-column passes of the tensor-core sparse step: parity, config-3 line
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02z
O=gpurun_out/r02z
(timeout 1800 python -m pytest tests/test_gpu_eigs.py tests/test_gpu_configs.py -q -m gpu -x -k "b32 or config3 or fused_sparse") > $O/tests.log 2>&1; tail -12 $O/tests.log
timeout 900 python bench.py --config 3 --no-e2e --no-cpu-baseline > $O/cfg3.json 2> $O/cfg3.err; echo rc=$?; head -c 500 $O/cfg3.json; echo
timeout 600 python scripts/family_times.py 3 > $O/family3.json 2>&1; head -c 700 $O/family3.json
