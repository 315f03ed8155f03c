# k_gram_tc with staged rows: eigs parity (every path that runs the Gram kernel), config-3 line
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/gram
O=gpurun_out/gram
(timeout 2400 python -m pytest tests/test_gpu_eigs.py tests/test_gpu_configs.py tests/test_gpu_bmds.py tests/test_gpu_shard.py -q -m gpu -x) > $O/tests.log 2>&1; tail -5 $O/tests.log
timeout 900 python bench.py --config 3 --no-e2e --no-cpu-baseline > $O/cfg3.json 2> $O/cfg3.err; echo rc=$?; head -c 300 $O/cfg3.json; echo
timeout 600 python scripts/family_times.py 3 > $O/family3.json 2>&1; head -c 420 $O/family3.json; echo
