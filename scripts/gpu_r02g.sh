# one readback for the X and Y1 checks: apply tests, apply lines at configs 3 and 4
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02g2
O=gpurun_out/r02g2
(timeout 1500 python -m pytest tests/test_gpu_apply.py tests/test_gpu_precision.py tests/test_gpu_shard.py -q -m gpu -x) > $O/tests.log 2>&1; tail -5 $O/tests.log
for i in 1 2; do timeout 600 python bench.py --mode apply --config 3 --b 32 --no-cpu-baseline > $O/apply3_$i.json 2> $O/apply3.err; echo rc=$?; head -c 330 $O/apply3_$i.json | tail -c 120; echo; done
timeout 600 python bench.py --mode apply --config 4 --no-cpu-baseline > $O/apply4.json 2> $O/apply4.err; echo rc=$?; head -c 330 $O/apply4.json | tail -c 120; echo
