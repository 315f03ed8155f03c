# 9 x 1 tile blocks in the int8 D stream: parity (apply, shard, eigs, configs), bench, D-stream ncu
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02h2
O=gpurun_out/r02h2
(timeout 2400 python -m pytest tests/test_gpu_apply.py tests/test_gpu_shard.py tests/test_gpu_eigs.py tests/test_gpu_configs.py tests/test_gpu_precision.py -q -m gpu -x) > $O/tests.log 2>&1; tail -5 $O/tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo rc=$?; head -c 330 $O/bench.json; echo
python scripts/eigs_once.py 4 6 && timeout 900 ncu --set full --clock-control none -k regex:"k_dstream_sym8|k_dreduce_y2d" -s 4 -c 2 -o $O/prof_d python scripts/eigs_once.py 4 6 > $O/ncu.log 2>&1; echo ncu rc=$?
