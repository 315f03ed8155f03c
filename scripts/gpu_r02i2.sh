# Philox init with four normals per call, wider final rotate: eigs parity, bench, launch list
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02i2
O=gpurun_out/r02i2
(timeout 2400 python -m pytest tests/test_gpu_eigs.py tests/test_gpu_shard.py tests/test_gpu_bmds.py tests/test_gpu_configs.py -q -m gpu -x) > $O/tests.log 2>&1; tail -4 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo rc=$?; head -c 330 $O/bench.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo launches rc=$?
python scripts/launch_shares.py $O/launches.csv > $O/launch_shares.txt 2>&1; grep -n "philox\|rotate\|gram_tc\|argmax\|k_rr\|csc_vec4" $O/launch_shares.txt
