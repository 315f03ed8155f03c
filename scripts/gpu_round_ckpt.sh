export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks.csv &
CLK=$!
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
kill $CLK
cat gpurun_out/bench.json
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
python scripts/profile_breakdown.py --config 4 --quick && \
ncu --set full --clock-control none --import-source on -k regex:k_dstream_tc -s 2 -c 1 -o gpurun_out/prof_dstream_tc python scripts/profile_breakdown.py --config 4 --quick > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
