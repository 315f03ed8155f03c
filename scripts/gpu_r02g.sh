# Round 2 measurement: full GPU suite, the default bench line, per-config lines (configs 3, 4
# apply, config 5 sweep), the round-2 additions' times.
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
(time timeout 2400 python -m pytest tests/ -q -m gpu) > gpurun_out/r02g_tests.log 2>&1; tail -5 gpurun_out/r02g_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err; echo bench rc=$?
cat gpurun_out/bench_r02g.json | head -c 600; echo
timeout 600 python bench.py --mode apply --config 4 --no-cpu-baseline > gpurun_out/bench_r02g_apply4.json 2>&1; echo rc=$?
timeout 900 python bench.py --config 3 --iters 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_r02g_cfg3.json 2>&1; echo rc=$?
timeout 600 python bench.py --mode apply --config 3 --b 32 --no-cpu-baseline > gpurun_out/bench_r02g_apply3.json 2>&1; echo rc=$?
for k in 8 16 64; do for b in 1 4 16 64; do
  timeout 600 python bench.py --mode apply --config 5 --k5 $k --b $b > gpurun_out/bench_r02g_cfg5_k${k}_b${b}.json 2>&1; echo cfg5 k=$k b=$b rc=$?
done; done
timeout 900 python scripts/time_next.py > gpurun_out/r02g_next.json 2>&1; echo next rc=$?
