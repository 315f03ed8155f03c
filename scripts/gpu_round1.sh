set -x
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
(time python -c "from gen import configs; configs.config(4)") 2>&1 | tail -4
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err; echo rc=$?
cat gpurun_out/bench_r01a.json; tail -5 gpurun_out/bench_r01a.err
