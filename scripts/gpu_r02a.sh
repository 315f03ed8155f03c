# Round-2 baseline: smoke, GPU suite, default bench line on the round-1 code.
set -x
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo bench rc=$?
cat gpurun_out/bench_r02a.json; tail -5 gpurun_out/bench_r02a.err
