# Re-entry check at HEAD (session 4): full GPU suite, smoke, default bench line
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
(time timeout 2700 python -m pytest tests/ -q -m gpu) > gpurun_out/r02j_tests.log 2>&1; tail -15 gpurun_out/r02j_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err; echo bench rc=$?
head -c 1500 gpurun_out/bench_r02j.json; echo
