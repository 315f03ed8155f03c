# Re-entry check at HEAD: GPU suite, smoke, default bench line.
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02k
O=gpurun_out/r02k
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
(time timeout 2400 python -m pytest tests/ -q -m gpu) > $O/tests.log 2>&1; tail -4 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
head -c 600 $O/bench.json; echo
