# Check at HEAD: GPU suite, smoke, default bench line, the config-5 sweep (standalone apply lines).
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
T=${1:-r02m}
mkdir -p gpurun_out/$T
O=gpurun_out/$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
(time timeout 2400 python -m pytest tests/ -q -m gpu) > $O/tests.log 2>&1; tail -4 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
head -c 300 $O/bench.json; echo
for k in 8 16 64; do for b in 1 4 16 64; do
  timeout 600 python bench.py --mode apply --config 5 --k5 $k --b $b > $O/cfg5_k${k}_b${b}.json 2>&1; echo cfg5 k=$k b=$b rc=$?
done; done
timeout 600 python bench.py --mode apply --config 4 --no-cpu-baseline > $O/apply4.json 2>&1; echo rc=$?
timeout 600 python bench.py --mode apply --config 3 --b 32 --no-cpu-baseline > $O/apply3.json 2>&1; echo rc=$?
