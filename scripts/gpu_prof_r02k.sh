# Round-2 final profiles (tensor-core sparse kernels behind the standalone apply and b = 32, split blocks):
# GPU suite, smoke, default bench line, per-config lines, the bench launch list (ncu) and one
# ncu --set full capture of the D stream, the sparse step and the two reduces; sBHA / BMDS times.
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02k
O=gpurun_out/r02k
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
(time timeout 2400 python -m pytest tests/ -q -m gpu) > $O/tests.log 2>&1; tail -4 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
head -c 400 $O/bench.json; echo
timeout 600 python bench.py --mode apply --config 4 --no-cpu-baseline > $O/apply4.json 2>&1; echo rc=$?
timeout 900 python bench.py --config 3 --no-e2e --no-cpu-baseline > $O/cfg3.json 2>&1; echo rc=$?
timeout 600 python bench.py --mode apply --config 3 --b 32 --no-cpu-baseline > $O/apply3.json 2>&1; echo rc=$?
for k in 8 16 64; do for b in 1 4 16 64; do
  timeout 600 python bench.py --mode apply --config 5 --k5 $k --b $b > $O/cfg5_k${k}_b${b}.json 2>&1; echo cfg5 k=$k b=$b rc=$?
done; done
timeout 900 python scripts/time_next.py > $O/next.json 2>&1; echo next rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo launches rc=$?
python scripts/launch_shares.py $O/launches.csv > $O/launch_shares.txt 2>&1; head -12 $O/launch_shares.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_dstream_sym8|k_sp8_step|k_blk_reduce_fold|k_dreduce_y2d" -s 8 -c 4 -o $O/prof_eigs python scripts/eigs_once.py 4 6 > $O/ncu_full.log 2>&1
echo full rc=$?
