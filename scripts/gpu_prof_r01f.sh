# Round-1 final profiles: default bench line, the bench launch list (ncu, cold-cache serialised
# per-launch times) and one ncu --set full capture each of the sparse step and the fold.
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r01f.json 2> gpurun_out/bench_r01f.err; echo bench rc=$?
cat gpurun_out/bench_r01f.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_f.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_f.log 2>&1
echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_blk_reduce_fold|k_sp8_step" -s 6 -c 2 -o gpurun_out/prof_f python scripts/eigs_once.py 4 6 > gpurun_out/ncu_f.log 2>&1
echo full rc=$?
