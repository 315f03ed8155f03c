# Round-1 profiles after the tensor-core sparse step: bench launch list (ncu, cold-cache
# serialised per-launch times) and one ncu --set full capture of k_sp8_step at config 4.
set -x
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_c.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
python scripts/eigs_once.py 4 6 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sp8_step -s 2 -c 1 -o gpurun_out/prof_sp8c python scripts/eigs_once.py 4 6 > gpurun_out/ncu_sp8c.log 2>&1
echo full rc=$?
