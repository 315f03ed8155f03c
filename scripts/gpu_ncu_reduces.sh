# ncu --set full of the two cooperative per-iteration reduces (config 4, eigs)
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
python scripts/eigs_once.py 4 6 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_blk_reduce_fold|k_dreduce_y2d" -s 6 -c 2 -o gpurun_out/prof_reduces2 python scripts/eigs_once.py 4 6 > gpurun_out/ncu_reduces.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu_reduces.log
