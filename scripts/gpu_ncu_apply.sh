# ncu of the standalone apply's kernels at config 4 (third apply) and of the width-32 int8 Gram at config 3.
# (hardware-counter sections only: the SASS-patched sections SourceCounters / InstructionStats of --set full
# fail on the TONLY variant under kernel replay -- every counter section and application replay pass)
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/ncu_apply
O=gpurun_out/ncu_apply
SECS="--section SpeedOfLight --section MemoryWorkloadAnalysis --section LaunchStats --section Occupancy --section WarpStateStats --section ComputeWorkloadAnalysis"
python scripts/apply_once.py 4 3 && timeout 900 ncu $SECS --clock-control none -k regex:"k_sp8_step|k_colsum4|k_blk_reduce|k_dstream_sym8|k_dreduce_pair" -s 10 -c 5 -o $O/prof_apply4 python scripts/apply_once.py 4 3 > $O/ncu_apply.log 2>&1; echo rc=$?
