# which ncu section makes the TONLY variant fail under kernel replay? (config 2)
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/ncu_tonly
O=gpurun_out/ncu_tonly
for sec in SourceCounters WarpStateStats SchedulerStats MemoryWorkloadAnalysis InstructionStats LaunchStats Occupancy ComputeWorkloadAnalysis MemoryWorkloadAnalysis_Tables; do
  timeout 200 ncu --section $sec --clock-control none -k regex:"k_sp8_step" -c 1 python scripts/apply_once.py 2 3 > $O/sec_$sec.log 2>&1; echo "$sec rc=$? passes: $(grep -o '[0-9]* passes' $O/sec_$sec.log | head -1)"
done
