# ncu --set full of the two fp32 SpMMs of a config-5 standalone apply (k = 16, b = 16): what bounds them
# (L1 wavefronts of the gathers vs L2 vs DRAM re-reads of X).
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/ncu_cfg5
O=gpurun_out/ncu_cfg5
python scripts/apply_once.py 5 3 16 16 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_csc_vec4|k_spmm_csr_vec4" -s 4 -c 2 -o $O/prof_cfg5 python scripts/apply_once.py 5 3 16 16 > $O/ncu.log 2>&1; echo rc=$?
tail -3 $O/ncu.log
