export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
python scripts/eigs_once.py 4 6 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sp8_step -s 2 -c 1 -o gpurun_out/prof_sp8 python scripts/eigs_once.py 4 6 > gpurun_out/ncu_sp8.log 2>&1
tail -2 gpurun_out/ncu_sp8.log
