export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
python scripts/profile_breakdown.py --config 5 --k5 16 --b 16 --dstream 3 --quick && \
ncu --set full --clock-control none --import-source on -k regex:k_dstream_sym -s 2 -c 1 -o gpurun_out/prof_sym python scripts/profile_breakdown.py --config 5 --k5 16 --b 16 --dstream 3 --quick > gpurun_out/ncu_sym.log 2>&1
tail -1 gpurun_out/ncu_sym.log
