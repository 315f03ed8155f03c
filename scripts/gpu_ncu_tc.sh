export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
timeout 600 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
python scripts/profile_breakdown.py --config 5 --k5 16 --b 16 --quick && \
ncu --set full --clock-control none --import-source on -k regex:k_dstream_tc -s 2 -c 1 -o gpurun_out/prof_tc2 python scripts/profile_breakdown.py --config 5 --k5 16 --b 16 --quick > gpurun_out/ncu_tc.log 2>&1
tail -1 gpurun_out/ncu_tc.log
