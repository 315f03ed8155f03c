export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -5
timeout 300 python scripts/profile_breakdown.py --config 4 --eigs 2>&1 | tail -1
python scripts/profile_breakdown.py --config 4 --quick && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 2 -c 2 -o gpurun_out/prof_spmm python scripts/profile_breakdown.py --config 4 --quick > gpurun_out/ncu_spmm.log 2>&1
tail -1 gpurun_out/ncu_spmm.log
