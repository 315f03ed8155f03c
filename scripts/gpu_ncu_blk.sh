export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -3
timeout 300 python scripts/profile_breakdown.py --config 4 --eigs 2>&1 | tail -1
python scripts/profile_breakdown.py --config 4 --quick && \
ncu --set full --clock-control none --import-source on -k regex:"k_blk_spmm|k_blk_reduce" -s 3 -c 3 -o gpurun_out/prof_blk2 python scripts/profile_breakdown.py --config 4 --quick > gpurun_out/ncu_blk.log 2>&1
tail -1 gpurun_out/ncu_blk.log
