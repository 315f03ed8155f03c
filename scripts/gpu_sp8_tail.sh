export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
timeout 600 python scripts/sp8_tail.py 4 2>&1 | tail -4
