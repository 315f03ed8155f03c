export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eigs.py tests/test_gpu_apply.py -x -q 2>&1 | tail -4
bash scripts/gpu_trace_e2e.sh | grep -B8 -A9 "D upload joined" | tail -10
grep -o '"e2e": {[^}]*}' gpurun_out/trace_e2e.json
