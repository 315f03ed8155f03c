export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
SBMDS_TRACE_EIGS=1 SBMDS_TRACE_CREATE=1 timeout 900 python bench.py --steps 1 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/trace_e2e.json 2> gpurun_out/trace_e2e.err
tail -60 gpurun_out/trace_e2e.err
