# compute-sanitizer (memcheck, racecheck) on small cases of the round-2 kernels: BMDS, sBHA,
# sharded stages, precision checks; and memcheck on the config-1 smoke (tcgen05/TMA kernels).
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out/r02s
O=gpurun_out/r02s
CS=/usr/local/cuda/bin/compute-sanitizer
$CS --version | head -2
timeout 900 $CS --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_sbha.py -q -x -k "icosphere or planar or degenerate" > $O/memcheck_sbha.log 2>&1; echo sbha rc=$?; tail -6 $O/memcheck_sbha.log
timeout 900 $CS --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_bmds.py -q -x -k "config1_vs_dense or rank_deficient" > $O/memcheck_bmds.log 2>&1; echo bmds rc=$?; tail -6 $O/memcheck_bmds.log
timeout 900 $CS --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_shard.py -q -x -k "ragged or communicator" > $O/memcheck_shard.log 2>&1; echo shard rc=$?; tail -6 $O/memcheck_shard.log
timeout 900 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_sbha.py -q -x -k "icosphere" > $O/racecheck_sbha.log 2>&1; echo race sbha rc=$?; tail -6 $O/racecheck_sbha.log
timeout 900 $CS --tool memcheck --leak-check no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1; echo smoke rc=$?; tail -6 $O/memcheck_smoke.log
