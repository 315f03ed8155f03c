# static Y_B scales in k_sp8_step: parity tests that run the tensor-core step, step times, timeline
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
(time timeout 1500 python -m pytest tests/test_gpu_eigs.py tests/test_gpu_configs.py tests/test_gpu_precision.py -q -m gpu -x -k "tensor_core or config4 or config2 or deferred or graph or precision or weights or range") > gpurun_out/r02l_tests.log 2>&1; tail -8 gpurun_out/r02l_tests.log
python scripts/sp8_modes.py 4 0,1,0 2>&1 | tee gpurun_out/r02l_modes.txt
python scripts/sp8_timeline.py 26 > gpurun_out/r02l_timeline_26.txt 2>&1; tail -12 gpurun_out/r02l_timeline_26.txt | cut -c1-200
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err; echo bench rc=$?; head -c 600 gpurun_out/r02l_bench.json; echo
