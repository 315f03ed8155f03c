# quick check of a k_sp8_step change: the tests that run it, step time, non-H timeline
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
T=${1:-q}
timeout 900 python -m pytest tests/test_gpu_eigs.py -q -m gpu -x -k "tensor_core or config4 or deferred" 2>&1 | tail -3
python scripts/sp8_modes.py 4 0,1,0 2>&1 | tee gpurun_out/${T}_modes.txt
python scripts/sp8_timeline.py 26 > gpurun_out/${T}_timeline_26.txt 2>&1; sed -n 1p gpurun_out/${T}_timeline_26.txt | cut -c1-200; tail -9 gpurun_out/${T}_timeline_26.txt | cut -c1-200
