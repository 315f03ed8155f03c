# check of the int8 Gram steps: tests, step time, timeline, bench
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
T=${1:-q}
timeout 1200 python -m pytest tests/test_gpu_eigs.py -q -m gpu -x -k "tensor_core or config4 or deferred or int8_gram" 2>&1 | tail -15
python scripts/sp8_modes.py 4 0,1,0 2>&1 | tee gpurun_out/${T}_modes.txt
python scripts/sp8_timeline.py 58 > gpurun_out/${T}_timeline_58.txt 2>&1; sed -n 1p gpurun_out/${T}_timeline_58.txt | cut -c1-200; tail -9 gpurun_out/${T}_timeline_58.txt | cut -c1-200
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc=$?; head -c 300 gpurun_out/${T}_bench.json; echo
