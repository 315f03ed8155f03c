# sparse-step diagnostics: normal / T off / stream-only times, stream-only timeline
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python scripts/sp8_modes.py 4 0,1,4,0 2>&1 | tee gpurun_out/r02k_modes.txt
python scripts/sp8_timeline.py 6 2>&1 | tee gpurun_out/r02k_timeline_stream.txt | head -60
python scripts/sp8_timeline.py 2 2>&1 | tee gpurun_out/r02k_timeline_full.txt | head -60
