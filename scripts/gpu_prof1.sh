export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
python scripts/profile_breakdown.py --config 4 --eigs > gpurun_out/breakdown_c4.json 2>&1; cat gpurun_out/breakdown_c4.json
python scripts/profile_breakdown.py --config 4 --eigs --order 0 > gpurun_out/breakdown_c4_noorder.json 2>&1; cat gpurun_out/breakdown_c4_noorder.json
for k in 8 16 64; do for b in 1 4 16 64; do python scripts/profile_breakdown.py --config 5 --k5 $k --b $b --applies 10; done; done > gpurun_out/breakdown_c5.jsonl 2>&1; cat gpurun_out/breakdown_c5.jsonl
python scripts/profile_breakdown.py --config 3 --eigs > gpurun_out/breakdown_c3.json 2>&1; cat gpurun_out/breakdown_c3.json
python scripts/profile_breakdown.py --config 4 --quick && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/profile_breakdown.py --config 4 --quick > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dstream -s 2 -c 1 -o gpurun_out/prof_dstream python scripts/profile_breakdown.py --config 4 --quick > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
