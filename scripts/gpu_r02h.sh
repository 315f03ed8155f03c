# Row order: stats per config, GPU suite, bench lines (config 4 eigs + apply, config 3, config 5 k16 b16)
export SBMDS_GEN_CACHE=/root/.cache/sbmds_gen
mkdir -p gpurun_out
python - <<'PY' 2>&1 | tail -12
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
for c in (1, 2, 3, 4):
    p = configs.config(c)
    with from_problem(p) as h:
        print(c, "permuted", h.stat("row_permuted"), "distinct nat/perm", h.stat("order_distinct_natural"), h.stat("order_distinct_permuted"), "umax", h.stat("blocked_umax"))
for k in (8, 64):
    p = configs.config(5, k5=k)
    with from_problem(p) as h:
        print("5 k", k, "permuted", h.stat("row_permuted"), h.stat("order_distinct_natural"), h.stat("order_distinct_permuted"), "umax", h.stat("blocked_umax"))
PY
timeout 2400 python -m pytest tests/ -q -m gpu -x > gpurun_out/r02h_tests.log 2>&1; tail -15 gpurun_out/r02h_tests.log
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_r02h.json 2>&1; echo rc=$?; head -c 700 gpurun_out/bench_r02h.json; echo
timeout 600 python bench.py --mode apply --config 4 > gpurun_out/bench_r02h_apply4.json 2>&1; echo rc=$?
timeout 900 python bench.py --config 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r02h_cfg3.json 2>&1; echo rc=$?
timeout 600 python bench.py --mode apply --config 3 --b 32 > gpurun_out/bench_r02h_apply3.json 2>&1; echo rc=$?
timeout 600 python bench.py --mode apply --config 5 --k5 16 --b 16 > gpurun_out/bench_r02h_cfg5_k16_b16.json 2>&1; echo rc=$?
timeout 600 python bench.py --mode apply --config 5 --k5 64 --b 64 > gpurun_out/bench_r02h_cfg5_k64_b64.json 2>&1; echo rc=$?
