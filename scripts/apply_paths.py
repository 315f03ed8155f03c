"""Standalone apply time with the tensor-core sparse kernels on / off (option sp8_apply) at a config."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = configs.config(cfg)
b = int(sys.argv[2]) if len(sys.argv) > 2 else (p.block or 16)
with from_problem(p) as h:
    X = torch.from_numpy(configs.x_block(p.n, b, seed=3)).cuda()
    Y = torch.empty_like(X)
    for on in (1, 0, 1, 0):
        h.set_option("sp8_apply", on)
        for _ in range(5): h.apply(X, out=Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): h.apply(X, out=Y)
        e1.record(); torch.cuda.synchronize()
        print(json.dumps({"config": cfg, "b": b, "sp8_apply": on, "ms_per_apply": round(e0.elapsed_time(e1) / 50, 4),
                          "t_launches": h.stat("sp8_apply_t_launches")}), flush=True)
