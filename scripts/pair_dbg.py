"""Per-role wait-cycle breakdown of k_dstream_pair (option pair_dbg)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
b = int(sys.argv[2]) if len(sys.argv) > 2 else 16
p = configs.config(cfg)
names = {0: "prod_partner", 1: "prod_empty", 4: "mma_acc_empty", 5: "mma_full", 6: "mma_lo_full",
         8: "conv_full", 9: "conv_lo_empty", 12: "epi_acc_full", 15: "total"}
with from_problem(p) as h:
    h.set_option("dstream", 3)
    X = torch.randn((p.n, b), device="cuda")
    Y = torch.empty_like(X)
    for _ in range(3):
        h.apply(X, Y)
    h.set_option("pair_dbg", 1)
    h.apply(X, Y)
    torch.cuda.synchronize()
    out = {r: {nm: h.stat(f"pair_dbg_{r}_{k}") for k, nm in names.items()} for r in "NT"}
    print(json.dumps(out))
