"""Why the tensor-core sparse kernels do or do not apply at a config: states and dictionary sizes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = configs.config(cfg)
b = p.block
with from_problem(p) as h:
    X = torch.randn(p.n, b, device="cuda")
    h.apply(X)
    torch.cuda.synchronize()
    for k in ["sp8_state", "sp8_umax", "sp8_range", "blocked_umax", "sp8_apply_launches", "sp8_apply_t_launches", "x_fallbacks", "sp8_bytes"]:
        print(k, h.stat(k))
