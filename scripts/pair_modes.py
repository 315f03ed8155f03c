"""Time k_dstream_pair under experiment modes (option pair_dbg bits 1..): 1 no converter TMEM stores,
2 no MMAs, 4 no epilogue TMEM work, 8 only the h1 MMA. Prints dstream ms per mode."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
b = int(sys.argv[2]) if len(sys.argv) > 2 else 16
modes = [int(m) for m in sys.argv[3:]] or [0, 1, 2, 4, 8, 5, 7]
p = configs.config(cfg)
out = {}
with from_problem(p) as h:
    h.set_option("dstream", int(os.environ.get("DS", "3")))
    X = torch.randn((p.n, b), device="cuda")
    Y = torch.empty_like(X)
    for _ in range(3):
        h.apply(X, Y)
    for m in modes:
        h.set_option("pair_dbg", 2 * m)
        h.set_option("profile", 1 << 2)
        h.apply(X, Y)
        h.set_option("profile_reset", 1)
        for _ in range(5):
            h.apply(X, Y)
        torch.cuda.synchronize()
        out[m] = h.stat("dstream_ns") / 5e6
    print(json.dumps(out))
