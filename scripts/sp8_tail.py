"""Per-CTA start / finish of the tensor-core sparse step at config 4 (sp8_dbg & 2 tail trace):
how much of the launch is the slowest CTA's excess over the median, and the last CTA's Gram
sums + Cholesky."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import configs
from paper_1705_10887_b200 import from_problem
p = configs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
with from_problem(p) as h:
    h.set_option("sp8_dbg", 2)
    for rep in range(3):
        h.eigs(p.m, p.block, max_iters=3, tol=0.0)
        torch.cuda.synchronize()
        ncta = min(148, h.stat("sp8_slots") if False else 148)
        st = [h.stat(f"sp8_trace_{768 + c}") for c in range(ncta)]
        dn = [h.stat(f"sp8_trace_{1024 + c}") for c in range(ncta)]
        end = h.stat("sp8_trace_1279")
        pw = sorted((h.stat(f"sp8_trace_{1280 + c}") - min(st)) / 1000 for c in range(ncta))
        dl = sorted((h.stat(f"sp8_trace_{1280 + c}") - dn[c]) / 1000 for c in range(ncta))
        a1 = sorted((h.stat(f"sp8_trace_{1536 + c}") - dn[c]) / 1000 for c in range(ncta))
        a2 = sorted((h.stat(f"sp8_trace_{1792 + c}") - dn[c]) / 1000 for c in range(ncta))
        print(f"  after fence+sync median {statistics.median(a1):.1f}, after red sync median {statistics.median(a2):.1f} us")
        print(f"  per-CTA partial phase: min {dl[0]:.1f} median {statistics.median(dl):.1f} max {dl[-1]:.1f} us")
        e1, e2 = h.stat("sp8_trace_1277"), h.stat("sp8_trace_1278")
        t0 = min(st)
        d = sorted((x - t0) / 1000 for x in dn)
        s = sorted((x - t0) / 1000 for x in st)
        print(f"rep {rep}: start spread {s[-1]:.1f} us; CTA done min {d[0]:.1f} median {statistics.median(d):.1f} "
              f"p90 {d[int(0.9 * len(d))]:.1f} max {d[-1]:.1f} us; partials written max {pw[-1]:.1f}; last CTA in "
              f"{(e1 - t0) / 1000:.1f}, sums {(e2 - t0) / 1000:.1f}, end {(end - t0) / 1000:.1f} us", flush=True)
