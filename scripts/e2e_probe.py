import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from gen import configs
from paper_1705_10887_b200 import Sbmds
p = configs.config(4)
rp = torch.from_numpy(np.ascontiguousarray(p.row_ptr, dtype=np.int64)).pin_memory()
ci = torch.from_numpy(np.ascontiguousarray(p.col_idx)).pin_memory()
vv = torch.from_numpy(p.val32()).pin_memory()
Dh = torch.from_numpy(p.D).pin_memory()
Dd = torch.empty_like(Dh, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    Dd.copy_(Dh, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    h = Sbmds(p.n, p.l, rp, ci, vv, Dh); torch.cuda.synchronize()
    t2 = time.perf_counter() - t
    t = time.perf_counter()
    h2 = Sbmds(p.n, p.l, rp.cuda(), ci.cuda(), vv.cuda(), Dd); torch.cuda.synchronize()
    t3 = time.perf_counter() - t
    print(f"H2D 10 GB torch copy {t1:.3f}s ({Dh.nbytes/t1/1e9:.1f} GB/s) | create from pinned host {t2:.3f}s | create from device {t3:.3f}s", flush=True)
    h.close(); h2.close()
