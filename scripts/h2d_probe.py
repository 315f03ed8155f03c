import torch, time, numpy as np
x = torch.empty(int(5.35e9 // 4), dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
for i in range(8):
    torch.cuda.synchronize(); t = time.perf_counter()
    y.copy_(x, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"h2d 5.35 GB: {dt:.3f} s = {5.35 / dt:.1f} GB/s", flush=True)
