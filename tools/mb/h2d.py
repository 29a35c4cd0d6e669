"""Host<->device copy rates on this box: pinned H2D/D2H and host memcpy."""
import time
import numpy as np
import torch
n = 1 << 30
p = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, f in [("H2D pinned", lambda: d.copy_(p, non_blocking=True)),
                ("D2H pinned", lambda: p.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    print(f"{name}: {5 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
a = np.ones(n, np.uint8); b = np.empty(n, np.uint8)
t = time.perf_counter(); np.copyto(b, a); print(f"host memcpy 1 thread: {n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
