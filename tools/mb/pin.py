"""Cost of page-locking an existing (pageable) host buffer in place."""
import time
import numpy as np
import torch
cr = torch.cuda.cudart()
for gb in (0.5, 2.56, 5.12):
    a = np.ones(int(gb * 1e9), np.uint8)  # touched
    t = time.perf_counter()
    r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data)
    t2 = time.perf_counter()
    print(f"{gb} GB: register {t1 - t:.3f} s ({r}), unregister {t2 - t1:.3f} s", flush=True)
