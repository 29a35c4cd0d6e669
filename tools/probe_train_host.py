"""train_l2_pq / train_apq repeated in one process at the config-5 shape:
wall time vs device phase time (host overhead, allocator behaviour)."""
import ctypes as C
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000
its = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = wl.config5(n=n)
s = aq.Session.default()
L = aq._L
ds = s.upload_dataset(w.base)
cfg = aq.TrainConfig(max_iterations=its, relative_tolerance=0.0, seed=0)
for rep in range(3):
    L.aq_session_timing(s.h, 1)
    for slot in range(9):
        L.aq_session_timer_read(s.h, slot, None, None, 1)
    s.sync()
    t = time.perf_counter()
    cb, codes = aq.dev_train_apq(ds, 128, 16, aq.ThresholdWeights(0.2), cfg, True, [])
    s.sync()
    tt = time.perf_counter() - t
    ph = {}
    for slot, nm in ((0, "encode"), (5, "assemble"), (6, "llt"), (7, "kmeans")):
        ms, cnt = C.c_double(0), C.c_uint64(0)
        L.aq_session_timer_read(s.h, slot, C.byref(ms), C.byref(cnt), 1)
        ph[nm] = round(ms.value, 1)
    L.aq_session_timing(s.h, 0)
    print(f"rep {rep}: wall {tt * 1e3:.0f} ms, device phases {ph}, "
          f"other {tt * 1e3 - sum(ph.values()):.0f} ms", flush=True)
