"""LLT factor + solve timing at the normal-equation dimensions (config 2:
1600, config 5: 4096) with bit-exact check against the oracle's pinned
blocked Cholesky (oracle/eigen_subset, orc_llt_solve)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq  # noqa: E402
from oracle import Port  # noqa: E402

s = aq.Session.default()
L = aq._L
dev = torch.device("cuda", 0)
stream = torch.cuda.ExternalStream(s.stream, device=dev)
for dim in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1600", "4096"])]:
    g = np.random.default_rng(dim)
    X = g.standard_normal((dim + 64, dim))
    A = X.T @ X / dim + np.eye(dim) * 0.5
    b = g.standard_normal(dim)
    want = Port().llt_solve(A, b) if dim <= 2048 else None
    Ad = torch.from_numpy(A).to(dev)
    times, ftimes = [], []
    for rep in range(4):
        Aw = Ad.clone()
        x = torch.from_numpy(b).to(dev)
        torch.cuda.synchronize()
        L.aq_session_timing(s.h, 1)
        L.aq_session_timer_read(s.h, 6, None, None, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        aq._check(L.aq_dev_solve_normal_equations(s.h, Aw.data_ptr(), x.data_ptr(), dim, 0.0))
        e1.record(stream)
        e1.synchronize()
        ms, cnt = C.c_double(0), C.c_uint64(0)
        L.aq_session_timer_read(s.h, 6, C.byref(ms), C.byref(cnt), 1)
        L.aq_session_timing(s.h, 0)
        times.append(e0.elapsed_time(e1))
        ftimes.append(ms.value)
    got = x.cpu().numpy()
    ok = "n/a" if want is None else bool(np.array_equal(got, want))
    import hashlib
    ok = f"{ok} sha {hashlib.sha1(got.tobytes()).hexdigest()[:12]}"
    print(f"dim {dim}: total {min(times):.3f} ms  factor {min(ftimes):.3f} ms  "
          f"solve+ridge {min(times) - min(ftimes):.3f} ms  bit-exact {ok}", flush=True)
