"""Block-Jacobi check on graded square cores: thin_svd through the path's
lazy-V variant; prints max |ds| / s1 or the error.  Usage: bj_debug.py n ..."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HYDOT_THIN_SVD_PATH"] = "1"
import paper_1410_0986_b200 as h  # noqa: E402
from paper_1410_0986_b200 import lowrank as lr  # noqa: E402

ctx = h.Context(0)
for n in [int(a) for a in sys.argv[1:]]:
    rng = np.random.default_rng(0)
    Q1 = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda"))[0]
    Q2 = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda"))[0]
    s = torch.logspace(0, -12, n, dtype=torch.float64, device="cuda")
    A = (Q1 * s) @ Q2.T
    try:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        U, sv, V = lr.thin_svd(ctx, A)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        err = float(np.max(np.abs(np.asarray(sv) - s.cpu().numpy())))
        print(f"n={n} ms={dt*1e3:.1f} max|ds|/s1={err:.2e}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"n={n} ERROR {e}", flush=True)
