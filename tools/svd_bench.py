"""Time the device thin SVD (the path's lazy-V variant with
HYDOT_THIN_SVD_PATH=1) on graded square cores like the path's R factors.
Usage: python tools/svd_bench.py [n ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_0986_b200 as h  # noqa: E402
from paper_1410_0986_b200 import lowrank as lr  # noqa: E402

ctx = h.Context(0)
sizes = [int(a) for a in sys.argv[1:]] or [300, 576, 1106, 2172]
rng = np.random.default_rng(0)
for n in sizes:
    Q1, _ = np.linalg.qr(rng.standard_normal((n, n)))
    Q2, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.logspace(0, -12, n)
    A = torch.as_tensor((Q1 * s) @ Q2.T).cuda()
    for _ in range(2):
        lr.thin_svd(ctx, A)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        U, sv, V = lr.thin_svd(ctx, A)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    err = float(np.max(np.abs(np.asarray(sv) - s) / s[0]))
    print(f"n={n} ms={dt * 1e3:.2f} max|ds|/s1={err:.2e}", flush=True)
