import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1410_0986_b200 as h
from paper_1410_0986_b200 import lowrank as lr
ctx = h.Context(0)
rng = np.random.default_rng(1)
for (m, n) in [(55, 8), (40, 21), (300, 70), (1000, 40), (20000, 33), (5000, 300)]:
    bad = 0
    A = rng.standard_normal((m, n))
    R2 = np.abs(np.diag(np.linalg.qr(A, mode="r")))
    for t in range(20):
        Q, R = lr.householder_qr(ctx, torch.as_tensor(A))
        Q, R = Q.cpu().numpy(), R.cpu().numpy()
        e = np.linalg.norm(Q @ R - A) / np.linalg.norm(A)
        d = np.max(np.abs(np.abs(np.diag(R)) - R2) / R2)
        if e > 1e-13 or d > 1e-10:
            bad += 1
            if bad < 3:
                print(m, n, "trial", t, "err", e, "diag", d, flush=True)
    print(m, n, "bad", bad, flush=True)
