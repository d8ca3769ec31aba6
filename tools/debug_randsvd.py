import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1410_0986_b200 as h
from paper_1410_0986_b200 import lowrank as lr
from oracle import oracle as o
ctx = h.Context(0)
rng = np.random.default_rng(1)
X = rng.standard_normal((40, 7)); Y = rng.standard_normal((55, 7)); A = X @ Y.T
for trial in range(3):
    f = lr.randsvd(ctx, A, 1e-10, 20, 10, 100)
    fo = o.randsvd(A, 1e-10, 20, 10, 100)
    print("rank", f.rank(), fo.rank, "err", np.linalg.norm(A - f.dense().cpu().numpy()) / np.linalg.norm(A), flush=True)
U, s, V = lr.thin_svd(ctx, torch.as_tensor(A))
print("thin_svd s", s[:8])
U, s, V = lr.thin_svd(ctx, torch.as_tensor(A[:, :21]))
print("thin_svd 40x21 s", s[:8])
