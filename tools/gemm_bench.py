"""DMMA GEMM throughput on the shapes of the path (CUDA events)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_0986_b200 as h  # noqa: E402

ctx = h.Context(0)
shapes = [
    ("square NN 4096^3", False, False, 4096, 4096, 4096, 0.0),
    ("sketch TN 300x330x110592", True, False, 300, 330, 110592, 0.0),
    ("qr W=V^T C TN 128x2044x110592", True, False, 128, 2044, 110592, 0.0),
    ("qr C-=V W NN 110592x2044x128 beta1", False, False, 110592, 2044, 128, 1.0),
    ("applyq NN 110592x2172x128 beta1", False, False, 110592, 2172, 128, 1.0),
    ("B=AtQ NN 110592x300x300", False, False, 110592, 300, 300, 0.0),
    ("matvec VtX TN 2131x256x110592", True, False, 2131, 256, 110592, 0.0),
    ("matvec UZ NN 4800x256x2131", False, False, 4800, 256, 2131, 0.0),
]
sel = os.environ.get("GEMM_SHAPES")
if sel:
    shapes = [shapes[int(i)] for i in sel.split(",")]
reps = int(os.environ.get("GEMM_REPS", "10"))
for name, ta, tb, m, n, k, beta in shapes:
    A = torch.randn((m * k,), dtype=torch.float64, device="cuda")
    B = torch.randn((k * n,), dtype=torch.float64, device="cuda")
    C = torch.randn((m * n,), dtype=torch.float64, device="cuda")
    lda = k if ta else m
    ldb = n if tb else k
    for _ in range(3):
        h.dgemm(ctx, ta, tb, m, n, k, 1.0, A, lda, B, ldb, beta, C, m)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        h.dgemm(ctx, ta, tb, m, n, k, 1.0, A, lda, B, ldb, beta, C, m)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    print(json.dumps({"shape": name, "tile": os.environ.get("HYDOT_GEMM_TILE", "auto"), "ms": t * 1e3, "tflops": 2.0 * m * n * k / t / 1e12}), flush=True)
