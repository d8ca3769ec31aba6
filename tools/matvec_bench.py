"""J~x / J~^T y throughput on a random factor of the config-1 shape
(N=110592, M=4800, R=2131, 4 chromophores).  Usage: python tools/matvec_bench.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_0986_b200 as h  # noqa: E402
from paper_1410_0986_b200 import lowrank as lr  # noqa: E402

N, M, R, NC, NL = 110592, 4800, 2131, 4, 50
ctx = h.Context(0)
U = torch.randn(M, R, dtype=torch.float64, device="cuda")
V = torch.randn(N, R, dtype=torch.float64, device="cuda")
f = lr.LowRankFactor.from_tensors(ctx, U, V)
perm = np.random.default_rng(0).permutation(M).astype(np.int32)
J = lr.JOperator(ctx, f, perm, np.random.default_rng(1).uniform(0.1, 1, (NL, NC)))
peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "MEASURED_PEAKS.json")))["hbm_gbs"])
for b in (1, 4, 16, 64):
    X = torch.randn(b, N * NC, dtype=torch.float64, device="cuda")
    Y = torch.randn(b, M, dtype=torch.float64, device="cuda")
    for name, fn in (("Jx", lambda: J.matmat_cm(X, Y, b)), ("JTy", lambda: J.rmatmat_cm(Y, X, b))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10 / 1e3
        nbytes = 8.0 * (N * R + M * R + b * NC * N + b * M)
        flops = 2.0 * R * b * NC * (N + M)
        print(json.dumps({"op": name, "b": b, "ms": round(t * 1e3, 3), "GB/s": round(nbytes / t / 1e9),
                          "hbm_frac": round(nbytes / t / 1e9 / peak, 3),
                          "TFLOP/s": round(flops / t / 1e12, 2)}), flush=True)
