"""Householder QR (R only) on the path's shapes, with the live stage split
(qr_panel / gemm inside geqrf).  Usage: python tools/qr_bench.py [m,n ...]"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_0986_b200 as h  # noqa: E402
from paper_1410_0986_b200._lib import lib  # noqa: E402
from paper_1410_0986_b200.core import dptr  # noqa: E402

shapes = [(300, 300), (593, 593), (1112, 1112), (2172, 2172), (110592, 300), (110592, 593),
          (110592, 1112), (110592, 2172)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
ctx = h.Context(0)
L = lib()
buf = ctypes.create_string_buffer(1 << 16)
reps = int(os.environ.get("QR_REPS", "5"))
for m, n in shapes:
    A = torch.randn((n, m), dtype=torch.float64, device="cuda")  # column-major m x n
    R = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for _ in range(2):
        L.hydot_householder_qr(ctx.h, m, n, dptr(A), m, dptr(R), None)
    torch.cuda.synchronize()
    L.hydot_ctx_set_timing(ctx.h, 1)
    L.hydot_ctx_timing_report(ctx.h, buf, len(buf))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.hydot_householder_qr(ctx.h, m, n, dptr(A), m, dptr(R), None)
    e1.record()
    torch.cuda.synchronize()
    L.hydot_ctx_timing_report(ctx.h, buf, len(buf))
    L.hydot_ctx_set_timing(ctx.h, 0)
    st = json.loads(buf.value.decode())
    ms = e0.elapsed_time(e1) / reps
    flops = 2.0 * m * n * n - 2.0 * n ** 3 / 3
    print(json.dumps({"m": m, "n": n, "ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 2),
                      "stages_ms": {k: round(v[0] / reps, 3) for k, v in st.items()},
                      "calls": {k: v[1] / reps for k, v in st.items()}}), flush=True)
