"""Wall-clock and CUDA-event time of the libstdc++ Gaussian stream on the GPU
(hydot_gaussian) for the sketch sizes of the path.  Usage: python tools/rng_bench.py [count ...]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_0986_b200 as h  # noqa: E402
from paper_1410_0986_b200 import core  # noqa: E402

ctx = h.Context(0)
counts = [int(float(a)) for a in sys.argv[1:]] or [262144 * 250, 262144 * 830, 262144 * 1580, 262144 * 2980]
for n in counts:
    for _ in range(2):
        core.gaussian(ctx, 7, 0, n)
    torch.cuda.synchronize()
    reps = 4
    t0 = time.perf_counter()
    for r in range(reps):
        core.gaussian(ctx, 11 + r, 0, n)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"normals={n} ({n * 8 / 1e9:.2f} GB) wall_ms={dt * 1e3:.2f} Gnormals/s={n / dt / 1e9:.2f}", flush=True)
