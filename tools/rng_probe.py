"""Generate one large Gaussian block (profiling target for the RNG kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_0986_b200 as h  # noqa: E402

ctx = h.Context(0)
x = h.gaussian(ctx, 12345, 0, 40_000_000)
torch.cuda.synchronize()
print(float(x[:1000].std()))
