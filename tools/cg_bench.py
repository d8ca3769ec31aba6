"""Fields (batched CG) throughput at a BASELINE config.  Usage: python tools/cg_bench.py [cfg]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_0986_b200 as h  # noqa: E402
from paper_1410_0986_b200 import born, configs  # noqa: E402

cfg = configs.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
st = configs.make_setup(cfg)
ctx = h.Context(0)
g = st.grid()
F, stats = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points[:4], tol=1e-10)
torch.cuda.synchronize()
times = []
for rep in range(int(os.environ.get("CG_REPS", "3"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    F, stats = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points, tol=1e-10)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) / 1e3)
    del F
s = min(times)
it = float(stats.iters.sum())
gbs = 48.0 * g.N * it / s / 1e9
print(json.dumps({"cfg": cfg.name, "systems": int(stats.iters.size), "s_min": round(s, 3),
                  "s_all": [round(t, 3) for t in times],
                  "iters_total": int(it), "alg_GB/s": round(gbs), "frac": round(gbs / 6554.9, 3),
                  "relres_max": float(stats.relres.max()),
                  "env": {k: v for k, v in os.environ.items() if k.startswith("HYDOT_CG")}}))
