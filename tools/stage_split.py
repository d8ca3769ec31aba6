"""One config-1 compress step with live CUDA-event stage timing; prints the
per-stage ms, calls and achieved TF/s.  Usage: python tools/stage_split.py"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_0986_b200 as h  # noqa: E402
from paper_1410_0986_b200 import born, configs, lowrank as lr  # noqa: E402

cfg = configs.CONFIGS[1]
st = configs.make_setup(cfg)
ctx = h.Context(0)
g = st.grid()
F, _ = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points, tol=1e-10)
w = torch.full((g.N,), cfg.h ** 3, dtype=torch.float64, device="cuda")
prov = lr.BornFieldsProvider([F[st.source_point[s]] for s in range(cfg.n_sources)],
                             [[F[st.detector_point[s, d]] for d in range(cfg.n_det)] for s in range(cfg.n_sources)], w, 1.0)
tree = lr.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
eps = configs.compression_tolerance(st, tree.depth())
for rep in range(2):
    if rep == 1:
        h.lib().hydot_ctx_timing_report(ctx.h, None, 0)
        h.lib().hydot_ctx_set_timing(ctx.h, 1)
    rec = lr.recursive_lowrank(ctx, tree, eps, prov, lr.RecursiveOptions(seed=cfg.seed))
    fr = lr.recompress(ctx, rec.factor, eps, -1, rec.ledger)
torch.cuda.synchronize()
buf = ctypes.create_string_buffer(1 << 16)
h.lib().hydot_ctx_timing_report(ctx.h, buf, 1 << 16)
d = json.loads(buf.value.decode())
for k, v in sorted(d.items(), key=lambda kv: -kv[1][0]):
    tf = v[2] / (v[0] / 1e3) / 1e12 if v[0] > 0 else 0.0
    print(f"{k:22s} {v[0]:9.1f} ms {int(v[1]):7d} calls {tf:6.2f} TF/s")
