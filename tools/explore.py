"""Exploration driver: fields -> recursive compression -> recompress at a
BASELINE config on one GPU, printing phase times, ranks and the ledger.
Usage: python tools/explore.py CFG_ID [--save-fields PATH]"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1410_0986_b200 as h  # noqa: E402
from paper_1410_0986_b200 import born, configs, lowrank as lr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--p", type=int, default=20)
    args = ap.parse_args()
    cfg = configs.CONFIGS[args.cfg]
    st = configs.make_setup(cfg)
    ctx = h.Context(0)
    g = st.grid()
    t0 = time.time()
    F, stats = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points, tol=1e-10)
    torch.cuda.synchronize()
    t_fields = time.time() - t0
    print(json.dumps(dict(cfg=cfg.name, points=len(st.points), fields_s=t_fields,
                          iters_max=int(stats.iters.max()), iters_mean=float(stats.iters.mean()),
                          relres_max=float(stats.relres.max()))), flush=True)
    w = torch.full((g.N,), cfg.h ** 3, dtype=torch.float64, device="cuda")
    inc = [F[st.source_point[s]] for s in range(cfg.n_sources)]
    adj = [[F[st.detector_point[s, d]] for d in range(cfg.n_det)] for s in range(cfg.n_sources)]
    tree = lr.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
    eps = configs.compression_tolerance(st, tree.depth())
    prov = lr.BornFieldsProvider(inc, adj, w, 1.0)
    for rep in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.time()
        rec = lr.recursive_lowrank(ctx, tree, eps, prov, lr.RecursiveOptions(seed=cfg.seed, p=args.p))
        torch.cuda.synchronize()
        t1 = time.time()
        fr = lr.recompress(ctx, rec.factor, eps)
        torch.cuda.synchronize()
        t2 = time.time()
        led = rec.ledger
        print(json.dumps(dict(rep=rep, eps=eps, depth=tree.depth(), rec_s=t1 - t0, recompress_s=t2 - t1,
                              rank=rec.factor.rank(), rank_recompressed=fr.rank(),
                              node_rank=rec.node_rank.tolist(), flagged=rec.factor.flagged,
                              ledger=dict(leaf=led.leaf, agg=led.agglomeration, tally=led.kernel_tally),
                              launches=ctx.launch_count())), flush=True)
        import ctypes
        buf = ctypes.create_string_buffer(1 << 16)
        h.lib().hydot_profile_dump(buf, 1 << 16)
        print(buf.value.decode(), flush=True)


if __name__ == "__main__":
    main()
