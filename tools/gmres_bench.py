"""Field solves on the reference's FEM operator: the device recycled
shifted-family GMRES (krylov.compute_fields_fem_gmres, csrc/gmres.cu) next to
the device batched CG (born.compute_fields_fem) on the same family, with the
BASELINE config's physics (configs.make_setup) on the FEM box of the same
spacing.  Optionally times the CPU oracle's solve_family on one rhs.

usage: python tools/gmres_bench.py CFG [--points P] [--oracle] [--tol T]
Prints one JSON line per solver."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--points", type=int, default=0, help="number of field points (0 = all of the config)")
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    import paper_1410_0986_b200 as h
    from paper_1410_0986_b200 import born, configs, krylov
    cfg = configs.CONFIGS[a.cfg] if hasattr(configs, "CONFIGS") else configs.config(a.cfg)
    st = configs.make_setup(cfg)
    n, hh = cfg.n, cfg.h
    half = (n - 1) * hh / 2
    geom = (n, n, n, half, half, (n - 1) * hh)
    pv = st.points if a.points <= 0 else st.points[: a.points]
    xyz = np.stack([(pv % n) * hh - half, ((pv // n) % n) * hh - half, (pv // (n * n)) * hh], axis=1)
    ctx = h.Context(0)
    nl = len(st.sigma)
    out = {}
    for name in ("cg", "gmres"):
        ts = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if name == "cg":
                F, stc = born.compute_fields_fem(ctx, geom, st.sigma, st.sigma_prime, st.inv_D, xyz, tol=a.tol)
                info = dict(iters_total=int(stc.iters.sum()), iters_max=int(stc.iters.max()),
                            relres_max=float(stc.relres.max()))
            else:
                F, fam = krylov.compute_fields_fem_gmres(ctx, geom, st.sigma, st.sigma_prime, st.inv_D, xyz,
                                                         krylov.SolverConfig(tol=a.tol))
                its = [s.iterations for f in fam for s in f.stats]
                info = dict(phase1_steps=[f.phase1_matvecs for f in fam][:4], deflation_k=fam[0].deflation_k,
                            phase2_iters_total=int(sum(its)), phase2_iters_max=int(max(its)),
                            relres_max=float(max(s.relres for f in fam for s in f.stats)),
                            matvecs_total=int(sum(s.matvecs for f in fam for s in f.stats)))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        out[name] = F
        print(json.dumps(dict(solver=name, cfg=a.cfg, N=cfg.N, points=len(pv), n_lambda=nl, systems=len(pv) * nl,
                              s=min(ts), s_all=ts, **info)), flush=True)
    d = (out["gmres"] - out["cg"]).norm(dim=2) / out["cg"].norm(dim=2)
    print(json.dumps(dict(gmres_vs_cg_max_rel=float(d.max()))), flush=True)
    if a.oracle:
        from oracle import oracle as o
        b = o.fem_point_source(geom, xyz[0])
        t0 = time.time()
        r = o.krylov_solve_family(geom, b, np.stack([st.sigma, st.sigma_prime], 1), o.SolverConfig(tol=a.tol))
        dt = time.time() - t0
        Xo = r["X"] * st.inv_D[None, :]
        Fg = out["gmres"][0].cpu().numpy().T
        rel = np.linalg.norm(Fg - Xo, axis=0) / np.linalg.norm(Xo, axis=0)
        print(json.dumps(dict(solver="oracle_cpu_1rhs", s=dt, cores=1, phase1_steps=r["phase1_steps"],
                              phase2_iters_total=int(r["iters"].sum()), device_vs_oracle_max_rel=float(rel.max()))),
              flush=True)


if __name__ == "__main__":
    main()
