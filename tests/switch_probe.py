"""Run by tests/test_gpu_switches.py in a subprocess (the library reads most
of its environment switches once per process): BASELINE config 0 through the
public API -- fields, recursive compression, recompress, one J~ product --
printed as one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1410_0986_b200 as h
    from paper_1410_0986_b200 import born, configs, lowrank as lr
    ctx = h.Context(0)
    cfg = configs.CONFIGS[0]
    st = configs.make_setup(cfg)
    g = st.grid()
    F, stats = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points, tol=1e-10)
    w = torch.full((g.N,), cfg.h ** 3, dtype=torch.float64, device="cuda")
    inc = [F[st.source_point[s]] for s in range(cfg.n_sources)]
    adj = [[F[st.detector_point[s, d]] for d in range(cfg.n_det)] for s in range(cfg.n_sources)]
    tree = lr.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
    eps = configs.compression_tolerance(st, tree.depth())
    rec = lr.recursive_lowrank(ctx, tree, eps, lr.BornFieldsProvider(inc, adj, w, 1.0),
                               lr.RecursiveOptions(seed=cfg.seed))
    fr = lr.recompress(ctx, rec.factor, eps)
    J = lr.JOperator(ctx, fr, rec.row_perm, st.eps_c)
    x = np.random.default_rng(5).standard_normal((g.N * cfg.n_chrom, 2))
    y = J.matvec(torch.as_tensor(x)).cpu().numpy()
    # a tall Householder QR + thin SVD outside the recursion (panel / Jacobi paths by themselves)
    A = np.random.default_rng(6).standard_normal((30000, 450)) * np.logspace(0, -9, 450)
    _, R = lr.householder_qr(ctx, torch.as_tensor(A))          # 450 columns: the look-ahead engages
    _, s, _ = lr.thin_svd(ctx, torch.as_tensor(A[:, :200]))
    print(json.dumps({
        "relres_max": float(stats.relres.max()), "iters": int(stats.iters.sum()),
        "fields_norm": float(torch.linalg.norm(F)),
        "node_rank": list(map(int, rec.node_rank)), "rank": int(fr.rank()),
        "sigma": np.linalg.norm(fr.V.cpu().numpy(), axis=0).tolist(),
        "y": y.ravel().tolist(),
        "qr_diag": np.abs(np.diag(R.cpu().numpy())).tolist(), "svd": np.asarray(s).tolist()}))


if __name__ == "__main__":
    main()
