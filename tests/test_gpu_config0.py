"""BASELINE config 0 (the reference's CPU-runnable case: n=32, N=32768, 8
sources x 4 detectors x 20 wavelengths, M=640, 4 chromophores) end to end
against the CPU oracle on identical inputs:

* fields: device CG vs the oracle CG at equal iteration counts <= 1e-12
  (only the dot-product summation order differs), and both converged to the
  1e-10 relative residual;
* compression: the device fields feed both sides (SURVEY 8d parity
  procedure), so node ranks must be equal, ||J~_gpu - J~_cpu||_F / ||J||_F
  <= 1e-8 after recompress, leading singular values within 1e-8 relative;
* J~x / J~^T y with the chromophore axis and the row permutation <= 1e-10.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def run():
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
    return dict(ctx=ctx, cfg=cfg, st=st, g=g, F=F, stats=stats, w=w, tree=tree, eps=eps,
                rec=rec, fr=fr)


def test_config0_fields_match_oracle(run, oracle):
    from paper_1410_0986_b200 import born
    d = run
    st, g = d["st"], d["g"]
    assert float(d["stats"].relres.max()) <= 1e-10
    pts = st.points[:3]
    gpu, _ = born.compute_fields(d["ctx"], g, st.sigma, st.sigma_prime, st.inv_D, pts, fixed_iters=40)
    want, _, _ = oracle.fields((g.nx, g.ny, g.nz), g.h, st.sigma, st.sigma_prime, st.inv_D, pts,
                               fixed_iters=40, threads=8)
    got = gpu.cpu().numpy().reshape(len(pts) * len(st.sigma), g.N).T
    rel = np.linalg.norm(got - want, axis=0) / np.linalg.norm(want, axis=0)
    assert rel.max() <= 1e-12, rel.max()


def test_config0_compression_and_products_match_oracle(run, oracle):
    d = run
    cfg, st, g = d["cfg"], d["st"], d["g"]
    Fh = d["F"].cpu().numpy()
    wh = d["w"].cpu().numpy()
    oinc = [Fh[st.source_point[s]].T for s in range(cfg.n_sources)]
    oadj = [[Fh[st.detector_point[s, k]].T for k in range(cfg.n_det)] for s in range(cfg.n_sources)]
    otree = oracle.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
    orec = oracle.recursive_lowrank_born(otree, d["eps"], oinc, oadj, wh, 1.0, seed=cfg.seed)
    rec = d["rec"]
    assert list(rec.node_rank) == list(orec.node_rank)
    assert np.array_equal(rec.row_perm, orec.row_perm)
    H = np.vstack([oracle.born_block(oinc[s], oadj[s], wh, 1.0) for s in range(cfg.n_sources)])
    of = oracle.recompress(orec.factor, d["eps"])
    fr = d["fr"]
    assert fr.rank() == of.rank
    Jg = np.zeros_like(H)
    Jg[rec.row_perm] = fr.dense().cpu().numpy()
    Jo = np.zeros_like(H)
    Jo[orec.row_perm] = of.dense()
    nH = np.linalg.norm(H)
    assert np.linalg.norm(Jg - Jo) <= 1e-8 * nH
    # compression error itself within the whole-tree budget eps_d = 1e-6
    assert np.linalg.norm(H - Jg) <= 1e-6 * nH
    # leading singular values of J~ (its V carries them)
    sg = np.linalg.norm(fr.V.cpu().numpy(), axis=0)[:10]
    so = np.linalg.svd(of.dense(), compute_uv=False)[:10]
    assert np.max(np.abs(sg - so) / so) <= 1e-8
    # J~ products, chromophore axis + permutation
    from paper_1410_0986_b200 import lowrank as lr
    J = lr.JOperator(d["ctx"], fr, rec.row_perm, st.eps_c)
    rng = np.random.default_rng(1)
    X = rng.standard_normal((g.N * cfg.n_chrom, 4))
    yg = J.matvec(torch.as_tensor(X)).cpu().numpy()
    yo = oracle.j_matmat(of, X, orec.row_perm, st.eps_c)
    assert np.linalg.norm(yg - yo) <= 1e-10 * np.linalg.norm(yo)
    Y = rng.standard_normal((cfg.M, 4))
    xg = J.rmatvec(torch.as_tensor(Y)).cpu().numpy()
    xo = oracle.j_matmat(of, Y, orec.row_perm, st.eps_c, trans=True)
    assert np.linalg.norm(xg - xo) <= 1e-10 * np.linalg.norm(xo)
