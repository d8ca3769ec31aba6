"""Compression and matvec parity on the B200 against the CPU oracle.

Same inputs, same seeds (the device generator reproduces the libstdc++ Gaussian
stream), so the adaptive rank path is replayed: ranks must be equal, leading
singular values within 1e-8 relative, ||J~_gpu - J~_cpu||_F / ||J||_F <= 1e-8,
matvecs within 1e-10 relative (BASELINE.json north_star tolerances).  The
reference's own lowrank tests (test_lowrank.cpp) are restated on the GPU path.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1410_0986_b200 as h
    return h.Context(0)


def random_lowrank(rng, m, n, r, noise=0.0):
    X = rng.standard_normal((m, r))
    Y = rng.standard_normal((n, r))
    A = X @ Y.T
    if noise > 0:
        E = rng.standard_normal((m, n))
        A = A + (noise * np.linalg.norm(A) / np.linalg.norm(E)) * E
    return A


def fro(a):
    return float(np.linalg.norm(a))


def test_randsvd_reference_cases(ctx):
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(1)
    for t in range(5):  # test_lowrank.cpp:53-62
        A = random_lowrank(rng, 40, 55, 7)
        f = lr.randsvd(ctx, A, 1e-10, 20, 10, 100 + t)
        assert fro(A - f.dense().cpu().numpy()) <= 1e-9 * fro(A)
        assert f.rank() <= 27 and not f.flagged
    rng = np.random.default_rng(2)
    for t in range(10):  # :64-72
        A = random_lowrank(rng, 30 + t % 20, 45, 5 + t % 6, 1e-4)
        f = lr.randsvd(ctx, A, 1e-3, 20, 10, 500 + t)
        assert fro(A - f.dense().cpu().numpy()) <= 10 * 1e-3 * fro(A)
    f = lr.randsvd(ctx, np.zeros((12, 9)), 1e-8)  # :74-79
    assert f.rank() == 0
    A = random_lowrank(np.random.default_rng(3), 25, 30, 6, 1e-6)  # :81-88
    f1 = lr.randsvd(ctx, A, 1e-6, 20, 10, 42)
    f2 = lr.randsvd(ctx, A, 1e-6, 20, 10, 42)
    assert torch.equal(f1.U, f2.U) and torch.equal(f1.V, f2.V)


@pytest.mark.parametrize("m,n,r,noise,eps,r0", [
    (40, 55, 7, 0.0, 1e-10, 1),         # Q = I branch (rs >= nmax)
    (200, 3000, 12, 1e-9, 1e-6, 1),     # adaptive sketch: several passes
    (80, 32768, 30, 1e-8, 6.6e-9, 43),  # cfg0-shaped leaf, warm start
    (300, 20000, 60, 1e-7, 1e-6, 1),
])
def test_randsvd_parity_with_oracle(ctx, oracle, m, n, r, noise, eps, r0):
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(m + n)
    A = random_lowrank(rng, m, n, r, noise) * np.exp(-np.arange(n) / n)[None, :]
    for seed in (7, 20240811 + 0x9e3779b97f4a7c15):
        fo = oracle.randsvd(A, eps, 20, 10, seed, oracle.LEAF, r0)
        fg = lr.randsvd(ctx, A, eps, 20, 10, seed, cat=lr.LEAF, r0=r0)
        assert fg.rank() == fo.rank
        assert fg.flagged == fo.flagged
        Dg = fg.dense().cpu().numpy()
        Do = fo.dense()
        assert fro(Dg - Do) <= 1e-8 * fro(A)
        sg = np.linalg.norm(fg.V.cpu().numpy(), axis=0)
        so = np.linalg.norm(fo.V, axis=0)
        assert np.all(np.abs(sg - so) <= 1e-8 * so[0])


def test_agglomerate_bound_and_parity(ctx, oracle):
    # test_lowrank.cpp:122-137 + parity of the merge with the oracle
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(6)
    for t in range(10):
        H1 = random_lowrank(rng, 24, 40, 5, 1e-3)
        H2 = random_lowrank(rng, 18, 40, 4, 1e-3)
        eps = 1e-2
        fs = []
        for Hx in (H1, H2):
            U, s, Vt = np.linalg.svd(Hx, full_matrices=False)
            k = int(np.sum(s > eps * s[0]))
            fs.append((U[:, :k], Vt[:k].T * s[:k]))
        g1 = lr.LowRankFactor.from_tensors(ctx, torch.as_tensor(fs[0][0]), torch.as_tensor(fs[0][1]))
        g2 = lr.LowRankFactor.from_tensors(ctx, torch.as_tensor(fs[1][0]), torch.as_tensor(fs[1][1]))
        o1 = oracle.Factor.make(*fs[0])
        o2 = oracle.Factor.make(*fs[1])
        g = lr.agglomerate(ctx, g1, g2, eps, 900 + t)
        o = oracle.agglomerate(o1, o2, eps, 900 + t)
        H = np.vstack([H1, H2])
        err = fro(H - g.dense().cpu().numpy())
        assert err <= (2 * eps + eps * eps) * (fro(H1) + fro(H2))
        assert g.rank() == o.rank
        assert fro(g.dense().cpu().numpy() - o.dense()) <= 1e-8 * fro(H)


def test_recursive_dense_provider_parity(ctx, oracle):
    # test_lowrank.cpp:176-218 on the device path, plus oracle parity
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(7)
    ns, rows_per, cols = 6, 8, 50
    H = random_lowrank(rng, ns * rows_per, cols, 6, 1e-5)
    pos = np.array([[(s % 3) / 2.0, (s // 3) * 1.0] for s in range(ns)])
    tree = lr.ClusterTree(pos, [0, 0], [1, 1])
    otree = oracle.ClusterTree(pos, [0, 0], [1, 1])
    Ht = torch.as_tensor(H).cuda()

    class Prov:
        rows_per_source = rows_per
        cols = 50

        @staticmethod
        def block(s):
            return Ht[s * rows_per:(s + 1) * rows_per]

    eps = 1e-4
    rec = lr.recursive_lowrank(ctx, tree, eps, Prov, lr.RecursiveOptions(seed=0))
    orec = oracle.recursive_lowrank(otree, eps, H, rows_per, seed=0)
    Hp = np.zeros_like(H)
    Hp[rec.row_perm] = rec.factor.dense().cpu().numpy()
    assert fro(H - Hp) <= 50 * eps * fro(H)
    assert list(rec.node_rank) == list(orec.node_rank)
    assert np.array_equal(rec.row_perm, orec.row_perm)
    led = rec.ledger
    assert abs(led.category_total() - led.kernel_tally) <= 0.05 * led.kernel_tally
    assert led.leaf > 0 and led.agglomeration > 0
    assert abs(led.kernel_tally - orec.ledger[4]) <= 1e-9 * orec.ledger[4]


def test_recompress_lazy_root_matches_dense(ctx):
    """The recursion's root keeps V as Q [Z; 0] (LazyV); recompress factors
    the small Z instead of the tall V.  Same singular values / rank / J~ as
    recompressing the materialised copy of the same factor."""
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(11)
    ns, rows_per, cols = 4, 20, 3000   # tall W^T: the root takes the Q = I / tall-QR path
    H = random_lowrank(rng, ns * rows_per, cols, 40, 1e-7)
    pos = np.array([[(s % 2) * 1.0, (s // 2) * 1.0] for s in range(ns)])
    tree = lr.ClusterTree(pos, [0, 0], [1, 1])
    Ht = torch.as_tensor(H).cuda()

    class Prov:
        rows_per_source = rows_per
        cols = 3000

        @staticmethod
        def block(s):
            return Ht[s * rows_per:(s + 1) * rows_per]

    eps = 1e-9
    rec = lr.recursive_lowrank(ctx, tree, eps, Prov, lr.RecursiveOptions(seed=3))
    lazy = lr.recompress(ctx, rec.factor, eps)          # first use: the implicit V
    U, V = rec.factor.U, rec.factor.V                    # materialises V
    dense = lr.recompress(ctx, lr.LowRankFactor.from_tensors(ctx, U, V), eps)
    assert lazy.rank() == dense.rank()
    A, B = lazy.dense().cpu().numpy(), dense.dense().cpu().numpy()
    assert fro(A - B) <= 1e-12 * fro(B)
    assert fro(U.cpu().numpy() @ V.cpu().numpy().T - B) <= 1e-9 * fro(B)


def _lazy_root(ctx, seed=3):
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(11)
    ns, rows_per, cols = 4, 20, 3000
    H = random_lowrank(rng, ns * rows_per, cols, 40, 1e-7)
    pos = np.array([[(s % 2) * 1.0, (s // 2) * 1.0] for s in range(ns)])
    tree = lr.ClusterTree(pos, [0, 0], [1, 1])
    Ht = torch.as_tensor(H).cuda()

    class Prov:
        rows_per_source = rows_per
        cols = 3000

        @staticmethod
        def block(s):
            return Ht[s * rows_per:(s + 1) * rows_per]

    return lr.recursive_lowrank(ctx, tree, 1e-9, Prov, lr.RecursiveOptions(seed=seed)), H


def test_lazy_root_every_consumer_sees_the_same_factor(ctx, tmp_path):
    """Each consumer of a fresh (lazy-V) root factor materialises V first:
    device pointers, products, save, agglomerate -- all equal to the same
    operations on the materialised copy."""
    from paper_1410_0986_b200 import lowrank as lr
    ref_rec, _ = _lazy_root(ctx)
    U, V = ref_rec.factor.U, ref_rec.factor.V            # materialised copy
    X = torch.randn(3000, 2, dtype=torch.float64, device="cuda")
    want = U @ (V.T @ X)
    rec, _ = _lazy_root(ctx)                             # fresh lazy root each time
    assert float(torch.linalg.norm(lr.lr_matvec(ctx, rec.factor, X) - want)) <= 1e-12 * float(torch.linalg.norm(want))
    rec, _ = _lazy_root(ctx)
    up, vp = rec.factor.device_ptrs()
    assert bool(up) and bool(vp)  # non-NULL device pointers
    assert torch.equal(rec.factor.V, V)
    rec, _ = _lazy_root(ctx)
    path = str(tmp_path / "f.bin")
    lr.save_factor(path, rec.factor)
    g, _ = lr.load_factor(ctx, path)
    assert torch.equal(g.V, V) and torch.equal(g.U, U)
    rec, _ = _lazy_root(ctx)
    dense = lr.LowRankFactor.from_tensors(ctx, U, V)
    a = lr.agglomerate(ctx, rec.factor, dense, 1e-9, 5)
    b = lr.agglomerate(ctx, lr.LowRankFactor.from_tensors(ctx, U, V), dense, 1e-9, 5)
    assert a.rank() == b.rank()
    assert torch.equal(a.dense(), b.dense())


def test_born_pipeline_parity_small(ctx, oracle):
    """fields -> Born blocks -> recursive compression -> recompress -> J~ products,
    device vs oracle on identical (device-computed) fields."""
    from paper_1410_0986_b200 import born, configs, lowrank as lr
    cfg = configs.small_config(n=14, ns_x=4, ns_y=2, n_det=3, n_lambda=6)
    st = configs.make_setup(cfg)
    g = st.grid()
    F, stats = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points,
                                   tol=1e-10)
    w = torch.full((g.N,), cfg.h ** 3, dtype=torch.float64, device="cuda")
    inc = [F[st.source_point[s]] for s in range(cfg.n_sources)]
    adj = [[F[st.detector_point[s, d]] for d in range(cfg.n_det)] for s in range(cfg.n_sources)]
    tree = lr.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
    otree = oracle.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
    eps = configs.compression_tolerance(st, tree.depth())
    rec = lr.recursive_lowrank(ctx, tree, eps, lr.BornFieldsProvider(inc, adj, w, 1.0),
                               lr.RecursiveOptions(seed=cfg.seed))
    Fh = F.cpu().numpy()
    oinc = [Fh[st.source_point[s]].T for s in range(cfg.n_sources)]
    oadj = [[Fh[st.detector_point[s, d]].T for d in range(cfg.n_det)] for s in range(cfg.n_sources)]
    orec = oracle.recursive_lowrank_born(otree, eps, oinc, oadj, w.cpu().numpy(), 1.0, seed=cfg.seed)
    assert list(rec.node_rank) == list(orec.node_rank)
    H = np.vstack([oracle.born_block(oinc[s], oadj[s], w.cpu().numpy(), 1.0)
                   for s in range(cfg.n_sources)])
    Jg = np.zeros_like(H)
    Jg[rec.row_perm] = rec.factor.dense().cpu().numpy()
    Jo = np.zeros_like(H)
    Jo[orec.row_perm] = orec.factor.dense()
    assert fro(Jg - Jo) <= 1e-8 * fro(H)
    err_g, err_o = fro(H - Jg) / fro(H), fro(H - Jo) / fro(H)
    # both errors sit far below eps_d; compare them at the 1e-8 parity bar
    # with a roundoff floor (they are O(1e-14) at this fixture size)
    assert abs(err_g - err_o) <= 1e-8 * err_o + 1e-12
    # recompress (experiments.cpp:249-250)
    fr = lr.recompress(ctx, rec.factor, eps)
    of = oracle.recompress(orec.factor, eps)
    assert fr.rank() == of.rank
    assert fro(fr.dense().cpu().numpy() - of.dense()) <= 1e-8 * fro(H)
    # J~ products with the chromophore axis and permutation
    J = lr.JOperator(ctx, fr, rec.row_perm, st.eps_c)
    rng = np.random.default_rng(0)
    for b in (1, 5):
        X = rng.standard_normal((g.N * cfg.n_chrom, b))
        yg = J.matvec(torch.as_tensor(X)).cpu().numpy()
        yo = oracle.j_matmat(of, X, orec.row_perm, st.eps_c)
        assert fro(yg - yo) <= 1e-10 * fro(yo)
        Y = rng.standard_normal((cfg.M, b))
        xg = J.rmatvec(torch.as_tensor(Y)).cpu().numpy()
        xo = oracle.j_matmat(of, Y, orec.row_perm, st.eps_c, trans=True)
        assert fro(xg - xo) <= 1e-10 * fro(xo)
        # adjoint consistency (test_lowrank.cpp:272-287)
        assert np.sum(Y * yg) == pytest.approx(np.sum(X * xg), rel=1e-12)


def test_lr_matvec_adjoint(ctx):
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(10)
    A = random_lowrank(rng, 22, 31, 5)
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    f = lr.LowRankFactor.from_tensors(ctx, torch.as_tensor(U[:, :5]), torch.as_tensor(Vt[:5].T * s[:5]))
    for _ in range(5):
        x, y = rng.standard_normal(31), rng.standard_normal(22)
        a = y @ lr.lr_matvec(ctx, f, torch.as_tensor(x)).cpu().numpy()
        b = x @ lr.lr_rmatvec(ctx, f, torch.as_tensor(y)).cpu().numpy()
        assert a == pytest.approx(b, rel=1e-12)
        assert fro(lr.lr_matvec(ctx, f, torch.as_tensor(x)).cpu().numpy() - A @ x) <= 1e-10 * fro(A @ x)
    with pytest.raises(ValueError):
        lr.lr_matvec(ctx, f, torch.zeros(30, dtype=torch.float64))


@pytest.mark.parametrize("b", [1, 2, 3, 5, 8, 13, 16, 17, 64])
def test_lr_matmat_widths(ctx, b):
    """skinny (b <= 16) and DMMA (b > 16) paths of U (V^T X) / V (U^T Y)."""
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(b)
    M, N, R = 700, 40000, 123
    U = rng.standard_normal((M, R))
    V = rng.standard_normal((N, R))
    f = lr.LowRankFactor.from_tensors(ctx, torch.as_tensor(U), torch.as_tensor(V))
    X = rng.standard_normal((N, b))
    Y = rng.standard_normal((M, b))
    want = U @ (V.T @ X)
    got = lr.lr_matmat if False else lr.lr_matvec(ctx, f, torch.as_tensor(X)).cpu().numpy()
    assert fro(got - want) <= 1e-13 * fro(want)
    want2 = V @ (U.T @ Y)
    got2 = lr.lr_rmatvec(ctx, f, torch.as_tensor(Y)).cpu().numpy()
    assert fro(got2 - want2) <= 1e-13 * fro(want2)


def test_voxel_engine_on_device_matches_the_library(ctx):
    """voxel.py's cooperative merge with the device kernels (DMMA GEMM,
    Householder QR, Jacobi SVD, device Gaussian stream) on one rank equals
    the library's agglomerate / recompress to rounding."""
    from paper_1410_0986_b200 import lowrank as lr, voxel as vx
    rng = np.random.default_rng(21)
    N = 4000
    fac = []
    for m in (60, 48):
        k = 40
        Q1, _ = np.linalg.qr(rng.standard_normal((m, k)))
        Q2, _ = np.linalg.qr(rng.standard_normal((N, k)))
        fac.append((Q1, Q2 * np.logspace(0, -9, k)))
    fac[1] = (fac[1][0], 0.5 * fac[0][1] + 0.5 * fac[1][1])
    ops = vx.DeviceOps(ctx)
    comm = vx.SimComm.group(1)[0]
    for hint in (-1, 200):
        f1 = vx.VFactor(ops.tensor(fac[0][0]), ops.tensor(fac[0][1]), N)
        f2 = vx.VFactor(ops.tensor(fac[1][0]), ops.tensor(fac[1][1]), N)
        fv = vx.agglomerate_voxel(ops, comm, f1, f2, 0, N, 1e-7, seed=99, rank_hint=hint)
        g1 = lr.LowRankFactor.from_tensors(ctx, torch.as_tensor(fac[0][0]), torch.as_tensor(fac[0][1]))
        g2 = lr.LowRankFactor.from_tensors(ctx, torch.as_tensor(fac[1][0]), torch.as_tensor(fac[1][1]))
        fg = lr.agglomerate(ctx, g1, g2, 1e-7, 99, rank_hint=hint)
        assert fv.rank == fg.rank()
        D = (fv.U @ fv.V_loc.T).cpu().numpy()
        Dg = fg.dense().cpu().numpy()
        assert fro(D - Dg) <= 1e-10 * fro(Dg)
        fr = vx.recompress_voxel(ops, comm, fv, 1e-7)
        fgr = lr.recompress(ctx, fg, 1e-7)
        assert fr.rank == fgr.rank()
        assert fro((fr.U @ fr.V_loc.T).cpu().numpy() - fgr.dense().cpu().numpy()) <= 1e-10 * fro(Dg)


def test_library_comm_j_matmat_voxel_single_rank(ctx):
    """hydot_comm (NCCL handle of the C ABI) and hydot_j_matmat_voxel on one
    rank reproduce hydot_j_matmat (the all-reduce is the identity)."""
    from paper_1410_0986_b200 import lowrank as lr, voxel as vx
    rng = np.random.default_rng(8)
    M, N, R, nl, nc, b = 90, 700, 17, 9, 3, 5
    U, V = rng.standard_normal((M, R)), rng.standard_normal((N, R))
    f = lr.LowRankFactor.from_tensors(ctx, torch.as_tensor(U), torch.as_tensor(V))
    perm = rng.permutation(M).astype(np.int32)
    eps_c = rng.uniform(0.5, 1.5, (nl, nc))
    J = lr.JOperator(ctx, f, perm, eps_c)
    comm = vx.LibComm(ctx)
    X = torch.as_tensor(rng.standard_normal((b, N * nc))).cuda()
    Y = torch.empty(b, M, dtype=torch.float64, device="cuda")
    J.matmat_cm(X, Y, b)
    Yv = vx.j_matmat_voxel_lib(comm, torch.as_tensor(U).cuda(), torch.as_tensor(V).cuda(), J.row_perm,
                               J.eps_c, nl, nc, X)
    assert float(torch.max(torch.abs(Yv - Y))) <= 1e-12 * float(torch.max(torch.abs(Y)))
    Xb = torch.empty(b, N * nc, dtype=torch.float64, device="cuda")
    J.rmatmat_cm(Y, Xb, b)
    Xv = vx.j_matmat_voxel_lib(comm, torch.as_tensor(U).cuda(), torch.as_tensor(V).cuda(), J.row_perm,
                               J.eps_c, nl, nc, Y, trans=True)
    assert float(torch.max(torch.abs(Xv - Xb))) <= 1e-12 * float(torch.max(torch.abs(Xb)))
    z = torch.arange(6, dtype=torch.float64, device="cuda")
    assert torch.equal(comm.allreduce(z), z)


def test_streamed_fields_provider_equals_resident_fields(ctx):
    """born.StreamedFieldsProvider (config 3's per-source CG -> block -> drop)
    gives the same compression as the provider over resident fields: every
    CG system is independent of the batch it runs in."""
    from paper_1410_0986_b200 import born, configs, lowrank as lr
    cfg = configs.small_config(n=12, ns_x=2, ns_y=2, n_det=2, n_lambda=4)
    st = configs.make_setup(cfg)
    g = st.grid()
    F, _ = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points, tol=1e-10)
    w = torch.full((g.N,), cfg.h ** 3, dtype=torch.float64, device="cuda")
    tree = lr.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
    eps = configs.compression_tolerance(st, tree.depth())
    inc = [F[st.source_point[s]] for s in range(cfg.n_sources)]
    adj = [[F[st.detector_point[s, d]] for d in range(cfg.n_det)] for s in range(cfg.n_sources)]
    r1 = lr.recursive_lowrank(ctx, tree, eps, lr.BornFieldsProvider(inc, adj, w, 1.0),
                              lr.RecursiveOptions(seed=cfg.seed))
    prov = born.StreamedFieldsProvider(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.source_vertex,
                                       st.detector_vertex, w, 1.0, tol=1e-10)
    r2 = lr.recursive_lowrank(ctx, tree, eps, prov, lr.RecursiveOptions(seed=cfg.seed))
    assert list(r1.node_rank) == list(r2.node_rank)
    assert len(prov.log) == cfg.n_sources and max(e["relres_max"] for e in prov.log) <= 1e-10
    D1, D2 = r1.factor.dense(), r2.factor.dense()
    assert float(torch.linalg.norm(D1 - D2)) <= 1e-13 * float(torch.linalg.norm(D1))


# ---- matrix-free LinOp (lowrank.hpp:56-63; hydot_randsvd_linop) -------------
@pytest.mark.gpu
@pytest.mark.parametrize("m,n,r,noise,eps,r0,block", [
    (60, 400, 8, 0.0, 1e-8, 1, True),       # exact rank, block products
    (60, 400, 8, 0.0, 1e-8, 1, False),      # the same through mv / rmv column by column
    (40, 55, 7, 0.0, 1e-10, 1, True),       # Q = I branch: A^T = rmm(I)
    (200, 3000, 12, 1e-9, 1e-6, 1, True),   # adaptive sketch: several passes
    (80, 32768, 30, 1e-8, 6.6e-9, 43, True),
])
def test_randsvd_linop_matches_dense_and_oracle(ctx, oracle, m, n, r, noise, eps, r0, block):
    from paper_1410_0986_b200 import lowrank as lr
    from paper_1410_0986_b200._lib import Ledger
    rng = np.random.default_rng(m + n)
    A = random_lowrank(rng, m, n, r, noise) * np.exp(-np.arange(n) / n)[None, :]
    Ad = torch.as_tensor(A).to(f"cuda:{ctx.device}")
    calls = {"mv": 0, "rmv": 0, "mm": 0, "rmm": 0}

    def count(name, fn):
        def g(x):
            calls[name] += 1
            return fn(x)
        return g
    op = lr.LinOp(rows=m, cols=n, mv=count("mv", lambda x: Ad @ x), rmv=count("rmv", lambda y: Ad.T @ y))
    if block:
        op.mm = count("mm", lambda X: Ad @ X)
        op.rmm = count("rmm", lambda Y: Ad.T @ Y)
    seed = 20240811 + 0x9e3779b97f4a7c15
    lo, ld = Ledger(), Ledger()
    fo = oracle.randsvd(A, eps, 20, 10, seed, oracle.LEAF, r0)
    fd = lr.randsvd(ctx, A, eps, 20, 10, seed, ledger=ld, cat=lr.LEAF, r0=r0)
    fg = lr.randsvd(ctx, op, eps, 20, 10, seed, ledger=lo, cat=lr.LEAF, r0=r0)
    assert fg.rank() == fo.rank == fd.rank()
    assert fg.flagged == fo.flagged
    Dg = fg.dense().cpu().numpy()
    assert fro(Dg - fo.dense()) <= 1e-8 * fro(A)
    assert fro(Dg - fd.dense().cpu().numpy()) <= 1e-10 * fro(A)
    sg = np.linalg.norm(fg.V.cpu().numpy(), axis=0)
    so = np.linalg.norm(fo.V, axis=0)
    assert np.all(np.abs(sg - so) <= 1e-8 * so[0])
    # apply_mm charges the same flops whichever form runs (lowrank.cpp:95-98)
    assert lo.leaf == ld.leaf and lo.kernel_tally == ld.kernel_tally
    if block:
        assert calls["mv"] == calls["rmv"] == 0 and calls["mm"] >= 0 and calls["rmm"] == 1
    else:
        assert calls["mm"] == calls["rmm"] == 0 and calls["rmv"] >= fg.rank()


@pytest.mark.gpu
def test_randsvd_linop_matrix_free_product_operator(ctx, oracle):
    # an operator that is never formed: A = diag(w) L R^T diag(c)
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(11)
    m, n, k = 96, 5000, 9
    L, R = rng.standard_normal((m, k)), rng.standard_normal((n, k))
    w, cs = np.exp(rng.standard_normal(m)), np.exp(-np.arange(n) / n)
    dev = f"cuda:{ctx.device}"
    Ld, Rd, wd, cd = (torch.as_tensor(a).to(dev) for a in (L, R, w, cs))
    op = lr.LinOp(rows=m, cols=n,
                  mm=lambda X: wd[:, None] * (Ld @ (Rd.T @ (cd[:, None] * X))),
                  rmm=lambda Y: cd[:, None] * (Rd @ (Ld.T @ (wd[:, None] * Y))))
    A = (w[:, None] * (L @ R.T)) * cs[None, :]
    fo = oracle.randsvd(A, 1e-9, 20, 10, 5, oracle.OTHER, 1)
    fg = lr.randsvd(ctx, op, 1e-9, 20, 10, 5)
    assert fg.rank() == fo.rank == k
    assert fro(fg.dense().cpu().numpy() - A) <= 10 * 1e-9 * fro(A)   # test_lowrank.cpp:48-63 bound
    assert fro(fg.dense().cpu().numpy() - fo.dense()) <= 1e-8 * fro(A)


@pytest.mark.gpu
def test_randsvd_linop_errors(ctx):
    from paper_1410_0986_b200 import lowrank as lr
    with pytest.raises(ValueError):
        lr.randsvd(ctx, lr.LinOp(rows=4, cols=5), 1e-6)            # no products at all
    with pytest.raises(ValueError):
        lr.randsvd(ctx, lr.LinOp(rows=4, cols=5, mv=lambda x: x), 1e-6)   # no adjoint

    def boom(X):
        raise KeyError("operator failed")
    with pytest.raises(KeyError):
        lr.randsvd(ctx, lr.LinOp(rows=4, cols=50, mm=boom, rmm=boom), 1e-6)
    f = lr.randsvd(ctx, lr.LinOp(rows=0, cols=5), 1e-6)            # lowrank.cpp:148-152
    assert f.rank() == 0


# ---- rejected sketch passes decided by the QR lower bound --------------------
def _graded(rng, m, n, decades):
    Q1, _ = np.linalg.qr(rng.standard_normal((m, m)))
    Q2, _ = np.linalg.qr(rng.standard_normal((n, m)))
    return (Q1 * np.logspace(0, -decades, m)) @ Q2.T


@pytest.mark.parametrize("m,n,decades,eps,r0,expect_bound", [
    (900, 6000, 10.0, 3e-10, 700, True),    # merge-like: slow decay, pass at r = 700 rejected (er ~ 7 thr), then Q = I
    (1300, 5000, 11.0, 3e-10, 950, True),   # er ~ 4.7 thr
    (1300, 5000, 11.0, 3e-10, 1000, None),  # er ~ 1.8 thr: the bound may or may not decide
    (900, 6000, 30.0, 3e-10, 700, False),   # fast decay: the pass is accepted (bound undecided -> full path)
])
def test_reject_bound_same_result_as_full_evaluation(ctx, oracle, capfd, monkeypatch, m, n, decades, eps, r0,
                                                     expect_bound):
    from paper_1410_0986_b200 import lowrank as lr
    from paper_1410_0986_b200._lib import Ledger
    rng = np.random.default_rng(m + r0)
    A = _graded(rng, m, n, decades)
    monkeypatch.setenv("HYDOT_TRACE_RANDSVD", "1")
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("HYDOT_REJECT_BOUND", mode)
        led = Ledger()
        capfd.readouterr()
        f = lr.randsvd(ctx, A, eps, 20, 10, 99, ledger=led, cat=lr.AGGLOMERATION, r0=r0)
        out[mode] = (f, led, capfd.readouterr().err)
    f0, l0, t0 = out["0"]
    f1, l1, t1 = out["1"]
    assert "(bound)" not in t0 and "undecided" not in t0
    # the decision sequence (accept / reject per pass, Q = I) is the same
    seq = lambda t: [("reject" if "reject" in ln else "accept" if "accept" in ln else "identity")
                     for ln in t.splitlines() if ln.startswith("[randsvd]") and "undecided" not in ln]
    assert seq(t0) == seq(t1)
    if expect_bound is not None:
        assert ("reject (bound)" in t1) == expect_bound   # the shortcut decided this pass
    assert f1.rank() == f0.rank() and f1.flagged == f0.flagged
    assert l1.kernel_tally == l0.kernel_tally and l1.agglomeration == l0.agglomeration
    D0, D1 = f0.dense().cpu().numpy(), f1.dense().cpu().numpy()
    if "reject (bound)" in t1 and "accept" not in t1:
        assert np.array_equal(D0, D1)          # a rejected pass leaves no trace in the result
    else:
        assert fro(D0 - D1) <= 1e-12 * fro(A)
    fo = oracle.randsvd(A, eps, 20, 10, 99, oracle.AGGLOMERATION, r0)
    assert f1.rank() == fo.rank and f1.flagged == fo.flagged
    assert fro(D1 - fo.dense()) <= 1e-8 * fro(A)


# ---- CholeskyQR panels that give up: the deferred Householder redo ----------
def test_speculative_tall_qr_redo_on_rank_deficient_input(ctx):
    # an exactly rank-deficient A with a tolerance no sketch pass can meet: the pass is
    # rejected, the Q = I branch consumes the speculative QR of A^T started on the side
    # stream, whose CholeskyQR panels cannot orthonormalise dependent columns -- the
    # consumer must notice (geqrf_verify) and redo it with Householder panels
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(21)
    m, n, k = 100, 20000, 10
    A = rng.standard_normal((m, k)) @ rng.standard_normal((k, n))
    f = lr.randsvd(ctx, A, 1e-17, 20, 10, 3, r0=60)
    assert f.rank() >= k
    assert fro(f.dense().cpu().numpy() - A) <= 1e-12 * fro(A)
    s = np.linalg.norm(f.V.cpu().numpy(), axis=0)
    s_ref = np.linalg.svd(A, compute_uv=False)
    assert np.all(np.abs(s[:k] - s_ref[:k]) <= 1e-12 * s_ref[0])


def test_recompress_redo_on_rank_deficient_factor(ctx, oracle):
    # QR(U) of recompress runs on the side stream with deferred verification
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(22)
    M, N, r, k = 3000, 5000, 64, 6
    U = rng.standard_normal((M, k)) @ rng.standard_normal((k, r))      # rank 6 of 64 columns
    V = rng.standard_normal((N, r))
    g = lr.LowRankFactor.from_tensors(ctx, torch.as_tensor(U), torch.as_tensor(V))
    out = lr.recompress(ctx, g, 1e-10)
    H = U @ V.T
    assert out.rank() == k
    assert fro(out.dense().cpu().numpy() - H) <= 1e-10 * fro(H)
    o = oracle.recompress(oracle.Factor.make(U, V), 1e-10)
    assert o.rank == out.rank()
