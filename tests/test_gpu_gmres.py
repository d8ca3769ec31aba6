"""Device recycled shifted-family solver (csrc/gmres.cu) against the CPU
oracle (oracle/krylov_oracle.cpp, itself pinned by the reference's
test_krylov.cpp cases in tests/test_krylov_oracle.py) and against dense direct
solves, on the reference's test family (test_krylov.cpp:14-45).

Bar: the device runs the reference's algorithm (same phase-1 step count,
same deflation dimension, same convergence decisions up to rounding), so its
solutions agree with the oracle's and with the direct solves to the
reference's own test tolerance 1e-7 at tol = 1e-10, every relres <= tol, and
the phase-2 iteration counts agree within a restart cycle's rounding
(|delta| <= 2 per shift)."""
import numpy as np
import pytest
import torch

from krylov_fixture import dense_system, small_family

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1410_0986_b200 as h
    return h.Context(0)


def _dev(ctx, geom, b, sh, **kw):
    from paper_1410_0986_b200 import krylov
    bt = torch.as_tensor(b, device="cuda:0")
    return krylov.solve_family(ctx, geom, bt, sh, krylov.SolverConfig(**kw))[0]


def _cmp(r, o, sh, geom, b, tol_x=1e-7, it_slack=2, direct=True):
    X = r.X.cpu().numpy().T
    assert r.all_converged and o["all_converged"]
    assert r.phase1_matvecs == o["phase1_steps"]
    assert r.deflation_k == o["defl_k"]
    for j in range(len(sh)):
        assert r.stats[j].relres <= 1e-10 or r.stats[j].relres <= o["relres"][j] * 10
        assert np.linalg.norm(X[:, j] - o["X"][:, j]) <= tol_x * np.linalg.norm(o["X"][:, j])
        assert abs(r.stats[j].iterations - int(o["iters"][j])) <= it_slack, (j, r.stats[j], o["iters"][j])
        if direct:
            xd = np.linalg.solve(dense_system(geom, sh[j]), b)
            assert np.linalg.norm(X[:, j] - xd) <= tol_x * np.linalg.norm(xd)


@pytest.mark.parametrize("n,nl", [(6, 10), (8, 20)])
def test_solve_family_matches_oracle_and_direct(ctx, oracle, n, nl):
    """test_krylov.cpp:173-186 on the device, against the oracle."""
    geom, sh, b = small_family(n, nl)
    r = _dev(ctx, geom, b, sh, tol=1e-10)
    o = oracle.krylov_solve_family(geom, b, sh, oracle.SolverConfig(tol=1e-10))
    _cmp(r, o, sh, geom, b)
    for j in range(nl):
        assert abs(r.stats[j].phase1_relres - o["phase1_relres"][j]) <= 1e-6 * max(o["phase1_relres"][j], 1e-12) \
            or max(r.stats[j].phase1_relres, o["phase1_relres"][j]) <= 1e-9


def test_solve_family_jacobi(ctx, oracle):
    """test_krylov.cpp:188-200: the Jacobi right preconditioner."""
    geom, sh, b = small_family(6, 4)
    r = _dev(ctx, geom, b, sh, tol=1e-10, jacobi=True)
    o = oracle.krylov_solve_family(geom, b, sh, oracle.SolverConfig(tol=1e-10, jacobi=True))
    _cmp(r, o, sh, geom, b)


def test_recycling_reduces_iterations_on_device(ctx, oracle):
    """test_krylov.cpp:202-218: deflation (k = 10) needs fewer iterations
    than none, with a short phase-1 basis; both match the oracle."""
    geom, sh, b = small_family(8, 20)
    kw = dict(arnoldi_steps=25, restart=25)
    rw = _dev(ctx, geom, b, sh, deflation_dim=10, **kw)
    rwo = _dev(ctx, geom, b, sh, deflation_dim=0, **kw)
    ow = oracle.krylov_solve_family(geom, b, sh, oracle.SolverConfig(deflation_dim=10, **kw))
    owo = oracle.krylov_solve_family(geom, b, sh, oracle.SolverConfig(deflation_dim=0, **kw))
    assert sum(s.iterations for s in rw.stats) < sum(s.iterations for s in rwo.stats)
    _cmp(rw, ow, sh, geom, b, tol_x=1e-6, direct=False)
    _cmp(rwo, owo, sh, geom, b, tol_x=1e-6, direct=False)


def test_explicit_qr_update_path(ctx, oracle):
    """ShiftedDeflation's QR path (krylov.cpp:237-246) via explicit_qr_update."""
    geom, sh, b = small_family(8, 6)
    kw = dict(arnoldi_steps=25, restart=25, tol=1e-10)
    r = _dev(ctx, geom, b, sh, explicit_qr_update=True, **kw)
    o = oracle.krylov_solve_family(geom, b, sh, oracle.SolverConfig(explicit_qr_update=True, **kw))
    _cmp(r, o, sh, geom, b)
    r2 = _dev(ctx, geom, b, sh, **kw)
    X1, X2 = r.X.cpu().numpy(), r2.X.cpu().numpy()
    assert np.linalg.norm(X1 - X2) <= 1e-7 * np.linalg.norm(X2)


def test_deterministic_and_batch_invariant(ctx):
    """test_krylov.cpp:220-235 (bitwise repeatable); a batch of right-hand
    sides gives each one exactly its single-rhs solution."""
    from paper_1410_0986_b200 import krylov
    from oracle import oracle as o
    geom, sh, b = small_family(7, 6)
    b2 = o.fem_point_source(geom, [-0.9, 0.4, 0.0])
    b3 = o.fem_point_source(geom, [1.1, 1.3, 1.0])
    B = torch.as_tensor(np.stack([b, b2, b3]), device="cuda:0")
    cfg = krylov.SolverConfig(arnoldi_steps=30, restart=20)
    rs = krylov.solve_family(ctx, geom, B, sh, cfg)
    rs2 = krylov.solve_family(ctx, geom, B, sh, cfg)
    for a, c in zip(rs, rs2):
        assert torch.equal(a.X, c.X)
    for i in range(3):
        one = krylov.solve_family(ctx, geom, B[i], sh, cfg)[0]
        assert torch.equal(one.X, rs[i].X)
        assert [s.iterations for s in one.stats] == [s.iterations for s in rs[i].stats]


def test_fields_gmres_matches_cg_fields(ctx, oracle):
    """compute_fields (born.cpp:39-80) with the recycled solver equals the CG
    fields of the same FEM family within the solve tolerance."""
    from paper_1410_0986_b200 import born, krylov
    geom, sh, _ = small_family(10, 8)
    invd = 1.0 / (1.0 + np.arange(len(sh)))
    pts = np.array([[0.2, -0.3, 2.0], [-1.0, 0.5, 0.0], [0.7, 0.7, 1.1]])
    F, fam = krylov.compute_fields_fem_gmres(ctx, geom, sh[:, 0], sh[:, 1], invd, pts,
                                             krylov.SolverConfig(tol=1e-10))
    Fc, st = born.compute_fields_fem(ctx, geom, sh[:, 0], sh[:, 1], invd, pts, tol=1e-12)
    d = (F - Fc).norm(dim=2) / Fc.norm(dim=2)
    assert float(d.max()) <= 1e-7
    assert all(f.all_converged for f in fam)


def test_zero_rhs_raises(ctx):
    from paper_1410_0986_b200 import krylov
    geom, sh, b = small_family(5, 2)
    with pytest.raises(ValueError, match="nonzero"):
        krylov.solve_family(ctx, geom, torch.zeros(len(b), dtype=torch.float64, device="cuda:0"), sh)
