"""The reference's test_krylov.cpp, restated against the CPU oracle
(oracle/krylov_oracle.cpp), so the oracle is pinned by the reference's own
known-answer and bound checks before it is used as the checker of the device
solver (tests/test_gpu_gmres.py).  Every case cites its reference test."""
import numpy as np
import pytest
import scipy.linalg as sla

from krylov_fixture import dense_system, small_family
from oracle import oracle as o


def _sbar(sh):
    return float(np.mean(sh[:, 1]))


def test_multishift_matches_dense_direct_solves():
    """test_krylov.cpp:47-63: one Arnoldi basis, every shift within 1e-7 of
    the direct solve, least-squares residual <= 1e-10."""
    geom, sh, b = small_family(6, 1)
    sigmas = [sh[0, 0], 2 * sh[0, 0], 0.5, 3.0]
    X, rel, V, T, _ = o.krylov_multishift(geom, sh[0, 1], b, sigmas, 120, 1e-10)
    _, d = o.krylov_apply(geom, sh[0, 1], b)
    bs = d * b
    for j, s in enumerate(sigmas):
        Ks = np.column_stack([o.krylov_apply(geom, sh[0, 1], e)[0] for e in np.eye(len(b))])
        xd = np.linalg.solve(Ks + s * np.eye(len(b)), bs)
        assert np.linalg.norm(X[:, j] - xd) <= 1e-7 * np.linalg.norm(xd)
        assert rel[j] <= 1e-10


def test_arnoldi_relation_and_orthonormal_basis():
    """test_krylov.cpp:65-83: Ks V_s = V_{s+1} Tbar, V orthonormal, beta = |bs|."""
    geom, sh, b = small_family(5, 1)
    X, rel, V, T, _ = o.krylov_multishift(geom, sh[0, 1], b, [sh[0, 0]], 40, 1e-14)
    s = T.shape[1]
    assert s > 0
    KV = np.column_stack([o.krylov_apply(geom, sh[0, 1], V[:, j])[0] for j in range(s)])
    kn = np.linalg.norm(np.column_stack([o.krylov_apply(geom, sh[0, 1], e)[0] for e in np.eye(len(b))]))
    assert np.linalg.norm(KV - V @ T) <= 1e-10 * kn
    assert np.linalg.norm(V.T @ V - np.eye(s + 1)) <= 1e-10


def test_harmonic_ritz_matches_dense_pencil():
    """test_krylov.cpp:85-125: retained |theta| ascending, the smallest equal
    to the pencil's smallest, each one a pencil eigenvalue (1e-6)."""
    geom, sh, b = small_family(5, 1)
    _, _, V, T, _ = o.krylov_multishift(geom, sh[0, 1], b, [sh[0, 0]], 40, 1e-14)
    s = T.shape[1]
    Z, th, _ = o.krylov_harmonic_ritz(T, 6)
    assert Z.shape[0] == s
    w = sla.eigvals(T.T @ T, T[:s, :s].T)
    mags = np.sort(np.abs(w))
    assert np.all(th[:-1] <= th[1:] * (1 + 1e-12))
    assert abs(th[0] - mags[0]) <= 1e-6 * mags[0]
    for t in th:
        assert np.min(np.abs(mags - t) / np.maximum(1.0, mags)) <= 1e-6


def test_deflation_basis_and_shifted_pair():
    """test_krylov.cpp:127-171: Ks U = C, C orthonormal; A_j U_j = C_j with
    C_j orthonormal; the Gram/Cholesky and QR paths span the same space."""
    geom, sh, b = small_family(6, 8)
    sbar = _sbar(sh)
    _, _, V, T, _ = o.krylov_multishift(geom, sbar, b, list(sh[:, 0]), 60, 1e-8)
    Z, th, _ = o.krylov_harmonic_ritz(T, 10)
    U, Cm, RU, _ = o.krylov_deflation(geom, sbar, V, T, Z)
    k = U.shape[1]
    assert k >= 1
    KU = np.column_stack([o.krylov_apply(geom, sbar, U[:, j])[0] for j in range(k)])
    assert np.linalg.norm(KU - Cm) <= 1e-8 * np.linalg.norm(Cm)
    assert np.linalg.norm(Cm.T @ Cm - np.eye(k)) <= 1e-8
    RU2 = np.column_stack([o.krylov_apply(geom, sbar, U[:, j], which=1)[0] for j in range(k)])
    assert np.array_equal(RU, RU2)
    sg, sp = sh[3, 0], sh[3, 1] - sbar
    Cg, Ug, failed = o.krylov_shifted_dense(U, Cm, RU, sg, sp, False)
    Cq, _, _ = o.krylov_shifted_dense(U, Cm, RU, sg, sp, True)
    assert not failed
    AU = np.column_stack([o.krylov_apply(geom, sbar, Ug[:, j], sg, sp)[0] for j in range(k)])
    assert np.linalg.norm(AU - Cg) <= 1e-7 * np.linalg.norm(Cg)
    assert np.linalg.norm(Cg.T @ Cg - np.eye(k)) <= 1e-8
    assert np.linalg.norm(Cg @ Cg.T - Cq @ Cq.T) <= 1e-7


@pytest.mark.parametrize("jacobi,nl", [(False, 10), (True, 4)])
def test_solve_family_matches_direct_solves(jacobi, nl):
    """test_krylov.cpp:173-200: every shift within 1e-7 of the direct solve,
    relres <= 1e-10 (with and without the Jacobi right preconditioner)."""
    geom, sh, b = small_family(6, nl)
    r = o.krylov_solve_family(geom, b, sh, o.SolverConfig(tol=1e-10, jacobi=jacobi))
    assert r["all_converged"]
    for j in range(nl):
        xd = np.linalg.solve(dense_system(geom, sh[j]), b)
        assert np.linalg.norm(r["X"][:, j] - xd) <= 1e-7 * np.linalg.norm(xd)
        assert r["relres"][j] <= 1e-10


def test_recycling_reduces_iterations():
    """test_krylov.cpp:202-218: a short phase-1 basis leaves work for the
    per-shift solves; deflation (k = 10) needs fewer total iterations."""
    geom, sh, b = small_family(8, 20)
    w = o.krylov_solve_family(geom, b, sh, o.SolverConfig(arnoldi_steps=25, restart=25, deflation_dim=10))
    wo = o.krylov_solve_family(geom, b, sh, o.SolverConfig(arnoldi_steps=25, restart=25, deflation_dim=0))
    assert w["all_converged"] and wo["all_converged"]
    assert w["iters"].sum() < wo["iters"].sum()


def test_solve_family_deterministic_and_thread_invariant():
    """test_krylov.cpp:220-235: bitwise repeatable, and identical with 4 threads."""
    geom, sh, b = small_family(5, 6)
    a = o.krylov_solve_family(geom, b, sh, o.SolverConfig())
    c = o.krylov_solve_family(geom, b, sh, o.SolverConfig())
    d = o.krylov_solve_family(geom, b, sh, o.SolverConfig(threads=4))
    assert np.array_equal(a["X"], c["X"])
    assert np.array_equal(a["X"], d["X"])


def test_zero_rhs_raises():
    """multishift_gmres: b must be nonzero (krylov.cpp:49-50)."""
    geom, sh, b = small_family(5, 2)
    with pytest.raises(ValueError, match="nonzero"):
        o.krylov_solve_family(geom, np.zeros_like(b), sh)
