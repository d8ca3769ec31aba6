"""Block one-sided Jacobi (bjacobi.cu: DMMA pair Grams, pair eigen-solve,
DMMA column update) on the path's large cores, against the oracle.

randsvd with r0 + p >= m takes the Q = I branch (lowrank.cpp:159-164), whose
core is the R factor of the presorted tall QR of A^T: an m x m SVD, above the
block driver's threshold for m >= 1800.  Parity with the oracle's LAPACK
(dgeqrf + dgesdd for Eigen's HouseholderQR + BDCSVD): equal kept rank,
singular values within 1e-8 relative (leading) and 1e-12 s_1 (all),
||U_g V_g^T - U_o V_o^T||_F <= 1e-8 ||A||_F.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1410_0986_b200 as h
    return h.Context(0)


def graded(rng, m, n, decades, clusters=False):
    k = min(m, n)
    Q1, _ = np.linalg.qr(rng.standard_normal((m, k)))
    Q2, _ = np.linalg.qr(rng.standard_normal((n, k)))
    s = np.logspace(0, -decades, k)
    if clusters:  # pairs and triples of nearly equal singular values
        s[1::3] = s[0::3][: len(s[1::3])] * (1 + 1e-9)
    return (Q1 * s) @ Q2.T, s


@pytest.mark.parametrize("m,n,decades,clusters", [(1900, 9000, 14, False), (2100, 12000, 12, True),
                                                  (2600, 16000, 16, False)])
def test_block_jacobi_core_matches_oracle(ctx, oracle, m, n, decades, clusters):
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(m)
    A, s = graded(rng, m, n, decades, clusters)
    eps = 1e-10
    fo = oracle.randsvd(A, eps, 20, 10, 11, oracle.LEAF, m)
    fg = lr.randsvd(ctx, A, eps, 20, 10, 11, cat=lr.LEAF, r0=m)
    assert fg.rank() == fo.rank
    sg = torch.linalg.norm(fg.V, dim=0).cpu().numpy()
    so = np.linalg.norm(fo.V, axis=0)
    assert np.max(np.abs(sg[:20] - so[:20]) / so[:20]) <= 1e-8
    assert np.max(np.abs(sg - so)) <= 1e-12 * so[0]
    Dg = (fg.U @ fg.V.T).cpu().numpy()
    nA = np.linalg.norm(A)
    assert np.linalg.norm(Dg - fo.dense()) <= 1e-8 * nA
    # the factor's leading U columns are orthonormal (the lazy-V recovery
    # V = X^T W S^-2 carries eps ||X|| / s_j per column: only columns with
    # s_j well above eps s_1 are orthonormal to working precision)
    k = int(np.sum(sg > 1e-4 * sg[0]))
    U = fg.U[:, :k]
    G = U.T @ U
    assert float(torch.max(torch.abs(G - torch.eye(k, dtype=G.dtype, device=G.device)))) <= 1e-9


def test_block_jacobi_thin_svd_square(ctx):
    """thin_svd on a graded square core through the lazy path: singular values
    against the exact ones, U orthonormal, U S V^T = A."""
    import os
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(5)
    n = 2000
    A, s = graded(rng, n, n, 12)
    os.environ["HYDOT_THIN_SVD_PATH"] = "1"
    try:
        U, sv, V = lr.thin_svd(ctx, torch.as_tensor(A).cuda())
    finally:
        del os.environ["HYDOT_THIN_SVD_PATH"]
    sv = np.asarray(sv)
    assert np.max(np.abs(sv - s)) <= 1e-13 * s[0]
    R = (U * torch.as_tensor(sv, device=U.device)) @ V.T
    assert float(torch.linalg.norm(R - torch.as_tensor(A, device=R.device))) <= 1e-12 * np.linalg.norm(A)
