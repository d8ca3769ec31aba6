"""The reference's own field operator (trilinear FEM, grid.cpp:12-174) and
point sources (grid.cpp:212-237, born.cpp:27-35): the oracle restatement is
pinned to closed-form element matrices and to a literal restatement of the
reference's triplet assembly; the device FEM mode is checked against it."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc

GEOMS = [(5, 4, 4, 2.0, 1.5, 3.0), (6, 5, 3, 3.0, 3.0, 2.0), (4, 4, 5, 1.0, 2.0, 4.0)]


def _1d(h):
    k = np.array([[1, -1], [-1, 1]]) / h
    m = np.array([[2, 1], [1, 2]]) * h / 6
    return k, m


def test_element_matrices_closed_form():
    hx, hy, hz = 0.7, 1.3, 0.4
    Ke, Me, Re = orc.fem_element(hx, hy, hz)
    kx, mx = _1d(hx)
    ky, my = _1d(hy)
    kz, mz = _1d(hz)
    # local vertex a: bit0 -> x, bit1 -> y, bit2 -> z  => kron(z, y, x)
    K = np.kron(mz, np.kron(my, kx)) + np.kron(mz, np.kron(ky, mx)) + np.kron(kz, np.kron(my, mx))
    M = np.kron(mz, np.kron(my, mx))
    R = np.kron(my, mx)
    np.testing.assert_allclose(Ke, K, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(Me, M, rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(Re, R, rtol=1e-13, atol=1e-16)


@pytest.mark.parametrize("geom", GEOMS)
def test_matrix_free_apply_matches_reference_assembly(geom):
    N = geom[0] * geom[1] * geom[2]
    rng = np.random.default_rng(N)
    for sigma, sigmap in ((0.0, 0.0), (0.37, 1.9)):
        A = orc.fem_dense(geom, sigma, sigmap)
        assert np.allclose(A, A.T, rtol=0, atol=1e-13 * np.abs(A).max())  # symmetric
        x = rng.standard_normal(N)
        np.testing.assert_allclose(orc.fem_apply(geom, sigma, sigmap, x), A @ x, rtol=1e-12,
                                   atol=1e-13 * np.abs(A @ x).max())
    # SPD with positive shifts (the CG precondition)
    assert np.linalg.eigvalsh(orc.fem_dense(geom, 0.37, 1.9)).min() > 0


def test_point_source_weights():
    geom = (6, 5, 3, 3.0, 3.0, 2.0)
    nx, ny, nz, Lx, Ly, Lz = geom
    b = orc.fem_point_source(geom, [0.1, -0.2, 0.7])
    assert np.count_nonzero(b) == 8 and abs(b.sum() - 1.0) < 1e-14  # interior cell: all 8 weights
    with pytest.raises(ValueError, match="Dirichlet boundary"):
        orc.fem_point_source(geom, [-Lx, -Ly, 0.0])
    with pytest.raises(ValueError, match="outside domain"):
        orc.fem_point_source(geom, [0.0, 0.0, -0.1])


def test_oracle_fields_match_dense_solve():
    geom = (6, 5, 4, 3.0, 3.0, 2.0)
    sig, sigp, invd = np.array([0.2, 0.9]), np.array([1.1, 0.4]), np.array([2.0, 3.0])
    pts = np.array([[0.1, -0.2, 0.0], [0.5, 0.3, 2.0]])
    F, it, rel = orc.fem_fields(geom, sig, sigp, invd, pts, tol=1e-13)
    assert rel.max() <= 1e-13
    N = 6 * 5 * 4
    for s in range(2):
        b = orc.fem_point_source(geom, pts[s])
        for l in range(2):
            x = np.linalg.solve(orc.fem_dense(geom, sig[l], sigp[l]), b) * invd[l]
            np.testing.assert_allclose(F[:, s * 2 + l], x, rtol=1e-10, atol=1e-12 * np.abs(x).max())
    assert F.shape == (N, 4)


@pytest.fixture(scope="module")
def ctx():
    import paper_1410_0986_b200 as h
    return h.Context(0)


@pytest.mark.gpu
@pytest.mark.parametrize("geom", GEOMS + [(17, 13, 11, 4.0, 3.0, 5.0)])
def test_gpu_apply_fem_matches_oracle(ctx, geom):
    from paper_1410_0986_b200 import born
    N = geom[0] * geom[1] * geom[2]
    x = np.random.default_rng(7).standard_normal(N)
    for sigma, sigmap in ((0.0, 0.0), (0.37, 1.9)):
        got = born.apply_operator_fem(ctx, geom, sigma, sigmap, torch.as_tensor(x).cuda()).cpu().numpy()
        np.testing.assert_array_equal(got, orc.fem_apply(geom, sigma, sigmap, x))


@pytest.mark.gpu
def test_gpu_fields_fem_match_oracle_and_dense(ctx):
    from paper_1410_0986_b200 import born
    geom = (9, 8, 7, 4.0, 3.5, 6.0)
    sig, sigp, invd = np.array([0.05, 0.3, 0.9]), np.array([1.5, 0.8, 0.2]), np.array([3.0, 2.5, 1.5])
    pts = np.array([[0.1, -0.2, 0.0], [1.3, 0.9, 6.0], [-2.0, 1.0, 3.3]])
    # fixed iterations: same recurrences, only the dot-product order differs
    Fg, _ = born.compute_fields_fem(ctx, geom, sig, sigp, invd, pts, fixed_iters=25)
    Fo, _, _ = orc.fem_fields(geom, sig, sigp, invd, pts, fixed_iters=25)
    got = Fg.cpu().numpy().reshape(-1, Fg.shape[-1]).T
    assert np.linalg.norm(got - Fo) <= 1e-12 * np.linalg.norm(Fo)
    # converged vs the dense reference-assembly solve
    Fc, st = born.compute_fields_fem(ctx, geom, sig, sigp, invd, pts, tol=1e-12)
    assert st.relres.max() <= 1e-12
    for s in range(3):
        b = orc.fem_point_source(geom, pts[s])
        for l in range(3):
            x = np.linalg.solve(orc.fem_dense(geom, sig[l], sigp[l]), b) * invd[l]
            np.testing.assert_allclose(Fc[s, l].cpu().numpy(), x, rtol=1e-9, atol=1e-11 * np.abs(x).max())
