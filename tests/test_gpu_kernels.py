"""Kernel-level parity on the B200 against the CPU oracle (same inputs).

Bars (BASELINE.json north_star): Born blocks bit-exact (1e-12 allowed),
fields 1e-12 relative at equal iteration counts, generator exact engine bits
and deviates within a few ulp, GEMM/QR/SVD at FP64 rounding level.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1410_0986_b200 as h
    return h.Context(0)


def cm(a):
    """numpy (m x n) -> column-major CUDA buffer (n x m row-major tensor)"""
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a).T)).cuda()


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (37, 29, 53), (64, 64, 16), (130, 70, 300),
                                   (800, 70, 40000), (5, 3, 200001)])
def test_dgemm_matches_numpy(ctx, ta, tb, m, n, k):
    import paper_1410_0986_b200 as h
    rng = np.random.default_rng(m * 7 + n * 13 + k)
    A = rng.standard_normal((k, m) if ta else (m, k))
    B = rng.standard_normal((n, k) if tb else (k, n))
    C0 = rng.standard_normal((m, n))
    ref = 1.5 * ((A.T if ta else A) @ (B.T if tb else B)) - 0.5 * C0
    dA, dB, dC = cm(A), cm(B), cm(C0)
    h.dgemm(ctx, bool(ta), bool(tb), m, n, k, 1.5, dA, A.shape[0], dB, B.shape[0], -0.5, dC, m)
    got = dC.cpu().numpy().T
    err = np.abs(got - ref).max() / (np.abs(A).max() * np.abs(B).max() * np.sqrt(k))
    assert err < 1e-14


def test_born_block_bitwise(ctx, oracle):
    from paper_1410_0986_b200 import born
    rng = np.random.default_rng(1)
    for N, nl, nd in [(1001, 3, 4), (4096, 7, 2), (12345, 5, 3)]:
        inc = rng.standard_normal((nl, N))
        adj = [rng.standard_normal((nl, N)) for _ in range(nd)]
        w = rng.random(N) + 0.5
        want = oracle.born_block(inc.T, [a.T for a in adj], w, 1.7)
        got = born.assemble_H_block(ctx, torch.as_tensor(inc).cuda(),
                                    [torch.as_tensor(a).cuda() for a in adj],
                                    torch.as_tensor(w).cuda(), 1.7).cpu().numpy()
        assert np.array_equal(got, want)


def test_mt19937_64_engine_bits(ctx, oracle):
    import paper_1410_0986_b200 as h
    for seed in (0, 5489, 20240811 + 0x9e3779b97f4a7c15, 2**64 - 1):
        want = oracle.mt19937_64(seed, 1000000)
        got = h.mt19937_64(ctx, seed, 0, 1000000).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want)
        # windows straddling jump-ahead chunk boundaries (S = 312 * 1024)
        for off, cnt in ((300000, 40000), (600000, 400000)):
            got2 = h.mt19937_64(ctx, seed, off, cnt).cpu().numpy().view(np.uint64)
            assert np.array_equal(got2, want[off:off + cnt])


def test_gaussian_stream_matches_libstdcxx(ctx, oracle):
    import paper_1410_0986_b200 as h
    for seed in (42, 20240811 + 0x9e3779b97f4a7c15 * 3):
        n = 700001
        want = oracle.gaussian(seed, n)
        got = h.gaussian(ctx, seed, 0, n).cpu().numpy()
        ulp = np.abs(got - want) / np.spacing(np.abs(want))
        assert np.max(ulp) <= 4.0, np.max(ulp)
        assert np.mean(got == want) > 0.9
        part = h.gaussian(ctx, seed, 123457, 1000).cpu().numpy()
        assert np.max(np.abs(part - want[123457:124457]) / np.spacing(np.abs(want[123457:124457]))) <= 4


def test_apply7_bitwise(ctx, oracle):
    from paper_1410_0986_b200 import born
    rng = np.random.default_rng(3)
    for shape in [(7, 6, 5), (16, 16, 16), (33, 20, 9)]:
        g = born.Grid7(*shape, 2.0)
        x = rng.standard_normal(g.N)
        want = oracle.apply7(shape, 2.0, 0.07, 1.6, x)
        got = born.apply_operator(ctx, g, 0.07, 1.6, torch.as_tensor(x).cuda()).cpu().numpy()
        assert np.array_equal(got, want)


def test_fields_match_oracle_cg(ctx, oracle):
    from paper_1410_0986_b200 import born, configs
    st = configs.make_setup(configs.small_config(n=16, n_lambda=5))
    g = st.grid()
    pts = st.points[:3]
    # equal iteration counts: only dot-product summation order differs
    gpu, stats = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, pts,
                                     fixed_iters=60)
    want, _, _ = oracle.fields((g.nx, g.ny, g.nz), g.h, st.sigma, st.sigma_prime, st.inv_D, pts,
                               fixed_iters=60)
    got = gpu.cpu().numpy().reshape(len(pts) * 5, g.N).T
    rel = np.linalg.norm(got - want, axis=0) / np.linalg.norm(want, axis=0)
    assert rel.max() <= 1e-12, rel.max()
    # converged mode: residual reaches tol, same answer as the oracle to tol
    gpu2, stats2 = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, pts, tol=1e-10)
    want2, it2, rr2 = oracle.fields((g.nx, g.ny, g.nz), g.h, st.sigma, st.sigma_prime, st.inv_D,
                                    pts, tol=1e-10)
    assert np.all(stats2.relres <= 1e-10)
    assert np.abs(stats2.iters.reshape(-1) - it2).max() <= 1
    got2 = gpu2.cpu().numpy().reshape(len(pts) * 5, g.N).T
    rel2 = np.linalg.norm(got2 - want2, axis=0) / np.linalg.norm(want2, axis=0)
    assert rel2.max() <= 1e-9


@pytest.mark.parametrize("shape", [(64, 40, 6), (100, 30, 3), (5, 9, 2), (48, 48, 3)])
def test_fields_tiled_shapes_match_oracle(ctx, oracle, shape):
    """Grids whose x-rows split into several z-marching tiles (ny > tile
    height), tiny tiles and two-plane grids: fields at equal iteration
    counts within 1e-12 of the oracle CG."""
    from paper_1410_0986_b200 import born
    nx, ny, nz = shape
    g = born.Grid7(nx, ny, nz, 2.0)
    sigma, sigp, invd = [0.02, 0.3], [1.4, 2.1], [3.0, 2.5]
    pts = [nx * (ny // 2) + nx // 2, (nz // 2) * nx * ny + nx * (ny - 2) + nx - 2]
    gpu, _ = born.compute_fields(ctx, g, sigma, sigp, invd, pts, fixed_iters=25)
    want, _, _ = oracle.fields(shape, 2.0, sigma, sigp, invd, pts, fixed_iters=25)
    got = gpu.cpu().numpy().reshape(len(pts) * 2, g.N).T
    rel = np.linalg.norm(got - want, axis=0) / np.linalg.norm(want, axis=0)
    assert rel.max() <= 1e-12, rel.max()


def test_fields_reject_dirichlet_source(ctx):
    from paper_1410_0986_b200 import born
    g = born.Grid7(8, 8, 8, 2.0)
    with pytest.raises(ValueError):
        born.compute_fields(ctx, g, [0.1], [1.5], [3.0], [0])  # corner vertex


@pytest.mark.parametrize("m,n", [(50, 7), (300, 70), (3000, 33), (200000, 40), (64, 64)])
def test_householder_qr(ctx, m, n):
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n)) * np.logspace(0, -12, n)
    Q, R = lr.householder_qr(ctx, torch.as_tensor(A))
    Q, R = Q.cpu().numpy(), R.cpu().numpy()
    assert np.allclose(np.triu(R), R)
    assert np.linalg.norm(Q @ R - A) <= 1e-14 * np.linalg.norm(A) * np.sqrt(n)
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13 * np.sqrt(n)
    # same R as LAPACK up to row signs
    R2 = np.linalg.qr(A, mode="r")
    assert np.allclose(np.abs(np.diag(R)), np.abs(np.diag(R2)), rtol=1e-10, atol=1e-14 * np.abs(R2).max())


def test_householder_qr_tall_rank_deficient(ctx):
    """The tall panels (shifted CholeskyQR3 + Householder reconstruction,
    qr_cqr.cu) on numerically rank-deficient input and an all-zero panel:
    still a backward-stable Householder QR with orthonormal Q."""
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(3)
    m, n, k = 120000, 96, 20
    A = (rng.standard_normal((m, k)) * np.logspace(0, -10, k)) @ rng.standard_normal((k, n))
    A[:, 40:72] = 0.0  # one whole 32-wide panel of zeros
    A[:, 75] *= 1e-300
    Q, R = lr.householder_qr(ctx, torch.as_tensor(A))
    Q, R = Q.cpu().numpy(), R.cpu().numpy()
    assert np.allclose(np.triu(R), R)
    assert np.linalg.norm(Q @ R - A) <= 1e-14 * np.linalg.norm(A) * np.sqrt(n)
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13 * np.sqrt(n)


@pytest.mark.parametrize("m,n", [(60000, 450), (60000, 384), (3000, 900), (40000, 515)])
def test_householder_qr_lookahead_equals_inline(ctx, monkeypatch, m, n):
    """geqrf with look-ahead (qr.cu: the next block's panels on a high-priority
    stream beside the rest of the trailing update) against the in-line order
    (HYDOT_QR_LOOKAHEAD=0): the same Householder QR -- bitwise identical R,
    orthonormal Q, A = Q R -- repeated to catch an ordering race."""
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n)) * np.logspace(0, -9, n)
    At = torch.as_tensor(A)
    out = {}
    for mode in ("0", "1", "1", "1"):
        monkeypatch.setenv("HYDOT_QR_LOOKAHEAD", mode)
        Q, R = lr.householder_qr(ctx, At)
        Q, R = Q.cpu().numpy(), R.cpu().numpy()
        assert np.allclose(np.triu(R), R)
        assert np.linalg.norm(Q @ R - A) <= 1e-14 * np.linalg.norm(A) * np.sqrt(n)
        assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13 * np.sqrt(n)
        if mode in out:   # run to run: bitwise
            assert np.array_equal(out[mode], R)
        out[mode] = R
    # every column sees the same kernels on the same operands in the same order (only the
    # k = 128 product C -= V W2 is split by columns, and it has no split-K): bitwise equal
    assert np.array_equal(out["0"], out["1"])


@pytest.mark.parametrize("m,n", [(40, 55), (70, 70), (300, 70), (20000, 60), (90, 400), (250, 250)])
def test_thin_svd_matches_oracle(ctx, oracle, m, n):
    from paper_1410_0986_b200 import lowrank as lr
    rng = np.random.default_rng(m * n)
    k = min(m, n)
    A = (rng.standard_normal((m, k)) * np.logspace(0, -14, k)) @ rng.standard_normal((k, n))
    U, s, V = lr.thin_svd(ctx, torch.as_tensor(A))
    U, V = U.cpu().numpy(), V.cpu().numpy()
    _, s2, _ = oracle.fast_thin_svd(A)
    assert np.all(np.abs(s - s2) <= 1e-13 * s2[0])
    assert np.linalg.norm(U * s @ V.T - A) <= 1e-13 * np.linalg.norm(A)
    assert np.linalg.norm(V.T @ V - np.eye(k)) <= 1e-13 * k
