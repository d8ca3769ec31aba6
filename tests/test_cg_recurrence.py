"""The single-pass CG recurrence of the GPU field solve (csrc/cg.cu cg1_step:
Chronopoulos-Gear scalars, alpha from gamma = (r, r) and delta = (r, A r) of
the previous pass) restated in numpy against the oracle's two-pass CG, the
reference's krylov::solve_family (krylov.cpp:400-463): at equal iteration
counts the iterates agree to rounding (1e-13 relative, ~1e-16 observed), and
in converged mode both stop at the same iteration.  This is what lets the GPU
kernel run one pass per iteration and still be checked against the
reference's CG at 1e-12 (test_gpu_kernels.py)."""
import numpy as np
import pytest

from paper_1410_0986_b200 import configs


def single_pass_cg(A, b, limit, tol=0.0):
    x = np.zeros_like(b)
    r = b.copy()
    p_old = np.zeros_like(b)
    gam = r @ r
    bn = np.sqrt(gam)
    dlt = r @ A(r)
    g_old = a_old = None
    for it in range(limit):
        if it == 0:
            beta, alpha = 0.0, gam / dlt
        else:
            if tol and np.sqrt(gam) / bn <= tol:
                return x, it
            beta = gam / g_old
            alpha = gam / (dlt - beta * gam / a_old)
        p = r + beta * p_old
        s = A(p)
        x = x + alpha * p
        r = r - alpha * s
        g_old, a_old = gam, alpha
        gam, dlt = r @ r, r @ A(r)
        p_old = p
    return x, limit


@pytest.mark.parametrize("n,fixed", [(12, 40), (16, 0)])
def test_single_pass_recurrence_matches_oracle_cg(oracle, n, fixed):
    st = configs.make_setup(configs.small_config(n=n, n_lambda=3))
    g = st.grid()
    shape = (g.nx, g.ny, g.nz)
    pts = st.points[:2]
    want, it_o, _ = oracle.fields(shape, g.h, st.sigma, st.sigma_prime, st.inv_D, pts,
                                  tol=1e-10, fixed_iters=fixed)
    for k, v in enumerate(pts):
        for l in range(len(st.sigma)):
            A = lambda u: oracle.apply7(shape, g.h, st.sigma[l], st.sigma_prime[l], u)
            b = np.zeros(g.N)
            b[v] = 1.0
            x, it = single_pass_cg(A, b, fixed or 10000, 0.0 if fixed else 1e-10)
            x = x * st.inv_D[l]
            col = want[:, k * len(st.sigma) + l]
            assert np.linalg.norm(x - col) <= 1e-13 * np.linalg.norm(col)
            if not fixed:
                assert it == it_o[k * len(st.sigma) + l]
