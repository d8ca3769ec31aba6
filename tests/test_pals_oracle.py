"""Pins the PaLS oracle restatement (oracle/pals_oracle.cpp) to the
reference's own PaLS tests (proj/tests/test_pals.cpp), re-expressed as
assertions on this build's fixtures.  CPU only."""
import numpy as np
import pytest

from oracle import oracle as orc

import pals_fixture as pf

GEOM = (7, 7, 6, 3.0, 3.0, 2.0)  # build_grid(7, 7, 6, 3, 3, 2) of test_pals.cpp


def test_wendland_values_and_derivative():  # test_pals.cpp:37-50
    w = lambda t: orc.pals_scalar("wendland", t)  # noqa: E731
    assert w(0.0) == pytest.approx(1.0)
    assert w(1.0) == 0.0 and w(2.0) == 0.0
    assert w(0.5) == pytest.approx(0.5 ** 4 * 3.0, rel=1e-15)
    for t in (0.1, 0.3, 0.7, 0.95):
        fd = (w(t + 1e-6) - w(t - 1e-6)) / 2e-6
        assert orc.pals_scalar("wendland_deriv", t) == pytest.approx(fd, rel=1e-7)
    assert orc.pals_scalar("wendland_deriv", 0.0) == 0.0
    assert orc.pals_scalar("wendland_deriv", 1.5) == 0.0


def test_smoothed_heaviside_and_delta():  # test_pals.cpp:52-76
    eps = 0.05
    H = lambda t: orc.pals_scalar("smooth_heaviside", t, eps)  # noqa: E731
    assert H(-2 * eps) == pytest.approx(0.0) and H(2 * eps) == pytest.approx(1.0)
    assert H(0.0) == pytest.approx(0.5, rel=1e-13)
    for t in (-0.04, -0.01, 0.0, 0.02, 0.045):
        fd = (H(t + 1e-7) - H(t - 1e-7)) / 2e-7
        assert orc.pals_scalar("smooth_delta", t, eps) == pytest.approx(fd, rel=1e-5)
    assert orc.pals_scalar("smooth_delta", 1.5 * eps, eps) == pytest.approx(0.0)
    prev, t = -1.0, -0.06
    while t <= 0.06:  # the reference's accumulated grid
        v = H(t)
        assert 0.0 <= v <= 1.0 and v >= prev - 1e-13
        prev = v
        t += 0.004


def _direct_level_set(geom, p):
    nx, ny, nz, Lx, Ly, Lz = geom
    hx, hy, hz = 2 * Lx / (nx - 1), 2 * Ly / (ny - 1), Lz / (nz - 1)
    n = np.arange(nx * ny * nz)
    r = np.stack([-Lx + (n % nx) * hx, -Ly + ((n // nx) % ny) * hy, (n // (nx * ny)) * hz], 1)
    phi = np.zeros(len(n))
    for k in range(len(p.alpha)):
        d = np.sqrt(((r - p.centers[k]) ** 2).sum(1) + p.nu_norm ** 2)
        t = p.beta[k] * d
        s = np.clip(1 - t, 0, None)
        phi += p.alpha[k] * np.where(t < 1, s ** 4 * (4 * t + 1), 0.0)
    return phi


def test_level_set_matches_direct_rbf_sum():  # test_pals.cpp:78-102
    rng = np.random.default_rng(2)
    p = pf.random_params(rng, GEOM, 3)
    phi = orc.pals_eval("level_set", GEOM, p)
    np.testing.assert_allclose(phi, _direct_level_set(GEOM, p), rtol=1e-13, atol=1e-15)
    mu = orc.pals_eval("shape", GEOM, p)
    assert np.all(mu >= 0) and np.all(mu <= 1)
    want = [orc.pals_scalar("smooth_heaviside", v - p.tau_level, p.eps_H) for v in phi]
    np.testing.assert_array_equal(mu, want)


def test_parameter_round_trip():  # test_pals.cpp:104-117
    p = pf.random_params(np.random.default_rng(1), GEOM, 4)
    v = p.to_vector()
    assert v.shape == (20,)
    q = p.with_vector(v)
    np.testing.assert_array_equal(q.alpha, p.alpha)
    np.testing.assert_array_equal(q.beta, p.beta)
    np.testing.assert_array_equal(q.centers, p.centers)
    assert v[0] == p.alpha[0] and v[4] == p.beta[0] and v[8] == p.centers[0, 0]


def test_shape_jacobian_matches_central_differences():  # test_pals.cpp:119-140
    rng = np.random.default_rng(3)
    for _ in range(3):
        p = pf.random_params(rng, GEOM, 2)
        J = orc.pals_eval("shape_jacobian", GEOM, p)
        assert J.shape == (7 * 7 * 6, 10)
        v = p.to_vector()
        for j in range(10):
            h = 1e-5 * max(1.0, abs(v[j]))
            vp, vm = v.copy(), v.copy()
            vp[j] += h
            vm[j] -= h
            fd = (orc.pals_eval("shape", GEOM, p.with_vector(vp))
                  - orc.pals_eval("shape", GEOM, p.with_vector(vm))) / (2 * h)
            tol = max(1e-6, 1e-4 * np.linalg.norm(J[:, j]))
            assert np.linalg.norm(J[:, j] - fd) <= tol


def test_lm_step_solves_damped_normal_equations():  # test_pals.cpp:142-155
    g = orc.gaussian(4, 30 * 8 + 30)
    J = g[:240].reshape(8, 30).T  # column-major fill
    r = g[240:]
    for nu in (1e-6, 1.0, 50.0):
        dp = orc.pals_lm_step(J, r, nu)
        want = np.linalg.solve(J.T @ J + nu * np.eye(8), -J.T @ r)
        assert np.linalg.norm(dp - want) <= 1e-9 * np.linalg.norm(want)


def test_concentration_solve_recovers_coefficients():  # test_pals.cpp:157-190
    geom = (6, 6, 5, 3.0, 3.0, 2.0)
    N = 6 * 6 * 5
    nl = 9
    ext = np.abs(orc.gaussian(11, nl * 4).reshape(4, nl).T) + 0.1
    M = 3 * nl
    H = orc.gaussian(5, M * N).reshape(N, M).T
    p = pf.random_params(np.random.default_rng(5), geom, 2)
    mu = orc.pals_eval("shape", geom, p)
    assert (mu > 0.5).sum() > 0
    c_true = np.array([8.0, 8.0, 0.1, -0.1])
    y = (ext @ c_true)[np.arange(M) % nl] * (H @ mu)
    w = np.ones(M)
    c, flagged = orc.pals_solve_concentrations(H, np.eye(N), None, mu, w, y, ext)
    assert not flagged
    np.testing.assert_allclose(c, c_true, rtol=1e-8)
    c0, bad = orc.pals_solve_concentrations(H, np.eye(N), None, np.zeros(N), w, y, ext)
    assert bad and np.all(c0 == 0)


def test_metrics_known_shapes():  # test_pals.cpp:192-205
    a = np.array([1, 1, 0, 0, 1, 0.0])
    b = np.array([1, 0, 0, 0, 1, 1.0])
    l2, dice, fl = orc.pals_metrics(a, b)
    assert dice == pytest.approx(2.0 * 2 / 6, rel=1e-13)
    assert l2 == pytest.approx(np.linalg.norm(a - b) / np.linalg.norm(a), rel=1e-13)
    l2, dice, fl = orc.pals_metrics(a, a)
    assert dice == 1.0 and l2 == 0.0
    assert orc.pals_metrics(np.zeros(6), np.zeros(6))[2]


def test_reconstruction_reaches_discrepancy_target():  # test_pals.cpp:207-269
    P = pf.recon_problem(9)
    assert (P["mu_true"] > 0.5).sum() > 0
    N = P["H"].shape[1]
    r = orc.pals_reconstruct(P["H"], np.eye(N), None, P["geom"], P["ext"], P["y"], P["w"],
                             P["init"], P["noise_norm"], max_outer=25, mu_truth=P["mu_true"])
    assert r["converged"]
    assert r["resnorm"] <= 1.2 * P["noise_norm"] * (1 + 1e-9)
    mu_hat = orc.pals_eval("shape", P["geom"], pf.Params(r["alpha"], r["beta"], r["centers"],
                                                         eps_H=0.3, nu_norm=2e-3))
    assert orc.pals_metrics(P["mu_true"], mu_hat)[1] >= 0.6
    outer = r["trace"][:, 0]
    assert len(outer) > 0 and np.all(np.diff(outer) >= 0)


def test_reconstruct_rejects_gamma_le_one():
    P = pf.recon_problem(9)
    N = P["H"].shape[1]
    with pytest.raises(ValueError):
        orc.pals_reconstruct(P["H"], np.eye(N), None, P["geom"], P["ext"], P["y"], P["w"],
                             P["init"], P["noise_norm"], gamma=1.0)
