"""Shared PaLS fixture (test infrastructure): a small 7-point-stencil Born
operator from the CPU oracle, a one-RBF truth and a perturbed start, and
noisy data built like born::add_noise (born.cpp:131-154) with the libstdc++
normal stream.  Mirrors the reconstruction fixture of
proj/tests/test_pals.cpp:207-269 on this build's operator."""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
from paper_1410_0986_b200 import configs  # noqa: E402


class Params:
    """Plain PaLSParams stand-in (the oracle wrapper takes any such object)."""

    def __init__(self, alpha, beta, centers, tau_level=0.1, eps_H=0.05, nu_norm=1e-3):
        self.alpha = np.asarray(alpha, dtype=np.float64).reshape(-1)
        self.beta = np.asarray(beta, dtype=np.float64).reshape(-1)
        self.centers = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
        self.tau_level, self.eps_H, self.nu_norm = tau_level, eps_H, nu_norm

    def to_vector(self):
        return np.concatenate([self.alpha, self.beta, self.centers[:, 0], self.centers[:, 1],
                               self.centers[:, 2]])

    def with_vector(self, v):
        n = len(self.alpha)
        return Params(v[:n], np.maximum(v[n:2 * n], 1e-8),
                      np.stack([v[2 * n:3 * n], v[3 * n:4 * n], v[4 * n:]], axis=1),
                      self.tau_level, self.eps_H, self.nu_norm)


def random_params(rng, geom, n_p):
    """random_params of test_pals.cpp:17-33 (numpy draws)."""
    nx, ny, nz, Lx, Ly, Lz = geom
    hmin = min(2 * Lx / (nx - 1), 2 * Ly / (ny - 1), Lz / (nz - 1))
    u = lambda: rng.uniform()  # noqa: E731
    alpha, beta, cen = [], [], []
    for _ in range(n_p):
        alpha.append(0.5 + 0.5 * u())
        beta.append(1.0 / ((0.3 + 0.4 * u()) * Lz))
        cen.append([(2 * u() - 1) * 0.4 * Lx, (2 * u() - 1) * 0.4 * Ly, (0.3 + 0.4 * u()) * Lz])
    return Params(alpha, beta, cen, nu_norm=1e-3 * hmin)


def add_noise(y, snr_db, seed):
    """born::add_noise (born.cpp:131-154) with the same mt19937_64/normal stream."""
    eta = orc.gaussian(seed, len(y))
    target = np.linalg.norm(y) * 10.0 ** (-snr_db / 20.0)
    eta = eta * (target / np.linalg.norm(eta))
    sigma = target / np.sqrt(len(y))
    w = np.full(len(y), 1.0 / sigma)
    return y + eta, eta, w


def born_fixture(n=9, ns=2, n_det=3, n_lambda=7):
    """Dense H (M x N), extinction (n_lambda x 4), geometry of an n^3 config grid."""
    cfg = configs.Config(f"pals{n}", n, ns, ns, n_det, n_lambda)
    st = configs.make_setup(cfg)
    g = st.grid()
    F, _, _ = orc.fields((g.nx, g.ny, g.nz), g.h, st.sigma, st.sigma_prime, st.inv_D, st.points,
                         tol=1e-12, threads=4)
    nl = n_lambda
    w = st.w
    blocks = []
    for s in range(cfg.n_sources):
        inc = F[:, st.source_point[s] * nl:(st.source_point[s] + 1) * nl]
        adj = [F[:, st.detector_point[s, d] * nl:(st.detector_point[s, d] + 1) * nl]
               for d in range(n_det)]
        blocks.append(orc.born_block(inc, adj, w, 1.0))
    H = np.vstack(blocks)
    L = (n - 1) * cfg.h / 2
    geom = (n, n, n, L, L, 2 * L)
    return H, st.eps_c.copy(), geom


def recon_problem(n=9):
    """Truth / init parameters and noisy data for the reconstruction tests."""
    H, ext, geom = born_fixture(n)
    Lz = geom[5]
    truth = Params([1.0], [1.0 / (0.45 * Lz)], [[0.0, 0.0, 0.5 * Lz]], eps_H=0.3,
                   nu_norm=1e-3 * 2.0)
    init = Params([0.9], [1.0 / (0.45 * Lz) * 0.85], [[0.1 * Lz / 2, -0.1 * Lz / 2, 0.55 * Lz]],
                  eps_H=0.3, nu_norm=1e-3 * 2.0)
    mu_true = orc.pals_eval("shape", geom, truth)
    c_true = np.array([8.0, 8.0, 0.1, -0.1])
    hm = H @ mu_true
    nl = ext.shape[0]
    scale = ext @ c_true
    y_clean = scale[np.arange(H.shape[0]) % nl] * hm
    y, eta, w = add_noise(y_clean, 40.0, 99)
    noise_norm = float(np.linalg.norm(w * eta))
    return dict(H=H, ext=ext, geom=geom, truth=truth, init=init, mu_true=mu_true, y=y, w=w,
                noise_norm=noise_norm, c_true=c_true)
