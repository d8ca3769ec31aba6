"""Fixture of the nonlinear forward model tests: a small BASELINE-recipe
setup, an interior absorption blob and the lumped-mass Born operator that
the full model linearises to (experiments.cpp:154-206 vs born.cpp:82-129)."""
import numpy as np

from paper_1410_0986_b200 import configs


def setup(n=12, ns_x=2, ns_y=2, n_det=2, n_lambda=4):
    cfg = configs.small_config(n=n, ns_x=ns_x, ns_y=ns_y, n_det=n_det, n_lambda=n_lambda)
    st = configs.make_setup(cfg)
    return cfg, st


def blob(cfg, centre=(0.5, 0.5, 0.45), radius=0.22):
    """A smooth interior anomaly in [0, 1] (compact support, zero on the
    faces), like a PaLS shape (pals.cpp:99-103)."""
    n = cfg.n
    t = np.arange(n) / (n - 1)
    z, y, x = np.meshgrid(t, t, t, indexing="ij")  # vertex id = ix + n (iy + n iz)
    r = np.sqrt((x - centre[0]) ** 2 + (y - centre[1]) ** 2 + (z - centre[2]) ** 2) / radius
    mu = np.where(r < 1.0, (1.0 - r) ** 4 * (4.0 * r + 1.0), 0.0)  # Wendland C2
    return mu.reshape(-1)


def lumped_mass(cfg):
    """Diagonal of the 7-point operator's mass: V = h^2 zext (h^3, h^3 / 2 on
    the z faces) -- the Born weight that matches the FV operator."""
    n, h = cfg.n, cfg.h
    zext = np.full(n, h)
    zext[0] = zext[-1] = 0.5 * h
    return np.repeat(h * h * zext, n * n)


def dsigma(st, c_pert):
    """dsigma_l = nu (sum_c c_c eps_c(lambda_l)) / D_l (experiments.cpp:168-177,
    nu = 1): the per-wavelength absorption scale of the anomaly."""
    return (st.eps_c @ c_pert) * st.inv_D


def born_prediction(st, cfg, H, mu, c_pert):
    """born::forward_measure (born.cpp:110-129): y[m] = (sum_c c_c
    eps_c(lambda_{m mod n_lambda})) (H mu)[m]."""
    e = st.eps_c @ c_pert
    Hm = H @ mu
    return e[np.arange(len(Hm)) % cfg.n_lambda] * Hm
