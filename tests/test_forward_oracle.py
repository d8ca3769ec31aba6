"""Nonlinear forward model, CPU oracle: the reference's own
tests of full_diffusion_forward restated on the 7-point operator
(test_harness.cpp:125-163):

* a zero anomaly gives exactly zero scattered data and nonzero incident data;
* the Born prediction is close for a weak anomaly (<= 15 % at a quarter of
  the contrast) and the gap grows monotonically with the contrast.
"""
import numpy as np

import forward_fixture as fx


def _H(oracle, cfg, st):
    g = st.grid() if False else None  # noqa: F841 (host only)
    n = cfg.n
    F, _, _ = oracle.fields((n, n, n), cfg.h, st.sigma, st.sigma_prime, st.inv_D, st.points, tol=1e-13)
    nl = cfg.n_lambda
    fld = lambda p: F[:, p * nl:(p + 1) * nl]  # N x nl
    w = fx.lumped_mass(cfg)
    blocks = []
    for s in range(cfg.n_sources):
        blocks.append(oracle.born_block(fld(st.source_point[s]),
                                        [fld(st.detector_point[s, d]) for d in range(cfg.n_det)], w, 1.0))
    return np.vstack(blocks)


def test_zero_anomaly_gives_zero_scattered_data(oracle):
    cfg, st = fx.setup()
    n = cfg.n
    mu0 = np.zeros(n ** 3)
    yt, yi, ys = oracle.full_forward((n, n, n), cfg.h, st.sigma, st.sigma_prime, st.inv_D,
                                     fx.dsigma(st, st.conc), mu0, st.source_vertex, st.detector_vertex,
                                     tol=1e-12)
    assert np.linalg.norm(ys) == 0.0
    assert np.linalg.norm(yt - yi) == 0.0
    assert np.linalg.norm(yi) > 0.0


def test_born_prediction_close_for_weak_anomaly_and_degrades_with_contrast(oracle):
    cfg, st = fx.setup()
    n = cfg.n
    mu = fx.blob(cfg)
    assert (mu > 0.5).sum() > 0
    H = _H(oracle, cfg, st)
    gaps, weak_rel = [], None
    for scale in (0.25, 0.5, 1.0, 2.0):
        c = scale * st.conc * 1.0  # anomaly contrast: 1x background per unit scale
        yt, yi, ys = oracle.full_forward((n, n, n), cfg.h, st.sigma, st.sigma_prime, st.inv_D,
                                         fx.dsigma(st, c), mu, st.source_vertex, st.detector_vertex, tol=1e-13)
        yb = fx.born_prediction(st, cfg, H, mu, c)
        gap = np.linalg.norm(ys - yb)
        gaps.append(gap)
        if scale == 0.25:
            weak_rel = gap / np.linalg.norm(yb)
    assert weak_rel <= 0.15, weak_rel
    assert all(b > a for a, b in zip(gaps, gaps[1:])), gaps
