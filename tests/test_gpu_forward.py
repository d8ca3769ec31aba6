"""Nonlinear forward model on the device (hydot_full_forward; SURVEY 8(f) #4,
experiments::full_diffusion_forward, experiments.cpp:154-206):

* against the oracle at equal CG iterations: y_total / y_incident <= 1e-12;
* a zero anomaly gives exactly zero scattered data (test_harness.cpp:125-136);
* the Born prediction from the device Born blocks (lumped-mass weight) is
  within 15 % for a weak anomaly and degrades monotonically with contrast
  (test_harness.cpp:138-163).
"""
import numpy as np
import pytest
import torch

import forward_fixture as fx

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1410_0986_b200 as h
    return h.Context(0)


def _run(ctx, cfg, st, mu, c, **kw):
    from paper_1410_0986_b200 import born
    return born.full_diffusion_forward(ctx, st.grid(), st.sigma, st.sigma_prime, st.inv_D, fx.dsigma(st, c),
                                       torch.as_tensor(mu), st.source_vertex, st.detector_vertex, **kw)


def test_full_forward_matches_oracle_at_equal_iterations(ctx, oracle):
    cfg, st = fx.setup(n=14, ns_x=2, ns_y=2, n_det=3, n_lambda=5)
    n = cfg.n
    mu = fx.blob(cfg)
    ff = _run(ctx, cfg, st, mu, 2.0 * st.conc, fixed_iters=60)
    yt, yi, ys = oracle.full_forward((n, n, n), cfg.h, st.sigma, st.sigma_prime, st.inv_D,
                                     fx.dsigma(st, 2.0 * st.conc), mu, st.source_vertex, st.detector_vertex,
                                     fixed_iters=60)
    for got, want in ((ff.y_total, yt), (ff.y_incident, yi)):
        got = got.cpu().numpy()
        assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-12


def test_full_forward_zero_anomaly_is_exactly_zero(ctx):
    cfg, st = fx.setup()
    ff = _run(ctx, cfg, st, np.zeros(cfg.N), st.conc, tol=1e-12)
    assert float(torch.linalg.norm(ff.y_scattered)) == 0.0
    assert float(torch.linalg.norm(ff.y_incident)) > 0.0


def test_full_forward_born_consistency(ctx):
    from paper_1410_0986_b200 import born
    cfg, st = fx.setup(n=16, ns_x=2, ns_y=2, n_det=3, n_lambda=5)
    g = st.grid()
    F, _ = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points, tol=1e-12)
    w = torch.as_tensor(fx.lumped_mass(cfg)).cuda()
    H = torch.cat([born.assemble_H_block(ctx, F[st.source_point[s]],
                                         [F[st.detector_point[s, d]] for d in range(cfg.n_det)], w, 1.0)
                   for s in range(cfg.n_sources)]).cpu().numpy()
    mu = fx.blob(cfg)
    gaps, weak = [], None
    for scale in (0.25, 0.5, 1.0, 2.0):
        c = scale * st.conc
        ys = _run(ctx, cfg, st, mu, c, tol=1e-12).y_scattered.cpu().numpy()
        yb = fx.born_prediction(st, cfg, H, mu, c)
        gaps.append(np.linalg.norm(ys - yb))
        if scale == 0.25:
            weak = gaps[-1] / np.linalg.norm(yb)
    assert weak <= 0.15, weak
    assert all(b > a for a, b in zip(gaps, gaps[1:])), gaps
