"""BASELINE config 1 at full size (n=48, N=110592, 16 sources x 6 detectors x
50 wavelengths, M=4800) through size-independent properties: the oracle is
too slow at this size, so the compressed operator is checked against the
exact Born operator applied block by block (never materialised), against
its own adjoint, and for reproducibility.

* ||H~x - Hx|| / ||Hx|| and ||H~^T y - H^T y|| / ||H^T y|| stay below the
  scheduled tolerance budget (eps_d = 1e-6, experiments.cpp:230-233);
* <H~x, y> = <x, H~^T y> to 1e-12 (test_lowrank.cpp:272-287 at full size);
* two compressions with the same seed give bit-identical factors
  (test_lowrank.cpp:83-88, determinism per seed);
* every field reaches the CG tolerance.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg1():
    import paper_1410_0986_b200 as h
    from paper_1410_0986_b200 import born, configs, lowrank as lr
    ctx = h.Context(0)
    cfg = configs.CONFIGS[1]
    st = configs.make_setup(cfg)
    g = st.grid()
    F, stats = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points, tol=1e-10)
    w = torch.full((g.N,), cfg.h ** 3, dtype=torch.float64, device="cuda")
    inc = [F[st.source_point[s]] for s in range(cfg.n_sources)]
    adj = [[F[st.detector_point[s, d]] for d in range(cfg.n_det)] for s in range(cfg.n_sources)]
    tree = lr.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
    eps = configs.compression_tolerance(st, tree.depth())
    prov = lr.BornFieldsProvider(inc, adj, w, 1.0)
    rec = lr.recursive_lowrank(ctx, tree, eps, prov, lr.RecursiveOptions(seed=cfg.seed))
    fr = lr.recompress(ctx, rec.factor, eps)
    return dict(ctx=ctx, cfg=cfg, st=st, g=g, stats=stats, inc=inc, adj=adj, w=w, tree=tree,
                eps=eps, prov=prov, rec=rec, fr=fr)


def exact_products(d, x, y):
    """H x and H^T y with H's blocks formed one source at a time."""
    from paper_1410_0986_b200 import born
    cfg = d["cfg"]
    m = cfg.n_det * cfg.n_lambda
    Hx = torch.empty(cfg.M, dtype=torch.float64, device="cuda")
    Hty = torch.zeros(d["g"].N, dtype=torch.float64, device="cuda")
    for s in range(cfg.n_sources):
        B = born.assemble_H_block(d["ctx"], d["inc"][s], d["adj"][s], d["w"], 1.0)
        Hx[s * m:(s + 1) * m] = B @ x
        Hty += B.T @ y[s * m:(s + 1) * m]
    return Hx, Hty


def test_fields_converged(cfg1):
    assert float(cfg1["stats"].relres.max()) <= 1e-10


def test_compressed_operator_matches_exact_born_products(cfg1):
    d = cfg1
    fr, perm = d["fr"], torch.as_tensor(np.asarray(d["rec"].row_perm), device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(d["g"].N, dtype=torch.float64, device="cuda", generator=gen)
    y = torch.randn(d["cfg"].M, dtype=torch.float64, device="cuda", generator=gen)
    Hx, Hty = exact_products(d, x, y)
    U, V = fr.U, fr.V
    Jx = torch.empty_like(Hx)
    Jx[perm] = U @ (V.T @ x)                  # permuted_matvec (experiments.cpp:255-262)
    Jty = V @ (U.T @ y[perm])
    budget = 1e-6  # eps_d: the whole-tree tolerance the schedule distributes
    assert float(torch.linalg.norm(Jx - Hx) / torch.linalg.norm(Hx)) <= budget
    assert float(torch.linalg.norm(Jty - Hty) / torch.linalg.norm(Hty)) <= budget
    # adjoint consistency of the compressed operator at full size
    lhs = float(torch.dot(Jx, y))
    rhs = float(torch.dot(x, Jty))
    assert lhs == pytest.approx(rhs, rel=1e-12)


def test_device_matvec_matches_factor_products(cfg1):
    from paper_1410_0986_b200 import lowrank as lr
    d = cfg1
    fr = d["fr"]
    gen = torch.Generator(device="cuda").manual_seed(9)
    X = torch.randn(d["g"].N, 3, dtype=torch.float64, device="cuda", generator=gen)
    got = lr.lr_matvec(d["ctx"], fr, X)
    want = fr.U @ (fr.V.T @ X)
    assert float(torch.linalg.norm(got - want) / torch.linalg.norm(want)) <= 1e-12


def test_compression_is_deterministic(cfg1):
    from paper_1410_0986_b200 import lowrank as lr
    d = cfg1
    rec2 = lr.recursive_lowrank(d["ctx"], d["tree"], d["eps"], d["prov"],
                                lr.RecursiveOptions(seed=d["cfg"].seed))
    assert list(rec2.node_rank) == list(d["rec"].node_rank)
    fr2 = lr.recompress(d["ctx"], rec2.factor, d["eps"])
    assert fr2.rank() == d["fr"].rank()
    assert torch.equal(fr2.U, d["fr"].U) and torch.equal(fr2.V, d["fr"].V)
