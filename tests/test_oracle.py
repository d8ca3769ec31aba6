"""CPU oracle pinned against the reference's own known-answer and bound tests.

Each test restates an assertion of /root/reference/proj/tests (cited) against
the oracle restatement (oracle/hydot_oracle.cpp).  No GPU needed.
"""
import math

import numpy as np
import pytest


def random_lowrank(rng, m, n, r, noise=0.0):
    # test_lowrank.cpp:14-30 (Gaussian factors, optional relative noise)
    X = rng.standard_normal((m, r))
    Y = rng.standard_normal((n, r))
    A = X @ Y.T
    if noise > 0:
        E = rng.standard_normal((m, n))
        A = A + (noise * np.linalg.norm(A) / np.linalg.norm(E)) * E
    return A


def truncated_svd(o, A, eps):
    # test_lowrank.cpp:33-49
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    total = float(np.sum(s * s))
    tail = total
    r = 0
    while r < len(s):
        if tail <= eps * eps * total:
            break
        tail -= s[r] * s[r]
        r += 1
    r = max(r, 1)
    return o.Factor.make(U[:, :r], Vt[:r].T * s[:r], tol=eps)


def test_mt19937_64_standard_known_answer(oracle):
    # C++ standard [rand.predef]: 10000th output of default-seeded mt19937_64
    v = oracle.mt19937_64(5489, 10000)
    assert int(v[-1]) == 9981545732273789042


def test_gaussian_stream_is_polar_pairs(oracle):
    # lowrank.cpp:136-143 through libstdc++ normal_distribution (polar method):
    # reproduce the first deviates from the raw engine in numpy.
    raw = oracle.mt19937_64(42, 64)
    u = raw.astype(np.float64) / 2.0**64
    g = oracle.gaussian(42, 8)
    outs = []
    t = 0
    while len(outs) < 8:
        x = 2.0 * u[t] - 1.0
        y = 2.0 * u[t + 1] - 1.0
        t += 2
        r2 = x * x + y * y
        if r2 > 1.0 or r2 == 0.0:
            continue
        mult = math.sqrt(-2 * math.log(r2) / r2)
        outs += [y * mult, x * mult]
    np.testing.assert_allclose(g, outs[:8], rtol=1e-15, atol=0)


def test_tolerance_schedule_formula(oracle):
    # test_lowrank.cpp:246-256
    for L in (0, 1, 2, 4):
        for Nr in (16, 400):
            want = 1e-6 / (2.0 ** (L / 2.0) * (L + 1) * math.sqrt(Nr))
            assert oracle.tolerance_schedule(1e-6, L, Nr) == pytest.approx(want, rel=1e-13)
    with pytest.raises(ValueError):
        oracle.tolerance_schedule(0.0, 1, 1)


def test_cluster_tree_five_on_a_line(oracle):
    # test_lowrank.cpp:139-159
    t = oracle.ClusterTree(np.array([0.1, 0.2, 0.6, 0.7, 0.95]), [0.0], [1.0])
    root = t.nodes[t.root]
    assert root["left"] >= 0
    L, R = t.nodes[root["left"]], t.nodes[root["right"]]
    assert L["idx"] == [0, 1] and L["left"] < 0
    assert R["left"] >= 0
    assert t.nodes[R["left"]]["idx"] == [2, 3]
    assert t.nodes[R["right"]]["idx"] == [4]
    assert t.depth() == 2
    assert t.leaf_order() == [0, 1, 2, 3, 4]


def test_cluster_tree_coincident_points(oracle):
    # test_lowrank.cpp:161-174
    pos = np.array([[0.1, 0.5], [0.9, 0.5], [0.1, 0.5], [0.9, 0.5]])
    t = oracle.ClusterTree(pos, [0, 0], [1, 1])
    assert sorted(t.leaf_order()) == [0, 1, 2, 3]
    for nd in t.nodes:
        if nd["left"] < 0:
            assert len(nd["idx"]) <= 2


def test_randsvd_exact_low_rank(oracle):
    # test_lowrank.cpp:53-62
    rng = np.random.default_rng(1)
    for t in range(5):
        A = random_lowrank(rng, 40, 55, 7)
        f = oracle.randsvd(A, 1e-10, 20, 10, 100 + t)
        assert np.linalg.norm(A - f.dense()) <= 1e-9 * np.linalg.norm(A)
        assert f.rank <= 27
        assert not f.flagged


def test_randsvd_error_within_tolerance(oracle):
    # test_lowrank.cpp:64-72
    rng = np.random.default_rng(2)
    for t in range(30):
        A = random_lowrank(rng, 30 + t % 20, 45, 5 + t % 6, 1e-4)
        f = oracle.randsvd(A, 1e-3, 20, 10, 500 + t)
        assert np.linalg.norm(A - f.dense()) <= 10 * 1e-3 * np.linalg.norm(A)


def test_randsvd_zero_matrix(oracle):
    # test_lowrank.cpp:74-79
    f = oracle.randsvd(np.zeros((12, 9)), 1e-8)
    assert f.rank == 0


def test_randsvd_deterministic(oracle):
    # test_lowrank.cpp:81-88
    rng = np.random.default_rng(3)
    A = random_lowrank(rng, 25, 30, 6, 1e-6)
    f1 = oracle.randsvd(A, 1e-6, 20, 10, 42)
    f2 = oracle.randsvd(A, 1e-6, 20, 10, 42)
    assert np.array_equal(f1.U, f2.U) and np.array_equal(f1.V, f2.V)


def test_randsvd_sketch_branch_taken(oracle):
    # a tall-wide block where the adaptive sketch (not Q = I) runs
    rng = np.random.default_rng(4)
    A = random_lowrank(rng, 200, 3000, 12, 1e-9)
    led = []
    f = oracle.randsvd(A, 1e-6, 20, 10, 7, oracle.LEAF, 1)
    assert 12 <= f.rank <= 14
    assert np.linalg.norm(A - f.dense()) <= 1e-5 * np.linalg.norm(A)
    assert f.ledger[0] > 0


def test_agglomeration_bound(oracle):
    # test_lowrank.cpp:122-137
    rng = np.random.default_rng(6)
    for t in range(40):
        H1 = random_lowrank(rng, 24, 40, 5, 1e-3)
        H2 = random_lowrank(rng, 18, 40, 4, 1e-3)
        eps = 1e-2
        f1, f2 = truncated_svd(oracle, H1, eps), truncated_svd(oracle, H2, eps)
        g = oracle.agglomerate(f1, f2, eps, 900 + t)
        H = np.vstack([H1, H2])
        err = np.linalg.norm(H - g.dense())
        assert err <= (2 * eps + eps * eps) * (np.linalg.norm(H1) + np.linalg.norm(H2))


def test_recursive_compression_through_row_perm(oracle):
    # test_lowrank.cpp:176-218
    rng = np.random.default_rng(7)
    ns, rows_per, cols = 6, 8, 50
    H = random_lowrank(rng, ns * rows_per, cols, 6, 1e-5)
    pos = np.array([[(s % 3) / 2.0, (s // 3) * 1.0] for s in range(ns)])
    tree = oracle.ClusterTree(pos, [0, 0], [1, 1])
    eps = 1e-4
    rec = oracle.recursive_lowrank(tree, eps, H, rows_per)
    assert len(rec.row_perm) == ns * rows_per
    Hhat = rec.factor.dense()
    Hp = np.zeros_like(H)
    Hp[rec.row_perm] = Hhat
    assert np.linalg.norm(H - Hp) <= 50 * eps * np.linalg.norm(H)
    tally = rec.ledger[4]
    assert tally > 0 and abs(rec.ledger[:4].sum() - tally) <= 0.05 * tally
    assert rec.ledger[0] > 0 and rec.ledger[1] > 0
    assert all(r >= 0 for r in rec.node_rank)


def test_recompress_removes_redundancy(oracle):
    # test_lowrank.cpp:258-270
    rng = np.random.default_rng(9)
    A = random_lowrank(rng, 30, 25, 4)
    f0 = truncated_svd(oracle, A, 1e-12)
    f = oracle.Factor.make(np.hstack([f0.U, f0.U]), np.hstack([0.5 * f0.V, 0.5 * f0.V]))
    g = oracle.recompress(f, 1e-10)
    assert g.rank <= f0.rank
    assert np.linalg.norm(g.dense() - A) <= 1e-9 * np.linalg.norm(A)


def test_matvec_adjoint_consistent(oracle):
    # test_lowrank.cpp:272-287
    rng = np.random.default_rng(10)
    A = random_lowrank(rng, 22, 31, 5)
    f = truncated_svd(oracle, A, 1e-12)
    for _ in range(10):
        x = rng.standard_normal(31)
        y = rng.standard_normal(22)
        a = y @ oracle.lr_matmat(f, x)[:, 0]
        b = x @ oracle.lr_matmat(f, y, trans=True)[:, 0]
        assert a == pytest.approx(b, rel=1e-12)
        assert np.linalg.norm(oracle.lr_matmat(f, x)[:, 0] - A @ x) <= 1e-10 * np.linalg.norm(A @ x)


def test_born_block_rows_and_ordering(oracle):
    # test_born.cpp:108-131: rows (d*nl + l) = -nu * phi_d .* phi_s .* w
    rng = np.random.default_rng(11)
    N, nl, nd = 300, 3, 4
    inc = rng.standard_normal((N, nl))
    adj = [rng.standard_normal((N, nl)) for _ in range(nd)]
    w = rng.random(N)
    B = oracle.born_block(inc, adj, w, 2.5)
    for d in range(nd):
        for l in range(nl):
            expect = (-2.5) * ((adj[d][:, l] * inc[:, l]) * w)
            assert np.array_equal(B[d * nl + l], expect)


def test_apply7_symmetric_positive(oracle):
    rng = np.random.default_rng(12)
    shape = (7, 6, 5)
    N = 7 * 6 * 5
    x, y = rng.standard_normal(N), rng.standard_normal(N)
    Ax = oracle.apply7(shape, 2.0, 0.1, 1.5, x)
    Ay = oracle.apply7(shape, 2.0, 0.1, 1.5, y)
    assert x @ Ay == pytest.approx(y @ Ax, rel=1e-12)
    assert x @ Ax > 0


def test_fields_match_dense_solve(oracle):
    # test_born.cpp:83-106: fields vs dense direct solves of the shifted system
    shape, h = (8, 7, 6), 2.0
    N = 8 * 7 * 6
    sig, sigp, invD = np.array([0.05, 0.2]), np.array([1.5, 1.6]), np.array([3.0, 3.2])
    v = 3 + 8 * (3 + 7 * 0)  # top plane interior vertex
    F, iters, rel = oracle.fields(shape, h, sig, sigp, invD, [v], tol=1e-12)
    for l in range(2):
        A = np.column_stack([oracle.apply7(shape, h, sig[l], sigp[l], e) for e in np.eye(N)])
        b = np.zeros(N)
        b[v] = 1.0
        phi = np.linalg.solve(A, b) * invD[l]
        assert np.linalg.norm(F[:, l] - phi) <= 1e-9 * np.linalg.norm(phi)
        assert rel[l] <= 1e-12
