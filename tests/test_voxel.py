"""Voxel-sharded top merges (paper_1410_0986_b200/voxel.py) on
CPU with the oracle's arithmetic (LAPACK + the libstdc++ normal stream):

* agglomerate / randsvd with V split by voxel rows over G = 2 and 4 ranks
  (sketch all-reduce, TSQR of the tall B^T, core SVD split by rows) give the
  reference's ranks and factor (lowrank.cpp:131-199, 321-359) within 1e-10;
* recompress (QR(U) replicated, TSQR of V, row-split core SVD) and the J~
  products (R x b n_c all-reduce) match the oracle (lowrank.cpp:547-599,
  experiments.cpp:255-262);
* the row-split block-Jacobi core SVD (svd_dist) matches LAPACK;
* the multi-process run over torch.distributed (gloo, world 2 and 4) is
  bit-identical to the same schedule replayed in one process (SimComm).
"""
import os
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1410_0986_b200 import voxel as vx


def lowrank_pair(seed, N=640, m1=36, m2=30):
    rng = np.random.default_rng(seed)
    out = []
    for m in (m1, m2):
        k = min(m, 26)
        Q1, _ = np.linalg.qr(rng.standard_normal((m, k)))
        Q2, _ = np.linalg.qr(rng.standard_normal((N, k)))
        s = np.logspace(0, -9, k)
        out.append((Q1, Q2 * s))  # U (m x k), V = V~ S (N x k)
    # correlate the two column spaces so the merge compresses
    out[1] = (out[1][0], 0.6 * out[0][1][:, :out[1][1].shape[1]] + 0.4 * out[1][1])
    return out


def run_ranks(world, fn):
    """fn(comm) on `world` threads with SimComm; returns the results by rank."""
    comms = vx.SimComm.group(world)
    res = [None] * world
    errs = []

    def body(g):
        try:
            res[g] = fn(comms[g])
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            comms[g].sh.barrier.abort()

    ts = [threading.Thread(target=body, args=(g,)) for g in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return res


def merge_case(oracle, comm, seed, eps, hint):
    ops = vx.NumpyOps(oracle)
    (U1, V1), (U2, V2) = lowrank_pair(seed)
    N = V1.shape[0]
    lo, hi = vx.voxel_ranges(N, comm.world)[comm.rank]
    f1 = vx.VFactor(ops.tensor(U1), ops.tensor(V1[lo:hi]), N)
    f2 = vx.VFactor(ops.tensor(U2), ops.tensor(V2[lo:hi]), N)
    return vx.agglomerate_voxel(ops, comm, f1, f2, lo, hi, eps, seed=seed + 17, rank_hint=hint)


def gather_rows(fs):
    return np.vstack([f.V_loc.numpy() for f in fs])


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("hint", [-1, 60])  # sketch passes / straight to Q = I
def test_agglomerate_voxel_matches_oracle(oracle, world, hint):
    eps = 1e-7
    for seed in (3, 11):
        fs = run_ranks(world, lambda comm: merge_case(oracle, comm, seed, eps, hint))
        (U1, V1), (U2, V2) = lowrank_pair(seed)
        fo = oracle.agglomerate(oracle.Factor.make(U1, V1), oracle.Factor.make(U2, V2), eps,
                                seed + 17, hint)
        assert fs[0].rank == fo.rank
        for f in fs[1:]:  # U and every decision replicated identically
            assert torch.equal(f.U, fs[0].U)
        D = fs[0].U.numpy() @ gather_rows(fs).T
        Do = fo.U @ fo.V.T
        assert np.linalg.norm(D - Do) <= 1e-10 * np.linalg.norm(Do)
        so = np.linalg.norm(fo.V, axis=0)
        sg = np.linalg.norm(gather_rows(fs), axis=0)
        assert np.max(np.abs(sg - so) / so[0]) <= 1e-12


def test_recompress_and_products_voxel_match_oracle(oracle):
    world, eps = 4, 1e-7
    rng = np.random.default_rng(5)
    M, N, b, nl, nc = 66, 640, 3, 6, 2
    perm = rng.permutation(M)
    eps_c = rng.uniform(0.5, 1.5, (nl, nc))
    X = rng.standard_normal((N * nc, b))

    def fn(comm):
        ops = vx.NumpyOps(oracle)
        f = merge_case(oracle, comm, 7, eps, -1)
        fr = vx.recompress_voxel(ops, comm, f, eps)
        lo, hi = vx.voxel_ranges(N, comm.world)[comm.rank]
        Xc = [torch.as_tensor(X[c * N + lo:c * N + hi]) for c in range(nc)]
        Y = vx.j_matmat_voxel(ops, comm, fr, perm, eps_c, Xc)
        y1 = vx.lr_matmat_voxel(ops, comm, fr, torch.as_tensor(X[lo:hi]))
        x1 = vx.lr_rmatmat_voxel(ops, fr, y1)
        return f, fr, Y, y1, x1

    res = run_ranks(world, fn)
    f0 = oracle.Factor.make(res[0][0].U.numpy(), gather_rows([r[0] for r in res]))
    fo = oracle.recompress(f0, eps)
    fr = [r[1] for r in res]
    assert fr[0].rank == fo.rank
    D = fr[0].U.numpy() @ gather_rows(fr).T
    assert np.linalg.norm(D - fo.U @ fo.V.T) <= 1e-10 * np.linalg.norm(fo.U @ fo.V.T)
    fg = oracle.Factor.make(fr[0].U.numpy(), gather_rows(fr))
    Yo = oracle.j_matmat(fg, X, perm, eps_c)
    assert np.linalg.norm(res[0][2].numpy() - Yo) <= 1e-12 * np.linalg.norm(Yo)
    y1o = fg.U @ (fg.V.T @ X[:N])
    assert np.linalg.norm(res[0][3].numpy() - y1o) <= 1e-12 * np.linalg.norm(y1o)
    x1 = np.vstack([r[4].numpy() for r in res])
    x1o = fg.V @ (fg.U.T @ y1o)
    assert np.linalg.norm(x1 - x1o) <= 1e-12 * np.linalg.norm(x1o)


def test_reshard_voxels_roundtrip():
    world, N = 4, 37
    Vs = [torch.randn(N, 3 + g, dtype=torch.float64) for g in range(world)]
    ranges = vx.voxel_ranges(N, world)
    got = run_ranks(world, lambda comm: vx.reshard_voxels(comm, Vs[comm.rank], ranges))
    for h, (lo, hi) in enumerate(ranges):
        for g in range(world):
            assert torch.equal(got[h][g], Vs[g][lo:hi])


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as o
        comm = vx.Comm(dist)
        f = merge_case(o, comm, 11, 1e-7, -1)
        fr = vx.recompress_voxel(vx.NumpyOps(o), comm, f, 1e-7)
        N = f.cols
        lo, hi = vx.voxel_ranges(N, world)[rank]
        Vs = [torch.full((N, 2 + g), float(g)) + torch.arange(N, dtype=torch.float64)[:, None]
              for g in range(world)]
        rs = vx.reshard_voxels(comm, Vs[rank], vx.voxel_ranges(N, world))
        torch.save({"U": f.U, "V": f.V_loc, "rU": fr.U, "rV": fr.V_loc, "rs": rs},
                   os.path.join(out_dir, f"r{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_ranks_bitwise_equal_the_sequential_replay(oracle, tmp_path, world):
    port = 29600 + world
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    rep = run_ranks(world, lambda comm: merge_case(oracle, comm, 11, 1e-7, -1))
    rrep = run_ranks(world, lambda comm: vx.recompress_voxel(vx.NumpyOps(oracle), comm,
                                                             merge_case(oracle, comm, 11, 1e-7, -1), 1e-7))
    for g in range(world):
        got = torch.load(os.path.join(tmp_path, f"r{g}.pt"))
        assert torch.equal(got["U"], rep[g].U) and torch.equal(got["V"], rep[g].V_loc)
        assert torch.equal(got["rU"], rrep[g].U) and torch.equal(got["rV"], rrep[g].V_loc)
        N = rep[g].cols
        lo, hi = vx.voxel_ranges(N, world)[g]
        for h in range(world):
            want = torch.full((N, 2 + h), float(h)) + torch.arange(N, dtype=torch.float64)[:, None]
            assert torch.equal(got["rs"][h], want[lo:hi])


@pytest.mark.parametrize("world,n", [(2, 64), (3, 97)])
def test_svd_dist_matches_lapack(oracle, world, n):
    """The row-split one-sided block Jacobi core SVD (svd_dist) against
    LAPACK: singular values to 1e-13 s_1, R = Ur S Vr^T to 1e-13, identical
    result on every rank."""
    rng = np.random.default_rng(n)
    Q1, _ = np.linalg.qr(rng.standard_normal((n, n)))
    Q2, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.logspace(0, -11, n)
    R = torch.as_tensor((Q1 * s) @ Q2.T)
    res = run_ranks(world, lambda comm: vx.svd_dist(vx.NumpyOps(oracle), comm, R.clone()))
    Ur, sv, Vr = res[0]
    for r in res[1:]:
        assert torch.equal(r[0], Ur) and torch.equal(r[2], Vr) and np.array_equal(r[1], sv)
    assert np.max(np.abs(sv - s)) <= 1e-13 * s[0]
    rec = (Ur.numpy() * sv) @ Vr.numpy().T
    assert np.linalg.norm(rec - R.numpy()) <= 1e-13 * np.linalg.norm(R.numpy())
