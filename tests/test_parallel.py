"""Multi-GPU sharding logic (paper_1410_0986_b200/parallel.py) on CPU.

The shard plan, the reduction-tree exchange (torch.distributed, gloo,
world_size 2 and 4) and the global seeds/row order are exercised with the CPU
oracle as the compute engine; the sharded result must equal the same schedule
replayed sequentially in one process, bit for bit, and approximate the
unsharded compression to the scheduled tolerance.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1410_0986_b200 import configs
from paper_1410_0986_b200.parallel import make_plan, reduce_tree, global_row_perm


class OracleEngine:
    def __init__(self, o, setup, F):
        self.o, self.st, self.F = o, setup, F

    def compress_subtree(self, sources, lo, hi, node_offset, eps, seed):
        o, st, F = self.o, self.st, self.F
        cfg = st.cfg
        sub = o.ClusterTree(st.source_xy[sources], lo, hi)
        inc = [F[st.source_point[s]].T for s in sources]
        adj = [[F[st.detector_point[s, d]].T for d in range(cfg.n_det)] for s in sources]
        w = np.full(cfg.N, cfg.h ** 3)
        rec = o.recursive_lowrank_born(sub, eps, inc, adj, w, 1.0, seed=seed, source_ids=sources,
                                       node_offset=node_offset)
        return rec, sub.leaf_order()

    def agglomerate(self, fa, fb, eps, seed, hint, p, kprobe):
        return self.o.agglomerate(fa, fb, eps, seed, hint, p, kprobe)

    def to_tensors(self, f):
        return torch.as_tensor(f.U.copy()), torch.as_tensor(f.V.copy()), f.flagged

    def from_tensors(self, U, V, flagged):
        return self.o.Factor.make(U.numpy(), V.numpy(), flagged=flagged)


def small_problem(oracle):
    cfg = configs.small_config(n=10, ns_x=4, ns_y=2, n_det=2, n_lambda=3)
    st = configs.make_setup(cfg)
    g = st.grid()
    Fo, _, _ = oracle.fields((g.nx, g.ny, g.nz), g.h, st.sigma, st.sigma_prime, st.inv_D,
                             st.points, tol=1e-12)
    F = Fo.T.reshape(len(st.points), cfg.n_lambda, g.N)
    return cfg, st, F


def box_of(tree, v, st):
    # replay the bisection boxes (lowrank.cpp:403-412) down to node v
    lo, hi = st.box_lo.astype(float).copy(), st.box_hi.astype(float).copy()

    def walk(u, lo, hi):
        if u == v:
            return lo, hi
        nd = tree.nodes[u]
        if nd["left"] < 0:
            return None
        idx = nd["idx"]
        ax = int(np.argmax(hi - lo)) if (hi - lo).max() > (hi - lo)[0] else 0
        mid = 0.5 * (lo[ax] + hi[ax])
        left = [i for i in idx if st.source_xy[i, ax] <= mid]
        l_hi, r_lo = hi.copy(), lo.copy()
        if 0 < len(left) < len(idx):
            l_hi[ax] = mid
            r_lo[ax] = mid
        return walk(nd["left"], lo, l_hi) or walk(nd["right"], r_lo, hi)

    return walk(tree.root, lo, hi)


def sequential_sharded(oracle, cfg, st, F, world):
    tree = oracle.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
    plan = make_plan(tree.nodes, tree.root, world)
    eps = configs.compression_tolerance(st, tree.depth())
    eng = OracleEngine(oracle, st, F)
    held, orders = {}, []
    for g, v in enumerate(plan.shard_roots):
        lo, hi = box_of(tree, v, st)
        rec, order = eng.compress_subtree(plan.shard_sources[g], lo, hi, v, eps, cfg.seed)
        held[v] = rec.factor
        orders.append([plan.shard_sources[g][i] for i in order])
    for (u, a, b, _d) in plan.merges:
        held[u] = eng.agglomerate(held.pop(a), held.pop(b), eps,
                                  (cfg.seed + 0x2545F4914F6CDD1D * (u + 1)) & (2**64 - 1), -1, 20, 10)
    root = plan.merges[-1][0] if plan.merges else plan.shard_roots[0]
    return held[root], global_row_perm(plan, cfg.rows_per_source, orders), tree, eps


def test_plan_on_baseline_trees(oracle):
    for cid, worlds in [(1, (1, 2, 4, 8)), (2, (1, 2, 4, 8)), (3, (1, 2, 4, 8))]:
        st = configs.make_setup(configs.CONFIGS[cid])
        t = oracle.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
        for w in worlds:
            plan = make_plan(t.nodes, t.root, w)
            assert len(plan.shard_roots) == w
            srcs = sorted(s for ss in plan.shard_sources for s in ss)
            assert srcs == list(range(st.cfg.n_sources))
            assert len(plan.merges) == w - 1
            assert plan.owner[t.root] == 0
            # every merge's children are owned before the merge runs (post-order)
            done = set(plan.shard_roots)
            for (u, a, b, _) in plan.merges:
                assert a in done and b in done
                done.add(u)
    with pytest.raises(ValueError):
        make_plan(t.nodes, t.root, 3)


def test_sharded_replay_approximates_unsharded(oracle):
    cfg, st, F = small_problem(oracle)
    f2, perm2, tree, eps = sequential_sharded(oracle, cfg, st, F, 2)
    w = np.full(cfg.N, cfg.h ** 3)
    inc = [F[st.source_point[s]].T for s in range(cfg.n_sources)]
    adj = [[F[st.detector_point[s, d]].T for d in range(cfg.n_det)] for s in range(cfg.n_sources)]
    full = oracle.recursive_lowrank_born(tree, eps, inc, adj, w, 1.0, seed=cfg.seed)
    H = np.vstack([oracle.born_block(inc[s], adj[s], w, 1.0) for s in range(cfg.n_sources)])
    J2 = np.zeros_like(H)
    J2[perm2] = f2.dense()
    J1 = np.zeros_like(H)
    J1[full.row_perm] = full.factor.dense()
    assert np.array_equal(np.sort(perm2), np.arange(cfg.M))
    nh = np.linalg.norm(H)
    assert np.linalg.norm(H - J2) <= 50 * cfg.eps_d * nh
    assert np.linalg.norm(J1 - J2) <= 50 * cfg.eps_d * nh


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as o
        cfg, st, F = small_problem(o)
        tree = o.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
        plan = make_plan(tree.nodes, tree.root, world)
        eps = configs.compression_tolerance(st, tree.depth())
        eng = OracleEngine(o, st, F)
        v = plan.shard_roots[rank]
        lo, hi = box_of(tree, v, st)
        rec, order = eng.compress_subtree(plan.shard_sources[rank], lo, hi, v, eps, cfg.seed)
        root = reduce_tree(plan, rank, rec.factor, eng, eps, cfg.seed, 20, 10, dist,
                           torch.device("cpu"))
        if rank == 0:
            q.put((root.U.copy(), root.V.copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_reduction_tree_matches_sequential(oracle, world):
    cfg, st, F = small_problem(oracle)
    f_seq, _, _, _ = sequential_sharded(oracle, cfg, st, F, world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 7 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    U, V = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert np.array_equal(U, f_seq.U) and np.array_equal(V, f_seq.V)
