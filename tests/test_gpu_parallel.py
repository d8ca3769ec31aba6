"""The source-sharded driver with the device engine (parallel.GpuEngine)
over torch.distributed at world 2 (gloo; both ranks on cuda:0, each working
independently -- factors cross through host memory, no kernel waits on
another rank): the sharded root factor and its global row order equal the
same schedule replayed sequentially by the CPU oracle on identical fields
(ranks equal, ||J~_gpu - J~_oracle|| <= 1e-8 ||J~||).  Covers
GpuEngine.to_tensors / from_tensors, _recv_factor's device placement and the
top merges with rank_hint = -1."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from test_parallel import box_of, sequential_sharded, small_problem

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, fpath, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1410_0986_b200 as h
        from paper_1410_0986_b200 import configs, lowrank as lr
        from paper_1410_0986_b200.parallel import GpuEngine, global_row_perm, make_plan, reduce_tree
        from oracle import oracle as o
        cfg = configs.small_config(n=10, ns_x=4, ns_y=2, n_det=2, n_lambda=3)
        st = configs.make_setup(cfg)
        F = np.load(fpath)  # (points, nl, N): the oracle's fields
        ctx = h.Context(0)
        dev = torch.device("cuda:0")
        tree = o.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
        plan = make_plan(tree.nodes, tree.root, world)
        eps = configs.compression_tolerance(st, tree.depth())
        v = plan.shard_roots[rank]
        srcs = plan.shard_sources[rank]
        lo, hi = box_of(tree, v, st)
        Fd = torch.as_tensor(F).to(dev)
        w = torch.full((cfg.N,), cfg.h ** 3, dtype=torch.float64, device=dev)
        prov = lr.BornFieldsProvider([Fd[st.source_point[s]] for s in srcs],
                                     [[Fd[st.detector_point[s, d]] for d in range(cfg.n_det)] for s in srcs],
                                     w, 1.0)
        eng = GpuEngine(ctx)
        rec = eng.compress_subtree(st.source_xy[srcs], lo, hi, srcs, v, eps, prov, cfg.seed, 20, 10)
        root = reduce_tree(plan, rank, rec.factor, eng, eps, cfg.seed, 20, 10, dist, dev)
        orders = [None] * world
        dist.all_gather_object(orders, [srcs[i] for i in lr.ClusterTree(st.source_xy[srcs], lo, hi).leaf_order()])
        if rank == 0:
            perm = global_row_perm(plan, cfg.rows_per_source, orders)
            np.savez(os.path.join(out_dir, "root.npz"), U=root.U.cpu().numpy(), V=root.V.cpu().numpy(), perm=perm)
    finally:
        dist.destroy_process_group()


def test_gpu_engine_reduction_tree_world2_matches_oracle_replay(oracle, tmp_path):
    world = 2
    cfg, st, F = small_problem(oracle)
    fpath = str(tmp_path / "fields.npy")
    np.save(fpath, np.ascontiguousarray(F))
    mp.spawn(_worker, args=(world, 29731, fpath, str(tmp_path)), nprocs=world, join=True)
    got = np.load(str(tmp_path / "root.npz"))
    f_seq, perm_seq, _, _ = sequential_sharded(oracle, cfg, st, F, world)
    assert got["U"].shape[1] == f_seq.rank
    assert np.array_equal(got["perm"], perm_seq)
    Dg = got["U"] @ got["V"].T
    Do = f_seq.U @ f_seq.V.T
    assert np.linalg.norm(Dg - Do) <= 1e-8 * np.linalg.norm(Do)
