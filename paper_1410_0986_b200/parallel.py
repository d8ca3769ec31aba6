"""Source-sharded compression across GPUs.

The cluster tree (lowrank.cpp:385-438) is cut at depth d = log2(world): rank g
owns the g-th subtree at that depth (left-to-right), computes the fields of its
own sources and detectors, assembles and compresses its subtree with no
communication, then the top d levels are merged by a reduction tree: the
owner of a right child sends its factor (U, V) to the owner of the left child,
which runs agglomerate (lowrank.cpp:321-359) with the node's reference seed.
Rank 0 ends with the root factor and recompresses it (experiments.cpp:249-250).

Semantics vs the sequential reference: seeds and row order are the global
ones (source ids / pre-order node ids are passed to the shard), the warm-start
hint chains (lowrank.cpp:466-471) restart on every shard, and the top merges
use rank_hint = -1.  The oracle replays exactly this schedule
(tests/test_parallel.py), so the sharded result has a CPU reference too.

The engine is pluggable (GPU engine below; tests inject an oracle engine) so
the exchange logic is testable with gloo on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import numpy as np
import torch

SEED_INTERNAL = 0x2545F4914F6CDD1D  # lowrank.cpp:500


@dataclass
class ShardPlan:
    world: int
    depth: int
    shard_roots: List[int]                 # node id per rank
    shard_sources: List[List[int]]         # global source ids per rank (node idx order)
    owner: Dict[int, int]                  # node -> rank holding its factor
    merges: List[Tuple[int, int, int, int]] = field(default_factory=list)  # (u, a, b, depth) post-order


def subtree_size(nodes, v) -> int:
    nd = nodes[v]
    if nd["left"] < 0:
        return 1
    return 1 + subtree_size(nodes, nd["left"]) + subtree_size(nodes, nd["right"])


def make_plan(nodes, root: int, world: int) -> ShardPlan:
    if world < 1 or (world & (world - 1)):
        raise ValueError("world size must be a power of two")
    d = world.bit_length() - 1
    frontier = [root]
    for _ in range(d):
        nxt = []
        for v in frontier:
            if nodes[v]["left"] < 0:
                raise ValueError("cluster tree too shallow for this many GPUs")
            nxt += [nodes[v]["left"], nodes[v]["right"]]
        frontier = nxt
    owner = {v: g for g, v in enumerate(frontier)}
    merges = []

    def post(v, depth):
        if v in owner:
            return owner[v]
        a, b = nodes[v]["left"], nodes[v]["right"]
        oa = post(a, depth + 1)
        post(b, depth + 1)
        merges.append((v, a, b, depth))
        owner[v] = oa
        return oa

    post(root, 0)
    return ShardPlan(world, d, frontier, [list(nodes[v]["idx"]) for v in frontier], owner, merges)


def _wire(dist, device):
    """the device messages travel on: the tensors' own device with NCCL, host
    memory with gloo (which has no device-tensor send / recv)"""
    return torch.device("cpu") if dist.get_backend() == "gloo" else device


def _send_factor(U: torch.Tensor, V: torch.Tensor, flagged: bool, dst: int, dist):
    w = _wire(dist, U.device)
    hdr = torch.tensor([U.shape[0], V.shape[0], U.shape[1], int(flagged)], dtype=torch.int64, device=w)
    dist.send(hdr, dst)
    if U.shape[1]:
        dist.send(U.contiguous().to(w), dst)
        dist.send(V.contiguous().to(w), dst)


def _recv_factor(src: int, device, dist):
    w = _wire(dist, device)
    hdr = torch.empty(4, dtype=torch.int64, device=w)
    dist.recv(hdr, src)
    rows, cols, rank, flagged = (int(x) for x in hdr.tolist())
    U = torch.empty(rows, rank, dtype=torch.float64, device=w)
    V = torch.empty(cols, rank, dtype=torch.float64, device=w)
    if rank:
        dist.recv(U, src)
        dist.recv(V, src)
    return U.to(device), V.to(device), bool(flagged)


def reduce_tree(plan: ShardPlan, rank: int, local_factor, engine, eps: float, seed: int, p: int,
                kprobe: int, dist, device):
    """Run the top merges; returns the root factor on rank 0, None elsewhere."""
    held = {plan.shard_roots[rank]: local_factor}
    for (u, a, b, _depth) in plan.merges:
        oa, ob = plan.owner[a], plan.owner[b]
        if rank == ob and oa != ob:
            U, V, fl = engine.to_tensors(held.pop(b))
            _send_factor(U, V, fl, oa, dist)
        elif rank == oa:
            fa = held.pop(a)
            if ob == oa:
                fb = held.pop(b)
            else:
                fb = engine.from_tensors(*_recv_factor(ob, device, dist))
            held[u] = engine.agglomerate(fa, fb, eps, (seed + SEED_INTERNAL * (u + 1)) & (2**64 - 1),
                                         -1, p, kprobe)
    return held.get(plan.merges[-1][0] if plan.merges else plan.shard_roots[0]) if rank == 0 else None


def global_row_perm(plan: ShardPlan, rows_per: int, leaf_orders: List[List[int]]) -> np.ndarray:
    """Factor row i <-> H row (experiments.cpp rows: source-major)."""
    out = []
    for order in leaf_orders:
        for s in order:
            out.extend(s * rows_per + q for q in range(rows_per))
    return np.asarray(out, dtype=np.int32)


# --------------------------------------------------------------- GPU engine --
class GpuEngine:
    """Engine over the CUDA library (paper_1410_0986_b200.lowrank)."""

    def __init__(self, ctx):
        from . import lowrank as lr
        self.ctx, self.lr = ctx, lr

    def compress_subtree(self, positions, lo, hi, sources, node_offset, eps, provider, seed, p,
                         kprobe):
        lr = self.lr
        sub = lr.ClusterTree(positions, lo, hi)
        opts = lr.RecursiveOptions(seed=seed, p=p, kprobe=kprobe, source_ids=list(sources),
                                   node_offset=node_offset)
        rec = lr.recursive_lowrank(self.ctx, sub, eps, provider, opts)
        return rec

    def agglomerate(self, fa, fb, eps, seed, hint, p, kprobe):
        return self.lr.agglomerate(self.ctx, fa, fb, eps, seed, None, hint, p, kprobe)

    def to_tensors(self, f):
        return f.U.contiguous(), f.V.contiguous(), f.flagged

    def from_tensors(self, U, V, flagged):
        return self.lr.LowRankFactor.from_tensors(self.ctx, U, V, flagged=flagged)

    def recompress(self, f, eps):
        return self.lr.recompress(self.ctx, f, eps)
