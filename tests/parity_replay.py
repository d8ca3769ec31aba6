"""Node-level parity replay of recursive_lowrank (lowrank.cpp:459-521) at the
benchmarked sizes.

The device path runs the reference recursion node by node through the
public per-node entry points (hydot_randsvd for every leaf source,
hydot_agglomerate for every merge) with the reference's seeds
(lowrank.cpp:485, 494, 500) and both warm-start chains (leaf_hint across
leaves in DFS order, depth_hint per depth, lowrank.cpp:480-488, 491-508).
At the nodes selected for checking, the CPU oracle runs the same node on the
SAME inputs -- the device's Born block for a leaf, the device's child factors
for a merge, downloaded -- so each comparison isolates one node:

* equal rank (the keep rule s_i > eps s_1, lowrank.cpp:187-190, and the
  sketch accept/reject chain, :176-181);
* leading singular values (the column norms of V = V~ S) within 1e-8
  relative;
* ||U_g V_g^T - U_o V_o^T||_F / ||U_o V_o^T||_F <= 1e-8, formed in row chunks
  on the device (torch matmul is the checker here, not the product).

The replay then continues with the device factor, so every later node is
again compared on identical inputs.  Oracle pinning caveat: the oracle's
QR/SVD are LAPACK's (dgeqrf/dgesdd for Eigen's HouseholderQR/BDCSVD), which
the reference pins only through bounds.
"""
from __future__ import annotations

import time

import numpy as np
import torch

SEED_LEAF = 0x9E3779B97F4A7C15  # lowrank.cpp:485
SEED_WITHIN = 0x517CC1B727220A95  # lowrank.cpp:494
SEED_INTERNAL = 0x2545F4914F6CDD1D  # lowrank.cpp:500
MASK = 2 ** 64 - 1
TOL_SIGMA = 1e-8
TOL_J = 1e-8


def factor_diff(Ug, Vg, Uo, Vo, chunk=1024):
    """||Ug Vg^T - Uo Vo^T||_F and ||Uo Vo^T||_F, row chunks on the device."""
    dev = Ug.device
    Uo = torch.as_tensor(Uo, device=dev)
    Vo = torch.as_tensor(Vo, device=dev)
    num = torch.zeros((), dtype=torch.float64, device=dev)
    den = torch.zeros((), dtype=torch.float64, device=dev)
    for i in range(0, Ug.shape[0], chunk):
        A = Ug[i:i + chunk] @ Vg.T
        B = Uo[i:i + chunk] @ Vo.T
        num += torch.sum((A - B) ** 2)
        den += torch.sum(B ** 2)
        del A, B
    return float(num.sqrt()), float(den.sqrt())


def compare(label, fg, fo, log):
    """fg: device LowRankFactor, fo: oracle Factor (same inputs)."""
    rg, ro = fg.rank(), fo.rank
    rec = {"node": label, "rank_gpu": rg, "rank_oracle": ro}
    if rg != ro:
        log.append(rec)
        raise AssertionError(f"{label}: rank {rg} (device) != {ro} (oracle)")
    if rg == 0:
        log.append(rec)
        return rec
    Ug, Vg = fg.U, fg.V
    sg = torch.linalg.norm(Vg, dim=0).cpu().numpy()
    so = np.linalg.norm(fo.V, axis=0)
    k = min(10, rg)
    rel_sigma = float(np.max(np.abs(sg[:k] - so[:k]) / so[:k]))
    abs_sigma = float(np.max(np.abs(sg - so)) / so[0])
    num, den = factor_diff(Ug, Vg, fo.U, fo.V)
    rec.update(rel_sigma_lead=rel_sigma, abs_sigma_all=abs_sigma, rel_J=num / den)
    log.append(rec)
    assert rel_sigma <= TOL_SIGMA, (label, rel_sigma)
    assert num <= TOL_J * den, (label, num / den)
    return rec


def oracle_factor(oracle, f):
    """Download a device factor into the oracle (same flagged bit)."""
    return oracle.Factor.make(f.U.cpu().numpy(), f.V.cpu().numpy(), f.tol, f.method, f.flagged)


class Replay:
    """Reference recursion, node by node on the device, oracle at `check`
    nodes.  block(s) -> (rows_per x N) CUDA tensor of source s (global id)."""

    def __init__(self, ctx, oracle, nodes, root, eps, seed, block, check=lambda v: True,
                 p=20, kprobe=10):
        self.ctx, self.o, self.nodes, self.root = ctx, oracle, nodes, root
        self.eps, self.seed, self.block, self.check = eps, seed, block, check
        self.p, self.kprobe = p, kprobe
        self.leaf_hint = -1
        self.depth_hint = {}
        self.node_rank = [-1] * len(nodes)
        self.log = []
        self.oracle_s = 0.0
        self.checked = 0

    def node_hint(self, depth):
        return self.depth_hint[depth] + 2 if depth in self.depth_hint else -1

    def _merge(self, label, f1, f2, seed, hint, do_check):
        from paper_1410_0986_b200 import lowrank as lr
        fg = lr.agglomerate(self.ctx, f1, f2, self.eps, seed, rank_hint=hint, p=self.p,
                            kprobe=self.kprobe)
        if do_check:
            t0 = time.perf_counter()
            fo = self.o.agglomerate(oracle_factor(self.o, f1), oracle_factor(self.o, f2), self.eps,
                                    seed, hint, self.p, self.kprobe)
            self.oracle_s += time.perf_counter() - t0
            compare(label, fg, fo, self.log)
            self.checked += 1
        return fg

    def go(self, v, depth=0):
        from paper_1410_0986_b200 import lowrank as lr
        nd = self.nodes[v]
        do_check = self.check(v)
        if nd["left"] < 0:
            parts = []
            for s in nd["idx"]:
                A = self.block(int(s))
                r0 = max(1, self.leaf_hint + 2)
                seed = (self.seed + SEED_LEAF * (int(s) + 1)) & MASK
                fg = lr.randsvd(self.ctx, A, self.eps, self.p, self.kprobe, seed, cat=lr.LEAF, r0=r0)
                if do_check:
                    t0 = time.perf_counter()
                    fo = self.o.randsvd(A.cpu().numpy(), self.eps, self.p, self.kprobe, seed,
                                        self.o.LEAF, r0)
                    self.oracle_s += time.perf_counter() - t0
                    compare(f"leaf s{s} (node {v})", fg, fo, self.log)
                    self.checked += 1
                del A
                self.leaf_hint = fg.rank()
                parts.append(fg)
            f = parts[0]
            for i in range(1, len(parts)):
                f = self._merge(f"within-leaf merge node {v}", f, parts[i],
                                (self.seed + SEED_WITHIN * (v + 1)) & MASK, self.node_hint(depth),
                                do_check)
        else:
            fl = self.go(nd["left"], depth + 1)
            fr = self.go(nd["right"], depth + 1)
            f = self._merge(f"merge node {v} (depth {depth})", fl, fr,
                            (self.seed + SEED_INTERNAL * (v + 1)) & MASK, self.node_hint(depth),
                            do_check)
        self.node_rank[v] = f.rank()
        self.depth_hint[depth] = f.rank()
        return f

    def run(self):
        return self.go(self.root, 0)


def subtree_nodes(nodes, v):
    out = [v]
    nd = nodes[v]
    if nd["left"] >= 0:
        out += subtree_nodes(nodes, nd["left"]) + subtree_nodes(nodes, nd["right"])
    return out
