"""Oracle parity at the benchmarked configurations (BASELINE configs 1 and 2),
node by node on identical inputs (tests/parity_replay.py):

* config 1 (n=48, N=110592, 16 sources x 6 detectors x 50 wavelengths,
  M=4800): all 31 nodes of the tree -- 16 leaf randsvds, 8 within-leaf
  merges, 7 internal merges -- then recompress of the root
  (lowrank.cpp:131-199, 321-359, 459-521, 547-587);
* config 2 (n=64, N=262144, 32 sources x 8 x 100, M=25600): the whole tree
  replayed on the device, the oracle on the first depth-2 subtree (8 leaf
  randsvds, 4 within-leaf merges, 3 internal merges), on the root merge
  (its core is the largest SVD of the path) and on the recompress.

Also (config 1): the library's own recursive_lowrank driver (speculation,
side-stream V, lazy root) reproduces the replay's node ranks and root factor.

Tolerances (BASELINE north_star): equal ranks; leading singular values 1e-8
relative; ||J~_gpu - J~_cpu||_F / ||J~||_F 1e-8; matvecs 1e-10.  Oracle
pinning: LAPACK stands in for Eigen's HouseholderQR / BDCSVD (bound-pinned
only).  PARITY_LOG=path writes the per-node records.
"""
import json
import os
import time

import numpy as np
import pytest
import torch

from conftest import session_seconds
from parity_replay import Replay, compare, factor_diff, oracle_factor, subtree_nodes

pytestmark = pytest.mark.gpu


def _setup(cfg_id):
    import paper_1410_0986_b200 as h
    from paper_1410_0986_b200 import born, configs, lowrank as lr
    ctx = h.Context(0)
    cfg = configs.CONFIGS[cfg_id]
    st = configs.make_setup(cfg)
    g = st.grid()
    F, stats = born.compute_fields(ctx, g, st.sigma, st.sigma_prime, st.inv_D, st.points, tol=1e-10)
    w = torch.full((g.N,), cfg.h ** 3, dtype=torch.float64, device="cuda")
    inc = [F[st.source_point[s]] for s in range(cfg.n_sources)]
    adj = [[F[st.detector_point[s, d]] for d in range(cfg.n_det)] for s in range(cfg.n_sources)]
    tree = lr.ClusterTree(st.source_xy, st.box_lo, st.box_hi)
    eps = configs.compression_tolerance(st, tree.depth())

    def block(s):
        return born.assemble_H_block(ctx, inc[s], adj[s], w, 1.0)

    return dict(ctx=ctx, cfg=cfg, st=st, g=g, F=F, stats=stats, w=w, inc=inc, adj=adj, tree=tree,
                eps=eps, block=block)


def _write_log(name, rep, extra):
    path = os.environ.get("PARITY_LOG")
    if not path:
        return
    rec = {"config": name, "nodes_checked": rep.checked, "oracle_seconds": rep.oracle_s,
           "node_rank": list(map(int, rep.node_rank)), "records": rep.log}
    rec.update(extra)
    with open(path, "a") as f:
        f.write(json.dumps(rec) + "\n")


def _driver_matches_replay(d, rep, froot):
    """The library's recursive_lowrank (speculation, side-stream V, lazy root
    V) gives the replay's ranks and root factor."""
    from paper_1410_0986_b200 import lowrank as lr
    torch.cuda.synchronize()
    torch.cuda.empty_cache()  # the replay's block and checker temporaries
    rec = lr.recursive_lowrank(d["ctx"], d["tree"], d["eps"],
                               lr.BornFieldsProvider(d["inc"], d["adj"], d["w"], 1.0),
                               lr.RecursiveOptions(seed=d["cfg"].seed))
    assert list(map(int, rec.node_rank)) == list(map(int, rep.node_rank))
    fr = rec.factor
    num, den = factor_diff(fr.U, fr.V, froot.U, froot.V)
    assert num <= 1e-12 * den, num / den
    return rec


def test_config1_every_node_matches_oracle(oracle):
    from paper_1410_0986_b200 import lowrank as lr
    d = _setup(1)
    oracle.set_threads(os.cpu_count() or 1)
    assert float(d["stats"].relres.max()) <= 1e-10
    tree = d["tree"]
    t0 = time.perf_counter()
    rep = Replay(d["ctx"], oracle, tree.nodes, tree.root, d["eps"], d["cfg"].seed, d["block"])
    froot = rep.run()
    assert rep.checked == 16 + 8 + 7
    rec = _driver_matches_replay(d, rep, froot)
    # recompress of the root on identical input
    fg = lr.recompress(d["ctx"], froot, d["eps"])
    fo_root = oracle_factor(oracle, froot)
    fo = oracle.recompress(fo_root, d["eps"])
    compare("recompress", fg, fo, rep.log)
    # J~ products through the chromophore axis and the row permutation
    st, cfg = d["st"], d["cfg"]
    J = lr.JOperator(d["ctx"], fg, rec.row_perm, st.eps_c)
    rng = np.random.default_rng(3)
    X = rng.standard_normal((d["g"].N * cfg.n_chrom, 4))
    yg = J.matvec(torch.as_tensor(X)).cpu().numpy()
    yo = oracle.j_matmat(fo, X, rec.row_perm, st.eps_c)
    assert np.linalg.norm(yg - yo) <= 1e-10 * np.linalg.norm(yo)
    Y = rng.standard_normal((cfg.M, 4))
    xg = J.rmatvec(torch.as_tensor(Y)).cpu().numpy()
    xo = oracle.j_matmat(fo, Y, rec.row_perm, st.eps_c, trans=True)
    assert np.linalg.norm(xg - xo) <= 1e-10 * np.linalg.norm(xo)
    _write_log("cfg1", rep, {"final_rank": fg.rank(), "seconds": time.perf_counter() - t0})


def test_config2_subtree_root_and_recompress_match_oracle(oracle):
    from paper_1410_0986_b200 import lowrank as lr
    d = _setup(2)
    oracle.set_threads(os.cpu_count() or 1)
    assert float(d["stats"].relres.max()) <= 1e-10
    tree = d["tree"]
    nodes = tree.nodes
    # the first depth-2 node on the left spine, and the root
    v2 = nodes[nodes[tree.root]["left"]]["left"]
    check = set(subtree_nodes(nodes, v2)) | {tree.root}
    t0 = time.perf_counter()
    rep = Replay(d["ctx"], oracle, nodes, tree.root, d["eps"], d["cfg"].seed, d["block"],
                 check=lambda v: v in check)
    froot = rep.run()
    assert rep.checked == 8 + 4 + 3 + 1
    _write_log("cfg2-replay", rep, {"seconds": time.perf_counter() - t0})
    # (the library driver is checked against the replay at config 1; here the
    # time goes to the oracle's root merge and recompress)
    del d["F"], d["inc"], d["adj"]
    torch.cuda.empty_cache()
    fg = lr.recompress(d["ctx"], froot, d["eps"])
    # The oracle's recompress of the rank-5686 root takes ~200 s of LAPACK on 16 cores.  The
    # GPU suite has a fixed wall-clock budget (1200 s on the driver's box, ~1000 s used on
    # the boxes measured so far): on a slower host this last check gives way, loudly, so
    # that every other result of the suite is still reported (config 1 checks recompress
    # against the oracle in any case).
    budget = float(os.environ.get("PARITY_SUITE_BUDGET_S", "900"))
    if session_seconds() > budget:
        _write_log("cfg2", rep, {"final_rank": fg.rank(), "seconds": time.perf_counter() - t0,
                                 "recompress_oracle": "skipped: suite time budget"})
        pytest.skip(f"config-2 recompress oracle check skipped after {session_seconds():.0f} s of "
                    f"suite time (budget {budget:.0f} s); subtree and root merge verified")
    fo = oracle.recompress(oracle_factor(oracle, froot), d["eps"])
    compare("recompress", fg, fo, rep.log)
    _write_log("cfg2", rep, {"final_rank": fg.rank(), "seconds": time.perf_counter() - t0})
