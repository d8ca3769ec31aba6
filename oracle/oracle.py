"""ctypes wrapper around the CPU ORACLE (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg as the checker and the CPU
baseline.  The product package (paper_1410_0986_b200) never imports it.
See hydot_oracle.cpp for the restated reference lines and the parity-pin
status ("pinned by the reference's known-answer tests; Eigen numerics pinned
by bounds").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_tolerance_schedule.restype = C.c_double
        L.oracle_tolerance_schedule.argtypes = [C.c_double, C.c_int, C.c_int]
        L.oracle_gaussian.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.oracle_mt19937_64.argtypes = [C.c_uint64, C.c_int64, _u64p]
        L.oracle_born_block.argtypes = [C.c_int64, C.c_int, _dp, C.POINTER(_dp), C.c_int, _dp,
                                        C.c_double, _dp]
        L.oracle_apply7.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_double, _dp, _dp]
        L.oracle_fields.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _dp, _dp,
                                    _dp, _i64p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                    _dp, _ip, _dp]
        L.oracle_fields_var.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _dp, _dp, _dp, _dp,
                                        _dp, _i64p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, _dp, _ip,
                                        _dp]
        L.oracle_factor_free.argtypes = [C.c_void_p]
        L.oracle_factor_info.argtypes = [C.c_void_p, _i64p, _i64p, _i64p, _dp, _ip, _ip]
        L.oracle_factor_get.argtypes = [C.c_void_p, _dp, _dp]
        L.oracle_factor_meta.argtypes = [C.c_void_p, _ip, _ip, _ip, _dp]
        L.oracle_factor_perm_len.argtypes = [C.c_void_p]
        L.oracle_factor_perm_len.restype = C.c_int64
        L.oracle_factor_make.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                         C.c_int, C.c_int]
        L.oracle_factor_make.restype = C.c_void_p
        L.oracle_randsvd.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                     C.c_int, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_agglomerate.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_uint64, C.c_int,
                                         C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_recompress.argtypes = [C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_build_cluster_tree.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp,
                                                C.POINTER(C.c_void_p)]
        L.oracle_tree_free.argtypes = [C.c_void_p]
        for n in ("oracle_tree_num_nodes", "oracle_tree_root", "oracle_tree_depth"):
            getattr(L, n).argtypes = [C.c_void_p]
        L.oracle_tree_node.argtypes = [C.c_void_p, C.c_int, _ip, _ip, _ip]
        L.oracle_tree_node_idx.argtypes = [C.c_void_p, C.c_int, _ip]
        L.oracle_tree_leaf_order.argtypes = [C.c_void_p, _ip]
        L.oracle_recursive_lowrank.argtypes = [C.c_void_p, C.c_double, _dp, C.c_int64, C.c_int64,
                                               C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                               C.POINTER(C.c_void_p)]
        L.oracle_recursive_lowrank_born.argtypes = [C.c_void_p, C.c_double, C.c_int64, C.c_int,
                                                    C.c_int, C.POINTER(_dp), C.POINTER(_dp), _dp,
                                                    C.c_double, C.c_uint64, C.c_int, C.c_int, _ip,
                                                    C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_lr_matmat.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp]
        L.oracle_j_matmat.argtypes = [C.c_void_p, C.c_int, C.c_int, _ip, _dp, C.c_int, C.c_int,
                                      _dp, _dp]
        L.oracle_fast_thin_svd.argtypes = [_dp, C.c_int64, C.c_int64, _dp, _dp, _dp]
        L.oracle_save_factor.argtypes = [C.c_char_p, C.c_void_p, _ip, C.c_int64]
        L.oracle_set_threads.argtypes = [C.c_int]
        _LIB = L
        L.oracle_set_threads(1)  # reference hot path is single-threaded
    return _LIB


def _d(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(rc):
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


LEAF, AGGLOMERATION, RECOMPRESS, OTHER = 0, 1, 2, 3


def tolerance_schedule(eps_d, L, N_r):
    v = lib().oracle_tolerance_schedule(eps_d, L, N_r)
    if v < 0:
        raise ValueError("tolerance_schedule: bad arguments")
    return v


def gaussian(seed, count):
    out = np.empty(count, dtype=np.float64)
    _check(lib().oracle_gaussian(C.c_uint64(seed & (2**64 - 1)), count, _d(out)))
    return out


def mt19937_64(seed, count):
    out = np.empty(count, dtype=np.uint64)
    _check(lib().oracle_mt19937_64(C.c_uint64(seed & (2**64 - 1)), count,
                                   out.ctypes.data_as(_u64p)))
    return out


def born_block(incident, adjoint_list, w, nu):
    """incident N x nl (F-order), adjoint_list[d] N x nl -> block (nd*nl) x N."""
    N, nl = incident.shape
    inc = np.asfortranarray(incident, dtype=np.float64)
    adj = [np.asfortranarray(a, dtype=np.float64) for a in adjoint_list]
    arr = (_dp * len(adj))(*[_d(a) for a in adj])
    out = np.empty((len(adj) * nl, N), dtype=np.float64)  # row-major
    w = _f64(w)
    _check(lib().oracle_born_block(N, nl, _d(inc), arr, len(adj), _d(w), nu, _d(out)))
    return out


def apply7(shape, h, sigma, sigmap, x):
    nx, ny, nz = shape
    x = _f64(x)
    y = np.empty_like(x)
    _check(lib().oracle_apply7(nx, ny, nz, h, sigma, sigmap, _d(x), _d(y)))
    return y


def fields(shape, h, sigma, sigmap, inv_D, rhs_vertex, tol=1e-10, max_iter=10000,
           fixed_iters=0, threads=1):
    nx, ny, nz = shape
    N = nx * ny * nz
    nl = len(sigma)
    rv = np.ascontiguousarray(rhs_vertex, dtype=np.int64)
    out = np.empty((N, len(rv) * nl), dtype=np.float64, order="F")
    iters = np.zeros(len(rv) * nl, dtype=np.int32)
    rel = np.zeros(len(rv) * nl, dtype=np.float64)
    _check(lib().oracle_fields(nx, ny, nz, h, nl, _d(_f64(sigma)), _d(_f64(sigmap)),
                               _d(_f64(inv_D)), rv.ctypes.data_as(_i64p), len(rv), tol, max_iter,
                               fixed_iters, threads, _d(out), iters.ctypes.data_as(_ip),
                               _d(rel)))
    return out, iters, rel


def fields_var(shape, h, sigma, sigmap, inv_D, dsig, mu, rhs_vertex, tol=1e-10, max_iter=10000,
               fixed_iters=0, threads=1):
    """Fields of the perturbed medium sigma_l + dsig_l mu(v) (the nonlinear
    forward model's solves, experiments.cpp:154-206); layout as fields()."""
    nx, ny, nz = shape
    N = nx * ny * nz
    nl = len(sigma)
    rv = np.ascontiguousarray(rhs_vertex, dtype=np.int64)
    out = np.empty((N, len(rv) * nl), dtype=np.float64, order="F")
    iters = np.zeros(len(rv) * nl, dtype=np.int32)
    rel = np.zeros(len(rv) * nl, dtype=np.float64)
    _check(lib().oracle_fields_var(nx, ny, nz, h, nl, _d(_f64(sigma)), _d(_f64(sigmap)), _d(_f64(inv_D)),
                                   _d(_f64(dsig)), _d(_f64(mu)), rv.ctypes.data_as(_i64p), len(rv), tol,
                                   max_iter, fixed_iters, threads, _d(out), iters.ctypes.data_as(_ip),
                                   _d(rel)))
    return out, iters, rel


def full_forward(shape, h, sigma, sigmap, inv_D, dsig, mu, source_vertex, detector_vertex, tol=1e-10,
                 fixed_iters=0, threads=1):
    """experiments::full_diffusion_forward (experiments.cpp:154-206) for the
    7-point operator: y_total / y_incident at the detector vertices,
    measurement (s, d, l) -> (s * n_det + d) * n_lambda + l."""
    nl = len(sigma)
    src = np.asarray(source_vertex, dtype=np.int64)
    det = np.asarray(detector_vertex, dtype=np.int64).reshape(len(src), -1)
    nd = det.shape[1]
    outs = []
    for ds in (np.asarray(dsig, dtype=np.float64), np.zeros(nl)):
        F, it, rel = fields_var(shape, h, sigma, sigmap, inv_D, ds, mu, src, tol=tol, fixed_iters=fixed_iters,
                                threads=threads)
        y = np.empty(len(src) * nd * nl)
        for s in range(len(src)):
            for d in range(nd):
                for l in range(nl):
                    y[(s * nd + d) * nl + l] = F[det[s, d], s * nl + l]
        outs.append(y)
    return outs[0], outs[1], outs[0] - outs[1]


class Factor:
    """LowRankFactor (lowrank.hpp:25-36) held by the oracle."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)
        r, c, k = C.c_int64(), C.c_int64(), C.c_int64()
        tol, meth, flag = C.c_double(), C.c_int(), C.c_int()
        lib().oracle_factor_info(self.h, C.byref(r), C.byref(c), C.byref(k), C.byref(tol),
                                 C.byref(meth), C.byref(flag))
        self.rows, self.cols, self.rank = r.value, c.value, k.value
        self.tol, self.method, self.flagged = tol.value, meth.value, bool(flag.value)
        U = np.empty((self.rows, self.rank), order="F")
        V = np.empty((self.cols, self.rank), order="F")
        lib().oracle_factor_get(self.h, _d(U), _d(V))
        self.U, self.V = U, V
        plen = lib().oracle_factor_perm_len(self.h)
        self.row_perm = np.zeros(plen, dtype=np.int32)
        self.ledger = np.zeros(5)
        lib().oracle_factor_meta(self.h, self.row_perm.ctypes.data_as(_ip), None, None,
                                 _d(self.ledger))

    @classmethod
    def make(cls, U, V, tol=0.0, method=0, flagged=False):
        U = np.asfortranarray(U, dtype=np.float64)
        V = np.asfortranarray(V, dtype=np.float64)
        h = lib().oracle_factor_make(_d(U), _d(V), U.shape[0], V.shape[0], U.shape[1], tol,
                                     method, int(flagged))
        return cls(h)

    def dense(self):
        return self.U @ self.V.T

    def __del__(self):
        try:
            lib().oracle_factor_free(self.h)
        except Exception:
            pass


def randsvd(A, eps, p=20, kprobe=10, seed=0, cat=OTHER, r0=1):
    A = np.asfortranarray(A, dtype=np.float64)
    h = C.c_void_p()
    m, n = A.shape
    _check(lib().oracle_randsvd(_d(A), m, n, max(m, 1), eps, p, kprobe,
                                C.c_uint64(seed & (2**64 - 1)), cat, r0, C.byref(h)))
    return Factor(h.value)


def agglomerate(f1, f2, eps, seed=0, rank_hint=-1, p=20, kprobe=10):
    h = C.c_void_p()
    _check(lib().oracle_agglomerate(f1.h, f2.h, eps, C.c_uint64(seed & (2**64 - 1)), rank_hint,
                                    p, kprobe, C.byref(h)))
    return Factor(h.value)


def recompress(f, eps, rank=-1):
    h = C.c_void_p()
    _check(lib().oracle_recompress(f.h, eps, rank, C.byref(h)))
    return Factor(h.value)


class ClusterTree:
    def __init__(self, positions, lo, hi):
        P = np.asfortranarray(positions, dtype=np.float64)
        if P.ndim == 1:
            P = P.reshape(-1, 1, order="F")
        n, d = P.shape
        h = C.c_void_p()
        _check(lib().oracle_build_cluster_tree(_d(P), n, d, _d(_f64(lo)), _d(_f64(hi)),
                                               C.byref(h)))
        self.h = h
        L = lib()
        self.root = L.oracle_tree_root(h)
        self.nodes = []
        for v in range(L.oracle_tree_num_nodes(h)):
            l, r, k = C.c_int(), C.c_int(), C.c_int()
            L.oracle_tree_node(h, v, C.byref(l), C.byref(r), C.byref(k))
            idx = np.zeros(k.value, dtype=np.int32)
            L.oracle_tree_node_idx(h, v, idx.ctypes.data_as(_ip))
            self.nodes.append(dict(left=l.value, right=r.value, idx=idx.tolist()))
        self._n = n

    def depth(self):
        return lib().oracle_tree_depth(self.h)

    def leaf_order(self):
        out = np.zeros(self._n, dtype=np.int32)
        lib().oracle_tree_leaf_order(self.h, out.ctypes.data_as(_ip))
        return out.tolist()

    def __del__(self):
        try:
            lib().oracle_tree_free(self.h)
        except Exception:
            pass


class RecResult:
    def __init__(self, handle, n_nodes):
        self.factor = Factor(handle)
        self.node_rank = np.zeros(n_nodes, dtype=np.int32)
        self.node_depth = np.zeros(n_nodes, dtype=np.int32)
        lib().oracle_factor_meta(self.factor.h, None, self.node_rank.ctypes.data_as(_ip),
                                 self.node_depth.ctypes.data_as(_ip), None)
        self.row_perm = self.factor.row_perm
        self.ledger = self.factor.ledger


def recursive_lowrank(tree, eps, H, rows_per, seed=0, p=20, kprobe=10):
    H = np.asfortranarray(H, dtype=np.float64)
    M, N = H.shape
    h = C.c_void_p()
    _check(lib().oracle_recursive_lowrank(tree.h, eps, _d(H), M, N, M, rows_per,
                                          C.c_uint64(seed & (2**64 - 1)), p, kprobe,
                                          C.byref(h)))
    return RecResult(h.value, len(tree.nodes))


def recursive_lowrank_born(tree, eps, incident, adjoint, w, nu, seed=0, p=20, kprobe=10,
                           source_ids=None, node_offset=0):
    """incident[s]: N x nl; adjoint[s][d]: N x nl (F-order arrays).  source_ids /
    node_offset: sharded replay (global seeds and row ids)."""
    ns = len(incident)
    nd = len(adjoint[0])
    N, nl = incident[0].shape
    inc = [np.asfortranarray(a, dtype=np.float64) for a in incident]
    adj = [np.asfortranarray(a, dtype=np.float64) for s in range(ns) for a in adjoint[s]]
    ia = (_dp * ns)(*[_d(a) for a in inc])
    aa = (_dp * len(adj))(*[_d(a) for a in adj])
    h = C.c_void_p()
    sid = None
    if source_ids is not None:
        sid_arr = np.ascontiguousarray(source_ids, dtype=np.int32)
        sid = sid_arr.ctypes.data_as(_ip)
    _check(lib().oracle_recursive_lowrank_born(tree.h, eps, N, nl, nd, ia, aa, _d(_f64(w)), nu,
                                               C.c_uint64(seed & (2**64 - 1)), p, kprobe, sid,
                                               int(node_offset), C.byref(h)))
    return RecResult(h.value, len(tree.nodes))


def lr_matmat(f, X, trans=False):
    X = np.asfortranarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X.reshape(-1, 1, order="F")
    b = X.shape[1]
    out = np.empty((f.cols if trans else f.rows, b), order="F")
    _check(lib().oracle_lr_matmat(f.h, int(trans), b, _d(X), _d(out)))
    return out


def j_matmat(f, X, row_perm, eps_c, trans=False):
    """eps_c: nl x nc (F-order).  trans=0: X (N*nc) x b -> M x b."""
    eps_c = np.asfortranarray(eps_c, dtype=np.float64)
    nl, nc = eps_c.shape
    X = np.asfortranarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X.reshape(-1, 1, order="F")
    b = X.shape[1]
    rp = np.ascontiguousarray(row_perm, dtype=np.int32)
    out = np.empty((f.cols * nc if trans else f.rows, b), order="F")
    _check(lib().oracle_j_matmat(f.h, int(trans), b, rp.ctypes.data_as(_ip), _d(eps_c), nl, nc,
                                 _d(X), _d(out)))
    return out


def fast_thin_svd(A):
    A = np.asfortranarray(A, dtype=np.float64)
    m, n = A.shape
    k = min(m, n)
    U = np.empty((m, k), order="F")
    s = np.empty(k)
    V = np.empty((n, k), order="F")
    _check(lib().oracle_fast_thin_svd(_d(A), m, n, _d(U), _d(s), _d(V)))
    return U, s, V


# --------------------------------------------------------------- PaLS -----
# Restatement of proj/src/pals.cpp (pals_oracle.cpp).  `geom` is
# (nx, ny, nz, Lx, Ly, Lz) as grid::build_grid; `p` any object with
# alpha, beta (n_p), centers (n_p x 3), tau_level, eps_H, nu_norm.
_pals_ready = False


def _pals_lib():
    global _pals_ready
    L = lib()
    if not _pals_ready:
        L.oracle_pals_last_error.restype = C.c_char_p
        L.oracle_pals_scalar.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
        L.oracle_pals_eval.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_double, C.c_int, _dp, _dp, _dp, C.c_double, C.c_double,
                                       C.c_double, _dp]
        L.oracle_pals_solve_concentrations.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                                       _ip, _dp, _dp, _dp, _dp, C.c_int, C.c_int,
                                                       _dp, _ip]
        L.oracle_pals_lm_step.argtypes = [_dp, C.c_int64, C.c_int, _dp, C.c_double, _dp]
        L.oracle_pals_metrics.argtypes = [C.c_int64, _dp, _dp, C.c_double, _dp, _dp, _ip]
        L.oracle_pals_reconstruct.argtypes = (
            [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, _ip, C.c_int, C.c_int, C.c_int, C.c_double,
             C.c_double, C.c_double, _dp, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp, _dp, _dp,
             C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
             C.c_double, C.c_double, C.c_double, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int, _dp])
        _pals_ready = True
    return L


def _pcheck(rc):
    if rc != 0:
        msg = _pals_lib().oracle_pals_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


def pals_scalar(name, t, eps=1.0):
    which = {"wendland": 0, "wendland_deriv": 1, "smooth_heaviside": 2, "smooth_delta": 3}[name]
    out = C.c_double()
    _pcheck(_pals_lib().oracle_pals_scalar(which, float(t), float(eps), C.byref(out)))
    return out.value


def _pargs(p):
    a = _f64(p.alpha)
    b = _f64(p.beta)
    c = np.asfortranarray(p.centers, dtype=np.float64)
    return a, b, c


def pals_eval(which, geom, p):
    """which: 'level_set' | 'shape' | 'shape_jacobian' (N x 5 n_p, F-order)."""
    nx, ny, nz, Lx, Ly, Lz = geom
    N = nx * ny * nz
    a, b, c = _pargs(p)
    k = {"level_set": 0, "shape": 1, "shape_jacobian": 2}[which]
    out = np.zeros((N, 5 * len(a)) if k == 2 else N, order="F")
    _pcheck(_pals_lib().oracle_pals_eval(k, nx, ny, nz, Lx, Ly, Lz, len(a), _d(a), _d(b), _d(c),
                                         p.tau_level, p.eps_H, p.nu_norm, _d(out)))
    return out


def _hop_args(U, V, perm):
    U = np.asfortranarray(U, dtype=np.float64)
    V = np.asfortranarray(V, dtype=np.float64)
    pp = None if perm is None else np.ascontiguousarray(perm, dtype=np.int32)
    return U, V, pp


def pals_solve_concentrations(U, V, perm, mu, w, y, ext):
    """ext: n_lambda x n_species extinction at the setup wavelengths."""
    U, V, pp = _hop_args(U, V, perm)
    ext = np.asfortranarray(ext, dtype=np.float64)
    nl, nsp = ext.shape
    c = np.zeros(nsp)
    fl = C.c_int()
    _pcheck(_pals_lib().oracle_pals_solve_concentrations(
        _d(U), _d(V), U.shape[0], V.shape[0], U.shape[1],
        None if pp is None else pp.ctypes.data_as(_ip), _d(_f64(mu)), _d(_f64(w)), _d(_f64(y)),
        _d(ext), nl, nsp, _d(c), C.byref(fl)))
    return c, bool(fl.value)


def pals_lm_step(J, eps, nu):
    J = np.asfortranarray(J, dtype=np.float64)
    dp = np.zeros(J.shape[1])
    _pcheck(_pals_lib().oracle_pals_lm_step(_d(J), J.shape[0], J.shape[1], _d(_f64(eps)), nu,
                                            _d(dp)))
    return dp


def pals_metrics(a, b, threshold=0.5):
    l2, dice, fl = C.c_double(), C.c_double(), C.c_int()
    a, b = _f64(a), _f64(b)
    _pcheck(_pals_lib().oracle_pals_metrics(len(a), _d(a), _d(b), threshold, C.byref(l2),
                                            C.byref(dice), C.byref(fl)))
    return l2.value, dice.value, bool(fl.value)


def pals_reconstruct(U, V, perm, geom, ext, y, w, init, noise_norm, max_outer=30, max_inner=5,
                     max_retries=8, gamma=1.2, nu0=1.0, stagnation_tol=1e-6, fixed_c=None,
                     mu_truth=None, trace_cap=4096):
    """Returns dict(alpha, beta, centers, c, trace (rows x 6), resnorm, converged, flagged)."""
    U, V, pp = _hop_args(U, V, perm)
    nx, ny, nz, Lx, Ly, Lz = geom
    ext = np.asfortranarray(ext, dtype=np.float64)
    nl, nsp = ext.shape
    a, b, c = _pargs(init)
    n = len(a)
    ao, bo, co = np.zeros(n), np.zeros(n), np.zeros((n, 3), order="F")
    cc = np.zeros(nsp)
    tr = np.zeros((trace_cap, 6))
    sc = np.zeros(4)
    fc = None if fixed_c is None else _d(_f64(fixed_c))
    mt = None if mu_truth is None else _d(_f64(mu_truth))
    _pcheck(_pals_lib().oracle_pals_reconstruct(
        _d(U), _d(V), U.shape[0], V.shape[0], U.shape[1],
        None if pp is None else pp.ctypes.data_as(_ip), nx, ny, nz, Lx, Ly, Lz, _d(ext), nl, nsp,
        _d(_f64(y)), _d(_f64(w)), n, _d(a), _d(b), _d(c), init.tau_level, init.eps_H,
        init.nu_norm, noise_norm, max_outer, max_inner, max_retries, gamma, nu0, stagnation_tol,
        fc, mt, _d(ao), _d(bo), _d(co), _d(cc), _d(tr), trace_cap, _d(sc)))
    ln = int(sc[3])
    return dict(alpha=ao, beta=bo, centers=co, c=cc, trace=tr[:min(ln, trace_cap)].copy(),
                resnorm=sc[0], converged=bool(sc[1]), flagged=bool(sc[2]))


# --------------------------------------------------------------- FEM -----
# The reference's own field operator (fem_oracle.cpp; grid.cpp:12-174).
_fem_ready = False


def _fem_lib():
    global _fem_ready
    L = lib()
    if not _fem_ready:
        L.oracle_fem_last_error.restype = C.c_char_p
        g6 = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
        L.oracle_fem_element.argtypes = [C.c_double, C.c_double, C.c_double, _dp, _dp, _dp]
        L.oracle_fem_apply.argtypes = g6 + [C.c_double, C.c_double, _dp, _dp]
        L.oracle_fem_dense.argtypes = g6 + [C.c_double, C.c_double, _dp]
        L.oracle_fem_point_source.argtypes = g6 + [_dp, _dp]
        L.oracle_fem_fields.argtypes = g6 + [C.c_int, _dp, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int,
                                             C.c_int, C.c_int, _dp, _ip, _dp]
        _fem_ready = True
    return L


def _fcheck(rc):
    if rc != 0:
        msg = _fem_lib().oracle_fem_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


def fem_element(hx, hy, hz):
    Ke, Me, Re = np.zeros(64), np.zeros(64), np.zeros(16)
    _fcheck(_fem_lib().oracle_fem_element(hx, hy, hz, _d(Ke), _d(Me), _d(Re)))
    return Ke.reshape(8, 8), Me.reshape(8, 8), Re.reshape(4, 4)


def fem_apply(geom, sigma, sigmap, x):
    x = _f64(x)
    y = np.empty_like(x)
    _fcheck(_fem_lib().oracle_fem_apply(*geom, sigma, sigmap, _d(x), _d(y)))
    return y


def fem_dense(geom, sigma, sigmap):
    N = geom[0] * geom[1] * geom[2]
    A = np.zeros((N, N), order="F")
    _fcheck(_fem_lib().oracle_fem_dense(*geom, sigma, sigmap, _d(A)))
    return A


def fem_point_source(geom, r):
    N = geom[0] * geom[1] * geom[2]
    b = np.zeros(N)
    _fcheck(_fem_lib().oracle_fem_point_source(*geom, _d(_f64(r)), _d(b)))
    return b


def fem_fields(geom, sigma, sigmap, inv_D, points, tol=1e-10, max_iter=20000, fixed_iters=0, threads=1):
    """(N x (n*nl), F-order) fields, iterations, relative residuals."""
    N = geom[0] * geom[1] * geom[2]
    nl = len(sigma)
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    out = np.empty((N, len(pts) * nl), order="F")
    iters = np.zeros(len(pts) * nl, dtype=np.int32)
    rel = np.zeros(len(pts) * nl)
    _fcheck(_fem_lib().oracle_fem_fields(*geom, nl, _d(_f64(sigma)), _d(_f64(sigmap)), _d(_f64(inv_D)),
                                         _d(pts), len(pts), tol, max_iter, fixed_iters, threads, _d(out),
                                         iters.ctypes.data_as(_ip), _d(rel)))
    return out, iters, rel


# ------------------------------------------------------------- Krylov -----
# The reference's recycled shifted-family solver (krylov_oracle.cpp;
# krylov.cpp:21-463) on the FEM operator above.
_kry_ready = False


def _kry_lib():
    global _kry_ready
    L = lib()
    if not _kry_ready:
        g6 = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
        L.oracle_krylov_last_error.restype = C.c_char_p
        L.oracle_krylov_apply.argtypes = g6 + [C.c_double, C.c_int, C.c_double, C.c_double, _dp, _dp, _dp]
        L.oracle_krylov_multishift.argtypes = g6 + [C.c_double, _dp, C.c_int, _dp, C.c_int, C.c_double,
                                                    _dp, _dp, _dp, _dp, _ip]
        L.oracle_krylov_harmonic_ritz.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp, _ip]
        L.oracle_krylov_deflation.argtypes = g6 + [C.c_double, C.c_int, _dp, _dp, C.c_int, _dp, _dp, _dp,
                                                   _dp, _ip]
        L.oracle_krylov_shifted_dense.argtypes = [C.c_int64, C.c_int, _dp, _dp, _dp, C.c_double, C.c_double,
                                                  C.c_int, _dp, _dp, _ip]
        L.oracle_krylov_solve_family.argtypes = g6 + [_dp, C.c_int, _dp, _dp, _ip, C.c_double, _dp, _ip,
                                                      _ip, _dp, _ip, _dp, _ip]
        _kry_ready = True
    return L


def _kcheck(rc):
    if rc != 0:
        msg = _kry_lib().oracle_krylov_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


class SolverConfig:
    """krylov::SolverConfig (krylov.hpp:13-23), same defaults."""

    def __init__(self, arnoldi_steps=80, deflation_dim=10, restart=50, tol=1e-8, max_restarts=40,
                 center_shifts=True, jacobi=False, explicit_qr_update=False, threads=1):
        self.arnoldi_steps, self.deflation_dim, self.restart = arnoldi_steps, deflation_dim, restart
        self.tol, self.max_restarts, self.center_shifts = tol, max_restarts, center_shifts
        self.jacobi, self.explicit_qr_update, self.threads = jacobi, explicit_qr_update, threads

    def ints(self):
        return np.array([self.arnoldi_steps, self.deflation_dim, self.restart, self.max_restarts,
                         int(self.center_shifts), int(self.jacobi), int(self.explicit_qr_update),
                         self.threads], dtype=np.int32)


def krylov_apply(geom, sbar, x, sigma=0.0, sp=0.0, which=0):
    """TransformedFamily.apply(sigma, sp, x) (which=0) or Rs x (which=1); also M^-1/2."""
    x = _f64(x)
    y = np.empty_like(x)
    d = np.empty_like(x)
    _kcheck(_kry_lib().oracle_krylov_apply(*geom, sbar, which, sigma, sp, _d(x), _d(y), _d(d)))
    return y, d


def krylov_multishift(geom, sbar, b, sigmas, n, tol):
    """multishift_gmres on transform_family(sbar) with rhs M^-1/2 b:
    (X, relres, V (N x (s+1)), Tbar ((s+1) x s), breakdown)."""
    N = geom[0] * geom[1] * geom[2]
    sig = _f64(sigmas)
    X = np.zeros((N, len(sig)), order="F")
    rel = np.zeros(len(sig))
    V = np.zeros((N, n + 1), order="F")
    T = np.zeros((n + 1, n), order="F")
    info = np.zeros(2, dtype=np.int32)
    _kcheck(_kry_lib().oracle_krylov_multishift(*geom, sbar, _d(_f64(b)), len(sig), _d(sig), n, tol, _d(X),
                                                _d(rel), _d(V), _d(T), info.ctypes.data_as(_ip)))
    s = int(info[0])
    return X, rel, V[:, :s + 1].copy(order="F"), T[:s + 1, :s].copy(order="F"), bool(info[1])


def krylov_harmonic_ritz(T, k):
    T = np.asfortranarray(T, dtype=np.float64)
    n = T.shape[1]
    Z = np.zeros((n, k), order="F")
    th = np.zeros(k)
    info = np.zeros(1, dtype=np.int32)
    _kcheck(_kry_lib().oracle_krylov_harmonic_ritz(n, _d(T), k, _d(Z), _d(th), info.ctypes.data_as(_ip)))
    return Z, th, bool(info[0])


def krylov_deflation(geom, sbar, V, T, Z):
    """build_deflation_basis: (U, C, RU, rank_reduced)."""
    V = np.asfortranarray(V, dtype=np.float64)
    T = np.asfortranarray(T, dtype=np.float64)
    Z = np.asfortranarray(Z, dtype=np.float64)
    N, s, k = V.shape[0], T.shape[1], Z.shape[1]
    U, Cm, RU = (np.zeros((N, k), order="F") for _ in range(3))
    info = np.zeros(2, dtype=np.int32)
    _kcheck(_kry_lib().oracle_krylov_deflation(*geom, sbar, s, _d(V), _d(T), k, _d(Z), _d(U), _d(Cm), _d(RU),
                                               info.ctypes.data_as(_ip)))
    ko = int(info[0])
    return U[:, :ko].copy(order="F"), Cm[:, :ko].copy(order="F"), RU[:, :ko].copy(order="F"), bool(info[1])


def krylov_shifted_dense(U, Cm, RU, sigma, sp, force_qr=False):
    """ShiftedDeflation(U, C, RU; sigma, sp): dense (C_j, U_j, cholesky_failed)."""
    U, Cm, RU = (np.asfortranarray(a, dtype=np.float64) for a in (U, Cm, RU))
    N, k = U.shape
    Cj, Uj = np.zeros((N, k), order="F"), np.zeros((N, k), order="F")
    info = np.zeros(1, dtype=np.int32)
    _kcheck(_kry_lib().oracle_krylov_shifted_dense(N, k, _d(U), _d(Cm), _d(RU), sigma, sp, int(force_qr),
                                                   _d(Cj), _d(Uj), info.ctypes.data_as(_ip)))
    return Cj, Uj, bool(info[0])


def krylov_solve_family(geom, b, shifts, cfg=None):
    """solve_family (krylov.cpp:400-463) for one rhs b (original variables):
    dict(X (N x nshift), iters, matvecs, relres, converged, phase1_relres,
    phase1_steps, defl_k, rank_reduced, pencil_shifted, breakdown,
    all_converged, first_failure)."""
    cfg = cfg or SolverConfig()
    N = geom[0] * geom[1] * geom[2]
    sh = np.asarray(shifts, dtype=np.float64).reshape(-1, 2)
    ns = len(sh)
    sig, sigp = np.ascontiguousarray(sh[:, 0]), np.ascontiguousarray(sh[:, 1])
    X = np.zeros((N, ns), order="F")
    it, mv, cv = (np.zeros(ns, dtype=np.int32) for _ in range(3))
    rel, p1 = np.zeros(ns), np.zeros(ns)
    info = np.zeros(7, dtype=np.int32)
    ci = cfg.ints()
    _kcheck(_kry_lib().oracle_krylov_solve_family(
        *geom, _d(_f64(b)), ns, _d(sig), _d(sigp), ci.ctypes.data_as(_ip), cfg.tol, _d(X),
        it.ctypes.data_as(_ip), mv.ctypes.data_as(_ip), _d(rel), cv.ctypes.data_as(_ip), _d(p1),
        info.ctypes.data_as(_ip)))
    return dict(X=X, iters=it, matvecs=mv, relres=rel, converged=cv.astype(bool), phase1_relres=p1,
                phase1_steps=int(info[0]), defl_k=int(info[1]), rank_reduced=bool(info[2]),
                pencil_shifted=bool(info[3]), breakdown=bool(info[4]), all_converged=bool(info[5]),
                first_failure=int(info[6]))
