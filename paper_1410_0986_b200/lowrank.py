"""hydot::lowrank on the B200 (mirror of proj/include/hydot/lowrank.hpp).

Same names, argument meaning and errors as the reference (std::invalid_argument
-> ValueError, std::runtime_error -> HydotError); matrices are torch float64
CUDA tensors.  Factors stay in HBM (``LowRankFactor``) until ``.U`` / ``.V``
are read.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import torch

from . import _lib
from ._lib import Ledger, check, lib
from .core import Context, dptr, iptr

# lowrank::Method (lowrank.hpp:14-22)
NONE, RANDSVD, ACA_FULL, ACA_PARTIAL, AGGLOMERATE, RECURSIVE, RECOMPRESS = range(7)
# FlopCategory (lowrank.hpp:54)
LEAF, AGGLOMERATION, RECOMPRESS_CAT, OTHER = range(4)


class LowRankFactor:
    """LowRankFactor (lowrank.hpp:25-36): A ~= U V^T, singular values in V."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx = ctx
        self.h = handle
        r, c, k = C.c_int64(), C.c_int64(), C.c_int64()
        tol, meth, flag = C.c_double(), C.c_int(), C.c_int()
        check(lib().hydot_factor_info(self.h, C.byref(r), C.byref(c), C.byref(k), C.byref(tol),
                                      C.byref(meth), C.byref(flag)))
        self._rows, self._cols, self._rank = r.value, c.value, k.value
        self.tol, self.method, self.flagged = tol.value, meth.value, bool(flag.value)

    @classmethod
    def from_tensors(cls, ctx: Context, U: torch.Tensor, V: torch.Tensor, tol=0.0,
                     method=NONE, flagged=False):
        """U (rows x r), V (cols x r) CUDA or CPU float64 tensors."""
        rows, r = U.shape
        cols = V.shape[0]
        Uc = U.T.contiguous()  # column-major
        Vc = V.T.contiguous()
        h = C.c_void_p()
        host = 0 if Uc.is_cuda else 1
        if host:
            Uc = Uc.numpy()
            Vc = Vc.numpy()
            up = Uc.ctypes.data_as(C.POINTER(C.c_double))
            vp = Vc.ctypes.data_as(C.POINTER(C.c_double))
        else:
            up, vp = dptr(Uc), dptr(Vc)
        check(lib().hydot_factor_create(ctx.h, rows, cols, r, up, max(rows, 1), vp, max(cols, 1),
                                        host, tol, method, int(flagged), C.byref(h)), ctx.h)
        return cls(ctx, h)

    def rank(self):
        return self._rank

    def rows(self):
        return self._rows

    def cols(self):
        return self._cols

    def _download(self):
        U = self.ctx.empty(max(self._rank, 1), max(self._rows, 1))
        V = self.ctx.empty(max(self._rank, 1), max(self._cols, 1))
        if self._rank:
            check(lib().hydot_factor_download(self.ctx.h, self.h, dptr(U), dptr(V), 0), self.ctx.h)
        return U[: self._rank, : self._rows].T, V[: self._rank, : self._cols].T

    @property
    def U(self) -> torch.Tensor:
        return self._download()[0]

    @property
    def V(self) -> torch.Tensor:
        return self._download()[1]

    def device_ptrs(self):
        u, v = _lib._dp(), _lib._dp()
        check(lib().hydot_factor_device_ptrs(self.h, C.byref(u), C.byref(v)))
        return u, v

    def dense(self) -> torch.Tensor:
        U, V = self._download()
        return U @ V.T

    def __del__(self):
        try:
            if self.h is not None and self.h.value:
                lib().hydot_factor_free(self.h)
                self.h = None
        except Exception:
            pass


_CUDART = None


def _cudart():
    global _CUDART
    if _CUDART is None:
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                _CUDART = C.CDLL(name)
                break
            except OSError:
                continue
        if _CUDART is None:
            raise RuntimeError("libcudart not found")
        _CUDART.cudaMemcpy2D.restype = C.c_int
    return _CUDART


def _seed(s):
    return C.c_uint64(int(s) & (2**64 - 1))


def _f64cuda(ctx, A):
    if not isinstance(A, torch.Tensor):
        A = torch.as_tensor(np.ascontiguousarray(A, dtype=np.float64))
    return A.to(device=f"cuda:{ctx.device}", dtype=torch.float64).contiguous()


@dataclass
class LinOp:
    """LinOp (lowrank.hpp:56-63): rows, cols and the products mv (A x), rmv
    (A^T y) and, optionally, the block forms mm (A X) / rmm (A^T Y).  The
    callables take and return float64 CUDA tensors (vectors for mv / rmv,
    (cols x k) -> (rows x k) matrices for mm, the reverse for rmm) and must
    work on the current torch stream."""
    rows: int = 0
    cols: int = 0
    mv: Optional[Callable] = None
    rmv: Optional[Callable] = None
    mm: Optional[Callable] = None
    rmm: Optional[Callable] = None


def dense_op(A: torch.Tensor) -> LinOp:
    """dense_op (lowrank.cpp:111-120): the four products of a dense CUDA
    matrix as a LinOp.  randsvd also takes the tensor itself (the library's
    own DMMA products); this form is for code written against LinOp."""
    return LinOp(rows=A.shape[0], cols=A.shape[1], mv=lambda x: A @ x, rmv=lambda y: A.T @ y,
                 mm=lambda X: A @ X, rmm=lambda Y: A.T @ Y)


def _randsvd_linop(ctx, A: LinOp, eps, p, kprobe, seed, ledger, cat, r0):
    dev = torch.device(f"cuda:{ctx.device}")
    err: list = []

    def view(ptr, rows, k, ld):
        # column-major (rows x k, ld) device memory as a (k, ld) row-major tensor
        n = (k - 1) * ld + rows
        flat = _tensor_from_ptr(ptr, n, dev)
        return flat.as_strided((k, rows), (ld, 1))

    def run(fn, stream, body):
        try:
            # a NULL cudaStream_t (the legacy default stream) arrives as None
            ext = (torch.cuda.ExternalStream(stream, device=dev) if stream
                   else torch.cuda.default_stream(dev))
            with torch.cuda.stream(ext):
                body()
            return 0
        except Exception as e:  # reported through the status code
            err.append(e)
            return 1

    def mk_mv(fn, nin, nout):
        if fn is None:
            return _lib.MV_FN()

        def cb(user, x, y, stream):
            def body():
                out = fn(view(x, nin, 1, nin)[0])
                view(y, nout, 1, nout)[0].copy_(out.reshape(nout))
            return run(fn, stream, body)
        return _lib.MV_FN(cb)

    def mk_mm(fn, nin, nout):
        if fn is None:
            return _lib.MM_FN()

        def cb(user, k, X, ldx, Y, ldy, stream):
            def body():
                out = fn(view(X, nin, k, ldx).T)
                view(Y, nout, k, ldy).copy_(out.reshape(nout, k).T)
            return run(fn, stream, body)
        return _lib.MM_FN(cb)

    op = _lib.LinOp(A.rows, A.cols, mk_mv(A.mv, A.cols, A.rows), mk_mv(A.rmv, A.rows, A.cols),
                    mk_mm(A.mm, A.cols, A.rows), mk_mm(A.rmm, A.rows, A.cols), None)
    h = C.c_void_p()
    led = Ledger()
    st = lib().hydot_randsvd_linop(ctx.h, C.byref(op), eps, p, kprobe, _seed(seed), cat, r0,
                                   C.byref(h), C.byref(led))
    if err:
        raise err[0]
    check(st, ctx.h)
    if ledger is not None:
        for f in ("leaf", "agglomeration", "recompress", "other", "kernel_tally"):
            setattr(ledger, f, getattr(ledger, f) + getattr(led, f))
    return LowRankFactor(ctx, h)


def _tensor_from_ptr(ptr, n, dev):
    """n float64 values at device address ptr as a torch tensor (no copy)."""
    class _Mem:
        pass
    m = _Mem()
    m.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                  "version": 2}
    return torch.as_tensor(m, device=dev)


def randsvd(ctx: Context, A, eps: float, p: int = 20, kprobe: int = 10,
            seed: int = 0, ledger: Optional[Ledger] = None, cat: int = OTHER, r0: int = 1):
    """randsvd (lowrank.hpp:70-72, lowrank.cpp:131-199).  A: a LinOp
    (matrix-free: hydot_randsvd_linop), or an m x n tensor standing for
    dense_op(A) (row-major torch tensor; any device)."""
    if isinstance(A, LinOp):
        return _randsvd_linop(ctx, A, eps, p, kprobe, seed, ledger, cat, r0)
    A = _f64cuda(ctx, A)
    m, n = A.shape
    h = C.c_void_p()
    led = Ledger()
    check(lib().hydot_randsvd(ctx.h, m, n, dptr(A) if A.numel() else None, max(n, 1), eps, p,
                              kprobe, _seed(seed), cat, r0, C.byref(h), C.byref(led)), ctx.h)
    if ledger is not None:
        for f in ("leaf", "agglomeration", "recompress", "other", "kernel_tally"):
            setattr(ledger, f, getattr(ledger, f) + getattr(led, f))
    return LowRankFactor(ctx, h)


def agglomerate(ctx: Context, f1: LowRankFactor, f2: LowRankFactor, eps: float, seed: int = 0,
                ledger: Optional[Ledger] = None, rank_hint: int = -1, p: int = 20,
                kprobe: int = 10):
    """agglomerate (lowrank.hpp:98-100, lowrank.cpp:321-359)."""
    h = C.c_void_p()
    led = Ledger()
    check(lib().hydot_agglomerate(ctx.h, f1.h, f2.h, eps, _seed(seed), rank_hint, p, kprobe,
                                  C.byref(h), C.byref(led)), ctx.h)
    if ledger is not None:
        for f in ("leaf", "agglomeration", "recompress", "other", "kernel_tally"):
            setattr(ledger, f, getattr(ledger, f) + getattr(led, f))
    return LowRankFactor(ctx, h)


def tolerance_schedule(eps_d: float, L: int, N_r: int) -> float:
    """eps = eps_d / (2^{L/2} (L+1) sqrt(N_r)) (lowrank.cpp:540-545)."""
    out = C.c_double()
    check(lib().hydot_tolerance_schedule(eps_d, L, N_r, C.byref(out)))
    return out.value


class ClusterTree:
    """ClusterTree / build_cluster_tree (lowrank.hpp:103-119, lowrank.cpp:385-438)."""

    def __init__(self, positions, lo, hi):
        P = np.asfortranarray(positions, dtype=np.float64)
        if P.ndim == 1:
            P = P.reshape(-1, 1, order="F")
        n, d = P.shape
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        if lo.size != d or hi.size != d:
            raise ValueError("build_cluster_tree: box dimension")
        h = C.c_void_p()
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        check(lib().hydot_tree_build(dp(P), n, d, dp(lo), dp(hi), C.byref(h)))
        self.h = h
        self.n_sources = n
        self.dim = d
        self.positions = P
        L = lib()
        self.root = L.hydot_tree_root(h)
        self.nodes = []
        for v in range(L.hydot_tree_num_nodes(h)):
            l, r, k = C.c_int(), C.c_int(), C.c_int()
            check(L.hydot_tree_node(h, v, C.byref(l), C.byref(r), C.byref(k), None))
            idx = np.zeros(max(k.value, 1), dtype=np.int32)
            check(L.hydot_tree_node(h, v, None, None, None, idx.ctypes.data_as(C.POINTER(C.c_int))))
            self.nodes.append(dict(left=l.value, right=r.value, idx=idx[: k.value].tolist()))

    def depth(self) -> int:
        return lib().hydot_tree_depth(self.h)

    def node_box(self, v: int):
        """(lo, hi) bounding box of node v (ClusterTree::Node::lo / hi)."""
        d = self.dim
        lo, hi = np.zeros(d), np.zeros(d)
        check(lib().hydot_tree_node_box(self.h, v, lo.ctypes.data_as(C.POINTER(C.c_double)),
                                        hi.ctypes.data_as(C.POINTER(C.c_double))))
        return lo, hi

    def leaf_order(self) -> List[int]:
        out = np.zeros(self.n_sources, dtype=np.int32)
        check(lib().hydot_tree_leaf_order(self.h, out.ctypes.data_as(C.POINTER(C.c_int))))
        return out.tolist()

    def __del__(self):
        try:
            lib().hydot_tree_free(self.h)
        except Exception:
            pass


def build_cluster_tree(positions, lo, hi) -> ClusterTree:
    return ClusterTree(positions, lo, hi)


@dataclass
class RecursiveOptions:
    """RecursiveOptions (lowrank.hpp:128-131) + the reference's hard-coded
    p=20 / kprobe=10 (lowrank.cpp:344, 448)."""
    seed: int = 0
    p: int = 20
    kprobe: int = 10
    hint_mode: int = 0
    # sharded execution: global ids of the local sources / pre-order offset
    source_ids: Optional[List[int]] = None
    node_offset: int = 0


@dataclass
class RecursiveResult:
    factor: LowRankFactor
    source_order: List[int]
    row_perm: np.ndarray
    node_rank: np.ndarray
    node_depth: np.ndarray
    ledger: Ledger = field(default_factory=Ledger)


@dataclass
class BornFieldsProvider:
    """Device BlockProvider: Born blocks formed from resident fields
    (compress_H's provider, experiments.cpp:235-240, without a dense H).
    incident[s]: (nl, N) CUDA tensor (rows = wavelengths);
    adjoint[s][d]: (nl, N); w: (N,); nu."""
    incident: list
    adjoint: list
    w: torch.Tensor
    nu: float = 1.0
    # optional torch.cuda.Event per source: the engine's stream waits on it
    # before forming that source's blocks (stream the fields in meanwhile)
    ready_events: Optional[list] = None


def recursive_lowrank(ctx: Context, tree: ClusterTree, eps: float, provider,
                      opts: RecursiveOptions = RecursiveOptions()) -> RecursiveResult:
    """recursive_lowrank (lowrank.hpp:142-144, lowrank.cpp:459-521).

    provider: BornFieldsProvider, or a callable block(s) -> (rows_per x cols)
    CUDA tensor together with attributes rows_per_source / cols (a
    lowrank::BlockProvider)."""
    nn = len(tree.nodes)
    row_perm = None
    node_rank = np.zeros(nn, dtype=np.int32)
    node_depth = np.zeros(nn, dtype=np.int32)
    h = C.c_void_p()
    led = Ledger()
    keep = []
    sid = None
    if opts.source_ids is not None:
        sid_arr = np.ascontiguousarray(opts.source_ids, dtype=np.int32)
        keep.append(sid_arr)
        sid = sid_arr.ctypes.data_as(C.POINTER(C.c_int))
    o = _lib.RecOpts(int(opts.seed) & (2**64 - 1), opts.p, opts.kprobe, opts.hint_mode, sid,
                     int(opts.node_offset))
    n_global = (max(opts.source_ids) + 1) if opts.source_ids is not None else tree.n_sources
    if isinstance(provider, BornFieldsProvider):
        ns = len(provider.incident)
        nd = len(provider.adjoint[0])
        nl, N = provider.incident[0].shape
        inc = (_lib._dp * ns)(*[dptr(t) for t in provider.incident])
        adj = (_lib._dp * (ns * nd))(*[dptr(t) for s in range(ns) for t in provider.adjoint[s]])
        keep += [inc, adj]
        evs = None
        if provider.ready_events is not None:
            if len(provider.ready_events) != ns:
                raise ValueError("BornFieldsProvider: one ready event per source")
            evs = (C.c_void_p * ns)(*[C.c_void_p(e.cuda_event) for e in provider.ready_events])
            keep.append(evs)
        bf = _lib.BornFields(N, nl, ns, nd, inc, adj, dptr(provider.w), provider.nu,
                             None if evs is None else C.cast(evs, C.POINTER(C.c_void_p)))
        rows_per = nd * nl
        row_perm = np.zeros(tree.n_sources * rows_per, dtype=np.int32)
        rc = lib().hydot_recursive_lowrank(ctx.h, tree.h, eps, None, C.byref(bf), C.byref(o),
                                           C.byref(h), row_perm.ctypes.data_as(C.POINTER(C.c_int)),
                                           node_rank.ctypes.data_as(C.POINTER(C.c_int)),
                                           node_depth.ctypes.data_as(C.POINTER(C.c_int)),
                                           C.byref(led))
    else:
        rows_per, cols = provider.rows_per_source, provider.cols
        errors = []

        def cb(user, s, out, ld):
            try:
                src = _f64cuda(ctx, provider.block(s))
                if tuple(src.shape) != (rows_per, cols):
                    raise ValueError("BlockProvider: block has the wrong shape")
                torch.cuda.synchronize(ctx.device)
                rc = _cudart().cudaMemcpy2D(C.c_void_p(C.cast(out, C.c_void_p).value),
                                            C.c_size_t(ld * 8), C.c_void_p(src.data_ptr()),
                                            C.c_size_t(cols * 8), C.c_size_t(cols * 8),
                                            C.c_size_t(rows_per), 3)
                return 0 if int(rc) == 0 else 1
            except Exception as e:  # surfaced as runtime_error by the library
                errors.append(e)
                return 1

        fn = _lib.BLOCK_FN(cb)
        keep.append(fn)
        pv = _lib.Provider(rows_per, cols, fn, None)
        row_perm = np.zeros(tree.n_sources * rows_per, dtype=np.int32)
        rc = lib().hydot_recursive_lowrank(ctx.h, tree.h, eps, C.byref(pv), None, C.byref(o),
                                           C.byref(h), row_perm.ctypes.data_as(C.POINTER(C.c_int)),
                                           node_rank.ctypes.data_as(C.POINTER(C.c_int)),
                                           node_depth.ctypes.data_as(C.POINTER(C.c_int)),
                                           C.byref(led))
        if rc != 0 and errors:
            raise errors[0]
    check(rc, ctx.h)
    return RecursiveResult(LowRankFactor(ctx, h), tree.leaf_order(), row_perm, node_rank,
                           node_depth, led)


def recompress(ctx: Context, f: LowRankFactor, eps: float, rank: int = -1,
               ledger: Optional[Ledger] = None) -> LowRankFactor:
    """recompress (lowrank.hpp:157-158, lowrank.cpp:547-587)."""
    h = C.c_void_p()
    led = Ledger()
    check(lib().hydot_recompress(ctx.h, f.h, eps, rank, C.byref(h), C.byref(led)), ctx.h)
    if ledger is not None:
        for fld in ("leaf", "agglomeration", "recompress", "other", "kernel_tally"):
            setattr(ledger, fld, getattr(ledger, fld) + getattr(led, fld))
    return LowRankFactor(ctx, h)


def _matmat(ctx, f, X, trans):
    X = _f64cuda(ctx, X)
    vec = X.dim() == 1
    Xc = X.reshape(-1, 1) if vec else X
    b = Xc.shape[1]
    rows_in = f.rows() if trans else f.cols()
    rows_out = f.cols() if trans else f.rows()
    if Xc.shape[0] != rows_in:
        raise ValueError("lr_rmatvec: dimension mismatch" if trans else "lr_matvec: dimension mismatch")
    Xcm = Xc.T.contiguous()  # column-major
    Y = ctx.empty(b, rows_out)
    check(lib().hydot_lr_matmat(ctx.h, f.h, int(trans), b, dptr(Xcm), rows_in, dptr(Y), rows_out),
          ctx.h)
    Y = Y.T
    return Y.reshape(-1) if vec else Y


def lr_matvec(ctx: Context, f: LowRankFactor, x) -> torch.Tensor:
    """U (V^T x) (lowrank.cpp:589-593); x may be N or N x b."""
    return _matmat(ctx, f, x, False)


def lr_rmatvec(ctx: Context, f: LowRankFactor, y) -> torch.Tensor:
    """V (U^T y) (lowrank.cpp:595-599)."""
    return _matmat(ctx, f, y, True)


class JOperator:
    """J~ = [E_1 H~, ..., E_nc H~] with the measurement permutation
    (permuted_matvec, experiments.cpp:255-262) and chromophore scaling
    (forward_measure, born.cpp:118-127).  Column-major device buffers:
    X (N*nc, b) for matvec, Y (M, b) for rmatvec."""

    def __init__(self, ctx: Context, f: LowRankFactor, row_perm, eps_c):
        self.ctx, self.f = ctx, f
        self.row_perm = torch.as_tensor(np.ascontiguousarray(row_perm, dtype=np.int32)).to(
            f"cuda:{ctx.device}")
        e = np.asfortranarray(eps_c, dtype=np.float64)  # nl x nc
        self.nl, self.nc = e.shape
        self.eps_c = torch.as_tensor(e.T.copy()).reshape(-1).to(f"cuda:{ctx.device}")
        self.M, self.N = f.rows(), f.cols()

    def matmat_cm(self, Xcm: torch.Tensor, Ycm: torch.Tensor, b: int):
        """column-major raw form: Xcm (b, N*nc) storage, Ycm (b, M) storage"""
        check(lib().hydot_j_matmat(self.ctx.h, self.f.h, 0, b, iptr(self.row_perm), dptr(self.eps_c),
                                   self.nl, self.nc, dptr(Xcm), self.N * self.nc, dptr(Ycm), self.M),
              self.ctx.h)

    def rmatmat_cm(self, Ycm: torch.Tensor, Xcm: torch.Tensor, b: int):
        check(lib().hydot_j_matmat(self.ctx.h, self.f.h, 1, b, iptr(self.row_perm), dptr(self.eps_c),
                                   self.nl, self.nc, dptr(Ycm), self.M, dptr(Xcm), self.N * self.nc),
              self.ctx.h)

    def matvec(self, X: torch.Tensor) -> torch.Tensor:
        X = _f64cuda(self.ctx, X)
        vec = X.dim() == 1
        Xc = (X.reshape(-1, 1) if vec else X).T.contiguous()
        b = Xc.shape[0]
        Y = self.ctx.empty(b, self.M)
        self.matmat_cm(Xc, Y, b)
        return Y.T.reshape(-1) if vec else Y.T

    def rmatvec(self, Y: torch.Tensor) -> torch.Tensor:
        Y = _f64cuda(self.ctx, Y)
        vec = Y.dim() == 1
        Yc = (Y.reshape(-1, 1) if vec else Y).T.contiguous()
        b = Yc.shape[0]
        X = self.ctx.empty(b, self.N * self.nc)
        self.rmatmat_cm(Yc, X, b)
        return X.T.reshape(-1) if vec else X.T


def thin_svd(ctx: Context, A: torch.Tensor):
    """fast_thin_svd (lowrank.cpp:62-93) on the device: returns U, s, V."""
    A = _f64cuda(ctx, A)
    m, n = A.shape
    k = min(m, n)
    Acm = A.T.contiguous()
    U = ctx.empty(max(k, 1), max(m, 1))
    V = ctx.empty(max(k, 1), max(n, 1))
    s = np.zeros(max(k, 1))
    check(lib().hydot_thin_svd(ctx.h, m, n, dptr(Acm), max(m, 1), dptr(U), s.ctypes.data_as(
        C.POINTER(C.c_double)), dptr(V)), ctx.h)
    return U[:k, :m].T, s[:k], V[:k, :n].T


def householder_qr(ctx: Context, A: torch.Tensor):
    A = _f64cuda(ctx, A)
    m, n = A.shape
    Acm = A.T.contiguous()
    R = ctx.empty(n, n)
    Q = ctx.empty(n, m)
    check(lib().hydot_householder_qr(ctx.h, m, n, dptr(Acm), m, dptr(R), dptr(Q)), ctx.h)
    return Q.T, R.T


def save_factor(path: str, f: LowRankFactor, row_perm=None) -> None:
    """save_factor (lowrank.hpp:165-166, lowrank.cpp:601-621): the reference's
    binary factor file, written from device memory."""
    perm = np.ascontiguousarray([] if row_perm is None else row_perm, dtype=np.int32)
    check(lib().hydot_factor_save(f.ctx.h, f.h, perm.ctypes.data_as(C.POINTER(C.c_int)),
                                  len(perm), os.fsencode(path)), f.ctx.h)


def load_factor(ctx: Context, path: str):
    """load_factor (lowrank.hpp:167, lowrank.cpp:623-655) into device memory:
    returns (LowRankFactor, row_perm int32 array)."""
    rows, cols, rank, plen = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().hydot_factor_file_info(os.fsencode(path), C.byref(rows), C.byref(cols),
                                       C.byref(rank), C.byref(plen)), None)
    perm = np.zeros(max(plen.value, 1), dtype=np.int32)
    h = C.c_void_p()
    check(lib().hydot_factor_load(ctx.h, os.fsencode(path), C.byref(h),
                                  perm.ctypes.data_as(C.POINTER(C.c_int)), len(perm)), ctx.h)
    return LowRankFactor(ctx, h), perm[:plen.value].copy()
