"""Voxel-sharded top merges and products.

After the source-sharded phase (parallel.py: each rank compresses its own
subtree with no communication), the top log2(G) merges of the cluster tree
hold factors whose V (N x r) are far too tall to ship to one GPU at config
3 (N = 1e6, r in the thousands).  Here every rank keeps the rows of V of its
own voxel range [lo_g, hi_g) and the merges run cooperatively:

* randsvd of W = [V1^T; V2^T] (lowrank.cpp:131-199, 321-359):
  - sketch Y = W Omega = sum_g W_g Omega_g: a local GEMM on the rank's voxel
    rows of Omega (the same libstdc++ stream, column-major N x (rs + k),
    lowrank.cpp:136-143) and an all-reduce of the (r1 + r2) x (rs + k)
    partials; the SVD of Y, the probe error and every accept / double / Q = I
    decision are then computed identically on all ranks;
  - B^T = W^T Q stays voxel-sharded (no communication);
  - the tall QR of B^T is a TSQR: local Householder QR of the rank's rows,
    all-gather of the q x q R factors, QR of the stacked R's (replicated),
    so B^T = (Q_g Q2_g) R with the rank's rows of the orthonormal factor
    formed locally; the core SVD of R is split by rows over the ranks
    (svd_dist: one-sided block Jacobi with one pair-Gram all-reduce per
    round);
  - U = blkdiag(U1, U2) inner.U is small and replicated.
* recompress (lowrank.cpp:547-587): QR(U) replicated, QR(V) by TSQR, core
  SVD split by rows (svd_dist), V rows formed locally.
* J~x / J~^T y (lowrank.cpp:589-599, experiments.cpp:255-262): Z = sum_g V_g^T
  X_g is an all-reduce of R x (b N_c) (the north_star's "r-length
  allreduce of V^T x"); J~^T y needs no communication (U replicated).

Collectives: all-reduce and all-gather only.  `Comm` sums all-reduce
contributions in rank order (all-gather + ordered sum), so a run over G
processes is bit-identical to the same schedule replayed in one process
(SimComm); NCCL's all_reduce can be selected for speed (ordered=False).

Compute goes through an ops object: `NumpyOps` (LAPACK through numpy, the
libstdc++ stream from the oracle -- test infrastructure) or `DeviceOps`
(the CUDA library: DMMA GEMM, device Householder QR / thin SVD, device
Gaussian stream).
"""
from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch


def voxel_ranges(N: int, world: int):
    """Contiguous voxel row ranges, as equal as possible."""
    base, extra = divmod(N, world)
    out, lo = [], 0
    for g in range(world):
        hi = lo + base + (1 if g < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


# ------------------------------------------------------------ collectives --
class Comm:
    """torch.distributed collectives over tensors of the ops' kind."""

    def __init__(self, dist, ordered: bool = True):
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.ordered = ordered

    def allreduce(self, x: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return x
        if not self.ordered:
            y = x.clone()
            self.dist.all_reduce(y)
            return y
        parts = [torch.empty_like(x) for _ in range(self.world)]
        self.dist.all_gather(parts, x.contiguous())
        out = parts[0].clone()
        for p in parts[1:]:
            out += p
        return out

    def allgather(self, x: torch.Tensor) -> List[torch.Tensor]:
        if self.world == 1:
            return [x]
        parts = [torch.empty_like(x) for _ in range(self.world)]
        self.dist.all_gather(parts, x.contiguous())
        return parts

    def allgather_rows(self, x: torch.Tensor, ranges) -> List[torch.Tensor]:
        """all-gather of row blocks of different heights (ranges[g] rows of
        rank g), padded to the largest"""
        width = max(b - a for a, b in ranges)
        pad = torch.zeros((width,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        pad[:x.shape[0]] = x
        parts = self.allgather(pad)
        return [p[:b - a] for p, (a, b) in zip(parts, ranges)]

    def alltoall(self, sends: List[torch.Tensor], shapes) -> List[torch.Tensor]:
        """sends[g] goes to rank g; returns the blocks received from every
        rank (shapes[g]); point-to-point, so it also runs on gloo."""
        out = [None] * self.world
        out[self.rank] = sends[self.rank].clone()
        reqs = []
        for g in range(self.world):
            if g == self.rank:
                continue
            out[g] = torch.empty(shapes[g], dtype=sends[g].dtype, device=sends[g].device)
            if self.rank < g:
                reqs.append(self.dist.isend(sends[g].contiguous(), g))
                reqs.append(self.dist.irecv(out[g], g))
            else:
                reqs.append(self.dist.irecv(out[g], g))
                reqs.append(self.dist.isend(sends[g].contiguous(), g))
        for r in reqs:
            r.wait()
        return out


class SimComm:
    """G virtual ranks on threads of one process (the sequential replay):
    all-reduce sums in rank order, exactly like Comm(ordered=True)."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared: "SimComm._Shared", rank: int):
        self.sh, self.rank, self.world = shared, rank, shared.world

    @classmethod
    def group(cls, world):
        sh = cls._Shared(world)
        return [cls(sh, g) for g in range(world)]

    def _exchange(self, x):
        self.sh.slots[self.rank] = x.clone()
        self.sh.barrier.wait()
        parts = [p.clone() for p in self.sh.slots]
        self.sh.barrier.wait()
        return parts

    def allreduce(self, x):
        parts = self._exchange(x)
        out = parts[0].clone()
        for p in parts[1:]:
            out += p
        return out

    def allgather(self, x):
        return self._exchange(x)

    def allgather_rows(self, x, ranges):
        return self._exchange(x)

    def alltoall(self, sends, shapes):
        self.sh.slots[self.rank] = [t.clone() for t in sends]
        self.sh.barrier.wait()
        out = [self.sh.slots[g][self.rank].clone() for g in range(self.world)]
        self.sh.barrier.wait()
        return out


class LibComm:
    """The library's own NCCL communicator (hydot_comm, include/hydot_b200.h)
    for a context, bootstrapped over torch.distributed: rank 0 draws the NCCL
    unique id, every rank receives it by broadcast.  Its all-reduce runs on
    the context's stream."""

    def __init__(self, ctx, dist=None):
        import ctypes as C
        from ._lib import check, lib
        self.ctx = ctx
        self.world = dist.get_world_size() if dist is not None else 1
        self.rank = dist.get_rank() if dist is not None else 0
        idb = (C.c_ubyte * 128)()
        if self.world > 1:
            if self.rank == 0:
                check(lib().hydot_comm_unique_id(idb))
            t = torch.tensor(list(bytes(idb)), dtype=torch.uint8,
                             device=f"cuda:{ctx.device}" if dist.get_backend() == "nccl" else "cpu")
            dist.broadcast(t, 0)
            idb = (C.c_ubyte * 128)(*t.cpu().tolist())
        self.h = C.c_void_p()
        check(lib().hydot_comm_create(ctx.h, self.world, self.rank, idb, C.byref(self.h)), ctx.h)

    def allreduce(self, x: torch.Tensor) -> torch.Tensor:
        from ._lib import check, lib
        from .core import dptr
        y = x.contiguous().clone()
        check(lib().hydot_comm_allreduce(self.ctx.h, self.h, dptr(y), y.numel()), self.ctx.h)
        return y

    def __del__(self):
        try:
            from ._lib import lib
            if self.h:
                lib().hydot_comm_destroy(self.h)
        except Exception:
            pass


def j_matmat_voxel_lib(comm: LibComm, U, V_loc, row_perm_dev, eps_c_dev, nl, nc, X, trans=False):
    """hydot_j_matmat_voxel: column-major device buffers as in JOperator;
    X (b, Nloc*nc) storage for trans=False (returns (b, M)), X (b, M) for
    trans=True (returns (b, Nloc*nc))."""
    from ._lib import check, lib
    from .core import dptr, iptr
    M, R = U.shape
    Nloc = V_loc.shape[0]
    Ucm, Vcm = U.T.contiguous(), V_loc.T.contiguous()
    b = X.shape[0]
    if not trans:
        Y = torch.empty((b, M), dtype=torch.float64, device=U.device)
        check(lib().hydot_j_matmat_voxel(comm.ctx.h, comm.h, 0, b, dptr(Ucm), M, dptr(Vcm), Nloc, R,
                                         iptr(row_perm_dev), dptr(eps_c_dev), nl, nc, dptr(X), Nloc * nc,
                                         dptr(Y), M), comm.ctx.h)
    else:
        Y = torch.empty((b, Nloc * nc), dtype=torch.float64, device=U.device)
        check(lib().hydot_j_matmat_voxel(comm.ctx.h, comm.h, 1, b, dptr(Ucm), M, dptr(Vcm), Nloc, R,
                                         iptr(row_perm_dev), dptr(eps_c_dev), nl, nc, dptr(X), M,
                                         dptr(Y), Nloc * nc), comm.ctx.h)
    return Y


# -------------------------------------------------------------- compute --
class NumpyOps:
    """LAPACK via numpy on CPU tensors; the libstdc++ normal stream from the
    oracle (test infrastructure only)."""

    def __init__(self, oracle):
        self.o = oracle
        self._cache = {}

    def tensor(self, a):
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64))

    def normals(self, seed, offset, count):
        key = seed
        have = self._cache.get(key)
        if have is None or have.size < offset + count:
            have = self.o.gaussian(seed, max(offset + count, 2 * (0 if have is None else have.size)))
            self._cache[key] = have
        return torch.as_tensor(have[offset:offset + count].copy())

    def mm(self, A, B):
        return A @ B

    def mtm(self, A, B):
        return A.T @ B

    def qr(self, A):
        """thin Householder QR: A = Q R (dgeqrf / HouseholderQR)."""
        Q, R = np.linalg.qr(A.numpy())
        return torch.as_tensor(Q), torch.as_tensor(R)

    def svd(self, A):
        """thin SVD, singular values descending (dgesdd / BDCSVD)."""
        U, s, Vt = np.linalg.svd(A.numpy(), full_matrices=False)
        return torch.as_tensor(U), s, torch.as_tensor(np.ascontiguousarray(Vt.T))


class DeviceOps:
    """The CUDA library's kernels on device tensors."""

    def __init__(self, ctx):
        from . import lowrank as lr
        from .core import gaussian
        self.ctx, self.lr, self._gauss = ctx, lr, gaussian
        self.dev = torch.device(f"cuda:{ctx.device}")

    def tensor(self, a):
        return torch.as_tensor(a, dtype=torch.float64, device=self.dev)

    def normals(self, seed, offset, count):
        return self._gauss(self.ctx, seed, offset, count)

    def mm(self, A, B):
        """A @ B on the DMMA GEMM (row-major tensors as column-major transposes)."""
        from .core import dgemm
        A, B = A.contiguous(), B.contiguous()
        m, k = A.shape
        n = B.shape[1]
        C = torch.empty((m, n), dtype=torch.float64, device=self.dev)
        if m and n:
            dgemm(self.ctx, False, False, n, m, k, 1.0, B, max(n, 1), A, max(k, 1), 0.0, C, max(n, 1))
        return C

    def mtm(self, A, B):
        """A^T @ B on the DMMA GEMM."""
        from .core import dgemm
        A, B = A.contiguous(), B.contiguous()
        k, m = A.shape
        n = B.shape[1]
        C = torch.empty((m, n), dtype=torch.float64, device=self.dev)
        if m and n:
            dgemm(self.ctx, False, True, n, m, k, 1.0, B, max(n, 1), A, max(m, 1), 0.0, C, max(n, 1))
        return C

    def qr(self, A):
        return self.lr.householder_qr(self.ctx, A)

    def svd(self, A):
        U, s, V = self.lr.thin_svd(self.ctx, A)
        return U, np.asarray(s), V


# -------------------------------------------------------- the algorithm --
@dataclass
class VFactor:
    """Low-rank factor with U replicated (rows x r) and the rank's voxel rows
    of V (N_g x r); V = V~ diag(s) like lowrank::LowRankFactor."""
    U: torch.Tensor
    V_loc: torch.Tensor
    cols: int
    flagged: bool = False

    @property
    def rank(self):
        return self.U.shape[1]


def _omega_rows(ops, seed, base, N, lo, hi, w):
    """Rows [lo, hi) of the column-major N x w Gaussian block starting at
    stream offset `base` (lowrank.cpp:136-143: G(i, j) = normal #(j N + i))."""
    cols = [ops.normals(seed, base + j * N + lo, hi - lo) for j in range(w)]
    return torch.stack(cols, dim=1)


def tsqr(ops, comm, B_loc):
    """B = [B_0; ...; B_{G-1}] (rows by rank) = Q R: returns the rank's rows of
    Q and the replicated R (Householder QR locally, QR of the stacked R's)."""
    if B_loc.shape[0] < B_loc.shape[1]:
        raise ValueError("tsqr: a rank holds fewer voxel rows than the factor has columns")
    Q1, R1 = ops.qr(B_loc)
    q = R1.shape[1]
    Rs = comm.allgather(R1.contiguous())
    Q2, R = ops.qr(torch.cat(Rs, dim=0))
    return ops.mm(Q1, Q2[comm.rank * q:(comm.rank + 1) * q].contiguous()), R


def _tournament(nb):
    """circle-method rounds of block pairs (nb even)"""
    p = list(range(nb))
    rounds = []
    for _ in range(nb - 1):
        rounds.append([(min(p[i], p[nb - 1 - i]), max(p[i], p[nb - 1 - i])) for i in range(nb // 2)])
        p = [p[0], p[-1]] + p[1:-1]
    return rounds


def svd_dist(ops, comm, R, bw=8, max_sweeps=60):
    """Thin SVD of the replicated square core R = Ur S Vr^T with the work
    split by rows over the ranks: one-sided block Jacobi (bjacobi.cu's
    scheme) on L = R^T, each rank holding rows [a_g, b_g) of L.  Per round,
    the pair Grams of all block pairs are one all-reduce (per x 2bw x 2bw);
    every rank then diagonalises the same Grams and rotates its own rows.
    Columns of L converge to Vr S; Ur = L^T (Vr S) S^-2 is one n x n
    all-reduce.  Replaces the replicated core SVD of the top merges (the term
    that capped the config-3 Amdahl estimate)."""
    n = R.shape[0]
    a, b = voxel_ranges(n, comm.world)[comm.rank]
    L0 = R.T[a:b].contiguous()
    L = L0.clone()
    nb = (n + bw - 1) // bw
    nbp = nb + (nb & 1)
    rounds = _tournament(nbp)
    tol = max(1e-15, (n ** 0.5) * 2.220446049250313e-16)

    def cols(blk):
        return list(range(blk * bw, min(n, (blk + 1) * bw)))

    for _sweep in range(max_sweeps):
        rotated = 0
        for rnd in rounds:
            pairs = [(cols(x) + cols(y)) for x, y in rnd if x < nb and y < nb and (cols(x) + cols(y))]
            if not pairs:
                continue
            w = max(len(c) for c in pairs)
            part = torch.zeros((len(pairs), w, w), dtype=L.dtype, device=L.device)
            for k, c in enumerate(pairs):
                Xp = L[:, c]
                part[k, :len(c), :len(c)] = ops.mtm(Xp, Xp)
            G = comm.allreduce(part)
            for k, c in enumerate(pairs):
                g = G[k, :len(c), :len(c)]
                d = torch.sqrt(torch.clamp(torch.diagonal(g), min=0.0))
                off = torch.abs(g) / torch.clamp(d[:, None] * d[None, :], min=1e-300)
                off.fill_diagonal_(0.0)
                if float(off.max()) <= 2.0 * tol:
                    continue
                Q, _, _ = ops.svd(g.contiguous())  # eigenvectors of the SPD pair Gram, descending
                L[:, c] = ops.mm(L[:, c].contiguous(), Q.contiguous())
                rotated += 1
        if rotated == 0:
            break
    s2 = comm.allreduce((L * L).sum(dim=0))
    sig = torch.sqrt(s2)
    order = torch.argsort(-sig, stable=True)
    L, sig = L[:, order], sig[order]
    Vr_loc = L / torch.where(sig > 0, sig, torch.ones_like(sig))
    Vr = torch.cat(comm.allgather_rows(Vr_loc, voxel_ranges(n, comm.world)), dim=0)
    inv2 = torch.where(sig > 1e-14 * sig[0], 1.0 / (sig * sig), torch.zeros_like(sig))
    Ur = comm.allreduce(ops.mtm(L0, L)) * inv2  # L^T (Vr S) S^-2
    return Ur, sig.cpu().numpy() if sig.is_cuda else sig.numpy(), Vr


def randsvd_voxel(ops, comm, Wt_loc, m, N, lo, hi, eps, p=20, kprobe=10, seed=0, r0=1):
    """randsvd(dense_op(W)) with W (m x N) held as the rank's rows of W^T
    (lowrank.cpp:131-199).  Returns VFactor (U m x keep replicated)."""
    nmax = min(m, N)
    if m == 0 or N == 0:
        return VFactor(ops.tensor(np.zeros((m, 0))), ops.tensor(np.zeros((hi - lo, 0))), N)
    r = int(np.clip(r0, 1, nmax))
    consumed = 0
    identity = False
    flagged = False
    Q = None
    while True:
        rs = min(r + p, nmax)
        if rs >= nmax and m <= N:  # :159-164, no RNG consumed
            identity = True
            break
        w = rs + kprobe
        Om = _omega_rows(ops, seed, consumed, N, lo, hi, w)
        consumed += N * w
        YP = comm.allreduce(ops.mtm(Wt_loc, Om))  # [Y | P], m x (rs + k)
        Uy, sy, _ = ops.svd(YP[:, :rs])      # fast_thin_svd(Y) (:165-170)
        qc = min(r, Uy.shape[1])
        Q = Uy[:, :qc]
        sigma_top = float(sy[0]) if len(sy) else 0.0
        P = YP[:, rs:]
        er = float(torch.linalg.norm(P - ops.mm(Q, ops.mtm(Q, P))))
        if er <= eps * sigma_top:  # :176
            break
        if r >= nmax:  # :177-180
            flagged = True
            break
        r = min(2 * r, nmax)  # :181
    Bt_loc = Wt_loc if identity else ops.mm(Wt_loc, Q)  # B^T = W^T Q, voxel rows
    # fast_thin_svd(B) with N >= 2 qc: the tall branch on B^T (:66-87)
    Qb_loc, R = tsqr(ops, comm, Bt_loc)
    # R = Ur S Vr^T  =>  B = Vr S (Qb Ur)^T; the core SVD split over the ranks
    Ur, s, Vr = svd_dist(ops, comm, R) if comm.world > 1 else ops.svd(R)
    s1 = float(s[0]) if len(s) else 0.0
    keep = int(sum(1 for x in s if x > eps * s1 and x > 0))  # :187-190
    Ub = Vr[:, :keep]
    U = Ub if identity else ops.mm(Q, Ub)  # :191
    sv = ops.tensor(np.asarray(s[:keep]))
    V_loc = ops.mm(Qb_loc, Ur[:, :keep]) * sv  # :192 (singular values folded into V)
    return VFactor(U, V_loc, N, flagged)


def agglomerate_voxel(ops, comm, f1: VFactor, f2: VFactor, lo, hi, eps, seed=0, rank_hint=-1, p=20,
                      kprobe=10) -> VFactor:
    """agglomerate (lowrank.cpp:321-359) on voxel-sharded V."""
    r1, r2 = f1.rank, f2.rank
    m1, m2 = f1.U.shape[0], f2.U.shape[0]
    N = f1.cols
    if r1 + r2 == 0:  # :333-337
        return VFactor(ops.tensor(np.zeros((m1 + m2, 0))), ops.tensor(np.zeros((hi - lo, 0))), N)
    Wt_loc = torch.cat([f1.V_loc, f2.V_loc], dim=1)
    inner = randsvd_voxel(ops, comm, Wt_loc, r1 + r2, N, lo, hi, eps, p, kprobe, seed,
                          max(r1, r2, rank_hint))
    U = torch.cat([ops.mm(f1.U, inner.U[:r1]), ops.mm(f2.U, inner.U[r1:])], dim=0)  # :349-356
    return VFactor(U, inner.V_loc, N, f1.flagged or f2.flagged or inner.flagged)


def recompress_voxel(ops, comm, f: VFactor, eps, rank=-1) -> VFactor:
    """recompress (lowrank.cpp:547-587) with V voxel-sharded."""
    r = f.rank
    if r == 0:
        return f
    Qu, Ru = ops.qr(f.U)
    Qv_loc, Rv = tsqr(ops, comm, f.V_loc)
    core = ops.mm(Ru, Rv.T.contiguous())
    Uc, s, Vc = svd_dist(ops, comm, core) if comm.world > 1 else ops.svd(core)
    s1 = float(s[0])
    keep = min(rank, len(s)) if rank >= 0 else int(sum(1 for x in s if x > eps * s1 and x > 0))
    sv = ops.tensor(np.asarray(s[:keep]))
    return VFactor(ops.mm(Qu, Uc[:, :keep]), ops.mm(Qv_loc, Vc[:, :keep]) * sv, f.cols, f.flagged)


def lr_matmat_voxel(ops, comm, f: VFactor, X_loc):
    """U (V^T X) with X's voxel rows local: the R x b all-reduce
    (lowrank.cpp:589-593)."""
    return ops.mm(f.U, comm.allreduce(ops.mtm(f.V_loc, X_loc)))


def lr_rmatmat_voxel(ops, f: VFactor, Y):
    """The rank's voxel rows of V (U^T Y) (lowrank.cpp:595-599): no
    communication with U replicated."""
    return ops.mm(f.V_loc, ops.mtm(f.U, Y))


def j_matmat_voxel(ops, comm, f: VFactor, row_perm, eps_c, X_loc_c: List[torch.Tensor]):
    """J~ X = P [E_1 U, ..., E_nc U] (V^T X_c) (experiments.cpp:255-262,
    born.cpp:118-127): X_loc_c[c] are the rank's voxel rows of chromophore
    block c (N_g x b); one all-reduce of R x (b n_c)."""
    nc = len(X_loc_c)
    b = X_loc_c[0].shape[1]
    Z = comm.allreduce(ops.mtm(f.V_loc, torch.cat(X_loc_c, dim=1)))  # R x (b nc)
    T = ops.mm(f.U, Z)
    M = f.U.shape[0]
    perm = torch.as_tensor(np.asarray(row_perm, dtype=np.int64), device=T.device)
    ec = torch.as_tensor(np.asarray(eps_c, dtype=np.float64), device=T.device)  # nl x nc
    lam = perm % ec.shape[0]
    Y = torch.zeros((M, b), dtype=T.dtype, device=T.device)
    tmp = torch.zeros((M, b), dtype=T.dtype, device=T.device)
    for c in range(nc):
        tmp += ec[lam, c][:, None] * T[:, c * b:(c + 1) * b]
    Y[perm] = tmp
    return Y


def reshard_voxels(comm, V_full: torch.Tensor, ranges) -> List[torch.Tensor]:
    """The one exchange before the voxel-sharded merges: every rank holds its
    subtree factor's full V (N x r_g); afterwards rank h holds rows
    [lo_h, hi_h) of every rank's V (a list over source ranks).  One
    all-to-all of ~N r_g / G rows per rank pair."""
    sends = [V_full[a:b].contiguous() for (a, b) in ranges]
    widths = comm.allgather(torch.tensor([V_full.shape[1]], dtype=torch.int64, device=V_full.device))
    lo, hi = ranges[comm.rank]
    shapes = [(hi - lo, int(w.item())) for w in widths]
    return comm.alltoall(sends, shapes)
