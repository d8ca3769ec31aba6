"""krylov -- the reference's recycled shifted-family solver on the device.

Mirrors ``hydot::krylov`` (/root/reference/proj/include/hydot/krylov.hpp,
src/krylov.cpp:21-463) over the C ABI (``hydot_solve_family_fem``,
``hydot_fields_solve_fem_gmres``; csrc/gmres.cu).  The operator is the
reference's FEM family K + sigma_j M + sigma'_j R (grid.cpp:112-174), applied
matrix-free; torch tensors are only the HBM allocator.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .core import Context, dptr


@dataclass
class SolverConfig:
    """krylov::SolverConfig (krylov.hpp:13-23); ``threads`` has no device
    meaning (every shift of a batch is solved together) and is ignored."""
    arnoldi_steps: int = 80
    deflation_dim: int = 10
    restart: int = 50
    tol: float = 1e-8
    max_restarts: int = 40
    center_shifts: bool = True
    jacobi: bool = False
    explicit_qr_update: bool = False
    threads: int = 1

    def c(self) -> _lib.KrylovConfig:
        return _lib.KrylovConfig(self.arnoldi_steps, self.deflation_dim, self.restart, self.tol,
                                 self.max_restarts, int(self.center_shifts), int(self.jacobi),
                                 int(self.explicit_qr_update))


@dataclass
class IterationStats:
    """krylov::IterationStats (krylov.hpp:109-114) + the phase-1 residual."""
    iterations: int
    matvecs: int
    relres: float
    converged: bool
    phase1_relres: float


@dataclass
class FamilyResult:
    """krylov::FamilyResult (krylov.hpp:128-134) for one right-hand side."""
    X: torch.Tensor                      # (n_shifts, N), original variables
    stats: List[IterationStats]
    phase1_matvecs: int
    all_converged: bool
    first_failure: int
    deflation_k: int = 0
    rank_reduced: bool = False
    pencil_shifted: bool = False
    breakdown: bool = False
    cholesky_failed: int = 0
    extra: dict = field(default_factory=dict)


def _geom(geom) -> _lib.GridGeom:
    from .born import _geom_c
    return _geom_c(geom)


def _results(X, st, fam, nsh):
    out = []
    for r in range(len(fam)):
        f = fam[r]
        sts = [IterationStats(int(s.iterations), int(s.matvecs), float(s.relres), bool(s.converged),
                              float(s.phase1_relres)) for s in st[r * nsh:(r + 1) * nsh]]
        out.append(FamilyResult(X[r], sts, int(f.phase1_steps), bool(f.all_converged), int(f.first_failure),
                                int(f.deflation_k), bool(f.rank_reduced), bool(f.pencil_shifted),
                                bool(f.breakdown), int(f.cholesky_failed)))
    return out


def solve_family(ctx: Context, geom, b: torch.Tensor, shifts, cfg: SolverConfig | None = None):
    """solve_family(K, M, R, b, shifts, cfg) (krylov.cpp:400-463) for every
    row of ``b`` ((n_rhs, N) or (N,), device float64): a list of FamilyResult
    (one per rhs).  Unconverged systems are reported, as in the reference."""
    cfg = cfg or SolverConfig()
    g = _geom(geom)
    N = g.nx * g.ny * g.nz
    b2 = b.reshape(-1, N).contiguous()
    sh = np.ascontiguousarray(np.asarray(shifts, dtype=np.float64).reshape(-1, 2))
    nsh = len(sh)
    sig, sigp = np.ascontiguousarray(sh[:, 0]), np.ascontiguousarray(sh[:, 1])
    nr = b2.shape[0]
    X = ctx.empty(nr, nsh, N)
    st = (_lib.KrylovStats * (nr * nsh))()
    fam = (_lib.KrylovFamily * nr)()
    cc = cfg.c()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    check(lib().hydot_solve_family_fem(ctx.h, C.byref(g), nsh, dp(sig), dp(sigp), dptr(b2), nr, C.byref(cc),
                                       dptr(X), st, fam), ctx.h)
    return _results(X, st, fam, nsh)


def compute_fields_fem_gmres(ctx: Context, geom, sigma, sigma_prime, inv_D, points_xyz,
                             cfg: SolverConfig | None = None):
    """compute_fields (born.cpp:39-80) with the reference's solver on its FEM
    operator: (n, n_lambda, N) fields x_l / D_l and the per-rhs FamilyResults
    (their X is the same tensor's rows).  Raises HydotError when a system
    does not converge ("field solve failed at ...", born.cpp:58-61)."""
    cfg = cfg or SolverConfig()
    g = _geom(geom)
    N = g.nx * g.ny * g.nz
    sig = np.ascontiguousarray(sigma, dtype=np.float64)
    sigp = np.ascontiguousarray(sigma_prime, dtype=np.float64)
    invd = np.ascontiguousarray(inv_D, dtype=np.float64)
    pts = np.ascontiguousarray(points_xyz, dtype=np.float64).reshape(-1, 3)
    nl, npt = sig.size, len(pts)
    out = ctx.empty(npt, nl, N)
    st = (_lib.KrylovStats * (npt * nl))()
    fam = (_lib.KrylovFamily * npt)()
    cc = cfg.c()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    check(lib().hydot_fields_solve_fem_gmres(ctx.h, C.byref(g), nl, dp(sig), dp(sigp), dp(invd), dp(pts), npt,
                                             C.byref(cc), dptr(out), st, fam), ctx.h)
    return out, _results(out, st, fam, nl)
