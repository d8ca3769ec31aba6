"""Parametric level-set (PaLS) reconstruction on the device -- the caller of
the compressed operator.

Mirrors proj/include/hydot/pals.hpp / src/pals.cpp: ``PaLSParams``
(to_vector / with_vector), ``level_set``, ``shape``, ``shape_jacobian``,
``solve_concentrations``, ``lm_step``, ``reconstruct``, ``metrics``,
``write_trace``.  The reference's ``Hmv`` closure is an ``HOperator``: a
device factor plus the factor's row permutation (experiments.cpp:255-262).
Everything N- or M-sized lives on the GPU; the kernels are in
csrc/pals.cu and the loop in csrc/pals_loop.cpp behind the C ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from ._lib import (GridGeom as _GridGeomC, Hop as _HopC, PalsParams as _ParamsC,
                   ReconConfig as _ReconConfigC, ReconResultC as _ResultC, TraceRowC, check, lib)
from .core import Context, dptr, iptr
from .lowrank import LowRankFactor, _f64cuda

_dp = C.POINTER(C.c_double)


@dataclass
class GridGeom:
    """grid::build_grid (grid.cpp:94-110): slab [-Lx,Lx] x [-Ly,Ly] x [0,Lz]."""
    nx: int
    ny: int
    nz: int
    Lx: float
    Ly: float
    Lz: float

    @property
    def hx(self):
        return 2 * self.Lx / (self.nx - 1)

    @property
    def hy(self):
        return 2 * self.Ly / (self.ny - 1)

    @property
    def hz(self):
        return self.Lz / (self.nz - 1)

    def num_vertices(self):
        return self.nx * self.ny * self.nz

    def vertex(self, n):  # grid.hpp:37-40
        ix, iy, iz = n % self.nx, (n // self.nx) % self.ny, n // (self.nx * self.ny)
        return np.array([-self.Lx + ix * self.hx, -self.Ly + iy * self.hy, iz * self.hz])

    def as_tuple(self):
        return (self.nx, self.ny, self.nz, self.Lx, self.Ly, self.Lz)

    def _c(self):
        return _GridGeomC(self.nx, self.ny, self.nz, self.Lx, self.Ly, self.Lz)

    @classmethod
    def for_grid7(cls, n: int, h: float):
        """The geometry of the config grids (configs.py): x = ix h - (n-1) h / 2, z = iz h."""
        L = (n - 1) * h / 2
        return cls(n, n, n, L, L, 2 * L)


def build_grid(nx, ny, nz, Lx, Ly, Lz) -> GridGeom:
    if nx < 2 or ny < 2 or nz < 2:
        raise ValueError("build_grid: vertex counts must be >= 2")
    if Lx <= 0 or Ly <= 0 or Lz <= 0:
        raise ValueError("build_grid: extents must be positive")
    return GridGeom(nx, ny, nz, Lx, Ly, Lz)


@dataclass
class PaLSParams:
    """PaLSParams (pals.hpp:16-32)."""
    alpha: np.ndarray
    beta: np.ndarray
    centers: np.ndarray  # n_p x 3
    tau_level: float = 0.1
    eps_H: float = 0.05
    nu_norm: float = 1e-3

    def __post_init__(self):
        self.alpha = np.asarray(self.alpha, dtype=np.float64).reshape(-1)
        self.beta = np.asarray(self.beta, dtype=np.float64).reshape(-1)
        self.centers = np.asarray(self.centers, dtype=np.float64).reshape(-1, 3)

    def np(self):
        return len(self.alpha)

    def num_params(self):
        return 5 * self.np()

    def to_vector(self):  # pals.cpp:14-23
        return np.concatenate([self.alpha, self.beta, self.centers[:, 0], self.centers[:, 1],
                               self.centers[:, 2]])

    def with_vector(self, v):  # pals.cpp:25-36
        n = self.np()
        v = np.asarray(v, dtype=np.float64)
        if v.shape != (5 * n,):
            raise ValueError("PaLSParams: parameter vector length")
        return PaLSParams(v[:n].copy(), np.maximum(v[n:2 * n], 1e-8),
                          np.stack([v[2 * n:3 * n], v[3 * n:4 * n], v[4 * n:]], axis=1),
                          self.tau_level, self.eps_H, self.nu_norm)

    def _c(self):
        self._keep = (np.ascontiguousarray(self.alpha), np.ascontiguousarray(self.beta),
                      np.asfortranarray(self.centers))
        a, b, c = self._keep
        return _ParamsC(self.np(), a.ctypes.data_as(_dp), b.ctypes.data_as(_dp),
                        c.ctypes.data_as(_dp), self.tau_level, self.eps_H, self.nu_norm)


class HOperator:
    """The reference's Hmv: y[row_perm[i]] = (U V^T x)[i] on the device."""

    def __init__(self, ctx: Context, factor: LowRankFactor, row_perm=None):
        self.ctx = ctx
        self.factor = factor
        self.perm = None
        if row_perm is not None:
            self.perm = torch.as_tensor(np.asarray(row_perm, dtype=np.int32)).to(
                f"cuda:{ctx.device}").contiguous()
        self._c = _HopC(factor.h, None if self.perm is None else iptr(self.perm))

    @property
    def M(self):
        return self.factor.rows()

    @property
    def N(self):
        return self.factor.cols()

    def matmat(self, X: torch.Tensor) -> torch.Tensor:
        """X: N or N x b (device) -> M or M x b."""
        X = _f64cuda(self.ctx, X)
        vec = X.dim() == 1
        Xc = X.reshape(-1, 1) if vec else X
        b = Xc.shape[1]
        Xcm = Xc.T.contiguous()
        Y = torch.empty((b, self.M), dtype=torch.float64, device=Xcm.device)
        check(lib().hydot_pals_hmv(self.ctx.h, C.byref(self._c), b, dptr(Xcm), self.N, dptr(Y),
                                   self.M), self.ctx.h)
        return Y[0] if vec else Y.T

    __call__ = matmat


def _eval(ctx, which, p: PaLSParams, g: GridGeom):
    N = g.num_vertices()
    cols = 5 * p.np() if which == 2 else 1
    out = torch.empty((cols, N), dtype=torch.float64, device=f"cuda:{ctx.device}")
    gc, pc = g._c(), p._c()
    check(lib().hydot_pals_eval(ctx.h, which, C.byref(gc), C.byref(pc), dptr(out), N), ctx.h)
    return out.T if which == 2 else out[0]


def level_set(ctx: Context, p: PaLSParams, g: GridGeom) -> torch.Tensor:
    """phi(r) = sum_k alpha_k psi(beta_k ||r - chi_k||_*) at every vertex (pals.cpp:74-86)."""
    return _eval(ctx, 0, p, g)


def shape(ctx: Context, p: PaLSParams, g: GridGeom) -> torch.Tensor:
    """mu_n = H_eps(phi_n - tau) (pals.cpp:88-94)."""
    return _eval(ctx, 1, p, g)


def shape_jacobian(ctx: Context, p: PaLSParams, g: GridGeom) -> torch.Tensor:
    """N x N_p analytic Jacobian [d/dalpha | d/dbeta | d/dcx | d/dcy | d/dcz] (pals.cpp:96-119)."""
    return _eval(ctx, 2, p, g)


@dataclass
class ConcentrationResult:
    c: List[float]
    flagged: bool = False


def solve_concentrations(ctx: Context, H: HOperator, mu, w, y, ext) -> ConcentrationResult:
    """c = (W D(p))^+ (W y) with D(p) columns E_i H mu (pals.cpp:139-156).
    ext: n_lambda x n_species extinction at the measurement wavelengths."""
    ext = np.asfortranarray(ext, dtype=np.float64)
    nl, nsp = ext.shape
    mu, w, y = (_f64cuda(ctx, t) for t in (mu, w, y))
    c = np.zeros(nsp)
    fl = C.c_int()
    check(lib().hydot_pals_solve_concentrations(ctx.h, C.byref(H._c), dptr(mu), dptr(w), dptr(y),
                                                ext.ctypes.data_as(_dp), nl, nsp,
                                                c.ctypes.data_as(_dp), C.byref(fl)), ctx.h)
    return ConcentrationResult(list(c), bool(fl.value))


def lm_step(ctx: Context, J, eps_residual, nu_damp: float) -> np.ndarray:
    """(J^T J + nu I) dp = -J^T eps via the stacked [J; sqrt(nu) I] system (pals.cpp:158-169)."""
    J = _f64cuda(ctx, J)
    M, n = J.shape
    Jc = J.T.contiguous()
    e = _f64cuda(ctx, eps_residual)
    dp = np.zeros(n)
    check(lib().hydot_pals_lm_step(ctx.h, M, n, dptr(Jc), M, dptr(e), float(nu_damp),
                                   dp.ctypes.data_as(_dp)), ctx.h)
    return dp


@dataclass
class Metrics:
    l2_rel: float = 0.0
    dice: float = 0.0
    flagged: bool = False


def metrics(ctx: Context, mu_true, mu_hat, threshold: float = 0.5) -> Metrics:
    """l2_rel and Dice overlap after binarisation (pals.cpp:307-329)."""
    a, b = _f64cuda(ctx, mu_true), _f64cuda(ctx, mu_hat)
    if a.numel() != b.numel():
        raise ValueError("metrics: length mismatch")
    l2, dice, fl = C.c_double(), C.c_double(), C.c_int()
    check(lib().hydot_pals_metrics(ctx.h, a.numel(), dptr(a), dptr(b), threshold, C.byref(l2),
                                   C.byref(dice), C.byref(fl)), ctx.h)
    return Metrics(l2.value, dice.value, bool(fl.value))


@dataclass
class ReconConfig:
    """ReconConfig (pals.hpp:67-75)."""
    max_outer: int = 30
    max_inner: int = 5
    max_retries: int = 8
    gamma: float = 1.2
    nu0: float = 1.0
    stagnation_tol: float = 1e-6
    fixed_c: List[float] = field(default_factory=list)
    # BASELINE config 4 knob: J~x / J~^T y normal-equation blocks per GN step
    normal_blocks: int = 0


@dataclass
class TraceRow:
    outer: int = 0
    inner: int = 0
    resnorm: float = 0.0
    nu: float = 0.0
    accepted: bool = False
    dice: float = -1.0


@dataclass
class ReconResult:
    p: PaLSParams
    c: List[float]
    trace: List[TraceRow]
    resnorm: float = 0.0
    converged: bool = False
    flagged: bool = False
    hmv_calls: int = 0
    hmv_columns: int = 0
    normal_columns: int = 0


def reconstruct(ctx: Context, y, H: HOperator, g: GridGeom, ext, init: PaLSParams, w_diag,
                noise_norm: float, cfg: Optional[ReconConfig] = None, mu_truth=None,
                trace_cap: int = 8192) -> ReconResult:
    """Alternating concentration / shape reconstruction with LM shape updates
    (pals.cpp:193-295); noise_norm = ||W eta|| for the discrepancy stop."""
    cfg = cfg or ReconConfig()
    if cfg.gamma <= 1.0:
        raise ValueError("reconstruct: gamma must exceed 1")
    ext = np.asfortranarray(ext, dtype=np.float64)
    nl, nsp = ext.shape
    y, w = _f64cuda(ctx, y), _f64cuda(ctx, w_diag)
    mt = None if mu_truth is None else _f64cuda(ctx, mu_truth)
    fixed = None
    if cfg.fixed_c:
        fixed = np.ascontiguousarray(cfg.fixed_c, dtype=np.float64)
    rc = _ReconConfigC(cfg.max_outer, cfg.max_inner, cfg.max_retries, cfg.gamma, cfg.nu0,
                       cfg.stagnation_tol, None if fixed is None else fixed.ctypes.data_as(_dp),
                       int(cfg.normal_blocks))
    n = init.np()
    ao, bo, co = np.zeros(n), np.zeros(n), np.zeros((n, 3), order="F")
    cc = np.zeros(max(nsp, 1))
    trace = (TraceRowC * trace_cap)()
    out = _ResultC()
    out.p = _ParamsC(n, ao.ctypes.data_as(_dp), bo.ctypes.data_as(_dp), co.ctypes.data_as(_dp),
                     0.0, 0.0, 0.0)
    out.c_h = cc.ctypes.data_as(_dp)
    out.trace_h = C.cast(trace, C.POINTER(TraceRowC))
    out.trace_cap = trace_cap
    gc, pc = g._c(), init._c()
    check(lib().hydot_pals_reconstruct(ctx.h, C.byref(H._c), C.byref(gc), ext.ctypes.data_as(_dp),
                                       nl, nsp, dptr(y), dptr(w), C.byref(pc), float(noise_norm),
                                       C.byref(rc), None if mt is None else dptr(mt),
                                       C.byref(out)), ctx.h)
    rows = [TraceRow(t.outer, t.inner, t.resnorm, t.nu, bool(t.accepted), t.dice)
            for t in trace[:min(out.trace_len, trace_cap)]]
    p = PaLSParams(ao, bo, np.ascontiguousarray(co), init.tau_level, init.eps_H, init.nu_norm)
    return ReconResult(p, list(cc[:nsp]), rows, out.resnorm, bool(out.converged),
                       bool(out.flagged), out.hmv_calls, out.hmv_columns, out.normal_columns)


def write_trace(path: str, trace: List[TraceRow]) -> None:
    """write_trace (pals.cpp:297-305)."""
    with open(path, "w") as f:
        f.write("outer_iter,inner_iter,resnorm,nu,accepted,dice_vs_truth\n")
        for r in trace:
            f.write(f"{r.outer},{r.inner},{r.resnorm:.12g},{r.nu:.12g},{int(r.accepted)},"
                    f"{r.dice:.12g}\n")
