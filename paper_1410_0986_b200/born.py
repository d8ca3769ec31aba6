"""hydot::born on the B200 (mirror of proj/include/hydot/born.hpp).

Fields come from the batched matrix-free 7-point CG (hydot_fields_solve);
Born blocks from the Hadamard kernel (hydot_born_block).  Device tensors are
row-major torch float64 tensors: a field set of one point is (n_lambda, N)
(each wavelength row voxel-contiguous, i.e. the reference's N x N_lambda
column-major Mat), a Born block is (n_det*n_lambda, N).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .core import Context, dptr


@dataclass
class Grid7:
    """Vertex grid, x-fastest (grid.hpp:22-28), spacing h; side faces
    Dirichlet, z faces Robin (grid.hpp:18-21)."""
    nx: int
    ny: int
    nz: int
    h: float

    @property
    def N(self) -> int:
        return self.nx * self.ny * self.nz

    def index(self, ix, iy, iz) -> int:
        return ix + self.nx * (iy + self.ny * iz)

    def c(self):
        return _lib.Grid7(self.nx, self.ny, self.nz, self.h)


@dataclass
class FieldStats:
    iters: np.ndarray
    relres: np.ndarray


def compute_fields(ctx: Context, grid: Grid7, sigma, sigma_prime, inv_D, points: Sequence[int],
                   tol: float = 1e-10, max_iter: int = 20000, fixed_iters: int = 0,
                   out: torch.Tensor = None):
    """Fields of unit point sources at vertex ids `points` for every
    wavelength: returns (len(points), n_lambda, N) = x_l / D_l with
    (K + sigma_l M + sigma'_l R) x_l = e_v (born.cpp:39-80, born.cpp:62-63).
    Raises HydotError when a system misses tol (born.cpp:58-61)."""
    sig = np.ascontiguousarray(sigma, dtype=np.float64)
    sigp = np.ascontiguousarray(sigma_prime, dtype=np.float64)
    invd = np.ascontiguousarray(inv_D, dtype=np.float64)
    nl = sig.size
    if nl == 0:
        raise ValueError("compute_fields: no wavelengths")
    pts = np.ascontiguousarray(points, dtype=np.int64)
    if out is None:
        out = ctx.empty(len(pts), nl, grid.N)
    iters = np.zeros(len(pts) * nl, dtype=np.int32)
    rel = np.zeros(len(pts) * nl, dtype=np.float64)
    g = grid.c()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    check(lib().hydot_fields_solve(ctx.h, C.byref(g), nl, dp(sig), dp(sigp), dp(invd),
                                   pts.ctypes.data_as(C.POINTER(C.c_int64)), len(pts), tol,
                                   max_iter, fixed_iters, dptr(out),
                                   iters.ctypes.data_as(C.POINTER(C.c_int)), dp(rel)), ctx.h)
    return out, FieldStats(iters.reshape(len(pts), nl), rel.reshape(len(pts), nl))


class StreamedFieldsProvider:
    """BlockProvider (lowrank.hpp:122-126) that solves the fields per source on
    demand -- the reference's per-source loop of compute_fields
    (born.cpp:39-80) fused with compress_H's provider (experiments.cpp:235-240):
    block(s) runs the batched CG for source s and its detectors, assembles
    the (N_ds N_lambda) x N Born block (born.cpp:82-98) and drops the fields,
    so only one source's fields are ever resident (config 3: 17.6 GB per
    source instead of 1.1 TB for all).

    source_point[s], detector_points[s] (vertex ids); `sources` maps the
    tree-local index the recursion passes to a global source id.  Records
    the CG time (CUDA events) and iteration counts per call in `log`."""

    def __init__(self, ctx: Context, grid: Grid7, sigma, sigma_prime, inv_D, source_vertex,
                 detector_vertices, w: torch.Tensor, nu: float = 1.0, tol: float = 1e-10,
                 sources=None):
        self.ctx, self.grid = ctx, grid
        self.sigma, self.sigma_prime, self.inv_D = sigma, sigma_prime, inv_D
        self.source_vertex = np.asarray(source_vertex, dtype=np.int64)
        self.detector_vertices = np.asarray(detector_vertices, dtype=np.int64)
        self.w, self.nu, self.tol = w, nu, tol
        self.sources = list(range(len(self.source_vertex))) if sources is None else list(sources)
        nd = self.detector_vertices.shape[1]
        self.rows_per_source = nd * len(np.atleast_1d(sigma))
        self.cols = grid.N
        self.log = []

    def block(self, s_local: int) -> torch.Tensor:
        s = self.sources[s_local]
        pts = [int(self.source_vertex[s])] + [int(v) for v in self.detector_vertices[s]]
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        F, st = compute_fields(self.ctx, self.grid, self.sigma, self.sigma_prime, self.inv_D, pts,
                               tol=self.tol)
        b.record()
        B = assemble_H_block(self.ctx, F[0], [F[1 + d] for d in range(len(pts) - 1)], self.w, self.nu)
        del F
        b.synchronize()
        self.log.append({"source": s, "cg_s": a.elapsed_time(b) / 1e3,
                         "iters_total": int(st.iters.sum()), "iters_max": int(st.iters.max()),
                         "relres_max": float(st.relres.max())})
        return B


@dataclass
class FullForward:
    """experiments::FullForward (experiments.hpp:39-45)."""
    y_total: torch.Tensor
    y_incident: torch.Tensor
    y_scattered: torch.Tensor
    iters_max: int


def full_diffusion_forward(ctx: Context, grid: Grid7, sigma, sigma_prime, inv_D, dsigma, mu: torch.Tensor,
                           source_vertex, detector_vertex, tol: float = 1e-10, max_iter: int = 20000,
                           fixed_iters: int = 0) -> FullForward:
    """full_diffusion_forward (experiments.cpp:154-206) on the device for the
    7-point operator: the perturbed medium sigma_l + dsigma_l mu(v) and the
    background, detector values (measurement (s, d, l) -> (s n_det + d)
    n_lambda + l).  dsigma_l = nu (sum_c c_pert_c eps_c(lambda_l)) / D_l."""
    sig = np.ascontiguousarray(sigma, dtype=np.float64)
    sigp = np.ascontiguousarray(sigma_prime, dtype=np.float64)
    invd = np.ascontiguousarray(inv_D, dtype=np.float64)
    dsg = np.ascontiguousarray(dsigma, dtype=np.float64)
    src = np.ascontiguousarray(source_vertex, dtype=np.int64)
    det = np.ascontiguousarray(detector_vertex, dtype=np.int64).reshape(len(src), -1)
    nl, ns, nd = sig.size, len(src), det.shape[1]
    if mu.numel() != grid.N:
        raise ValueError("full_forward: mu must hold one value per vertex")
    mu = mu.to(device=f"cuda:{ctx.device}", dtype=torch.float64).contiguous()
    yt = ctx.empty(ns * nd * nl)
    yi = ctx.empty(ns * nd * nl)
    it = C.c_int(0)
    g = grid.c()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    ip64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))
    check(lib().hydot_full_forward(ctx.h, C.byref(g), nl, dp(sig), dp(sigp), dp(invd), dp(dsg), dptr(mu),
                                   ip64(src), ns, ip64(det), nd, tol, max_iter, fixed_iters, dptr(yt), dptr(yi),
                                   C.byref(it)), ctx.h)
    return FullForward(yt, yi, yt - yi, it.value)


def apply_operator(ctx: Context, grid: Grid7, sigma: float, sigma_prime: float,
                   x: torch.Tensor) -> torch.Tensor:
    y = torch.empty_like(x)
    g = grid.c()
    check(lib().hydot_apply7(ctx.h, C.byref(g), sigma, sigma_prime, dptr(x), dptr(y)), ctx.h)
    return y


def assemble_H_block(ctx: Context, incident: torch.Tensor, adjoint: List[torch.Tensor],
                     lumped_w: torch.Tensor, nu: float = 1.0, out: torch.Tensor = None):
    """assemble_H_block (born.hpp:61-62, born.cpp:82-98): rows (d*nl + l) =
    (-nu) * phi_d[:, l] .* phi_s[:, l] .* w.  incident (nl, N), adjoint[d]
    (nl, N) CUDA tensors; returns (n_det*nl, N)."""
    nl, N = incident.shape
    nd = len(adjoint)
    if lumped_w.numel() != N:
        raise ValueError("assemble_H_block: weight size mismatch")
    for a in adjoint:
        if tuple(a.shape) != (nl, N):
            raise ValueError("assemble_H_block: adjoint field shape mismatch")
    if out is None:
        out = ctx.empty(nd * nl, N)
    arr = (_lib._dp * max(nd, 1))(*[dptr(a) for a in adjoint])
    check(lib().hydot_born_block(ctx.h, N, nl, dptr(incident.contiguous()), arr, nd,
                                 dptr(lumped_w.contiguous()), nu, dptr(out), out.stride(0)), ctx.h)
    return out


def assemble_H_dense(ctx: Context, incident: List[torch.Tensor], adjoint: List[List[torch.Tensor]],
                     lumped_w: torch.Tensor, nu: float = 1.0) -> torch.Tensor:
    """All blocks stacked in source order (born.cpp:100-108; fixture scale)."""
    nl, N = incident[0].shape
    nd = len(adjoint[0])
    H = ctx.empty(len(incident) * nd * nl, N)
    for s in range(len(incident)):
        assemble_H_block(ctx, incident[s], adjoint[s], lumped_w, nu,
                         out=H[s * nd * nl:(s + 1) * nd * nl])
    return H


def save_block(ctx: Context, path: str, block: torch.Tensor) -> None:
    """save_block (born.hpp:85, born.cpp:156-167) from a device block
    (rows, cols) -- the (n_det*n_lambda) x N layout of assemble_H_block."""
    if block.dim() != 2 or block.stride(1) != 1:
        raise ValueError("save_block: expected a row-major 2-D tensor")
    rows, cols = block.shape
    check(lib().hydot_block_save(ctx.h, dptr(block), rows, cols, block.stride(0),
                                 os.fsencode(path)), ctx.h)


def load_block(ctx: Context, path: str) -> torch.Tensor:
    """load_block (born.hpp:86, born.cpp:169-185) into device memory."""
    rows, cols = C.c_int64(), C.c_int64()
    check(lib().hydot_block_file_info(os.fsencode(path), C.byref(rows), C.byref(cols)), None)
    out = ctx.empty(max(rows.value, 1), max(cols.value, 1))[:rows.value, :cols.value]
    r2, c2 = C.c_int64(), C.c_int64()
    check(lib().hydot_block_load(ctx.h, os.fsencode(path), dptr(out), max(cols.value, 1),
                                 rows.value, C.byref(r2), C.byref(c2)), ctx.h)
    return out


def _geom_c(geom):
    """(nx, ny, nz, Lx, Ly, Lz) or any object with those attributes."""
    if hasattr(geom, "Lx"):
        t = (geom.nx, geom.ny, geom.nz, geom.Lx, geom.Ly, geom.Lz)
    else:
        t = tuple(geom)
    return _lib.GridGeom(int(t[0]), int(t[1]), int(t[2]), float(t[3]), float(t[4]), float(t[5]))


def apply_operator_fem(ctx: Context, geom, sigma: float, sigma_prime: float,
                       x: torch.Tensor) -> torch.Tensor:
    """(K + sigma M + sigma' R) x with the reference's trilinear-FEM K, lumped M
    and z-face R (grid.cpp:112-174), matrix-free on the device."""
    y = torch.empty_like(x)
    g = _geom_c(geom)
    check(lib().hydot_apply_fem(ctx.h, C.byref(g), sigma, sigma_prime, dptr(x), dptr(y)), ctx.h)
    return y


def compute_fields_fem(ctx: Context, geom, sigma, sigma_prime, inv_D, points_xyz,
                       tol: float = 1e-10, max_iter: int = 20000, fixed_iters: int = 0):
    """compute_fields (born.cpp:39-80) on the reference's own FEM operator with
    its trilinear point sources (points_xyz: n x 3 coordinates); returns
    (n, n_lambda, N) fields x_l / D_l and the CG statistics."""
    sig = np.ascontiguousarray(sigma, dtype=np.float64)
    sigp = np.ascontiguousarray(sigma_prime, dtype=np.float64)
    invd = np.ascontiguousarray(inv_D, dtype=np.float64)
    nl = sig.size
    pts = np.ascontiguousarray(points_xyz, dtype=np.float64).reshape(-1, 3)
    g = _geom_c(geom)
    N = g.nx * g.ny * g.nz
    out = ctx.empty(len(pts), nl, N)
    iters = np.zeros(len(pts) * nl, dtype=np.int32)
    rel = np.zeros(len(pts) * nl, dtype=np.float64)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    check(lib().hydot_fields_solve_fem(ctx.h, C.byref(g), nl, dp(sig), dp(sigp), dp(invd), dp(pts),
                                       len(pts), tol, max_iter, fixed_iters, dptr(out),
                                       iters.ctypes.data_as(C.POINTER(C.c_int)), dp(rel)), ctx.h)
    return out, FieldStats(iters.reshape(len(pts), nl), rel.reshape(len(pts), nl))
