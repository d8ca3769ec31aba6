// cg.cu -- batched matrix-free CG for the forward / adjoint fields
// (SURVEY 8a A4).  Replaces born::compute_fields' per-source calls of
// krylov::solve_family (born.cpp:54-65, krylov.cpp:400-463): every (point,
// wavelength) system (K + sigma_l M + sigma'_l R) x = e_v is SPD, so all of
// them run as one batch of independent CG iterations.
//
// Per iteration two HBM-streaming kernels, each CTA owning 1024 vertices of
// one system (grid.y = system):
//   cg_pa : p <- r + beta p (on the fly for the 6 neighbours), store p,
//           partial p.Ap                                   (reads r,p; writes p)
//   cg_xr : alpha = rr / p.Ap, x += alpha p, r -= alpha A p, partial r.r
//                                                         (reads p,x,r; writes x,r)
// For the 7-point operator (the BASELINE fields) the same two kernels run
// z-marching (cgz_pa / cgz_xr below): a CTA owns full x-rows of one system
// and walks the z planes with three planes of p in shared memory -- config 1
// fields 0.93 -> 0.63 s (36 -> 53 % of the 48 N B/iteration HBM figure).
// With even nx the planes are streamed by bulk copies (cp.async.bulk +
// mbarrier rings, cgzt_pa / cgzt_xr): 0.63 -> 0.50 s on config 1 (68 %),
// 6.96 -> 5.45 s on config 2 (69 %).
// Scalars never leave the device: each CTA sums its system's partials in a
// fixed order (deterministic), CTA 0 publishes rr into a parity slot.  The
// stencil and the vector updates use explicit _rn intrinsics in the oracle's
// operation order (no FMA contraction), so only the dot-product summation
// order differs from the CPU restatement.
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "internal.h"

namespace hydot {
namespace {

constexpr int CT = 256;       // threads per CTA
constexpr int VPT = 16;       // vertices per thread (amortises the scalar prologue)
constexpr int CV = CT * VPT;  // vertices per CTA

struct Stencil {
    int nx, ny, nz;
    double h;
    float inv_nx, inv_ny;  // for the division-free vertex decode
};

inline Stencil make_stencil(const hydot_grid7& g) {
    return Stencil{g.nx, g.ny, g.nz, g.h, 1.0f / float(g.nx), 1.0f / float(g.ny)};
}

// q = i / d, r = i % d for i < 2^24 without an integer division: a float
// estimate corrected by one step (64-bit div/mod dominated the CG kernels)
__device__ __forceinline__ void fdivmod(unsigned i, unsigned d, float inv_d, unsigned& q,
                                        unsigned& r) {
    q = __float2uint_rz(__uint2float_rn(i) * inv_d);
    int rr = int(i) - int(q * d);
    if (rr < 0) {
        --q;
        rr += int(d);
    } else if (rr >= int(d)) {
        ++q;
        rr -= int(d);
    }
    r = unsigned(rr);
}

// The 7-point operator row at vertex (ix, iy, iz) from its centre and six
// neighbour values, in the reference operation order.  Masked neighbours are
// selected away (not multiplied), so stale or clamped values never matter.
__device__ __forceinline__ double stencil7(int nx, int ny, int nz, double h, int ix, int iy, int iz,
                                           double sigma, double sigmap, double xi, double vxm,
                                           double vxp, double vym, double vyp, double vzm,
                                           double vzp) {
    const bool dir = (ix == 0 || ix == nx - 1 || iy == 0 || iy == ny - 1);
    const bool bxm = ix - 1 > 0, bxp = ix + 1 < nx - 1, bym = iy - 1 > 0, byp = iy + 1 < ny - 1;
    const bool bzm = iz > 0, bzp = iz < nz - 1;
    const bool zb = (iz == 0 || iz == nz - 1);
    const double zext = zb ? 0.5 * h : h;
    const double V = __dmul_rn(__dmul_rn(h, h), zext);
    const double S = zb ? __dmul_rn(h, h) : 0.0;
    const double xm = bxm ? vxm : 0.0;
    const double xp = bxp ? vxp : 0.0;
    const double ym = bym ? vym : 0.0;
    const double yp = byp ? vyp : 0.0;
    double wsum = 4.0 * zext;
    double nb = __dmul_rn(zext, xm);
    nb = __dadd_rn(nb, __dmul_rn(zext, xp));
    nb = __dadd_rn(nb, __dmul_rn(zext, ym));
    nb = __dadd_rn(nb, __dmul_rn(zext, yp));
    if (bzm) {
        wsum = __dadd_rn(wsum, h);
        nb = __dadd_rn(nb, __dmul_rn(h, vzm));
    }
    if (bzp) {
        wsum = __dadd_rn(wsum, h);
        nb = __dadd_rn(nb, __dmul_rn(h, vzp));
    }
    const double diag = __dadd_rn(__dadd_rn(wsum, __dmul_rn(sigma, V)), __dmul_rn(sigmap, S));
    const double y = __dsub_rn(__dmul_rn(diag, xi), nb);
    return dir ? xi : y;
}

// stencil7 split for the z-marching kernels: the diagonal depends only on
// the plane (zdiag, once per plane), the neighbour sum on the vertex
// (stencil7_nb); together they are stencil7's operations in its order.
struct ZDiag {
    double zext, diag;
    bool bzm, bzp;
};

__device__ __forceinline__ ZDiag zdiag(int nz, double h, int iz, double sigma, double sigmap) {
    ZDiag d;
    d.bzm = iz > 0;
    d.bzp = iz < nz - 1;
    const bool zb = (iz == 0 || iz == nz - 1);
    d.zext = zb ? 0.5 * h : h;
    const double V = __dmul_rn(__dmul_rn(h, h), d.zext);
    const double S = zb ? __dmul_rn(h, h) : 0.0;
    double wsum = 4.0 * d.zext;
    if (d.bzm) wsum = __dadd_rn(wsum, h);
    if (d.bzp) wsum = __dadd_rn(wsum, h);
    d.diag = __dadd_rn(__dadd_rn(wsum, __dmul_rn(sigma, V)), __dmul_rn(sigmap, S));
    return d;
}

__device__ __forceinline__ double stencil7_nb(int nx, int ny, double h, const ZDiag& d, int ix, int iy,
                                              double xi, double vxm, double vxp, double vym,
                                              double vyp, double vzm, double vzp) {
    const bool dir = (ix == 0 || ix == nx - 1 || iy == 0 || iy == ny - 1);
    const bool bxm = ix - 1 > 0, bxp = ix + 1 < nx - 1, bym = iy - 1 > 0, byp = iy + 1 < ny - 1;
    const double xm = bxm ? vxm : 0.0;
    const double xp = bxp ? vxp : 0.0;
    const double ym = bym ? vym : 0.0;
    const double yp = byp ? vyp : 0.0;
    double nb = __dmul_rn(d.zext, xm);
    nb = __dadd_rn(nb, __dmul_rn(d.zext, xp));
    nb = __dadd_rn(nb, __dmul_rn(d.zext, ym));
    nb = __dadd_rn(nb, __dmul_rn(d.zext, yp));
    if (d.bzm) nb = __dadd_rn(nb, __dmul_rn(h, vzm));
    if (d.bzp) nb = __dadd_rn(nb, __dmul_rn(h, vzp));
    const double y = __dsub_rn(__dmul_rn(d.diag, xi), nb);
    return dir ? xi : y;
}

// y_i = (A x)_i with x(j) supplied by a functor; reference operation order.
// Branch-free: every neighbour is loaded from a clamped in-range index, so
// the compiler can issue all loads of the unrolled vertices before their
// first use (the branchy form stalled on each load).
template <class Get>
__device__ __forceinline__ double stencil_at(const Stencil& g, double sigma, double sigmap,
                                             int64_t i, Get get) {
    const int64_t plane = int64_t(g.nx) * g.ny;
    const int64_t N = plane * g.nz;
    unsigned q1, ux, uy, uz;
    fdivmod(unsigned(i), unsigned(g.nx), g.inv_nx, q1, ux);
    fdivmod(q1, unsigned(g.ny), g.inv_ny, uz, uy);
    const double xi = get(i);
    const double vxm = get(i > 0 ? i - 1 : i);
    const double vxp = get(i + 1 < N ? i + 1 : i);
    const double vym = get(i >= g.nx ? i - g.nx : i);
    const double vyp = get(i + g.nx < N ? i + g.nx : i);
    const double vzm = get(i >= plane ? i - plane : i);
    const double vzp = get(i + plane < N ? i + plane : i);
    return stencil7(g.nx, g.ny, g.nz, g.h, int(ux), int(uy), int(uz), sigma, sigmap, xi, vxm, vxp,
                    vym, vyp, vzm, vzp);
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < CT / 32; ++i) t += sh[i];
    __syncthreads();
    return t;
}

// deterministic sum of nparts partials (all threads get the result)
__device__ __forceinline__ double sum_parts(const double* __restrict__ parts, int nparts,
                                            double* sh, double* bc) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nparts; i += CT) v += parts[i];
    double t = block_sum(v, sh);
    if (threadIdx.x == 0) *bc = t;
    __syncthreads();
    return *bc;
}

// ---------------------------------------------------------- operators --
// Op7: the BASELINE 7-point vertex-centred FV operator (stencil_at).
struct Op7 {
    Stencil g;
    template <class Get>
    __device__ __forceinline__ double operator()(int64_t i, double sigma, double sigmap, int, Get get) const {
        return stencil_at(g, sigma, sigmap, i, get);
    }
};

// Op7Var: the same operator with a per-vertex absorption -- the lumped mass
// weighted by sigma_l + dsig_l mu(v) (the nonlinear forward model's
// K + M_w + sp R with w = nu (mu_bg + dmu_l mu) / D, experiments.cpp:154-206)
struct Op7Var {
    Stencil g;
    const double* __restrict__ mu;    // N
    const double* __restrict__ dsig;  // n_lambda
    template <class Get>
    __device__ __forceinline__ double operator()(int64_t i, double sigma, double sigmap, int l, Get get) const {
        return stencil_at(g, __dadd_rn(sigma, __dmul_rn(dsig[l], mu[i])), sigmap, i, get);
    }
};

// OpFem: the reference's operator K + sigma M + sigma' R (grid.cpp:112-174)
// applied matrix-free: K trilinear-element stiffness with the Dirichlet
// side vertices eliminated (unit diagonal), M row-sum-lumped element mass,
// R bilinear face mass on the z = 0 and z = Lz faces -- not restricted to
// non-Dirichlet vertices, as in assemble_robin (the SURVEY A1 quirk).
// Element matrices come from the reference's 2x2x2 Gauss rule (host).
// Row sums run cell by cell in (cz, cy, cx) order, local vertex b inner.
struct OpFem {
    int nx, ny, nz;
    float inv_nx, inv_ny;
    const double* __restrict__ em;  // Ke (64) | Me (64) | Re (16)
    template <class Get>
    __device__ __forceinline__ double operator()(int64_t i, double sigma, double sigmap, int, Get get) const {
        unsigned q1, ux, uy, uz;
        fdivmod(unsigned(i), unsigned(nx), inv_nx, q1, ux);
        fdivmod(q1, unsigned(ny), inv_ny, uz, uy);
        const int ix = int(ux), iy = int(uy), iz = int(uz);
        auto dir = [&](int jx, int jy) { return jx == 0 || jx == nx - 1 || jy == 0 || jy == ny - 1; };
        const bool di = dir(ix, iy);
        const double xi = get(i);
        double kx = 0.0, m = 0.0;
        for (int oz = -1; oz <= 0; ++oz) {
            const int cz = iz + oz;
            if (cz < 0 || cz > nz - 2) continue;
            for (int oy = -1; oy <= 0; ++oy) {
                const int cy = iy + oy;
                if (cy < 0 || cy > ny - 2) continue;
                for (int ox = -1; ox <= 0; ++ox) {
                    const int cx = ix + ox;
                    if (cx < 0 || cx > nx - 2) continue;
                    const int a = (ox ? 1 : 0) | (oy ? 2 : 0) | (oz ? 4 : 0);
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const int jx = cx + (b & 1), jy = cy + ((b >> 1) & 1), jz = cz + ((b >> 2) & 1);
                        m = __dadd_rn(m, em[64 + a * 8 + b]);
                        if (!di && !dir(jx, jy)) {
                            const int64_t j = (int64_t(jz) * ny + jy) * nx + jx;
                            kx = __dadd_rn(kx, __dmul_rn(em[a * 8 + b], get(j)));
                        }
                    }
                }
            }
        }
        double y = di ? xi : kx;
        y = __dadd_rn(y, __dmul_rn(sigma, __dmul_rn(m, xi)));
        if (iz == 0 || iz == nz - 1) {
            double rx = 0.0;
            for (int oy = -1; oy <= 0; ++oy) {
                const int cy = iy + oy;
                if (cy < 0 || cy > ny - 2) continue;
                for (int ox = -1; ox <= 0; ++ox) {
                    const int cx = ix + ox;
                    if (cx < 0 || cx > nx - 2) continue;
                    const int a = (ox ? 1 : 0) | (oy ? 2 : 0);
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int64_t j = (int64_t(iz) * ny + cy + ((b >> 1) & 1)) * nx + cx + (b & 1);
                        rx = __dadd_rn(rx, __dmul_rn(em[128 + a * 4 + b], get(j)));
                    }
                }
            }
            y = __dadd_rn(y, __dmul_rn(sigmap, rx));
        }
        return y;
    }
};

struct SysState {
    double rr[2];   // r.r published per iteration parity
    double bnorm;   // ||b||
    int done;       // converged (or stopped)
    int iters;
    double relres;
};

// zero x, r, p; scalars from ||b||^2 (b set by cg_rhs)
__global__ void cg_init(int64_t N, int nl, const double* __restrict__ rhs_b2, int k0, double* __restrict__ X,
                        double* __restrict__ R, double* __restrict__ P, SysState* __restrict__ st) {
    const int sys = blockIdx.y;
    const int kglob = k0 + sys;
    double* x = X + int64_t(sys) * N;  // x lives in the output (caller column)
    double* r = R + int64_t(sys) * N;
    double* p = P + int64_t(sys) * N;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < N;
         i += int64_t(gridDim.x) * blockDim.x) {
        x[i] = 0.0;
        r[i] = 0.0;
        p[i] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const double b2 = rhs_b2[kglob / nl];
        st[sys].rr[0] = b2;
        st[sys].rr[1] = 0.0;
        st[sys].bnorm = sqrt(b2);
        st[sys].done = 0;
        st[sys].iters = 0;
        st[sys].relres = 1.0;
    }
}

// r = b: up to 8 (vertex, weight) entries per right-hand side
__global__ void cg_rhs(int64_t N, int nl, int k0, int nb, const int64_t* __restrict__ ridx,
                       const double* __restrict__ rw, double* __restrict__ R) {
    const int sys = blockIdx.x * blockDim.y + threadIdx.y;
    const int e = threadIdx.x;  // 0..7
    if (sys >= nb) return;
    const int rhs = (k0 + sys) / nl;
    const int64_t v = ridx[int64_t(rhs) * 8 + e];
    if (v >= 0) R[int64_t(sys) * N + v] = rw[int64_t(rhs) * 8 + e];
}

template <class Op>
__global__ void __launch_bounds__(CT, 4) cg_pa(Op op, int64_t N, int nl, int k0, int it,
                                            const double* __restrict__ sig,
                                            const double* __restrict__ sigp,
                                            const double* __restrict__ R,
                                            const double* __restrict__ Pold,
                                            double* __restrict__ Pnew, double* __restrict__ partA,
                                            const double* __restrict__ partB, int nparts,
                                            SysState* __restrict__ st, double tol, int fixed,
                                            const int* __restrict__ act) {
    __shared__ double sh[CT / 32];
    __shared__ double bc;
    const int sys = act[blockIdx.y];  // compacted list of unconverged systems
    SysState& S = st[sys];
    if (S.done) return;
    const int l = (k0 + sys) % nl;
    double beta = 0.0;
    const int slot = it & 1;
    if (it > 0) {
        const double rr_new = sum_parts(partB + int64_t(sys) * nparts, nparts, sh, &bc);
        const double rr_old = S.rr[slot ^ 1];
        const double relres = sqrt(rr_new) / S.bnorm;
        if (!fixed && relres <= tol) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                S.done = 1;
                S.iters = it;
                S.relres = relres;
            }
            return;
        }
        beta = rr_new / rr_old;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            S.rr[slot] = rr_new;
            S.relres = relres;
            S.iters = it;
        }
    }
    const double* r = R + int64_t(sys) * N;
    const double* po = Pold + int64_t(sys) * N;
    double* p = Pnew + int64_t(sys) * N;
    const double sigma = sig[l], sigmap = sigp[l];
    auto pnew = [&](int64_t j) { return __dadd_rn(r[j], __dmul_rn(beta, po[j])); };
    // p is double-buffered across iterations: neighbours in other CTAs
    // still read p_old while this CTA stores p_new.
    double acc = 0.0;
    const int64_t base = int64_t(blockIdx.x) * CV + threadIdx.x;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int64_t i = base + int64_t(k) * CT;
        if (i < N) {
            const double pi = pnew(i);
            const double ap = op(i, sigma, sigmap, l, pnew);
            p[i] = pi;
            acc += pi * ap;
        }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partA[int64_t(sys) * nparts + blockIdx.x] = t;
}

template <class Op>
__global__ void __launch_bounds__(CT, 4) cg_xr(Op op, int64_t N, int nl, int k0, int it,
                                            const double* __restrict__ sig,
                                            const double* __restrict__ sigp,
                                            double* __restrict__ X, double* __restrict__ R,
                                            const double* __restrict__ P,
                                            const double* __restrict__ partA,
                                            double* __restrict__ partB, int nparts,
                                            SysState* __restrict__ st,
                                            const int* __restrict__ act) {
    __shared__ double sh[CT / 32];
    __shared__ double bc;
    const int sys = act[blockIdx.y];
    SysState& S = st[sys];
    if (S.done) return;
    const int l = (k0 + sys) % nl;
    const double pq = sum_parts(partA + int64_t(sys) * nparts, nparts, sh, &bc);
    const double alpha = S.rr[it & 1] / pq;
    double* x = X + int64_t(sys) * N;
    double* r = R + int64_t(sys) * N;
    const double* p = P + int64_t(sys) * N;
    const double sigma = sig[l], sigmap = sigp[l];
    auto getp = [&](int64_t j) { return p[j]; };
    double acc = 0.0;
    const int64_t base = int64_t(blockIdx.x) * CV + threadIdx.x;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int64_t i = base + int64_t(k) * CT;
        if (i < N) {
            const double q = op(i, sigma, sigmap, l, getp);
            x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
            const double rn = __dsub_rn(r[i], __dmul_rn(alpha, q));
            r[i] = rn;
            acc += rn * rn;
        }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partB[int64_t(sys) * nparts + blockIdx.x] = t;
}

// ------------------------------------------------------ z-marching (Op7) --
// The same two kernels for the 7-point operator with a 2.5-D tiling: a CTA
// owns `ty` full x-rows of one system and marches through the z planes,
// keeping three planes of its (ty+2)-row halo'ed tile in shared memory.
// Each vertex's p_new is formed once per plane (instead of once per stencil
// use), every load is a coalesced x-row, and the next plane is prefetched
// into registers while the current one is computed.  Arithmetic is
// stencil7 in the reference order, so the result is bit-identical to the
// vertex-parallel kernels above (only the dot-product partition differs).
constexpr int ZT = 256;  // threads per CTA
constexpr int ZE = 6;    // halo'ed tile elements per thread: (ty + 2) nx <= ZT ZE
constexpr int ZO = 5;    // own-tile elements per thread:     ty nx <= ZT ZO

struct ZGeo {
    int nx, ny, nz, ty;
    double h;
};

// Tile geometry: halo'ed element e (row-major over ty+2 rows) lives at plane
// offset base + e and is inside the grid for lo <= e < hi; own element e
// (e < Wo) lives at base + nx + e and at tile index e + nx.  Only the own
// elements' (ix, iy) are kept per thread (packed), for the stencil masks.
struct ZIdx {
    int base, lo, hi, W, Wo;
    int oxy[ZO];  // ix | iy << 16
};

__device__ __forceinline__ void zidx(const ZGeo& g, ZIdx& z) {
    const int y0 = blockIdx.x * g.ty;
    const int rows = min(g.ty, g.ny - y0);
    z.W = (rows + 2) * g.nx;
    z.Wo = rows * g.nx;
    z.base = (y0 - 1) * g.nx;
    z.lo = y0 == 0 ? g.nx : 0;
    z.hi = y0 + rows == g.ny ? (rows + 1) * g.nx : z.W;
#pragma unroll
    for (int k = 0; k < ZO; ++k) {
        const int e = threadIdx.x + k * ZT;
        const int ry = e / g.nx, ix = e - ry * g.nx;
        z.oxy[k] = ix | ((y0 + ry) << 16);
    }
}

// stencil at own element e of plane iz from the three shared planes
__device__ __forceinline__ double zstencil(const ZGeo& g, const ZIdx& z, int k, int e, const ZDiag& d,
                                           const double* __restrict__ c, const double* __restrict__ dn,
                                           const double* __restrict__ up) {
    const int si = e + g.nx, ix = z.oxy[k] & 0xffff, iy = z.oxy[k] >> 16;
    return stencil7_nb(g.nx, g.ny, g.h, d, ix, iy, c[si], c[ix > 0 ? si - 1 : si],
                       c[ix < g.nx - 1 ? si + 1 : si], c[si - g.nx], c[si + g.nx], dn[si], up[si]);
}

template <int MINB>
__global__ void __launch_bounds__(ZT, MINB) cgz_pa(ZGeo g, int64_t N, int nl, int k0, int it,
                                              const double* __restrict__ sig,
                                              const double* __restrict__ sigp,
                                              const double* __restrict__ R,
                                              const double* __restrict__ Pold,
                                              double* __restrict__ Pnew, double* __restrict__ partA,
                                              const double* __restrict__ partB, int nparts,
                                              SysState* __restrict__ st, double tol, int fixed,
                                              const int* __restrict__ act) {
    extern __shared__ double zs[];  // 3 planes of the halo'ed tile
    __shared__ double sh[ZT / 32];
    __shared__ double bc;
    const int sys = act[blockIdx.y];
    SysState& S = st[sys];
    if (S.done) return;
    const int l = (k0 + sys) % nl;
    double beta = 0.0;
    const int slot = it & 1;
    if (it > 0) {
        const double rr_new = sum_parts(partB + int64_t(sys) * nparts, nparts, sh, &bc);
        const double rr_old = S.rr[slot ^ 1];
        const double relres = sqrt(rr_new) / S.bnorm;
        if (!fixed && relres <= tol) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                S.done = 1;
                S.iters = it;
                S.relres = relres;
            }
            return;
        }
        beta = rr_new / rr_old;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            S.rr[slot] = rr_new;
            S.relres = relres;
            S.iters = it;
        }
    }
    ZIdx z;
    zidx(g, z);
    const int64_t plane = int64_t(g.nx) * g.ny;
    const double* r = R + int64_t(sys) * N;
    const double* po = Pold + int64_t(sys) * N;
    double* p = Pnew + int64_t(sys) * N;
    const double sigma = sig[l], sigmap = sigp[l];
    double rv[ZE], pv[ZE];
    auto load = [&](int iz) {
#pragma unroll
        for (int k = 0; k < ZE; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e >= z.lo && e < z.hi) {
                const int64_t i = iz * plane + z.base + e;
                rv[k] = __ldcs(r + i);
                pv[k] = __ldcs(po + i);
            }
        }
    };
    auto put = [&](int iz) {
        double* s = zs + (iz % 3) * z.W;
#pragma unroll
        for (int k = 0; k < ZE; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e < z.W) s[e] = (e >= z.lo && e < z.hi) ? __dadd_rn(rv[k], __dmul_rn(beta, pv[k])) : 0.0;
        }
    };
    load(0);
    put(0);
    if (g.nz > 1) load(1);
    double acc = 0.0;
    for (int iz = 0; iz < g.nz; ++iz) {
        if (iz + 1 < g.nz) put(iz + 1);
        if (iz + 2 < g.nz) load(iz + 2);
        __syncthreads();
        const double* c = zs + (iz % 3) * z.W;
        const double* dn = zs + ((iz + 2) % 3) * z.W;
        const double* up = zs + ((iz + 1) % 3) * z.W;
        const ZDiag d = zdiag(g.nz, g.h, iz, sigma, sigmap);
#pragma unroll
        for (int k = 0; k < ZO; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e < z.Wo) {
                const double pi = c[e + g.nx];
                const double ap = zstencil(g, z, k, e, d, c, dn, up);
                __stcs(p + iz * plane + z.base + g.nx + e, pi);
                acc += pi * ap;
            }
        }
        __syncthreads();
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partA[int64_t(sys) * nparts + blockIdx.x] = t;
}

template <int MINB>
__global__ void __launch_bounds__(ZT, MINB) cgz_xr(ZGeo g, int64_t N, int nl, int k0, int it,
                                              const double* __restrict__ sig,
                                              const double* __restrict__ sigp,
                                              double* __restrict__ X, double* __restrict__ R,
                                              const double* __restrict__ P,
                                              const double* __restrict__ partA,
                                              double* __restrict__ partB, int nparts,
                                              SysState* __restrict__ st,
                                              const int* __restrict__ act) {
    extern __shared__ double zs[];
    __shared__ double sh[ZT / 32];
    __shared__ double bc;
    const int sys = act[blockIdx.y];
    SysState& S = st[sys];
    if (S.done) return;
    const int l = (k0 + sys) % nl;
    const double pq = sum_parts(partA + int64_t(sys) * nparts, nparts, sh, &bc);
    const double alpha = S.rr[it & 1] / pq;
    ZIdx z;
    zidx(g, z);
    const int64_t plane = int64_t(g.nx) * g.ny;
    double* x = X + int64_t(sys) * N;
    double* r = R + int64_t(sys) * N;
    const double* p = P + int64_t(sys) * N;
    const double sigma = sig[l], sigmap = sigp[l];
    double pv[ZE], xv[ZO], rv[ZO];
    auto loadp = [&](int iz) {
#pragma unroll
        for (int k = 0; k < ZE; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e >= z.lo && e < z.hi) pv[k] = __ldcs(p + iz * plane + z.base + e);
        }
    };
    auto loadxr = [&](int iz) {
#pragma unroll
        for (int k = 0; k < ZO; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e < z.Wo) {
                xv[k] = __ldcs(x + iz * plane + z.base + g.nx + e);
                rv[k] = __ldcs(r + iz * plane + z.base + g.nx + e);
            }
        }
    };
    auto put = [&](int iz) {
        double* s = zs + (iz % 3) * z.W;
#pragma unroll
        for (int k = 0; k < ZE; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e < z.W) s[e] = (e >= z.lo && e < z.hi) ? pv[k] : 0.0;
        }
    };
    loadp(0);
    put(0);
    if (g.nz > 1) loadp(1);
    loadxr(0);
    double acc = 0.0;
    for (int iz = 0; iz < g.nz; ++iz) {
        if (iz + 1 < g.nz) put(iz + 1);
        if (iz + 2 < g.nz) loadp(iz + 2);
        __syncthreads();
        const double* c = zs + (iz % 3) * z.W;
        const double* dn = zs + ((iz + 2) % 3) * z.W;
        const double* up = zs + ((iz + 1) % 3) * z.W;
        const ZDiag d = zdiag(g.nz, g.h, iz, sigma, sigmap);
#pragma unroll
        for (int k = 0; k < ZO; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e < z.Wo) {
                const double q = zstencil(g, z, k, e, d, c, dn, up);
                const int64_t i = iz * plane + z.base + g.nx + e;
                __stcs(x + i, __dadd_rn(xv[k], __dmul_rn(alpha, c[e + g.nx])));
                const double rn = __dsub_rn(rv[k], __dmul_rn(alpha, q));
                __stcs(r + i, rn);
                acc += rn * rn;
            }
        }
        if (iz + 1 < g.nz) loadxr(iz + 1);  // in flight across the barrier and the next put
        __syncthreads();
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partB[int64_t(sys) * nparts + blockIdx.x] = t;
}

// ------------------------------------------- z-marching with bulk copies --
// cgzt_xr: cgz_xr with the planes streamed by the bulk-copy engine (one
// cp.async.bulk per plane and array, mbarrier completion) into shared-memory
// rings -- p: 5 planes (3 in use, 2 in flight), x / r: 3 planes (1 in use,
// 2 in flight).  No load instructions or prefetch registers in the loop and
// one block barrier per plane.  Needs 16-byte aligned rows (nx even).
constexpr int NSP = 5, NSX = 3;

__device__ __forceinline__ uint32_t su32(const void* q) { return uint32_t(__cvta_generic_to_shared(q)); }
__device__ __forceinline__ void mb_init(uint64_t* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n\t.reg .pred P;\nWAIT%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra WAIT%=;\n}" ::"r"(
            su32(b)),
        "r"(par)
        : "memory");
}

__global__ void __launch_bounds__(ZT, 2) cgzt_xr(ZGeo g, int64_t N, int nl, int k0, int it,
                                               const double* __restrict__ sig,
                                               const double* __restrict__ sigp,
                                               double* __restrict__ X, double* __restrict__ R,
                                               const double* __restrict__ P,
                                               const double* __restrict__ partA,
                                               double* __restrict__ partB, int nparts,
                                               SysState* __restrict__ st,
                                               const int* __restrict__ act) {
    extern __shared__ __align__(16) double zs[];
    __shared__ __align__(8) uint64_t bar[NSP + NSX];
    __shared__ double sh[ZT / 32];
    __shared__ double bc;
    const int sys = act[blockIdx.y];
    SysState& S = st[sys];
    if (S.done) return;
    const int l = (k0 + sys) % nl;
    const double pq = sum_parts(partA + int64_t(sys) * nparts, nparts, sh, &bc);
    const double alpha = S.rr[it & 1] / pq;
    ZIdx z;
    zidx(g, z);
    const int64_t plane = int64_t(g.nx) * g.ny;
    double* x = X + int64_t(sys) * N;
    double* r = R + int64_t(sys) * N;
    const double* p = P + int64_t(sys) * N;
    const double sigma = sig[l], sigmap = sigp[l];
    double* pring = zs;                   // NSP x W
    double* xring = zs + NSP * z.W;       // NSX x (x | r) x Wo
    const uint32_t pbytes = uint32_t(z.hi - z.lo) * 8u, xbytes = uint32_t(z.Wo) * 8u;
    auto issue_p = [&](int j) {
        const int sl = j % NSP;
        mb_expect(&bar[sl], pbytes);
        bulk_load(pring + sl * z.W + z.lo, p + j * plane + z.base + z.lo, pbytes, &bar[sl]);
    };
    auto issue_xr = [&](int j) {
        const int sl = j % NSX;
        mb_expect(&bar[NSP + sl], 2u * xbytes);
        const int64_t o = j * plane + z.base + g.nx;
        bulk_load(xring + (2 * sl) * z.Wo, x + o, xbytes, &bar[NSP + sl]);
        bulk_load(xring + (2 * sl + 1) * z.Wo, r + o, xbytes, &bar[NSP + sl]);
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSP + NSX; ++i) mb_init(&bar[i]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int j = 0; j < 3 && j < g.nz; ++j) issue_p(j);
        for (int j = 0; j < 2 && j < g.nz; ++j) issue_xr(j);
    }
    double acc = 0.0;
    for (int iz = 0; iz < g.nz; ++iz) {
        if (iz > 0) __syncthreads();  // plane iz-1's reads are done: its slots may refill
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (iz + 3 < g.nz) issue_p(iz + 3);    // into p(iz-2)'s slot
            if (iz + 2 < g.nz) issue_xr(iz + 2);   // into x/r(iz-1)'s slot
        }
        if (iz == 0) mb_wait(&bar[0], 0);
        if (iz + 1 < g.nz) mb_wait(&bar[(iz + 1) % NSP], uint32_t(((iz + 1) / NSP) & 1));
        mb_wait(&bar[NSP + iz % NSX], uint32_t((iz / NSX) & 1));
        const double* c = pring + (iz % NSP) * z.W;
        const double* dn = pring + ((iz + NSP - 1) % NSP) * z.W;
        const double* up = pring + ((iz + 1) % NSP) * z.W;
        const double* xs = xring + (2 * (iz % NSX)) * z.Wo;
        const double* rs = xs + z.Wo;
        const ZDiag d = zdiag(g.nz, g.h, iz, sigma, sigmap);
#pragma unroll
        for (int k = 0; k < ZO; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e < z.Wo) {
                const double q = zstencil(g, z, k, e, d, c, dn, up);
                const int64_t i = iz * plane + z.base + g.nx + e;
                __stcs(x + i, __dadd_rn(xs[e], __dmul_rn(alpha, c[e + g.nx])));
                const double rn = __dsub_rn(rs[e], __dmul_rn(alpha, q));
                __stcs(r + i, rn);
                acc += rn * rn;
            }
        }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partB[int64_t(sys) * nparts + blockIdx.x] = t;
}

// cgzt_pa: cgz_pa with r and p_old streamed by bulk copies into a 3-plane
// ring; p_new = r + beta p_old is formed once per vertex into a 4-plane ring
// (4 slots: the plane written at step iz was last read two barriers ago, so
// one block barrier per plane suffices).
constexpr int NSR = 3;

// NS raw planes in the ring, NPN p_new planes (4: one barrier per plane;
// 3: a second barrier per plane, one more raw plane in flight in the same
// shared memory)
template <int NS, int NPN>
__global__ void __launch_bounds__(ZT, 2) cgzt_pa(ZGeo g, int64_t N, int nl, int k0, int it,
                                               const double* __restrict__ sig,
                                               const double* __restrict__ sigp,
                                               const double* __restrict__ R,
                                               const double* __restrict__ Pold,
                                               double* __restrict__ Pnew, double* __restrict__ partA,
                                               const double* __restrict__ partB, int nparts,
                                               SysState* __restrict__ st, double tol, int fixed,
                                               const int* __restrict__ act) {
    extern __shared__ __align__(16) double zs[];
    __shared__ __align__(8) uint64_t bar[NS];
    __shared__ double sh[ZT / 32];
    __shared__ double bc;
    const int sys = act[blockIdx.y];
    SysState& S = st[sys];
    if (S.done) return;
    const int l = (k0 + sys) % nl;
    double beta = 0.0;
    const int slot = it & 1;
    if (it > 0) {
        const double rr_new = sum_parts(partB + int64_t(sys) * nparts, nparts, sh, &bc);
        const double rr_old = S.rr[slot ^ 1];
        const double relres = sqrt(rr_new) / S.bnorm;
        if (!fixed && relres <= tol) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                S.done = 1;
                S.iters = it;
                S.relres = relres;
            }
            return;
        }
        beta = rr_new / rr_old;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            S.rr[slot] = rr_new;
            S.relres = relres;
            S.iters = it;
        }
    }
    ZIdx z;
    zidx(g, z);
    const int64_t plane = int64_t(g.nx) * g.ny;
    const double* r = R + int64_t(sys) * N;
    const double* po = Pold + int64_t(sys) * N;
    double* p = Pnew + int64_t(sys) * N;
    const double sigma = sig[l], sigmap = sigp[l];
    double* raw = zs;                 // NS x (r | p_old) x W
    double* pn = zs + 2 * NS * z.W;  // NPN x W
    const uint32_t bytes = uint32_t(z.hi - z.lo) * 8u;
    auto issue = [&](int j) {
        const int sl = j % NS;
        mb_expect(&bar[sl], 2u * bytes);
        const int64_t o = j * plane + z.base + z.lo;
        bulk_load(raw + (2 * sl) * z.W + z.lo, r + o, bytes, &bar[sl]);
        bulk_load(raw + (2 * sl + 1) * z.W + z.lo, po + o, bytes, &bar[sl]);
    };
    auto convert = [&](int j) {  // pn[j % 4] = r + beta p_old on the in-grid rows
        const int sl = j % NS;
        mb_wait(&bar[sl], uint32_t((j / NS) & 1));
        const double* rs = raw + (2 * sl) * z.W;
        const double* ps = rs + z.W;
        double* out = pn + (j % NPN) * z.W;
#pragma unroll
        for (int k = 0; k < ZE; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e >= z.lo && e < z.hi) out[e] = __dadd_rn(rs[e], __dmul_rn(beta, ps[e]));
        }
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) mb_init(&bar[i]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = threadIdx.x; e < NPN * z.W; e += ZT) pn[e] = 0.0;  // out-of-grid halo rows
    __syncthreads();
    if (threadIdx.x == 0)
        for (int j = 0; j < NS && j < g.nz; ++j) issue(j);
    convert(0);
    __syncthreads();
    if (threadIdx.x == 0 && NS < g.nz) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(NS);
    }
    double acc = 0.0;
    for (int iz = 0; iz < g.nz; ++iz) {
        const int j = iz + 1;
        if (j < g.nz) convert(j);
        __syncthreads();
        if (threadIdx.x == 0 && j + NS < g.nz) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(j + NS);  // into raw(j)'s slot, converted above
        }
        const double* c = pn + (iz % NPN) * z.W;
        const double* dn = pn + ((iz + NPN - 1) % NPN) * z.W;
        const double* up = pn + ((iz + 1) % NPN) * z.W;
        const ZDiag d = zdiag(g.nz, g.h, iz, sigma, sigmap);
#pragma unroll
        for (int k = 0; k < ZO; ++k) {
            const int e = threadIdx.x + k * ZT;
            if (e < z.Wo) {
                const double pi = c[e + g.nx];
                const double ap = zstencil(g, z, k, e, d, c, dn, up);
                __stcs(p + iz * plane + z.base + g.nx + e, pi);
                acc += pi * ap;
            }
        }
        if (NPN == 3) __syncthreads();  // pn(iz-1)'s slot is refilled next
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partA[int64_t(sys) * nparts + blockIdx.x] = t;
}

// CTAs per SM the z-marching kernels are compiled for (3: 80 registers;
// 4 forces 64 and spills: 0.84 vs 0.63 s on config 1)
#define ZSEL(k) (k<3>)

// (a cgzt_pa with 4 raw planes and 3 p_new planes -- one more plane in
// flight, one more barrier per plane -- measured 0.493 -> 0.503 s on config 1)

// bulk-copy x/r kernel for even nx (HYDOT_CG_BULK=0 keeps the register one)
bool zbulk_on() {
    static const bool on = [] {
        const char* e = std::getenv("HYDOT_CG_BULK");
        return !(e && e[0] == '0');
    }();
    return on;
}

// z-march tile height for an nx x ny plane (0 = tile does not fit: use the
// vertex-parallel kernels); balanced over the tiles
int zmarch_ty(int nx, int ny) {
    static const bool on = [] {
        const char* e = std::getenv("HYDOT_CG_ZMARCH");
        return !(e && e[0] == '0');
    }();
    if (!on) return 0;
    const int tmax = std::min(ny, std::min(ZT * ZE / nx - 2, ZT * ZO / nx));
    if (tmax < 1) return 0;
    const int ntiles = (ny + tmax - 1) / tmax;
    return (ny + ntiles - 1) / ntiles;
}

// fixed-iteration / max-iteration finish: final relres, scale by inv_D
__global__ void cg_finish(int64_t N, int nl, int k0, int it_total, double* __restrict__ X,
                          const double* __restrict__ invD, const double* __restrict__ partB,
                          int nparts, SysState* __restrict__ st) {
    __shared__ double sh[CT / 32];
    __shared__ double bc;
    const int sys = blockIdx.y;
    SysState& S = st[sys];
    const int l = (k0 + sys) % nl;
    if (!S.done && blockIdx.x == 0) {
        double rr = sum_parts(partB + int64_t(sys) * nparts, nparts, sh, &bc);
        if (threadIdx.x == 0) {
            S.relres = sqrt(rr) / S.bnorm;
            S.iters = it_total;
        }
    }
    const double s = invD[l];
    double* x = X + int64_t(sys) * N;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < N;
         i += int64_t(gridDim.x) * blockDim.x)
        x[i] = x[i] * s;
}

template <class Op>
__global__ void apply_k(Op op, int64_t N, double sigma, double sigmap, const double* __restrict__ x,
                        double* __restrict__ y) {
    auto get = [&](int64_t j) { return x[j]; };
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < N;
         i += int64_t(gridDim.x) * blockDim.x)
        y[i] = op(i, sigma, sigmap, 0, get);
}

__global__ void count_active(int n, const SysState* __restrict__ st, int* __restrict__ out) {
    int a = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) a += st[i].done ? 0 : 1;
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    __shared__ int sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
        *out = t;
    }
}

}  // namespace

namespace {

// the batched CG over any operator: rhs n_rhs sparse vectors (ridx / rw, 8
// entries each, -1 = unused) times n_lambda shifts
template <class Op>
void cg_batch(Ctx& c, const Op& op, int64_t N, int nl, const double* sigma, const double* sigmap,
              const double* inv_D, const std::vector<int64_t>& ridx, const std::vector<double>& rw,
              const std::vector<double>& b2, int n_rhs, double tol, int max_iter, int fixed_iters, double* out,
              CGStats* stats) {
    if (N >= (int64_t(1) << 24)) throw std::invalid_argument("fields_solve: grid too large for the 24-bit vertex decode");
    const int total = n_rhs * nl;
    int nparts = int((N + CV - 1) / CV);
    // 7-point operator: z-marching kernels when the halo'ed tile fits
    ZGeo zg{};
    size_t zsmem = 0, ztsmem = 0, ztpsmem = 0;
    if constexpr (std::is_same_v<Op, Op7>) {
        const int ty = zmarch_ty(op.g.nx, op.g.ny);
        if (ty > 0) {
            zg = ZGeo{op.g.nx, op.g.ny, op.g.nz, ty, op.g.h};
            nparts = (op.g.ny + ty - 1) / ty;
            zsmem = size_t(3) * size_t(ty + 2) * size_t(op.g.nx) * sizeof(double);
            if (op.g.nx % 2 == 0 && zbulk_on()) {
                ztsmem = size_t(NSP * (ty + 2) + NSX * 2 * ty) * size_t(op.g.nx) * sizeof(double);
                ztpsmem = size_t((2 * NSR + 4) * (ty + 2)) * size_t(op.g.nx) * sizeof(double);
                static AttrGate attr;
                attr_once(attr, c.device, [&] {
                    HYDOT_CUDA(cudaFuncSetAttribute(cgzt_xr, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    200 * 1024));
                    HYDOT_CUDA(cudaFuncSetAttribute(cgzt_pa<NSR, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    200 * 1024));
                });
            }
        }
    }
    // One batch of up to 24 GB (all systems iterate together, HBM-bound).
    // L2-sized groups (32 N bytes per system) measured slower on config 1
    // (1.4-2.8 s vs 0.96 s: small groups make the iterations launch- and
    // sync-bound).
    int64_t per_sys = 2 * N * 8;
    int batch = int(std::max<int64_t>(1, std::min<int64_t>(total, (int64_t(24) << 30) / per_sys)));
    batch = std::min(batch, 65535);
    DBuf dsig = dalloc(c, size_t(nl)), dsigp = dalloc(c, size_t(nl)), dinv = dalloc(c, size_t(nl));
    HYDOT_CUDA(cudaMemcpyAsync(dsig.d(), sigma, size_t(nl) * 8, cudaMemcpyHostToDevice, c.stream));
    HYDOT_CUDA(cudaMemcpyAsync(dsigp.d(), sigmap, size_t(nl) * 8, cudaMemcpyHostToDevice, c.stream));
    HYDOT_CUDA(cudaMemcpyAsync(dinv.d(), inv_D, size_t(nl) * 8, cudaMemcpyHostToDevice, c.stream));
    // sparse right-hand sides: 8 (vertex, weight) entries each, and ||b||^2
    DBuf dridx(c, size_t(n_rhs) * 8 * sizeof(int64_t));
    DBuf drw = dalloc(c, size_t(n_rhs) * 8), db2 = dalloc(c, size_t(n_rhs));
    HYDOT_CUDA(cudaMemcpyAsync(dridx.as<void>(), ridx.data(), ridx.size() * 8, cudaMemcpyHostToDevice, c.stream));
    HYDOT_CUDA(cudaMemcpyAsync(drw.d(), rw.data(), rw.size() * 8, cudaMemcpyHostToDevice, c.stream));
    HYDOT_CUDA(cudaMemcpyAsync(db2.d(), b2.data(), b2.size() * 8, cudaMemcpyHostToDevice, c.stream));
    DBuf R = dalloc(c, size_t(batch) * size_t(N));
    DBuf P = dalloc(c, 2 * size_t(batch) * size_t(N));  // double-buffered p
    DBuf pA = dalloc(c, size_t(batch) * size_t(nparts));
    DBuf pB = dalloc(c, size_t(batch) * size_t(nparts));
    DBuf S(c, size_t(batch) * sizeof(SysState));
    DBuf dact(c, sizeof(int) * size_t(batch));
    if (stats) {
        stats->iters.assign(size_t(total), 0);
        stats->relres.assign(size_t(total), 0.0);
    }
    const int limit = fixed_iters > 0 ? fixed_iters : max_iter;
    for (int k0 = 0; k0 < total; k0 += batch) {
        const int nb = std::min(batch, total - k0);
        double* X = out + int64_t(k0) * N;
        SysState* ss = S.as<SysState>();
        {
            dim3 gi = dim3(unsigned(std::min<int64_t>((N + 255) / 256, 1024)), unsigned(nb));
            // p_old of iteration 0 is buffer 1 (zeroed); p_it lives in buffer it&1
            cg_init<<<gi, 256, 0, c.stream>>>(N, nl, db2.d(), k0, X, R.d(),
                                              P.d() + size_t(batch) * size_t(N), ss);
            c.check_launch();
            dim3 gr = dim3(unsigned((nb + 31) / 32));
            cg_rhs<<<gr, dim3(8, 32), 0, c.stream>>>(N, nl, k0, nb, dridx.as<int64_t>(), drw.d(), R.d());
            c.check_launch();
        }
        auto pbuf = [&](int i) { return P.d() + size_t(i & 1) * size_t(batch) * size_t(N); };
        // active-system list: converged systems are dropped from the grid
        // every 8 iterations (systems converge between ~70 and ~135 iterations)
        std::vector<int> active(static_cast<size_t>(nb));
        for (int k = 0; k < nb; ++k) active[size_t(k)] = k;
        std::vector<SysState> hst(static_cast<size_t>(nb));
        HYDOT_CUDA(cudaMemcpyAsync(dact.as<void>(), active.data(), active.size() * sizeof(int),
                                   cudaMemcpyHostToDevice, c.stream));
        int it = 0;
        for (; it < limit; ++it) {
            dim3 grid = dim3(unsigned(nparts), unsigned(active.size()));
            if (zsmem) {
                if (ztpsmem)
                    cgzt_pa<NSR, 4><<<grid, ZT, ztpsmem, c.stream>>>(zg, N, nl, k0, it, dsig.d(), dsigp.d(), R.d(),
                                                             pbuf(it + 1), pbuf(it), pA.d(), pB.d(), nparts, ss,
                                                             tol, fixed_iters > 0, dact.as<int>());
                else
                    ZSEL(cgz_pa)<<<grid, ZT, zsmem, c.stream>>>(zg, N, nl, k0, it, dsig.d(), dsigp.d(), R.d(),
                                                                pbuf(it + 1), pbuf(it), pA.d(), pB.d(), nparts,
                                                                ss, tol, fixed_iters > 0, dact.as<int>());
                c.check_launch();
                if (ztsmem)
                    cgzt_xr<<<grid, ZT, ztsmem, c.stream>>>(zg, N, nl, k0, it, dsig.d(), dsigp.d(), X, R.d(),
                                                            pbuf(it), pA.d(), pB.d(), nparts, ss, dact.as<int>());
                else
                    ZSEL(cgz_xr)<<<grid, ZT, zsmem, c.stream>>>(zg, N, nl, k0, it, dsig.d(), dsigp.d(), X,
                                                                R.d(), pbuf(it), pA.d(), pB.d(), nparts, ss,
                                                                dact.as<int>());
                c.check_launch();
            } else {
            cg_pa<<<grid, CT, 0, c.stream>>>(op, N, nl, k0, it, dsig.d(), dsigp.d(), R.d(),
                                            pbuf(it + 1), pbuf(it), pA.d(), pB.d(), nparts, ss,
                                            tol, fixed_iters > 0, dact.as<int>());
            c.check_launch();
            cg_xr<<<grid, CT, 0, c.stream>>>(op, N, nl, k0, it, dsig.d(), dsigp.d(), X, R.d(),
                                            pbuf(it), pA.d(), pB.d(), nparts, ss, dact.as<int>());
            c.check_launch();
            }
            if (fixed_iters <= 0 && (it % 8) == 7) {
                HYDOT_CUDA(cudaMemcpyAsync(hst.data(), ss, size_t(nb) * sizeof(SysState),
                                           cudaMemcpyDeviceToHost, c.stream));
                c.sync();
                std::vector<int> still;
                for (int k : active)
                    if (!hst[size_t(k)].done) still.push_back(k);
                if (still.empty()) {
                    ++it;
                    break;
                }
                if (still.size() < active.size()) {
                    active.swap(still);
                    HYDOT_CUDA(cudaMemcpyAsync(dact.as<void>(), active.data(),
                                               active.size() * sizeof(int), cudaMemcpyHostToDevice,
                                               c.stream));
                    c.sync();  // host vector is reused
                }
            }
        }
        if (fixed_iters <= 0 && it >= limit) {
            // one more convergence check for systems finishing on the last step
            dim3 grid = dim3(unsigned(nparts), unsigned(active.size()));
            if (ztpsmem)
                cgzt_pa<NSR, 4><<<grid, ZT, ztpsmem, c.stream>>>(zg, N, nl, k0, it, dsig.d(), dsigp.d(), R.d(),
                                                         pbuf(it + 1), pbuf(it), pA.d(), pB.d(), nparts, ss,
                                                         tol, 0, dact.as<int>());
            else if (zsmem)
                ZSEL(cgz_pa)<<<grid, ZT, zsmem, c.stream>>>(zg, N, nl, k0, it, dsig.d(), dsigp.d(), R.d(),
                                                      pbuf(it + 1), pbuf(it), pA.d(), pB.d(), nparts, ss,
                                                      tol, 0, dact.as<int>());
            else
                cg_pa<<<grid, CT, 0, c.stream>>>(op, N, nl, k0, it, dsig.d(), dsigp.d(), R.d(),
                                                pbuf(it + 1), pbuf(it), pA.d(), pB.d(), nparts, ss,
                                                tol, 0, dact.as<int>());
            c.check_launch();
        }
        {
            dim3 gf = dim3(unsigned(std::min<int64_t>((N + 255) / 256, 1024)), unsigned(nb));
            cg_finish<<<gf, CT, 0, c.stream>>>(N, nl, k0, it, X, dinv.d(), pB.d(), nparts, ss);
            c.check_launch();
        }
        if (stats) {
            std::vector<SysState> hs(static_cast<size_t>(nb));
            HYDOT_CUDA(cudaMemcpyAsync(hs.data(), ss, size_t(nb) * sizeof(SysState),
                                       cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            for (int k = 0; k < nb; ++k) {
                stats->iters[size_t(k0 + k)] = hs[size_t(k)].iters;
                stats->relres[size_t(k0 + k)] = hs[size_t(k)].relres;
            }
        }
    }
    c.sync();
}

void check_grid(int nx, int ny, int nz) {
    if (nx < 3 || ny < 3 || nz < 2) throw std::invalid_argument("fields_solve: bad grid");
}

}  // namespace

void apply7(Ctx& c, const hydot_grid7& g, double sigma, double sigmap, const double* x, double* y) {
    const int64_t N = int64_t(g.nx) * g.ny * g.nz;
    Op7 op{make_stencil(g)};
    int blocks = int(std::min<int64_t>((N + 255) / 256, int64_t(c.num_sms) * 16));
    apply_k<<<blocks, 256, 0, c.stream>>>(op, N, sigma, sigmap, x, y);
    c.check_launch();
}

void fields_solve(Ctx& c, const hydot_grid7& g, int nl, const double* sigma, const double* sigmap,
                  const double* inv_D, const int64_t* rhs_vertex, int n_rhs, double tol, int max_iter,
                  int fixed_iters, double* out, CGStats* stats) {
    check_grid(g.nx, g.ny, g.nz);
    if (g.h <= 0) throw std::invalid_argument("fields_solve: bad grid");
    if (nl <= 0 || n_rhs <= 0) throw std::invalid_argument("compute_fields: no wavelengths");
    const int64_t N = int64_t(g.nx) * g.ny * g.nz;
    std::vector<int64_t> ridx(size_t(n_rhs) * 8, -1);
    std::vector<double> rw(size_t(n_rhs) * 8, 0.0), b2(size_t(n_rhs), 1.0);
    for (int s = 0; s < n_rhs; ++s) {
        int64_t v = rhs_vertex[s];
        if (v < 0 || v >= N) throw std::invalid_argument("point_source_vector: point outside domain");
        int ix = int(v % g.nx), iy = int((v / g.nx) % g.ny);
        if (ix == 0 || ix == g.nx - 1 || iy == 0 || iy == g.ny - 1)
            throw std::invalid_argument("source support falls entirely on the Dirichlet boundary");
        ridx[size_t(s) * 8] = v;
        rw[size_t(s) * 8] = 1.0;
    }
    cg_batch(c, Op7{make_stencil(g)}, N, nl, sigma, sigmap, inv_D, ridx, rw, b2, n_rhs, tol, max_iter,
             fixed_iters, out, stats);
}

// fields of the perturbed medium: sigma_l + dsig_l mu(v) per vertex (mu, dsig
// device arrays; the vertex-parallel kernels -- this is not the hot path)
void fields_solve_var(Ctx& c, const hydot_grid7& g, int nl, const double* sigma, const double* sigmap,
                      const double* inv_D, const double* dsig_dev, const double* mu_dev, const int64_t* rhs_vertex,
                      int n_rhs, double tol, int max_iter, int fixed_iters, double* out, CGStats* stats) {
    check_grid(g.nx, g.ny, g.nz);
    if (g.h <= 0) throw std::invalid_argument("fields_solve: bad grid");
    if (nl <= 0 || n_rhs <= 0) throw std::invalid_argument("compute_fields: no wavelengths");
    const int64_t N = int64_t(g.nx) * g.ny * g.nz;
    std::vector<int64_t> ridx(size_t(n_rhs) * 8, -1);
    std::vector<double> rw(size_t(n_rhs) * 8, 0.0), b2(size_t(n_rhs), 1.0);
    for (int s = 0; s < n_rhs; ++s) {
        int64_t v = rhs_vertex[s];
        if (v < 0 || v >= N) throw std::invalid_argument("point_source_vector: point outside domain");
        int ix = int(v % g.nx), iy = int((v / g.nx) % g.ny);
        if (ix == 0 || ix == g.nx - 1 || iy == 0 || iy == g.ny - 1)
            throw std::invalid_argument("source support falls entirely on the Dirichlet boundary");
        ridx[size_t(s) * 8] = v;
        rw[size_t(s) * 8] = 1.0;
    }
    cg_batch(c, Op7Var{make_stencil(g), mu_dev, dsig_dev}, N, nl, sigma, sigmap, inv_D, ridx, rw, b2, n_rhs, tol,
             max_iter, fixed_iters, out, stats);
}

// ------------------------------------------------------------- FEM mode --
namespace {

constexpr double kGaussPt = 0.57735026918962576451;  // grid.cpp:14

// element stiffness / mass (grid.cpp:39-64) and face mass (:67-88) by the
// reference's 2x2x2 (2x2) Gauss rule, same summation order
void fem_element_matrices(double hx, double hy, double hz, double Ke[64], double Me[64], double Re[16]) {
    for (int e = 0; e < 64; ++e) Ke[e] = Me[e] = 0.0;
    for (int e = 0; e < 16; ++e) Re[e] = 0.0;
    const double detJ = hx * hy * hz / 8.0;
    const double ih[3] = {2.0 / hx, 2.0 / hy, 2.0 / hz};
    auto sgn = [](int a, int bit) { return (a & bit) ? 1.0 : -1.0; };
    for (int qx = 0; qx < 2; ++qx)
        for (int qy = 0; qy < 2; ++qy)
            for (int qz = 0; qz < 2; ++qz) {
                const double xi = qx ? kGaussPt : -kGaussPt, eta = qy ? kGaussPt : -kGaussPt,
                             zeta = qz ? kGaussPt : -kGaussPt;
                double N[8], G[8][3];
                for (int a = 0; a < 8; ++a) {
                    const double sx = sgn(a, 1), sy = sgn(a, 2), sz = sgn(a, 4);
                    N[a] = 0.125 * (1 + sx * xi) * (1 + sy * eta) * (1 + sz * zeta);
                    G[a][0] = 0.125 * sx * (1 + sy * eta) * (1 + sz * zeta) * ih[0];
                    G[a][1] = 0.125 * sy * (1 + sx * xi) * (1 + sz * zeta) * ih[1];
                    G[a][2] = 0.125 * sz * (1 + sx * xi) * (1 + sy * eta) * ih[2];
                }
                for (int a = 0; a < 8; ++a)
                    for (int b = 0; b < 8; ++b) {
                        const double dot = G[a][0] * G[b][0] + G[a][1] * G[b][1] + G[a][2] * G[b][2];
                        Ke[a * 8 + b] += detJ * dot;
                        Me[a * 8 + b] += detJ * N[a] * N[b];
                    }
            }
    const double detF = hx * hy / 4.0;
    for (int qx = 0; qx < 2; ++qx)
        for (int qy = 0; qy < 2; ++qy) {
            const double xi = qx ? kGaussPt : -kGaussPt, eta = qy ? kGaussPt : -kGaussPt;
            for (int a = 0; a < 4; ++a) {
                const double Na = 0.25 * (1 + sgn(a, 1) * xi) * (1 + sgn(a, 2) * eta);
                for (int b = 0; b < 4; ++b) {
                    const double Nb = 0.25 * (1 + sgn(b, 1) * xi) * (1 + sgn(b, 2) * eta);
                    Re[a * 4 + b] += detF * Na * Nb;
                }
            }
        }
}

struct FemSetup {
    OpFem op{};
    DBuf em;
    int64_t N = 0;
    double hx = 0, hy = 0, hz = 0;
};

FemSetup fem_setup(Ctx& c, const hydot_grid_geom& g) {
    check_grid(g.nx, g.ny, g.nz);
    if (g.Lx <= 0 || g.Ly <= 0 || g.Lz <= 0) throw std::invalid_argument("build_grid: extents must be positive");
    FemSetup f;
    f.hx = 2 * g.Lx / (g.nx - 1);
    f.hy = 2 * g.Ly / (g.ny - 1);
    f.hz = g.Lz / (g.nz - 1);
    double h[144];
    fem_element_matrices(f.hx, f.hy, f.hz, h, h + 64, h + 128);
    f.em = dalloc(c, 144);
    HYDOT_CUDA(cudaMemcpyAsync(f.em.d(), h, sizeof h, cudaMemcpyHostToDevice, c.stream));
    c.sync();
    f.op = OpFem{g.nx, g.ny, g.nz, 1.0f / float(g.nx), 1.0f / float(g.ny), f.em.d()};
    f.N = int64_t(g.nx) * g.ny * g.nz;
    return f;
}

}  // namespace

void fem_element_host(double hx, double hy, double hz, double Ke[64], double Me[64], double Re[16]) {
    fem_element_matrices(hx, hy, hz, Ke, Me, Re);
}

void apply_fem(Ctx& c, const hydot_grid_geom& g, double sigma, double sigmap, const double* x, double* y) {
    FemSetup f = fem_setup(c, g);
    int blocks = int(std::min<int64_t>((f.N + 255) / 256, int64_t(c.num_sms) * 16));
    apply_k<<<blocks, 256, 0, c.stream>>>(f.op, f.N, sigma, sigmap, x, y);
    c.check_launch();
    c.sync();
}

// source_rhs (born.cpp:27-35): trilinear point_source_vector (grid.cpp:212-237)
// with the Dirichlet vertices zeroed -- 8 (vertex, weight) pairs per point
// (vertex -1 = no entry) and the squared norm of each source vector
void fem_point_weights(const hydot_grid_geom& g, const double* points, int n_pts, std::vector<int64_t>& ridx,
                       std::vector<double>& rw, std::vector<double>& b2) {
    const double hx = 2 * g.Lx / (g.nx - 1), hy = 2 * g.Ly / (g.ny - 1), hz = g.Lz / (g.nz - 1);
    ridx.assign(size_t(n_pts) * 8, -1);
    rw.assign(size_t(n_pts) * 8, 0.0);
    b2.assign(size_t(n_pts), 0.0);
    auto clamp_cell = [](double t, int ncells) {
        int cc = int(std::floor(t));
        return cc < 0 ? 0 : (cc > ncells - 1 ? ncells - 1 : cc);
    };
    for (int s = 0; s < n_pts; ++s) {
        const double rx = points[3 * s], ry = points[3 * s + 1], rz = points[3 * s + 2];
        if (!(rx >= -g.Lx && rx <= g.Lx && ry >= -g.Ly && ry <= g.Ly && rz >= 0.0 && rz <= g.Lz))
            throw std::invalid_argument("point_source_vector: point outside domain");
        const double tx = (rx + g.Lx) / hx, ty = (ry + g.Ly) / hy, tz = rz / hz;
        const int cx = clamp_cell(tx, g.nx - 1), cy = clamp_cell(ty, g.ny - 1), cz = clamp_cell(tz, g.nz - 1);
        const double xi = 2 * (tx - cx) - 1, eta = 2 * (ty - cy) - 1, zeta = 2 * (tz - cz) - 1;
        double nrm2 = 0.0;
        for (int a = 0; a < 8; ++a) {
            const int jx = cx + (a & 1), jy = cy + ((a >> 1) & 1), jz = cz + ((a >> 2) & 1);
            const double sx = (a & 1) ? 1.0 : -1.0, sy = (a & 2) ? 1.0 : -1.0, sz = (a & 4) ? 1.0 : -1.0;
            double w = 0.125 * (1 + sx * xi) * (1 + sy * eta) * (1 + sz * zeta);
            if (jx == 0 || jx == g.nx - 1 || jy == 0 || jy == g.ny - 1) w = 0.0;
            ridx[size_t(s) * 8 + a] = w != 0.0 ? (int64_t(jz) * g.ny + jy) * g.nx + jx : -1;
            rw[size_t(s) * 8 + a] = w;
            nrm2 += w * w;
        }
        if (nrm2 == 0.0) throw std::invalid_argument("source support falls entirely on the Dirichlet boundary");
        b2[size_t(s)] = nrm2;
    }
}

void fields_solve_fem(Ctx& c, const hydot_grid_geom& g, int nl, const double* sigma, const double* sigmap,
                      const double* inv_D, const double* points, int n_pts, double tol, int max_iter,
                      int fixed_iters, double* out, CGStats* stats) {
    if (nl <= 0 || n_pts <= 0) throw std::invalid_argument("compute_fields: no wavelengths");
    FemSetup f = fem_setup(c, g);
    std::vector<int64_t> ridx;
    std::vector<double> rw, b2;
    fem_point_weights(g, points, n_pts, ridx, rw, b2);
    cg_batch(c, f.op, f.N, nl, sigma, sigmap, inv_D, ridx, rw, b2, n_pts, tol, max_iter, fixed_iters, out, stats);
}

}  // namespace hydot
