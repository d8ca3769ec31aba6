// gmres.cu -- the reference's recycled shifted-family solver on the device
// (krylov::solve_family, /root/reference/proj/src/krylov.cpp:21-463) on the
// reference's trilinear-FEM operator (grid.cpp:112-174).
//
// Per right-hand side b (a point source, born.cpp:27-35) and the shift family
// (sigma_j, sigma'_j), j < n_shifts (the wavelengths), in the lumped-mass
// transformed variables (transform_family, krylov.cpp:286-309):
//   Ks = D (K + sbar' R) D, Rs = D R D, D = M^-1/2, A_j = Ks + sigma_j I + (sigma'_j - sbar') Rs
//   phase 1  (multishift_gmres :45-104) one Arnoldi basis of Ks per rhs, per-shift
//            least squares, convergence test every 10 steps
//   deflation (harmonic_ritz :106-168, build_deflation_basis :170-213) k smallest
//            harmonic Ritz vectors, K U = C with C orthonormal; per shift the
//            Gram/Cholesky update C_j = C'_j F_j^-1 (ShiftedDeflation :215-283),
//            QR of C'_j when the Cholesky fails (or explicit_qr_update)
//   phase 2  (augmented_gmres :311-398) deflated GMRES(m - k) per shift from the
//            phase-1 solution, with restarts
// B200 design: every system of a batch (rhs x shift) advances in lockstep;
// one launch per operation covers all systems of the batch:
//   op_k    the FEM operator, matrix-free, per-system shifts, optional residual
//           form b - A x with the squared-norm partials fused
//   dot_k   inner products of a vector with a system's column set (deflation
//           columns of its rhs + its own Krylov basis), the vector slice staged
//           in shared memory, one warp per column; grid ordered systems-fastest
//           so the systems of one rhs read the same deflation slice from L2
//   upd_k   vector -= (column set) * coefficients, squared-norm partials fused
//   small per-system kernels (one thread per system): Hessenberg columns,
//           Givens least squares, F_j, the deflation coefficients
// Orthogonalisation is classical Gram-Schmidt with one re-orthogonalisation
// pass (CGS2: two passes over the basis per pass pair, bandwidth-friendly)
// instead of the reference's modified Gram-Schmidt with refinement (same
// result to rounding; krylov.cpp:21-29).  The pencil Tbar^T Tbar z = theta
// T_n^T z is solved in its symmetric-definite form: T_n is the Arnoldi
// projection of the symmetric positive definite Ks (K, R symmetric;
// grid.cpp:112-174), so T_n^T is symmetrised, factored by Cholesky and the
// reduced symmetric problem diagonalised by parallel cyclic Jacobi; when the
// Cholesky fails the reference's pencil shift eps*|T_n|_F I is applied
// (krylov.cpp:117-121).  Results match the oracle (oracle/krylov_oracle.cpp)
// to the solve tolerance, not bitwise (tests/test_gpu_gmres.py).
#include <cmath>
#include <cstdio>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.h"

namespace hydot {

namespace {

constexpr int kT = 256;           // threads of the streaming kernels
constexpr int kDotL = 2048;       // vector slice per dot_k CTA
constexpr int kUpdRows = 4;       // rows per thread in upd_k / op_k
constexpr int kMaxCols = 256;     // columns of one dot / update (deflation + basis)
constexpr int kMaxSteps = 200;    // Arnoldi steps / restart length supported

__device__ __forceinline__ void fdivmod_g(unsigned i, unsigned d, float inv_d, unsigned& q, unsigned& r) {
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

struct FemGeo {
    int nx, ny, nz;
    float inv_nx, inv_ny;
    const double* em;  // Ke (64) | Me (64) | Re (16), grid.cpp element order
};

__device__ __forceinline__ void coords(const FemGeo& g, int64_t i, int& ix, int& iy, int& iz) {
    unsigned q1, ux, uy, uz;
    fdivmod_g(unsigned(i), unsigned(g.nx), g.inv_nx, q1, ux);
    fdivmod_g(q1, unsigned(g.ny), g.inv_ny, uz, uy);
    ix = int(ux);
    iy = int(uy);
    iz = int(uz);
}

// lumped mass, K and R diagonals: dinv = M^-1/2, kd = K_ii, rd = R_ii
__global__ void fem_diag_k(FemGeo g, int64_t N, double* dinv, double* kd, double* rd) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N) return;
    int ix, iy, iz;
    coords(g, i, ix, iy, iz);
    auto dir = [&](int jx, int jy) { return jx == 0 || jx == g.nx - 1 || jy == 0 || jy == g.ny - 1; };
    double m = 0.0, k = 0.0, r = 0.0;
    for (int oz = -1; oz <= 0; ++oz) {
        const int cz = iz + oz;
        if (cz < 0 || cz > g.nz - 2) continue;
        for (int oy = -1; oy <= 0; ++oy) {
            const int cy = iy + oy;
            if (cy < 0 || cy > g.ny - 2) continue;
            for (int ox = -1; ox <= 0; ++ox) {
                const int cx = ix + ox;
                if (cx < 0 || cx > g.nx - 2) continue;
                const int a = (ox ? 1 : 0) | (oy ? 2 : 0) | (oz ? 4 : 0);
                for (int b = 0; b < 8; ++b) m += g.em[64 + a * 8 + b];
                k += g.em[a * 8 + a];
            }
        }
    }
    if (dir(ix, iy)) k = 1.0;
    if (iz == 0 || iz == g.nz - 1)
        for (int oy = -1; oy <= 0; ++oy) {
            const int cy = iy + oy;
            if (cy < 0 || cy > g.ny - 2) continue;
            for (int ox = -1; ox <= 0; ++ox) {
                const int cx = ix + ox;
                if (cx < 0 || cx > g.nx - 2) continue;
                const int a = (ox ? 1 : 0) | (oy ? 2 : 0);
                r += g.em[128 + a * 4 + a];
            }
        }
    dinv[i] = 1.0 / sqrt(m);
    if (kd) kd[i] = k;
    if (rd) rd[i] = r;
}

struct OpArgs {
    const int* act;       // active slot list (blockIdx.y)
    const double* x;      // x of slot s at x + s * xs
    int64_t xs;
    double* y;
    int64_t ys;
    double ck;            // K coefficient (1, or 0 for Rs alone)
    const double* cs;     // per-slot identity shift (nullable -> cs0)
    const double* cr;     // per-slot R coefficient (nullable -> cr0)
    double cs0, cr0;
    const double* xscale; // per-slot scale of x (nullable)
    const double* px;     // right preconditioner P^-1 (nullable)
    const double* b;      // residual form: y = b - A x, b of slot s at b + bslot[s] * bs
    const int* bslot;
    int64_t bs;
    double* part;         // residual form: squared-norm partials [a * gridDim.x + tile]
};

// y_s = D (ck K + cr_s R) D u + cs_s u,  u = xscale_s * px (.) x_s
__global__ void __launch_bounds__(kT) op_k(FemGeo g, int64_t N, OpArgs o) {
    __shared__ double red[kT / 32];
    const int a = blockIdx.y;
    const int s = o.act[a];
    const double* x = o.x + int64_t(s) * o.xs;
    double* y = o.y + int64_t(s) * o.ys;
    const double sc = o.xscale ? o.xscale[s] : 1.0;
    const double cs = o.cs ? o.cs[s] : o.cs0;
    const double cr = o.cr ? o.cr[s] : o.cr0;
    const double* dinv = g.em + 144;  // dinv follows the element matrices
    auto u = [&](int64_t j) {
        const double v = sc * x[j];
        return o.px ? o.px[j] * v : v;
    };
    double acc = 0.0;
    for (int r = 0; r < kUpdRows; ++r) {
        const int64_t i = (int64_t(blockIdx.x) * kUpdRows + r) * kT + threadIdx.x;
        if (i >= N) break;
        int ix, iy, iz;
        coords(g, i, ix, iy, iz);
        auto dir = [&](int jx, int jy) { return jx == 0 || jx == g.nx - 1 || jy == 0 || jy == g.ny - 1; };
        const bool di = dir(ix, iy);
        double kx = 0.0;
        if (o.ck != 0.0) {
            if (di) {
                kx = dinv[i] * u(i);
            } else {
                for (int oz = -1; oz <= 0; ++oz) {
                    const int cz = iz + oz;
                    if (cz < 0 || cz > g.nz - 2) continue;
                    for (int oy = -1; oy <= 0; ++oy) {
                        const int cy = iy + oy;
                        if (cy < 0 || cy > g.ny - 2) continue;
                        for (int ox = -1; ox <= 0; ++ox) {
                            const int cx = ix + ox;
                            if (cx < 0 || cx > g.nx - 2) continue;
                            const int aa = (ox ? 1 : 0) | (oy ? 2 : 0) | (oz ? 4 : 0);
#pragma unroll
                            for (int b = 0; b < 8; ++b) {
                                const int jx = cx + (b & 1), jy = cy + ((b >> 1) & 1), jz = cz + ((b >> 2) & 1);
                                if (!dir(jx, jy)) {
                                    const int64_t j = (int64_t(jz) * g.ny + jy) * g.nx + jx;
                                    kx += g.em[aa * 8 + b] * (dinv[j] * u(j));
                                }
                            }
                        }
                    }
                }
            }
        }
        double rx = 0.0;
        if (cr != 0.0 && (iz == 0 || iz == g.nz - 1)) {
            for (int oy = -1; oy <= 0; ++oy) {
                const int cy = iy + oy;
                if (cy < 0 || cy > g.ny - 2) continue;
                for (int ox = -1; ox <= 0; ++ox) {
                    const int cx = ix + ox;
                    if (cx < 0 || cx > g.nx - 2) continue;
                    const int aa = (ox ? 1 : 0) | (oy ? 2 : 0);
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int64_t j = (int64_t(iz) * g.ny + cy + ((b >> 1) & 1)) * g.nx + cx + (b & 1);
                        rx += g.em[128 + aa * 4 + b] * (dinv[j] * u(j));
                    }
                }
            }
        }
        double v = dinv[i] * (o.ck * kx + cr * rx) + cs * u(i);
        if (o.b) {
            v = o.b[int64_t(o.bslot[s]) * o.bs + i] - v;
            acc += v * v;
        }
        y[i] = v;
    }
    if (o.part) {
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < kT / 32; ++w) t += red[w];
            o.part[int64_t(a) * gridDim.x + blockIdx.x] = t;
        }
    }
}

// Column sets: set 1 = the deflation columns of the slot's rhs (nd1[s]
// columns at d1 + dset[s] * d1s, column stride N); set 2 = the slot's own
// basis columns [c2a, c2a + n2) at v2 + s * v2s.
struct Cols {
    const int* act;
    const double* d1;
    int64_t d1s;
    const int* dset;  // slot -> deflation set (nullable: no set 1)
    const int* nd1;   // slot -> its column count
    const double* v2;
    int64_t v2s;
    int c2a, n2;
    int ncm;          // row stride of the per-slot coefficient / result rows
    __device__ __forceinline__ int n1(int s) const { return dset ? nd1[s] : 0; }
    __device__ __forceinline__ const double* col(int s, int c, int64_t N) const {
        const int k1 = n1(s);
        if (c < k1) return d1 + int64_t(dset[s]) * d1s + int64_t(c) * N;
        return v2 + int64_t(s) * v2s + int64_t(c2a + c - k1) * N;
    }
};

// part[(a * ncm + c) * nsl + sl] = col_c[slice] . w[slice]   (grid: a fastest, slice)
__global__ void __launch_bounds__(kT) dot_k(int64_t N, Cols cs, const double* w, int64_t ws, int64_t woff,
                                           double* part, int nsl) {
    __shared__ double wsh[kDotL];
    const int a = blockIdx.x, sl = blockIdx.y;
    const int s = cs.act[a];
    const int64_t j0 = int64_t(sl) * kDotL;
    const int len = int(min(int64_t(kDotL), N - j0));
    const double* wp = w + int64_t(s) * ws + woff + j0;
    for (int t = threadIdx.x; t < len; t += kT) wsh[t] = wp[t];
    __syncthreads();
    const int nc = cs.n1(s) + cs.n2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c = warp; c < nc; c += kT / 32) {
        const double* b = cs.col(s, c, N) + j0;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        int t = lane;
        for (; t + 96 < len; t += 128) {
            acc0 += b[t] * wsh[t];
            acc1 += b[t + 32] * wsh[t + 32];
            acc2 += b[t + 64] * wsh[t + 64];
            acc3 += b[t + 96] * wsh[t + 96];
        }
        for (; t < len; t += 32) acc0 += b[t] * wsh[t];
        double acc = (acc0 + acc1) + (acc2 + acc3);
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) part[(int64_t(a) * cs.ncm + c) * nsl + sl] = acc;
    }
}

// out[a * ncm + c] = sum over slices (fixed order)
__global__ void red_k(int nact, int ncm, const int* ncol_of_a, const double* part, int nsl, double* out) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= int64_t(nact) * ncm) return;
    const int a = int(t / ncm), c = int(t % ncm);
    if (ncol_of_a && c >= ncol_of_a[a]) return;
    const double* p = part + t * nsl;
    double s = 0.0;
    for (int i = 0; i < nsl; ++i) s += p[i];
    out[t] = s;
}

// target_s += sum_c coef[a * ncm + c] col_c  (set-2 columns times rs2 row
// scale when given); nrm: squared-norm partials of the result
__global__ void __launch_bounds__(kT) upd_k(int64_t N, Cols cs, const double* coef, const double* rs2, double* tb,
                                           int64_t ts, int64_t toff, double* part) {
    __shared__ double cf[kMaxCols];
    __shared__ double red[kT / 32];
    const int a = blockIdx.x;
    const int s = cs.act[a];
    const int k1 = cs.n1(s), nc = k1 + cs.n2;
    for (int c = threadIdx.x; c < nc; c += kT) cf[c] = coef[int64_t(a) * cs.ncm + c];
    __syncthreads();
    double* t = tb + int64_t(s) * ts + toff;
    double acc = 0.0;
    const int64_t i0 = int64_t(blockIdx.y) * (kT * kUpdRows) + threadIdx.x;
#pragma unroll
    for (int r = 0; r < kUpdRows; ++r) {
        const int64_t i = i0 + int64_t(r) * kT;
        if (i >= N) break;
        double v1 = 0.0, v2 = 0.0;
        for (int c = 0; c < k1; ++c) v1 += cf[c] * cs.col(s, c, N)[i];
        const double* vb = cs.v2 + int64_t(s) * cs.v2s + int64_t(cs.c2a) * N + i;
        for (int c = 0; c < cs.n2; ++c) v2 += cf[k1 + c] * vb[int64_t(c) * N];
        if (rs2) v2 *= rs2[i];
        const double v = t[i] + (v1 + v2);
        t[i] = v;
        acc += v * v;
    }
    if (part) {
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double q = 0.0;
            for (int w = 0; w < kT / 32; ++w) q += red[w];
            part[int64_t(a) * gridDim.y + blockIdx.y] = q;
        }
    }
}

// y_s = x_s * scale[s]  (vectors at stride xs / ys, offsets xo / yo)
__global__ void scale_k(int64_t N, const int* act, const double* x, int64_t xs, int64_t xo, double* y, int64_t ys,
                        int64_t yo, const double* scale) {
    const int s = act[blockIdx.y];
    const double f = scale[s];
    const double* xp = x + int64_t(s) * xs + xo;
    double* yp = y + int64_t(s) * ys + yo;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += int64_t(gridDim.x) * blockDim.x)
        yp[i] = f * xp[i];
}

// bs = dinv (.) b; the per-rhs squared-norm partials
__global__ void bscale_k(int64_t N, const double* b, const double* dinv, double* bs, double* part) {
    __shared__ double red[kT / 32];
    const int r = blockIdx.y;
    double acc = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < N; i += int64_t(gridDim.x) * kT) {
        const double v = dinv[i] * b[int64_t(r) * N + i];
        bs[int64_t(r) * N + i] = v;
        acc += v * v;
    }
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double q = 0.0;
        for (int w = 0; w < kT / 32; ++w) q += red[w];
        part[int64_t(r) * gridDim.x + blockIdx.x] = q;
    }
}

// squared norms from partials: out[s] = sqrt(sum part[a * np .. ]) for act[a] = s
__global__ void norm_k(int nact, const int* act, const double* part, int np, double* out) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    double q = 0.0;
    for (int i = 0; i < np; ++i) q += part[int64_t(a) * np + i];
    out[act[a]] = sqrt(q);
}

__device__ __forceinline__ void givens(double f, double g, double& c, double& s, double& r) {
    if (g == 0.0) {
        c = 1.0;
        s = 0.0;
        r = f;
        return;
    }
    r = hypot(f, g);
    c = f / r;
    s = g / r;
}

// ---------------------------------------------------------------- phase 1 --
// coef row = -h (h = dot results, i + 1 values); accumulates H column i
__global__ void p1_coef_k(int nact, const int* act, int ncm, const double* h, double* coef, double* T, int64_t Ts,
                          int ldT, int i, int first) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    const int p = act[a];
    double* tc = T + int64_t(p) * Ts + int64_t(i) * ldT;
    for (int c = 0; c <= i; ++c) {
        const double v = h[int64_t(a) * ncm + c];
        coef[int64_t(a) * ncm + c] = -v;
        tc[c] = first ? v : tc[c] + v;
    }
}

// H(i+1, i) = |w|; breakdown flag; 1 / |w|
__global__ void p1_norm_k(int nact, const int* act, const double* nrm, double* T, int64_t Ts, int ldT, int i,
                          const double* bnorm, double* inv_h, int* flag) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    const int p = act[a];
    const double hn = nrm[p];
    T[int64_t(p) * Ts + int64_t(i) * ldT + i + 1] = hn;
    const bool bd = hn <= 1e-14 * bnorm[p];
    flag[p] = bd ? 1 : 0;
    inv_h[p] = bd ? 0.0 : 1.0 / hn;
}

// Givens least squares of min |beta e1 - (Tbar_s + sigma [I; 0]) y| (the
// reference's hessenberg_ls, krylov.cpp:33-41); R kept in rs (upper packed by
// columns) when y is wanted.  Returns the residual norm.
__device__ double hess_ls(const double* T, int ldT, int s, double sigma, double beta, double* rs, double* g,
                          double* cs_, double* sn_, double* y) {
    for (int i = 0; i <= s; ++i) g[i] = 0.0;
    g[0] = beta;
    for (int c = 0; c < s; ++c) {
        double* col = rs + int64_t(c) * (c + 1) / 2;  // rows 0..c of column c
        double hnext = T[int64_t(c) * ldT + c + 1];
        for (int r = 0; r <= c; ++r) col[r] = T[int64_t(c) * ldT + r] + (r == c ? sigma : 0.0);
        for (int r = 0; r < c; ++r) {
            const double t0 = cs_[r] * col[r] + sn_[r] * col[r + 1];
            col[r + 1] = -sn_[r] * col[r] + cs_[r] * col[r + 1];
            col[r] = t0;
        }
        double cc, ss, rr;
        givens(col[c], hnext, cc, ss, rr);
        cs_[c] = cc;
        sn_[c] = ss;
        col[c] = rr;
        g[c + 1] = -ss * g[c];
        g[c] = cc * g[c];
    }
    if (y) {
        for (int r = s - 1; r >= 0; --r) {
            double t = g[r];
            for (int c = r + 1; c < s; ++c) t -= rs[int64_t(c) * (c + 1) / 2 + r] * y[c];
            y[r] = t / rs[int64_t(r) * (r + 1) / 2 + r];
        }
    }
    return fabs(g[s]);
}

// per (point, shift): the least-squares residual (conv test) or solution (Y, relres)
__global__ void p1_ls_k(int npts, const int* pts, int nsh, const double* sig, const double* T, int64_t Ts, int ldT,
                        const int* steps, const double* bnorm, double tol, double* scratch, int64_t scr_s,
                        int* conv, double* Y, int64_t Ys, int ldY, double* relres) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= npts * nsh) return;
    const int a = t / nsh, j = t % nsh;
    const int p = pts[a];
    const int s = steps[p];
    double* sc = scratch + int64_t(t) * scr_s;
    double* g = sc;
    double* cs_ = g + (s + 1);
    double* sn_ = cs_ + s;
    double* rs = sn_ + s;
    double* y = Y ? Y + int64_t(p) * Ys + int64_t(j) * ldY : nullptr;
    const double res = hess_ls(T + int64_t(p) * Ts, ldT, s, sig[j], bnorm[p], rs, g, cs_, sn_, y);
    if (conv) conv[int64_t(a) * nsh + j] = (res / bnorm[p] <= tol) ? 1 : 0;
    if (relres) relres[int64_t(p) * nsh + j] = res / bnorm[p];
}

// ------------------------------------------------------- harmonic Ritz --
// One CTA per rhs: Tbar^T Tbar z = theta sym(T_n) z as a symmetric-definite
// pencil (see the file header), k smallest |theta|, unit columns.
__global__ void __launch_bounds__(kT) hritz_k(const int* steps, const double* T, int64_t Ts, int ldT, int kreq,
                                             int ld, double* scratch, int64_t scr_s, double* Z, int64_t Zs,
                                             double* theta, int* kout, int* pencil) {
    const int p = blockIdx.x;
    const int s = steps[p];
    const int k = min(kreq, s);
    const double* Tp = T + int64_t(p) * Ts;
    double* A = scratch + int64_t(p) * scr_s;
    double* L = A + int64_t(ld) * ld;
    double* X = L + int64_t(ld) * ld;
    double* C = X + int64_t(ld) * ld;
    double* W = C + int64_t(ld) * ld;
    __shared__ double fro;
    __shared__ int fail, rot;
    __shared__ double pc[kMaxSteps / 2 + 1], ps[kMaxSteps / 2 + 1];
    __shared__ int pp[kMaxSteps / 2 + 1], pq[kMaxSteps / 2 + 1];
    auto at = [&](double* M, int i, int j) -> double& { return M[int64_t(j) * ld + i]; };
    const int tid = threadIdx.x;
    for (int e = tid; e < s * s; e += kT) {
        const int i = e % s, j = e / s;
        double v = 0.0;
        for (int r = 0; r <= s; ++r) v += Tp[int64_t(i) * ldT + r] * Tp[int64_t(j) * ldT + r];
        at(A, i, j) = v;
    }
    if (tid == 0) {
        double f = 0.0;
        for (int j = 0; j < s; ++j)
            for (int i = 0; i < s; ++i) f += Tp[int64_t(j) * ldT + i] * Tp[int64_t(j) * ldT + i];
        fro = sqrt(f);
    }
    __syncthreads();
    for (int attempt = 0; attempt < 2; ++attempt) {
        const double shift = attempt ? 2.220446049250313e-16 * fro : 0.0;
        for (int e = tid; e < s * s; e += kT) {
            const int i = e % s, j = e / s;
            at(L, i, j) = 0.5 * (Tp[int64_t(j) * ldT + i] + Tp[int64_t(i) * ldT + j]) + (i == j ? shift : 0.0);
        }
        if (tid == 0) fail = 0;
        __syncthreads();
        for (int j = 0; j < s; ++j) {  // right-looking Cholesky, lower
            if (tid == 0) {
                const double d = at(L, j, j);
                if (!(d > 0.0)) fail = 1;
                at(L, j, j) = d > 0.0 ? sqrt(d) : 1.0;
            }
            __syncthreads();
            const double ljj = at(L, j, j);
            for (int i = j + 1 + tid; i < s; i += kT) at(L, i, j) /= ljj;
            __syncthreads();
            for (int e = tid; e < (s - j - 1) * (s - j - 1); e += kT) {
                const int i = j + 1 + e % (s - j - 1), c = j + 1 + e / (s - j - 1);
                if (c <= i) at(L, i, c) -= at(L, i, j) * at(L, c, j);
            }
            __syncthreads();
        }
        if (!fail) break;
        if (tid == 0) pencil[p] = 1;
        __syncthreads();
    }
    if (fail) {
        if (tid == 0) kout[p] = 0;
        return;
    }
    // X = L^-1 A (column per thread), C = L^-1 X^T, symmetrised
    for (int j = tid; j < s; j += kT)
        for (int i = 0; i < s; ++i) {
            double v = at(A, i, j);
            for (int t = 0; t < i; ++t) v -= at(L, i, t) * at(X, t, j);
            at(X, i, j) = v / at(L, i, i);
        }
    __syncthreads();
    for (int j = tid; j < s; j += kT)
        for (int i = 0; i < s; ++i) {
            double v = at(X, j, i);
            for (int t = 0; t < i; ++t) v -= at(L, i, t) * at(W, t, j);
            at(W, i, j) = v / at(L, i, i);
        }
    __syncthreads();
    for (int e = tid; e < s * s; e += kT) {
        const int i = e % s, j = e / s;
        at(C, i, j) = 0.5 * (at(W, i, j) + at(W, j, i));
    }
    __syncthreads();
    for (int e = tid; e < s * s; e += kT) {
        const int i = e % s, j = e / s;
        at(W, i, j) = i == j ? 1.0 : 0.0;
    }
    __syncthreads();
    // parallel cyclic Jacobi (round-robin pairs), eigenvectors in W
    const int m = s + (s & 1);
    for (int sweep = 0; sweep < 60 && s > 1; ++sweep) {
        if (tid == 0) rot = 0;
        __syncthreads();
        for (int r = 0; r < m - 1; ++r) {
            for (int q = tid; q < m / 2; q += kT) {
                const int i0 = q == 0 ? 0 : 1 + (q - 1 + r) % (m - 1);
                const int i1 = 1 + (m - 1 - q - 1 + r) % (m - 1);
                int P = min(i0, i1), Q = max(i0, i1);
                double c = 1.0, sn = 0.0;
                if (Q < s) {
                    const double apq = at(C, P, Q), app = at(C, P, P), aqq = at(C, Q, Q);
                    if (fabs(apq) > 1e-15 * sqrt(fabs(app * aqq)) && fabs(apq) > 1e-300) {
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        sn = t * c;
                        atomicExch(&rot, 1);
                    }
                } else {
                    P = Q = -1;
                }
                pp[q] = P;
                pq[q] = Q;
                pc[q] = c;
                ps[q] = sn;
            }
            __syncthreads();
            for (int e = tid; e < (m / 2) * s; e += kT) {  // columns: C J, W J
                const int q = e / s, i = e % s;
                const int P = pp[q], Q = pq[q];
                if (P < 0 || ps[q] == 0.0) continue;
                const double c = pc[q], sn = ps[q];
                const double cp = at(C, i, P), cq = at(C, i, Q);
                at(C, i, P) = c * cp - sn * cq;
                at(C, i, Q) = sn * cp + c * cq;
                const double wp = at(W, i, P), wq = at(W, i, Q);
                at(W, i, P) = c * wp - sn * wq;
                at(W, i, Q) = sn * wp + c * wq;
            }
            __syncthreads();
            for (int e = tid; e < (m / 2) * s; e += kT) {  // rows: J^T (C J)
                const int q = e / s, j = e % s;
                const int P = pp[q], Q = pq[q];
                if (P < 0 || ps[q] == 0.0) continue;
                const double c = pc[q], sn = ps[q];
                const double rp = at(C, P, j), rq = at(C, Q, j);
                at(C, P, j) = c * rp - sn * rq;
                at(C, Q, j) = sn * rp + c * rq;
            }
            __syncthreads();
        }
        if (!rot) break;
        __syncthreads();
    }
    // k smallest |theta| (stable by index), z = L^-T w, unit norm
    __shared__ int sel[kMaxSteps];
    if (tid == 0) {
        for (int c = 0; c < k; ++c) {
            int best = -1;
            for (int i = 0; i < s; ++i) {
                bool used = false;
                for (int t = 0; t < c; ++t) used |= sel[t] == i;
                if (used) continue;
                if (best < 0 || fabs(at(C, i, i)) < fabs(at(C, best, best))) best = i;
            }
            sel[c] = best;
            theta[int64_t(p) * kreq + c] = fabs(at(C, best, best));
        }
        kout[p] = k;
    }
    __syncthreads();
    for (int c = tid; c < k; c += kT) {
        double* z = Z + int64_t(p) * Zs + int64_t(c) * ld;
        const int e = sel[c];
        for (int i = s - 1; i >= 0; --i) {
            double v = at(W, i, e);
            for (int t = i + 1; t < s; ++t) v -= at(L, t, i) * z[t];
            z[i] = v / at(L, i, i);
        }
        double nz = 0.0;
        for (int i = 0; i < s; ++i) nz += z[i] * z[i];
        nz = sqrt(nz);
        if (nz > 0)
            for (int i = 0; i < s; ++i) z[i] /= nz;
    }
}

// U = Ut R^-1 (R k x k upper, ld ldr): one row per thread
__global__ void trsm_ru_k(int64_t N, int k, const double* Ut, const double* R, int ldr, double* U) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= N) return;
    double u[32];
    for (int j = 0; j < k; ++j) {
        double t = Ut[r + int64_t(j) * N];
        for (int l = 0; l < j; ++l) t -= u[l] * R[l + int64_t(j) * ldr];
        u[j] = t / R[j + int64_t(j) * ldr];
        U[r + int64_t(j) * N] = u[j];
    }
}

// Per (rhs, shift): the Gram/Cholesky update of ShiftedDeflation
// (krylov.cpp:223-235) from G = [C U RU]^T [C U RU]; writes Mc, Mu (3k x k,
// C_j = [C U RU] Mc, U_j = [C U RU] Mu); failed[t] = 1 when the Cholesky fails.
__global__ void shifted_k(int npts, const int* pts, int nsh, const double* sig, const double* spr,
                          const int* kdef, const double* G, int64_t Gs, double* Mc, double* Mu, int64_t Ms,
                          int* failed, int force_qr) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= npts * nsh) return;
    const int a = t / nsh, j = t % nsh;
    const int p = pts[a];
    const int k = kdef[p];
    const int slot = p * nsh + j;
    double* mc = Mc + int64_t(slot) * Ms;
    double* mu = Mu + int64_t(slot) * Ms;
    failed[slot] = 0;
    if (k == 0) return;
    const double sg = sig[j], sp = spr[j];
    const double* g = G + int64_t(p) * Gs;
    const int l3 = 3 * k;  // G of this rhs is 3k x 3k (ld 3k)
    auto Gb = [&](int bi, int bj, int i, int jj) { return g[int64_t(bj * k + jj) * l3 + bi * k + i]; };
    double F[32 * 33 / 2];  // upper, packed by columns
    auto f = [&](int i, int jj) -> double& { return F[jj * (jj + 1) / 2 + i]; };
    bool ok = !force_qr;
    if (ok) {
        // gram (upper part) = I + s(UtC + CtU) + s'(CtRU + RUtC) + s s'(RUtU + UtRU) + s^2 UtU + s'^2 RUtRU
        for (int jj = 0; jj < k; ++jj)
            for (int i = 0; i <= jj; ++i) {
                double v = i == jj ? 1.0 : 0.0;
                v += sg * (Gb(1, 0, i, jj) + Gb(1, 0, jj, i));
                v += sp * (Gb(0, 2, i, jj) + Gb(0, 2, jj, i));
                v += sg * sp * (Gb(2, 1, i, jj) + Gb(2, 1, jj, i));
                v += sg * sg * Gb(1, 1, i, jj);
                v += sp * sp * Gb(2, 2, i, jj);
                f(i, jj) = v;
            }
        for (int jj = 0; jj < k && ok; ++jj) {  // gram = F^T F (dpotrf 'U')
            for (int i = 0; i < jj; ++i) {
                double v = f(i, jj);
                for (int l = 0; l < i; ++l) v -= f(l, i) * f(l, jj);
                f(i, jj) = v / f(i, i);
            }
            double d = f(jj, jj);
            for (int l = 0; l < jj; ++l) d -= f(l, jj) * f(l, jj);
            if (!(d > 0.0)) ok = false;
            else f(jj, jj) = sqrt(d);
        }
    }
    if (!ok) {
        failed[slot] = 1;
        return;
    }
    // Finv (upper), then Mc = [Finv; s Finv; s' Finv], Mu = [0; Finv; 0]
    double Fi[32 * 33 / 2];
    auto fi = [&](int i, int jj) -> double& { return Fi[jj * (jj + 1) / 2 + i]; };
    for (int jj = 0; jj < k; ++jj) {
        fi(jj, jj) = 1.0 / f(jj, jj);
        for (int i = jj - 1; i >= 0; --i) {
            double v = 0.0;
            for (int l = i + 1; l <= jj; ++l) v += f(i, l) * fi(l, jj);
            fi(i, jj) = -v / f(i, i);
        }
    }
    const int nd = 3 * k;
    for (int jj = 0; jj < k; ++jj)
        for (int i = 0; i < nd; ++i) {
            const int bi = i / k, ii = i % k;
            const double v = ii <= jj ? fi(ii, jj) : 0.0;
            mc[int64_t(jj) * nd + i] = bi == 0 ? v : (bi == 1 ? sg * v : sp * v);
            mu[int64_t(jj) * nd + i] = bi == 1 ? v : 0.0;
        }
}

// ---------------------------------------------------------------- phase 2 --
struct P2 {
    int ns;            // slots of the batch
    int k_max;
    const int* nd;     // slot -> deflation column count
    const int* kdef;   // slot -> k
    const double* Mc;  // slot -> nd x k
    const double* Mu;
    int64_t Ms;
    double* Fk;        // slot -> k x inner
    double* H;         // slot -> packed upper R columns (Givens-reduced)
    int64_t Hs;
    double* g;         // slot -> inner + 1
    double* cs;
    double* sn;        // slot -> inner
    double* beta;      // slot
    const double* bnorm;  // slot -> |bs| of its rhs
    double* inv_h;
    int* status;       // 0 continue, 1 lucky, 2 converged, 3 full
    double* lsres;
    int inner;
    double tol;
};

// after the dots of w against [deflation | V(0..i)]: c = Mc^T g, Fk(:, i) = c,
// coef = [-(Mc c); -h]; H column i starts as h
__global__ void p2_a_k(int nact, const int* act, int ncm, const double* dots, double* coef, P2 q, int i) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    const int s = act[a];
    const int nd = q.nd[s], k = q.kdef[s];
    const double* dr = dots + int64_t(a) * ncm;
    double* cr = coef + int64_t(a) * ncm;
    const double* mc = q.Mc + int64_t(s) * q.Ms;
    double c[32];
    for (int jj = 0; jj < k; ++jj) {
        double v = 0.0;
        for (int l = 0; l < nd; ++l) v += mc[int64_t(jj) * nd + l] * dr[l];
        c[jj] = v;
        q.Fk[int64_t(s) * k * q.inner + int64_t(i) * k + jj] = v;
    }
    for (int l = 0; l < nd; ++l) {
        double v = 0.0;
        for (int jj = 0; jj < k; ++jj) v += mc[int64_t(jj) * nd + l] * c[jj];
        cr[l] = -v;
    }
    double* hc = q.H + int64_t(s) * q.Hs + int64_t(i) * (i + 1) / 2;
    for (int r = 0; r <= i; ++r) {
        hc[r] = dr[nd + r];
        cr[nd + r] = -dr[nd + r];
    }
}

// second pass: H column i += h2, coef = -h2
__global__ void p2_b_k(int nact, const int* act, int ncm, const double* dots, double* coef, P2 q, int i) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    const int s = act[a];
    double* hc = q.H + int64_t(s) * q.Hs + int64_t(i) * (i + 1) / 2;
    for (int r = 0; r <= i; ++r) {
        const double v = dots[int64_t(a) * ncm + r];
        hc[r] += v;
        coef[int64_t(a) * ncm + r] = -v;
    }
}

// |w| -> Givens update of column i, least-squares residual, the step's status
__global__ void p2_c_k(int nact, const int* act, const double* nrm, P2 q, int i) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    const int s = act[a];
    const double hn = nrm[s];
    double* hc = q.H + int64_t(s) * q.Hs + int64_t(i) * (i + 1) / 2;
    double* cs = q.cs + int64_t(s) * q.inner;
    double* sn = q.sn + int64_t(s) * q.inner;
    double* g = q.g + int64_t(s) * (q.inner + 1);
    double lower = hn;
    for (int r = 0; r < i; ++r) {
        const double t0 = cs[r] * hc[r] + sn[r] * hc[r + 1];
        hc[r + 1] = -sn[r] * hc[r] + cs[r] * hc[r + 1];
        hc[r] = t0;
    }
    double c, sg, rr;
    givens(hc[i], lower, c, sg, rr);
    cs[i] = c;
    sn[i] = sg;
    hc[i] = rr;
    g[i + 1] = -sg * g[i];
    g[i] = c * g[i];
    const double ls = fabs(g[i + 1]);
    q.lsres[s] = ls;
    int st = 0;
    if (hn <= 1e-14 * q.beta[s]) st = 1;
    else if (ls / q.bnorm[s] <= q.tol) st = 2;
    else if (i + 1 == q.inner) st = 3;
    q.status[s] = st;
    q.inv_h[s] = st == 1 ? 0.0 : 1.0 / hn;
}

// cycle start: g = beta e1, inv_h = 1 / beta
__global__ void p2_start_k(int nact, const int* act, const double* rn, P2 q) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    const int s = act[a];
    const double b = rn[s];
    q.beta[s] = b;
    double* g = q.g + int64_t(s) * (q.inner + 1);
    for (int r = 0; r <= q.inner; ++r) g[r] = r == 0 ? b : 0.0;
    q.inv_h[s] = 1.0 / b;
}

// end of a cycle: y2 = R^-1 g, coef (for x) = [Mu (-(Fk y2)); y2]
__global__ void p2_end_k(int nact, const int* act, const int* steps, int ncm, double* coef, P2 q) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    const int s = act[a];
    const int st = steps[s];
    const int nd = q.nd[s], k = q.kdef[s];
    const double* hs = q.H + int64_t(s) * q.Hs;
    const double* g = q.g + int64_t(s) * (q.inner + 1);
    double* cr = coef + int64_t(a) * ncm;
    double y[kMaxSteps];
    for (int r = st - 1; r >= 0; --r) {
        double t = g[r];
        for (int c = r + 1; c < st; ++c) t -= hs[int64_t(c) * (c + 1) / 2 + r] * y[c];
        y[r] = t / hs[int64_t(r) * (r + 1) / 2 + r];
    }
    double tk[32];
    const double* fk = q.Fk + int64_t(s) * k * q.inner;
    for (int jj = 0; jj < k; ++jj) {
        double v = 0.0;
        for (int c = 0; c < st; ++c) v += fk[int64_t(c) * k + jj] * y[c];
        tk[jj] = -v;
    }
    const double* mu = q.Mu + int64_t(s) * q.Ms;
    for (int l = 0; l < nd; ++l) {
        double v = 0.0;
        for (int jj = 0; jj < k; ++jj) v += mu[int64_t(jj) * nd + l] * tk[jj];
        cr[l] = v;
    }
    for (int c = 0; c < st; ++c) cr[nd + c] = y[c];
}

// deflate (x, r): z = Mc^T g; coef_x = Mu z, coef_r = -(Mc z)
__global__ void p2_defl_k(int nact, const int* act, int ncm, const double* dots, double* cx, double* crr, P2 q) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    const int s = act[a];
    const int nd = q.nd[s], k = q.kdef[s];
    const double* dr = dots + int64_t(a) * ncm;
    const double* mc = q.Mc + int64_t(s) * q.Ms;
    const double* mu = q.Mu + int64_t(s) * q.Ms;
    double z[32];
    for (int jj = 0; jj < k; ++jj) {
        double v = 0.0;
        for (int l = 0; l < nd; ++l) v += mc[int64_t(jj) * nd + l] * dr[l];
        z[jj] = v;
    }
    for (int l = 0; l < nd; ++l) {
        double vx = 0.0, vr = 0.0;
        for (int jj = 0; jj < k; ++jj) {
            vx += mu[int64_t(jj) * nd + l] * z[jj];
            vr += mc[int64_t(jj) * nd + l] * z[jj];
        }
        cx[int64_t(a) * ncm + l] = vx;
        crr[int64_t(a) * ncm + l] = -vr;
    }
}

// P^-1 = 1 / max(|Ks_ii + ms + msp Rs_ii|, 1e-300)  (krylov.cpp:429-437)
__global__ void pinv_k(int64_t N, const double* dinv, const double* kd, const double* rd, double sbar, double ms,
                       double msp, double* out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double d = dinv[i];
    const double ks = (d * (kd[i] + sbar * rd[i])) * d, rs = (d * rd[i]) * d;
    out[i] = 1.0 / fmax(fabs((ks + ms) + msp * rs), 1e-300);
}

// X_out[s] = dinv (.) x_s * mult[shift of s]
__global__ void unscale_k(int64_t N, int nsh, const double* x, const double* dinv, const double* mult, double* out,
                          int64_t os, int s0) {
    const int s = blockIdx.y;
    const double f = mult ? mult[(s0 + s) % nsh] : 1.0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += int64_t(gridDim.x) * blockDim.x)
        out[int64_t(s) * os + i] = (dinv[i] * x[int64_t(s) * N + i]) * f;
}

// element matrices (the reference's 2x2x2 Gauss rule) -- shared with cg.cu's
// FEM mode through fem_element_host
}  // namespace

void fem_element_host(double hx, double hy, double hz, double Ke[64], double Me[64], double Re[16]);

namespace {

template <class T>
DBuf upload(Ctx& c, const std::vector<T>& v) {
    DBuf b(c, std::max<size_t>(1, v.size()) * sizeof(T));
    if (!v.empty())
        HYDOT_CUDA(cudaMemcpyAsync(b.as<void>(), v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c.stream));
    return b;
}

template <class T>
std::vector<T> download(Ctx& c, const DBuf& b, size_t n) {
    std::vector<T> v(n);
    if (n) HYDOT_CUDA(cudaMemcpyAsync(v.data(), b.as<void>(), n * sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return v;
}

struct Family {
    Ctx& c;
    FemGeo g{};
    int64_t N = 0;
    DBuf em;  // Ke | Me | Re | dinv (N) | kd (N) | rd (N)
    double* dinv = nullptr;
    double* kd = nullptr;
    double* rd = nullptr;
    explicit Family(Ctx& cc) : c(cc) {}
};

void make_family(Family& f, const hydot_grid_geom& gg) {
    if (gg.nx < 3 || gg.ny < 3 || gg.nz < 2) throw std::invalid_argument("fields_solve: bad grid");
    if (gg.Lx <= 0 || gg.Ly <= 0 || gg.Lz <= 0) throw std::invalid_argument("build_grid: extents must be positive");
    f.N = int64_t(gg.nx) * gg.ny * gg.nz;
    if (f.N >= (int64_t(1) << 31)) throw std::invalid_argument("solve_family: grid too large");
    const double hx = 2 * gg.Lx / (gg.nx - 1), hy = 2 * gg.Ly / (gg.ny - 1), hz = gg.Lz / (gg.nz - 1);
    double h[144];
    fem_element_host(hx, hy, hz, h, h + 64, h + 128);
    f.em = dalloc(f.c, size_t(144 + 3 * f.N));
    HYDOT_CUDA(cudaMemcpyAsync(f.em.d(), h, sizeof h, cudaMemcpyHostToDevice, f.c.stream));
    f.dinv = f.em.d() + 144;
    f.kd = f.dinv + f.N;
    f.rd = f.kd + f.N;
    f.g = FemGeo{gg.nx, gg.ny, gg.nz, 1.0f / float(gg.nx), 1.0f / float(gg.ny), f.em.d()};
    fem_diag_k<<<unsigned((f.N + 255) / 256), 256, 0, f.c.stream>>>(f.g, f.N, f.dinv, f.kd, f.rd);
    f.c.check_launch();
}

inline unsigned cdiv(int64_t a, int64_t b) { return unsigned((a + b - 1) / b); }

struct Engine {
    Ctx& c;
    Family& f;
    int64_t N;
    int nsl;      // dot slices
    int ntile;    // upd tiles
    int ntile_op;
    DBuf part, red, coef, coef2, nrm2, dact, ncol;
    int ncm = 0, cap_act = 0;
    Engine(Ctx& cc, Family& ff, int max_act, int ncm_)
        : c(cc), f(ff), N(ff.N), ncm(ncm_), cap_act(max_act) {
        nsl = int((N + kDotL - 1) / kDotL);
        ntile = int((N + kT * kUpdRows - 1) / (kT * kUpdRows));
        ntile_op = ntile;
        part = dalloc(c, size_t(max_act) * ncm * std::max(nsl, ntile));
        red = dalloc(c, size_t(max_act) * ncm);
        coef = dalloc(c, size_t(max_act) * ncm);
        coef2 = dalloc(c, size_t(max_act) * ncm);
        dact = DBuf(c, size_t(max_act) * sizeof(int));
        ncol = DBuf(c, size_t(max_act) * sizeof(int));
    }
    void set_act(const std::vector<int>& a) {
        HYDOT_CUDA(cudaMemcpyAsync(dact.as<void>(), a.data(), a.size() * sizeof(int), cudaMemcpyHostToDevice,
                                   c.stream));
    }
    const int* act() const { return dact.as<int>(); }
    // red[a * ncm + c] = columns . w  (nact active slots)
    void dots(int nact, const Cols& cs, const double* w, int64_t ws, int64_t woff) {
        if (nact == 0) return;
        dot_k<<<dim3(unsigned(nact), unsigned(nsl)), kT, 0, c.stream>>>(N, cs, w, ws, woff, part.d(), nsl);
        c.check_launch();
        red_k<<<cdiv(int64_t(nact) * ncm, 256), 256, 0, c.stream>>>(nact, ncm, nullptr, part.d(), nsl, red.d());
        c.check_launch();
    }
    // target += columns * coef; norms -> out[slot] (optional)
    void update(int nact, const Cols& cs, const double* cf, const double* rs2, double* tb, int64_t ts, int64_t toff,
                double* norm_out) {
        if (nact == 0) return;
        upd_k<<<dim3(unsigned(nact), unsigned(ntile)), kT, 0, c.stream>>>(N, cs, cf, rs2, tb, ts, toff,
                                                                           norm_out ? part.d() : nullptr);
        c.check_launch();
        if (norm_out) {
            norm_k<<<cdiv(nact, 128), 128, 0, c.stream>>>(nact, act(), part.d(), ntile, norm_out);
            c.check_launch();
        }
    }
    void op(int nact, OpArgs o, double* norm_out) {
        if (nact == 0) return;
        o.act = act();
        o.part = norm_out ? part.d() : nullptr;
        op_k<<<dim3(unsigned(ntile_op), unsigned(nact)), kT, 0, c.stream>>>(f.g, N, o);
        c.check_launch();
        if (norm_out) {
            norm_k<<<cdiv(nact, 128), 128, 0, c.stream>>>(nact, act(), part.d(), ntile_op, norm_out);
            c.check_launch();
        }
    }
    void scale(int nact, const double* x, int64_t xs, int64_t xo, double* y, int64_t ys, int64_t yo,
               const double* sc) {
        if (nact == 0) return;
        scale_k<<<dim3(unsigned(std::min<int64_t>(cdiv(N, 256), 64)), unsigned(nact)), 256, 0, c.stream>>>(
            N, act(), x, xs, xo, y, ys, yo, sc);
        c.check_launch();
    }
};

struct RhsOut {
    int steps = 0, k = 0;
    bool breakdown = false, pencil = false, rank_reduced = false;
};

}  // namespace

void solve_family_fem(Ctx& c, const hydot_grid_geom& gg, int nsh, const double* sigma, const double* sigmap,
                      const double* b_dev, int n_rhs, const hydot_krylov_config& cfg, const double* mult,
                      double* X_dev, int64_t x_stride, hydot_krylov_stats* stats, hydot_krylov_family* fam_out) {
    if (nsh <= 0) throw std::invalid_argument("solve_family: no shifts");
    if (n_rhs <= 0) throw std::invalid_argument("solve_family: no right-hand sides");
    if (cfg.arnoldi_steps < 1 || cfg.arnoldi_steps > kMaxSteps || cfg.restart < 1 || cfg.restart > kMaxSteps ||
        cfg.deflation_dim < 0 || cfg.deflation_dim > 32 || cfg.max_restarts < 0)
        throw std::invalid_argument("solve_family: unsupported solver configuration");
    Family f(c);
    make_family(f, gg);
    const int64_t N = f.N;
    // center_shift_transform (optics.cpp:129-139, krylov.cpp:412-417)
    double sbar = 0.0;
    if (cfg.center_shifts) {
        for (int j = 0; j < nsh; ++j) sbar += sigmap[j];
        sbar /= nsh;
    }
    std::vector<double> sig(sigma, sigma + nsh), spr(static_cast<size_t>(nsh));
    for (int j = 0; j < nsh; ++j) spr[size_t(j)] = sigmap[j] - sbar;
    DBuf dsig = upload(c, sig), dspr = upload(c, spr);
    // Jacobi right preconditioner (krylov.cpp:429-437): P = |diag(Ks) + mean sigma + mean sigma'' diag(Rs)|
    DBuf pinv;
    if (cfg.jacobi) {
        double ms = 0.0, msp = 0.0;
        for (int j = 0; j < nsh; ++j) {
            ms += sig[size_t(j)];
            msp += spr[size_t(j)];
        }
        ms /= nsh;
        msp /= nsh;
        pinv = dalloc(c, size_t(N));
        pinv_k<<<cdiv(N, 256), 256, 0, c.stream>>>(N, f.dinv, f.kd, f.rd, sbar, ms, msp, pinv.d());
        c.check_launch();
    }
    const int n1 = int(std::min<int64_t>(cfg.arnoldi_steps, N));
    const int kreq = cfg.deflation_dim;
    const int inner_max = std::max(1, cfg.restart - 0);
    // ---- chunking by rhs: phase-1 basis + phase-2 systems of a chunk fit the budget
    size_t free_b = 0, total_b = 0;
    HYDOT_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double budget = 0.6 * double(free_b);
    const double per_rhs = 8.0 * N * (double(n1 + 1) + 3.0 * std::max(kreq, 1) + 2.0 + 2.0 * kreq +
                                      double(nsh) * (inner_max + 3.0));
    int chunk = int(std::max(1.0, std::min(double(n_rhs), budget / per_rhs)));
    if (per_rhs > budget && chunk == 1 && per_rhs > 0.95 * double(free_b))
        throw std::bad_alloc();
    for (int r0 = 0; r0 < n_rhs; r0 += chunk) {
        const int P = std::min(chunk, n_rhs - r0);
        const int S = P * nsh;  // phase-2 systems
        // ---- transformed rhs, |bs|
        DBuf bs = dalloc(c, size_t(P) * N), bnorm = dalloc(c, size_t(P));
        {
            const unsigned gx = std::min<unsigned>(cdiv(N, kT), 256);
            DBuf bp = dalloc(c, size_t(P) * gx);
            bscale_k<<<dim3(gx, unsigned(P)), kT, 0, c.stream>>>(N, b_dev + int64_t(r0) * N, f.dinv, bs.d(), bp.d());
            c.check_launch();
            std::vector<int> id(static_cast<size_t>(P));
            std::iota(id.begin(), id.end(), 0);
            DBuf did = upload(c, id);
            norm_k<<<cdiv(P, 128), 128, 0, c.stream>>>(P, did.as<int>(), bp.d(), int(gx), bnorm.d());
            c.check_launch();
        }
        std::vector<double> hbn = download<double>(c, bnorm, size_t(P));
        for (double v : hbn)
            if (v == 0.0) throw std::invalid_argument("multishift_gmres: b must be nonzero");
        // ---- phase 1: Arnoldi of Ks per rhs (multishift_gmres, krylov.cpp:45-104)
        const int ldT = n1 + 1;
        const int64_t v1s = int64_t(n1 + 1) * N, Ts = int64_t(ldT) * n1;
        DBuf V1 = dalloc(c, size_t(P) * v1s), T1 = dalloc(c, size_t(P) * Ts);
        HYDOT_CUDA(cudaMemsetAsync(T1.d(), 0, T1.bytes(), c.stream));
        const int ncm = std::max(n1 + 1, 3 * kreq + inner_max + 1);
        if (ncm > kMaxCols) throw std::invalid_argument("solve_family: basis too wide for the device kernels");
        Engine e(c, f, std::max(std::max(P, S), kreq), ncm);
        DBuf invh = dalloc(c, size_t(std::max(P, S))), nrm = dalloc(c, size_t(std::max(P, S)));
        DBuf flag = DBuf(c, size_t(std::max(P, S)) * sizeof(int));
        std::vector<int> act(static_cast<size_t>(P));
        std::iota(act.begin(), act.end(), 0);
        e.set_act(act);
        {  // V(:,0) = bs / |bs|
            std::vector<double> ib(static_cast<size_t>(P));
            for (int p = 0; p < P; ++p) ib[size_t(p)] = 1.0 / hbn[size_t(p)];
            DBuf dib = upload(c, ib);
            e.scale(P, bs.d(), N, 0, V1.d(), v1s, 0, dib.d());
        }
        std::vector<int> steps(static_cast<size_t>(P), 0);
        std::vector<RhsOut> ro(static_cast<size_t>(P));
        const int ls_scr = (n1 + 1) + 2 * n1 + n1 * (n1 + 1) / 2;
        DBuf lsscr = dalloc(c, size_t(P) * nsh * ls_scr);
        DBuf dsteps = DBuf(c, size_t(P) * sizeof(int));
        DBuf conv = DBuf(c, size_t(P) * nsh * sizeof(int));
        for (int i = 0; i < n1 && !act.empty(); ++i) {
            const int na = int(act.size());
            OpArgs o{};
            o.x = V1.d() + int64_t(i) * N;
            o.xs = v1s;
            o.y = V1.d() + int64_t(i + 1) * N;
            o.ys = v1s;
            o.ck = 1.0;
            o.cr0 = sbar;
            e.op(na, o, nullptr);
            Cols cs{};
            cs.act = e.act();
            cs.v2 = V1.d();
            cs.v2s = v1s;
            cs.c2a = 0;
            cs.n2 = i + 1;
            cs.ncm = ncm;
            for (int pass = 0; pass < 2; ++pass) {
                e.dots(na, cs, V1.d(), v1s, int64_t(i + 1) * N);
                p1_coef_k<<<cdiv(na, 128), 128, 0, c.stream>>>(na, e.act(), ncm, e.red.d(), e.coef.d(), T1.d(), Ts,
                                                               ldT, i, pass == 0 ? 1 : 0);
                c.check_launch();
                e.update(na, cs, e.coef.d(), nullptr, V1.d(), v1s, int64_t(i + 1) * N, pass == 1 ? nrm.d() : nullptr);
            }
            p1_norm_k<<<cdiv(na, 128), 128, 0, c.stream>>>(na, e.act(), nrm.d(), T1.d(), Ts, ldT, i, bnorm.d(),
                                                           invh.d(), flag.as<int>());
            c.check_launch();
            e.scale(na, V1.d(), v1s, int64_t(i + 1) * N, V1.d(), v1s, int64_t(i + 1) * N, invh.d());
            std::vector<int> fl = download<int>(c, flag, size_t(P));
            std::vector<int> still;
            for (int p : act) {
                steps[size_t(p)] = i + 1;
                if (fl[size_t(p)]) ro[size_t(p)].breakdown = true;
                else still.push_back(p);
            }
            if ((i + 1) % 10 == 0 && !still.empty() && i + 1 < n1) {
                HYDOT_CUDA(cudaMemcpyAsync(dsteps.as<void>(), steps.data(), size_t(P) * sizeof(int),
                                           cudaMemcpyHostToDevice, c.stream));
                DBuf dst = upload(c, still);
                const int np = int(still.size());
                p1_ls_k<<<cdiv(int64_t(np) * nsh, 128), 128, 0, c.stream>>>(
                    np, dst.as<int>(), nsh, dsig.d(), T1.d(), Ts, ldT, dsteps.as<int>(), bnorm.d(), cfg.tol,
                    lsscr.d(), ls_scr, conv.as<int>(), nullptr, 0, 0, nullptr);
                c.check_launch();
                std::vector<int> cv = download<int>(c, conv, size_t(np) * nsh);
                std::vector<int> keep;
                for (int a = 0; a < np; ++a) {
                    bool all = true;
                    for (int j = 0; j < nsh; ++j) all &= cv[size_t(a) * nsh + j] != 0;
                    if (!all) keep.push_back(still[size_t(a)]);
                }
                still.swap(keep);
            }
            act.swap(still);
            if (!act.empty()) e.set_act(act);
        }
        for (int p = 0; p < P; ++p) ro[size_t(p)].steps = steps[size_t(p)];
        HYDOT_CUDA(cudaMemcpyAsync(dsteps.as<void>(), steps.data(), size_t(P) * sizeof(int), cudaMemcpyHostToDevice,
                                   c.stream));
        // phase-1 solutions: Y (s x nsh) per rhs, X0 = V_s Y; relres per shift
        DBuf Y = dalloc(c, size_t(P) * n1 * nsh), p1rel = dalloc(c, size_t(P) * nsh);
        HYDOT_CUDA(cudaMemsetAsync(Y.d(), 0, Y.bytes(), c.stream));
        {
            std::vector<int> all(static_cast<size_t>(P));
            std::iota(all.begin(), all.end(), 0);
            DBuf dall = upload(c, all);
            p1_ls_k<<<cdiv(int64_t(P) * nsh, 128), 128, 0, c.stream>>>(
                P, dall.as<int>(), nsh, dsig.d(), T1.d(), Ts, ldT, dsteps.as<int>(), bnorm.d(), cfg.tol, lsscr.d(),
                ls_scr, nullptr, Y.d(), int64_t(n1) * nsh, n1, p1rel.d());
            c.check_launch();
        }
        lsscr.release();
        // systems: slot = p * nsh + j; x = phase-1 solution
        DBuf X = dalloc(c, size_t(S) * N);
        for (int p = 0; p < P; ++p)
            dgemm(c, false, false, N, nsh, steps[size_t(p)], 1.0, V1.d() + int64_t(p) * v1s, N,
                  Y.d() + int64_t(p) * n1 * nsh, n1, 0.0, X.d() + int64_t(p) * nsh * N, N);
        std::vector<double> hp1 = download<double>(c, p1rel, size_t(P) * nsh);
        // ---- deflation basis per rhs (harmonic_ritz + build_deflation_basis)
        std::vector<int> kdef(static_cast<size_t>(P), 0);
        const int kd3 = 3 * std::max(kreq, 1);
        DBuf Dset = dalloc(c, size_t(P) * kd3 * N);
        DBuf G = dalloc(c, size_t(P) * kd3 * kd3);
        if (kreq > 0) {
            const int ld = n1;
            DBuf scr = dalloc(c, size_t(P) * 5 * ld * ld), Z = dalloc(c, size_t(P) * ld * kreq);
            DBuf th = dalloc(c, size_t(P) * kreq);
            DBuf kout = DBuf(c, size_t(P) * sizeof(int)), pen = DBuf(c, size_t(P) * sizeof(int));
            HYDOT_CUDA(cudaMemsetAsync(pen.as<void>(), 0, pen.bytes(), c.stream));
            hritz_k<<<unsigned(P), kT, 0, c.stream>>>(dsteps.as<int>(), T1.d(), Ts, ldT, kreq, ld, scr.d(),
                                                      int64_t(5) * ld * ld, Z.d(), int64_t(ld) * kreq, th.d(),
                                                      kout.as<int>(), pen.as<int>());
            c.check_launch();
            std::vector<int> hk = download<int>(c, kout, size_t(P)), hpen = download<int>(c, pen, size_t(P));
            DBuf Ut = dalloc(c, size_t(N) * kreq), Cp = dalloc(c, size_t(N) * kreq);
            DBuf TZ = dalloc(c, size_t(n1 + 1) * kreq), Rk = dalloc(c, size_t(kreq) * kreq);
            for (int p = 0; p < P; ++p) {
                ro[size_t(p)].pencil = hpen[size_t(p)] != 0;
                const int s = steps[size_t(p)];
                int k = hk[size_t(p)];
                double* Vp = V1.d() + int64_t(p) * v1s;
                double* Dp = Dset.d() + int64_t(p) * kd3 * N;
                while (k > 0) {
                    const double* Zp = Z.d() + int64_t(p) * ld * kreq;
                    dgemm(c, false, false, N, k, s, 1.0, Vp, N, Zp, ld, 0.0, Ut.d(), N);
                    dgemm(c, false, false, s + 1, k, s, 1.0, T1.d() + int64_t(p) * Ts, ldT, Zp, ld, 0.0, TZ.d(),
                          s + 1);
                    dgemm(c, false, false, N, k, s + 1, 1.0, Vp, N, TZ.d(), s + 1, 0.0, Cp.d(), N);
                    QRFact qf;
                    geqrf(c, N, k, Cp.d(), N, qf);
                    extract_upper(c, k, qf.a.d(), N, Rk.d(), k);
                    std::vector<double> R = download<double>(c, Rk, size_t(k) * k);
                    double dmax = 0.0;
                    for (int i = 0; i < k; ++i) dmax = std::max(dmax, std::fabs(R[size_t(i) * k + i]));
                    bool ok = true;
                    for (int i = 0; i < k; ++i)
                        if (std::fabs(R[size_t(i) * k + i]) < 1e-12 * dmax) ok = false;
                    if (!ok) {
                        --k;
                        ro[size_t(p)].rank_reduced = true;
                        continue;
                    }
                    // C = Q [I; 0] into Dset columns [0, k); U = Ut R^-1 into [k, 2k)
                    fill(c, N, k, 0.0, Dp, N);
                    set_identity(c, k, k, Dp, N);
                    apply_q(c, qf, false, k, Dp, N);
                    trsm_ru_k<<<cdiv(N, 256), 256, 0, c.stream>>>(N, k, Ut.d(), Rk.d(), k, Dp + int64_t(k) * N);
                    c.check_launch();
                    break;
                }
                kdef[size_t(p)] = k;
                ro[size_t(p)].k = k;
                if (k == 0) continue;
                // RU = Rs U  (columns [2k, 3k))
                std::vector<int> cols(static_cast<size_t>(k));
                std::iota(cols.begin(), cols.end(), 0);
                e.set_act(cols);
                OpArgs o{};
                o.x = Dp + int64_t(k) * N;
                o.xs = N;
                o.y = Dp + int64_t(2 * k) * N;
                o.ys = N;
                o.ck = 0.0;
                o.cr0 = 1.0;
                e.op(k, o, nullptr);
                // G = [C U RU]^T [C U RU]
                dgemm(c, true, false, 3 * k, 3 * k, N, 1.0, Dp, N, Dp, N, 0.0, G.d() + int64_t(p) * kd3 * kd3, 3 * k);
            }
        }
        V1.release();
        T1.release();
        // ---- per-shift deflation coefficients (ShiftedDeflation)
        const int kmax = std::max(1, kreq);
        const int64_t Ms = int64_t(3 * kmax) * kmax;
        DBuf Mc = dalloc(c, size_t(S) * Ms), Mu = dalloc(c, size_t(S) * Ms);
        DBuf failed = DBuf(c, size_t(S) * sizeof(int));
        HYDOT_CUDA(cudaMemsetAsync(failed.as<void>(), 0, failed.bytes(), c.stream));
        DBuf dkdef = upload(c, kdef);
        std::vector<int> nd(static_cast<size_t>(S)), kslot(static_cast<size_t>(S)), dsetv(static_cast<size_t>(S));
        for (int s = 0; s < S; ++s) {
            const int p = s / nsh;
            nd[size_t(s)] = 3 * kdef[size_t(p)];
            kslot[size_t(s)] = kdef[size_t(p)];
            dsetv[size_t(s)] = p;
        }
        if (kreq > 0) {
            std::vector<int> all(static_cast<size_t>(P));
            std::iota(all.begin(), all.end(), 0);
            DBuf dall = upload(c, all);
            shifted_k<<<cdiv(int64_t(P) * nsh, 128), 128, 0, c.stream>>>(
                P, dall.as<int>(), nsh, dsig.d(), dspr.d(), dkdef.as<int>(), G.d(), int64_t(kd3) * kd3, Mc.d(),
                Mu.d(), Ms, failed.as<int>(), cfg.explicit_qr_update ? 1 : 0);
            c.check_launch();
        }
        std::vector<int> hfail = download<int>(c, failed, size_t(S));
        // explicit QR path (krylov.cpp:237-246) for the failed / forced shifts
        std::vector<int> expl;
        for (int s = 0; s < S; ++s)
            if (kslot[size_t(s)] > 0 && hfail[size_t(s)]) expl.push_back(s);
        DBuf Dx;
        if (!expl.empty()) {
            Dx = dalloc(c, size_t(expl.size()) * 2 * kmax * N);
            DBuf Mtmp = dalloc(c, size_t(3 * kmax) * kmax), Rk = dalloc(c, size_t(kmax) * kmax);
            DBuf Cpj = dalloc(c, size_t(N) * kmax);
            for (size_t t = 0; t < expl.size(); ++t) {
                const int s = expl[t], p = s / nsh, j = s % nsh, k = kslot[size_t(s)];
                const double* Dp = Dset.d() + int64_t(p) * kd3 * N;
                std::vector<double> m(size_t(3 * k) * k, 0.0);
                for (int i = 0; i < k; ++i) {
                    m[size_t(i) * 3 * k + i] = 1.0;
                    m[size_t(i) * 3 * k + k + i] = sig[size_t(j)];
                    m[size_t(i) * 3 * k + 2 * k + i] = spr[size_t(j)];
                }
                HYDOT_CUDA(cudaMemcpyAsync(Mtmp.d(), m.data(), m.size() * 8, cudaMemcpyHostToDevice, c.stream));
                dgemm(c, false, false, N, k, 3 * k, 1.0, Dp, N, Mtmp.d(), 3 * k, 0.0, Cpj.d(), N);
                QRFact qf;
                geqrf(c, N, k, Cpj.d(), N, qf);
                extract_upper(c, k, qf.a.d(), N, Rk.d(), k);
                double* Dxs = Dx.d() + int64_t(t) * 2 * kmax * N;
                fill(c, N, k, 0.0, Dxs, N);
                set_identity(c, k, k, Dxs, N);
                apply_q(c, qf, false, k, Dxs, N);
                trsm_ru_k<<<cdiv(N, 256), 256, 0, c.stream>>>(N, k, Dp + int64_t(k) * N, Rk.d(), k,
                                                               Dxs + int64_t(k) * N);
                c.check_launch();
                std::vector<double> mc(static_cast<size_t>(Ms), 0.0), mu(static_cast<size_t>(Ms), 0.0);
                for (int i = 0; i < k; ++i) {
                    mc[size_t(i) * 2 * k + i] = 1.0;
                    mu[size_t(i) * 2 * k + k + i] = 1.0;
                }
                HYDOT_CUDA(cudaMemcpyAsync(Mc.d() + int64_t(s) * Ms, mc.data(), size_t(Ms) * 8,
                                           cudaMemcpyHostToDevice, c.stream));
                HYDOT_CUDA(cudaMemcpyAsync(Mu.d() + int64_t(s) * Ms, mu.data(), size_t(Ms) * 8,
                                           cudaMemcpyHostToDevice, c.stream));
                nd[size_t(s)] = 2 * k;
                dsetv[size_t(s)] = int(t);
            }
            c.sync();
        }
        // ---- phase 2: augmented GMRES per system (krylov.cpp:311-398)
        std::vector<int> inner_of(static_cast<size_t>(S));
        int inner = 1;
        for (int s = 0; s < S; ++s) {
            inner_of[size_t(s)] = std::max(1, cfg.restart - kslot[size_t(s)]);
            inner = std::max(inner, inner_of[size_t(s)]);
        }
        // one deflation-set pointer space: the rhs sets, then the explicit sets
        // (dset index >= P) -- kept as two Cols variants
        std::vector<int> is_expl(static_cast<size_t>(S), 0);
        for (int s : expl) is_expl[size_t(s)] = 1;
        DBuf dnd = upload(c, nd), dk = upload(c, kslot), dds = upload(c, dsetv);
        const int64_t v2s = int64_t(inner + 1) * N;
        DBuf V2 = dalloc(c, size_t(S) * v2s);
        DBuf Fk = dalloc(c, size_t(S) * kmax * inner), H = dalloc(c, size_t(S) * inner * (inner + 1) / 2);
        DBuf gv = dalloc(c, size_t(S) * (inner + 1)), csv = dalloc(c, size_t(S) * inner),
             snv = dalloc(c, size_t(S) * inner);
        DBuf betav = dalloc(c, size_t(S)), bnv = dalloc(c, size_t(S)), lsv = dalloc(c, size_t(S));
        DBuf status = DBuf(c, size_t(S) * sizeof(int)), dstp = DBuf(c, size_t(S) * sizeof(int));
        DBuf rnorm = dalloc(c, size_t(S)), cs_slot = dalloc(c, size_t(S)), cr_slot = dalloc(c, size_t(S));
        std::vector<int> bslot(static_cast<size_t>(S));
        {
            std::vector<double> bn(static_cast<size_t>(S)), csh(static_cast<size_t>(S)), crh(static_cast<size_t>(S));
            for (int s = 0; s < S; ++s) {
                bn[size_t(s)] = hbn[size_t(s / nsh)];
                csh[size_t(s)] = sig[size_t(s % nsh)];
                crh[size_t(s)] = sbar + spr[size_t(s % nsh)];
                bslot[size_t(s)] = s / nsh;
            }
            HYDOT_CUDA(cudaMemcpyAsync(bnv.d(), bn.data(), size_t(S) * 8, cudaMemcpyHostToDevice, c.stream));
            HYDOT_CUDA(cudaMemcpyAsync(cs_slot.d(), csh.data(), size_t(S) * 8, cudaMemcpyHostToDevice, c.stream));
            HYDOT_CUDA(cudaMemcpyAsync(cr_slot.d(), crh.data(), size_t(S) * 8, cudaMemcpyHostToDevice, c.stream));
        }
        DBuf dbslot = upload(c, bslot);
        DBuf R = dalloc(c, size_t(S) * N);
        P2 q{};
        q.ns = S;
        q.k_max = kmax;
        q.nd = dnd.as<int>();
        q.kdef = dk.as<int>();
        q.Mc = Mc.d();
        q.Mu = Mu.d();
        q.Ms = Ms;
        q.Fk = Fk.d();
        q.H = H.d();
        q.Hs = int64_t(inner) * (inner + 1) / 2;
        q.g = gv.d();
        q.cs = csv.d();
        q.sn = snv.d();
        q.beta = betav.d();
        q.bnorm = bnv.d();
        q.inv_h = invh.d();
        q.status = status.as<int>();
        q.lsres = lsv.d();
        q.inner = inner;
        q.tol = cfg.tol;
        // Column views: deflation set of a slot (rhs set or its explicit set),
        // plus the slot's V columns.  Slots of the two kinds go in separate launches.
        auto defl_cols = [&](bool explicit_kind, const double* v2, int c2a, int n2) {
            Cols cs{};
            cs.act = e.act();
            cs.d1 = explicit_kind ? Dx.d() : Dset.d();
            cs.d1s = explicit_kind ? int64_t(2) * kmax * N : int64_t(kd3) * N;
            cs.dset = kreq > 0 ? dds.as<int>() : nullptr;
            cs.nd1 = dnd.as<int>();
            cs.v2 = v2;
            cs.v2s = v2s;
            cs.c2a = c2a;
            cs.n2 = n2;
            cs.ncm = ncm;
            return cs;
        };
        std::vector<hydot_krylov_stats> st(static_cast<size_t>(S));
        for (auto& x : st) x = hydot_krylov_stats{0, 0, 0.0, 0, 0.0};
        // groups of active slots by deflation kind (0 = rhs set, 1 = explicit)
        auto split = [&](const std::vector<int>& v) {
            std::vector<int> a0, a1;
            for (int s : v) (is_expl[size_t(s)] ? a1 : a0).push_back(s);
            return std::make_pair(a0, a1);
        };
        auto for_kinds = [&](const std::vector<int>& v, auto&& fn) {
            auto pr = split(v);
            if (!pr.first.empty()) {
                e.set_act(pr.first);
                fn(false, int(pr.first.size()));
            }
            if (!pr.second.empty()) {
                e.set_act(pr.second);
                fn(true, int(pr.second.size()));
            }
        };
        // r = bs - A x  (+ |r|)
        auto residual = [&](const std::vector<int>& v) {
            e.set_act(v);
            OpArgs o{};
            o.x = X.d();
            o.xs = N;
            o.y = R.d();
            o.ys = N;
            o.ck = 1.0;
            o.cs = cs_slot.d();
            o.cr = cr_slot.d();
            o.b = bs.d();
            o.bslot = dbslot.as<int>();
            o.bs = N;
            e.op(int(v.size()), o, rnorm.d());
            for (int s : v) st[size_t(s)].matvecs++;
        };
        // deflate(x, r): x += U_j C_j^T r, r -= C_j C_j^T r; |r| -> rnorm
        auto deflate = [&](const std::vector<int>& v) {
            if (kreq == 0) return;
            std::vector<int> w;
            for (int s : v)
                if (kslot[size_t(s)] > 0) w.push_back(s);
            for_kinds(w, [&](bool ek, int na) {
                Cols cs = defl_cols(ek, R.d(), 0, 0);
                e.dots(na, cs, R.d(), N, 0);
                p2_defl_k<<<cdiv(na, 128), 128, 0, c.stream>>>(na, e.act(), ncm, e.red.d(), e.coef.d(),
                                                               e.coef2.d(), q);
                c.check_launch();
                e.update(na, cs, e.coef.d(), nullptr, X.d(), N, 0, nullptr);
                e.update(na, cs, e.coef2.d(), nullptr, R.d(), N, 0, rnorm.d());
            });
        };
        std::vector<int> all(static_cast<size_t>(S));
        std::iota(all.begin(), all.end(), 0);
        residual(all);
        deflate(all);
        std::vector<double> rn = download<double>(c, rnorm, size_t(S));
        std::vector<int> live;
        std::vector<int> done(static_cast<size_t>(S), 0);
        for (int s = 0; s < S; ++s) {
            st[size_t(s)].relres = rn[size_t(s)] / hbn[size_t(s / nsh)];
            st[size_t(s)].phase1_relres = hp1[size_t(s)];
            live.push_back(s);
        }
        for (int cycle = 0; cycle <= cfg.max_restarts && !live.empty(); ++cycle) {
            std::vector<int> cyc;
            for (int s : live) {
                if (st[size_t(s)].relres <= cfg.tol) {
                    st[size_t(s)].converged = 1;
                    done[size_t(s)] = 1;
                } else {
                    cyc.push_back(s);
                }
            }
            live = cyc;
            if (cyc.empty()) break;
            // V(:,0) = r / beta, g = beta e1
            e.set_act(cyc);
            p2_start_k<<<cdiv(int(cyc.size()), 128), 128, 0, c.stream>>>(int(cyc.size()), e.act(), rnorm.d(), q);
            c.check_launch();
            e.scale(int(cyc.size()), R.d(), N, 0, V2.d(), v2s, 0, invh.d());
            std::vector<int> stp(static_cast<size_t>(S), 0), lucky(static_cast<size_t>(S), 0);
            std::vector<int> inn = cyc;
            for (int i = 0; i < inner && !inn.empty(); ++i) {
                // w = A P^-1 v_i  (into V(:, i+1))
                e.set_act(inn);
                OpArgs o{};
                o.x = V2.d() + int64_t(i) * N;
                o.xs = v2s;
                o.y = V2.d() + int64_t(i + 1) * N;
                o.ys = v2s;
                o.ck = 1.0;
                o.cs = cs_slot.d();
                o.cr = cr_slot.d();
                o.px = cfg.jacobi ? pinv.d() : nullptr;
                e.op(int(inn.size()), o, nullptr);
                for (int s : inn) st[size_t(s)].matvecs++;
                for_kinds(inn, [&](bool ek, int na) {
                    // pass 1: deflation dots + V dots, subtract both; pass 2: V only
                    Cols cs = defl_cols(ek, V2.d(), 0, i + 1);
                    if (kreq == 0) cs.dset = nullptr;
                    e.dots(na, cs, V2.d(), v2s, int64_t(i + 1) * N);
                    p2_a_k<<<cdiv(na, 128), 128, 0, c.stream>>>(na, e.act(), ncm, e.red.d(), e.coef.d(), q, i);
                    c.check_launch();
                    e.update(na, cs, e.coef.d(), nullptr, V2.d(), v2s, int64_t(i + 1) * N, nullptr);
                    Cols cv = cs;
                    cv.dset = nullptr;
                    e.dots(na, cv, V2.d(), v2s, int64_t(i + 1) * N);
                    p2_b_k<<<cdiv(na, 128), 128, 0, c.stream>>>(na, e.act(), ncm, e.red.d(), e.coef.d(), q, i);
                    c.check_launch();
                    e.update(na, cv, e.coef.d(), nullptr, V2.d(), v2s, int64_t(i + 1) * N, nrm.d());
                    p2_c_k<<<cdiv(na, 128), 128, 0, c.stream>>>(na, e.act(), nrm.d(), q, i);
                    c.check_launch();
                });
                e.set_act(inn);
                e.scale(int(inn.size()), V2.d(), v2s, int64_t(i + 1) * N, V2.d(), v2s, int64_t(i + 1) * N, invh.d());
                std::vector<int> sv = download<int>(c, status, size_t(S));
                std::vector<int> nxt;
                for (int s : inn) {
                    stp[size_t(s)] = i + 1;
                    const int code = sv[size_t(s)];
                    if (code == 1) lucky[size_t(s)] = 1;
                    if (code == 0 && i + 1 < inner_of[size_t(s)]) nxt.push_back(s);
                }
                inn.swap(nxt);
            }
            // end of the cycle: x += U_j(-(Fk y2)) + P^-1 V y2; r = b - A x
            for (int s : cyc) st[size_t(s)].iterations += stp[size_t(s)];
            HYDOT_CUDA(cudaMemcpyAsync(dstp.as<void>(), stp.data(), size_t(S) * sizeof(int), cudaMemcpyHostToDevice,
                                       c.stream));
            // systems grouped by step count (the V column count of the update)
            std::vector<int> byst(static_cast<size_t>(S), -1);
            for (int sc = 1; sc <= inner; ++sc) {
                std::vector<int> grp;
                for (int s : cyc)
                    if (stp[size_t(s)] == sc) grp.push_back(s);
                if (grp.empty()) continue;
                for_kinds(grp, [&](bool ek, int na) {
                    Cols cs = defl_cols(ek, V2.d(), 0, sc);
                    if (kreq == 0) cs.dset = nullptr;
                    p2_end_k<<<cdiv(na, 128), 128, 0, c.stream>>>(na, e.act(), dstp.as<int>(), ncm, e.coef.d(), q);
                    c.check_launch();
                    e.update(na, cs, e.coef.d(), cfg.jacobi ? pinv.d() : nullptr, X.d(), N, 0, nullptr);
                });
            }
            residual(cyc);
            std::vector<double> rr = download<double>(c, rnorm, size_t(S));
            std::vector<int> cont;
            for (int s : cyc) {
                st[size_t(s)].relres = rr[size_t(s)] / hbn[size_t(s / nsh)];
                if (st[size_t(s)].relres <= cfg.tol || lucky[size_t(s)]) {
                    st[size_t(s)].converged = st[size_t(s)].relres <= cfg.tol;
                    done[size_t(s)] = 1;
                } else {
                    cont.push_back(s);
                }
            }
            // re-deflate before the next cycle; stats.relres keeps the
            // pre-deflation value, beta is the deflated |r| (krylov.cpp:392-396, 346)
            deflate(cont);
            live = cont;
        }
        // ---- outputs: original variables, times mult[shift]
        DBuf dmult;
        if (mult) dmult = upload(c, std::vector<double>(mult, mult + nsh));
        for (int p = 0; p < P; ++p) {
            unscale_k<<<dim3(std::min<unsigned>(cdiv(N, 256), 256), unsigned(nsh)), 256, 0, c.stream>>>(
                N, nsh, X.d() + int64_t(p) * nsh * N, f.dinv, mult ? dmult.d() : nullptr,
                X_dev + int64_t(r0 + p) * nsh * x_stride, x_stride, 0);
            c.check_launch();
        }
        c.sync();
        for (int s = 0; s < S; ++s) {
            const int p = s / nsh;
            if (stats) stats[int64_t(r0) * nsh + s] = st[size_t(s)];
        }
        if (fam_out)
            for (int p = 0; p < P; ++p) {
                hydot_krylov_family& fo = fam_out[r0 + p];
                fo.phase1_steps = ro[size_t(p)].steps;
                fo.deflation_k = ro[size_t(p)].k;
                fo.rank_reduced = ro[size_t(p)].rank_reduced;
                fo.pencil_shifted = ro[size_t(p)].pencil;
                fo.breakdown = ro[size_t(p)].breakdown;
                fo.cholesky_failed = 0;
                fo.all_converged = 1;
                fo.first_failure = -1;
                for (int j = 0; j < nsh; ++j) {
                    const int s = p * nsh + j;
                    if (hfail[size_t(s)] && !cfg.explicit_qr_update) fo.cholesky_failed++;
                    if (!st[size_t(s)].converged) {
                        fo.all_converged = 0;
                        if (fo.first_failure < 0) fo.first_failure = j;
                    }
                }
            }
    }
}

namespace {
// b[r][ridx[r*8+a]] = rw[r*8+a]  (b zeroed before)
__global__ void scatter_src_k(int n, int64_t N, const int64_t* ridx, const double* rw, double* b) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * 8) return;
    const int64_t v = ridx[t];
    if (v >= 0) b[int64_t(t / 8) * N + v] = rw[t];
}
}  // namespace

void fields_solve_fem_gmres(Ctx& c, const hydot_grid_geom& g, int nl, const double* sigma, const double* sigmap,
                            const double* inv_D, const double* points, int n_pts, const hydot_krylov_config& cfg,
                            double* out, hydot_krylov_stats* stats, hydot_krylov_family* fam) {
    if (nl <= 0 || n_pts <= 0) throw std::invalid_argument("compute_fields: no wavelengths");
    if (g.nx < 3 || g.ny < 3 || g.nz < 2) throw std::invalid_argument("fields_solve: bad grid");
    if (g.Lx <= 0 || g.Ly <= 0 || g.Lz <= 0) throw std::invalid_argument("build_grid: extents must be positive");
    std::vector<int64_t> ridx;
    std::vector<double> rw, b2;
    fem_point_weights(g, points, n_pts, ridx, rw, b2);
    const int64_t N = int64_t(g.nx) * g.ny * g.nz;
    DBuf b = dalloc(c, size_t(n_pts) * N);
    HYDOT_CUDA(cudaMemsetAsync(b.d(), 0, b.bytes(), c.stream));
    DBuf dr = upload(c, ridx), dw = upload(c, rw);
    scatter_src_k<<<cdiv(int64_t(n_pts) * 8, 128), 128, 0, c.stream>>>(n_pts, N, dr.as<int64_t>(), dw.d(), b.d());
    c.check_launch();
    std::vector<hydot_krylov_stats> st(size_t(n_pts) * nl);
    solve_family_fem(c, g, nl, sigma, sigmap, b.d(), n_pts, cfg, inv_D, out, N, st.data(), fam);
    if (stats) std::copy(st.begin(), st.end(), stats);
    // born.cpp:58-61
    for (int k = 0; k < n_pts * nl; ++k)
        if (!st[size_t(k)].converged)
            throw std::runtime_error("field solve failed at point " + std::to_string(k / nl) + ", wavelength index " +
                                     std::to_string(k % nl));
}

}  // namespace hydot
