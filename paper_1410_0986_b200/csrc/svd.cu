// svd.cu -- one-sided (Hestenes) Jacobi thin SVD on the GPU, replacing
// Eigen::BDCSVD on the small cores of the path (lowrank.cpp:43-49, 79, 88,
// 568): the R factors of Y, B^T, W^T and the recompress core.
//
// Columns of X (m x n, m >= n) are orthogonalised by plane rotations in
// round-robin (circle-method) order; each rotation is computed from the
// actual column dot products, so small singular values keep high relative
// accuracy (no Gram matrix is formed).  Two drivers:
//   * small: (m + n) n doubles fit in shared memory -- one CTA runs every
//     sweep on-chip, one warp per column pair;
//   * large: one cooperative persistent kernel runs all sweeps with a
//     grid-wide barrier between rounds and a per-sweep rotation counter for
//     convergence (no host round trips).  With lazy V (the path's default)
//     and m <= 2560 it is the register block-Jacobi jacobi_rblk_k (blocks of
//     4 columns, a 28-pair mini-sweep per block pair in registers: 4x fewer
//     barriers and passes over U; 1.24x faster over config 1's cores than the
//     point driver); otherwise one CTA per column pair.  Measured slower and
//     kept out of the default: a dataflow variant with per-column completion
//     flags (a release fence per pair serialises each CTA, 1.75x) and a
//     shared-memory block variant (bound by per-SM shared-memory bandwidth).
// Afterwards sigma_j = ||u_j||, U = u_j / sigma_j, sorted descending.
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <numeric>
#include <string>

#include "internal.h"

namespace cg = cooperative_groups;

namespace hydot {
namespace {

constexpr int kMaxSweeps = 40;
constexpr int JT = 256;  // threads per CTA of the large driver

// Jacobi rotation annihilating g for the 2x2 Gram [[a, g], [g, b]]:
// t = sign(d) g / (|d| + sqrt(d^2 + g^2)), d = (b - a) / 2 -- the usual
// zeta = d / g form multiplied through by |g| (one division, one sqrt and
// one rsqrt on the critical path instead of three divisions and two sqrts)
//
// Default form: two reciprocal square roots on the critical path, no
// division or square root -- with r = 1/rho, rho = sqrt(d^2 + g^2),
// x = |d|/rho = cos 2theta:  cs = sqrt((1 + x)/2),  sn = sign(d) g r / (2 cs)
// = sign(d) (g r / 2) rsqrt((1 + x)/2); cs^2 + sn^2 = 1 identically.
// HYDOT_ROT_FORM=0 (compile time) keeps the t-form.
#ifndef HYDOT_ROT_FORM
#define HYDOT_ROT_FORM 1
#endif
__device__ __forceinline__ void rot_params(double a, double b, double g, double& cs, double& sn) {
    const double d = 0.5 * (b - a);
#if HYDOT_ROT_FORM
    const double r = rsqrt(fma(d, d, g * g));
    const double h = fma(0.5 * fabs(d), r, 0.5);  // (1 + x) / 2 in (1/2, 1]
    const double ih = rsqrt(h);
    cs = h * ih;
    sn = copysign(1.0, d) * (0.5 * g * r) * ih;
#else
    const double t = copysign(1.0, d) * g / (fabs(d) + sqrt(fma(d, d, g * g)));
    cs = rsqrt(fma(t, t, 1.0));
    sn = cs * t;
#endif
}

// one warp orthogonalises columns p, q of U (m rows) and rotates V (n rows);
// returns true when a rotation was applied
__device__ __forceinline__ bool warp_pair(int lane, int64_t m, int64_t n, double* __restrict__ up,
                                          double* __restrict__ uq, double* __restrict__ vp,
                                          double* __restrict__ vq, double tol, double atol) {
    double a = 0, b = 0, g = 0;
    for (int64_t i = lane; i < m; i += 32) {
        double x = up[i], y = uq[i];
        a += x * x;
        b += y * y;
        g += x * y;
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        g += __shfl_xor_sync(0xffffffffu, g, o);
    }
    // relative criterion (high relative accuracy) AND an absolute floor at
    // the backward-error level eps*||A||*max(|u_p|,|u_q|) (BDCSVD-grade)
    if (!(g != 0.0 && fabs(g) > tol * sqrt(a * b) && fabs(g) > atol * sqrt(fmax(a, b))))
        return false;  // atol = 0 keeps the pure relative criterion
    double cs, sn;
    rot_params(a, b, g, cs, sn);
    for (int64_t i = lane; i < m; i += 32) {
        double x = up[i], y = uq[i];
        up[i] = cs * x - sn * y;
        uq[i] = sn * x + cs * y;
    }
    for (int64_t i = lane; i < n; i += 32) {
        double x = vp[i], y = vq[i];
        vp[i] = cs * x - sn * y;
        vq[i] = sn * x + cs * y;
    }
    return true;
}

// ---------------------------------------------------------- single CTA ----
__global__ void __launch_bounds__(1024) jacobi_smem_k(int m, int n, int np,
                                                      const int2* __restrict__ pairs,
                                                      double* __restrict__ Ug, int64_t ldu,
                                                      double* __restrict__ Vg, int64_t ldv,
                                                      double tol, double atol,
                                                      int* __restrict__ sweeps_out) {
    // Vg == nullptr: lazy V (only U lives in shared memory, V is recovered
    // by the caller's GEMM) -- lets n up to ~160 run on one SM
    extern __shared__ double sm[];
    const bool withV = Vg != nullptr;
    const int vn = withV ? n : 0;
    double* U = sm;                   // m x n, ld m
    double* V = sm + int64_t(m) * n;  // n x n, ld n (withV)
    __shared__ int changed;
    for (int64_t e = threadIdx.x; e < int64_t(m) * n; e += blockDim.x) {
        int64_t i = e % m, j = e / m;
        U[e] = Ug[i + j * ldu];
    }
    for (int64_t e = threadIdx.x; e < int64_t(vn) * vn; e += blockDim.x) {
        int64_t i = e % vn, j = e / vn;
        V[e] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int rounds = np - 1, per = np / 2;
    int sweep = 0;
    for (; sweep < kMaxSweeps; ++sweep) {
        if (threadIdx.x == 0) changed = 0;
        __syncthreads();
        for (int r = 0; r < rounds; ++r) {
            for (int q = warp; q < per; q += nwarp) {
                int2 pr = pairs[r * per + q];
                if (pr.x >= n || pr.y >= n) continue;
                if (warp_pair(lane, m, vn, U + int64_t(pr.x) * m, U + int64_t(pr.y) * m,
                              V + int64_t(pr.x) * vn, V + int64_t(pr.y) * vn, tol, atol) &&
                    lane == 0)
                    changed = 1;
            }
            __syncthreads();
        }
        if (!changed) break;
        __syncthreads();
    }
    for (int64_t e = threadIdx.x; e < int64_t(m) * n; e += blockDim.x) {
        int64_t i = e % m, j = e / m;
        Ug[i + j * ldu] = U[e];
    }
    for (int64_t e = threadIdx.x; e < int64_t(vn) * vn; e += blockDim.x) {
        int64_t i = e % vn, j = e / vn;
        Vg[i + j * ldv] = V[e];
    }
    if (threadIdx.x == 0 && sweeps_out) *sweeps_out = sweep;
}

// ------------------------------------------------------- cooperative ------
// CTA-per-pair variant for long columns
__global__ void __launch_bounds__(JT) jacobi_coop_k(int64_t m, int n, int np,
                                                    const int2* __restrict__ pairs,
                                                    double* __restrict__ U, int64_t ldu,
                                                    double* __restrict__ V, int64_t ldv,
                                                    double tol, double atol,
                                                    int* __restrict__ counters,
                                                    int* __restrict__ sweeps_out) {
    // one CTA (JT threads) per column pair: long columns need the memory
    // parallelism of a whole CTA, a warp per pair was latency-bound
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[3][JT / 32];
    __shared__ double rot[3];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int rounds = np - 1, per = np / 2;
    int sweep = 0;
    for (; sweep < kMaxSweeps; ++sweep) {
        int mine = 0;
        for (int r = 0; r < rounds; ++r) {
            for (int q = blockIdx.x; q < per; q += gridDim.x) {
                int2 pr = pairs[r * per + q];
                if (pr.x >= n || pr.y >= n) continue;
                double* up = U + int64_t(pr.x) * ldu;
                double* uq = U + int64_t(pr.y) * ldu;
                double a = 0, b = 0, g = 0;
                for (int64_t i = threadIdx.x; i < m; i += JT) {
                    double x = up[i], y = uq[i];
                    a += x * x;
                    b += y * y;
                    g += x * y;
                }
                for (int o = 16; o > 0; o >>= 1) {
                    a += __shfl_xor_sync(0xffffffffu, a, o);
                    b += __shfl_xor_sync(0xffffffffu, b, o);
                    g += __shfl_xor_sync(0xffffffffu, g, o);
                }
                if (lane == 0) {
                    red[0][w] = a;
                    red[1][w] = b;
                    red[2][w] = g;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    double A = 0, B = 0, Gm = 0;
                    for (int k = 0; k < JT / 32; ++k) {
                        A += red[0][k];
                        B += red[1][k];
                        Gm += red[2][k];
                    }
                    rot[2] = 0.0;
                    if (Gm != 0.0 && fabs(Gm) > tol * sqrt(A * B) && fabs(Gm) > atol * sqrt(fmax(A, B))) {
                        double cs, sn;
                        rot_params(A, B, Gm, cs, sn);
                        rot[0] = cs;
                        rot[1] = sn;
                        rot[2] = 1.0;
                    }
                }
                __syncthreads();
                if (rot[2] != 0.0) {
                    const double cs = rot[0], sn = rot[1];
                    for (int64_t i = threadIdx.x; i < m; i += JT) {
                        double x = up[i], y = uq[i];
                        up[i] = cs * x - sn * y;
                        uq[i] = sn * x + cs * y;
                    }
                    if (V) {  // V == nullptr: right vectors recovered after the sweeps
                        double* vp = V + int64_t(pr.x) * ldv;
                        double* vq = V + int64_t(pr.y) * ldv;
                        for (int64_t i = threadIdx.x; i < n; i += JT) {
                            double x = vp[i], y = vq[i];
                            vp[i] = cs * x - sn * y;
                            vq[i] = sn * x + cs * y;
                        }
                    }
                    ++mine;
                }
                __syncthreads();
            }
            grid.sync();
        }
        if (threadIdx.x == 0 && mine) atomicAdd(&counters[sweep], mine);
        grid.sync();
        if (*((volatile int*)&counters[sweep]) == 0) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

// CTA-per-pair variant with the column pair held in registers (m <= EPT*JT):
// one read and (when rotated) one write of each column per round instead
// of read / re-read / write; every thread derives the rotation from the
// shared partial sums (no second block barrier).  V is never rotated here
// (lazy V only).
template <int EPT>
__global__ void __launch_bounds__(JT, EPT <= 4 ? 4 : (EPT <= 8 ? 3 : 2)) jacobi_coop_reg_k(int64_t m, int n, int np,
                                                        const int2* __restrict__ pairs,
                                                        double* __restrict__ U, int64_t ldu,
                                                        double tol, int* __restrict__ counters,
                                                        int* __restrict__ sweeps_out) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[2][3][JT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int rounds = np - 1, per = np / 2;
    int sweep = 0, parity = 0;
    for (; sweep < kMaxSweeps; ++sweep) {
        int mine = 0;
        for (int r = 0; r < rounds; ++r) {
            for (int q = blockIdx.x; q < per; q += gridDim.x) {
                int2 pr = pairs[r * per + q];
                if (pr.x >= n || pr.y >= n) continue;
                double* up = U + int64_t(pr.x) * ldu;
                double* uq = U + int64_t(pr.y) * ldu;
                double x[EPT], y[EPT];
                double a = 0, b = 0, g = 0;
#pragma unroll
                for (int e = 0; e < EPT; ++e) {
                    const int64_t i = threadIdx.x + int64_t(e) * JT;
                    x[e] = i < m ? up[i] : 0.0;
                    y[e] = i < m ? uq[i] : 0.0;
                }
#pragma unroll
                for (int e = 0; e < EPT; ++e) {
                    a += x[e] * x[e];
                    b += y[e] * y[e];
                    g += x[e] * y[e];
                }
                for (int o = 16; o > 0; o >>= 1) {
                    a += __shfl_xor_sync(0xffffffffu, a, o);
                    b += __shfl_xor_sync(0xffffffffu, b, o);
                    g += __shfl_xor_sync(0xffffffffu, g, o);
                }
                if (lane == 0) {
                    red[parity][0][w] = a;
                    red[parity][1][w] = b;
                    red[parity][2][w] = g;
                }
                __syncthreads();
                double A = 0, B = 0, Gm = 0;
#pragma unroll
                for (int k = 0; k < JT / 32; ++k) {
                    A += red[parity][0][k];
                    B += red[parity][1][k];
                    Gm += red[parity][2][k];
                }
                parity ^= 1;  // the next pair writes the other buffer: no trailing barrier
                if (Gm != 0.0 && fabs(Gm) > tol * sqrt(A * B)) {
                    double cs, sn;
                    rot_params(A, B, Gm, cs, sn);
#pragma unroll
                    for (int e = 0; e < EPT; ++e) {
                        const int64_t i = threadIdx.x + int64_t(e) * JT;
                        if (i < m) {
                            up[i] = cs * x[e] - sn * y[e];
                            uq[i] = sn * x[e] + cs * y[e];
                        }
                    }
                    ++mine;
                }
            }
            grid.sync();
        }
        if (threadIdx.x == 0 && mine) atomicAdd(&counters[sweep], mine);
        grid.sync();
        if (*((volatile int*)&counters[sweep]) == 0) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

// Block one-sided Jacobi for the lazy-V driver, register resident.  Columns
// are grouped in blocks of RB = 4; a global round pairs the blocks (circle
// method over nb blocks) and each CTA loads its block pair into registers --
// thread t holds rows t, t + 512, ... of all 8 columns -- and runs one full
// mini-sweep over the 28 column pairs: 7 sub-rounds of 4 disjoint pairs whose
// indices are compile-time constants (unrolled circle method), each sub-round
// one block reduction of the 12 dot products, rotations computed from the
// actual column dots (the point driver's accuracy) and applied in registers.
// Per sweep: nb-1 grid barriers and passes over U instead of n-1.
constexpr int RB = 4;            // default block width (columns)
constexpr int RMAXR = 5;         // max rows per thread at RB = 4 (5-9 measured: 5 fastest)

__host__ __device__ constexpr int circ_col(int pos, int r, int np) {
    return pos == 0 ? 0 : ((pos - 1 + r) % (np - 1)) + 1;
}

// Sub-round schedules of a block pair (columns 0..RBk-1 = block A, RBk..2RBk-1
// = block B), RBk disjoint column pairs each:
//   kind 0 "mini":  circle method over all 2 RBk columns (2 RBk - 1 sub-rounds)
//   kind 1 "cross": pair (k, RBk + (k + t) % RBk) (RBk sub-rounds: A x B once)
//   kind 2 "intra": circle method inside A and inside B (RBk - 1 sub-rounds)
template <int RBk>
__device__ __forceinline__ void sched_pair(int kind, int sr, int k, int& p, int& o) {
    constexpr int RC = 2 * RBk;
    if (kind == 0) {
        p = circ_col(k, sr, RC);
        o = circ_col(RC - 1 - k, sr, RC);
    } else if (kind == 1) {
        p = k;
        o = RBk + (k + sr) % RBk;
    } else {
        const int blk = k / (RBk / 2), kk = k % (RBk / 2);
        p = blk * RBk + circ_col(kk, sr, RBk);
        o = blk * RBk + circ_col(RBk - 1 - kk, sr, RBk);
    }
}

// One sub-round on the register-resident block pair x: the RBk column-pair
// dot products reduced over the CTA (warp transpose-reduce, one partial per
// warp), a warp per pair forms the rotation from the actual column dots,
// every thread applies the rotations to its rows.
template <int R, int RT, int RBk>
__device__ __forceinline__ void rblk_subround(int kind, int sr, double (&x)[R][2 * RBk], double (*red)[RT / 32],
                                              double* tot, int lane, int warp, double tol, int& mine) {
    constexpr int NW = RT / 32;
    constexpr int RNV = 3 * RBk;
    constexpr int NVP = RNV <= 8 ? 8 : RNV <= 16 ? 16 : 32;
    double part[NVP];  // the sub-round's dot products, padded
#pragma unroll
    for (int k = 0; k < RBk; ++k) {
        int p, o;
        sched_pair<RBk>(kind, sr, k, p, o);
        double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            a += x[rr][p] * x[rr][p];
            b += x[rr][o] * x[rr][o];
            g += x[rr][p] * x[rr][o];
        }
        part[3 * k] = a;
        part[3 * k + 1] = b;
        part[3 * k + 2] = g;
    }
#pragma unroll
    for (int v = RNV; v < NVP; ++v) part[v] = 0.0;
    // warp reduce: plain butterflies down to NVP lanes, then a
    // transpose-reduce -- lane l ends with quantity (l % NVP)
#pragma unroll
    for (int sft = 16; sft >= NVP; sft >>= 1)
#pragma unroll
        for (int v = 0; v < RNV; ++v) part[v] += __shfl_xor_sync(0xffffffffu, part[v], sft);
#pragma unroll
    for (int sft = NVP / 2; sft >= 1; sft >>= 1) {
        const bool upper = (lane & sft) != 0;
#pragma unroll
        for (int j = 0; j < sft; ++j) {
            const double send = upper ? part[j] : part[j + sft];
            const double keep = upper ? part[j + sft] : part[j];
            part[j] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
        }
    }
    if (lane < RNV) red[lane][warp] = part[0];
    __syncthreads();
    for (int k = warp; k < RBk; k += NW) {  // a warp finishes pair k, forms its rotation once
        double A = lane < NW ? red[3 * k][lane] : 0.0;
        double Bv = lane < NW ? red[3 * k + 1][lane] : 0.0;
        double G = lane < NW ? red[3 * k + 2][lane] : 0.0;
#pragma unroll
        for (int sft = NW / 2; sft > 0; sft >>= 1) {
            A += __shfl_xor_sync(0xffffffffu, A, sft);
            Bv += __shfl_xor_sync(0xffffffffu, Bv, sft);
            G += __shfl_xor_sync(0xffffffffu, G, sft);
        }
        if (lane == 0) {
            double cs = 1.0, sn = 0.0, on = 0.0;
            if (G != 0.0 && fabs(G) > tol * sqrt(A * Bv)) {
                rot_params(A, Bv, G, cs, sn);
                on = 1.0;
            }
            tot[3 * k] = cs;
            tot[3 * k + 1] = sn;
            tot[3 * k + 2] = on;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < RBk; ++k) {
        int p, o;
        sched_pair<RBk>(kind, sr, k, p, o);
        if (tot[3 * k + 2] != 0.0) {
            const double cs = tot[3 * k], sn = tot[3 * k + 1];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                const double xp = x[rr][p], xo = x[rr][o];
                x[rr][p] = cs * xp - sn * xo;
                x[rr][o] = sn * xp + cs * xo;
            }
            if (threadIdx.x == 0) ++mine;
        }
    }
}

// RBk = block width: 4 (8 columns per pair) or 2 (4 columns) -- the narrow
// form keeps cores up to 6144 rows in registers (12 rows x 4 columns per
// thread at 512 threads).
// Schedule per sweep (cross = 1, the default): in the sweep's first round
// every block's own column pairs (intra, RBk - 1 sub-rounds), then in every
// round the A x B cross pairs of the block pair (RBk sub-rounds): each
// column pair once per sweep, ~n sub-rounds per sweep.  cross = 0 runs the
// full 2 RBk - 1 sub-round mini-sweep on every block-pair visit (~2n per
// sweep): on the path's cores cross needs 0-1 more sweeps but 34-42 % fewer
// sub-rounds (offline, dumped cores).
template <int R, int RT, int RBk>
__global__ void __launch_bounds__(RT, 1) jacobi_rblk_k(int64_t m, int n, int nb, const int2* __restrict__ bpairs,
                                                      double* __restrict__ U, int64_t ldu, double tol,
                                                      int* __restrict__ counters, int* __restrict__ sweeps_out,
                                                      int cross, int stop_thr) {
    constexpr int NW = RT / 32;
    constexpr int RC = 2 * RBk;          // columns per block pair
    constexpr int RNV = 3 * RBk;         // dot products per sub-round
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[RNV][NW];
    __shared__ double tot[RNV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nbp = nb + (nb & 1);
    const int rounds = nbp - 1, per = nbp / 2;
    int sweep = 0;
    double x[R][RC];
    for (; sweep < kMaxSweeps; ++sweep) {
        int mine = 0;
        for (int r = 0; r < rounds; ++r) {
            for (int q = blockIdx.x; q < per; q += gridDim.x) {
                const int2 bp = bpairs[r * per + q];
                int col[RC];
#pragma unroll
                for (int j = 0; j < RC; ++j) {
                    const int blk = j < RBk ? bp.x : bp.y;
                    const int cj = blk * RBk + (j % RBk);
                    col[j] = (blk < nb && cj < n) ? cj : -1;
                }
#pragma unroll
                for (int j = 0; j < RC; ++j)
#pragma unroll
                    for (int rr = 0; rr < R; ++rr) {
                        const int64_t i = threadIdx.x + int64_t(rr) * RT;
                        x[rr][j] = (col[j] >= 0 && i < m) ? __ldcg(U + i + int64_t(col[j]) * ldu) : 0.0;
                    }
                if (cross) {
                    if (r == 0) {
#pragma unroll
                        for (int sr = 0; sr < RBk - 1; ++sr)
                            rblk_subround<R, RT, RBk>(2, sr, x, red, tot, lane, warp, tol, mine);
                    }
#pragma unroll
                    for (int t = 0; t < RBk; ++t)
                        rblk_subround<R, RT, RBk>(1, t, x, red, tot, lane, warp, tol, mine);
                } else {
#pragma unroll
                    for (int sr = 0; sr < RC - 1; ++sr)
                        rblk_subround<R, RT, RBk>(0, sr, x, red, tot, lane, warp, tol, mine);
                }
#pragma unroll
                for (int j = 0; j < RC; ++j)
#pragma unroll
                    for (int rr = 0; rr < R; ++rr) {
                        const int64_t i = threadIdx.x + int64_t(rr) * RT;
                        if (col[j] >= 0 && i < m) __stcg(U + i + int64_t(col[j]) * ldu, x[rr][j]);
                    }
            }
            grid.sync();
        }
        if (threadIdx.x == 0 && mine) atomicAdd(&counters[sweep], mine);
        grid.sync();
        if (*((volatile int*)&counters[sweep]) <= stop_thr) break;  // stop_thr > 0: the host checks the rest
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

__global__ void colnorm_k(int64_t m, int n, const double* __restrict__ U, int64_t ldu,
                          double* __restrict__ s) {
    __shared__ double sh[8];
    const double* u = U + int64_t(blockIdx.x) * ldu;
    double a = 0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) a += u[i] * u[i];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
        s[blockIdx.x] = sqrt(t);
    }
}

// U_out(:, j) = U(:, perm[j]) / s[perm[j]] ; V_out(:, j) = V(:, perm[j])
__global__ void finish_k(int64_t m, int n, const int* __restrict__ perm, const double* __restrict__ s,
                         const double* __restrict__ U, int64_t ldu, double* __restrict__ Uo,
                         int64_t lduo, const double* __restrict__ V, int64_t ldv,
                         double* __restrict__ Vo, int64_t ldvo) {
    int j = blockIdx.y;
    int src = perm[j];
    double sv = s[src];
    double inv = sv > 0.0 ? 1.0 / sv : 0.0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x)
        Uo[i + int64_t(j) * lduo] = sv > 0.0 ? U[i + int64_t(src) * ldu] * inv : 0.0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        Vo[i + int64_t(j) * ldvo] = V[i + int64_t(src) * ldv];
}

// Convergence check on the Gram matrix G = U^T U (one DMMA GEMM): list the
// pairs i < j with |g_ij| > tol sqrt(g_ii g_jj) -- the one-sided Jacobi
// rotation test of every pair on the current U.  The list order is made
// deterministic on the host (sorted).
__global__ void jacobi_violations_k(int n, const double* __restrict__ G, int64_t ldg, double tol,
                                    int cap, int* __restrict__ count, int2* __restrict__ list) {
    const int j = blockIdx.x;
    const double gjj = G[j + int64_t(j) * ldg];
    for (int i = threadIdx.x; i < j; i += blockDim.x) {
        const double g = G[i + int64_t(j) * ldg];
        const double gii = G[i + int64_t(i) * ldg];
        if (g != 0.0 && fabs(g) > tol * sqrt(gii * gjj)) {
            const int k = atomicAdd(count, 1);
            if (k < cap) list[k] = make_int2(i, j);
        }
    }
}

// Rotate the listed column pairs in order (one CTA), each from its actual
// column dot products -- the point driver's rotation.
__global__ void __launch_bounds__(512) jacobi_fix_k(int64_t m, int np, const int2* __restrict__ list,
                                                    double* __restrict__ U, int64_t ldu, double tol) {
    __shared__ double red[3][16];
    __shared__ double rot[3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = 0; k < np; ++k) {
        const int2 pq = list[k];
        double* up = U + int64_t(pq.x) * ldu;
        double* uq = U + int64_t(pq.y) * ldu;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
            const double x = up[i], y = uq[i];
            a += x * x;
            b += y * y;
            g += x * y;
        }
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (lane == 0) {
            red[0][warp] = a;
            red[1][warp] = b;
            red[2][warp] = g;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double A = 0.0, B = 0.0, Gv = 0.0;
            for (int w = 0; w < int(blockDim.x >> 5); ++w) {
                A += red[0][w];
                B += red[1][w];
                Gv += red[2][w];
            }
            double cs = 1.0, sn = 0.0, on = 0.0;
            if (Gv != 0.0 && fabs(Gv) > tol * sqrt(A * B)) {
                rot_params(A, B, Gv, cs, sn);
                on = 1.0;
            }
            rot[0] = cs;
            rot[1] = sn;
            rot[2] = on;
        }
        __syncthreads();
        if (rot[2] != 0.0) {
            const double cs = rot[0], sn = rot[1];
            for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
                const double x = up[i], y = uq[i];
                up[i] = cs * x - sn * y;
                uq[i] = sn * x + cs * y;
            }
        }
        __syncthreads();
    }
}

// circle-method tournament: rounds x (np/2) pairs
std::vector<int2> tournament(int n, int& np) {
    np = n + (n & 1);
    std::vector<int> p(static_cast<size_t>(np));
    std::iota(p.begin(), p.end(), 0);
    std::vector<int2> out;
    out.reserve(size_t(np / 2) * size_t(np - 1));
    for (int r = 0; r < np - 1; ++r) {
        for (int i = 0; i < np / 2; ++i) {
            int a = p[size_t(i)], b = p[size_t(np - 1 - i)];
            out.push_back(make_int2(std::min(a, b), std::max(a, b)));
        }
        int last = p[size_t(np - 1)];
        for (int i = np - 1; i > 1; --i) p[size_t(i)] = p[size_t(i - 1)];
        p[1] = last;
    }
    return out;
}

// per-process cache of tournament tables in device memory, keyed by
// (device, n); contexts on several devices may use it from several threads
struct PairCache {
    int device = -1, n = -1, np = 0;
    int2* dev = nullptr;
};

const int2* device_pairs(Ctx& c, int n, int& np) {
    static std::mutex mu;
    static std::vector<PairCache> cache;
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : cache)
        if (e.n == n && e.device == c.device) {
            np = e.np;
            return e.dev;
        }
    std::vector<int2> pairs = tournament(n, np);
    PairCache pc;
    pc.device = c.device;
    pc.n = n;
    pc.np = np;
    HYDOT_CUDA(cudaMalloc(&pc.dev, std::max<size_t>(pairs.size(), 1) * sizeof(int2)));
    if (!pairs.empty())
        HYDOT_CUDA(cudaMemcpy(pc.dev, pairs.data(), pairs.size() * sizeof(int2), cudaMemcpyHostToDevice));
    if (cache.size() > 256) {
        int cur = 0;  // cudaFree synchronises the device: in-flight users finish first
        cudaGetDevice(&cur);
        cudaSetDevice(cache.front().device);
        cudaFree(cache.front().dev);
        cudaSetDevice(cur);
        cache.erase(cache.begin());
    }
    cache.push_back(pc);
    return pc.dev;
}

// register block-Jacobi for the lazy-V driver: 4-column blocks with the
// fewest threads T (a power of two >= 64) holding <= RMAXR rows each -- the
// per-sub-round reduction costs instructions per warp, so fat threads win;
// cores too long for that use 2-column blocks at 512 threads (<= 12 rows
// per thread, m <= 6144).  false = not used.
bool rblk_shape(int64_t m, int64_t n, int& R, int& T, int& B) {
    // at least 128 threads: with 64 each of the 2 warps forms two rotations
    // per sub-round in sequence (111-320-row cores: 242 -> 174 ms per
    // config-1 step at 128; 206 ms at 256)
    constexpr int tmin = 128;
    // 256 threads may hold 9 rows each (1153-2304-row cores): fewer warps
    // per sub-round reduction, 2172^2 core 131 -> 112 ms; at 128 threads 9
    // rows measured slower than 256 x 5
    constexpr int rmax256 = 9;
    B = RB;
    if ((n + RB - 1) / RB >= 4) {
        for (T = tmin; T <= 512; T *= 2) {
            R = int((m + T - 1) / T);
            const int cap = T == 512 ? 5 : T == 256 ? rmax256 : RMAXR;  // 512 threads: 128 registers each
            if (R <= cap) {
                R = R <= 3 ? 3 : R <= 5 ? 5 : 9;  // instantiated row counts
                // (8-column blocks measured slower: Jacobi 454 -> 566 ms per
                // config-1 step, 24-value reductions and register pressure)
                return true;
            }
        }
    }
    // 2-column blocks only beyond the register point driver's reach (m >
    // 4096): at 3000 rows they measured on par with it (681 vs 650 ms), at
    // 5686 rows 1.65x faster than the CTA-per-pair driver (5.1 vs 8.5 s)
    if (m <= 16 * JT) return false;
    B = 2;
    T = 512;
    R = int((m + T - 1) / T);
    if (R > 12 || (n + 1) / 2 < 4) return false;
    R = R <= 6 ? 6 : R <= 9 ? 9 : 12;
    return true;
}

template <int R, int T, int B>
void launch_rblk_t(Ctx& c, int64_t m, int64_t n, double* U, int64_t ldu, double tol, int* counters,
                   int* sweeps_out, int stop_thr) {
    int nb = int((n + B - 1) / B);
    int npb = 0;
    const int2* bp = device_pairs(c, nb, npb);
    int per_sm = 0;
    HYDOT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_rblk_k<R, T, B>, T, 0));
    int grid = std::max(1, std::min(npb / 2, per_sm * c.num_sms));
    int64_t mm = m;
    int nn = int(n), nbb = nb;
    int cross = 1;  // cross schedule (a full mini-sweep per visit needs 34-42 % more sub-rounds)
    void* args[] = {&mm, &nn, &nbb, &bp, &U, &ldu, &tol, &counters, &sweeps_out, &cross, &stop_thr};
    c.coop_launch((void*)jacobi_rblk_k<R, T, B>, dim3(grid), dim3(T), args, 0);
    c.count();
}

void launch_rblk(Ctx& c, int R, int T, int B, int64_t m, int64_t n, double* U, int64_t ldu, double tol,
                 int* counters, int* sweeps_out, int stop_thr) {
    if (B == 2) {
        switch (R) {
            case 6: launch_rblk_t<6, 512, 2>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr); break;
            case 9: launch_rblk_t<9, 512, 2>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr); break;
            default: launch_rblk_t<12, 512, 2>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr); break;
        }
        return;
    }
    if (R == 9) {
        if (T == 128) launch_rblk_t<9, 128, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr);
        else launch_rblk_t<9, 256, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr);
        return;
    }
    const bool r3 = R == 3;
    switch (T) {
        case 64: r3 ? launch_rblk_t<3, 64, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr)
                    : launch_rblk_t<5, 64, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr); break;
        case 128: r3 ? launch_rblk_t<3, 128, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr)
                     : launch_rblk_t<5, 128, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr); break;
        case 256: r3 ? launch_rblk_t<3, 256, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr)
                     : launch_rblk_t<5, 256, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr); break;
        default: r3 ? launch_rblk_t<3, 512, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr)
                    : launch_rblk_t<5, 512, RB>(c, m, n, U, ldu, tol, counters, sweeps_out, stop_thr); break;
    }
}

thread_local bool g_strict_svd = false;
bool strict_svd_flag() { return g_strict_svd; }
bool lazy_v_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("HYDOT_JACOBI_LAZYV");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool stats_on() {
    static int on = [] {
        const char* e = std::getenv("HYDOT_JACOBI_STATS");
        return (e && e[0] == '1') ? 1 : 0;
    }();
    return on != 0;
}

}  // namespace

namespace {
// HYDOT_JACOBI_TAIL=0: plain sweeps to a zero-rotation sweep
bool gram_tail_on() {
    static const bool on = [] {
        const char* e = std::getenv("HYDOT_JACOBI_TAIL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Register block-Jacobi to convergence.  The last sweeps of a one-sided
// Jacobi rotate a handful of pairs (e.g. ... 3791, 8, 0 on the 2172^2 root
// core) and the final one only verifies.  Sweeps therefore stop once a sweep
// rotates <= 12 n pairs; then the rotation test of every pair is evaluated at
// once on G = U^T U (one GEMM), the few violating pairs are rotated from
// their actual columns (jacobi_fix_k), and the test repeats -- the stopping
// state is the sweep criterion (no pair fails the test, at 2 tol: see
// below).  Too many violations fall back to sweeps.
void rblk_converge(Ctx& c, int R, int T, int B, int64_t m, int64_t n, double* U, double tol, DBuf& sw) {
    int* counters = sw.as<int>();
    int* sweeps_out = sw.as<int>() + kMaxSweeps;
    if (!gram_tail_on() || n < 64) {
        launch_rblk(c, R, T, B, m, n, U, m, tol, counters, sweeps_out, 0);
        return;
    }
    // a sweep of <= 12 n rotations is followed by one of at most a few hundred
    // on the path's cores; fixing a pair costs ~1/100 of a sweep at n = 300
    const int cap = int(std::clamp<int64_t>(n / 4, 16, 256));
    constexpr int tailk = 12;  // the stop threshold in units of n (12 / 20 / 30 measured within noise)
    launch_rblk(c, R, T, B, m, n, U, m, tol, counters, sweeps_out, int(std::min<int64_t>(tailk * n, 1 << 30)));
    DBuf G = dalloc(c, size_t(n * n));
    DBuf cnt(c, sizeof(int));
    DBuf lst(c, sizeof(int2) * cap);
    for (int round = 0; round < 4; ++round) {
        dgemm(c, true, false, n, n, m, 1.0, U, m, U, m, 0.0, G.d(), n);
        HYDOT_CUDA(cudaMemsetAsync(cnt.as<void>(), 0, sizeof(int), c.stream));
        // test at 2 tol: tol = sqrt(m) eps is the rounding level of a column
        // dot product itself, so pairs within a factor 2 of it are noise
        // (the GEMM and the fix kernel sum in different orders and would
        // disagree on them forever); real violations are far above
        jacobi_violations_k<<<unsigned(n), 128, 0, c.stream>>>(int(n), G.d(), n, 2.0 * tol, cap, cnt.as<int>(),
                                                             lst.as<int2>());
        c.check_launch();
        int nv = 0;
        HYDOT_CUDA(cudaMemcpyAsync(&nv, cnt.as<void>(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (stats_on()) fprintf(stderr, "[jacobi-tail] n=%lld round=%d violations=%d\n", (long long)n, round, nv);
        if (nv == 0) return;
        if (nv > cap) break;
        std::vector<int2> h(static_cast<size_t>(nv));
        HYDOT_CUDA(cudaMemcpyAsync(h.data(), lst.as<void>(), sizeof(int2) * size_t(nv), cudaMemcpyDeviceToHost,
                                   c.stream));
        c.sync();
        std::sort(h.begin(), h.end(), [](int2 a, int2 b) { return a.y != b.y ? a.y < b.y : a.x < b.x; });
        HYDOT_CUDA(cudaMemcpyAsync(lst.as<void>(), h.data(), sizeof(int2) * size_t(nv), cudaMemcpyHostToDevice,
                                   c.stream));
        jacobi_fix_k<<<1, 512, 0, c.stream>>>(m, nv, lst.as<int2>(), U, m, tol);
        c.check_launch();
        c.sync();  // h goes out of scope
    }
    // many violations left: plain sweeps to convergence
    HYDOT_CUDA(cudaMemsetAsync(counters, 0, sizeof(int) * kMaxSweeps, c.stream));
    launch_rblk(c, R, T, B, m, n, U, m, tol, counters, sweeps_out, 0);
}
}  // namespace

StrictSVD::StrictSVD() : prev_(g_strict_svd) { g_strict_svd = true; }
StrictSVD::~StrictSVD() { g_strict_svd = prev_; }

void jacobi_svd(Ctx& c, int64_t m, int64_t n, const double* X, int64_t ldx, double* Uo,
                int64_t lduo, std::vector<double>& s, double* Vo, int64_t ldvo) {
    StageTimer _t(c, n > 96 ? "svd_jacobi_large" : "svd_jacobi_small", m, n, -1,
                  14.0 * double(std::max(m, n)) * double(std::min(m, n)) * double(std::min(m, n)));
    s.assign(static_cast<size_t>(std::max<int64_t>(n, 0)), 0.0);
    if (n <= 0) return;
    if (m < n) throw std::invalid_argument("jacobi_svd: needs m >= n");
    // LAPACK dgesvj's convergence threshold: sqrt(m) * eps
    const double tol = std::max(1e-15, std::sqrt(double(m)) * 2.220446049250313e-16);
    if (stats_on()) c.sync();
    const auto t_start = std::chrono::steady_clock::now();
    int np = 0;
    const int2* dpairs = device_pairs(c, int(n), np);
    DBuf U = dalloc(c, size_t(m * n));
    DBuf V = dalloc(c, size_t(n * n));
    copy2d(c, m, n, X, ldx, U.d(), m);
    // No absolute rotation floor (atol = 0): one at eps ||A|| saved few sweeps
    // on the path's cores and leaves the vectors of negligible singular
    // values non-orthonormal, unlike BDCSVD.
    const double atol = 0.0;
    DBuf sw(c, sizeof(int) * (kMaxSweeps + 1));
    HYDOT_CUDA(cudaMemsetAsync(sw.as<void>(), 0, sizeof(int) * (kMaxSweeps + 1), c.stream));
    bool lazy_v = false;
    const size_t smem = size_t((m + n) * n) * sizeof(double);
    // (a U-only single-CTA variant for 110 < n <= 160 measured 2x slower
    // than the multi-SM block driver: one SM's FP64 rate bounds each round)
    if (n >= 2 && smem <= 200 * 1024) {
        static AttrGate attr;
        attr_once(attr, c.device, [&] {
            HYDOT_CUDA(cudaFuncSetAttribute(jacobi_smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            210 * 1024));
        });
        jacobi_smem_k<<<1, 1024, smem, c.stream>>>(int(m), int(n), np, dpairs, U.d(), m, V.d(), n,
                                                    tol, atol, sw.as<int>() + kMaxSweeps);
        c.check_launch();
    } else if (n >= bjacobi_min_n() && !strict_svd_flag() && lazy_v_enabled() && atol == 0.0) {
        lazy_v = true;
        const int sweeps = bjacobi_converge(c, m, n, U.d(), tol);
        HYDOT_CUDA(cudaMemcpyAsync(sw.as<int>() + kMaxSweeps, &sweeps, sizeof(int), cudaMemcpyHostToDevice,
                                   c.stream));
        c.sync();
    } else if (int rbR = 0, rbT = 0, rbB = 0; n >= 2 && !strict_svd_flag() && lazy_v_enabled() && atol == 0.0 &&
                                               rblk_shape(m, n, rbR, rbT, rbB)) {
        lazy_v = true;
        rblk_converge(c, rbR, rbT, rbB, m, n, U.d(), tol, sw);
    } else {
        set_identity(c, n, n, V.d(), n);
        if (n >= 2) {
            int per_sm = 0;
            static const bool reg_env = [] {
                const char* e = std::getenv("HYDOT_JACOBI_REG");
                return !(e && e[0] == '0');
            }();
            lazy_v = !strict_svd_flag() && lazy_v_enabled();
            const bool reg_mode = lazy_v && atol == 0.0 && reg_env && m <= 16 * JT;
            void* kern = (void*)jacobi_coop_k;
            if (reg_mode) {
                kern = m <= 4 * JT   ? (void*)jacobi_coop_reg_k<4>
                       : m <= 8 * JT ? (void*)jacobi_coop_reg_k<8>
                                     : (void*)jacobi_coop_reg_k<16>;
            }
            HYDOT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, JT, 0));
            const int per = np / 2;
            int want = per;
            int grid = std::max(1, std::min(want, per_sm * c.num_sms));
            int64_t mm = m;
            int nn = int(n), npp = np;
            double* up = U.d();
            double* vp = lazy_v ? nullptr : V.d();
            int64_t ldu = m, ldv = n;
            double tl = tol, at = atol;
            int* cnt = sw.as<int>();
            int* so = sw.as<int>() + kMaxSweeps;
            const int2* pp = dpairs;
            void* args[] = {&mm, &nn, &npp, &pp, &up, &ldu, &vp, &ldv, &tl, &at, &cnt, &so};
            void* rargs[] = {&mm, &nn, &npp, &pp, &up, &ldu, &tl, &cnt, &so};
            c.coop_launch(kern, dim3(grid), dim3(JT), reg_mode ? rargs : args, 0);
            c.count();
        }
    }
    if (stats_on()) {
        int sweeps = 0;
        HYDOT_CUDA(cudaMemcpyAsync(&sweeps, sw.as<int>() + kMaxSweeps, sizeof(int),
                                   cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        int rots[kMaxSweeps + 1];
        HYDOT_CUDA(cudaMemcpyAsync(rots, sw.as<int>(), sizeof(int) * (kMaxSweeps + 1), cudaMemcpyDeviceToHost,
                                   c.stream));
        c.sync();
        std::string rs;
        for (int i = 0; i <= sweeps && i < kMaxSweeps; ++i) rs += std::to_string(rots[i]) + " ";
        fprintf(stderr, "[jacobi] m=%lld n=%lld sweeps=%d ms=%.3f rot/sweep: %s\n", (long long)m, (long long)n,
                sweeps, dt * 1e3, rs.c_str());
    }
    DBuf sd = dalloc(c, size_t(n));
    colnorm_k<<<unsigned(n), 256, 0, c.stream>>>(m, int(n), U.d(), m, sd.d());
    c.check_launch();
    std::vector<double> sv(static_cast<size_t>(n));
    c.d2h(sv.data(), sd.d(), size_t(n));
    if (lazy_v) {
        // right vectors from X = U S V^T:  V = X^T W S^-2 with W = U S the
        // rotated columns (one DMMA GEMM instead of rotating V every round);
        // column j carries an error eps ||X|| / s_j, i.e. backward-stable
        // for every kept triple (s_j > eps_tol s_1 >> eps s_1); columns
        // with s_j below 1e-14 s_1 are set to zero (never kept).
        dgemm(c, true, false, n, n, m, 1.0, X, ldx, U.d(), m, 0.0, V.d(), n);
        const double smax = *std::max_element(sv.begin(), sv.end());
        std::vector<double> inv(static_cast<size_t>(n));
        for (int64_t j = 0; j < n; ++j) {
            const double sj = sv[size_t(j)];
            inv[size_t(j)] = (sj > 1e-14 * smax && sj > 0.0) ? 1.0 / (sj * sj) : 0.0;
        }
        DBuf dinv = dalloc(c, size_t(n));
        HYDOT_CUDA(cudaMemcpyAsync(dinv.d(), inv.data(), size_t(n) * 8, cudaMemcpyHostToDevice,
                                   c.stream));
        scale_cols(c, n, n, V.d(), n, dinv.d());
        c.sync();
    }
    std::vector<int> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(),
                     [&](int a, int b) { return sv[size_t(a)] > sv[size_t(b)]; });
    for (int64_t j = 0; j < n; ++j) s[size_t(j)] = sv[size_t(perm[size_t(j)])];
    DBuf dperm(c, size_t(n) * sizeof(int));
    HYDOT_CUDA(cudaMemcpyAsync(dperm.as<void>(), perm.data(), size_t(n) * sizeof(int),
                               cudaMemcpyHostToDevice, c.stream));
    int gx = int(std::min<int64_t>((std::max(m, n) + 255) / 256, 64));
    finish_k<<<dim3(unsigned(gx), unsigned(n)), 256, 0, c.stream>>>(
        m, int(n), dperm.as<int>(), sd.d(), U.d(), m, Uo, lduo, V.d(), n, Vo, ldvo);
    c.check_launch();
    c.sync();
}

}  // namespace hydot
