// qr_cqr.cu -- Householder panels of very tall matrices without a grid
// barrier per column.
//
// The cooperative panel (qr.cu) needs one grid-wide reduction per column; on
// the path's tallest panels (N = 262 144 rows at config 2: a 67 MB panel that
// no longer fits on chip) that cost ~30 us per column.  Here the mr x jb
// (jb <= 32) panel is factored by shifted CholeskyQR3 (Fukaya, Nakatsukasa,
// Yanagisawa, Yamamoto 2020): three passes of "Gram -> Cholesky -> row-wise
// triangular solve", the first with the shift s = 11 (mr jb + jb (jb + 1)) u
// tr(P^T P) so that it is stable for ill-conditioned and rank-deficient
// panels, giving P = Q R with Q orthonormal to working precision.  The
// Householder representation the blocked QR needs (unit-lower V, tau, the
// upper R; LAPACK dgeqrf / Eigen HouseholderQR layout, lowrank.cpp:77-83) is
// then reconstructed from Q (Ballard, Demmel, Grigori, Jacquelin, Nguyen,
// Solomonik 2014): the LU factorisation Q - [S; 0] = V U with the signs
// s_k = -sign of the running pivot (|u_kk| >= 1, no pivoting needed) gives
// H_1 ... H_jb = I - V T V^T with first jb columns Q S, T = -U S V_1^-T, so
// tau_k = -s_k u_kk and R_house = S R.  Four launches per panel, each one
// pass over the panel: Gram(P) | Q1 = P R1^-1 + Gram | Q2 = Q1 R2^-1 + Gram
// (+ the top block's LU) | V = Q2 R3^-1 U^-1 below the top block.  Gram
// partials are reduced by the last CTA in CTA order (deterministic).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace hydot {
namespace {

constexpr int W = 32;       // panel width handled (jb <= W)
constexpr int RT = 128;     // threads = rows per tile
constexpr int GSZ = W * W;  // Gram entries
constexpr int XS = RT + 4;  // tile stride ([col][row])
constexpr int GRP = 16;     // CTAs per first-level reduction group
constexpr int CTAS_PER_SM = 2;  // resident CTAs streaming the panel (tiles in flight per SM)
constexpr int MAXGRP = 64;

__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// stage rows [r0, r0 + RT) of the panel's jb columns into buf[col][row]
// (zero-filled outside), 8-byte copies (any leading dimension)
__device__ __forceinline__ void stage_tile(double* buf, const double* __restrict__ X, int64_t ldx, int64_t r0,
                                           int64_t mr, int jb) {
#pragma unroll 8
    for (int e = threadIdx.x; e < RT * W; e += RT) {
        const int i = e % RT, j = e / RT;
        const bool ok = r0 + i < mr && j < jb;
        cp_async8(buf + j * XS + i, ok ? X + r0 + i + int64_t(j) * ldx : X, ok);
    }
}

struct CqrBufs {
    double* part;      // gridDim x GSZ partial Grams
    double* gpart;     // group sums (MAXGRP x GSZ)
    unsigned* ticket;  // last-group ticket (self-resetting)
    unsigned* gticket;  // per-group last-CTA tickets (self-resetting)
    double* R;         // 3 x W x W: R1, R2, R3 (upper, column-major W x W)
    double* U;         // W x W: U of the top block's LU
    int* status;       // [0]: 1 = zero panel, 2 = Q not orthonormal (panel left untouched)
    int* sticky;       // the factorisation's flag: raised to 2 when any panel is left untouched
    double* T;         // jb x jb compact-WY triangle of the panel's reflectors (ld ldt), may be null
    int64_t ldt;
};

// |G3 - I| bound below which Q2 is treated as orthonormal (then Q = Q2 R3^-1
// is orthonormal to working precision); above it the panel is left to the
// Householder kernel
constexpr double kOrthTol = 1e-6;

// y = x R^-1 for a row vector x (jb), R upper triangular (column-major W x W
// in shared memory), invd[j] = 1 / R_jj: y_j = (x_j - sum_{i<j} y_i R_ij) /
// R_jj by substitution (backward stable per row), the inner sum split in
// four independent chains
__device__ __forceinline__ void row_solve(double (&x)[W], const double* __restrict__ R,
                                          const double* __restrict__ invd, int jb) {
#pragma unroll
    for (int j = 0; j < W; ++j) {
        if (j < jb) {
            double s0 = x[j], s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int i = 0; i < W; i += 4) {
                if (i < j) s0 -= x[i] * R[i + j * W];
                if (i + 1 < j) s1 -= x[i + 1] * R[i + 1 + j * W];
                if (i + 2 < j) s2 -= x[i + 2] * R[i + 2 + j * W];
                if (i + 3 < j) s3 -= x[i + 3] * R[i + 3 + j * W];
            }
            x[j] = ((s0 + s1) + (s2 + s3)) * invd[j];
        }
    }
}

// v[k] for a runtime k without dynamic register indexing
__device__ __forceinline__ double pick(const double (&v)[W], int k) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < W; ++i) r = i == k ? v[i] : r;
    return r;
}

// Cholesky of the jb x jb Gram (+ shift) by one warp, lane j holding column
// j in registers: G + s I = R^T R, R upper (column-major W x W in shared
// memory; identity outside jb, zero below the diagonal).  Retries with a
// 10x larger shift if a pivot is not positive.
__device__ void warp_cholesky(const double* __restrict__ G, double* __restrict__ R, int jb, double shift,
                              double* tr_out) {
    const int lane = threadIdx.x;
    double tr = 0.0;
    for (int i = 0; i < jb; ++i) tr += G[i + i * W];
    if (tr_out && lane == 0) *tr_out = tr;
    double s = shift * tr;
    for (int attempt = 0; attempt < 12; ++attempt) {
        double col[W];
#pragma unroll
        for (int i = 0; i < W; ++i) col[i] = (lane < jb && i < jb) ? G[i + lane * W] + (i == lane ? s : 0.0) : 0.0;
        bool ok = true;
        for (int k = 0; k < jb; ++k) {
            const double akj = pick(col, k);
            const double akk = __shfl_sync(0xffffffffu, akj, k);
            if (!(akk > 0.0)) {
                ok = false;
                break;
            }
            const double d = sqrt(akk);
            const double rkj = (lane >= k && lane < jb) ? (lane == k ? d : akj / d) : 0.0;
            if (lane < jb) R[k + lane * W] = rkj;
#pragma unroll
            for (int i = 0; i < W; ++i) {  // a_ij -= r_ki r_kj for i > k
                const double rki = __shfl_sync(0xffffffffu, rkj, i);
                if (i > k) col[i] -= rki * rkj;
            }
        }
        if (ok) {
            __syncwarp();
            for (int e = lane; e < W * W; e += 32) {
                const int i = e % W, j = e / W;
                if (i >= jb || j >= jb) R[e] = i == j ? 1.0 : 0.0;
                else if (i > j) R[e] = 0.0;
            }
            __syncwarp();
            return;
        }
        s = s > 0.0 ? s * 10.0 : 1e-16 * tr + 1e-300;
    }
}

// One pass over the panel rows: optionally y = x Rin^-1 (stored to Y), and the
// Gram of y (or x) reduced by the last CTA, which then factors it (mode 0:
// shifted, into R slot `slot`; the last pass also does the reconstruction).
// mode: 0 = Gram(P) + shifted Cholesky -> R1
//       1 = Q1 = P R1^-1 (-> Y) + Gram + Cholesky -> R2
//       2 = Q2 = Q1 R2^-1 (-> Y) + Gram + Cholesky -> R3, then the top
//           block's modified LU -> U, tau, R_house, V_1 written into P
template <int MODE>
__global__ void __launch_bounds__(RT) cqr_pass_k(int64_t mr, int jb, const double* __restrict__ X, int64_t ldx,
                                                 double* __restrict__ Y, int64_t ldy, double* __restrict__ P,
                                                 int64_t ldp, double* __restrict__ tau, CqrBufs b, double shift) {
    extern __shared__ __align__(16) double dyn[];  // 2 x W x XS: double-buffered row tiles
    double* tile = dyn;
    __shared__ double Rin[W * W];
    __shared__ double invd[W];
    __shared__ bool last;
    // the last CTA reuses the tile after the row loop
    double* Gs = tile;              // Gram, then Q's top block / LU
    double* Rs = tile + W * W;      // this pass's Cholesky factor
    double* R12 = tile + 2 * W * W;  // R2 R1 (last pass)
    double* R1s = tile + 3 * W * W;  // R1, then R2 staged from global (4 W W <= W XS)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wi = (warp & 1) * 16, wj = (warp >> 1) * 16;
    if (MODE > 0 && b.status[0]) return;  // zero panel: nothing to do
    if (MODE > 0) {
        for (int e = threadIdx.x; e < W * W; e += RT) Rin[e] = b.R[(MODE - 1) * W * W + e];
        __syncthreads();
        if (threadIdx.x < W) invd[threadIdx.x] = 1.0 / Rin[threadIdx.x * (W + 1)];
    }
    __syncthreads();
    double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    const int64_t ntiles = (mr + RT - 1) / RT;
    // tile k of this CTA lives in buffer k & 1; the next tile's copies are
    // in flight while the current one is solved and accumulated
    int64_t tt = blockIdx.x;
    if (tt < ntiles) stage_tile(dyn, X, ldx, tt * RT, mr, jb);
    cp_commit();
    for (int k = 0; tt < ntiles; tt += gridDim.x, ++k) {
        double* cur = dyn + (k & 1) * (W * XS);
        double* nxt = dyn + ((k + 1) & 1) * (W * XS);
        if (tt + gridDim.x < ntiles) stage_tile(nxt, X, ldx, (tt + gridDim.x) * RT, mr, jb);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const int64_t i = tt * RT + threadIdx.x;
        if (MODE > 0) {
            double x[W];
#pragma unroll
            for (int j = 0; j < W; ++j) x[j] = cur[j * XS + threadIdx.x];
            if (i < mr) row_solve(x, Rin, invd, jb);
#pragma unroll
            for (int j = 0; j < W; ++j) {
                if (i < mr && j < jb) __stcg(Y + i + int64_t(j) * ldy, x[j]);
                cur[j * XS + threadIdx.x] = x[j];
            }
            __syncthreads();
        }
#pragma unroll
        for (int kk = 0; kk < RT; kk += 4) {
            const double a0 = cur[(wi + g) * XS + kk + t];
            const double a1 = cur[(wi + g + 8) * XS + kk + t];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) dmma(acc[ni], a0, a1, cur[(wj + ni * 8 + g) * XS + kk + t]);
        }
        __syncthreads();  // cur is refilled two tiles later
    }
    cp_wait<0>();
    double* mine = b.part + int64_t(blockIdx.x) * GSZ;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int r = wi + g + ((v & 2) ? 8 : 0);
            const int cc = wj + ni * 8 + 2 * t + (v & 1);
            __stcg(mine + r + cc * W, acc[ni][v]);
        }
    // Two-level reduction in a fixed order (deterministic): the last CTA of
    // each group of GRP consecutive CTAs sums the group's partials in CTA
    // order, the last group to finish sums the group sums in group order.
    // (One CTA walking all ~300 partials was an L2 round trip per four of
    // them: the tail of every pass.)
    const int ngrp = (int(gridDim.x) + GRP - 1) / GRP, grp = int(blockIdx.x) / GRP;
    const int gfirst = grp * GRP, gcount = min(GRP, int(gridDim.x) - gfirst);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(b.gticket + grp, 1u) == unsigned(gcount - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    constexpr int EPT = W * W / RT;  // 8 entries per thread
    auto sum_in_order = [&](const double* base, int np, double (&s)[EPT]) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) s[k] = 0.0;
        int p = 0;
        for (; p + 4 <= np; p += 4) {  // four partials per step, all 32 loads in flight
            double v[4][EPT];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int k = 0; k < EPT; ++k) v[q][k] = __ldcg(base + int64_t(p + q) * GSZ + threadIdx.x + k * RT);
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int k = 0; k < EPT; ++k) s[k] += v[q][k];
        }
        for (; p < np; ++p)
#pragma unroll
            for (int k = 0; k < EPT; ++k) s[k] += __ldcg(base + int64_t(p) * GSZ + threadIdx.x + k * RT);
    };
    {
        double s[EPT];
        sum_in_order(b.part + int64_t(gfirst) * GSZ, gcount, s);
#pragma unroll
        for (int k = 0; k < EPT; ++k) __stcg(b.gpart + int64_t(grp) * GSZ + threadIdx.x + k * RT, s[k]);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        b.gticket[grp] = 0u;  // ready for the next launch on this stream
        last = atomicAdd(b.ticket, 1u) == unsigned(ngrp - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    {
        double s[EPT];
        sum_in_order(b.gpart, ngrp, s);
#pragma unroll
        for (int k = 0; k < EPT; ++k) Gs[threadIdx.x + k * RT] = s[k];
    }
    __syncthreads();
    __shared__ double tr0;
    if (warp == 0) warp_cholesky(Gs, Rs, jb, MODE == 0 ? shift : 0.0, MODE == 0 ? &tr0 : nullptr);
    __syncthreads();
    if (MODE == 0 && tr0 == 0.0) {  // zero panel: H = I, R = 0
        if (threadIdx.x == 0) b.status[0] = 1;
        for (int e = threadIdx.x; e < jb * jb; e += RT) {
            const int r = e % jb, cc = e / jb;
            P[r + int64_t(cc) * ldp] = 0.0;
        }
        for (int j = threadIdx.x; j < jb; j += RT) tau[j] = 0.0;
        if (b.T)
            for (int e = threadIdx.x; e < jb * jb; e += RT) b.T[e % jb + int64_t(e / jb) * b.ldt] = 0.0;
        for (int64_t e = threadIdx.x; e < (mr - jb) * jb; e += RT)
            P[jb + e % (mr - jb) + int64_t(e / (mr - jb)) * ldp] = 0.0;
        if (threadIdx.x == 0) *b.ticket = 0u;
        return;
    }
    if (MODE == 2) {  // Q2 must be orthonormal to O(sqrt u) for the reconstruction
        __shared__ int bad;
        if (threadIdx.x == 0) bad = 0;
        __syncthreads();
        for (int e = threadIdx.x; e < jb * jb; e += RT) {
            const int r = e % jb, cc = e / jb;
            const double v = Gs[r + cc * W] - (r == cc ? 1.0 : 0.0);
            if (!(fabs(v) <= kOrthTol)) bad = 1;
        }
        __syncthreads();
        if (bad) {
            if (threadIdx.x == 0) {
                b.status[0] = 2;
                atomicMax(b.sticky, 2);
                *b.ticket = 0u;
            }
            return;
        }
    }
    for (int e = threadIdx.x; e < W * W; e += RT) b.R[MODE * W * W + e] = Rs[e];
    if (MODE == 2) {
        // top block of Q = Q2 R3^-1 (rows 0..jb-1), then the modified LU
        __shared__ double invr[W];
        __shared__ double sgn[W];
        if (threadIdx.x < W) invr[threadIdx.x] = 1.0 / Rs[threadIdx.x * (W + 1)];
        // R12 = R2 R1 (upper), both staged in shared memory (R2 into R12's
        // space first, R1 beside it)
        for (int e = threadIdx.x; e < W * W; e += RT) {
            R12[e] = __ldcg(b.R + W * W + e);
            R1s[e] = __ldcg(b.R + e);
        }
        __syncthreads();
        double r12v[W * W / RT];
#pragma unroll
        for (int k = 0; k < W * W / RT; ++k) {
            const int e = threadIdx.x + k * RT;
            const int r = e % W, cc = e / W;
            double v = 0.0;
            if (r <= cc && cc < jb)
                for (int a2 = r; a2 <= cc; ++a2) v += R12[r + a2 * W] * R1s[a2 + cc * W];
            r12v[k] = v;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < W * W / RT; ++k) R12[threadIdx.x + k * RT] = r12v[k];
        __syncthreads();
        double* Qt = Gs;  // Qt[i + j W]
        if (threadIdx.x < W) {
            const int i = threadIdx.x;
            double x[W];
#pragma unroll
            for (int j = 0; j < W; ++j) x[j] = (i < jb && j < jb) ? __ldcg(Y + i + int64_t(j) * ldy) : 0.0;
            if (i < jb) row_solve(x, Rs, invr, jb);
#pragma unroll
            for (int j = 0; j < W; ++j) Qt[i + j * W] = x[j];
        }
        __syncthreads();
        if (warp == 0) {  // LU of Qt - S without pivoting: lane = row, in registers
            double row[W];
#pragma unroll
            for (int j = 0; j < W; ++j) row[j] = Qt[lane + j * W];
            for (int k = 0; k < jb; ++k) {
                const double pk = __shfl_sync(0xffffffffu, pick(row, k), k);  // running pivot
                const double sk = pk >= 0.0 ? -1.0 : 1.0;  // s_k = -sign(pivot): |u_kk| >= 1
                if (lane == 0) sgn[k] = sk;
                if (lane == k) {
#pragma unroll
                    for (int j = 0; j < W; ++j)
                        if (j == k) row[j] -= sk;
                }
                const double l = (lane > k && lane < jb) ? pick(row, k) / (pk - sk) : 0.0;
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    const double ukj = __shfl_sync(0xffffffffu, row[j], k);
                    if (j > k) row[j] -= l * ukj;
                    else if (j == k && lane > k && lane < jb) row[j] = l;
                }
            }
#pragma unroll
            for (int j = 0; j < W; ++j) Qt[lane + j * W] = row[j];
        }
        __syncthreads();
        // R_house = S (R3 R2 R1) (upper), V_1 = strict lower of the LU,
        // tau_k = -s_k u_kk; U kept for the last pass
        for (int e = threadIdx.x; e < jb * jb; e += RT) {
            const int r = e % jb, cc = e / jb;
            double v;
            if (r <= cc) {
                double s = 0.0;
                for (int a2 = r; a2 <= cc; ++a2) s += Rs[r + a2 * W] * R12[a2 + cc * W];
                v = sgn[r] * s;
            } else {
                v = Qt[r + cc * W];
            }
            P[r + int64_t(cc) * ldp] = v;
        }
        for (int e = threadIdx.x; e < W * W; e += RT) {
            const int r = e % W, cc = e / W;
            b.U[e] = (r < jb && cc < jb) ? (r <= cc ? Qt[e] : 0.0) : (r == cc ? 1.0 : 0.0);
        }
        for (int k = threadIdx.x; k < jb; k += RT) tau[k] = -sgn[k] * Qt[k + k * W];
        if (b.T) {
            // T = -U S V_1^-T (Ballard et al.; equal to dlarft's T of these
            // reflectors to rounding): row r of T solves t V_1^T = -(U S)(r, :),
            // a unit upper triangular system
            double* Vt = R1s;  // V_1^T (unit upper); R1 is no longer needed
            __shared__ double one[W];
            for (int e = threadIdx.x; e < W * W; e += RT) {
                const int r = e % W, cc = e / W;
                Vt[e] = r < cc ? ((r < jb && cc < jb) ? Qt[cc + r * W] : 0.0) : (r == cc ? 1.0 : 0.0);
            }
            if (threadIdx.x < W) one[threadIdx.x] = 1.0;
            __syncthreads();
            if (threadIdx.x < W) {
                const int r = threadIdx.x;
                double x[W];
#pragma unroll
                for (int j = 0; j < W; ++j) x[j] = (r < jb && j >= r && j < jb) ? -Qt[r + j * W] * sgn[j] : 0.0;
                if (r < jb) {
                    row_solve(x, Vt, one, jb);
#pragma unroll
                    for (int j = 0; j < W; ++j)
                        if (j < jb) b.T[r + int64_t(j) * b.ldt] = x[j];
                }
            }
        }
    }
    if (threadIdx.x == 0) *b.ticket = 0u;
}

// rows >= jb: V = Q2 R3^-1 U^-1 written below the panel's top block
// Vout (ld mr, may be null): the explicit unit lower-trapezoidal V of the
// panel (ones on the diagonal, zeros above) that the block update consumes
__global__ void __launch_bounds__(RT) cqr_v_k(int64_t mr, int jb, const double* __restrict__ Q2, int64_t ldq,
                                              double* __restrict__ P, int64_t ldp, double* __restrict__ Vout,
                                              CqrBufs b) {
    extern __shared__ __align__(16) double dyn[];
    __shared__ double R3[W * W], Us[W * W], i3[W], iu[W];
    if (b.status[0]) return;
    for (int e = threadIdx.x; e < W * W; e += RT) {
        R3[e] = b.R[2 * W * W + e];
        Us[e] = b.U[e];
    }
    __syncthreads();
    if (threadIdx.x < W) {
        i3[threadIdx.x] = 1.0 / R3[threadIdx.x * (W + 1)];
        iu[threadIdx.x] = 1.0 / Us[threadIdx.x * (W + 1)];
    }
    if (Vout && blockIdx.x == 0)  // top block: the LU's strict lower part (written by the previous launch)
        for (int e = threadIdx.x; e < jb * jb; e += RT) {
            const int r = e % jb, cc = e / jb;
            Vout[r + int64_t(cc) * mr] = r > cc ? P[r + int64_t(cc) * ldp] : (r == cc ? 1.0 : 0.0);
        }
    const int64_t ntiles = (mr + RT - 1) / RT;
    int64_t tt = blockIdx.x;
    if (tt < ntiles) stage_tile(dyn, Q2, ldq, tt * RT, mr, jb);
    cp_commit();
    for (int k = 0; tt < ntiles; tt += gridDim.x, ++k) {
        double* cur = dyn + (k & 1) * (W * XS);
        double* nxt = dyn + ((k + 1) & 1) * (W * XS);
        if (tt + gridDim.x < ntiles) stage_tile(nxt, Q2, ldq, (tt + gridDim.x) * RT, mr, jb);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const int64_t i = tt * RT + threadIdx.x;
        if (i >= jb && i < mr) {
            double x[W];
#pragma unroll
            for (int j = 0; j < W; ++j) x[j] = cur[j * XS + threadIdx.x];
            row_solve(x, R3, i3, jb);
            row_solve(x, Us, iu, jb);
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (j < jb) {
                    P[i + int64_t(j) * ldp] = x[j];
                    if (Vout) Vout[i + int64_t(j) * mr] = x[j];
                }
        }
        __syncthreads();
    }
    cp_wait<0>();
}

}  // namespace

// Factor the mr x jb (jb <= 32) panel P (ld) in place like the Householder
// panels of qr.cu: R above the diagonal, V below (unit diagonal implied),
// tau.  `work` holds 2 mr x 32 doubles (Q1, Q2), `scratch` cqr_scratch_doubles()
// (per-panel state).  A panel whose Q does not come out orthonormal is left
// untouched and raises *sticky (device) to 2: the caller then redoes the
// whole factorisation by Householder panels (geqrf, qr.cu).
int64_t cqr_scratch_doubles(const Ctx& c) {
    return int64_t(c.num_sms) * CTAS_PER_SM * GSZ + int64_t(MAXGRP) * GSZ + 4 * W * W + 2 + MAXGRP;
}

// T (ld ldt, may be null) receives the panel's compact-WY triangle and, when
// form_v is set, work[0 .. mr jb) the explicit V (ld mr) -- Q1's space, free
// by the last pass.
void panel_cqr(Ctx& c, int64_t mr, int jb, double* P, int64_t ld, double* tau, double* work,
               double* scratch, int* sticky, double* T, int64_t ldt, bool form_v) {
    if (jb < 1 || jb > W || mr < int64_t(W)) throw std::invalid_argument("panel_cqr: shape");
    // CTAS_PER_SM CTAs per SM stream the rows: one CTA keeps a single 32 KB
    // tile in flight and one warp per scheduler in the row substitution,
    // which left both the memory system and the FP64 pipe waiting (ncu: a
    // 67 MB panel read at 0.9 TB/s)
    const int grid = int(std::min<int64_t>((mr + RT - 1) / RT, int64_t(c.num_sms) * CTAS_PER_SM));
    if ((grid + GRP - 1) / GRP > MAXGRP) throw std::runtime_error("panel_cqr: grid too large");
    double* part = scratch;
    double* gpart = scratch + int64_t(c.num_sms) * CTAS_PER_SM * GSZ;
    double* small = gpart + int64_t(MAXGRP) * GSZ;
    unsigned* ints = reinterpret_cast<unsigned*>(small + 4 * W * W);  // ticket, status, group tickets
    HYDOT_CUDA(cudaMemsetAsync(ints, 0, (2 + MAXGRP) * sizeof(unsigned), c.stream));
    CqrBufs b{part, gpart, ints, ints + 2, small, small + 3 * W * W, reinterpret_cast<int*>(ints + 1), sticky, T, ldt};
    double* Q1 = work;
    double* Q2 = work + mr * W;
    const double shift = 11.0 * (double(mr) * jb + double(jb) * (jb + 1)) * 1.1102230246251565e-16;
    const size_t smem = size_t(2) * W * XS * sizeof(double);
    static AttrGate attr;
    attr_once(attr, c.device, [&] {
        HYDOT_CUDA(cudaFuncSetAttribute(cqr_pass_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        HYDOT_CUDA(cudaFuncSetAttribute(cqr_pass_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        HYDOT_CUDA(cudaFuncSetAttribute(cqr_pass_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        HYDOT_CUDA(cudaFuncSetAttribute(cqr_v_k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    });
    cqr_pass_k<0><<<grid, RT, smem, c.stream>>>(mr, jb, P, ld, nullptr, 0, P, ld, tau, b, shift);
    c.check_launch();
    cqr_pass_k<1><<<grid, RT, smem, c.stream>>>(mr, jb, P, ld, Q1, mr, P, ld, tau, b, 0.0);
    c.check_launch();
    cqr_pass_k<2><<<grid, RT, smem, c.stream>>>(mr, jb, Q1, mr, Q2, mr, P, ld, tau, b, 0.0);
    c.check_launch();
    cqr_v_k<<<grid, RT, smem, c.stream>>>(mr, jb, Q2, mr, P, ld, form_v ? Q1 : nullptr, b);
    c.check_launch();
}

}  // namespace hydot
