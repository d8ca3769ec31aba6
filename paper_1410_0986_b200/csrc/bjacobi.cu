// bjacobi.cu -- block one-sided Jacobi on the FP64 tensor cores (DMMA) for
// the large SVD cores of the path: the R factors behind Eigen's BDCSVD calls
// (lowrank.cpp:43-49, 79, 88, 568) once they reach hundreds to thousands of
// columns (config 2's root merge core is 5686 x 5686).
//
// The point drivers of svd.cu orthogonalise one column pair per rotation, so
// every sub-round costs an m-long CTA reduction and a barrier, and a sweep
// streams the matrix once per block round at ~1 flop/byte.  Here the columns
// are grouped in blocks of BW = 16; a tournament (circle method) over the
// blocks pairs them up, and one visit of a block pair X_p = [X_i X_j]
// (m x 32) is
//   1. G_p = X_p^T X_p             (DMMA, rows split in chunks, partial
//                                    Grams summed in a fixed chunk order)
//   2. G_p = Q_p D Q_p^T           (cyclic two-sided Jacobi on the 32 x 32
//                                    Gram in shared memory, by the CTA that
//                                    completes the pair's last chunk)
//   3. X_p <- X_p Q_p              (DMMA, in place, row chunks)
// so a sweep is 8 m n^2 tensor-core flops plus ~3 passes over the matrix per
// block round, with two grid barriers per round (one cooperative launch per
// sweep).  Accuracy: the Gram entries carry errors ~ m eps |x_k| |x_l|, i.e.
// relative to each column pair, and two-sided Jacobi on a positive
// semidefinite matrix with the relative stopping test |g_kl| <= tol
// sqrt(g_kk g_ll) is relatively accurate (Demmel-Veselic); the update is an
// orthogonal transformation of the columns, as in the point method.  A pair
// whose Gram passes the test is left untouched; a sweep in which no pair
// rotates ends the iteration, and the columns are then those of a converged
// one-sided Jacobi (sigma_j = |x_j|, U = x_j / sigma_j).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "internal.h"

namespace hydot {
namespace {

// Block width BW = 16 (32-column pairs, warp eigen-solve) or 32 (64-column
// pairs, CTA eigen-solve: half the block rounds per sweep, so half the passes
// over a matrix too large for L2).
constexpr int SUB = 64;       // rows per shared-memory sub-tile
constexpr int NTH = 128;      // threads per CTA (4 warps)
constexpr int XS = SUB + 4;   // X sub-tile stride ([col][row], conflict-free fragments)
template <int BW>
struct Geo {
    static constexpr int PW = 2 * BW;  // columns per block pair
    static constexpr int QS = PW + 4;  // Q stride ([out col][in col])
    static constexpr int GS = PW + 1;  // eigen-solver stride
    static constexpr int QD = PW / 2;  // a warp's Gram quadrant (QD x QD)
    static constexpr int MI = QD / 16, NI = QD / 8;
    static constexpr int NU = PW / 8;  // update: n8 tiles per warp row block
    static constexpr int SMEM = 2 * PW * XS + PW * QS > 2 * PW * GS ? 2 * PW * XS + PW * QS : 2 * PW * GS;
};
// Inner sweeps per pair visit: one cyclic sweep over the pair Gram (to a
// threshold 1e-4 x its initial largest scaled off-diagonal, floor tol) --
// the eigen-solve is the latency chain of a round, and the outer sweeps
// converge quadratically anyway.  Measured (graded cores, total ms for
// 2000 / 2800 / 5686): 4 inner sweeps 179 / 319 / 1149, 2: 139 / 252 / 987,
// 1: 116 / 217 / 992 (one more outer sweep).  An uncapped solve ran 30
// sweeps on strongly graded pairs, where the inner rotations' own rounding
// keeps tiny off-diagonals above tol.
constexpr int kInner = 1;
constexpr double kInnerRel = 1e-4;
constexpr int kMaxBSweeps = 40;

struct BJArgs {
    int64_t m;
    int n, nbp, per, rounds;
    const int2* pairs;  // rounds x per block pairs (circle method)
    double* U;
    int64_t ldu;
    double tol, flag_tol;
    int inner_cap;     // inner sweeps per pair visit (kInner)
    double inner_rel;  // inner threshold relative to the pair's largest off-diagonal (kInnerRel)
    int nch, rch;
    // ring buffers over rounds (slot r % RING): a pair slot's Gram partials,
    // rotation and flag of round r live until round r + RING reuses them
    double* gws;  // RING x per x nch x PW*PW partial Grams
    double* qws;  // RING x per x PW*PW rotations
    int* flag;    // RING x per: 1 = rotate
    int* cnt;     // RING x per: chunk arrival counters (self-resetting)
    int* ver;     // nbp x nch: rounds of updates applied to (block, chunk)
    int* epoch;   // RING x per: r + 1 once round r's eigen-solve of the slot is published
    int* udone;   // RING x per: update units finished (rounds of that ring slot)
    int* work;    // item dispenser
    int* stats;   // [0] pairs rotated this sweep, [1] inner rotations, [2] non-finite pair Grams, [3] inner sweeps
};
constexpr int RING = 4;

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_geq(const int* p, int v) {
    if (ld_acquire(p) >= v) return;
    unsigned ns = 32;
    while (ld_acquire(p) < v) {
        __nanosleep(ns);
        if (ns < 512) ns *= 2;
    }
}
// publish: every thread's prior stores, then the counter (release)
__device__ __forceinline__ void publish_add(int* p, int v) {
    __threadfence();
    atomicAdd(p, v);
}

__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

// rotation annihilating g of the 2x2 Gram [[a, g], [g, b]] (svd.cu's form:
// cos 2theta from a reciprocal square root, no division)
__device__ __forceinline__ void rot2(double a, double b, double g, double& cs, double& sn) {
    const double d = 0.5 * (b - a);
    const double r = rsqrt(fma(d, d, g * g));
    const double h = fma(0.5 * fabs(d), r, 0.5);
    const double ih = rsqrt(h);
    cs = h * ih;
    sn = copysign(1.0, d) * (0.5 * g * r) * ih;
}

__device__ __forceinline__ int circ(int pos, int r, int np) {
    if (pos == 0) return 0;
    int v = pos - 1 + r;  // < 2 (np - 1)
    if (v >= np - 1) v -= np - 1;
    return v + 1;
}

// global column of pair-local column j (-1: padding / dummy block)
template <int BW>
__device__ __forceinline__ int pair_col(int2 bp, int j, int n) {
    const int blk = j < BW ? bp.x : bp.y;
    const int c = blk * BW + (j & (BW - 1));
    return c < n ? c : -1;
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

// asynchronous load_sub: the copies land in xs while the previous sub-tile
// is processed (double buffering inside a unit)
template <int PW>
__device__ __forceinline__ void stage_sub(double* xs, const double* __restrict__ U, int64_t ldu,
                                          const int* col, int64_t r, int64_t rend) {
#pragma unroll
    for (int k = 0; k < SUB * PW / NTH; ++k) {
        const int e = threadIdx.x + k * NTH;
        const int i = e & (SUB - 1), j = e / SUB;
        const int64_t gi = r + i;
        const int cj = col[j];
        const bool ok = cj >= 0 && gi < rend;
        cp_async8(xs + j * XS + i, ok ? U + gi + int64_t(cj) * ldu : U, ok);
    }
}

// ---- phase 1: partial Gram of one (pair, row chunk) unit; the CTA that
// completes a pair's last chunk diagonalises its Gram
template <int BW>
__device__ void eig_pair(const BJArgs& a, int q, int rnd, double* smem);

template <int BW>
__device__ void gram_unit(const BJArgs& a, int2 bp, int q, int rnd, int ch, double* smem, int* col) {
    using Gm = Geo<BW>;
    constexpr int PW = Gm::PW, QD = Gm::QD, MI = Gm::MI, NI = Gm::NI;
    double* xs = smem;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wi = (warp & 1) * QD, wj = (warp >> 1) * QD;
    double acc[MI][NI][4];
#pragma unroll
    for (int x = 0; x < MI; ++x)
#pragma unroll
        for (int y = 0; y < NI; ++y)
#pragma unroll
            for (int z = 0; z < 4; ++z) acc[x][y][z] = 0.0;
    const int64_t r0 = int64_t(ch) * a.rch, r1 = min(a.m, r0 + a.rch);
    const int nsub = int((r1 - r0 + SUB - 1) / SUB);
    __syncthreads();
    stage_sub<PW>(xs, a.U, a.ldu, col, r0, r1);
    cp_commit();
    for (int sb = 0; sb < nsub; ++sb) {
        const double* cur = xs + (sb & 1) * (PW * XS);
        if (sb + 1 < nsub)
            stage_sub<PW>(xs + ((sb + 1) & 1) * (PW * XS), a.U, a.ldu, col, r0 + int64_t(sb + 1) * SUB, r1);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < SUB; kk += 4) {
            // A = X^T (i = column, k = row), B = X (k = row, j = column)
            double a0[MI], a1[MI];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
                a0[mi] = cur[(wi + mi * 16 + g) * XS + kk + t];
                a1[mi] = cur[(wi + mi * 16 + g + 8) * XS + kk + t];
            }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
                const double b0 = cur[(wj + ni * 8 + g) * XS + kk + t];
#pragma unroll
                for (int mi = 0; mi < MI; ++mi) dmma(acc[mi][ni], a0[mi], a1[mi], b0);
            }
        }
        __syncthreads();
    }
    cp_wait<0>();
    const int slot = rnd % RING;
    double* out = a.gws + ((int64_t(slot) * a.per + q) * a.nch + ch) * (PW * PW);
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int i = wi + mi * 16 + g + ((v & 2) ? 8 : 0);
                const int j = wj + ni * 8 + 2 * t + (v & 1);
                __stcg(out + i + j * PW, acc[mi][ni][v]);
            }
    __threadfence();
    __syncthreads();
    __shared__ int last;
    int* cnt = a.cnt + slot * a.per + q;
    if (threadIdx.x == 0) last = atomicAdd(cnt, 1) == a.nch - 1;
    __syncthreads();
    if (last) {
        __threadfence();
        // the rotation / flag ring slot is free once round rnd - RING's
        // update units of this pair slot are done
        if (threadIdx.x == 0) {
            *cnt = 0;
            wait_geq(a.udone + slot * a.per + q, (rnd / RING) * a.nch);
        }
        __syncthreads();
        eig_pair<BW>(a, q, rnd, smem);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicExch(a.epoch + slot * a.per + q, rnd + 1);  // publish this round's rotation
        }
    }
}

// Cyclic two-sided Jacobi on the pair Gram: G <- J^T G J, Q <- Q J, 16
// disjoint rotations per round (circle method over 32 indices), run by one
// warp in shared memory (warp barriers only: a CTA barrier per step made the
// eigen-solve the latency bottleneck of a round).  The eigenvector columns
// leave sorted by decreasing diagonal.
template <int BW>
__device__ void eig_pair(const BJArgs& a, int q, int rnd, double* smem) {
    constexpr int PW = Geo<BW>::PW, GS = Geo<BW>::GS;
    const int slot = rnd % RING;
    double* G = smem;              // PW x GS
    double* Q = smem + PW * GS;    // PW x GS
    __shared__ double rc[PW / 2], rs[PW / 2];
    __shared__ int rp[PW / 2], ro[PW / 2];
    __shared__ int any, bad, rot_total, sweeps_total;
    __shared__ unsigned long long off0_bits;
    __shared__ double dsum[PW];
    __shared__ int perm[PW];
    const double* part = a.gws + (int64_t(slot) * a.per + q) * a.nch * (PW * PW);
    if (threadIdx.x == 0) {
        any = 0;
        bad = 0;
        rot_total = 0;
        sweeps_total = 0;
        off0_bits = 0ull;
    }
    for (int e = threadIdx.x; e < PW * PW; e += NTH) {
        double s = 0.0;
        for (int c = 0; c < a.nch; ++c) s += __ldcg(part + int64_t(c) * (PW * PW) + e);
        const int i = e % PW, j = e / PW;
        G[i * GS + j] = s;
        Q[i * GS + j] = i == j ? 1.0 : 0.0;
    }
    __syncthreads();
    // the pair decision: any scaled off-diagonal above flag_tol
    for (int e = threadIdx.x; e < PW * PW; e += NTH) {
        const int i = e % PW, j = e / PW;
        const double gij = G[i * GS + j];
        if (!isfinite(gij)) bad = 1;
        if (i < j && gij != 0.0) {
            const double sc = fabs(gij) / sqrt(G[i * GS + i] * G[j * GS + j]);
            if (sc > a.flag_tol) {
                any = 1;
                // non-negative doubles order like their bit patterns
                atomicMax(&off0_bits, (unsigned long long)__double_as_longlong(sc));
            }
        }
    }
    __syncthreads();
    if (bad && threadIdx.x == 0) atomicAdd(a.stats + 2, 1);
    if (!any) {
        if (threadIdx.x == 0) a.flag[slot * a.per + q] = 0;
        return;
    }
    const double tin = fmax(a.tol, a.inner_rel * __longlong_as_double((long long)off0_bits));
    if constexpr (BW == 32) {
        // CTA solve of the 64 x 64 Gram: 32 rotations per round; the row and
        // column phases are spread over the 4 warps (CTA barriers)
        __shared__ int rmask[2];
        for (int sw = 0; sw < a.inner_cap; ++sw) {
            int rotated = 0;
            for (int r = 0; r < PW - 1; ++r) {
                if (threadIdx.x < PW / 2) {
                    const int k = threadIdx.x;
                    int p = circ(k, r, PW), o = circ(PW - 1 - k, r, PW);
                    if (p > o) {
                        const int tmp = p;
                        p = o;
                        o = tmp;
                    }
                    const double app = G[p * GS + p], aoo = G[o * GS + o], apo = G[p * GS + o];
                    double cs = 1.0, sn = 0.0;
                    bool on = false;
                    if (apo != 0.0 && fabs(apo) > tin * sqrt(app * aoo)) {
                        rot2(app, aoo, apo, cs, sn);
                        on = true;
                    }
                    rc[k] = cs;
                    rs[k] = on ? sn : 0.0;
                    rp[k] = p;
                    ro[k] = o;
                    const unsigned mask = __ballot_sync(0xffffffffu, on);
                    if (k == 0) rmask[r & 1] = int(__popc(mask));
                }
                __syncthreads();
                const int nrot = rmask[r & 1];
                if (nrot == 0) continue;  // uniform: no one wrote G this round
                rotated += nrot;
                // rows: G <- J^T G; item (slot k, column x)
                for (int e = threadIdx.x; e < (PW / 2) * PW; e += NTH) {
                    const int k = e / PW, x = e % PW;
                    const double sn = rs[k];
                    if (sn != 0.0) {
                        const double c = rc[k];
                        const int p = rp[k], o = ro[k];
                        const double gp = G[p * GS + x], go = G[o * GS + x];
                        G[p * GS + x] = c * gp - sn * go;
                        G[o * GS + x] = sn * gp + c * go;
                    }
                }
                __syncthreads();
                // columns: G <- G J, Q <- Q J; item (slot k, row x)
                for (int e = threadIdx.x; e < (PW / 2) * PW; e += NTH) {
                    const int k = e / PW, x = e % PW;
                    const double sn = rs[k];
                    if (sn != 0.0) {
                        const double c = rc[k];
                        const int p = rp[k], o = ro[k];
                        const double gp = G[x * GS + p], go = G[x * GS + o];
                        G[x * GS + p] = c * gp - sn * go;
                        G[x * GS + o] = sn * gp + c * go;
                        const double qp = Q[x * GS + p], qo = Q[x * GS + o];
                        Q[x * GS + p] = c * qp - sn * qo;
                        Q[x * GS + o] = sn * qp + c * qo;
                    }
                }
                __syncthreads();
                if (threadIdx.x < PW / 2 && rs[threadIdx.x] != 0.0) {  // annihilated exactly
                    G[rp[threadIdx.x] * GS + ro[threadIdx.x]] = 0.0;
                    G[ro[threadIdx.x] * GS + rp[threadIdx.x]] = 0.0;
                }
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                rot_total += rotated;
                ++sweeps_total;
            }
            if (rotated == 0) break;
        }
    } else if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        for (int sw = 0; sw < a.inner_cap; ++sw) {
            int rotated = 0;
            for (int r = 0; r < PW - 1; ++r) {
                // circle-method pair of slot k = lane (k < 16) in round r
                bool on = false;
                if (lane < PW / 2) {
                    int p = circ(lane, r, PW), o = circ(PW - 1 - lane, r, PW);
                    if (p > o) {
                        const int tmp = p;
                        p = o;
                        o = tmp;
                    }
                    const double app = G[p * GS + p], aoo = G[o * GS + o], apo = G[p * GS + o];
                    double cs = 1.0, sn = 0.0;
                    if (apo != 0.0 && fabs(apo) > tin * sqrt(app * aoo)) {
                        rot2(app, aoo, apo, cs, sn);
                        on = true;
                    }
                    rc[lane] = cs;
                    rs[lane] = on ? sn : 0.0;
                    rp[lane] = p;
                    ro[lane] = o;
                }
                const unsigned mask = __ballot_sync(0xffffffffu, on);
                if (mask == 0u) continue;
                rotated += __popc(mask);
                __syncwarp();
                // every index is in exactly one slot: a lane updates a whole
                // column (rows phase) or row (columns phase), 8 slots at a
                // time with all their loads issued before any store
                constexpr int H = PW / 4;
#pragma unroll
                for (int h0 = 0; h0 < PW / 2; h0 += H) {  // rows: G <- J^T G (lane = column)
                    double vp[H], vo[H];
#pragma unroll
                    for (int k = 0; k < H; ++k) {
                        vp[k] = G[rp[h0 + k] * GS + lane];
                        vo[k] = G[ro[h0 + k] * GS + lane];
                    }
#pragma unroll
                    for (int k = 0; k < H; ++k) {
                        const double c = rc[h0 + k], sn = rs[h0 + k];
                        G[rp[h0 + k] * GS + lane] = c * vp[k] - sn * vo[k];
                        G[ro[h0 + k] * GS + lane] = sn * vp[k] + c * vo[k];
                    }
                }
                __syncwarp();
#pragma unroll
                for (int h0 = 0; h0 < PW / 2; h0 += H) {  // columns: G <- G J, Q <- Q J (lane = row)
                    double vp[H], vo[H], wp[H], wo[H];
#pragma unroll
                    for (int k = 0; k < H; ++k) {
                        vp[k] = G[lane * GS + rp[h0 + k]];
                        vo[k] = G[lane * GS + ro[h0 + k]];
                        wp[k] = Q[lane * GS + rp[h0 + k]];
                        wo[k] = Q[lane * GS + ro[h0 + k]];
                    }
#pragma unroll
                    for (int k = 0; k < H; ++k) {
                        const double c = rc[h0 + k], sn = rs[h0 + k];
                        G[lane * GS + rp[h0 + k]] = c * vp[k] - sn * vo[k];
                        G[lane * GS + ro[h0 + k]] = sn * vp[k] + c * vo[k];
                        Q[lane * GS + rp[h0 + k]] = c * wp[k] - sn * wo[k];
                        Q[lane * GS + ro[h0 + k]] = sn * wp[k] + c * wo[k];
                    }
                }
                __syncwarp();
                if (on) {  // annihilated exactly
                    G[rp[lane] * GS + ro[lane]] = 0.0;
                    G[ro[lane] * GS + rp[lane]] = 0.0;
                }
                __syncwarp();
            }
            if (lane == 0) {
                rot_total += rotated;
                ++sweeps_total;
            }
            if (rotated == 0) break;
        }
    }
    __syncthreads();
    // sort by decreasing diagonal (stable rank order)
    if (threadIdx.x < PW) dsum[threadIdx.x] = G[threadIdx.x * GS + threadIdx.x];
    __syncthreads();
    if (threadIdx.x < PW) {
        const int j = threadIdx.x;
        const double dj = dsum[j];
        int rank = 0;
        for (int k = 0; k < PW; ++k) {
            const double dk = dsum[k];
            rank += (dk > dj) || (dk == dj && k < j);
        }
        perm[rank] = j;
    }
    __syncthreads();
    double* qo = a.qws + (int64_t(slot) * a.per + q) * (PW * PW);
    for (int e = threadIdx.x; e < PW * PW; e += NTH) {
        const int i = e % PW, j = e / PW;
        __stcg(qo + i + j * PW, Q[i * GS + perm[j]]);
    }
    if (threadIdx.x == 0) {
        a.flag[slot * a.per + q] = 1;
        atomicAdd(a.stats, 1);
        atomicAdd(a.stats + 1, rot_total);
        atomicAdd(a.stats + 3, sweeps_total);
    }
    __threadfence();
}

// ---- phase 3: X_p(rows of the chunk) <- X_p Q_p
template <int BW>
__device__ void update_unit(const BJArgs& a, int q, int rnd, int ch, double* smem, const int* col) {
    using Gm = Geo<BW>;
    constexpr int PW = Gm::PW, QS = Gm::QS, NU = Gm::NU;
    double* xs = smem;                // 2 x PW x XS (double-buffered sub-tiles)
    double* qs = smem + 2 * PW * XS;  // PW x QS: qs[j * QS + k] = Q(k, j)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const double* qg = a.qws + (int64_t(rnd % RING) * a.per + q) * (PW * PW);
    __syncthreads();
    for (int e = threadIdx.x; e < PW * PW; e += NTH) {
        const int k = e % PW, j = e / PW;
        qs[j * QS + k] = __ldcg(qg + e);
    }
    const int64_t r0 = int64_t(ch) * a.rch, r1 = min(a.m, r0 + a.rch);
    const int wr = warp * 16;  // the warp's 16 rows of the 64-row sub-tile
    const int nsub = int((r1 - r0 + SUB - 1) / SUB);
    __syncthreads();
    stage_sub<PW>(xs, a.U, a.ldu, col, r0, r1);
    cp_commit();
    for (int sb = 0; sb < nsub; ++sb) {
        const int64_t r = r0 + int64_t(sb) * SUB;
        double* cur = xs + (sb & 1) * (PW * XS);
        if (sb + 1 < nsub) stage_sub<PW>(xs + ((sb + 1) & 1) * (PW * XS), a.U, a.ldu, col, r + SUB, r1);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        double acc[NU][4];
#pragma unroll
        for (int x = 0; x < NU; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
#pragma unroll
        for (int kk = 0; kk < PW; kk += 4) {
            // A = X (i = row, k = column): xs[k * XS + i]
            const double a0 = cur[(kk + t) * XS + wr + g];
            const double a1 = cur[(kk + t) * XS + wr + g + 8];
#pragma unroll
            for (int ni = 0; ni < NU; ++ni) dmma(acc[ni], a0, a1, qs[(ni * 8 + g) * QS + kk + t]);
        }
        __syncthreads();
#pragma unroll
        for (int ni = 0; ni < NU; ++ni)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int i = wr + g + ((v & 2) ? 8 : 0);
                const int j = ni * 8 + 2 * t + (v & 1);
                cur[j * XS + i] = acc[ni][v];
            }
        __syncthreads();
#pragma unroll
        for (int e = threadIdx.x; e < SUB * PW; e += NTH) {
            const int i = e & (SUB - 1), j = e / SUB;
            const int64_t gi = r + i;
            const int cj = col[j];
            if (cj >= 0 && gi < r1) __stcg(a.U + gi + int64_t(cj) * a.ldu, cur[j * XS + i]);
        }
        __syncthreads();  // cur is refilled by the next iteration's staging
    }
    cp_wait<0>();
}



// One sweep as a dataflow over work items taken in a fixed global order
// (round-major; per round the Gram units, then the update units), so
// every item only waits on items handed out before it (no deadlock, no grid
// barrier): a Gram unit waits until its two blocks' chunk carries the
// previous round's update, an update unit until its pair's eigen-solve is
// published.  A slow eigen-solve then delays only the pairs that depend on
// it instead of the whole grid.
template <int BW>
__global__ void __launch_bounds__(NTH, BW == 16 ? 4 : 2) bjacobi_sweep_k(BJArgs a) {
    constexpr int PW = Geo<BW>::PW;
    extern __shared__ __align__(16) double smem[];  // Geo<BW>::SMEM doubles
    __shared__ int col[PW];
    __shared__ int item_s;
    const int units = a.per * a.nch;
    const int64_t items = int64_t(a.rounds) * 2 * units;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) item_s = atomicAdd(a.work, 1);
        __syncthreads();
        const int64_t it = item_s;
        if (it >= items) break;
        const int rnd = int(it / (2 * units));
        const int rem = int(it % (2 * units));
        const bool upd = rem >= units;
        const int u = upd ? rem - units : rem;
        const int q = u / a.nch, ch = u % a.nch;
        const int2 bp = a.pairs[int64_t(rnd) * a.per + q];
        if (threadIdx.x < PW) col[threadIdx.x] = pair_col<BW>(bp, threadIdx.x, a.n);
        if (!upd) {
            if (threadIdx.x == 0) {
                wait_geq(a.ver + bp.x * a.nch + ch, rnd);
                wait_geq(a.ver + bp.y * a.nch + ch, rnd);
                // partial / counter ring slot free: round rnd - RING's eigen-solve done
                wait_geq(a.epoch + (rnd % RING) * a.per + q, rnd - RING + 1);
            }
            __syncthreads();
            gram_unit<BW>(a, bp, q, rnd, ch, smem, col);
        } else {
            if (threadIdx.x == 0) wait_geq(a.epoch + (rnd % RING) * a.per + q, rnd + 1);
            __syncthreads();
            if (__ldcg(a.flag + (rnd % RING) * a.per + q)) update_unit<BW>(a, q, rnd, ch, smem, col);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(a.ver + bp.x * a.nch + ch, 1);
                atomicAdd(a.ver + bp.y * a.nch + ch, 1);
                atomicAdd(a.udone + (rnd % RING) * a.per + q, 1);
            }
        }
    }
}

std::vector<int2> block_tournament(int nbp) {
    std::vector<int> p(static_cast<size_t>(nbp));
    std::iota(p.begin(), p.end(), 0);
    std::vector<int2> out;
    out.reserve(size_t(nbp / 2) * size_t(nbp - 1));
    for (int r = 0; r < nbp - 1; ++r) {
        for (int i = 0; i < nbp / 2; ++i) {
            const int x = p[size_t(i)], y = p[size_t(nbp - 1 - i)];
            out.push_back(make_int2(std::min(x, y), std::max(x, y)));
        }
        const int last = p[size_t(nbp - 1)];
        for (int i = nbp - 1; i > 1; --i) p[size_t(i)] = p[size_t(i - 1)];
        p[1] = last;
    }
    return out;
}

bool bj_stats() {
    static const bool on = [] {
        const char* e = std::getenv("HYDOT_JACOBI_STATS");
        return e && e[0] == '1';
    }();
    return on;
}

}  // namespace

// Minimum core order for the block driver (below it the register point
// drivers of svd.cu are latency-optimal).  HYDOT_BJACOBI_MIN overrides.
int64_t bjacobi_min_n() {
    static const int64_t v = [] {
        const char* e = std::getenv("HYDOT_BJACOBI_MIN");
        return e ? int64_t(std::atoll(e)) : int64_t(1800);
    }();
    return v;
}

// Orthogonalise the columns of U (m x n, ld m, m >= n) in place to the
// one-sided Jacobi criterion (pairs within flag_tol = 2 tol).  Returns the
// number of sweeps.
namespace {
template <int BW>
int bjacobi_run(Ctx& c, int64_t m, int64_t n, double* U, double tol) {
    constexpr int PW = Geo<BW>::PW;
    const size_t smem = size_t(Geo<BW>::SMEM) * sizeof(double);
    static AttrGate attr;
    attr_once(attr, c.device, [&] {
        HYDOT_CUDA(cudaFuncSetAttribute(bjacobi_sweep_k<BW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    });
    const int nb = int((n + BW - 1) / BW);
    const int nbp = nb + (nb & 1);
    const int per = nbp / 2, rounds = nbp - 1;
    std::vector<int2> pairs = block_tournament(nbp);
    DBuf dpairs(c, pairs.size() * sizeof(int2));
    HYDOT_CUDA(cudaMemcpyAsync(dpairs.as<void>(), pairs.data(), pairs.size() * sizeof(int2),
                               cudaMemcpyHostToDevice, c.stream));
    int per_sm = 0;
    HYDOT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bjacobi_sweep_k<BW>, NTH, smem));
    const int max_grid = std::max(1, per_sm) * c.num_sms;
    // row chunks: enough (pair, chunk) units to fill the grid twice
    const int64_t subs = (m + SUB - 1) / SUB;
    int64_t nch = std::clamp<int64_t>((2 * int64_t(max_grid) + per - 1) / per, 1, subs);
    const int64_t rch = ((m + nch - 1) / nch + SUB - 1) / SUB * SUB;
    nch = (m + rch - 1) / rch;
    const int units = int(per * nch);
    const int grid = std::min(units, max_grid);
    DBuf gws = dalloc(c, size_t(RING) * size_t(per) * size_t(nch) * PW * PW);
    DBuf qws = dalloc(c, size_t(RING) * size_t(per) * PW * PW);
    // flag, cnt (RING x per each), ver (nbp x nch), epoch, udone (RING x per each), work, stats (4)
    const size_t nints = size_t(2 * RING * per) + size_t(nbp) * size_t(nch) + size_t(2 * RING * per) + 1 + 4;
    DBuf ints(c, sizeof(int) * nints);
    HYDOT_CUDA(cudaMemsetAsync(ints.as<void>(), 0, sizeof(int) * nints, c.stream));
    BJArgs a;
    a.m = m;
    a.n = int(n);
    a.nbp = nbp;
    a.per = per;
    a.rounds = rounds;
    a.pairs = dpairs.as<int2>();
    a.U = U;
    a.ldu = m;
    a.tol = tol;
    a.flag_tol = 2.0 * tol;  // tol is itself the rounding level of a column dot product
    // (experiment knobs: HYDOT_BJ_INNER=cap,rel)
    a.inner_cap = kInner;
    a.inner_rel = kInnerRel;
    if (const char* e = std::getenv("HYDOT_BJ_INNER")) {
        int cap = kInner;
        double rel = kInnerRel;
        if (sscanf(e, "%d,%lf", &cap, &rel) >= 1) {
            a.inner_cap = std::max(1, cap);
            a.inner_rel = rel;
        }
    }
    a.nch = int(nch);
    a.rch = int(rch);
    a.gws = gws.d();
    a.qws = qws.d();
    a.flag = ints.as<int>();
    a.cnt = a.flag + RING * per;
    a.ver = a.cnt + RING * per;
    a.epoch = a.ver + size_t(nbp) * size_t(nch);
    a.udone = a.epoch + RING * per;
    a.work = a.udone + RING * per;
    a.stats = a.work + 1;
    // everything but the ring contents restarts every sweep
    const size_t reset = size_t(nbp) * size_t(nch) + size_t(2 * RING * per) + 1 + 4;
    int sweeps = 0;
    for (; sweeps < kMaxBSweeps; ++sweeps) {
        HYDOT_CUDA(cudaMemsetAsync(a.ver, 0, reset * sizeof(int), c.stream));
        bjacobi_sweep_k<BW><<<grid, NTH, smem, c.stream>>>(a);
        c.check_launch();
        int st[4] = {0, 0, 0, 0};
        HYDOT_CUDA(cudaMemcpyAsync(st, a.stats, sizeof st, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (bj_stats())
            fprintf(stderr,
                    "[bjacobi] bw=%d m=%lld n=%lld sweep=%d pairs_rotated=%d inner_rotations=%d inner_sweeps=%d (of "
                    "%d pairs) nonfinite=%d\n",
                    BW, (long long)m, (long long)n, sweeps, st[0], st[1], st[3], per * rounds, st[2]);
        if (st[2] > 0) throw std::runtime_error("block Jacobi: non-finite column Gram (input not finite?)");
        if (st[0] == 0) break;
    }
    return sweeps + 1;
}
}  // namespace

// Block width by core order: 32-column blocks once the core no longer fits
// L2 (the sweep is then bound by the passes over the matrix, and BW = 32
// halves them); 16 below.  HYDOT_BJACOBI_BW overrides (16 / 32).
int bjacobi_converge(Ctx& c, int64_t m, int64_t n, double* U, double tol) {
    static const int force = [] {
        const char* e = std::getenv("HYDOT_BJACOBI_BW");
        return e ? std::atoi(e) : 0;
    }();
    const bool wide = force ? force == 32 : n >= 4000;
    return wide ? bjacobi_run<32>(c, m, n, U, tol) : bjacobi_run<16>(c, m, n, U, tol);
}

}  // namespace hydot
