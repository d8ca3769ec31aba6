// qr.cu -- blocked Householder QR on the GPU (LAPACK dgeqrf / dlarft /
// dlarfb semantics), replacing Eigen::HouseholderQR in fast_thin_svd
// (lowrank.cpp:73-87) and recompress (lowrank.cpp:564-566, 579-580).
//
// The scheduled leaf tolerance reaches 8e-11, below sqrt(eps),
// so Gram/Cholesky QR is not admissible: this is true Householder.
// Two-level blocking:
//   panel  (32 columns)  one cooperative persistent kernel: every CTA owns a
//          contiguous row slab (kept in shared memory when it fits) and ONE
//          grid-wide barrier per column.  Look-ahead: while applying the
//          reflector of column c, each CTA already accumulates the partial
//          norm of column c+1 and its partial dot products x^T P_q with the
//          remaining columns; with the published row c+1 the reflector data
//          w_q = P_cq + scal (x^T P_q - alpha P_cq) of the next column need no
//          second reduction.  Partial sums are reduced redundantly by every
//          CTA in fixed order: deterministic.
//   block  (128 columns) the 32-wide sub-panels update the rest of their
//          128-block with DMMA GEMMs; the 128-wide block reflector
//          I - V T V^T then updates the trailing matrix with three DMMA GEMMs
//          (4x fewer passes over the trailing matrix than 32-wide blocking).
#include <cooperative_groups.h>

#include <cstdlib>
#include <exception>

#include "internal.h"

namespace cg = cooperative_groups;

namespace hydot {
namespace {

constexpr int PB = 32;        // panel width (cooperative kernel)
constexpr int NB = kQRBlock;  // block-reflector width (128)
constexpr int PT = 512;       // threads per panel CTA
constexpr int GMAX = 512;     // max CTAs of a panel grid (buffer sizing)

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Buffers (double-buffered by column parity):
//   nrm[2][GMAX]      partial ||x||^2 below the diagonal
//   dot[2][GMAX][PB]  partial x^T P_q (rows >= diagonal)
//   row[2][PB]        the diagonal row of the panel (published by its owner)
struct PanelBufs {
    double* nrm;
    double* dot;
    double* row;
};

// Factor the mr x jb panel P (ld) in place: R above the diagonal, unit-lower
// Householder vectors below, tau[0..jb).
template <bool SMEM>
__global__ void __launch_bounds__(PT) qr_panel_coop(int64_t mr, int jb, double* __restrict__ P,
                                                    int64_t ld, int64_t rows_per,
                                                    double* __restrict__ tau_out, PanelBufs buf,
                                                    const int* __restrict__ only_if) {
    // only_if (device flag, may be null): run only when it is 2 -- the
    // CholeskyQR panel found its Q not orthonormal and left P untouched
    if (only_if && *only_if != 2) return;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double slab[];  // rows_per x PB (ld rows_per) when SMEM
    __shared__ double red[2][PT / 32][PB + 1];  // by partial parity: no barrier before reuse
    __shared__ double wraw[PB], wsh[PB];
    __shared__ double sc[3];
    const int G = gridDim.x;
    const int64_t r0 = int64_t(blockIdx.x) * rows_per;
    const int64_t r1 = min(mr, r0 + rows_per);
    const int nrow = r1 > r0 ? int(r1 - r0) : 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto at = [&](int64_t i, int q) -> double& {
        if (SMEM) return slab[(i - r0) + int64_t(q) * rows_per];
        return P[i + int64_t(q) * ld];
    };
    if (SMEM) {
        for (int q = 0; q < jb; ++q)
            for (int k = threadIdx.x; k < nrow; k += PT) slab[k + int64_t(q) * rows_per] = P[r0 + k + q * ld];
        __syncthreads();
    }
    // partials of column `col` (after all previous updates): norm below the
    // diagonal, dots with the later columns, diagonal row -> slot `par`
    auto partials = [&](int col, int par) {
        double nacc = 0.0;
        double acc[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q) acc[q] = 0.0;
        for (int64_t i = max(r0, int64_t(col)) + threadIdx.x; i < r1; i += PT) {
            const double x = at(i, col);
            if (i > col) nacc += x * x;
#pragma unroll
            for (int q = 0; q < PB; ++q)
                if (q > col && q < jb) acc[q] += x * at(i, q);
            if (i == col)
                for (int q = col; q < jb; ++q) buf.row[par * PB + q] = at(i, q);
        }
        nacc = warp_sum(nacc);
        // transpose-reduce: afterwards lane q holds sum over lanes of acc[q]
        // (31 shuffles instead of 32 full butterflies)
#pragma unroll
        for (int sft = PB / 2; sft >= 1; sft >>= 1) {
            const bool upper = (lane & sft) != 0;
#pragma unroll
            for (int j = 0; j < sft; ++j) {
                const double send = upper ? acc[j] : acc[j + sft];
                const double keep = upper ? acc[j + sft] : acc[j];
                acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
            }
        }
        red[par][warp][lane] = acc[0];
        if (lane == 0) red[par][warp][PB] = nacc;
        __syncthreads();
        // the 32 dots and the norm summed over the 16 warps with shuffles,
        // one half-warp per quantity; slot 0 (dot 0 is never needed: q > col
        // >= 0) carries the norm
        {
            const int slot = 2 * warp + (lane >> 4), hl = lane & 15;
            const int q = slot == 0 ? PB : slot;
            double t = (q <= PB && hl < PT / 32) ? red[par][hl][q] : 0.0;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (hl == 0 && q <= PB) {
                if (q == PB) buf.nrm[par * GMAX + blockIdx.x] = t;
                else if (q > col && q < jb) buf.dot[(int64_t(par) * GMAX + blockIdx.x) * PB + q] = t;
            }
        }
    };
    partials(0, 0);
    for (int c = 0; c < jb; ++c) {
        const int par = c & 1;
        grid.sync();
        // ---- reflector of column c from the published partials (every CTA,
        // identical fixed-order warp reductions -> identical results).  Warp 0
        // reduces the G norm partials, the other warps the dot partials of
        // their columns; lanes stride over the partials so the L2 loads are
        // issued together instead of as one dependent chain.
        if (warp == 0) {
            double xn2 = 0.0;
            for (int p = lane; p < G; p += 32) xn2 += buf.nrm[par * GMAX + p];
            xn2 = warp_sum(xn2);
            if (lane == 0) {
                const double alpha = buf.row[par * PB + c];
                double tau = 0.0, beta = alpha, scal = 1.0;
                if (xn2 > 0.0) {
                    beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
                    tau = (beta - alpha) / beta;
                    scal = 1.0 / (alpha - beta);
                }
                sc[0] = tau;
                sc[1] = beta;
                sc[2] = scal;
            }
        } else {
            for (int q = c + warp; q < jb; q += PT / 32 - 1) {  // q = c+1, c+2, ...
                double s = 0.0;
                for (int p = lane; p < G; p += 32) s += buf.dot[(int64_t(par) * GMAX + p) * PB + q];
                s = warp_sum(s);
                if (lane == 0) wraw[q] = s;  // raw x^T P_q; scaled below
            }
        }
        __syncthreads();
        const double tau = sc[0], beta = sc[1], scal = sc[2];
        if (threadIdx.x < PB) {
            const int q = threadIdx.x;
            double wq = 0.0;
            if (q > c && q < jb) {
                const double pc = buf.row[par * PB + q];
                wq = pc + scal * (wraw[q] - buf.row[par * PB + c] * pc);  // v^T P_q, v_c = 1
            }
            wsh[q] = wq;
        }
        __syncthreads();
        // ---- apply H_c to the rest of the panel (own rows), store v
        for (int64_t i = max(r0, int64_t(c)) + threadIdx.x; i < r1; i += PT) {
            double v = 1.0;
            if (i > c) {
                v = at(i, c);
                if (tau != 0.0) {
                    v *= scal;
                    at(i, c) = v;
                }
            }
            if (tau != 0.0)
                for (int q = c + 1; q < jb; ++q) at(i, q) -= tau * v * wsh[q];
            if (i == c) at(i, c) = beta;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) tau_out[c] = tau;
        __syncthreads();
        // ---- look-ahead partials of column c+1
        if (c + 1 < jb) partials(c + 1, par ^ 1);
    }
    if (SMEM) {
        __syncthreads();
        for (int q = 0; q < jb; ++q)
            for (int k = threadIdx.x; k < nrow; k += PT) P[r0 + k + q * ld] = slab[k + int64_t(q) * rows_per];
    }
}

// Single-CTA panel for short panels (mr <= kCtaRows): the mr x jb slab lives
// in shared memory and each column costs two block barriers.  Phase 1: warp
// w computes s_q = x^T P[c+1:, q] for its columns q > c (x the unscaled
// sub-column below the diagonal) and the last warps the norm ||x||^2; phase
// 2: every thread forms (beta, tau, scal) redundantly, w_q = P_cq + scal
// s_q, and applies H_c = I - tau v v^T (v = [1; scal x]) to its (row, q)
// entries, storing v and beta.
constexpr int kCtaRows = 768;
constexpr int CT = 512;  // (1024 measured slower: barriers + 32-way norm reduction)
__global__ void __launch_bounds__(CT) qr_panel_cta(int mr, int jb, double* __restrict__ P, int64_t ld,
                                                   double* __restrict__ tau_out) {
    extern __shared__ double slab[];  // mr x jb, ld mr
    __shared__ double s_dot[PB], s_pc[PB];
    __shared__ double s_nrm[CT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = CT / 32;
    for (int q = 0; q < jb; ++q)
        for (int i = threadIdx.x; i < mr; i += CT) slab[i + q * mr] = P[i + int64_t(q) * ld];
    __syncthreads();
    for (int c = 0; c < jb; ++c) {
        const double* x = slab + int64_t(c) * mr;
        // ---- phase 1: dots with the later columns (warp per column) + norm
        const int nq = jb - c - 1;
        for (int t = warp; t < nq; t += NW) {
            const double* pq = slab + int64_t(c + 1 + t) * mr;
            // four independent partial sums: the dependent FMA chain over
            // the column was the critical path
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int i = c + 1 + lane;
            for (; i + 96 < mr; i += 128) {
                s0 += x[i] * pq[i];
                s1 += x[i + 32] * pq[i + 32];
                s2 += x[i + 64] * pq[i + 64];
                s3 += x[i + 96] * pq[i + 96];
            }
            for (; i < mr; i += 32) s0 += x[i] * pq[i];
            double s = (s0 + s1) + (s2 + s3);
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) {
                s_dot[c + 1 + t] = s;
                s_pc[c + 1 + t] = pq[c];  // P_cq before the update (phase 2 rewrites it)
            }
        }
        double nacc = 0.0;
#pragma unroll 2
        for (int i = c + 1 + threadIdx.x; i < mr; i += CT) nacc += x[i] * x[i];
        for (int o = 16; o > 0; o >>= 1) nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
        if (lane == 0) s_nrm[warp] = nacc;
        __syncthreads();
        // ---- phase 2: reflector (redundantly per warp) and update; the 16
        // warp partials are summed with shuffles, not a dependent load chain
        double xn2 = lane < NW ? s_nrm[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) xn2 += __shfl_xor_sync(0xffffffffu, xn2, o);  // all lanes get the sum
        const double alpha = x[c];
        double tau = 0.0, beta = alpha, scal = 1.0;
        if (xn2 > 0.0) {
            beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        if (tau != 0.0) {
            for (int q = c + 1 + warp; q < jb; q += NW) {  // warp per column, lanes over rows
                const double wq = s_pc[q] + scal * s_dot[q];
                double* pq = slab + int64_t(q) * mr;
                if (lane == 0) pq[c] -= tau * wq;  // v_c = 1
#pragma unroll 4
                for (int i = c + 1 + lane; i < mr; i += 32) pq[i] -= tau * (x[i] * scal) * wq;
            }
        }
        __syncthreads();  // column c, s_dot, s_pc and s_nrm fully consumed
        // scale column c into v; the next column's phase 1 touches only
        // columns > c, so no barrier is needed before it
        if (tau != 0.0)
            for (int i = c + 1 + threadIdx.x; i < mr; i += CT) slab[i + int64_t(c) * mr] *= scal;
        if (threadIdx.x == 0) {
            slab[c + int64_t(c) * mr] = beta;
            tau_out[c] = tau;
        }
    }
    __syncthreads();
    for (int q = 0; q < jb; ++q)
        for (int i = threadIdx.x; i < mr; i += CT) P[i + int64_t(q) * ld] = slab[i + q * mr];
}

// Vp (mr x jb, ld mr): unit lower trapezoid of the factored columns
__global__ void form_v(int64_t mr, int jb, const double* __restrict__ P, int64_t ld,
                       double* __restrict__ V) {
    int64_t total = mr * jb;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % mr;
        int q = int(e / mr);
        V[e] = i == q ? 1.0 : (i > q ? P[i + int64_t(q) * ld] : 0.0);
    }
}

// dlarft (forward, columnwise): T upper triangular jb x jb (ld NB) with
// H_0 ... H_{jb-1} = I - V T V^T, from G = V^T V and tau.  The 32 x 32
// diagonal blocks follow LAPACK's column recurrence (one warp per block, in
// parallel); they are then joined by the compact-WY merge
//   T = [[T1, -T1 (V1^T V2) T2], [0, T2]]
// at widths 32 -> 64 -> 128 with small shared-memory products.
constexpr int LT = 512;
__global__ void __launch_bounds__(LT) larft_k(int jb, const double* __restrict__ G, int64_t ldg,
                                              const double* __restrict__ tau, double* __restrict__ T) {
    extern __shared__ double Ts[];  // NB x (NB+1): T
    double* X = Ts + NB * (NB + 1);  // (NB/2) x (NB/2 + 1): merge scratch
    auto t = [&](int i, int j) -> double& { return Ts[i * (NB + 1) + j]; };
    constexpr int XL = NB / 2 + 1;
    for (int e = threadIdx.x; e < NB * (NB + 1); e += LT) Ts[e] = 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // ---- diagonal 32-blocks: warp w owns columns [32w, 32w+32)
    {
        const int b0 = warp * 32;
        if (b0 < jb) {
            const int bn = min(32, jb - b0);
            const int r = b0 + lane;  // this lane's row
            for (int ii = 0; ii < bn; ++ii) {
                const int i = b0 + ii;
                // t(r, i) = sum_{q=r}^{i-1} t(r, q) * (-tau_i G(q, i)),  r < i in the block
                double s = 0.0;
                if (lane < ii) {
                    const double ti = -tau[i];
                    for (int q = r; q < i; ++q) s += t(r, q) * (ti * G[q + int64_t(i) * ldg]);
                }
                __syncwarp();
                if (lane < ii) t(r, i) = s;
                if (lane == ii) t(i, i) = tau[i];
                __syncwarp();
            }
        }
    }
    __syncthreads();
    // ---- merges: width w blocks (w = 32, 64) pairwise into 2w
    for (int w = 32; w < jb; w *= 2) {
        for (int a0 = 0; a0 + w < jb; a0 += 2 * w) {
            const int b0 = a0 + w;
            const int na = w, nb = min(w, jb - b0);
            // X = G(a-block, b-block) * T2   (na x nb)
            for (int e = threadIdx.x; e < na * nb; e += LT) {
                const int i = e % na, j = e / na;
                double s = 0.0;
                for (int q = 0; q <= j; ++q) s += G[(a0 + i) + int64_t(b0 + q) * ldg] * t(b0 + q, b0 + j);
                X[i * XL + j] = s;
            }
            __syncthreads();
            // T12 = -T1 * X   (T1 upper triangular na x na)
            for (int e = threadIdx.x; e < na * nb; e += LT) {
                const int i = e % na, j = e / na;
                double s = 0.0;
                for (int q = i; q < na; ++q) s += t(a0 + i, a0 + q) * X[q * XL + j];
                t(a0 + i, b0 + j) = -s;
            }
            __syncthreads();
        }
    }
    for (int e = threadIdx.x; e < NB * jb; e += LT) {
        const int r = e % NB, j = e / NB;
        T[r + int64_t(j) * NB] = t(r, j);  // only jb columns exist
    }
}

}  // namespace
// a panel left untouched (Q not orthonormal) raises *sticky to 2
// (T, ldt): the panel's compact-WY triangle; form_v: work[0 .. mr jb) = explicit V on return
void panel_cqr(Ctx& c, int64_t mr, int jb, double* P, int64_t ld, double* tau, double* work,
               double* scratch, int* sticky, double* T, int64_t ldt, bool form_v);
int64_t cqr_scratch_doubles(const Ctx& c);
namespace {

// sticky != nullptr: tall panels by CholeskyQR (a failed panel raises
// *sticky and the caller redoes the factorisation with sticky == nullptr:
// cooperative Householder panels)
// Returns true when the CholeskyQR path also produced the sub-panel's T
// (into Tsub, ld NB) and, with want_v, its explicit V in work.
bool panel(Ctx& c, int64_t mr, int jb, double* P, int64_t ld, double* tau, const PanelBufs& pbuf,
           double* work, double* cqr_scratch, int* sticky, double* Tsub, bool want_v) {
    StageTimer _t(c, "qr_panel", mr, jb, -1, 2.0 * double(mr) * jb * jb, 16.0 * double(mr) * jb);
    // the same launches split by kind (one CTA on-chip / cooperative tall)
    StageTimer _k(c, mr <= kCtaRows ? "qr_panel_cta" : (sticky ? "qr_panel_cqr" : "qr_panel_coop"), mr, jb, -1,
                  2.0 * double(mr) * jb * jb, 16.0 * double(mr) * jb);
    const int* only_if = nullptr;
    if (mr > kCtaRows && sticky) {
        // tall: shifted CholeskyQR3 + Householder reconstruction (qr_cqr.cu).
        // A panel whose Q comes out non-orthonormal (numerically rank-deficient
        // within the panel) is left untouched and flagged; geqrf checks the
        // flag once at its end and redoes the factorisation with the
        // cooperative Householder kernel below.  (Launching that kernel after
        // every panel on the device flag cost a cooperative launch -- a full
        // drain of both streams -- per panel.)
        panel_cqr(c, mr, jb, P, ld, tau, work, cqr_scratch, sticky, Tsub, NB, want_v);
        return true;
    }
    static AttrGate attr;
    const size_t smem_cap = 200 * 1024;
    if (mr <= kCtaRows) {  // short panels: one CTA, the whole panel on-chip
        static AttrGate cattr;
        attr_once(cattr, c.device, [&] {
            HYDOT_CUDA(cudaFuncSetAttribute(qr_panel_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            int(smem_cap)));
        });
        qr_panel_cta<<<1, CT, size_t(mr) * jb * sizeof(double), c.stream>>>(int(mr), jb, P, ld, tau);
        c.check_launch();
        return false;
    }
    int G = c.num_sms;
    int64_t rows_per = (mr + G - 1) / G;
    if (rows_per < 64) {
        G = int(std::max<int64_t>(1, (mr + 63) / 64));
        rows_per = (mr + G - 1) / G;
    }
    if (G > GMAX) throw std::runtime_error("qr panel: grid too large");
    const size_t smem = size_t(rows_per) * PB * sizeof(double);
    const bool use_smem = smem <= smem_cap;
    attr_once(attr, c.device, [&] {
        HYDOT_CUDA(cudaFuncSetAttribute(qr_panel_coop<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(smem_cap)));
    });
    int per_sm = 0;
    if (use_smem)
        HYDOT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qr_panel_coop<true>, PT, smem));
    else
        HYDOT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qr_panel_coop<false>, PT, 0));
    if (per_sm * c.num_sms < G) throw std::runtime_error("qr panel: cooperative grid does not fit");
    PanelBufs b = pbuf;
    void* args[] = {&mr, &jb, &P, &ld, &rows_per, &tau, &b, &only_if};
    if (use_smem)
        c.coop_launch((void*)qr_panel_coop<true>, dim3(G), dim3(PT), args, smem);
    else
        c.coop_launch((void*)qr_panel_coop<false>, dim3(G), dim3(PT), args, 0);
    c.count();
    return false;
}

void form_v_launch(Ctx& c, int64_t mr, int jb, const double* P, int64_t ld, double* V) {
    int blocks = int(std::max<int64_t>(1, std::min<int64_t>((mr * jb + 255) / 256, int64_t(c.num_sms) * 8)));
    form_v<<<blocks, 256, 0, c.stream>>>(mr, jb, P, ld, V);
    c.check_launch();
}

// Sub-panel T in one launch: G = V^T V of the mr x jb (jb <= 32) unit
// lower-trapezoidal V held in the factored panel P (implicit unit diagonal,
// zeros above), reduced over row chunks, then T by the dlarft forward
// recurrence T(0:c, c) = -tau_c T(0:c, 0:c) G(0:c, c), T(c, c) = tau_c.
// Replaces form_v + the V^T V GEMM (+ split-K reduce) + larft_k of every
// 32-wide sub-panel.  The last CTA to finish (atomic ticket) reduces the
// per-CTA partial Grams in CTA order (deterministic) and forms T.
constexpr int GT = 256;     // threads
constexpr int GTILE = 128;  // rows staged per tile
__global__ void __launch_bounds__(GT) gram_t32_k(int64_t mr, int jb, const double* __restrict__ P, int64_t ld,
                                                 int64_t rows_per, const double* __restrict__ tau,
                                                 double* __restrict__ T, double* __restrict__ part,
                                                 unsigned* __restrict__ ticket) {
    __shared__ double tile[GTILE][PB + 1];
    __shared__ double Gs[PB][PB + 1];
    __shared__ bool last;
    const int npairs = jb * (jb + 1) / 2;
    int ep[3], eq[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // entry e -> (p, q), p <= q, column-major upper
        const int e = threadIdx.x + k * GT;
        int q = 0;
        while ((q + 1) * (q + 2) / 2 <= e) ++q;
        ep[k] = e < npairs ? e - q * (q + 1) / 2 : -1;
        eq[k] = q;
    }
    double acc[3] = {0.0, 0.0, 0.0};
    const int64_t r0 = int64_t(blockIdx.x) * rows_per, r1 = min(mr, r0 + rows_per);
    for (int64_t t0 = r0; t0 < r1; t0 += GTILE) {
        const int nt = int(min(int64_t(GTILE), r1 - t0));
        for (int e = threadIdx.x; e < GTILE * jb; e += GT) {
            const int rr = e % GTILE, q = e / GTILE;
            const int64_t i = t0 + rr;
            double v = 0.0;
            if (rr < nt) v = i > q ? P[i + int64_t(q) * ld] : (i == q ? 1.0 : 0.0);
            tile[rr][q] = v;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (ep[k] >= 0)
                for (int rr = 0; rr < nt; ++rr) acc[k] += tile[rr][ep[k]] * tile[rr][eq[k]];
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (ep[k] >= 0) part[int64_t(blockIdx.x) * npairs + threadIdx.x + k * GT] = acc[k];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (ep[k] >= 0) {
            // 8 independent partial sums (the loads overlap instead of one
            // dependent L2 round trip per CTA), combined in a fixed order
            const double* pp = part + threadIdx.x + k * GT;
            double g8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            int b = 0;
            for (; b + 8 <= int(gridDim.x); b += 8)
#pragma unroll
                for (int u = 0; u < 8; ++u) g8[u] += __ldcg(pp + int64_t(b + u) * npairs);
            for (; b < int(gridDim.x); ++b) g8[0] += __ldcg(pp + int64_t(b) * npairs);
            Gs[ep[k]][eq[k]] = ((g8[0] + g8[1]) + (g8[2] + g8[3])) + ((g8[4] + g8[5]) + (g8[6] + g8[7]));
        }
    __syncthreads();
    if (threadIdx.x < 32) {  // one warp: the column recurrence, lane i owns row i of T
        const int i = threadIdx.x;
        double trow[PB];
#pragma unroll
        for (int j = 0; j < PB; ++j) trow[j] = 0.0;
        for (int c = 0; c < jb; ++c) {
            const double tc = tau[c];
            // y_i = sum_{j=i..c-1} T(i, j) G(j, c)  (T upper triangular)
            double y = 0.0;
#pragma unroll
            for (int j = 0; j < PB; ++j)
                if (j >= i && j < c) y += trow[j] * Gs[j][c];
#pragma unroll
            for (int j = 0; j < PB; ++j)
                if (j == c) trow[j] = i < c ? -tc * y : (i == c ? tc : 0.0);
        }
        if (i < jb) {
#pragma unroll
            for (int j = 0; j < PB; ++j)
                if (j < jb) T[i + int64_t(j) * NB] = trow[j];
        }
        if (i == 0) *ticket = 0u;  // ready for the next launch on this stream
    }
}

void gram_t32(Ctx& c, int64_t mr, int jb, const double* P, int64_t ld, const double* tau, double* T,
              double* part, unsigned* ticket) {
    int G = int(std::min<int64_t>(c.num_sms, (mr + GTILE - 1) / GTILE));
    G = std::max(G, 1);
    const int64_t rows_per = (mr + G - 1) / G;
    gram_t32_k<<<G, GT, 0, c.stream>>>(mr, jb, P, ld, rows_per, tau, T, part, ticket);
    c.check_launch();
}

void larft(Ctx& c, int jb, const double* G, int64_t ldg, const double* tau, double* T) {
    static AttrGate attr;
    const int smem = (NB * (NB + 1) + (NB / 2) * (NB / 2 + 1)) * sizeof(double);
    attr_once(attr, c.device, [&] {
        HYDOT_CUDA(cudaFuncSetAttribute(larft_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    });
    larft_k<<<1, LT, smem, c.stream>>>(jb, G, ldg, tau, T);
    c.check_launch();
}

}  // namespace

namespace {
// HYDOT_QR_LOOKAHEAD=1 turns the look-ahead below on (read per call: the
// tests run both ways in one process).  Off by default: measured on the
// B200 it takes 3-6 % off an isolated tall factorisation (262144 x 1542:
// 78.9 -> 74.5 ms) but the config-2 step stays within its run-to-run noise
// (the tall QRs already run beside other work on the side stream), while the
// products that share the SMs with the panels stretch (GEMM class 0.69 ->
// 0.64 of the FP64 peak).  profiles/lookahead_r02.txt.
bool lookahead_on() {
    const char* e = std::getenv("HYDOT_QR_LOOKAHEAD");
    return e && e[0] == '1';
}

// restores the context stream; on an exception the panel stream is drained
// first (the buffers it uses are released in the caller's stream order)
struct StreamScope {
    Ctx& c;
    cudaStream_t keep, drain;
    int depth = std::uncaught_exceptions();
    ~StreamScope() {
        c.stream = keep;
        if (drain != keep && std::uncaught_exceptions() > depth) cudaStreamSynchronize(drain);
    }
};

// C -= V T^T V^T C for the nc columns at C (ld ldc): the block reflector of
// the jb columns factored last (V mr x jb explicit, T jb x jb, ld NB)
void block_update(Ctx& c, int64_t mr, int jb, const double* V, const double* T, int64_t nc, double* C,
                  int64_t ldc, double* W, double* W2) {
    dgemm(c, true, false, jb, nc, mr, 1.0, V, mr, C, ldc, 0.0, W, jb);
    dgemm(c, true, false, jb, nc, jb, 1.0, T, NB, W, jb, 0.0, W2, jb);
    dgemm(c, false, false, mr, nc, jb, -1.0, V, mr, W2, jb, 1.0, C, ldc);
}

// one pass of the blocked factorisation; sticky (device int, may be null):
// see panel().
//
// Look-ahead (tall mode, n >= 3 blocks): the panel chain is latency-bound
// (four streaming passes + three single-CTA tails per 32 columns) and the
// trailing update is DMMA work, so part of it runs beside the next block's
// panels.  Of block j's update C -= V (T^T (V^T C)), the products W = V^T C
// and W2 = T^T W are formed for all trailing columns on a high-priority
// stream H (W = V^T C is a split-K product whose CTAs live for ~1 ms: beside
// it the panel kernels would wait that long for SM slots, which an earlier
// version that overlapped the whole update measured), then C -= V W2 is
// applied on H to the next block's columns only, H goes on to factor block
// j + 1, and the rest of C -= V W2 (short CTAs) runs meanwhile on the caller's
// stream S.  Order: S waits for W2 (event evH); H waits for S's update (evR)
// before it reads the trailing columns again for block j + 1's V^T C.  Every
// column sees the same operations in the same order as in line.
void geqrf_run(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, QRFact& f, int* sticky) {
    f.m = m;
    f.n = n;
    // buffers may be preallocated by the caller (on another stream)
    if (f.a.bytes() < size_t(std::max<int64_t>(m * n, 1)) * 8) f.a = dalloc(c, size_t(std::max<int64_t>(m * n, 1)));
    if (f.tau.bytes() < size_t(std::max<int64_t>(n, 1)) * 8) f.tau = dalloc(c, size_t(std::max<int64_t>(n, 1)));
    if (f.T.bytes() < size_t(NB) * size_t(std::max<int64_t>(n, 1)) * 8)
        f.T = dalloc(c, size_t(NB) * size_t(std::max<int64_t>(n, 1)));
    copy2d(c, m, n, A, lda, f.a.d(), m);
    const int64_t k = std::min(m, n);
    if (k <= 0) return;
    double* a = f.a.d();
    const bool ahead = sticky && n >= 3 * NB && lookahead_on();
    DBuf pb_mem = dalloc(c, size_t(2) * GMAX + size_t(2) * GMAX * PB + 2 * PB);
    PanelBufs pbuf{pb_mem.d(), pb_mem.d() + 2 * GMAX, pb_mem.d() + 2 * GMAX + 2 * GMAX * PB};
    DBuf V = dalloc(c, size_t(m) * NB);  // panel scratch and the sub-panel's explicit V
    // the 128-wide block V: with look-ahead block j's is still read by R(j)
    // while block j + 1 is factored, so two alternate (else V serves)
    DBuf Vb[2];
    if (ahead)
        for (auto& v : Vb) v = dalloc(c, size_t(m) * NB);
    DBuf cqr = dalloc(c, size_t(cqr_scratch_doubles(c)));
    DBuf G = dalloc(c, size_t(NB) * NB);
    DBuf W = dalloc(c, size_t(NB) * size_t(std::max<int64_t>(n, 1)));
    DBuf W2 = dalloc(c, size_t(NB) * size_t(std::max<int64_t>(n, 1)));
    DBuf Wr, W2r;  // the block-level products (W2r is read on S while H factors the next block)
    if (ahead) {
        Wr = dalloc(c, size_t(NB) * size_t(n));
        W2r = dalloc(c, size_t(NB) * size_t(n));
    }
    DBuf Tp = dalloc(c, size_t(NB) * NB);
    DBuf gpart = dalloc(c, size_t(c.num_sms) * (PB * (PB + 1) / 2));
    DBuf gticket(c, sizeof(unsigned));
    HYDOT_CUDA(cudaMemsetAsync(gticket.as<void>(), 0, sizeof(unsigned), c.stream));
    const cudaStream_t S = c.stream;
    const cudaStream_t H = ahead ? c.hp_stream(S == c.side ? 1 : 0) : S;
    cudaEvent_t evH = nullptr, evR = nullptr;
    bool r_pending = false;
    StreamScope scope{c, S, H};
    struct EvGuard {
        cudaEvent_t &a, &b;
        ~EvGuard() {
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } evg{evH, evR};
    if (ahead) {
        HYDOT_CUDA(cudaEventCreateWithFlags(&evH, cudaEventDisableTiming));
        HYDOT_CUDA(cudaEventCreateWithFlags(&evR, cudaEventDisableTiming));
        HYDOT_CUDA(cudaEventRecord(evR, S));  // the copy and the buffers above
        HYDOT_CUDA(cudaStreamWaitEvent(H, evR, 0));
    }
    int64_t blk = 0;
    for (int64_t j0 = 0; j0 < k; j0 += NB, ++blk) {
        const int jb = int(std::min<int64_t>(NB, k - j0));
        const int64_t mr = m - j0;
        double* Pb = a + j0 + j0 * m;  // top-left of the 128-block
        c.stream = H;
        // ---- factor the block with 32-wide panels
        for (int p0 = 0; p0 < jb; p0 += PB) {
            const int pb = std::min(PB, jb - p0);
            const int64_t pr = mr - p0;
            double* Pp = Pb + p0 + int64_t(p0) * m;
            const int rest = jb - p0 - pb;
            const bool have_tv =
                panel(c, pr, pb, Pp, m, f.tau.d() + j0 + p0, pbuf, V.d(), cqr.d(), sticky, Tp.d(), rest > 0);
            if (rest > 0) {
                // apply this sub-panel's reflector to the rest of the block
                // (the CholeskyQR panel leaves V and T behind)
                if (!have_tv) {
                    form_v_launch(c, pr, pb, Pp, m, V.d());
                    gram_t32(c, pr, pb, Pp, m, f.tau.d() + j0 + p0, Tp.d(), gpart.d(), gticket.as<unsigned>());
                }
                block_update(c, pr, pb, V.d(), Tp.d(), rest, Pp + int64_t(pb) * m, m, W.d(), W2.d());
            }
        }
        // ---- 128-wide block reflector: T and the trailing update
        double* Vblk = ahead ? Vb[blk & 1].d() : V.d();
        form_v_launch(c, mr, jb, Pb, m, Vblk);
        dgemm(c, true, false, jb, jb, mr, 1.0, Vblk, mr, Vblk, mr, 0.0, G.d(), jb);
        larft(c, jb, G.d(), jb, f.tau.d() + j0, f.T.d() + j0 * NB);
        const int64_t nr = n - j0 - jb;
        if (nr <= 0) continue;
        double* Cm = a + j0 + (j0 + jb) * m;
        const double* Tj = f.T.d() + j0 * NB;
        if (!ahead) {
            block_update(c, mr, jb, Vblk, Tj, nr, Cm, m, W.d(), W2.d());
            continue;
        }
        // on H: W2 = T^T (V^T C) for every trailing column (S's part of the
        // previous update must have landed), C -= V W2 on the next block
        const int64_t nn = std::min<int64_t>(NB, nr);
        if (r_pending) HYDOT_CUDA(cudaStreamWaitEvent(H, evR, 0));
        r_pending = false;
        dgemm(c, true, false, jb, nr, mr, 1.0, Vblk, mr, Cm, m, 0.0, Wr.d(), jb);
        dgemm(c, true, false, jb, nr, jb, 1.0, Tj, NB, Wr.d(), jb, 0.0, W2r.d(), jb);
        dgemm(c, false, false, mr, nn, jb, -1.0, Vblk, mr, W2r.d(), jb, 1.0, Cm, m);
        if (nr > nn) {
            HYDOT_CUDA(cudaEventRecord(evH, H));
            // on S: the remaining columns, beside block j + 1's panels
            c.stream = S;
            HYDOT_CUDA(cudaStreamWaitEvent(S, evH, 0));
            dgemm(c, false, false, mr, nr - nn, jb, -1.0, Vblk, mr, W2r.d() + nn * jb, jb, 1.0, Cm + nn * m, m);
            HYDOT_CUDA(cudaEventRecord(evR, S));
            r_pending = true;
        }
    }
    if (ahead) {  // join: the caller's stream owns every buffer above
        HYDOT_CUDA(cudaEventRecord(evH, H));
        HYDOT_CUDA(cudaStreamWaitEvent(S, evH, 0));
    }
    c.stream = S;
}
}  // namespace

void geqrf(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, QRFact& f, QRCheck chk) {
    StageTimer _t(c, "qr_geqrf", m, n, -1, 2.0 * double(m) * double(n) * double(n));
    f.unverified = false;
    // CholeskyQR panels only exist above kCtaRows rows
    const bool tall = chk != QRCheck::Safe && m > kCtaRows && std::min(m, n) > 0;
    if (!tall) {
        geqrf_run(c, m, n, A, lda, f, nullptr);
        return;
    }
    if (f.flag.bytes() < sizeof(int)) f.flag = DBuf(c, sizeof(int));
    HYDOT_CUDA(cudaMemsetAsync(f.flag.as<void>(), 0, sizeof(int), c.stream));
    geqrf_run(c, m, n, A, lda, f, f.flag.as<int>());
    f.unverified = true;
    if (chk == QRCheck::Now && !geqrf_verify(c, f)) geqrf(c, m, n, A, lda, f, QRCheck::Safe);
}

bool geqrf_verify(Ctx& c, QRFact& f) {
    if (!f.unverified) return true;
    int v = 0;
    HYDOT_CUDA(cudaMemcpyAsync(&v, f.flag.as<void>(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    f.unverified = false;
    static const bool stats = [] {  // HYDOT_QR_STATS=1: report factorisations that are redone
        const char* e = std::getenv("HYDOT_QR_STATS");
        return e && e[0] == '1';
    }();
    if (stats) {
        static long n_all = 0, n_redo = 0;
        ++n_all;
        n_redo += v != 0;
        if (v != 0 || n_all % 100 == 0)
            fprintf(stderr, "[geqrf] m=%lld n=%lld %s (factorisations %ld, redone %ld)\n", (long long)f.m,
                    (long long)f.n, v ? "redo by Householder panels" : "ok", n_all, n_redo);
    }
    return v == 0;
}

void apply_q(Ctx& c, const QRFact& f, bool trans, int64_t k, double* Y, int64_t ldy, int64_t nz_rows) {
    StageTimer _t(c, "qr_apply_q", f.m, f.n, k, 4.0 * double(f.m) * double(std::min(f.m, f.n)) * double(k));
    const int64_t m = f.m, kk = std::min(f.m, f.n);
    if (k <= 0 || kk <= 0) return;
    DBuf V = dalloc(c, size_t(m) * NB);
    DBuf W = dalloc(c, size_t(NB) * size_t(k));
    DBuf W2 = dalloc(c, size_t(NB) * size_t(k));
    const int64_t nblk = (kk + NB - 1) / NB;
    // Q [Z; 0] (nz_rows = rows of Z): rows >= nzr of Y are still zero, so
    // the first block applied reads only Y[j0, nzr) in W = V^T Y, and blocks
    // entirely below nzr leave Y unchanged
    int64_t nzr = (nz_rows >= 0 && !trans) ? std::min(nz_rows, m) : m;
    for (int64_t bi = 0; bi < nblk; ++bi) {
        const int64_t b = trans ? bi : (nblk - 1 - bi);
        const int64_t j0 = b * NB;
        const int jb = int(std::min<int64_t>(NB, kk - j0));
        const int64_t mr = m - j0;
        if (j0 >= nzr) continue;  // H_b acts on zero rows only
        const int64_t kr = std::min(mr, nzr - j0);
        form_v_launch(c, mr, jb, f.a.d() + j0 + j0 * m, m, V.d());
        double* Ys = Y + j0;
        dgemm(c, true, false, jb, k, kr, 1.0, V.d(), mr, Ys, ldy, 0.0, W.d(), jb);
        // Q Y uses T, Q^T Y uses T^T
        dgemm(c, trans, false, jb, k, jb, 1.0, f.T.d() + j0 * NB, NB, W.d(), jb, 0.0, W2.d(), jb);
        dgemm(c, false, false, mr, k, jb, -1.0, V.d(), mr, W2.d(), jb, 1.0, Ys, ldy);
        nzr = m;  // rows >= j0 are dense from here on
    }
}

}  // namespace hydot
