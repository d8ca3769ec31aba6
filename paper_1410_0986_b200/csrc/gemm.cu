// gemm.cu -- FP64 tensor-core (DMMA, mma.sync m16n8k4 .f64) GEMM for sm_100a.
//
// Replaces every dense product of the reference hot path: Eigen A*B in
// lowrank::gemm (lowrank.cpp:31-36), apply_mm / dense_op (lowrank.cpp:95-120)
// and the matvecs (lowrank.cpp:589-599).  sm_100 has no FP64 tcgen05 kind
// (SURVEY 0.4), so FP64 tensor math is the DMMA path.
//
// Column-major C = alpha op(A) op(B) + beta C.  64x64x16 tiles, 4 warps
// (2x2, 32x32 warp tiles), 3 resident CTAs per SM, 3-stage cp.async pipeline
// (16-byte copies when the operand is aligned), bank-conflict-free shared
// layouts.  The beta != 0 epilogue issues all C reads of a fragment before
// any store (the QR trailing updates are K=128 and were epilogue-latency
// bound: 16 -> 27.6 TF/s).  A 128x128 / 8-warp variant of the same template
// measured slower on every path shape (1 CTA/SM at 254 registers).  K-long shapes use split-K: each z-slice writes a
// partial tile to a workspace and a second kernel sums the slices in fixed
// z order, so results are deterministic run to run.
#include <cstdlib>

#include "internal.h"

namespace hydot {
namespace {

constexpr int BK = 16, STAGES = 3;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int bytes) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma16x8x4(double (&d)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

// Stage an RC x SC block of a column-major operand (RC along the contiguous
// dimension) into shared memory laid out dst[s * L + r]: the global
// contiguous dimension stays contiguous, so aligned operands move in 16-byte
// cp.async pairs.  Out-of-range elements are zero-filled.
template <int RC, int SC, int L, int NT>
__device__ __forceinline__ void load_block(double* dst, const double* __restrict__ g, int64_t ld,
                                           int64_t r0, int64_t rmax, int64_t s0, int64_t smax,
                                           bool vec, int tid) {
    if (vec && r0 + RC <= rmax && s0 + SC <= smax) {  // interior block: no predicates
        const double* base = g + r0 + s0 * ld;
#pragma unroll
        for (int e = 0; e < (RC * SC) / (2 * NT); ++e) {
            const int idx = tid + e * NT;
            const int r = (idx % (RC / 2)) * 2, sidx = idx / (RC / 2);
            cp_async16(dst + sidx * L + r, base + r + int64_t(sidx) * ld, 16);
        }
    } else if (vec) {
#pragma unroll
        for (int e = 0; e < (RC * SC) / (2 * NT); ++e) {
            int idx = tid + e * NT;
            int r = (idx % (RC / 2)) * 2, sidx = idx / (RC / 2);
            int64_t gr = r0 + r, gs = s0 + sidx;
            int bytes = gs < smax ? (gr + 1 < rmax ? 16 : (gr < rmax ? 8 : 0)) : 0;
            cp_async16(dst + sidx * L + r, bytes ? g + gr + gs * ld : g, bytes);
        }
    } else {
#pragma unroll
        for (int e = 0; e < (RC * SC) / NT; ++e) {
            int idx = tid + e * NT;
            int r = idx % RC, sidx = idx / RC;
            int64_t gr = r0 + r, gs = s0 + sidx;
            bool ok = gr < rmax && gs < smax;
            cp_async8(dst + sidx * L + r, ok ? g + gr + gs * ld : g, ok);
        }
    }
}

// Shared layouts (all conflict-free for the m16n8k4 fragment reads):
//   A, !TA: [k][i] stride BM+4      A, TA: [i][k] stride BK+4
//   B, !TB: [j][k] stride BK+4      B, TB: [k][j] stride BN+4
template <int BM, int BN, int WM, int WN>
struct Tile {
    static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
    static constexpr int NT = 32 * WARPS_M * WARPS_N;
    static constexpr int MI = WM / 16, NI = WN / 8;
    static constexpr int A_ELEMS = (BM + 4) * BK > BM * (BK + 4) ? (BM + 4) * BK : BM * (BK + 4);
    static constexpr int B_ELEMS = (BN + 4) * BK > BN * (BK + 4) ? (BN + 4) * BK : BN * (BK + 4);
    static constexpr size_t SMEM = size_t(STAGES) * (A_ELEMS + B_ELEMS) * sizeof(double);
    // 64x64: 3 CTAs (12 warps) per SM; 128x64 (64x32 warp tiles): 2
    static constexpr int MIN_CTAS = NT <= 128 ? (BM * BN <= 4096 ? 3 : 2) : 1;
};

template <bool TA, bool TB, int BM, int BN, int WM, int WN>
__global__ void __launch_bounds__(Tile<BM, BN, WM, WN>::NT, Tile<BM, BN, WM, WN>::MIN_CTAS)
    dgemm_kernel(int64_t M, int64_t N, int64_t K, const double* __restrict__ A, int64_t lda,
                 const double* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t ldc,
                 double alpha, double beta, int64_t kchunk, double* __restrict__ ws, bool vecA,
                 bool vecB) {
    using T = Tile<BM, BN, WM, WN>;
    constexpr int NT = T::NT, MI = T::MI, NI = T::NI;
    constexpr int LA = TA ? BK + 4 : BM + 4, LB = TB ? BN + 4 : BK + 4;
    extern __shared__ __align__(16) double smem_[];
    double* As = smem_;
    double* Bs = smem_ + STAGES * T::A_ELEMS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t m0 = int64_t(blockIdx.x) * BM, n0 = int64_t(blockIdx.y) * BN;
    const int64_t kbeg = int64_t(blockIdx.z) * kchunk;
    const int64_t kend = min(K, kbeg + kchunk);
    const int ktiles = kend > kbeg ? int((kend - kbeg + BK - 1) / BK) : 0;
    const bool split = gridDim.z > 1;

    auto load_tile = [&](int stage, int64_t k0) {
        double* a = As + stage * T::A_ELEMS;
        double* b = Bs + stage * T::B_ELEMS;
        if (!TA) load_block<BM, BK, LA, NT>(a, A, lda, m0, M, k0, kend, vecA, tid);
        else load_block<BK, BM, LA, NT>(a, A, lda, k0, kend, m0, M, vecA, tid);
        if (!TB) load_block<BK, BN, LB, NT>(b, B, ldb, k0, kend, n0, N, vecB, tid);
        else load_block<BN, BK, LB, NT>(b, B, ldb, n0, N, k0, kend, vecB, tid);
    };

    const int wm = (warp % T::WARPS_M) * WM, wn = (warp / T::WARPS_M) * WN;
    const int g = lane >> 2, t = lane & 3;

    double acc[MI][NI][4];
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
        for (int b = 0; b < NI; ++b)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[a][b][q] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_tile(s, kbeg + int64_t(s) * BK);
        cp_async_commit();
    }
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        int nk = kt + STAGES - 1;
        if (nk < ktiles) load_tile(nk % STAGES, kbeg + int64_t(nk) * BK);
        cp_async_commit();
        const double* a_s = As + (kt % STAGES) * T::A_ELEMS;
        const double* b_s = Bs + (kt % STAGES) * T::B_ELEMS;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[MI][2], b[NI];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
                int i = wm + mi * 16 + g;
                a[mi][0] = TA ? a_s[i * LA + kk + t] : a_s[(kk + t) * LA + i];
                a[mi][1] = TA ? a_s[(i + 8) * LA + kk + t] : a_s[(kk + t) * LA + i + 8];
            }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
                int j = wn + ni * 8 + g;
                b[ni] = TB ? b_s[(kk + t) * LB + j] : b_s[j * LB + kk + t];
            }
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) dmma16x8x4(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
        }
    }
    cp_async_wait<0>();

    if (split) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    int64_t r = m0 + wm + mi * 16 + g + ((q & 2) ? 8 : 0);
                    int64_t cc = n0 + wn + ni * 8 + 2 * t + (q & 1);
                    if (r < M && cc < N) ws[int64_t(blockIdx.z) * M * N + r + cc * M] = acc[mi][ni][q];
                }
        return;
    }
    // beta != 0: issue every C read of the fragment before the first store so
    // the loads overlap instead of serialising one round trip per element
    if (beta != 0.0) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    int64_t r = m0 + wm + mi * 16 + g + ((q & 2) ? 8 : 0);
                    int64_t cc = n0 + wn + ni * 8 + 2 * t + (q & 1);
                    double cold = (r < M && cc < N) ? __ldcs(C + r + cc * ldc) : 0.0;
                    acc[mi][ni][q] = alpha * acc[mi][ni][q] + beta * cold;
                }
    } else {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[mi][ni][q] = alpha * acc[mi][ni][q];
    }
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                int64_t r = m0 + wm + mi * 16 + g + ((q & 2) ? 8 : 0);
                int64_t cc = n0 + wn + ni * 8 + 2 * t + (q & 1);
                if (r < M && cc < N) C[r + cc * ldc] = acc[mi][ni][q];
            }
}

// sum the split-K slices in a fixed order: threadIdx.x over 32 consecutive
// elements (coalesced), threadIdx.y over z-slices, then a fixed-order
// shared-memory combine -- a long serial load chain per element was the
// reduce's cost when one GEMM had hundreds of slices
constexpr int RZ = 8;
__global__ void __launch_bounds__(32 * RZ) splitk_reduce(int64_t M, int64_t N, int splits,
                                                         const double* __restrict__ ws,
                                                         double* __restrict__ C, int64_t ldc,
                                                         double alpha, double beta) {
    __shared__ double part[RZ][33];
    const int64_t total = M * N;
    for (int64_t e0 = blockIdx.x * int64_t(32); e0 < total; e0 += int64_t(gridDim.x) * 32) {
        const int64_t e = e0 + threadIdx.x;
        double s = 0.0;
        if (e < total)
            for (int z = threadIdx.y; z < splits; z += RZ) s += ws[int64_t(z) * total + e];
        part[threadIdx.y][threadIdx.x] = s;
        __syncthreads();
        if (threadIdx.y == 0 && e < total) {
            double t = 0.0;
#pragma unroll
            for (int y = 0; y < RZ; ++y) t += part[y][threadIdx.x];
            const int64_t r = e % M, cc = e / M;
            double* cp = C + r + cc * ldc;
            *cp = beta == 0.0 ? alpha * t : alpha * t + beta * *cp;
        }
        __syncthreads();
    }
}

// few slices: one thread per element
__global__ void splitk_reduce_1d(int64_t M, int64_t N, int splits, const double* __restrict__ ws,
                                 double* __restrict__ C, int64_t ldc, double alpha, double beta) {
    const int64_t total = M * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < splits; ++z) s += ws[int64_t(z) * total + e];
        const int64_t r = e % M, cc = e / M;
        double* cp = C + r + cc * ldc;
        *cp = beta == 0.0 ? alpha * s : alpha * s + beta * *cp;
    }
}

__global__ void scale_kernel(int64_t M, int64_t N, double beta, double* C, int64_t ldc) {
    int64_t total = M * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t r = e % M, cc = e / M;
        C[r + cc * ldc] = beta == 0.0 ? 0.0 : beta * C[r + cc * ldc];
    }
}

template <int BM, int BN, int WM, int WN>
void run_tiles(Ctx& c, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
               const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
               int64_t ldc) {
    using T = Tile<BM, BN, WM, WN>;
    int64_t tm = (m + BM - 1) / BM, tn = (n + BN - 1) / BN;
    int64_t tiles = tm * tn;
    // Split K when the output tiles alone leave the device under-filled.  The
    // slice count minimises waves x (k per slice + fixed per-CTA cost) + the
    // slice reduction, with a wave = the CTAs resident at once (MIN_CTAS per
    // SM): filling 4/3 of a wave (the earlier 4-per-SM target with 3
    // resident) ran two rounds for the price of 1.33 (ncu: 592 CTAs, 70 % of
    // the DMMA pipe on W = V^T C of the tall QRs).
    const int64_t wave = int64_t(c.num_sms) * T::MIN_CTAS;
    int64_t splits = 1;
    if (tiles < wave) {
        int64_t smax = std::min<int64_t>((k + 255) / 256, 128);          // >= 256 k per slice
        const int64_t cap = (int64_t(512) << 20) / (8 * m * n);          // workspace <= 512 MB
        smax = std::max<int64_t>(1, std::min(smax, std::max<int64_t>(cap, 1)));
        double best = 0.0;
        for (int64_t sp = 1; sp <= smax; ++sp) {
            int64_t kc = (k + sp - 1) / sp;
            kc = (kc + BK - 1) / BK * BK;
            const int64_t ns = (k + kc - 1) / kc;
            if (ns != sp) continue;  // same slices as a smaller count
            const double waves = double((tiles * sp + wave - 1) / wave);
            // k-steps of one CTA: its slice + prologue / epilogue; the
            // reduction reads sp partial tiles (in k-steps of a full wave)
            double cost = waves * (double(kc) + 48.0);
            if (sp > 1) cost += 32.0 + 2.7e-5 * double(sp) * double(m) * double(n);
            if (sp == 1 || cost < best) {
                best = cost;
                splits = sp;
            }
        }
    }
    int64_t kchunk = (k + splits - 1) / splits;
    kchunk = (kchunk + BK - 1) / BK * BK;
    splits = (k + kchunk - 1) / kchunk;
    if (tn > 65535) throw std::invalid_argument("dgemm: n too large");
    if (splits > 65535) throw std::invalid_argument("dgemm: split too large");
    dim3 grid = dim3(unsigned(tm), unsigned(tn), unsigned(splits));
    DBuf ws;
    if (splits > 1) ws = dalloc(c, size_t(splits * m * n));
    static AttrGate attr;
    attr_once(attr, c.device, [&] {
        HYDOT_CUDA(cudaFuncSetAttribute(dgemm_kernel<false, false, BM, BN, WM, WN>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(T::SMEM)));
        HYDOT_CUDA(cudaFuncSetAttribute(dgemm_kernel<false, true, BM, BN, WM, WN>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(T::SMEM)));
        HYDOT_CUDA(cudaFuncSetAttribute(dgemm_kernel<true, false, BM, BN, WM, WN>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(T::SMEM)));
        HYDOT_CUDA(cudaFuncSetAttribute(dgemm_kernel<true, true, BM, BN, WM, WN>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(T::SMEM)));
    });
    const bool vecA = (lda % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0);
    const bool vecB = (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0);
    auto launch = [&](auto kern) {
        kern<<<grid, T::NT, T::SMEM, c.stream>>>(m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, kchunk,
                                                ws.d(), vecA, vecB);
    };
    if (!ta && !tb) launch(dgemm_kernel<false, false, BM, BN, WM, WN>);
    else if (!ta && tb) launch(dgemm_kernel<false, true, BM, BN, WM, WN>);
    else if (ta && !tb) launch(dgemm_kernel<true, false, BM, BN, WM, WN>);
    else launch(dgemm_kernel<true, true, BM, BN, WM, WN>);
    c.check_launch();
    if (splits > 8) {
        int blocks = int(std::min<int64_t>((m * n + 31) / 32, int64_t(c.num_sms) * 16));
        splitk_reduce<<<blocks, dim3(32, RZ), 0, c.stream>>>(m, n, int(splits), ws.d(), C, ldc, alpha,
                                                             beta);
        c.check_launch();
    } else if (splits > 1) {
        int blocks = int(std::min<int64_t>((m * n + 255) / 256, int64_t(c.num_sms) * 8));
        splitk_reduce_1d<<<blocks, 256, 0, c.stream>>>(m, n, int(splits), ws.d(), C, ldc, alpha, beta);
        c.check_launch();
    }
}

}  // namespace

void dgemm(Ctx& c, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
           const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
           int64_t ldc) {
    StageTimer _t(c, "gemm", m, n, k, 2.0 * double(m) * double(n) * double(k),
                  8.0 * (double(m) * k + double(k) * n + double(m) * n * (beta != 0.0 ? 2 : 1)));
    // HYDOT_GEMM_CLASSES=1: also time by shape class (profiling aid)
    static const bool classes = [] {
        const char* e = std::getenv("HYDOT_GEMM_CLASSES");
        return e && e[0] == '1';
    }();
    std::unique_ptr<StageTimer> t2;
    if (classes) {
        const char* cls = (m <= 32 || n <= 32) ? (k >= 4096 ? "gemm_c_thin_longk" : "gemm_c_thin")
                          : k <= 32            ? "gemm_c_k32"
                          : k <= 128           ? "gemm_c_k128"
                          : k >= 4096          ? "gemm_c_longk"
                                               : "gemm_c_mid";
        t2.reset(new StageTimer(c, cls, m, n, k, 2.0 * double(m) * double(n) * double(k), 0.0));
    }
    if (m <= 0 || n <= 0) return;
    if (k <= 0 || alpha == 0.0) {
        int blocks = int(std::min<int64_t>((m * n + 255) / 256, 4096));
        scale_kernel<<<blocks, 256, 0, c.stream>>>(m, n, beta, C, ldc);
        c.check_launch();
        return;
    }
    // 64x64 CTA tiles (a 128x64 / 64x32-warp-tile variant measured slower on
    // every path shape: 254 registers, 2 CTAs/SM, QR W = V^T C 28 -> 18.6 TF/s)
    run_tiles<64, 64, 32, 32>(c, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

}  // namespace hydot
