// gemm.cu -- FP64 tensor-core (DMMA, mma.sync m16n8k4 .f64) GEMM for sm_100a.
//
// Replaces every dense product of the reference hot path: Eigen A*B in
// lowrank::gemm (lowrank.cpp:31-36), apply_mm / dense_op (lowrank.cpp:95-120)
// and the matvecs (lowrank.cpp:589-599).  sm_100 has no FP64 tcgen05 kind
// (SURVEY 0.4), so FP64 tensor math is the DMMA path.
//
// Column-major C = alpha op(A) op(B) + beta C.  64x64x16 CTA tiles, 4 warps
// (2x2, 32x32 warp tiles = 2x4 m16n8 fragments), 3-stage cp.async pipeline,
// bank-conflict-free k-major shared tiles (row stride 68 doubles).  K-long
// shapes (the sketch A*Omega with K = N voxels) use split-K: each z-slice
// writes a partial tile to a workspace and a second kernel sums the slices
// in fixed z order, so results are deterministic run to run.
#include "internal.h"

namespace hydot {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, LDS = 68, NT = 128;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
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

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) dgemm_kernel(int64_t M, int64_t N, int64_t K,
                                                   const double* __restrict__ A, int64_t lda,
                                                   const double* __restrict__ B, int64_t ldb,
                                                   double* __restrict__ C, int64_t ldc,
                                                   double alpha, double beta, int64_t kchunk,
                                                   double* __restrict__ ws) {
    extern __shared__ __align__(16) double smem_[];
    auto As = reinterpret_cast<double (*)[BK][LDS]>(smem_);
    auto Bs = reinterpret_cast<double (*)[BK][LDS]>(smem_ + STAGES * BK * LDS);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t m0 = int64_t(blockIdx.x) * BM, n0 = int64_t(blockIdx.y) * BN;
    const int64_t kbeg = int64_t(blockIdx.z) * kchunk;
    const int64_t kend = min(K, kbeg + kchunk);
    const int ktiles = kend > kbeg ? int((kend - kbeg + BK - 1) / BK) : 0;

    auto load_tile = [&](int stage, int64_t k0) {
#pragma unroll
        for (int e = 0; e < (BM * BK) / NT; ++e) {
            int idx = tid + e * NT;
            int i, kk;
            if (!TA) {
                i = idx % BM;
                kk = idx / BM;
            } else {
                kk = idx % BK;
                i = idx / BK;
            }
            int64_t gi = m0 + i, gk = k0 + kk;
            bool ok = gi < M && gk < kend;
            const double* src = ok ? (TA ? A + gk + gi * lda : A + gi + gk * lda) : A;
            cp_async8(&As[stage][kk][i], src, ok);
        }
#pragma unroll
        for (int e = 0; e < (BN * BK) / NT; ++e) {
            int idx = tid + e * NT;
            int j, kk;
            if (!TB) {
                kk = idx % BK;
                j = idx / BK;
            } else {
                j = idx % BN;
                kk = idx / BN;
            }
            int64_t gj = n0 + j, gk = k0 + kk;
            bool ok = gj < N && gk < kend;
            const double* src = ok ? (TB ? B + gj + gk * ldb : B + gk + gj * ldb) : B;
            cp_async8(&Bs[stage][kk][j], src, ok);
        }
    };

    double acc[2][4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[a][b][q] = 0.0;

    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    const int g = lane >> 2, t = lane & 3;

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
        const int st = kt % STAGES;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[2][2], b[4];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) {
                a[mi][0] = As[st][kk + t][wm + mi * 16 + g];
                a[mi][1] = As[st][kk + t][wm + mi * 16 + g + 8];
            }
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[st][kk + t][wn + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma16x8x4(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
        }
    }
    cp_async_wait<0>();

    const bool split = gridDim.z > 1;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                int64_t r = m0 + wm + mi * 16 + g + ((q & 2) ? 8 : 0);
                int64_t cc = n0 + wn + ni * 8 + 2 * t + (q & 1);
                if (r >= M || cc >= N) continue;
                double v = acc[mi][ni][q];
                if (split) {
                    ws[int64_t(blockIdx.z) * M * N + r + cc * M] = v;
                } else {
                    double* cp = C + r + cc * ldc;
                    *cp = beta == 0.0 ? alpha * v : alpha * v + beta * *cp;
                }
            }
}

__global__ void splitk_reduce(int64_t M, int64_t N, int splits, const double* __restrict__ ws,
                              double* __restrict__ C, int64_t ldc, double alpha, double beta) {
    int64_t total = M * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < splits; ++z) s += ws[int64_t(z) * total + e];
        int64_t r = e % M, cc = e / M;
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

}  // namespace

void dgemm(Ctx& c, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
           const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
           int64_t ldc) {
    StageTimer _t(c, "gemm", m, n, k, 2.0 * double(m) * double(n) * double(k),
                  8.0 * (double(m) * k + double(k) * n + double(m) * n * (beta != 0.0 ? 2 : 1)));
    if (m <= 0 || n <= 0) return;
    if (k <= 0 || alpha == 0.0) {
        int blocks = int(std::min<int64_t>((m * n + 255) / 256, 4096));
        scale_kernel<<<blocks, 256, 0, c.stream>>>(m, n, beta, C, ldc);
        c.check_launch();
        return;
    }
    int64_t tm = (m + BM - 1) / BM, tn = (n + BN - 1) / BN;
    int64_t tiles = tm * tn;
    int64_t target = int64_t(c.num_sms) * 4;
    int64_t splits = 1;
    if (tiles < target) {
        splits = (target + tiles - 1) / tiles;
        splits = std::min<int64_t>(splits, (k + 255) / 256);  // >= 256 k per slice
        // bound the workspace to 512 MB
        int64_t cap = (int64_t(512) << 20) / (8 * m * n);
        splits = std::max<int64_t>(1, std::min(splits, std::max<int64_t>(cap, 1)));
    }
    int64_t kchunk = (k + splits - 1) / splits;
    kchunk = (kchunk + BK - 1) / BK * BK;
    splits = (k + kchunk - 1) / kchunk;
    if (tn > 65535) throw std::invalid_argument("dgemm: n too large");
    if (splits > 65535) throw std::invalid_argument("dgemm: split too large");
    dim3 grid = dim3(unsigned(tm), unsigned(tn), unsigned(splits));
    DBuf ws;
    if (splits > 1) ws = dalloc(c, size_t(splits * m * n));
    constexpr size_t smem = size_t(2) * STAGES * BK * LDS * sizeof(double);
    static bool attr = false;
    if (!attr) {
        HYDOT_CUDA(cudaFuncSetAttribute(dgemm_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        HYDOT_CUDA(cudaFuncSetAttribute(dgemm_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        HYDOT_CUDA(cudaFuncSetAttribute(dgemm_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        HYDOT_CUDA(cudaFuncSetAttribute(dgemm_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr = true;
    }
    auto launch = [&](auto kern) {
        kern<<<grid, NT, smem, c.stream>>>(m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, kchunk,
                                        ws.d());
    };
    if (!ta && !tb) launch(dgemm_kernel<false, false>);
    else if (!ta && tb) launch(dgemm_kernel<false, true>);
    else if (ta && !tb) launch(dgemm_kernel<true, false>);
    else launch(dgemm_kernel<true, true>);
    c.check_launch();
    if (splits > 1) {
        int blocks = int(std::min<int64_t>((m * n + 255) / 256, int64_t(c.num_sms) * 8));
        splitk_reduce<<<blocks, 256, 0, c.stream>>>(m, n, int(splits), ws.d(), C, ldc, alpha,
                                                    beta);
        c.check_launch();
    }
}

}  // namespace hydot
