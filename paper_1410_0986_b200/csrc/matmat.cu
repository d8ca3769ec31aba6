// matmat.cu -- epilogues of the low-rank J~ products.
//
// J~ X = P [E_1 U, ..., E_nc U] (V^T X_c): the two GEMMs run on the DMMA
// kernel; these kernels apply the chromophore scaling E_c (forward_measure,
// born.cpp:118-127: row m scaled by sum_c c_c eps_c(lambda_{m mod nl})) and
// the measurement permutation (permuted_matvec, experiments.cpp:255-262:
// out[row_perm[i]] = tmp[i]).
#include "internal.h"

namespace hydot {
namespace {

// Y[row_perm[i], j] = sum_c eps_c[l, c] * T[i, j*nc + c],  l = row_perm[i] % nl
__global__ void j_combine_k(int64_t M, int b, int nc, int nl, const double* __restrict__ T,
                            int64_t ldt, const int* __restrict__ rp, const double* __restrict__ eps,
                            double* __restrict__ Y, int64_t ldy) {
    int64_t total = M * b;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % M;
        int j = int(e / M);
        int row = rp[i];
        int l = row % nl;
        double s = 0.0;
        for (int c = 0; c < nc; ++c) s += eps[l + c * nl] * T[i + int64_t(j * nc + c) * ldt];
        Y[row + int64_t(j) * ldy] = s;
    }
}

// G[i, j*nc + c] = eps_c[l, c] * X[row_perm[i], j]
__global__ void j_gather_scale_k(int64_t M, int b, int nc, int nl, const double* __restrict__ X,
                                 int64_t ldx, const int* __restrict__ rp,
                                 const double* __restrict__ eps, double* __restrict__ G,
                                 int64_t ldg) {
    int64_t total = M * b;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % M;
        int j = int(e / M);
        int row = rp[i];
        int l = row % nl;
        double x = X[row + int64_t(j) * ldx];
        for (int c = 0; c < nc; ++c) G[i + int64_t(j * nc + c) * ldg] = eps[l + c * nl] * x;
    }
}

// X[c*N + v, j] = conc[c] * D[v, j]  (the chromophore axis of a shape
// perturbation: delta c_c(v) = conc_c * dmu(v), pals.cpp:124-135)
__global__ void kron_conc_k(int64_t N, int b, int nc, const double* __restrict__ conc,
                            const double* __restrict__ D, int64_t ldd, double* __restrict__ X, int64_t ldx) {
    const int64_t total = N * b * nc;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t v = e % N;
        const int64_t rest = e / N;
        const int c = int(rest % nc), j = int(rest / nc);
        X[int64_t(c) * N + v + int64_t(j) * ldx] = conc[c] * D[v + int64_t(j) * ldd];
    }
}

// Y[i, j] = w[i]^2 * X[i, j]
__global__ void wsq_rows_k(int64_t M, int b, const double* __restrict__ w, const double* __restrict__ X,
                           int64_t ldx, double* __restrict__ Y, int64_t ldy) {
    const int64_t total = M * b;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e % M;
        const int j = int(e / M);
        Y[i + int64_t(j) * ldy] = w[i] * w[i] * X[i + int64_t(j) * ldx];
    }
}

}  // namespace

void kron_conc(Ctx& c, int64_t N, int b, int nc, const double* conc_dev, const double* D, int64_t ldd,
               double* X, int64_t ldx) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((N * b * nc + 255) / 256, int64_t(c.num_sms) * 8)));
    kron_conc_k<<<blocks, 256, 0, c.stream>>>(N, b, nc, conc_dev, D, ldd, X, ldx);
    c.check_launch();
}

void wsq_rows(Ctx& c, int64_t M, int b, const double* w, const double* X, int64_t ldx, double* Y, int64_t ldy) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((M * b + 255) / 256, int64_t(c.num_sms) * 8)));
    wsq_rows_k<<<blocks, 256, 0, c.stream>>>(M, b, w, X, ldx, Y, ldy);
    c.check_launch();
}

// J~ X (trans = false: X (N nc) x b -> Y M x b) or J~^T X (X M x b -> Y
// (N nc) x b): permuted_matvec (experiments.cpp:255-262) with the E_c axis
// (born.cpp:118-127, pals.cpp:124-135) on the factor U V^T of H.
void j_matmat(Ctx& c, const double* U, const double* V, int64_t M, int64_t N, int64_t R, bool trans, int b,
              const int* row_perm, const double* eps_c, int nl, int nc, const double* X, int64_t ldx, double* Y,
              int64_t ldy) {
    const int64_t q = int64_t(b) * nc;
    if (b == 0) return;
    const double flops = 2.0 * double(R) * double(q) * double(N + M);
    const double bytes = 8.0 * (double(N) * R + double(M) * R + double(q) * N + double(b) * M);
    StageTimer _t(c, trans ? "j_matmat_adj" : "j_matmat_fwd", M, N, b, flops, bytes);
    if (!trans) {
        if (ldx != N * nc || ldy < M) throw std::invalid_argument("J matvec: dimension mismatch");
        if (R == 0) {
            fill(c, M, b, 0.0, Y, ldy);
            return;
        }
        DBuf Z = dalloc(c, size_t(R * q)), T = dalloc(c, size_t(M * q));
        if (skinny_ok(int(q))) {
            skinny_tn(c, N, R, int(q), V, N, X, N, Z.d(), R);
            skinny_nn(c, M, R, int(q), U, M, Z.d(), R, T.d(), M);
        } else {
            dgemm(c, true, false, R, q, N, 1.0, V, N, X, N, 0.0, Z.d(), R);
            dgemm(c, false, false, M, q, R, 1.0, U, M, Z.d(), R, 0.0, T.d(), M);
        }
        j_combine(c, M, b, nc, nl, T.d(), M, row_perm, eps_c, Y, ldy);
    } else {
        if (ldx < M || ldy != N * nc) throw std::invalid_argument("J rmatvec: dimension mismatch");
        if (R == 0) {
            fill(c, N * nc, b, 0.0, Y, ldy);
            return;
        }
        DBuf G = dalloc(c, size_t(M * q)), W = dalloc(c, size_t(R * q));
        j_gather_scale(c, M, b, nc, nl, X, ldx, row_perm, eps_c, G.d(), M);
        if (skinny_ok(int(q))) {
            skinny_tn(c, M, R, int(q), U, M, G.d(), M, W.d(), R);
            skinny_nn(c, N, R, int(q), V, N, W.d(), R, Y, N);
        } else {
            dgemm(c, true, false, R, q, M, 1.0, U, M, G.d(), M, 0.0, W.d(), R);
            dgemm(c, false, false, N, q, R, 1.0, V, N, W.d(), R, 0.0, Y, N);
        }
    }
}

void j_combine(Ctx& c, int64_t M, int b, int nc, int nl, const double* T, int64_t ldt,
               const int* row_perm, const double* eps_c, double* Y, int64_t ldy) {
    int blocks = int(std::max<int64_t>(1, std::min<int64_t>((M * b + 255) / 256, int64_t(c.num_sms) * 8)));
    j_combine_k<<<blocks, 256, 0, c.stream>>>(M, b, nc, nl, T, ldt, row_perm, eps_c, Y, ldy);
    c.check_launch();
}

void j_gather_scale(Ctx& c, int64_t M, int b, int nc, int nl, const double* X, int64_t ldx,
                    const int* row_perm, const double* eps_c, double* G, int64_t ldg) {
    int blocks = int(std::max<int64_t>(1, std::min<int64_t>((M * b + 255) / 256, int64_t(c.num_sms) * 8)));
    j_gather_scale_k<<<blocks, 256, 0, c.stream>>>(M, b, nc, nl, X, ldx, row_perm, eps_c, G, ldg);
    c.check_launch();
}

}  // namespace hydot

// --------------------------------------------------------- skinny GEMMs --
// The b = 1 J~ products are two tall-skinny matrix products (R x q and
// M x q with q = b * n_c <= 16): HBM-bound streams of V (N x R) and U
// (M x R).  The DMMA tile kernel wastes its 64-wide N tile there, so these
// kernels read every factor element exactly once with coalesced loads,
// keep the skinny operand in shared memory and reduce split partials in a
// fixed order (deterministic).
namespace hydot {
namespace {

constexpr int SK_T = 256;  // threads per CTA

// partial Z_chunk[j, c] = sum_{i in chunk} A[i, j] X[i, c]
template <int Q>
constexpr int skinny_rows() { return 4096 / Q > 256 ? 4096 / Q : 256; }

template <int Q>
__global__ void __launch_bounds__(SK_T) skinny_tn_k(int64_t K, int64_t R, int64_t T,
                                                    const double* __restrict__ A, int64_t lda,
                                                    const double* __restrict__ X, int64_t ldx,
                                                    double* __restrict__ part, int64_t jgroup,
                                                    int q) {
    extern __shared__ double xs[];  // T x Q (columns >= q are zero)
    constexpr int TT = skinny_rows<Q>();  // == T
    const int64_t i0 = int64_t(blockIdx.x) * T;
    const int64_t rows = min(T, K - i0);
    for (int64_t e = threadIdx.x; e < rows * Q; e += SK_T) {
        const int64_t i = e % rows;
        const int c = int(e / rows);
        xs[i + c * T] = c < q ? X[i0 + i + int64_t(c) * ldx] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t j0 = int64_t(blockIdx.y) * jgroup;
    const int64_t j1 = min(R, j0 + jgroup);
    for (int64_t j = j0 + warp; j < j1; j += SK_T / 32) {
        const double* a = A + i0 + j * lda;
        double acc[Q];
#pragma unroll
        for (int c = 0; c < Q; ++c) acc[c] = 0.0;
        if (rows == TT && (reinterpret_cast<uintptr_t>(a) & 15) == 0) {
            // full chunk: groups of 8 independent 128-bit loads per lane in
            // flight before they are consumed (HBM needs the bytes in flight)
            constexpr int KK = TT / 64;  // double2 per lane
#pragma unroll 1
            for (int k0 = 0; k0 < KK; k0 += 8) {
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(a + 2 * lane + 64 * (k0 + u)));
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = 2 * lane + 64 * (k0 + u);
#pragma unroll
                    for (int c = 0; c < Q; ++c) acc[c] += v[u].x * xs[i + c * TT] + v[u].y * xs[i + 1 + c * TT];
                }
            }
        } else if ((reinterpret_cast<uintptr_t>(a) & 15) == 0) {
            // 128-bit streaming loads: two rows per lane per step, two steps
            // in flight
            const int64_t rows2 = rows & ~int64_t(1);
            int64_t i = 2 * lane;
            for (; i + 64 < rows2; i += 128) {
                const double2 v = __ldcs(reinterpret_cast<const double2*>(a + i));
                const double2 u = __ldcs(reinterpret_cast<const double2*>(a + i + 64));
#pragma unroll
                for (int c = 0; c < Q; ++c)
                    acc[c] += v.x * xs[i + c * T] + v.y * xs[i + 1 + c * T] + u.x * xs[i + 64 + c * T] +
                              u.y * xs[i + 65 + c * T];
            }
            if (i < rows2) {
                const double2 v = __ldcs(reinterpret_cast<const double2*>(a + i));
#pragma unroll
                for (int c = 0; c < Q; ++c) acc[c] += v.x * xs[i + c * T] + v.y * xs[i + 1 + c * T];
            }
            if ((rows & 1) && lane == 0) {
                const double v = a[rows - 1];
#pragma unroll
                for (int c = 0; c < Q; ++c) acc[c] += v * xs[rows - 1 + c * T];
            }
        } else {
            for (int64_t i = lane; i < rows; i += 32) {
                const double v = __ldcs(a + i);
#pragma unroll
                for (int c = 0; c < Q; ++c) acc[c] += v * xs[i + c * T];
            }
        }
#pragma unroll
        for (int c = 0; c < Q; ++c)
            for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
        if (lane < q) {
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < Q; ++c)
                if (c == lane) v = acc[c];
            part[(int64_t(blockIdx.x) * R + j) * q + lane] = v;
        }
    }
}

// Z[j, c] = sum_chunks part[chunk][j][c] (fixed order)
// sum the chunk partials: threadIdx.x over 32 consecutive outputs, threadIdx.y
// over chunks, fixed-order shared-memory combine (no long dependent chain)
constexpr int SRZ = 8;
__global__ void __launch_bounds__(32 * SRZ) skinny_reduce_k(int64_t nchunks, int64_t R, int Q,
                                                            const double* __restrict__ part,
                                                            double* __restrict__ Z, int64_t ldz) {
    __shared__ double sh[SRZ][33];
    const int64_t total = R * Q;
    for (int64_t e0 = blockIdx.x * int64_t(32); e0 < total; e0 += int64_t(gridDim.x) * 32) {
        const int64_t e = e0 + threadIdx.x;
        double s = 0.0;
        if (e < total)
            for (int64_t k = threadIdx.y; k < nchunks; k += SRZ) s += part[k * total + e];
        sh[threadIdx.y][threadIdx.x] = s;
        __syncthreads();
        if (threadIdx.y == 0 && e < total) {
            double t = 0.0;
#pragma unroll
            for (int y = 0; y < SRZ; ++y) t += sh[y][threadIdx.x];
            Z[e / Q + (e % Q) * ldz] = t;
        }
        __syncthreads();
    }
}

// partial Y_chunk[i, c] = sum_{j in chunk} A[i, j] Z[j, c]
template <int Q>
__global__ void __launch_bounds__(SK_T) skinny_nn_k(int64_t M, int64_t R, int64_t RC,
                                                    const double* __restrict__ A, int64_t lda,
                                                    const double* __restrict__ Z, int64_t ldz,
                                                    double* __restrict__ part, int q) {
    extern __shared__ double zs[];  // RC x Q (columns >= q are zero)
    const int64_t j0 = int64_t(blockIdx.y) * RC;
    const int64_t cols = min(RC, R - j0);
    for (int64_t e = threadIdx.x; e < cols * Q; e += SK_T) {
        const int64_t j = e / Q;
        const int c = int(e % Q);
        zs[j * Q + c] = c < q ? Z[j0 + j + int64_t(c) * ldz] : 0.0;
    }
    __syncthreads();
    const int64_t i = int64_t(blockIdx.x) * SK_T + threadIdx.x;
    if (i >= M) return;
    double acc[Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) acc[c] = 0.0;
    const double* a = A + i + j0 * lda;
    int64_t j = 0;
    for (; j + 8 <= cols; j += 8) {  // 8 independent column loads in flight
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(a + (j + u) * lda);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < Q; ++c) acc[c] += v[u] * zs[(j + u) * Q + c];
    }
    for (; j < cols; ++j) {
        const double v = __ldcs(a + j * lda);
#pragma unroll
        for (int c = 0; c < Q; ++c) acc[c] += v * zs[j * Q + c];
    }
#pragma unroll
    for (int c = 0; c < Q; ++c)
        if (c < q) part[(int64_t(blockIdx.y) * q + c) * M + i] = acc[c];
}

__global__ void skinny_nn_reduce_k(int64_t M, int64_t nchunks, int Q, const double* __restrict__ part,
                                   double* __restrict__ Y, int64_t ldy) {
    const int64_t total = M * Q;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e % M;
        const int c = int(e / M);
        double s = 0.0;
        for (int64_t k = 0; k < nchunks; ++k) s += part[(k * Q + c) * M + i];
        Y[i + int64_t(c) * ldy] = s;
    }
}

template <int Q>
void skinny_tn_t(Ctx& c, int64_t K, int64_t R, int q, const double* A, int64_t lda, const double* X,
                 int64_t ldx, double* Z, int64_t ldz) {
    // 32 KB of X per CTA (several CTAs per SM: enough loads in flight to
    // stream A at HBM rate), at least 256 rows
    const int64_t T = skinny_rows<Q>();
    const int64_t nchunks = (K + T - 1) / T;
    const int64_t want = int64_t(c.num_sms) * 4;
    int64_t groups = std::max<int64_t>(1, (want + nchunks - 1) / nchunks);
    int64_t jgroup = std::max<int64_t>(8, (R + groups - 1) / groups);
    groups = (R + jgroup - 1) / jgroup;
    DBuf part = dalloc(c, size_t(nchunks * R * q));
    static AttrGate attr;
    attr_once(attr, c.device, [&] {
        HYDOT_CUDA(cudaFuncSetAttribute(skinny_tn_k<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(T * Q * 8)));
    });
    skinny_tn_k<Q><<<dim3(unsigned(nchunks), unsigned(groups)), SK_T, size_t(T * Q * 8), c.stream>>>(
        K, R, T, A, lda, X, ldx, part.d(), jgroup, q);
    c.check_launch();
    int blocks = int(std::max<int64_t>(1, std::min<int64_t>((R * q + 31) / 32, int64_t(c.num_sms) * 16)));
    skinny_reduce_k<<<blocks, dim3(32, SRZ), 0, c.stream>>>(nchunks, R, q, part.d(), Z, ldz);
    c.check_launch();
}

template <int Q>
void skinny_nn_t(Ctx& c, int64_t M, int64_t R, int q, const double* A, int64_t lda, const double* Z,
                 int64_t ldz, double* Y, int64_t ldy) {
    const int64_t rb = (M + SK_T - 1) / SK_T;
    const int64_t want = int64_t(c.num_sms) * 8;
    int64_t nch = std::max<int64_t>(1, std::min<int64_t>((want + rb - 1) / rb, (R + 63) / 64));
    int64_t RC = (R + nch - 1) / nch;
    RC = std::min<int64_t>(RC, 16384 / Q);
    nch = (R + RC - 1) / RC;
    DBuf part = dalloc(c, size_t(nch * q * M));
    static AttrGate attr;
    attr_once(attr, c.device, [&] {
        HYDOT_CUDA(cudaFuncSetAttribute(skinny_nn_k<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        16384 * 8));
    });
    skinny_nn_k<Q><<<dim3(unsigned(rb), unsigned(nch)), SK_T, size_t(RC * Q * 8), c.stream>>>(
        M, R, RC, A, lda, Z, ldz, part.d(), q);
    c.check_launch();
    int blocks = int(std::max<int64_t>(1, std::min<int64_t>((M * q + 255) / 256, int64_t(c.num_sms) * 8)));
    skinny_nn_reduce_k<<<blocks, 256, 0, c.stream>>>(M, nch, q, part.d(), Y, ldy);
    c.check_launch();
}

}  // namespace

// <= 8 right-hand sides: the streaming kernels; wider goes to the DMMA GEMM
// (16-wide skinny measured 2.7 ms vs 1.25 ms through DMMA on config-1 factors)
bool skinny_ok(int q) { return q >= 1 && q <= 8; }

void skinny_tn(Ctx& c, int64_t K, int64_t R, int q, const double* A, int64_t lda, const double* X,
               int64_t ldx, double* Z, int64_t ldz) {
    StageTimer _t(c, "skinny_tn", K, R, q, 2.0 * double(K) * R * q, 8.0 * (double(K) * R + double(K) * q));
    switch (q) {
        case 1: skinny_tn_t<1>(c, K, R, q, A, lda, X, ldx, Z, ldz); break;
        case 2: skinny_tn_t<2>(c, K, R, q, A, lda, X, ldx, Z, ldz); break;
        case 3: case 4: skinny_tn_t<4>(c, K, R, q, A, lda, X, ldx, Z, ldz); break;
        case 5: case 6: case 7: case 8: skinny_tn_t<8>(c, K, R, q, A, lda, X, ldx, Z, ldz); break;
        default: skinny_tn_t<16>(c, K, R, q, A, lda, X, ldx, Z, ldz); break;
    }
    (void)q;
}

void skinny_nn(Ctx& c, int64_t M, int64_t R, int q, const double* A, int64_t lda, const double* Z,
               int64_t ldz, double* Y, int64_t ldy) {
    StageTimer _t(c, "skinny_nn", M, R, q, 2.0 * double(M) * R * q, 8.0 * (double(M) * R + double(M) * q));
    switch (q) {
        case 1: skinny_nn_t<1>(c, M, R, q, A, lda, Z, ldz, Y, ldy); break;
        case 2: skinny_nn_t<2>(c, M, R, q, A, lda, Z, ldz, Y, ldy); break;
        case 3: case 4: skinny_nn_t<4>(c, M, R, q, A, lda, Z, ldz, Y, ldy); break;
        case 5: case 6: case 7: case 8: skinny_nn_t<8>(c, M, R, q, A, lda, Z, ldz, Y, ldy); break;
        default: skinny_nn_t<16>(c, M, R, q, A, lda, Z, ldz, Y, ldy); break;
    }
}

}  // namespace hydot
