// svd.cu -- one-sided (Hestenes) Jacobi thin SVD on the GPU, replacing
// Eigen::BDCSVD on the small cores of the path (lowrank.cpp:43-49, 79, 88,
// 568): the R factors of Y, B^T, W^T and the recompress core.
//
// Columns of X (m x n, m >= n) are orthogonalised by plane rotations in
// round-robin (circle-method) order; each rotation is computed from the
// actual column dot products, so small singular values keep high relative
// accuracy (no Gram matrix is formed).  Two drivers:
//   * small  (m + n) n doubles fit in shared memory: one CTA runs every sweep
//     on-chip, one warp per column pair;
//   * large: one launch per round, one CTA per pair, convergence flag read
//     once per sweep.
// Afterwards sigma_j = ||u_j||, U = u_j / sigma_j, sorted descending.
#include <algorithm>
#include <numeric>

#include "internal.h"

namespace hydot {
namespace {

constexpr double kTol = 1.0e-15;
constexpr int kMaxSweeps = 60;

__device__ __forceinline__ void rot_params(double a, double b, double g, double& cs, double& sn) {
    double zeta = (b - a) / (2.0 * g);
    double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    cs = 1.0 / sqrt(1.0 + t * t);
    sn = cs * t;
}

// ---------------------------------------------------------- single CTA ----
__global__ void __launch_bounds__(1024) jacobi_smem_k(int m, int n, int np,
                                                      const int2* __restrict__ pairs,
                                                      double* __restrict__ Ug, int64_t ldu,
                                                      double* __restrict__ Vg, int64_t ldv,
                                                      int* __restrict__ sweeps_out) {
    extern __shared__ double sm[];
    double* U = sm;               // m x n, ld m
    double* V = sm + int64_t(m) * n;  // n x n, ld n
    __shared__ int changed;
    for (int64_t e = threadIdx.x; e < int64_t(m) * n; e += blockDim.x) {
        int64_t i = e % m, j = e / m;
        U[e] = Ug[i + j * ldu];
    }
    for (int64_t e = threadIdx.x; e < int64_t(n) * n; e += blockDim.x) {
        int64_t i = e % n, j = e / n;
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
                double* up = U + int64_t(pr.x) * m;
                double* uq = U + int64_t(pr.y) * m;
                double a = 0, b = 0, g = 0;
                for (int i = lane; i < m; i += 32) {
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
                if (g != 0.0 && fabs(g) > kTol * sqrt(a * b)) {
                    double cs, sn;
                    rot_params(a, b, g, cs, sn);
                    for (int i = lane; i < m; i += 32) {
                        double x = up[i], y = uq[i];
                        up[i] = cs * x - sn * y;
                        uq[i] = sn * x + cs * y;
                    }
                    double* vp = V + int64_t(pr.x) * n;
                    double* vq = V + int64_t(pr.y) * n;
                    for (int i = lane; i < n; i += 32) {
                        double x = vp[i], y = vq[i];
                        vp[i] = cs * x - sn * y;
                        vq[i] = sn * x + cs * y;
                    }
                    if (lane == 0) changed = 1;
                }
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
    for (int64_t e = threadIdx.x; e < int64_t(n) * n; e += blockDim.x) {
        int64_t i = e % n, j = e / n;
        Vg[i + j * ldv] = V[e];
    }
    if (threadIdx.x == 0 && sweeps_out) *sweeps_out = sweep;
}

// ------------------------------------------------------------ multi CTA ----
__global__ void __launch_bounds__(256) jacobi_round_k(int64_t m, int n, const int2* __restrict__ pairs,
                                                      double* __restrict__ U, int64_t ldu,
                                                      double* __restrict__ V, int64_t ldv,
                                                      int* __restrict__ changed) {
    __shared__ double sh[3][8];
    __shared__ double s_cs, s_sn;
    __shared__ int s_rot;
    int2 pr = pairs[blockIdx.x];
    if (pr.x >= n || pr.y >= n) return;
    double* up = U + int64_t(pr.x) * ldu;
    double* uq = U + int64_t(pr.y) * ldu;
    double a = 0, b = 0, g = 0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        double x = up[i], y = uq[i];
        a += x * x;
        b += y * y;
        g += x * y;
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        g += __shfl_down_sync(0xffffffffu, g, o);
    }
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        sh[0][w] = a;
        sh[1][w] = b;
        sh[2][w] = g;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double A = 0, B = 0, G = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) {
            A += sh[0][i];
            B += sh[1][i];
            G += sh[2][i];
        }
        s_rot = (G != 0.0 && fabs(G) > kTol * sqrt(A * B)) ? 1 : 0;
        if (s_rot) {
            double cs, sn;
            rot_params(A, B, G, cs, sn);
            s_cs = cs;
            s_sn = sn;
            *changed = 1;
        }
    }
    __syncthreads();
    if (!s_rot) return;
    const double cs = s_cs, sn = s_sn;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        double x = up[i], y = uq[i];
        up[i] = cs * x - sn * y;
        uq[i] = sn * x + cs * y;
    }
    double* vp = V + int64_t(pr.x) * ldv;
    double* vq = V + int64_t(pr.y) * ldv;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double x = vp[i], y = vq[i];
        vp[i] = cs * x - sn * y;
        vq[i] = sn * x + cs * y;
    }
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
        // rotate p[1..np-1]
        int last = p[size_t(np - 1)];
        for (int i = np - 1; i > 1; --i) p[size_t(i)] = p[size_t(i - 1)];
        p[1] = last;
    }
    return out;
}

}  // namespace

void jacobi_svd(Ctx& c, int64_t m, int64_t n, const double* X, int64_t ldx, double* Uo,
                int64_t lduo, std::vector<double>& s, double* Vo, int64_t ldvo) {
    StageTimer _t(c, n > 96 ? "svd_jacobi_large" : "svd_jacobi_small");
    s.assign(size_t(std::max<int64_t>(n, 0)), 0.0);
    if (n <= 0) return;
    if (m < n) throw std::invalid_argument("jacobi_svd: needs m >= n");
    int np = 0;
    std::vector<int2> pairs = tournament(int(n), np);
    DBuf dpairs(c, std::max<size_t>(pairs.size(), 1) * sizeof(int2));
    if (!pairs.empty())
        HYDOT_CUDA(cudaMemcpyAsync(dpairs.as<void>(), pairs.data(), pairs.size() * sizeof(int2),
                                   cudaMemcpyHostToDevice, c.stream));
    DBuf U = dalloc(c, size_t(m * n));
    DBuf V = dalloc(c, size_t(n * n));
    copy2d(c, m, n, X, ldx, U.d(), m);
    const size_t smem = size_t((m + n) * n) * sizeof(double);
    if (n >= 2 && smem <= 200 * 1024) {
        static bool attr = false;
        if (!attr) {
            HYDOT_CUDA(cudaFuncSetAttribute(jacobi_smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            210 * 1024));
            attr = true;
        }
        jacobi_smem_k<<<1, 1024, smem, c.stream>>>(int(m), int(n), np, dpairs.as<int2>(), U.d(), m,
                                                    V.d(), n, nullptr);
        c.check_launch();
    } else {
        set_identity(c, n, n, V.d(), n);
        if (n >= 2) {
            DBuf flag(c, sizeof(int));
            const int per = np / 2;
            for (int sw = 0; sw < kMaxSweeps; ++sw) {
                HYDOT_CUDA(cudaMemsetAsync(flag.as<void>(), 0, sizeof(int), c.stream));
                for (int r = 0; r < np - 1; ++r) {
                    jacobi_round_k<<<per, 256, 0, c.stream>>>(m, int(n), dpairs.as<int2>() + r * per,
                                                             U.d(), m, V.d(), n, flag.as<int>());
                    c.check_launch();
                }
                int h = 0;
                HYDOT_CUDA(cudaMemcpyAsync(&h, flag.as<void>(), sizeof(int), cudaMemcpyDeviceToHost,
                                           c.stream));
                c.sync();
                if (!h) break;
            }
        }
    }
    DBuf sd = dalloc(c, size_t(n));
    colnorm_k<<<unsigned(n), 256, 0, c.stream>>>(m, int(n), U.d(), m, sd.d());
    c.check_launch();
    std::vector<double> sv(static_cast<size_t>(n));
    c.d2h(sv.data(), sd.d(), size_t(n));
    std::vector<int> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return sv[size_t(a)] > sv[size_t(b)]; });
    for (int64_t j = 0; j < n; ++j) s[size_t(j)] = sv[size_t(perm[size_t(j)])];
    DBuf dperm(c, size_t(n) * sizeof(int));
    HYDOT_CUDA(cudaMemcpyAsync(dperm.as<void>(), perm.data(), size_t(n) * sizeof(int),
                               cudaMemcpyHostToDevice, c.stream));
    int gx = int(std::min<int64_t>((std::max(m, n) + 255) / 256, 64));
    finish_k<<<dim3(unsigned(gx), unsigned(n)), 256, 0, c.stream>>>(
        m, int(n), dperm.as<int>(), sd.d(), U.d(), m, Uo, lduo, V.d(), n, Vo, ldvo);
    c.check_launch();
    c.sync();  // host vectors (pairs, perm) go out of scope
}

}  // namespace hydot
