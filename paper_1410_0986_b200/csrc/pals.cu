// pals.cu -- voxel- and measurement-parallel kernels of the PaLS loop
// (proj/src/pals.cpp).  The level set, the smoothed shape
// and the analytic shape Jacobian are evaluated one vertex per thread with
// the RBF parameters staged in shared memory; the arithmetic follows the
// reference expressions operation by operation with explicitly rounded
// intrinsics (no FMA contraction), so only sin/cos may differ from glibc
// (<= 1-2 ulp).  The Jacobian (N x 5 n_p, column-major, coalesced per
// column) is HBM-write bound: 8 * 5 n_p B per vertex.
#include "pals.h"

namespace hydot {
namespace pals {
namespace {

constexpr double kPi = 3.14159265358979323846;  // M_PI

struct GD {
    int nx, ny, nz;
    double Lx, Ly, hx, hy, hz;
};
struct PD {
    int np;
    const double* v;  // [alpha | beta | cx | cy | cz], n_p each
    double tau, epsH, nu;
};

__device__ __forceinline__ double wend(double t) {  // pals.cpp:38-43
    if (t >= 1.0) return 0.0;
    const double s = __dsub_rn(1.0, t);
    const double s2 = __dmul_rn(s, s);
    return __dmul_rn(__dmul_rn(s2, s2), __dadd_rn(__dmul_rn(4.0, t), 1.0));
}
__device__ __forceinline__ double wend_d(double t) {  // pals.cpp:45-49
    if (t >= 1.0) return 0.0;
    const double s = __dsub_rn(1.0, t);
    return __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(-20.0, t), s), s), s);
}
__device__ __forceinline__ double heav(double t, double eps) {  // pals.cpp:51-55
    if (t < -eps) return 0.0;
    if (t > eps) return 1.0;
    const double a = __dadd_rn(1.0, __ddiv_rn(t, eps));
    const double arg = __ddiv_rn(__dmul_rn(kPi, t), eps);
    return __dmul_rn(0.5, __dadd_rn(a, __ddiv_rn(sin(arg), kPi)));
}
__device__ __forceinline__ double dlt(double t, double eps) {  // pals.cpp:57-60
    if (t < -eps || t > eps) return 0.0;
    const double arg = __ddiv_rn(__dmul_rn(kPi, t), eps);
    return __dmul_rn(__ddiv_rn(0.5, eps), __dadd_rn(1.0, cos(arg)));
}
// ||r - chi_k||_* (pals.cpp:64-70)
__device__ __forceinline__ double star(const double r[3], double cx, double cy, double cz, double nu) {
    const double dx = __dsub_rn(r[0], cx), dy = __dsub_rn(r[1], cy), dz = __dsub_rn(r[2], cz);
    double s = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    s = __dadd_rn(s, __dmul_rn(dz, dz));
    s = __dadd_rn(s, __dmul_rn(nu, nu));
    return __dsqrt_rn(s);
}

template <int WHICH>
__global__ void __launch_bounds__(256) pals_eval_k(int64_t N, GD g, PD p, double* __restrict__ out,
                                                   int64_t ldo) {
    extern __shared__ double sp[];
    const int np = p.np;
    for (int e = threadIdx.x; e < 5 * np; e += blockDim.x) sp[e] = p.v[e];
    __syncthreads();
    const double *al = sp, *be = sp + np, *cx = sp + 2 * np, *cy = sp + 3 * np, *cz = sp + 4 * np;
    for (int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; n < N;
         n += int64_t(gridDim.x) * blockDim.x) {
        const int ix = int(n % g.nx);
        const int iy = int((n / g.nx) % g.ny);
        const int iz = int(n / (int64_t(g.nx) * g.ny));
        double r[3];  // grid.hpp:37-40
        r[0] = __dadd_rn(-g.Lx, __dmul_rn(double(ix), g.hx));
        r[1] = __dadd_rn(-g.Ly, __dmul_rn(double(iy), g.hy));
        r[2] = __dmul_rn(double(iz), g.hz);
        double phi = 0.0;  // level_set (pals.cpp:79-83)
        for (int k = 0; k < np; ++k)
            phi = __dadd_rn(phi, __dmul_rn(al[k], wend(__dmul_rn(be[k], star(r, cx[k], cy[k], cz[k], p.nu)))));
        if (WHICH == EVAL_LEVEL_SET) {
            out[n] = phi;
        } else if (WHICH == EVAL_SHAPE) {
            out[n] = heav(__dsub_rn(phi, p.tau), p.epsH);
        } else {  // shape_jacobian (pals.cpp:101-116)
            const double d = dlt(__dsub_rn(phi, p.tau), p.epsH);
            for (int k = 0; k < np; ++k) {
                double j0 = 0.0, j1 = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
                if (d != 0.0) {
                    const double nr = star(r, cx[k], cy[k], cz[k], p.nu);
                    const double t = __dmul_rn(be[k], nr);
                    const double psi = wend(t), dpsi = wend_d(t);
                    j0 = __dmul_rn(d, psi);
                    j1 = __dmul_rn(__dmul_rn(__dmul_rn(d, al[k]), dpsi), nr);
                    const double fac =
                        __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(-d, al[k]), be[k]), dpsi), nr);
                    jx = __dmul_rn(fac, __dsub_rn(r[0], cx[k]));
                    jy = __dmul_rn(fac, __dsub_rn(r[1], cy[k]));
                    jz = __dmul_rn(fac, __dsub_rn(r[2], cz[k]));
                }
                out[n + int64_t(k) * ldo] = j0;
                out[n + int64_t(np + k) * ldo] = j1;
                out[n + int64_t(2 * np + k) * ldo] = jx;
                out[n + int64_t(3 * np + k) * ldo] = jy;
                out[n + int64_t(4 * np + k) * ldo] = jz;
            }
        }
    }
}

__global__ void pals_residual_k(int64_t M, int nl, int nsp, const double* __restrict__ ext,
                                const double* __restrict__ cv, const double* __restrict__ y,
                                const double* __restrict__ w, const double* __restrict__ hmu,
                                double* __restrict__ eps) {
    for (int64_t m = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; m < M;
         m += int64_t(gridDim.x) * blockDim.x) {
        const int l = int(m % nl);
        const double h = hmu[m];
        double dc = 0.0;  // (D c)_m, D(m, i) = e_i[l] * hmu[m] (pals.cpp:132, 187)
        for (int i = 0; i < nsp; ++i) dc = __dadd_rn(dc, __dmul_rn(__dmul_rn(ext[l + int64_t(i) * nl], h), cv[i]));
        eps[m] = __dmul_rn(w[m], __dsub_rn(y[m], dc));
    }
}

__global__ void pals_jscale_k(int64_t M, int ncols, int nl, const double* __restrict__ w,
                              const double* __restrict__ ebar, const double* __restrict__ HJ,
                              int64_t ldh, double* __restrict__ J, int64_t ldj) {
    const int64_t total = M * ncols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t m = e % M, j = e / M;
        J[m + j * ldj] = __dmul_rn(__dmul_rn(-w[m], ebar[m % nl]), HJ[m + j * ldh]);
    }
}

constexpr int RB = 256;     // threads per reduction block
constexpr int RGRID = 512;  // fixed partial count: deterministic order

template <int K, class F>
__device__ __forceinline__ void block_sums(F f, int64_t n, double* __restrict__ part) {
    __shared__ double sh[K][RB / 32];
    double acc[K];
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] = 0.0;
    for (int64_t i = blockIdx.x * int64_t(RB) + threadIdx.x; i < n; i += int64_t(gridDim.x) * RB) f(i, acc);
#pragma unroll
    for (int q = 0; q < K; ++q)
        for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int q = 0; q < K; ++q) sh[q][threadIdx.x >> 5] = acc[q];
    __syncthreads();
    if (threadIdx.x < K) {
        double s = 0.0;
        for (int w = 0; w < RB / 32; ++w) s += sh[threadIdx.x][w];
        part[int64_t(threadIdx.x) * gridDim.x + blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(RB) sumsq_k(int64_t n, const double* __restrict__ x, double* part) {
    block_sums<1>([&](int64_t i, double* a) { a[0] += x[i] * x[i]; }, n, part);
}

__global__ void __launch_bounds__(RB) metric_k(int64_t n, const double* __restrict__ a,
                                               const double* __restrict__ b, double thr, double* part) {
    block_sums<6>(
        [&](int64_t i, double* s) {
            const double x = a[i], y = b[i], d = x - y;
            s[0] += d * d;
            s[1] += x * x;
            s[2] += y * y;
            const bool ta = x > thr, tb = y > thr;
            s[3] += ta ? 1.0 : 0.0;
            s[4] += tb ? 1.0 : 0.0;
            s[5] += (ta && tb) ? 1.0 : 0.0;
        },
        n, part);
}

// K partial rows of `parts` partials -> out[K] (one warp per quantity, fixed order)
__global__ void finish_sums_k(int K, int parts, const double* __restrict__ part, double* __restrict__ out) {
    const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (q >= K) return;
    double s = 0.0;
    for (int i = lane; i < parts; i += 32) s += part[int64_t(q) * parts + i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[q] = s;
}

__global__ void stack_damped_k(int64_t M, int n, const double* __restrict__ J, int64_t ldj,
                               const double* __restrict__ eps, double snu, double* __restrict__ A,
                               double* __restrict__ rhs) {
    const int64_t rows = M + n, total = rows * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e % rows, j = e / rows;
        A[e] = i < M ? J[i + j * ldj] : ((i - M) == j ? snu : 0.0);
        if (j == 0) rhs[i] = i < M ? -eps[i] : 0.0;
    }
}

int grid_for(Ctx& c, int64_t n) {
    return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(c.num_sms) * 8)));
}

template <int K>
void reduce(Ctx& c, DBuf& part, double* out_h) {
    DBuf res = dalloc(c, K);
    finish_sums_k<<<1, 32 * K, 0, c.stream>>>(K, RGRID, part.d(), res.d());
    c.check_launch();
    c.d2h(out_h, res.d(), K);
}

}  // namespace

Geom Geom::make(const hydot_grid_geom& g) {  // build_grid (grid.cpp:94-110)
    if (g.nx < 2 || g.ny < 2 || g.nz < 2) throw std::invalid_argument("build_grid: vertex counts must be >= 2");
    if (g.Lx <= 0 || g.Ly <= 0 || g.Lz <= 0) throw std::invalid_argument("build_grid: extents must be positive");
    Geom o;
    o.nx = g.nx;
    o.ny = g.ny;
    o.nz = g.nz;
    o.Lx = g.Lx;
    o.Ly = g.Ly;
    o.Lz = g.Lz;
    o.hx = 2 * g.Lx / (g.nx - 1);
    o.hy = 2 * g.Ly / (g.ny - 1);
    o.hz = g.Lz / (g.nz - 1);
    return o;
}

void eval(Ctx& c, int which, const Geom& g, const Params& p, double* out, int64_t ldo) {
    StageTimer _t(c, which == EVAL_JACOBIAN ? "pals_jacobian" : "pals_shape", g.N(), p.np(), -1, 0.0,
                  8.0 * double(g.N()) * (which == EVAL_JACOBIAN ? 5 * p.np() : 1));
    const int np = p.np();
    if (np < 0 || int64_t(p.beta.size()) != np || int64_t(p.centers.size()) != 3 * int64_t(np))
        throw std::invalid_argument("PaLS: parameter array lengths");
    std::vector<double> v = p.to_vector();
    DBuf pv = dalloc(c, size_t(std::max(1, 5 * np)));
    if (np > 0)
        HYDOT_CUDA(cudaMemcpyAsync(pv.d(), v.data(), v.size() * 8, cudaMemcpyHostToDevice, c.stream));
    GD gd{g.nx, g.ny, g.nz, g.Lx, g.Ly, g.hx, g.hy, g.hz};
    PD pd{np, pv.d(), p.tau_level, p.eps_H, p.nu_norm};
    const int64_t N = g.N();
    const size_t smem = size_t(std::max(1, 5 * np)) * 8;
    if (smem > 48 * 1024) throw std::invalid_argument("PaLS: too many basis functions");
    const int blocks = grid_for(c, N);
    if (which == EVAL_LEVEL_SET) pals_eval_k<EVAL_LEVEL_SET><<<blocks, 256, smem, c.stream>>>(N, gd, pd, out, ldo);
    else if (which == EVAL_SHAPE) pals_eval_k<EVAL_SHAPE><<<blocks, 256, smem, c.stream>>>(N, gd, pd, out, ldo);
    else pals_eval_k<EVAL_JACOBIAN><<<blocks, 256, smem, c.stream>>>(N, gd, pd, out, ldo);
    c.check_launch();
}

void residual(Ctx& c, int64_t M, int nl, int nsp, const double* ext_dev, const double* c_dev,
              const double* y, const double* w, const double* hmu, double* eps) {
    pals_residual_k<<<grid_for(c, M), 256, 0, c.stream>>>(M, nl, nsp, ext_dev, c_dev, y, w, hmu, eps);
    c.check_launch();
}

void jscale(Ctx& c, int64_t M, int ncols, int nl, const double* w, const double* ebar_dev,
            const double* HJ, int64_t ldh, double* J, int64_t ldj) {
    pals_jscale_k<<<grid_for(c, M * ncols), 256, 0, c.stream>>>(M, ncols, nl, w, ebar_dev, HJ, ldh, J, ldj);
    c.check_launch();
}

double norm2(Ctx& c, int64_t n, const double* x) {
    DBuf part = dalloc(c, RGRID);
    sumsq_k<<<RGRID, RB, 0, c.stream>>>(n, x, part.d());
    c.check_launch();
    double s = 0.0;
    reduce<1>(c, part, &s);
    return std::sqrt(s);
}

void stack_damped(Ctx& c, int64_t M, int n, const double* J, int64_t ldj, const double* eps, double nu,
                  double* A, double* rhs) {
    stack_damped_k<<<grid_for(c, (M + n) * n), 256, 0, c.stream>>>(M, n, J, ldj, eps, std::sqrt(nu), A, rhs);
    c.check_launch();
}

void metric_sums(Ctx& c, int64_t N, const double* a, const double* b, double thr, double out[6]) {
    DBuf part = dalloc(c, size_t(6) * RGRID);
    metric_k<<<RGRID, RB, 0, c.stream>>>(N, a, b, thr, part.d());
    c.check_launch();
    reduce<6>(c, part, out);
}

}  // namespace pals
}  // namespace hydot
