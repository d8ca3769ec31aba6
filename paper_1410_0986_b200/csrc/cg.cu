// cg.cu -- batched matrix-free CG for the forward / adjoint fields
// (SURVEY 8a A4).  Replaces born::compute_fields' per-source calls of
// krylov::solve_family (born.cpp:54-65, krylov.cpp:400-463): every (point,
// wavelength) system (K + sigma_l M + sigma'_l R) x = e_v is SPD, so all of
// them run as one batch of independent CG iterations.
//
// Per iteration two HBM-streaming kernels, each CTA owning 1024 vertices of
// one system (grid.y = system):
//   cg_pa : p <- r + beta p (on the fly for the 6 neighbours), store p,
//           partial p.Ap                                   (reads r,p; writes p)
//   cg_xr : alpha = rr / p.Ap, x += alpha p, r -= alpha A p, partial r.r
//                                                         (reads p,x,r; writes x,r)
// Scalars never leave the device: each CTA sums its system's partials in a
// fixed order (deterministic), CTA 0 publishes rr into a parity slot.  The
// stencil and the vector updates use explicit _rn intrinsics in the oracle's
// operation order (no FMA contraction), so only the dot-product summation
// order differs from the CPU restatement.
#include <cstdlib>

#include "internal.h"

namespace hydot {
namespace {

constexpr int CT = 256;       // threads per CTA
constexpr int VPT = 16;       // vertices per thread (amortises the scalar prologue)
constexpr int CV = CT * VPT;  // vertices per CTA

struct Stencil {
    int nx, ny, nz;
    double h;
    float inv_nx, inv_ny;  // for the division-free vertex decode
};

inline Stencil make_stencil(const hydot_grid7& g) {
    return Stencil{g.nx, g.ny, g.nz, g.h, 1.0f / float(g.nx), 1.0f / float(g.ny)};
}

// q = i / d, r = i % d for i < 2^24 without an integer division: a float
// estimate corrected by one step (64-bit div/mod dominated the CG kernels)
__device__ __forceinline__ void fdivmod(unsigned i, unsigned d, float inv_d, unsigned& q,
                                        unsigned& r) {
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

// y_i = (A x)_i with x(j) supplied by a functor; reference operation order.
// Branch-free: every neighbour is loaded from a clamped in-range index and
// masked by a select, so the compiler can issue all loads of the unrolled
// vertices before their first use (the branchy form stalled on each load).
// The masked terms add +0.0, leaving every sum as in the reference order.
template <class Get>
__device__ __forceinline__ double stencil_at(const Stencil& g, double sigma, double sigmap,
                                             int64_t i, Get get) {
    const int64_t plane = int64_t(g.nx) * g.ny;
    const int64_t N = plane * g.nz;
    unsigned q1, ux, uy, uz;
    fdivmod(unsigned(i), unsigned(g.nx), g.inv_nx, q1, ux);
    fdivmod(q1, unsigned(g.ny), g.inv_ny, uz, uy);
    const int ix = int(ux), iy = int(uy), iz = int(uz);
    const double xi = get(i);
    const bool dir = (ix == 0 || ix == g.nx - 1 || iy == 0 || iy == g.ny - 1);
    const bool bxm = ix - 1 > 0, bxp = ix + 1 < g.nx - 1, bym = iy - 1 > 0, byp = iy + 1 < g.ny - 1;
    const bool bzm = iz > 0, bzp = iz < g.nz - 1;
    const double vxm = get(i > 0 ? i - 1 : i);
    const double vxp = get(i + 1 < N ? i + 1 : i);
    const double vym = get(i >= g.nx ? i - g.nx : i);
    const double vyp = get(i + g.nx < N ? i + g.nx : i);
    const double vzm = get(i >= plane ? i - plane : i);
    const double vzp = get(i + plane < N ? i + plane : i);
    const double h = g.h;
    const bool zb = (iz == 0 || iz == g.nz - 1);
    const double zext = zb ? 0.5 * h : h;
    const double V = __dmul_rn(__dmul_rn(h, h), zext);
    const double S = zb ? __dmul_rn(h, h) : 0.0;
    const double xm = bxm ? vxm : 0.0;
    const double xp = bxp ? vxp : 0.0;
    const double ym = bym ? vym : 0.0;
    const double yp = byp ? vyp : 0.0;
    double wsum = 4.0 * zext;
    double nb = __dmul_rn(zext, xm);
    nb = __dadd_rn(nb, __dmul_rn(zext, xp));
    nb = __dadd_rn(nb, __dmul_rn(zext, ym));
    nb = __dadd_rn(nb, __dmul_rn(zext, yp));
    if (bzm) {
        wsum = __dadd_rn(wsum, h);
        nb = __dadd_rn(nb, __dmul_rn(h, vzm));
    }
    if (bzp) {
        wsum = __dadd_rn(wsum, h);
        nb = __dadd_rn(nb, __dmul_rn(h, vzp));
    }
    const double diag = __dadd_rn(__dadd_rn(wsum, __dmul_rn(sigma, V)), __dmul_rn(sigmap, S));
    const double y = __dsub_rn(__dmul_rn(diag, xi), nb);
    return dir ? xi : y;
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < CT / 32; ++i) t += sh[i];
    __syncthreads();
    return t;
}

// deterministic sum of nparts partials (all threads get the result)
__device__ __forceinline__ double sum_parts(const double* __restrict__ parts, int nparts,
                                            double* sh, double* bc) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nparts; i += CT) v += parts[i];
    double t = block_sum(v, sh);
    if (threadIdx.x == 0) *bc = t;
    __syncthreads();
    return *bc;
}

struct SysState {
    double rr[2];   // r.r published per iteration parity
    double bnorm;   // ||b||
    int done;       // converged (or stopped)
    int iters;
    double relres;
};

__global__ void cg_init(int64_t N, int nl, const int64_t* __restrict__ rhs_vertex, int k0,
                        double* __restrict__ X, double* __restrict__ R, double* __restrict__ P,
                        SysState* __restrict__ st) {
    const int sys = blockIdx.y;
    const int kglob = k0 + sys;
    const int64_t v = rhs_vertex[kglob / nl];
    double* x = X + int64_t(sys) * N;  // x lives in the output (caller column)
    double* r = R + int64_t(sys) * N;
    double* p = P + int64_t(sys) * N;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < N;
         i += int64_t(gridDim.x) * blockDim.x) {
        x[i] = 0.0;
        r[i] = (i == v) ? 1.0 : 0.0;
        p[i] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st[sys].rr[0] = 1.0;
        st[sys].rr[1] = 0.0;
        st[sys].bnorm = 1.0;
        st[sys].done = 0;
        st[sys].iters = 0;
        st[sys].relres = 1.0;
    }
}

__global__ void __launch_bounds__(CT, 4) cg_pa(Stencil g, int64_t N, int nl, int k0, int it,
                                            const double* __restrict__ sig,
                                            const double* __restrict__ sigp,
                                            const double* __restrict__ R,
                                            const double* __restrict__ Pold,
                                            double* __restrict__ Pnew, double* __restrict__ partA,
                                            const double* __restrict__ partB, int nparts,
                                            SysState* __restrict__ st, double tol, int fixed,
                                            const int* __restrict__ act) {
    __shared__ double sh[CT / 32];
    __shared__ double bc;
    const int sys = act[blockIdx.y];  // compacted list of unconverged systems
    SysState& S = st[sys];
    if (S.done) return;
    const int l = (k0 + sys) % nl;
    double beta = 0.0;
    const int slot = it & 1;
    if (it > 0) {
        const double rr_new = sum_parts(partB + int64_t(sys) * nparts, nparts, sh, &bc);
        const double rr_old = S.rr[slot ^ 1];
        const double relres = sqrt(rr_new) / S.bnorm;
        if (!fixed && relres <= tol) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                S.done = 1;
                S.iters = it;
                S.relres = relres;
            }
            return;
        }
        beta = rr_new / rr_old;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            S.rr[slot] = rr_new;
            S.relres = relres;
            S.iters = it;
        }
    }
    const double* r = R + int64_t(sys) * N;
    const double* po = Pold + int64_t(sys) * N;
    double* p = Pnew + int64_t(sys) * N;
    const double sigma = sig[l], sigmap = sigp[l];
    auto pnew = [&](int64_t j) { return __dadd_rn(r[j], __dmul_rn(beta, po[j])); };
    // p is double-buffered across iterations: neighbours in other CTAs
    // still read p_old while this CTA stores p_new.
    double acc = 0.0;
    const int64_t base = int64_t(blockIdx.x) * CV + threadIdx.x;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int64_t i = base + int64_t(k) * CT;
        if (i < N) {
            const double pi = pnew(i);
            const double ap = stencil_at(g, sigma, sigmap, i, pnew);
            p[i] = pi;
            acc += pi * ap;
        }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partA[int64_t(sys) * nparts + blockIdx.x] = t;
}

__global__ void __launch_bounds__(CT, 4) cg_xr(Stencil g, int64_t N, int nl, int k0, int it,
                                            const double* __restrict__ sig,
                                            const double* __restrict__ sigp,
                                            double* __restrict__ X, double* __restrict__ R,
                                            const double* __restrict__ P,
                                            const double* __restrict__ partA,
                                            double* __restrict__ partB, int nparts,
                                            SysState* __restrict__ st,
                                            const int* __restrict__ act) {
    __shared__ double sh[CT / 32];
    __shared__ double bc;
    const int sys = act[blockIdx.y];
    SysState& S = st[sys];
    if (S.done) return;
    const int l = (k0 + sys) % nl;
    const double pq = sum_parts(partA + int64_t(sys) * nparts, nparts, sh, &bc);
    const double alpha = S.rr[it & 1] / pq;
    double* x = X + int64_t(sys) * N;
    double* r = R + int64_t(sys) * N;
    const double* p = P + int64_t(sys) * N;
    const double sigma = sig[l], sigmap = sigp[l];
    auto getp = [&](int64_t j) { return p[j]; };
    double acc = 0.0;
    const int64_t base = int64_t(blockIdx.x) * CV + threadIdx.x;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int64_t i = base + int64_t(k) * CT;
        if (i < N) {
            const double q = stencil_at(g, sigma, sigmap, i, getp);
            x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
            const double rn = __dsub_rn(r[i], __dmul_rn(alpha, q));
            r[i] = rn;
            acc += rn * rn;
        }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partB[int64_t(sys) * nparts + blockIdx.x] = t;
}

// fixed-iteration / max-iteration finish: final relres, scale by inv_D
__global__ void cg_finish(int64_t N, int nl, int k0, int it_total, double* __restrict__ X,
                          const double* __restrict__ invD, const double* __restrict__ partB,
                          int nparts, SysState* __restrict__ st) {
    __shared__ double sh[CT / 32];
    __shared__ double bc;
    const int sys = blockIdx.y;
    SysState& S = st[sys];
    const int l = (k0 + sys) % nl;
    if (!S.done && blockIdx.x == 0) {
        double rr = sum_parts(partB + int64_t(sys) * nparts, nparts, sh, &bc);
        if (threadIdx.x == 0) {
            S.relres = sqrt(rr) / S.bnorm;
            S.iters = it_total;
        }
    }
    const double s = invD[l];
    double* x = X + int64_t(sys) * N;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < N;
         i += int64_t(gridDim.x) * blockDim.x)
        x[i] = x[i] * s;
}

__global__ void apply7_k(Stencil g, int64_t N, double sigma, double sigmap,
                         const double* __restrict__ x, double* __restrict__ y) {
    auto get = [&](int64_t j) { return x[j]; };
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < N;
         i += int64_t(gridDim.x) * blockDim.x)
        y[i] = stencil_at(g, sigma, sigmap, i, get);
}

__global__ void count_active(int n, const SysState* __restrict__ st, int* __restrict__ out) {
    int a = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) a += st[i].done ? 0 : 1;
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    __shared__ int sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
        *out = t;
    }
}

}  // namespace

void apply7(Ctx& c, const hydot_grid7& g, double sigma, double sigmap, const double* x,
            double* y) {
    const int64_t N = int64_t(g.nx) * g.ny * g.nz;
    Stencil s = make_stencil(g);
    int blocks = int(std::min<int64_t>((N + 255) / 256, int64_t(c.num_sms) * 16));
    apply7_k<<<blocks, 256, 0, c.stream>>>(s, N, sigma, sigmap, x, y);
    c.check_launch();
}

void fields_solve(Ctx& c, const hydot_grid7& g, int nl, const double* sigma,
                  const double* sigmap, const double* inv_D, const int64_t* rhs_vertex, int n_rhs,
                  double tol, int max_iter, int fixed_iters, double* out, CGStats* stats) {
    if (g.nx < 3 || g.ny < 3 || g.nz < 2 || g.h <= 0)
        throw std::invalid_argument("fields_solve: bad grid");
    if (nl <= 0 || n_rhs <= 0) throw std::invalid_argument("compute_fields: no wavelengths");
    const int64_t N = int64_t(g.nx) * g.ny * g.nz;
    for (int s = 0; s < n_rhs; ++s) {
        int64_t v = rhs_vertex[s];
        if (v < 0 || v >= N) throw std::invalid_argument("point_source_vector: point outside domain");
        int ix = int(v % g.nx), iy = int((v / g.nx) % g.ny);
        if (ix == 0 || ix == g.nx - 1 || iy == 0 || iy == g.ny - 1)
            throw std::invalid_argument("source support falls entirely on the Dirichlet boundary");
    }
    Stencil st = make_stencil(g);
    if (int64_t(g.nx) * g.ny * g.nz >= (int64_t(1) << 24))
        throw std::invalid_argument("fields_solve: grid too large for the 24-bit vertex decode");
    const int total = n_rhs * nl;
    const int nparts = int((N + CV - 1) / CV);
    // One batch of up to 24 GB (all systems iterate together, HBM-bound).
    // HYDOT_CG_L2_MB > 0 instead iterates L2-sized groups (32 N bytes per
    // system): measured slower on config 1 (1.4-2.8 s vs 0.96 s -- small
    // groups make the iterations launch- and sync-bound), kept for experiments.
    // A z-marching shared-memory stencil (one CTA per x-y tile walking z)
    // also measured slower (1.35 s: one plane of loads in flight per CTA).
    static const int l2_mb = [] {
        const char* e = std::getenv("HYDOT_CG_L2_MB");
        return e ? std::atoi(e) : 0;
    }();
    int64_t per_sys = 2 * N * 8;
    int batch = int(std::max<int64_t>(1, std::min<int64_t>(total, (int64_t(24) << 30) / per_sys)));
    if (l2_mb > 0)
        batch = int(std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t(l2_mb) << 20) / (4 * per_sys))));
    batch = std::min(batch, 65535);
    DBuf dsig = dalloc(c, size_t(nl)), dsigp = dalloc(c, size_t(nl)), dinv = dalloc(c, size_t(nl));
    HYDOT_CUDA(cudaMemcpyAsync(dsig.d(), sigma, size_t(nl) * 8, cudaMemcpyHostToDevice, c.stream));
    HYDOT_CUDA(cudaMemcpyAsync(dsigp.d(), sigmap, size_t(nl) * 8, cudaMemcpyHostToDevice, c.stream));
    HYDOT_CUDA(cudaMemcpyAsync(dinv.d(), inv_D, size_t(nl) * 8, cudaMemcpyHostToDevice, c.stream));
    DBuf drhs(c, size_t(n_rhs) * 8);
    HYDOT_CUDA(cudaMemcpyAsync(drhs.as<void>(), rhs_vertex, size_t(n_rhs) * 8,
                               cudaMemcpyHostToDevice, c.stream));
    DBuf R = dalloc(c, size_t(batch) * size_t(N));
    DBuf P = dalloc(c, 2 * size_t(batch) * size_t(N));  // double-buffered p
    DBuf pA = dalloc(c, size_t(batch) * size_t(nparts));
    DBuf pB = dalloc(c, size_t(batch) * size_t(nparts));
    DBuf S(c, size_t(batch) * sizeof(SysState));
    DBuf dact(c, sizeof(int) * size_t(batch));
    if (stats) {
        stats->iters.assign(size_t(total), 0);
        stats->relres.assign(size_t(total), 0.0);
    }
    const int limit = fixed_iters > 0 ? fixed_iters : max_iter;
    for (int k0 = 0; k0 < total; k0 += batch) {
        const int nb = std::min(batch, total - k0);
        double* X = out + int64_t(k0) * N;
        SysState* ss = S.as<SysState>();
        {
            dim3 gi = dim3(unsigned(std::min<int64_t>((N + 255) / 256, 1024)), unsigned(nb));
            // p_old of iteration 0 is buffer 1 (zeroed); p_it lives in buffer it&1
            cg_init<<<gi, 256, 0, c.stream>>>(N, nl, drhs.as<int64_t>(), k0, X, R.d(),
                                              P.d() + size_t(batch) * size_t(N), ss);
            c.check_launch();
        }
        auto pbuf = [&](int i) { return P.d() + size_t(i & 1) * size_t(batch) * size_t(N); };
        // active-system list: converged systems are dropped from the grid
        // every 8 iterations (systems converge between ~70 and ~135 iterations)
        std::vector<int> active(static_cast<size_t>(nb));
        for (int k = 0; k < nb; ++k) active[size_t(k)] = k;
        std::vector<SysState> hst(static_cast<size_t>(nb));
        HYDOT_CUDA(cudaMemcpyAsync(dact.as<void>(), active.data(), active.size() * sizeof(int),
                                   cudaMemcpyHostToDevice, c.stream));
        int it = 0;
        for (; it < limit; ++it) {
            dim3 grid = dim3(unsigned(nparts), unsigned(active.size()));
            cg_pa<<<grid, CT, 0, c.stream>>>(st, N, nl, k0, it, dsig.d(), dsigp.d(), R.d(),
                                            pbuf(it + 1), pbuf(it), pA.d(), pB.d(), nparts, ss,
                                            tol, fixed_iters > 0, dact.as<int>());
            c.check_launch();
            cg_xr<<<grid, CT, 0, c.stream>>>(st, N, nl, k0, it, dsig.d(), dsigp.d(), X, R.d(),
                                            pbuf(it), pA.d(), pB.d(), nparts, ss, dact.as<int>());
            c.check_launch();
            if (fixed_iters <= 0 && (it % 8) == 7) {
                HYDOT_CUDA(cudaMemcpyAsync(hst.data(), ss, size_t(nb) * sizeof(SysState),
                                           cudaMemcpyDeviceToHost, c.stream));
                c.sync();
                std::vector<int> still;
                for (int k : active)
                    if (!hst[size_t(k)].done) still.push_back(k);
                if (still.empty()) {
                    ++it;
                    break;
                }
                if (still.size() < active.size()) {
                    active.swap(still);
                    HYDOT_CUDA(cudaMemcpyAsync(dact.as<void>(), active.data(),
                                               active.size() * sizeof(int), cudaMemcpyHostToDevice,
                                               c.stream));
                    c.sync();  // host vector is reused
                }
            }
        }
        if (fixed_iters <= 0 && it >= limit) {
            // one more convergence check for systems finishing on the last step
            dim3 grid = dim3(unsigned(nparts), unsigned(active.size()));
            cg_pa<<<grid, CT, 0, c.stream>>>(st, N, nl, k0, it, dsig.d(), dsigp.d(), R.d(),
                                            pbuf(it + 1), pbuf(it), pA.d(), pB.d(), nparts, ss,
                                            tol, 0, dact.as<int>());
            c.check_launch();
        }
        {
            dim3 gf = dim3(unsigned(std::min<int64_t>((N + 255) / 256, 1024)), unsigned(nb));
            cg_finish<<<gf, CT, 0, c.stream>>>(N, nl, k0, it, X, dinv.d(), pB.d(), nparts, ss);
            c.check_launch();
        }
        if (stats) {
            std::vector<SysState> hs(static_cast<size_t>(nb));
            HYDOT_CUDA(cudaMemcpyAsync(hs.data(), ss, size_t(nb) * sizeof(SysState),
                                       cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            for (int k = 0; k < nb; ++k) {
                stats->iters[size_t(k0 + k)] = hs[size_t(k)].iters;
                stats->relres[size_t(k0 + k)] = hs[size_t(k)].relres;
            }
        }
    }
    c.sync();
}

}  // namespace hydot
