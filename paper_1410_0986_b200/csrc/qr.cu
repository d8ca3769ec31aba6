// qr.cu -- blocked Householder QR on the GPU (LAPACK dgeqrf / dlarft /
// dlarfb semantics), replacing Eigen::HouseholderQR in fast_thin_svd
// (lowrank.cpp:73-87) and recompress (lowrank.cpp:564-566, 579-580).
//
// The scheduled leaf tolerance reaches 8e-11, below sqrt(eps),
// so Gram/Cholesky QR is not admissible: this is true Householder.
// Right-looking, panel width 32:
//   panel   column-by-column reflectors over all rows; each column takes two
//           grid-wide passes (reflector + dot products, then rank-1 update
//           fused with the next column's norm); reductions are per-CTA
//           partials summed in fixed order by every CTA (deterministic).
//   T       block-reflector triangle from G = V^T V (DMMA GEMM) and tau.
//   update  C -= V (T^T (V^T C)): three DMMA GEMMs (the first is split-K over
//           the long row dimension).
#include "internal.h"

namespace hydot {
namespace {

constexpr int NB = kQRPanel;  // 32
constexpr int PT = 256;       // threads per panel CTA

struct PanelScalars {
    double tau, beta, scal;
};

inline int panel_ctas(Ctx& c, int64_t rows) {
    int64_t p = (rows + 1023) / 1024;
    return int(std::max<int64_t>(1, std::min<int64_t>(p, int64_t(c.num_sms) * 2)));
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
    return t;  // valid in thread 0
}

// partial sum of squares of column c, rows [c+1, mr)
__global__ void __launch_bounds__(PT) pf_norm(int64_t mr, int c, const double* __restrict__ P,
                                              int64_t ld, int64_t rows_per,
                                              double* __restrict__ part) {
    __shared__ double sh[32];
    int64_t r0 = int64_t(blockIdx.x) * rows_per, r1 = min(mr, r0 + rows_per);
    double acc = 0.0;
    for (int64_t i = max(r0, int64_t(c) + 1) + threadIdx.x; i < r1; i += blockDim.x) {
        double x = P[i + int64_t(c) * ld];
        acc += x * x;
    }
    double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// dlarfg on column c (every CTA recomputes it from the partials), scale v in
// this CTA's rows, partial dots w_cc = v^T P[:, cc] for cc in (c, jb).
__global__ void __launch_bounds__(PT) pf_reflect(int64_t mr, int jb, int c, double* __restrict__ P,
                                                 int64_t ld, int64_t rows_per, int nparts,
                                                 const double* __restrict__ part,
                                                 double* __restrict__ part2,
                                                 PanelScalars* __restrict__ sc) {
    __shared__ double sh[32];
    __shared__ double s_scal, s_tau;
    if (threadIdx.x == 0) {
        double xn2 = 0.0;
        for (int p = 0; p < nparts; ++p) xn2 += part[p];
        double alpha = P[c + int64_t(c) * ld];
        double tau = 0.0, beta = alpha, scal = 1.0;
        if (xn2 > 0.0) {
            double xnorm = sqrt(xn2);
            beta = -copysign(hypot(alpha, xnorm), alpha);
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        s_scal = scal;
        s_tau = tau;
        if (blockIdx.x == 0) {
            sc->tau = tau;
            sc->beta = beta;
            sc->scal = scal;
        }
    }
    __syncthreads();
    const double scal = s_scal;
    const bool active = s_tau != 0.0;
    int64_t r0 = int64_t(blockIdx.x) * rows_per, r1 = min(mr, r0 + rows_per);
    double acc[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) acc[q] = 0.0;
    for (int64_t i = max(r0, int64_t(c)) + threadIdx.x; i < r1; i += blockDim.x) {
        double v;
        if (i == c) {
            v = 1.0;
        } else {
            v = P[i + int64_t(c) * ld];
            if (active) {
                v *= scal;
                P[i + int64_t(c) * ld] = v;
            }
        }
#pragma unroll
        for (int q = 0; q < NB; ++q)
            if (q > c && q < jb) acc[q] += v * P[i + int64_t(q) * ld];
    }
    for (int q = c + 1; q < jb; ++q) {
        double t = block_sum(acc[q], sh);
        if (threadIdx.x == 0) part2[int64_t(blockIdx.x) * NB + q] = t;
    }
}

// P[:, cc] -= tau v w_cc for cc in (c, jb); diagonal <- beta; partial norm of
// the next column below its diagonal.
__global__ void __launch_bounds__(PT) pf_update(int64_t mr, int jb, int c, double* __restrict__ P,
                                                int64_t ld, int64_t rows_per, int nparts,
                                                const double* __restrict__ part2,
                                                const PanelScalars* __restrict__ sc,
                                                double* __restrict__ part) {
    __shared__ double sh[32];
    __shared__ double w[NB];
    const double tau = sc->tau;
    if (threadIdx.x < NB) {
        int q = threadIdx.x;
        double s = 0.0;
        if (q > c && q < jb)
            for (int p = 0; p < nparts; ++p) s += part2[int64_t(p) * NB + q];
        w[q] = s;
    }
    __syncthreads();
    int64_t r0 = int64_t(blockIdx.x) * rows_per, r1 = min(mr, r0 + rows_per);
    double nacc = 0.0;
    for (int64_t i = max(r0, int64_t(c)) + threadIdx.x; i < r1; i += blockDim.x) {
        double v = (i == c) ? 1.0 : P[i + int64_t(c) * ld];
        if (tau != 0.0) {
            for (int q = c + 1; q < jb; ++q) P[i + int64_t(q) * ld] -= tau * v * w[q];
        }
        if (i == c) P[i + int64_t(c) * ld] = sc->beta;
        if (c + 1 < jb && i >= c + 2) {
            double x = P[i + int64_t(c + 1) * ld];
            nacc += x * x;
        }
    }
    double t = block_sum(nacc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void store_tau(const PanelScalars* sc, double* tau) { *tau = sc->tau; }

// Vp (mr x jb): unit lower trapezoid of the factored panel
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

// dlarft (forward, columnwise): T upper triangular jb x jb (ld NB)
__global__ void larft_k(int jb, const double* __restrict__ G, const double* __restrict__ tau,
                        double* __restrict__ T) {
    __shared__ double Ts[NB][NB + 1];
    __shared__ double wv[NB];
    int r = threadIdx.x;
    for (int i = 0; i < jb; ++i) {
        // w = -tau_i G[0:i, i]; T[0:i, i] = T[0:i,0:i] w
        if (r < i) wv[r] = -tau[i] * G[r + i * jb];
        __syncthreads();
        if (r < i) {
            double s = 0.0;
            for (int q = r; q < i; ++q) s += Ts[r][q] * wv[q];
            Ts[r][i] = s;
        }
        if (r == i) Ts[i][i] = tau[i];
        if (r > i && r < NB) Ts[r][i] = 0.0;
        __syncthreads();
    }
    for (int i = 0; i < jb; ++i)
        if (r < NB) T[r + i * NB] = r < jb ? Ts[r][i] : 0.0;
}

}  // namespace

void geqrf(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, QRFact& f) {
    StageTimer _t(c, "qr_geqrf");
    f.m = m;
    f.n = n;
    f.a = dalloc(c, size_t(std::max<int64_t>(m * n, 1)));
    f.tau = dalloc(c, size_t(std::max<int64_t>(n, 1)));
    f.T = dalloc(c, size_t(NB) * size_t(std::max<int64_t>(n, 1)));
    copy2d(c, m, n, A, lda, f.a.d(), m);
    const int64_t k = std::min(m, n);
    if (k <= 0) return;
    double* a = f.a.d();
    int maxp = panel_ctas(c, m);
    DBuf part = dalloc(c, size_t(maxp));
    DBuf part2 = dalloc(c, size_t(maxp) * NB);
    DBuf scal(c, sizeof(PanelScalars));
    DBuf V = dalloc(c, size_t(m) * NB);
    DBuf G = dalloc(c, size_t(NB) * NB);
    DBuf W = dalloc(c, size_t(NB) * size_t(std::max<int64_t>(n, 1)));
    DBuf W2 = dalloc(c, size_t(NB) * size_t(std::max<int64_t>(n, 1)));
    for (int64_t j0 = 0; j0 < k; j0 += NB) {
        const int jb = int(std::min<int64_t>(NB, k - j0));
        const int64_t mr = m - j0;
        double* P = a + j0 + j0 * m;
        const int np = panel_ctas(c, mr);
        const int64_t rows_per = (mr + np - 1) / np;
        pf_norm<<<np, PT, 0, c.stream>>>(mr, 0, P, m, rows_per, part.d());
        c.check_launch();
        for (int cc = 0; cc < jb; ++cc) {
            pf_reflect<<<np, PT, 0, c.stream>>>(mr, jb, cc, P, m, rows_per, np, part.d(),
                                                part2.d(), scal.as<PanelScalars>());
            c.check_launch();
            pf_update<<<np, PT, 0, c.stream>>>(mr, jb, cc, P, m, rows_per, np, part2.d(),
                                               scal.as<PanelScalars>(), part.d());
            c.check_launch();
            store_tau<<<1, 1, 0, c.stream>>>(scal.as<PanelScalars>(), f.tau.d() + j0 + cc);
            c.check_launch();
        }
        // block reflector
        {
            int blocks = int(std::min<int64_t>((mr * jb + 255) / 256, int64_t(c.num_sms) * 8));
            form_v<<<blocks, 256, 0, c.stream>>>(mr, jb, P, m, V.d());
            c.check_launch();
        }
        dgemm(c, true, false, jb, jb, mr, 1.0, V.d(), mr, V.d(), mr, 0.0, G.d(), jb);
        larft_k<<<1, NB, 0, c.stream>>>(jb, G.d(), f.tau.d() + j0, f.T.d() + j0 * NB);
        c.check_launch();
        const int64_t nr = n - j0 - jb;
        if (nr > 0) {
            double* Cm = a + j0 + (j0 + jb) * m;
            dgemm(c, true, false, jb, nr, mr, 1.0, V.d(), mr, Cm, m, 0.0, W.d(), jb);
            dgemm(c, true, false, jb, nr, jb, 1.0, f.T.d() + j0 * NB, NB, W.d(), jb, 0.0, W2.d(),
                  jb);
            dgemm(c, false, false, mr, nr, jb, -1.0, V.d(), mr, W2.d(), jb, 1.0, Cm, m);
        }
    }
}

void apply_q(Ctx& c, const QRFact& f, bool trans, int64_t k, double* Y, int64_t ldy) {
    StageTimer _t(c, "qr_apply_q");
    const int64_t m = f.m, kk = std::min(f.m, f.n);
    if (k <= 0 || kk <= 0) return;
    DBuf V = dalloc(c, size_t(m) * NB);
    DBuf W = dalloc(c, size_t(NB) * size_t(k));
    DBuf W2 = dalloc(c, size_t(NB) * size_t(k));
    const int64_t npan = (kk + NB - 1) / NB;
    for (int64_t pi = 0; pi < npan; ++pi) {
        const int64_t p = trans ? pi : (npan - 1 - pi);
        const int64_t j0 = p * NB;
        const int jb = int(std::min<int64_t>(NB, kk - j0));
        const int64_t mr = m - j0;
        int blocks = int(std::min<int64_t>((mr * jb + 255) / 256, int64_t(c.num_sms) * 8));
        form_v<<<blocks, 256, 0, c.stream>>>(mr, jb, f.a.d() + j0 + j0 * m, m, V.d());
        c.check_launch();
        double* Ys = Y + j0;
        dgemm(c, true, false, jb, k, mr, 1.0, V.d(), mr, Ys, ldy, 0.0, W.d(), jb);
        // Q Y uses T, Q^T Y uses T^T
        dgemm(c, trans, false, jb, k, jb, 1.0, f.T.d() + j0 * NB, NB, W.d(), jb, 0.0, W2.d(), jb);
        dgemm(c, false, false, mr, k, jb, -1.0, V.d(), mr, W2.d(), jb, 1.0, Ys, ldy);
    }
}

}  // namespace hydot
