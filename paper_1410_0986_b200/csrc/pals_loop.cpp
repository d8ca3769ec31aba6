// pals_loop.cpp -- host control of the device PaLS reconstruction
// (SURVEY 8a A19), following proj/src/pals.cpp:139-295 step by step.  Every
// N- and M-length array stays on the device; the host holds the n_p
// parameters, the n_species concentrations, the 5n_p-vector dp and the
// scalar norms that drive the accept / retry / stop decisions.
#include <algorithm>
#include <cmath>

#include "pals.h"

namespace hydot {
namespace pals {

std::vector<double> Params::to_vector() const {
    const int n = np();
    std::vector<double> v(static_cast<size_t>(5 * n));
    for (int k = 0; k < n; ++k) {
        v[size_t(k)] = alpha[size_t(k)];
        v[size_t(n + k)] = beta[size_t(k)];
        for (int a = 0; a < 3; ++a) v[size_t((2 + a) * n + k)] = centers[size_t(k + a * n)];
    }
    return v;
}

Params Params::with_vector(const std::vector<double>& v) const {
    Params o = *this;
    const int n = np();
    if (int64_t(v.size()) != 5 * int64_t(n)) throw std::invalid_argument("PaLSParams: parameter vector length");
    for (int k = 0; k < n; ++k) {
        o.alpha[size_t(k)] = v[size_t(k)];
        o.beta[size_t(k)] = std::max(v[size_t(n + k)], 1e-8);  // widths stay positive (pals.cpp:31)
        for (int a = 0; a < 3; ++a) o.centers[size_t(k + a * n)] = v[size_t((2 + a) * n + k)];
    }
    return o;
}

Params Params::from(const hydot_pals_params& p) {
    if (p.np < 0 || (p.np > 0 && (!p.alpha || !p.beta || !p.centers)))
        throw std::invalid_argument("PaLS: bad parameter arrays");
    Params o;
    o.alpha.assign(p.alpha, p.alpha + p.np);
    o.beta.assign(p.beta, p.beta + p.np);
    o.centers.assign(p.centers, p.centers + 3 * p.np);
    o.tau_level = p.tau_level;
    o.eps_H = p.eps_H;
    o.nu_norm = p.nu_norm;
    return o;
}

void hmv(Ctx& c, const Hop& h, int b, const double* X, int64_t ldx, double* Y, int64_t ldy) {
    const Factor& F = *h.f;
    const int64_t M = F.rows, N = F.cols, R = F.rank;
    if (b <= 0) return;
    if (ldx < N || ldy < M) throw std::invalid_argument("Hmv: dimension mismatch");
    if (R == 0) {
        fill(c, M, b, 0.0, Y, ldy);
        return;
    }
    DBuf Z = dalloc(c, size_t(R) * b);
    DBuf T;
    double* out = Y;
    int64_t ldo = ldy;
    if (h.perm) {
        T = dalloc(c, size_t(M) * b);
        out = T.d();
        ldo = M;
    }
    if (skinny_ok(b)) {
        skinny_tn(c, N, R, b, F.V.d(), N, X, ldx, Z.d(), R);
        skinny_nn(c, M, R, b, F.U.d(), M, Z.d(), R, out, ldo);
    } else {
        dgemm(c, true, false, R, b, N, 1.0, F.V.d(), N, X, ldx, 0.0, Z.d(), R);
        dgemm(c, false, false, M, b, R, 1.0, F.U.d(), M, Z.d(), R, 0.0, out, ldo);
    }
    if (h.perm) scatter_rows(c, M, b, T.d(), M, h.perm, Y, ldy);  // out[perm[i]] = t[i]
}

namespace {

// Eigen ColPivHouseholderQR(A).solve(b) for a tall A with few columns
// (pals.cpp:147-153): Householder with column pivoting on the largest
// remaining column norm; rank() counts |R_ii| > thr * max|R_jj|, solve()
// uses the pivots before the remaining norm^2 drops below
// (eps * max initial norm)^2 (m - k) / m.
struct CPQR {
    std::vector<double> x;
    int rank = 0;
};
CPQR colpiv_solve(std::vector<double> A, int64_t m, int n, std::vector<double> b, double thr) {
    CPQR out;
    out.x.assign(size_t(n), 0.0);
    if (n == 0 || m == 0) return out;
    std::vector<int> perm(static_cast<size_t>(n));
    for (int j = 0; j < n; ++j) perm[size_t(j)] = j;
    auto col = [&](int j) { return A.data() + int64_t(j) * m; };
    auto tail_norm2 = [&](int j, int64_t k) {
        double s = 0.0;
        const double* a = col(j);
        for (int64_t i = k; i < m; ++i) s += a[i] * a[i];
        return s;
    };
    double max0 = 0.0;
    for (int j = 0; j < n; ++j) max0 = std::max(max0, std::sqrt(tail_norm2(j, 0)));
    const double eps = 2.220446049250313e-16;
    const double helper = (max0 * eps) * (max0 * eps) / double(m);
    const int kmax = int(std::min<int64_t>(m, n));
    int nonzero = kmax;
    double maxpiv = 0.0;
    std::vector<double> diag(static_cast<size_t>(kmax), 0.0);
    for (int k = 0; k < kmax; ++k) {
        int best = k;
        double bn = -1.0;
        for (int j = k; j < n; ++j) {
            const double t = tail_norm2(j, k);
            if (t > bn) {
                bn = t;
                best = j;
            }
        }
        if (nonzero == kmax && bn < helper * double(m - k)) nonzero = k;
        if (best != k) {
            std::swap_ranges(col(k), col(k) + m, col(best));
            std::swap(perm[size_t(k)], perm[size_t(best)]);
        }
        double* a = col(k);
        const double alpha = a[k];
        double xn2 = 0.0;
        for (int64_t i = k + 1; i < m; ++i) xn2 += a[i] * a[i];
        double beta = alpha, tau = 0.0;
        if (xn2 > 0.0) {
            beta = -std::copysign(std::hypot(alpha, std::sqrt(xn2)), alpha);
            tau = (beta - alpha) / beta;
            const double scal = 1.0 / (alpha - beta);
            for (int64_t i = k + 1; i < m; ++i) a[i] *= scal;
        }
        a[k] = 1.0;
        // apply H = I - tau v v^T to the remaining columns and to b
        for (int j = k + 1; j < n; ++j) {
            double* cj = col(j);
            double s = 0.0;
            for (int64_t i = k; i < m; ++i) s += a[i] * cj[i];
            s *= tau;
            for (int64_t i = k; i < m; ++i) cj[i] -= s * a[i];
        }
        {
            double s = 0.0;
            for (int64_t i = k; i < m; ++i) s += a[i] * b[size_t(i)];
            s *= tau;
            for (int64_t i = k; i < m; ++i) b[size_t(i)] -= s * a[i];
        }
        a[k] = beta;
        diag[size_t(k)] = beta;
        maxpiv = std::max(maxpiv, std::fabs(beta));
    }
    for (int k = 0; k < kmax; ++k)
        if (std::fabs(diag[size_t(k)]) > maxpiv * thr) ++out.rank;
    std::vector<double> cc(b.begin(), b.begin() + nonzero);
    for (int i = nonzero - 1; i >= 0; --i) {
        double s = cc[size_t(i)];
        for (int j = i + 1; j < nonzero; ++j) s -= A[size_t(i + int64_t(j) * m)] * cc[size_t(j)];
        cc[size_t(i)] = s / A[size_t(i + int64_t(i) * m)];
    }
    for (int i = 0; i < nonzero; ++i) out.x[size_t(perm[size_t(i)])] = cc[size_t(i)];
    return out;
}

}  // namespace

Conc solve_concentrations(Ctx& c, const Hop& h, const double* mu, const double* w, const double* y,
                          const double* ext_h, int nl, int nsp) {
    StageTimer _t(c, "pals_concentrations");
    if (nl < 1 || nsp < 0) throw std::invalid_argument("solve_concentrations: bad spectra");
    const int64_t M = h.f->rows;
    Conc res;
    res.c.assign(size_t(nsp), 0.0);
    DBuf hmu = dalloc(c, size_t(M));
    hmv(c, h, 1, mu, h.f->cols, hmu.d(), M);
    // W D(p) is M x n_species: the pivoted least-squares solve runs on the
    // host like the reference's Eigen call (three M-vectors cross the bus)
    std::vector<double> hh(static_cast<size_t>(M)), wh(static_cast<size_t>(M)), yh(static_cast<size_t>(M));
    c.d2h(hh.data(), hmu.d(), size_t(M));
    c.d2h(wh.data(), w, size_t(M));
    c.d2h(yh.data(), y, size_t(M));
    std::vector<double> WD(static_cast<size_t>(M * nsp)), wy(static_cast<size_t>(M));
    for (int i = 0; i < nsp; ++i)
        for (int64_t m = 0; m < M; ++m)
            WD[size_t(m + i * M)] = wh[size_t(m)] * (ext_h[(m % nl) + int64_t(i) * nl] * hh[size_t(m)]);
    for (int64_t m = 0; m < M; ++m) wy[size_t(m)] = wh[size_t(m)] * yh[size_t(m)];
    CPQR q = colpiv_solve(std::move(WD), M, nsp, std::move(wy), 1e-12);
    if (q.rank < nsp) {
        res.flagged = true;
        if (q.rank == 0) return res;  // empty anomaly: c = 0
    }
    res.c = q.x;
    return res;
}

std::vector<double> lm_step(Ctx& c, int64_t M, int n, const double* J, int64_t ldj, const double* eps,
                            double nu) {
    StageTimer _t(c, "pals_lm_step", M, n);
    if (nu < 0) throw std::invalid_argument("lm_step: damping must be nonnegative");
    if (n <= 0) return {};
    if (ldj < M) throw std::invalid_argument("lm_step: dimension mismatch");
    const int64_t rows = M + n;
    DBuf A = dalloc(c, size_t(rows) * n), rhs = dalloc(c, size_t(rows));
    stack_damped(c, M, n, J, ldj, eps, nu, A.d(), rhs.d());
    QRFact f;
    geqrf(c, rows, n, A.d(), rows, f);
    apply_q(c, f, true, 1, rhs.d(), rows);
    DBuf Rc = dalloc(c, size_t(n) * n);
    copy2d(c, n, n, f.a.d(), rows, Rc.d(), n);
    std::vector<double> R(static_cast<size_t>(n) * n), q(static_cast<size_t>(n));
    c.d2h(R.data(), Rc.d(), R.size());
    c.d2h(q.data(), rhs.d(), q.size());
    std::vector<double> dp(static_cast<size_t>(n), 0.0);
    for (int i = n - 1; i >= 0; --i) {  // R dp = (Q^T rhs)[0:n]
        double s = q[size_t(i)];
        for (int j = i + 1; j < n; ++j) s -= R[size_t(i + int64_t(j) * n)] * dp[size_t(j)];
        const double d = R[size_t(i + int64_t(i) * n)];
        dp[size_t(i)] = d != 0.0 ? s / d : 0.0;
    }
    return dp;
}

Metrics metrics(Ctx& c, int64_t N, const double* a, const double* b, double thr) {
    double s[6];
    metric_sums(c, N, a, b, thr, s);
    Metrics m;
    const double tn = std::sqrt(s[1]);
    m.l2_rel = tn > 0 ? std::sqrt(s[0]) / tn : (std::sqrt(s[2]) > 0 ? 1.0 : 0.0);
    const double na = s[3], nb = s[4], inter = s[5];
    if (na + nb == 0) {
        m.dice = 1.0;
        m.flagged = true;
    } else {
        m.dice = 2.0 * inter / (na + nb);
    }
    return m;
}

Recon reconstruct(Ctx& c, const Hop& h, const Geom& g, const double* ext_h, int nl, int nsp,
                  const double* y, const double* w, const Params& init, double noise_norm,
                  const ReconCfg& cfg, const double* mu_truth) {
    StageTimer _t(c, "pals_reconstruct");
    if (cfg.gamma <= 1.0) throw std::invalid_argument("reconstruct: gamma must exceed 1");
    const int64_t M = h.f->rows, N = h.f->cols;
    if (g.N() != N) throw std::invalid_argument("reconstruct: grid / operator size mismatch");
    if (!cfg.fixed_c.empty() && int(cfg.fixed_c.size()) != nsp)
        throw std::invalid_argument("reconstruct: fixed concentration length");
    Recon res;
    res.p = init;
    const int np5 = 5 * init.np();
    DBuf mu = dalloc(c, size_t(N)), hmu = dalloc(c, size_t(M));
    DBuf eps = dalloc(c, size_t(M)), eps_try = dalloc(c, size_t(M));
    DBuf ext_d = dalloc(c, size_t(nl) * std::max(nsp, 1)), c_d = dalloc(c, size_t(std::max(nsp, 1)));
    DBuf ebar_d = dalloc(c, size_t(nl));
    DBuf dmudp = dalloc(c, size_t(N) * std::max(np5, 1));
    DBuf HJ = dalloc(c, size_t(M) * std::max(np5, 1)), J = dalloc(c, size_t(M) * std::max(np5, 1));
    DBuf tmp = mu_truth ? dalloc(c, size_t(N)) : DBuf();
    HYDOT_CUDA(cudaMemcpyAsync(ext_d.d(), ext_h, size_t(nl) * nsp * 8, cudaMemcpyHostToDevice, c.stream));
    // normal-equation blocks (cfg.normal_blocks): X (N nsp) x b, Y M x b, Z (N nsp) x b
    const int nbk = nsp > 0 ? std::min(cfg.normal_blocks, std::max(np5, 0)) : 0;
    DBuf nX, nY, nW, nZ, nconc, nperm;
    if (nbk > 0) {
        nX = dalloc(c, size_t(N) * nsp * nbk);
        nY = dalloc(c, size_t(M) * nbk);
        nW = dalloc(c, size_t(M) * nbk);
        nZ = dalloc(c, size_t(N) * nsp * nbk);
        nconc = dalloc(c, size_t(nsp));
        if (!h.perm) {
            std::vector<int> id(static_cast<size_t>(M));
            for (int64_t i = 0; i < M; ++i) id[size_t(i)] = int(i);
            nperm = DBuf(c, size_t(M) * sizeof(int));
            HYDOT_CUDA(cudaMemcpyAsync(nperm.as<void>(), id.data(), size_t(M) * sizeof(int), cudaMemcpyHostToDevice,
                                       c.stream));
            c.sync();
        }
    }
    auto normal_products = [&]() {
        HYDOT_CUDA(cudaMemcpyAsync(nconc.d(), res.c.data(), size_t(nsp) * 8, cudaMemcpyHostToDevice, c.stream));
        kron_conc(c, N, nbk, nsp, nconc.d(), dmudp.d(), N, nX.d(), N * nsp);
        const int* perm = h.perm ? h.perm : nperm.as<int>();
        j_matmat(c, h.f->U.d(), h.f->V.d(), M, N, h.f->rank, false, nbk, perm, ext_d.d(), nl, nsp, nX.d(), N * nsp,
                 nY.d(), M);
        wsq_rows(c, M, nbk, w, nY.d(), M, nW.d(), M);
        j_matmat(c, h.f->U.d(), h.f->V.d(), M, N, h.f->rank, true, nbk, perm, ext_d.d(), nl, nsp, nW.d(), M,
                 nZ.d(), N * nsp);
        res.normal_columns += nbk;
    };

    auto Hmv = [&](int b, const double* X, double* Y) {
        hmv(c, h, b, X, N, Y, M);
        res.hmv_calls += 1;
        res.hmv_columns += b;
    };
    // Objective::residual (pals.cpp:180-188) -> ||eps||
    auto residual_of = [&](const Params& p, const std::vector<double>& cv, double* out) {
        eval(c, EVAL_SHAPE, g, p, mu.d(), N);
        Hmv(1, mu.d(), hmu.d());
        HYDOT_CUDA(cudaMemcpyAsync(c_d.d(), cv.data(), cv.size() * 8, cudaMemcpyHostToDevice, c.stream));
        residual(c, M, nl, nsp, ext_d.d(), c_d.d(), y, w, hmu.d(), out);
        return norm2(c, M, out);
    };
    auto dice_now = [&](const Params& p) {
        if (!mu_truth) return -1.0;
        eval(c, EVAL_SHAPE, g, p, tmp.d(), N);
        return metrics(c, N, mu_truth, tmp.d(), 0.5).dice;
    };

    const double target = cfg.gamma * noise_norm;
    double nu = cfg.nu0;
    std::vector<double> outer_norms;
    for (int outer = 0; outer < cfg.max_outer; ++outer) {
        if (cfg.fixed_c.empty()) {
            eval(c, EVAL_SHAPE, g, res.p, mu.d(), N);
            const int64_t calls = res.hmv_calls;
            res.c = solve_concentrations(c, h, mu.d(), w, y, ext_h, nl, nsp).c;
            res.hmv_calls = calls + 1;
            res.hmv_columns += 1;
        } else {
            res.c = cfg.fixed_c;
        }
        res.resnorm = residual_of(res.p, res.c, eps.d());
        res.trace.push_back({outer, -1, res.resnorm, nu, true, dice_now(res.p)});
        if (res.resnorm <= target) {
            res.converged = true;
            break;
        }
        outer_norms.push_back(res.resnorm);
        if (outer_norms.size() >= 4) {
            const double past = outer_norms[outer_norms.size() - 4];
            if (std::fabs(past - res.resnorm) <= cfg.stagnation_tol * std::max(past, 1e-300)) break;
        }
        // per-measurement extinction mix (pals.cpp:240-246)
        std::vector<double> ebar(static_cast<size_t>(nl));
        for (int l = 0; l < nl; ++l) {
            double e = 0.0;
            for (size_t i = 0; i < res.c.size(); ++i) e += res.c[i] * ext_h[l + int64_t(i) * nl];
            ebar[size_t(l)] = e;
        }
        HYDOT_CUDA(cudaMemcpyAsync(ebar_d.d(), ebar.data(), size_t(nl) * 8, cudaMemcpyHostToDevice, c.stream));

        bool stalled = false;
        for (int inner = 0; inner < cfg.max_inner; ++inner) {
            // J = -W Ebar H dmu/dp: one blocked product of 5 n_p columns
            eval(c, EVAL_JACOBIAN, g, res.p, dmudp.d(), N);
            Hmv(np5, dmudp.d(), HJ.d());
            jscale(c, M, np5, nl, w, ebar_d.d(), HJ.d(), M, J.d(), M);
            if (nbk > 0) normal_products();
            bool accepted = false;
            double nu_try = nu;
            for (int attempt = 0; attempt < cfg.max_retries; ++attempt) {
                std::vector<double> dp = lm_step(c, M, np5, J.d(), M, eps.d(), nu_try);
                std::vector<double> v = res.p.to_vector();
                for (size_t i = 0; i < v.size(); ++i) v[i] += dp[i];
                Params p_try = res.p.with_vector(v);
                const double rn = residual_of(p_try, res.c, eps_try.d());
                res.trace.push_back({outer, inner, rn, nu_try, rn < res.resnorm, dice_now(p_try)});
                if (rn < res.resnorm) {
                    res.p = p_try;
                    std::swap(eps, eps_try);
                    res.resnorm = rn;
                    nu = std::max(nu_try / 10.0, 1e-12);
                    accepted = true;
                    break;
                }
                nu_try *= 10.0;
            }
            if (!accepted) {
                stalled = true;
                break;
            }
            if (res.resnorm <= target) break;
        }
        if (res.resnorm <= target) {
            res.converged = true;
            res.trace.push_back({cfg.max_outer, -1, res.resnorm, nu, true, dice_now(res.p)});
            break;
        }
        if (stalled) {
            res.flagged = true;
            break;
        }
    }
    c.sync();
    return res;
}

}  // namespace pals
}  // namespace hydot
