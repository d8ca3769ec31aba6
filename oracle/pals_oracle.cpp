// pals_oracle.cpp -- CPU ORACLE (test infrastructure only).
//
// Restatement of the reference PaLS reconstruction loop (SURVEY 8a A19,
// /root/reference/proj/src/pals.cpp, include/hydot/pals.hpp) used ONLY by
// tests/ and bench.py's cpu_baseline as the checker of the device PaLS path
// (paper_1410_0986_b200/csrc/pals.*).  The product never links this file.
//
// The operator Hmv is the permuted low-rank matvec the reference hands to
// reconstruct (experiments.cpp:255-262 over lowrank.cpp:589-593):
// out[perm[i]] = (U (V^T x))[i]; a dense H is the special case U = H,
// V = I.  Eigen's ColPivHouseholderQR (pals.cpp:147-153, 168) is LAPACK
// dgeqp3 + dormqr + a triangular solve here, with Eigen's rank rule
// (|R_ii| > threshold * max|R_jj|) and its nonzero-pivot rule for solve().
//
// Parity status: pinned by the reference's own pals tests restated in
// tests/test_pals_oracle.py (Wendland/Heaviside known values, level set vs
// the direct RBF sum, parameter round trip, Jacobian vs central
// differences, LM step vs the damped normal equations, concentration
// recovery, overlap metrics, reconstruction reaching the discrepancy
// target); Eigen's own arithmetic is not reproducible here (no Eigen).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

extern "C" {
void scipy_dgeqp3_(const int*, const int*, double*, const int*, int*, double*, double*,
                   const int*, int*);
void scipy_dormqr_(const char*, const char*, const int*, const int*, const int*, const double*,
                   const int*, const double*, double*, const int*, double*, const int*, int*);
}

namespace pals_oracle {

// grid::Grid / build_grid (grid.hpp:22-45, grid.cpp:94-110)
struct Geom {
    int nx, ny, nz;
    double Lx, Ly, Lz, hx, hy, hz;
    Geom(int x, int y, int z, double lx, double ly, double lz)
        : nx(x), ny(y), nz(z), Lx(lx), Ly(ly), Lz(lz) {
        if (nx < 2 || ny < 2 || nz < 2) throw std::invalid_argument("build_grid: vertex counts must be >= 2");
        if (Lx <= 0 || Ly <= 0 || Lz <= 0) throw std::invalid_argument("build_grid: extents must be positive");
        hx = 2 * Lx / (nx - 1);
        hy = 2 * Ly / (ny - 1);
        hz = Lz / (nz - 1);
    }
    int64_t N() const { return int64_t(nx) * ny * nz; }
    void vertex(int64_t n, double r[3]) const {  // grid.hpp:37-40
        int ix = int(n % nx), iy = int((n / nx) % ny), iz = int(n / (int64_t(nx) * ny));
        r[0] = -Lx + ix * hx;
        r[1] = -Ly + iy * hy;
        r[2] = iz * hz;
    }
};

// PaLSParams (pals.hpp:16-32); centers n_p x 3 column-major
struct Params {
    std::vector<double> alpha, beta, centers;
    double tau_level = 0.1, eps_H = 0.05, nu_norm = 1e-3;
    int np() const { return int(alpha.size()); }
    double c(int k, int a) const { return centers[size_t(k + a * np())]; }
    std::vector<double> to_vector() const {  // pals.cpp:14-23
        const int n = np();
        std::vector<double> v(static_cast<size_t>(5 * n));
        for (int k = 0; k < n; ++k) {
            v[size_t(k)] = alpha[size_t(k)];
            v[size_t(n + k)] = beta[size_t(k)];
            for (int a = 0; a < 3; ++a) v[size_t((2 + a) * n + k)] = c(k, a);
        }
        return v;
    }
    Params with_vector(const std::vector<double>& v) const {  // pals.cpp:25-36
        Params o = *this;
        const int n = np();
        if (int64_t(v.size()) != 5 * n) throw std::invalid_argument("PaLSParams: parameter vector length");
        for (int k = 0; k < n; ++k) {
            o.alpha[size_t(k)] = v[size_t(k)];
            o.beta[size_t(k)] = std::max(v[size_t(n + k)], 1e-8);  // widths stay positive
            for (int a = 0; a < 3; ++a) o.centers[size_t(k + a * n)] = v[size_t((2 + a) * n + k)];
        }
        return o;
    }
};

// pals.cpp:38-60
double wendland(double t) {
    if (t >= 1.0) return 0.0;
    double s = 1.0 - t;
    double s2 = s * s;
    return s2 * s2 * (4.0 * t + 1.0);
}
double wendland_deriv(double t) {
    if (t >= 1.0) return 0.0;
    double s = 1.0 - t;
    return -20.0 * t * s * s * s;
}
double smooth_heaviside(double t, double eps) {
    if (t < -eps) return 0.0;
    if (t > eps) return 1.0;
    return 0.5 * (1.0 + t / eps + std::sin(M_PI * t / eps) / M_PI);
}
double smooth_delta(double t, double eps) {
    if (t < -eps || t > eps) return 0.0;
    return 0.5 / eps * (1.0 + std::cos(M_PI * t / eps));
}

// pals.cpp:64-70
double star_norm(const double r[3], const Params& p, int k) {
    double dx = r[0] - p.c(k, 0);
    double dy = r[1] - p.c(k, 1);
    double dz = r[2] - p.c(k, 2);
    return std::sqrt(dx * dx + dy * dy + dz * dz + p.nu_norm * p.nu_norm);
}

// pals.cpp:74-86
std::vector<double> level_set(const Params& p, const Geom& g) {
    std::vector<double> phi(size_t(g.N()), 0.0);
    for (int64_t n = 0; n < g.N(); ++n) {
        double r[3];
        g.vertex(n, r);
        double v = 0.0;
        for (int k = 0; k < p.np(); ++k) v += p.alpha[size_t(k)] * wendland(p.beta[size_t(k)] * star_norm(r, p, k));
        phi[size_t(n)] = v;
    }
    return phi;
}

// pals.cpp:88-94
std::vector<double> shape(const Params& p, const Geom& g) {
    std::vector<double> mu = level_set(p, g);
    for (double& v : mu) v = smooth_heaviside(v - p.tau_level, p.eps_H);
    return mu;
}

// pals.cpp:96-119 ; J is N x 5 n_p column-major
std::vector<double> shape_jacobian(const Params& p, const Geom& g) {
    const int64_t N = g.N();
    const int n_p = p.np();
    std::vector<double> J(size_t(N * 5 * n_p), 0.0);
    std::vector<double> phi = level_set(p, g);
    for (int64_t n = 0; n < N; ++n) {
        double d = smooth_delta(phi[size_t(n)] - p.tau_level, p.eps_H);
        if (d == 0.0) continue;
        double r[3];
        g.vertex(n, r);
        for (int k = 0; k < n_p; ++k) {
            double nr = star_norm(r, p, k);
            double t = p.beta[size_t(k)] * nr;
            double psi = wendland(t);
            double dpsi = wendland_deriv(t);
            J[size_t(n + int64_t(k) * N)] = d * psi;
            J[size_t(n + int64_t(n_p + k) * N)] = d * p.alpha[size_t(k)] * dpsi * nr;
            double fac = -d * p.alpha[size_t(k)] * p.beta[size_t(k)] * dpsi / nr;
            for (int a = 0; a < 3; ++a) J[size_t(n + int64_t((2 + a) * n_p + k) * N)] = fac * (r[a] - p.c(k, a));
        }
    }
    return J;
}

// The permuted low-rank operator (experiments.cpp:255-262, lowrank.cpp:589-593)
struct Hop {
    const double *U, *V;
    int64_t M, N, R;
    const int* perm;  // M entries, or null
    std::vector<double> operator()(const std::vector<double>& x) const {
        std::vector<double> z(size_t(R), 0.0), t(size_t(M), 0.0), y(size_t(M), 0.0);
        for (int64_t k = 0; k < R; ++k) {
            double s = 0.0;
            for (int64_t i = 0; i < N; ++i) s += V[i + k * N] * x[size_t(i)];
            z[size_t(k)] = s;
        }
        for (int64_t k = 0; k < R; ++k)
            for (int64_t i = 0; i < M; ++i) t[size_t(i)] += U[i + k * M] * z[size_t(k)];
        for (int64_t i = 0; i < M; ++i) y[size_t(perm ? perm[i] : i)] = t[size_t(i)];
        return y;
    }
};

double norm2(const std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
}

// Eigen ColPivHouseholderQR(A).solve(b) with setThreshold(thr) for rank():
// returns x (n), rank and the nonzero-pivot count.
struct CPQR {
    std::vector<double> x;
    int rank = 0, nonzero = 0;
};
CPQR colpiv_solve(std::vector<double> A, int64_t m, int n, std::vector<double> b, double thr) {
    CPQR out;
    out.x.assign(size_t(n), 0.0);
    if (n == 0) return out;
    int M = int(m), Nn = n, lda = std::max(1, M), info = 0;
    std::vector<int> jpvt(static_cast<size_t>(n), 0);
    std::vector<double> tau(static_cast<size_t>(n));
    int lwork = -1;
    double wq = 0;
    scipy_dgeqp3_(&M, &Nn, A.data(), &lda, jpvt.data(), tau.data(), &wq, &lwork, &info);
    lwork = std::max(1, int(wq));
    std::vector<double> work(static_cast<size_t>(lwork));
    scipy_dgeqp3_(&M, &Nn, A.data(), &lda, jpvt.data(), tau.data(), work.data(), &lwork, &info);
    if (info != 0) throw std::runtime_error("dgeqp3 failed");
    const int kmax = int(std::min<int64_t>(m, n));
    double maxpiv = 0.0;
    for (int i = 0; i < kmax; ++i) maxpiv = std::max(maxpiv, std::fabs(A[size_t(i + int64_t(i) * m)]));
    for (int i = 0; i < kmax; ++i)
        if (std::fabs(A[size_t(i + int64_t(i) * m)]) > maxpiv * thr) ++out.rank;
    // Eigen: pivots count until the largest remaining column norm^2 drops
    // below (eps * max initial column norm)^2 / m * (m - k)
    const double eps = 2.220446049250313e-16;
    const double r00 = std::fabs(A[0]);
    const double helper = (r00 * eps) * (r00 * eps) / double(m);
    out.nonzero = kmax;
    for (int k = 0; k < kmax; ++k) {
        const double rk = A[size_t(k + int64_t(k) * m)];
        if (rk * rk < helper * double(m - k)) {
            out.nonzero = k;
            break;
        }
    }
    if (out.nonzero == 0) return out;
    int one = 1, ldb = std::max(1, M), nz = out.nonzero;
    lwork = -1;
    scipy_dormqr_("L", "T", &M, &one, &nz, A.data(), &lda, tau.data(), b.data(), &ldb, &wq, &lwork, &info);
    lwork = std::max(1, int(wq));
    work.assign(size_t(lwork), 0.0);
    scipy_dormqr_("L", "T", &M, &one, &nz, A.data(), &lda, tau.data(), b.data(), &ldb, work.data(), &lwork,
                  &info);
    if (info != 0) throw std::runtime_error("dormqr failed");
    std::vector<double> c(b.begin(), b.begin() + nz);
    for (int i = nz - 1; i >= 0; --i) {
        double s = c[size_t(i)];
        for (int j = i + 1; j < nz; ++j) s -= A[size_t(i + int64_t(j) * m)] * c[size_t(j)];
        c[size_t(i)] = s / A[size_t(i + int64_t(i) * m)];
    }
    for (int i = 0; i < nz; ++i) out.x[size_t(jpvt[size_t(i)] - 1)] = c[size_t(i)];
    return out;
}

// assemble_D (pals.cpp:124-135); ext is n_lambda x n_species column-major
std::vector<double> assemble_D(const std::vector<double>& hmu, const double* ext, int nl, int nsp) {
    const int64_t M = int64_t(hmu.size());
    std::vector<double> D(static_cast<size_t>(M * nsp));
    for (int i = 0; i < nsp; ++i)
        for (int64_t m = 0; m < M; ++m) D[size_t(m + i * M)] = ext[(m % nl) + int64_t(i) * nl] * hmu[size_t(m)];
    return D;
}

struct Conc {
    std::vector<double> c;
    bool flagged = false;
};

// solve_concentrations (pals.cpp:139-156)
Conc solve_concentrations(const Hop& H, const std::vector<double>& mu, const std::vector<double>& w,
                          const std::vector<double>& y, const double* ext, int nl, int nsp) {
    Conc res;
    res.c.assign(size_t(nsp), 0.0);
    std::vector<double> hmu = H(mu);
    const int64_t M = int64_t(hmu.size());
    std::vector<double> WD = assemble_D(hmu, ext, nl, nsp);
    for (int i = 0; i < nsp; ++i)
        for (int64_t m = 0; m < M; ++m) WD[size_t(m + i * M)] = w[size_t(m)] * WD[size_t(m + i * M)];
    std::vector<double> wy(static_cast<size_t>(M));
    for (int64_t m = 0; m < M; ++m) wy[size_t(m)] = w[size_t(m)] * y[size_t(m)];
    CPQR q = colpiv_solve(WD, M, nsp, wy, 1e-12);
    if (q.rank < nsp) {
        res.flagged = true;
        if (q.rank == 0) return res;  // empty anomaly: c = 0
    }
    res.c = q.x;
    return res;
}

// lm_step (pals.cpp:158-169); J is M x n column-major
std::vector<double> lm_step(const std::vector<double>& J, int64_t M, int n, const std::vector<double>& eps,
                            double nu) {
    if (nu < 0) throw std::invalid_argument("lm_step: damping must be nonnegative");
    const int64_t rows = M + n;
    std::vector<double> A(size_t(rows * n), 0.0), rhs(size_t(rows), 0.0);
    for (int j = 0; j < n; ++j) {
        for (int64_t i = 0; i < M; ++i) A[size_t(i + j * rows)] = J[size_t(i + j * M)];
        A[size_t(M + j + j * rows)] = std::sqrt(nu);
    }
    for (int64_t i = 0; i < M; ++i) rhs[size_t(i)] = -eps[size_t(i)];
    return colpiv_solve(A, rows, n, rhs, 2.220446049250313e-16).x;
}

// Objective::residual (pals.cpp:180-188)
std::vector<double> residual(const Hop& H, const Geom& g, const Params& p, const std::vector<double>& c,
                             const std::vector<double>& y, const std::vector<double>& w, const double* ext,
                             int nl) {
    std::vector<double> hmu = H(shape(p, g));
    const int64_t M = int64_t(hmu.size());
    const int nsp = int(c.size());
    std::vector<double> D = assemble_D(hmu, ext, nl, nsp);
    std::vector<double> e(static_cast<size_t>(M));
    for (int64_t m = 0; m < M; ++m) {
        double dc = 0.0;
        for (int i = 0; i < nsp; ++i) dc += D[size_t(m + i * M)] * c[size_t(i)];
        e[size_t(m)] = w[size_t(m)] * (y[size_t(m)] - dc);
    }
    return e;
}

struct Metrics {
    double l2_rel = 0.0, dice = 0.0;
    bool flagged = false;
};
// metrics (pals.cpp:307-329)
Metrics metrics(const std::vector<double>& a, const std::vector<double>& b, double thr) {
    if (a.size() != b.size()) throw std::invalid_argument("metrics: length mismatch");
    Metrics m;
    double tn = norm2(a);
    std::vector<double> d(a.size());
    for (size_t i = 0; i < a.size(); ++i) d[i] = a[i] - b[i];
    m.l2_rel = tn > 0 ? norm2(d) / tn : (norm2(b) > 0 ? 1.0 : 0.0);
    long na = 0, nb = 0, inter = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        bool ta = a[i] > thr, tb = b[i] > thr;
        na += ta;
        nb += tb;
        inter += ta && tb;
    }
    if (na + nb == 0) {
        m.dice = 1.0;
        m.flagged = true;
    } else {
        m.dice = 2.0 * double(inter) / double(na + nb);
    }
    return m;
}

struct TraceRow {
    int outer, inner;
    double resnorm, nu;
    int accepted;
    double dice;
};
struct ReconCfg {
    int max_outer = 30, max_inner = 5, max_retries = 8;
    double gamma = 1.2, nu0 = 1.0, stagnation_tol = 1e-6;
    std::vector<double> fixed_c;
};
struct Recon {
    Params p;
    std::vector<double> c;
    std::vector<TraceRow> trace;
    double resnorm = 0.0;
    bool converged = false, flagged = false;
};

// reconstruct (pals.cpp:193-295)
Recon reconstruct(const std::vector<double>& y, const Hop& H, const Geom& g, const double* ext, int nl,
                  int nsp, const Params& init, const std::vector<double>& w, double noise_norm,
                  const ReconCfg& cfg, const std::vector<double>* mu_truth) {
    if (cfg.gamma <= 1.0) throw std::invalid_argument("reconstruct: gamma must exceed 1");
    Recon res;
    res.p = init;
    const int64_t M = int64_t(y.size());
    const double target = cfg.gamma * noise_norm;
    double nu = cfg.nu0;
    std::vector<double> outer_norms;
    auto dice_now = [&](const Params& p) {
        if (!mu_truth) return -1.0;
        return metrics(*mu_truth, shape(p, g), 0.5).dice;
    };
    for (int outer = 0; outer < cfg.max_outer; ++outer) {
        if (cfg.fixed_c.empty()) res.c = solve_concentrations(H, shape(res.p, g), w, y, ext, nl, nsp).c;
        else res.c = cfg.fixed_c;
        std::vector<double> eps = residual(H, g, res.p, res.c, y, w, ext, nl);
        res.resnorm = norm2(eps);
        res.trace.push_back({outer, -1, res.resnorm, nu, 1, dice_now(res.p)});
        if (res.resnorm <= target) {
            res.converged = true;
            break;
        }
        outer_norms.push_back(res.resnorm);
        if (outer_norms.size() >= 4) {
            double past = outer_norms[outer_norms.size() - 4];
            if (std::fabs(past - res.resnorm) <= cfg.stagnation_tol * std::max(past, 1e-300)) break;
        }
        std::vector<double> ebar(static_cast<size_t>(nl));
        for (int l = 0; l < nl; ++l) {
            double e = 0.0;
            for (size_t i = 0; i < res.c.size(); ++i) e += res.c[i] * ext[l + int64_t(i) * nl];
            ebar[size_t(l)] = e;
        }
        bool stalled = false;
        for (int inner = 0; inner < cfg.max_inner; ++inner) {
            std::vector<double> dmudp = shape_jacobian(res.p, g);
            const int np5 = 5 * res.p.np();
            const int64_t N = g.N();
            std::vector<double> J(static_cast<size_t>(M * np5));
            for (int j = 0; j < np5; ++j) {
                std::vector<double> col(dmudp.begin() + j * N, dmudp.begin() + (j + 1) * N);
                std::vector<double> hj = H(col);
                for (int64_t m = 0; m < M; ++m)
                    J[size_t(m + j * M)] = -w[size_t(m)] * ebar[size_t(m % nl)] * hj[size_t(m)];
            }
            bool accepted = false;
            double nu_try = nu;
            for (int attempt = 0; attempt < cfg.max_retries; ++attempt) {
                std::vector<double> dp = lm_step(J, M, np5, eps, nu_try);
                std::vector<double> v = res.p.to_vector();
                for (size_t i = 0; i < v.size(); ++i) v[i] += dp[i];
                Params p_try = res.p.with_vector(v);
                std::vector<double> eps_try = residual(H, g, p_try, res.c, y, w, ext, nl);
                double rn = norm2(eps_try);
                res.trace.push_back({outer, inner, rn, nu_try, rn < res.resnorm ? 1 : 0, dice_now(p_try)});
                if (rn < res.resnorm) {
                    res.p = p_try;
                    eps = eps_try;
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
            res.trace.push_back({cfg.max_outer, -1, res.resnorm, nu, 1, dice_now(res.p)});
            break;
        }
        if (stalled) {
            res.flagged = true;
            break;
        }
    }
    return res;
}

}  // namespace pals_oracle

// ----------------------------------------------------------------- C ABI --
// Geometry (nx, ny, nz, Lx, Ly, Lz) as grid::build_grid; params as
// (np, alpha, beta, centers n_p x 3 column-major, tau, eps_H, nu_norm).
using namespace pals_oracle;

namespace {
thread_local std::string g_perr;
template <class F>
int pguard(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_perr = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_perr = e.what();
        return 2;
    }
}
Params make_params(int np, const double* alpha, const double* beta, const double* centers, double tau,
                   double epsH, double nu) {
    Params p;
    p.alpha.assign(alpha, alpha + np);
    p.beta.assign(beta, beta + np);
    p.centers.assign(centers, centers + 3 * np);
    p.tau_level = tau;
    p.eps_H = epsH;
    p.nu_norm = nu;
    return p;
}
}  // namespace

extern "C" {

const char* oracle_pals_last_error() { return g_perr.c_str(); }

int oracle_pals_scalar(int which, double t, double eps, double* out) {
    return pguard([&] {
        switch (which) {
            case 0: *out = wendland(t); break;
            case 1: *out = wendland_deriv(t); break;
            case 2: *out = smooth_heaviside(t, eps); break;
            case 3: *out = smooth_delta(t, eps); break;
            default: throw std::invalid_argument("pals scalar: unknown function");
        }
    });
}

// which: 0 level set, 1 shape, 2 shape Jacobian (N x 5np)
int oracle_pals_eval(int which, int nx, int ny, int nz, double Lx, double Ly, double Lz, int np,
                     const double* alpha, const double* beta, const double* centers, double tau, double epsH,
                     double nu, double* out) {
    return pguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        Params p = make_params(np, alpha, beta, centers, tau, epsH, nu);
        std::vector<double> r = which == 0 ? level_set(p, g) : which == 1 ? shape(p, g) : shape_jacobian(p, g);
        std::copy(r.begin(), r.end(), out);
    });
}

int oracle_pals_solve_concentrations(const double* U, const double* V, int64_t M, int64_t N, int64_t R,
                                     const int* perm, const double* mu, const double* w, const double* y,
                                     const double* ext, int nl, int nsp, double* c_out, int* flagged) {
    return pguard([&] {
        Hop H{U, V, M, N, R, perm};
        Conc r = solve_concentrations(H, std::vector<double>(mu, mu + N), std::vector<double>(w, w + M),
                                      std::vector<double>(y, y + M), ext, nl, nsp);
        std::copy(r.c.begin(), r.c.end(), c_out);
        *flagged = r.flagged ? 1 : 0;
    });
}

int oracle_pals_lm_step(const double* J, int64_t M, int n, const double* eps, double nu, double* dp) {
    return pguard([&] {
        std::vector<double> r = lm_step(std::vector<double>(J, J + M * n), M, n,
                                        std::vector<double>(eps, eps + M), nu);
        std::copy(r.begin(), r.end(), dp);
    });
}

int oracle_pals_metrics(int64_t n, const double* a, const double* b, double thr, double* l2_rel, double* dice,
                        int* flagged) {
    return pguard([&] {
        Metrics m = metrics(std::vector<double>(a, a + n), std::vector<double>(b, b + n), thr);
        *l2_rel = m.l2_rel;
        *dice = m.dice;
        *flagged = m.flagged ? 1 : 0;
    });
}

// trace_out: trace_cap rows of 6 doubles (outer, inner, resnorm, nu,
// accepted, dice); scalars_out: resnorm, converged, flagged, trace_len.
int oracle_pals_reconstruct(const double* U, const double* V, int64_t M, int64_t N, int64_t R, const int* perm,
                            int nx, int ny, int nz, double Lx, double Ly, double Lz, const double* ext, int nl,
                            int nsp, const double* y, const double* w, int np, const double* alpha,
                            const double* beta, const double* centers, double tau, double epsH, double nu,
                            double noise_norm, int max_outer, int max_inner, int max_retries, double gamma,
                            double nu0, double stagnation_tol, const double* fixed_c, const double* mu_truth,
                            double* alpha_out, double* beta_out, double* centers_out, double* c_out,
                            double* trace_out, int trace_cap, double* scalars_out) {
    return pguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        if (g.N() != N) throw std::invalid_argument("reconstruct: grid / operator size mismatch");
        Hop H{U, V, M, N, R, perm};
        ReconCfg cfg;
        cfg.max_outer = max_outer;
        cfg.max_inner = max_inner;
        cfg.max_retries = max_retries;
        cfg.gamma = gamma;
        cfg.nu0 = nu0;
        cfg.stagnation_tol = stagnation_tol;
        if (fixed_c) cfg.fixed_c.assign(fixed_c, fixed_c + nsp);
        std::vector<double> mt;
        if (mu_truth) mt.assign(mu_truth, mu_truth + N);
        Recon r = reconstruct(std::vector<double>(y, y + M), H, g, ext, nl, nsp,
                              make_params(np, alpha, beta, centers, tau, epsH, nu), std::vector<double>(w, w + M),
                              noise_norm, cfg, mu_truth ? &mt : nullptr);
        std::copy(r.p.alpha.begin(), r.p.alpha.end(), alpha_out);
        std::copy(r.p.beta.begin(), r.p.beta.end(), beta_out);
        std::copy(r.p.centers.begin(), r.p.centers.end(), centers_out);
        std::copy(r.c.begin(), r.c.end(), c_out);
        const int len = int(r.trace.size());
        for (int i = 0; i < std::min(len, trace_cap); ++i) {
            const TraceRow& t = r.trace[size_t(i)];
            double* o = trace_out + 6 * i;
            o[0] = t.outer;
            o[1] = t.inner;
            o[2] = t.resnorm;
            o[3] = t.nu;
            o[4] = t.accepted;
            o[5] = t.dice;
        }
        scalars_out[0] = r.resnorm;
        scalars_out[1] = r.converged ? 1 : 0;
        scalars_out[2] = r.flagged ? 1 : 0;
        scalars_out[3] = len;
    });
}

}  // extern "C"
