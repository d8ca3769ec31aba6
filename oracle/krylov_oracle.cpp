// krylov_oracle.cpp -- CPU ORACLE (test infrastructure only).
//
// Restatement of the reference's recycled shifted-family solver
// (/root/reference/proj/src/krylov.cpp, header include/hydot/krylov.hpp):
//   transform_family   krylov.cpp:286-309   Ks = M^-1/2 (K + sbar' R) M^-1/2, Rs = M^-1/2 R M^-1/2
//   orthogonalize      krylov.cpp:21-29     modified Gram-Schmidt, two passes
//   hessenberg_ls      krylov.cpp:33-41     HouseholderQR least squares of min |beta e1 - Tbar y|
//   multishift_gmres   krylov.cpp:45-104    one Arnoldi basis for every shift, convergence test every 10 steps
//   harmonic_ritz      krylov.cpp:106-168   Tbar^T Tbar z = theta T_n^T z, k smallest |theta|
//   build_deflation_basis krylov.cpp:170-213 K U = C, C^T C = I (QR of Cp, trailing-column drop)
//   ShiftedDeflation   krylov.cpp:215-283   C_j = C'_j F^-1 via the Gram/Cholesky update (QR fallback)
//   augmented_gmres    krylov.cpp:311-398   deflated GMRES(m - k) with restarts
//   solve_family       krylov.cpp:400-463   the pipeline, per-shift parallel
// on the reference's FEM operator (fem_oracle.cpp: K, lumped M, R assembled
// as CSR from the same element matrices and triplet order as grid.cpp:112-174).
// Eigen's dense kernels are replaced by LAPACK from scipy's OpenBLAS:
// HouseholderQR -> dgeqrf/dormqr/dorgqr, GeneralizedEigenSolver -> dggev,
// LLT -> dpotrf, FullPivLU::rank -> the singular values of dgesdd at Eigen's
// threshold (eps * n relative to the largest).  Parity of these pieces with
// Eigen is by bounds (the reference's own test_krylov.cpp checks, restated in
// tests/test_krylov_oracle.py), not bitwise.
// Used only by tests/ (and nothing in the product) as the checker of
// csrc/gmres.cu.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fem_oracle.h"

extern "C" {
void scipy_dgeqrf_(const int*, const int*, double*, const int*, double*, double*, const int*, int*);
void scipy_dormqr_(const char*, const char*, const int*, const int*, const int*, const double*, const int*,
                   const double*, double*, const int*, double*, const int*, int*);
void scipy_dorgqr_(const int*, const int*, const int*, double*, const int*, const double*, double*, const int*,
                   int*);
void scipy_dggev_(const char*, const char*, const int*, double*, const int*, double*, const int*, double*,
                  double*, double*, double*, const int*, double*, const int*, double*, const int*, int*);
void scipy_dpotrf_(const char*, const int*, double*, const int*, int*);
void scipy_dgesdd_(const char*, const int*, const int*, double*, const int*, double*, double*, const int*,
                   double*, const int*, double*, const int*, int*, int*);
}

namespace krylov_oracle {

using fem_oracle::Geom;
using Vec = std::vector<double>;

// column-major dense matrix
struct Mat {
    int64_t r = 0, c = 0;
    Vec d;
    Mat() = default;
    Mat(int64_t rows, int64_t cols) : r(rows), c(cols), d(size_t(rows * cols), 0.0) {}
    double& operator()(int64_t i, int64_t j) { return d[size_t(i + j * r)]; }
    double operator()(int64_t i, int64_t j) const { return d[size_t(i + j * r)]; }
    double* col(int64_t j) { return d.data() + j * r; }
    const double* col(int64_t j) const { return d.data() + j * r; }
};

double dot(const double* a, const double* b, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
double nrm(const double* a, int64_t n) { return std::sqrt(dot(a, a, n)); }

// A (m x k) * B (k x n)
Mat mul(const Mat& A, const Mat& B) {
    Mat C(A.r, B.c);
    for (int64_t j = 0; j < B.c; ++j)
        for (int64_t l = 0; l < A.c; ++l) {
            const double b = B(l, j);
            if (b == 0.0) continue;
            const double* a = A.col(l);
            double* c = C.col(j);
            for (int64_t i = 0; i < A.r; ++i) c[i] += a[i] * b;
        }
    return C;
}
// A^T (k x m) * B (m x n)
Mat tmul(const Mat& A, const Mat& B) {
    Mat C(A.c, B.c);
    for (int64_t j = 0; j < B.c; ++j)
        for (int64_t i = 0; i < A.c; ++i) C(i, j) = dot(A.col(i), B.col(j), A.r);
    return C;
}
Mat left_cols(const Mat& A, int64_t k) {
    Mat B(A.r, k);
    std::copy(A.d.begin(), A.d.begin() + A.r * k, B.d.begin());
    return B;
}
Mat top_left(const Mat& A, int64_t r, int64_t c) {
    Mat B(r, c);
    for (int64_t j = 0; j < c; ++j)
        for (int64_t i = 0; i < r; ++i) B(i, j) = A(i, j);
    return B;
}

// CSR matrix (Eigen RowMajor SpMat; duplicates summed in insertion order)
struct Csr {
    int64_t n = 0;
    std::vector<int64_t> rp, ci;
    Vec v;
    void mv(const double* x, double* y) const {
        for (int64_t i = 0; i < n; ++i) {
            double s = 0.0;
            for (int64_t e = rp[size_t(i)]; e < rp[size_t(i + 1)]; ++e) s += v[size_t(e)] * x[ci[size_t(e)]];
            y[i] = s;
        }
    }
    double diag(int64_t i) const {
        for (int64_t e = rp[size_t(i)]; e < rp[size_t(i + 1)]; ++e)
            if (ci[size_t(e)] == i) return v[size_t(e)];
        return 0.0;
    }
};

struct Trip {
    int64_t r, c;
    double v;
};

Csr from_triplets(int64_t n, std::vector<Trip>& t) {
    std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
        return a.r != b.r ? a.r < b.r : a.c < b.c;
    });
    Csr m;
    m.n = n;
    m.rp.assign(static_cast<size_t>(n + 1), 0);
    for (size_t e = 0; e < t.size();) {
        size_t f = e;
        double s = t[e].v;
        while (++f < t.size() && t[f].r == t[e].r && t[f].c == t[e].c) s += t[f].v;
        m.ci.push_back(t[e].c);
        m.v.push_back(s);
        m.rp[size_t(t[e].r + 1)]++;
        e = f;
    }
    for (int64_t i = 0; i < n; ++i) m.rp[size_t(i + 1)] += m.rp[size_t(i)];
    return m;
}

// sum of two CSR matrices with a scale on the second (Kc = K + SpMat(s R))
Csr add_scaled(const Csr& A, const Csr& B, double s) {
    std::vector<Trip> t;
    for (int64_t i = 0; i < A.n; ++i) {
        for (int64_t e = A.rp[size_t(i)]; e < A.rp[size_t(i + 1)]; ++e) t.push_back({i, A.ci[size_t(e)], A.v[size_t(e)]});
        for (int64_t e = B.rp[size_t(i)]; e < B.rp[size_t(i + 1)]; ++e)
            t.push_back({i, B.ci[size_t(e)], s * B.v[size_t(e)]});
    }
    return from_triplets(A.n, t);
}

Csr scale_both(const Csr& A, const Vec& d) {  // D * A * D = (d_i a_ij) d_j
    Csr m = A;
    for (int64_t i = 0; i < A.n; ++i)
        for (int64_t e = A.rp[size_t(i)]; e < A.rp[size_t(i + 1)]; ++e)
            m.v[size_t(e)] = (d[size_t(i)] * A.v[size_t(e)]) * d[size_t(A.ci[size_t(e)])];
    return m;
}

// grid.cpp:112-174: K (Dirichlet eliminated, unit diagonal), lumped M, R
void assemble(const Geom& g, Csr& K, Vec& Mdiag, Csr& R) {
    const int64_t N = g.N();
    double Ke[64], Me[64], Re[16];
    fem_oracle::element(g.hx, g.hy, g.hz, Ke, Me, Re);
    std::vector<Trip> tk, tr;
    Mdiag.assign(static_cast<size_t>(N), 0.0);
    for (int cz = 0; cz < g.nz - 1; ++cz)
        for (int cy = 0; cy < g.ny - 1; ++cy)
            for (int cx = 0; cx < g.nx - 1; ++cx) {
                int64_t v[8];
                bool d[8];
                for (int a = 0; a < 8; ++a) {
                    const int jx = cx + (a & 1), jy = cy + ((a >> 1) & 1), jz = cz + ((a >> 2) & 1);
                    v[a] = g.idx(jx, jy, jz);
                    d[a] = g.dir(jx, jy);
                }
                for (int a = 0; a < 8; ++a) {
                    if (d[a]) continue;
                    for (int b = 0; b < 8; ++b)
                        if (!d[b]) tk.push_back({v[a], v[b], Ke[a * 8 + b]});
                }
                for (int a = 0; a < 8; ++a)
                    for (int b = 0; b < 8; ++b) Mdiag[size_t(v[a])] += Me[a * 8 + b];
            }
    for (int iz = 0; iz < g.nz; ++iz)
        for (int iy = 0; iy < g.ny; ++iy)
            for (int ix = 0; ix < g.nx; ++ix)
                if (g.dir(ix, iy)) tk.push_back({g.idx(ix, iy, iz), g.idx(ix, iy, iz), 1.0});
    for (int iz : {0, g.nz - 1})
        for (int cy = 0; cy < g.ny - 1; ++cy)
            for (int cx = 0; cx < g.nx - 1; ++cx) {
                int64_t v[4];
                for (int a = 0; a < 4; ++a) v[a] = g.idx(cx + (a & 1), cy + ((a >> 1) & 1), iz);
                for (int a = 0; a < 4; ++a)
                    for (int b = 0; b < 4; ++b) tr.push_back({v[a], v[b], Re[a * 4 + b]});
            }
    K = from_triplets(N, tk);
    R = from_triplets(N, tr);
}

// TransformedFamily (krylov.hpp:112-121, krylov.cpp:286-309)
struct Family {
    Csr Ks, Rs;
    Vec minv_sqrt;
    double sbar = 0.0;
    void apply(double sigma, double sp, const double* x, double* y) const {
        const int64_t N = Ks.n;
        Vec t(static_cast<size_t>(N));
        Ks.mv(x, y);
        Rs.mv(x, t.data());
        for (int64_t i = 0; i < N; ++i) y[i] = (y[i] + sigma * x[i]) + sp * t[size_t(i)];
    }
};

Family transform_family(const Geom& g, double sbar) {
    Csr K, R;
    Vec Md;
    assemble(g, K, Md, R);
    Family f;
    for (double d : Md)
        if (d <= 0) throw std::invalid_argument("transform_family: lumped mass diagonal must be positive");
    f.minv_sqrt.resize(Md.size());
    for (size_t i = 0; i < Md.size(); ++i) f.minv_sqrt[i] = 1.0 / std::sqrt(Md[i]);
    Csr Kc = sbar != 0.0 ? add_scaled(K, R, sbar) : K;
    f.Ks = scale_both(Kc, f.minv_sqrt);
    f.Rs = scale_both(R, f.minv_sqrt);
    f.sbar = sbar;
    return f;
}

// krylov.cpp:21-29
void orthogonalize(const Mat& V, int ncols, double* w, Vec& h) {
    h.assign(static_cast<size_t>(ncols), 0.0);
    for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j < ncols; ++j) {
            const double c = dot(V.col(j), w, V.r);
            const double* v = V.col(j);
            for (int64_t i = 0; i < V.r; ++i) w[i] -= c * v[i];
            h[size_t(j)] += c;
        }
}

// Householder QR of A (m x n, m >= n) in place; returns tau
Vec geqrf(Mat& A) {
    const int M = int(A.r), N = int(A.c), lda = std::max(1, M);
    Vec tau(size_t(std::max(1, N)));
    int info = 0, lw = -1;
    double wq = 0;
    scipy_dgeqrf_(&M, &N, A.d.data(), &lda, tau.data(), &wq, &lw, &info);
    lw = std::max(1, int(wq));
    Vec work(static_cast<size_t>(lw));
    scipy_dgeqrf_(&M, &N, A.d.data(), &lda, tau.data(), work.data(), &lw, &info);
    if (info != 0) throw std::runtime_error("dgeqrf failed");
    return tau;
}

// Q^T b for the QR held in (A, tau)
void ormqr_t(const Mat& A, const Vec& tau, double* b) {
    const int M = int(A.r), N = 1, K = int(A.c), lda = std::max(1, M), ldc = std::max(1, M);
    int info = 0, lw = -1;
    double wq = 0;
    scipy_dormqr_("L", "T", &M, &N, &K, A.d.data(), &lda, tau.data(), b, &ldc, &wq, &lw, &info);
    lw = std::max(1, int(wq));
    Vec work(static_cast<size_t>(lw));
    scipy_dormqr_("L", "T", &M, &N, &K, A.d.data(), &lda, tau.data(), b, &ldc, work.data(), &lw, &info);
    if (info != 0) throw std::runtime_error("dormqr failed");
}

// the first k columns of Q
Mat orgqr(const Mat& A, const Vec& tau, int k) {
    Mat Q(A.r, k);
    std::copy(A.d.begin(), A.d.begin() + A.r * k, Q.d.begin());
    const int M = int(A.r), N = k, lda = std::max(1, M);
    int info = 0, lw = -1;
    double wq = 0;
    scipy_dorgqr_(&M, &N, &N, Q.d.data(), &lda, tau.data(), &wq, &lw, &info);
    lw = std::max(1, int(wq));
    Vec work(static_cast<size_t>(lw));
    scipy_dorgqr_(&M, &N, &N, Q.d.data(), &lda, tau.data(), work.data(), &lw, &info);
    if (info != 0) throw std::runtime_error("dorgqr failed");
    return Q;
}

// krylov.cpp:33-41
Vec hessenberg_ls(const Mat& Tbar, int s, double beta, double& resnorm) {
    Mat A = top_left(Tbar, s + 1, s);
    Vec rhs(static_cast<size_t>(s + 1), 0.0);
    rhs[0] = beta;
    Mat qr = A;
    Vec tau = geqrf(qr);
    Vec qtb = rhs;
    ormqr_t(qr, tau, qtb.data());
    Vec y(static_cast<size_t>(s), 0.0);
    for (int i = s - 1; i >= 0; --i) {  // R y = (Q^T rhs)[0:s]
        double t = qtb[size_t(i)];
        for (int j = i + 1; j < s; ++j) t -= qr(i, j) * y[size_t(j)];
        y[size_t(i)] = t / qr(i, i);
    }
    double r2 = 0.0;
    for (int i = 0; i <= s; ++i) {
        double t = rhs[size_t(i)];
        for (int j = 0; j < s; ++j) t -= A(i, j) * y[size_t(j)];
        r2 += t * t;
    }
    resnorm = std::sqrt(r2);
    return y;
}

struct Arnoldi {
    Mat V, T;
    double beta = 0.0;
    int steps = 0;
    bool breakdown = false;
};

struct Multishift {
    Mat X;
    Vec relres;
    Arnoldi a;
};

// krylov.cpp:45-104
Multishift multishift_gmres(const Csr& Ks, const Vec& b, const Vec& sigmas, int n, double tol) {
    const int64_t N = int64_t(b.size());
    const double bnorm = nrm(b.data(), N);
    if (bnorm == 0.0) throw std::invalid_argument("multishift_gmres: b must be nonzero");
    n = int(std::min<int64_t>(n, N));
    Arnoldi a;
    a.V = Mat(N, n + 1);
    a.T = Mat(n + 1, n);
    a.beta = bnorm;
    for (int64_t i = 0; i < N; ++i) a.V(i, 0) = b[size_t(i)] / bnorm;
    auto all_converged = [&](int s) {
        for (double sigma : sigmas) {
            Mat Ts = top_left(a.T, s + 1, s);
            for (int i = 0; i < s; ++i) Ts(i, i) += sigma;
            double rn;
            hessenberg_ls(Ts, s, bnorm, rn);
            if (rn / bnorm > tol) return false;
        }
        return true;
    };
    int steps = 0;
    Vec w(static_cast<size_t>(N)), h;
    for (int i = 0; i < n; ++i) {
        Ks.mv(a.V.col(i), w.data());
        orthogonalize(a.V, i + 1, w.data(), h);
        for (int j = 0; j <= i; ++j) a.T(j, i) = h[size_t(j)];
        const double hnext = nrm(w.data(), N);
        a.T(i + 1, i) = hnext;
        steps = i + 1;
        if (hnext <= 1e-14 * bnorm) {
            a.breakdown = true;
            break;
        }
        for (int64_t r = 0; r < N; ++r) a.V(r, i + 1) = w[size_t(r)] / hnext;
        if ((i + 1) % 10 == 0 && all_converged(i + 1)) break;
    }
    a.steps = steps;
    a.V = left_cols(a.V, steps + 1);
    a.T = top_left(a.T, steps + 1, steps);
    Multishift res;
    const int ns = int(sigmas.size());
    res.X = Mat(N, ns);
    res.relres.resize(static_cast<size_t>(ns));
    for (int j = 0; j < ns; ++j) {
        Mat Ts = a.T;
        for (int i = 0; i < steps; ++i) Ts(i, i) += sigmas[size_t(j)];
        double rn;
        Vec y = hessenberg_ls(Ts, steps, bnorm, rn);
        for (int c = 0; c < steps; ++c) {
            const double* v = a.V.col(c);
            double* x = res.X.col(j);
            for (int64_t r = 0; r < N; ++r) x[r] += v[r] * y[size_t(c)];
        }
        res.relres[size_t(j)] = rn / bnorm;
    }
    res.a = std::move(a);
    return res;
}

struct HarmonicRitz {
    Mat Z;
    Vec theta;
    bool pencil_shifted = false;
};

// krylov.cpp:106-168
HarmonicRitz harmonic_ritz(const Mat& Tbar, int n, int k) {
    if (k > n) throw std::invalid_argument("harmonic_ritz: k > Arnoldi steps");
    Mat Tn = top_left(Tbar, n, n);
    Mat A = tmul(Tbar, Tbar);
    Mat B(n, n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) B(i, j) = Tn(j, i);
    HarmonicRitz hr;
    {  // FullPivLU(B).rank() < n  <=>  smallest singular value below eps * n * largest
        Mat S = B;
        Vec s(static_cast<size_t>(n));
        int info = 0, lw = -1, ldu = 1;
        std::vector<int> iw(size_t(8 * n));
        double wq = 0, du = 0;
        const int lda = n;
        scipy_dgesdd_("N", &n, &n, S.d.data(), &lda, s.data(), &du, &ldu, &du, &ldu, &wq, &lw, iw.data(), &info);
        lw = std::max(1, int(wq));
        Vec work(static_cast<size_t>(lw));
        scipy_dgesdd_("N", &n, &n, S.d.data(), &lda, s.data(), &du, &ldu, &du, &ldu, work.data(), &lw, iw.data(),
                      &info);
        if (info != 0) throw std::runtime_error("dgesdd failed");
        const double thr = std::numeric_limits<double>::epsilon() * n * s[0];
        int rank = 0;
        for (double v : s) rank += v > thr;
        if (rank < n) {
            double fro = 0.0;
            for (double v : Tn.d) fro += v * v;
            const double shift = std::numeric_limits<double>::epsilon() * std::sqrt(fro);
            for (int i = 0; i < n; ++i) B(i, i) += shift;
            hr.pencil_shifted = true;
        }
    }
    Vec ar(static_cast<size_t>(n)), ai(static_cast<size_t>(n)), be(static_cast<size_t>(n));
    Mat VR(n, n);
    {
        Mat A2 = A, B2 = B;
        int info = 0, lw = -1, one = 1;
        double wq = 0, dl = 0;
        scipy_dggev_("N", "V", &n, A2.d.data(), &n, B2.d.data(), &n, ar.data(), ai.data(), be.data(), &dl, &one,
                     VR.d.data(), &n, &wq, &lw, &info);
        lw = std::max(1, int(wq));
        Vec work(static_cast<size_t>(lw));
        scipy_dggev_("N", "V", &n, A2.d.data(), &n, B2.d.data(), &n, ar.data(), ai.data(), be.data(), &dl, &one,
                     VR.d.data(), &n, work.data(), &lw, &info);
        if (info != 0) throw std::runtime_error("dggev failed");
    }
    std::vector<std::complex<double>> theta(static_cast<size_t>(n));
    std::vector<std::vector<std::complex<double>>> Z(static_cast<size_t>(n), std::vector<std::complex<double>>(size_t(n)));
    for (int j = 0; j < n; ++j) {
        theta[size_t(j)] = std::complex<double>(ar[size_t(j)], ai[size_t(j)]) / be[size_t(j)];
        if (ai[size_t(j)] == 0.0) {
            for (int i = 0; i < n; ++i) Z[size_t(j)][size_t(i)] = VR(i, j);
        } else if (ai[size_t(j)] > 0.0 && j + 1 < n) {  // pair (j, j+1): VR(:,j) +- i VR(:,j+1)
            for (int i = 0; i < n; ++i) {
                Z[size_t(j)][size_t(i)] = {VR(i, j), VR(i, j + 1)};
                Z[size_t(j + 1)][size_t(i)] = {VR(i, j), -VR(i, j + 1)};
            }
        }
    }
    std::vector<int> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(),
              [&](int i, int j) { return std::abs(theta[size_t(i)]) < std::abs(theta[size_t(j)]); });
    hr.Z = Mat(n, k);
    hr.theta.assign(static_cast<size_t>(k), 0.0);
    std::vector<bool> used(static_cast<size_t>(n), false);
    int col = 0;
    for (int idx : order) {
        if (col >= k) break;
        if (used[size_t(idx)]) continue;
        used[size_t(idx)] = true;
        const auto& z = Z[size_t(idx)];
        double re2 = 0, im2 = 0;
        for (auto& c : z) {
            re2 += c.real() * c.real();
            im2 += c.imag() * c.imag();
        }
        if (std::sqrt(im2) > 1e-12 * std::sqrt(re2)) {
            for (int i = 0; i < n; ++i) hr.Z(i, col) = z[size_t(i)].real();
            hr.theta[size_t(col)] = std::abs(theta[size_t(idx)]);
            ++col;
            for (int other : order)
                if (!used[size_t(other)] &&
                    std::abs(theta[size_t(other)] - std::conj(theta[size_t(idx)])) <=
                        1e-10 * (1.0 + std::abs(theta[size_t(idx)]))) {
                    used[size_t(other)] = true;
                    break;
                }
            if (col < k) {
                for (int i = 0; i < n; ++i) hr.Z(i, col) = z[size_t(i)].imag();
                hr.theta[size_t(col)] = std::abs(theta[size_t(idx)]);
                ++col;
            }
        } else {
            for (int i = 0; i < n; ++i) hr.Z(i, col) = z[size_t(i)].real();
            hr.theta[size_t(col)] = std::abs(theta[size_t(idx)]);
            ++col;
        }
    }
    for (int c = 0; c < k; ++c) {
        const double nz = nrm(hr.Z.col(c), n);
        if (nz > 0)
            for (int i = 0; i < n; ++i) hr.Z(i, c) /= nz;
    }
    return hr;
}

struct Deflation {
    Mat U, C, RU, UtC, CtRU, RUtU, UtU, RUtRU;
    int k = 0;
    bool rank_reduced = false;
};

// krylov.cpp:170-213
Deflation build_deflation_basis(const Family& fam, const Arnoldi& a, const Mat& Zall) {
    const int n = a.steps;
    int k = int(Zall.c);
    const int64_t N = a.V.r;
    Deflation basis;
    while (k > 0) {
        Mat Zk = left_cols(Zall, k);
        Mat Ut = mul(left_cols(a.V, n), Zk);
        Mat Cp = mul(a.V, mul(a.T, Zk));
        Mat qr = Cp;
        Vec tau = geqrf(qr);
        double dmax = 0.0;
        for (int i = 0; i < k; ++i) dmax = std::max(dmax, std::abs(qr(i, i)));
        bool ok = true;
        for (int i = 0; i < k; ++i)
            if (std::abs(qr(i, i)) < 1e-12 * dmax) ok = false;
        if (!ok) {
            --k;
            basis.rank_reduced = true;
            continue;
        }
        basis.C = orgqr(qr, tau, k);
        basis.U = Mat(N, k);  // U = Ut Y^-1, row by row: u Y = ut
        for (int64_t r = 0; r < N; ++r)
            for (int j = 0; j < k; ++j) {
                double t = Ut(r, j);
                for (int l = 0; l < j; ++l) t -= basis.U(r, l) * qr(l, j);
                basis.U(r, j) = t / qr(j, j);
            }
        break;
    }
    basis.k = k;
    if (k == 0) return basis;
    basis.RU = Mat(N, k);
    for (int j = 0; j < k; ++j) fam.Rs.mv(basis.U.col(j), basis.RU.col(j));
    basis.UtC = tmul(basis.U, basis.C);
    basis.CtRU = tmul(basis.C, basis.RU);
    basis.RUtU = tmul(basis.RU, basis.U);
    basis.UtU = tmul(basis.U, basis.U);
    basis.RUtRU = tmul(basis.RU, basis.RU);
    return basis;
}

// ShiftedDeflation (krylov.hpp:83-107, krylov.cpp:215-283)
struct Shifted {
    const Deflation* base = nullptr;
    double sigma = 0, sp = 0;
    Mat F, Cx, Ux;
    bool expl = false, chol_failed = false;
    int dim() const { return base ? base->k : 0; }

    Shifted() = default;
    Shifted(const Deflation& b, double s, double spr, bool force_qr) : base(&b), sigma(s), sp(spr) {
        const int k = b.k;
        if (k == 0) {
            base = nullptr;
            return;
        }
        if (!force_qr) {
            Mat g(k, k);
            for (int i = 0; i < k; ++i) g(i, i) = 1.0;
            for (int j = 0; j < k; ++j)
                for (int i = 0; i < k; ++i) g(i, j) += sigma * (b.UtC(i, j) + b.UtC(j, i));
            for (int j = 0; j < k; ++j)
                for (int i = 0; i < k; ++i) g(i, j) += sp * (b.CtRU(i, j) + b.CtRU(j, i));
            for (int j = 0; j < k; ++j)
                for (int i = 0; i < k; ++i) g(i, j) += sigma * sp * (b.RUtU(i, j) + b.RUtU(j, i));
            for (int j = 0; j < k; ++j)
                for (int i = 0; i < k; ++i) g(i, j) += sigma * sigma * b.UtU(i, j);
            for (int j = 0; j < k; ++j)
                for (int i = 0; i < k; ++i) g(i, j) += sp * sp * b.RUtRU(i, j);
            int info = 0;
            scipy_dpotrf_("U", &k, g.d.data(), &k, &info);
            if (info == 0) {
                F = Mat(k, k);
                for (int j = 0; j < k; ++j)
                    for (int i = 0; i <= j; ++i) F(i, j) = g(i, j);
                return;
            }
            chol_failed = true;
        }
        expl = true;
        const int64_t N = b.U.r;
        Mat Cp(N, k);
        for (int64_t e = 0; e < N * k; ++e)
            Cp.d[size_t(e)] = (b.C.d[size_t(e)] + sigma * b.U.d[size_t(e)]) + sp * b.RU.d[size_t(e)];
        Vec tau = geqrf(Cp);
        Cx = orgqr(Cp, tau, k);
        Ux = Mat(N, k);
        for (int64_t r = 0; r < N; ++r)
            for (int j = 0; j < k; ++j) {
                double t = b.U(r, j);
                for (int l = 0; l < j; ++l) t -= Ux(r, l) * Cp(l, j);
                Ux(r, j) = t / Cp(j, j);
            }
    }
    // F^{-1} w (upper) and F^{-T} t (lower)
    Vec solve_F(const Vec& w) const {
        const int k = dim();
        Vec s(w);
        for (int i = k - 1; i >= 0; --i) {
            double t = s[size_t(i)];
            for (int j = i + 1; j < k; ++j) t -= F(i, j) * s[size_t(j)];
            s[size_t(i)] = t / F(i, i);
        }
        return s;
    }
    Vec solve_Ft(const Vec& t) const {
        const int k = dim();
        Vec s(t);
        for (int i = 0; i < k; ++i) {
            double v = s[size_t(i)];
            for (int j = 0; j < i; ++j) v -= F(j, i) * s[size_t(j)];
            s[size_t(i)] = v / F(i, i);
        }
        return s;
    }
    Vec apply_Ct(const double* v) const {
        const int k = dim();
        const int64_t N = base->U.r;
        Vec t(static_cast<size_t>(k));
        if (expl) {
            for (int j = 0; j < k; ++j) t[size_t(j)] = dot(Cx.col(j), v, N);
            return t;
        }
        for (int j = 0; j < k; ++j)
            t[size_t(j)] = (dot(base->C.col(j), v, N) + sigma * dot(base->U.col(j), v, N)) +
                           sp * dot(base->RU.col(j), v, N);
        return solve_Ft(t);
    }
    void add_C(const Vec& w, double* out, double alpha) const {  // out += alpha * C_j w
        const int k = dim();
        const int64_t N = base->U.r;
        if (expl) {
            for (int j = 0; j < k; ++j)
                for (int64_t r = 0; r < N; ++r) out[r] += alpha * (Cx(r, j) * w[size_t(j)]);
            return;
        }
        Vec s = solve_F(w);
        Vec y(static_cast<size_t>(N), 0.0);
        for (int j = 0; j < k; ++j)
            for (int64_t r = 0; r < N; ++r)
                y[size_t(r)] += (base->C(r, j) * s[size_t(j)] + sigma * (base->U(r, j) * s[size_t(j)])) +
                                sp * (base->RU(r, j) * s[size_t(j)]);
        for (int64_t r = 0; r < N; ++r) out[r] += alpha * y[size_t(r)];
    }
    void add_U(const Vec& w, double* out, double alpha) const {  // out += alpha * U_j w
        const int k = dim();
        const int64_t N = base->U.r;
        const Mat& Uu = expl ? Ux : base->U;
        Vec s = expl ? w : solve_F(w);
        for (int j = 0; j < k; ++j)
            for (int64_t r = 0; r < N; ++r) out[r] += alpha * (Uu(r, j) * s[size_t(j)]);
    }
};

struct Stats {
    int iterations = 0, matvecs = 0;
    double relres = 0.0;
    bool converged = false;
};

// krylov.cpp:311-398
Vec augmented_gmres(const Family& fam, double sigma, double sp, const Vec& b, const Shifted& defl, const Vec& x0,
                    int m, double tol, int max_restarts, Stats& st, const Vec* pdiag) {
    const int64_t N = int64_t(b.size());
    const int k = defl.dim();
    const int inner = std::max(1, m - k);
    const double bnorm = nrm(b.data(), N);
    if (bnorm == 0.0) throw std::invalid_argument("augmented_gmres: b must be nonzero");
    Vec pinv;
    if (pdiag) {
        pinv.resize(pdiag->size());
        for (size_t i = 0; i < pinv.size(); ++i) pinv[i] = 1.0 / (*pdiag)[i];
    }
    auto applyA = [&](const double* v, double* y) {
        ++st.matvecs;
        fam.apply(sigma, sp, v, y);
    };
    auto applyB = [&](const double* v, double* y) {
        if (!pdiag) return applyA(v, y);
        Vec t(static_cast<size_t>(N));
        for (int64_t i = 0; i < N; ++i) t[size_t(i)] = pinv[size_t(i)] * v[i];
        applyA(t.data(), y);
    };
    Vec x = x0, r(static_cast<size_t>(N)), t(static_cast<size_t>(N));
    applyA(x.data(), t.data());
    for (int64_t i = 0; i < N; ++i) r[size_t(i)] = b[size_t(i)] - t[size_t(i)];
    auto deflate = [&](Vec& xi, Vec& ri) {
        if (k == 0) return;
        Vec z = defl.apply_Ct(ri.data());
        defl.add_U(z, xi.data(), 1.0);
        defl.add_C(z, ri.data(), -1.0);
    };
    deflate(x, r);
    st.relres = nrm(r.data(), N) / bnorm;
    for (int cycle = 0; cycle <= max_restarts; ++cycle) {
        if (st.relres <= tol) {
            st.converged = true;
            break;
        }
        const double beta = nrm(r.data(), N);
        Mat V(N, inner + 1), Tbar(inner + 1, inner), Fk(std::max(k, 0), inner);
        for (int64_t i = 0; i < N; ++i) V(i, 0) = r[size_t(i)] / beta;
        int steps = 0;
        bool lucky = false;
        double lsres = beta;
        Vec w(static_cast<size_t>(N)), h;
        for (int i = 0; i < inner; ++i) {
            applyB(V.col(i), w.data());
            if (k > 0) {
                Vec c = defl.apply_Ct(w.data());
                for (int j = 0; j < k; ++j) Fk(j, i) = c[size_t(j)];
                defl.add_C(c, w.data(), -1.0);
            }
            orthogonalize(V, i + 1, w.data(), h);
            for (int j = 0; j <= i; ++j) Tbar(j, i) = h[size_t(j)];
            const double hnext = nrm(w.data(), N);
            Tbar(i + 1, i) = hnext;
            steps = i + 1;
            hessenberg_ls(Tbar, steps, beta, lsres);
            if (hnext <= 1e-14 * beta) {
                lucky = true;
                break;
            }
            for (int64_t r2 = 0; r2 < N; ++r2) V(r2, i + 1) = w[size_t(r2)] / hnext;
            if (lsres / bnorm <= tol) break;
        }
        st.iterations += steps;
        double resnorm;
        Vec y2 = hessenberg_ls(Tbar, steps, beta, resnorm);
        Vec dx(static_cast<size_t>(N), 0.0);
        for (int c = 0; c < steps; ++c)
            for (int64_t i = 0; i < N; ++i) dx[size_t(i)] += V(i, c) * y2[size_t(c)];
        if (pdiag)
            for (int64_t i = 0; i < N; ++i) dx[size_t(i)] = pinv[size_t(i)] * dx[size_t(i)];
        if (k > 0) {
            Vec fy(static_cast<size_t>(k), 0.0);
            for (int j = 0; j < k; ++j)
                for (int c = 0; c < steps; ++c) fy[size_t(j)] += Fk(j, c) * y2[size_t(c)];
            for (auto& v : fy) v = -v;
            defl.add_U(fy, x.data(), 1.0);
        }
        for (int64_t i = 0; i < N; ++i) x[size_t(i)] += dx[size_t(i)];
        applyA(x.data(), t.data());
        for (int64_t i = 0; i < N; ++i) r[size_t(i)] = b[size_t(i)] - t[size_t(i)];
        st.relres = nrm(r.data(), N) / bnorm;
        if (st.relres <= tol || lucky) {
            st.converged = st.relres <= tol;
            break;
        }
        deflate(x, r);
    }
    return x;
}

struct Config {
    int arnoldi_steps = 80, deflation_dim = 10, restart = 50, max_restarts = 40;
    double tol = 1e-8;
    bool center_shifts = true, jacobi = false, explicit_qr_update = false;
    int threads = 1;
};

struct FamilyOut {
    int phase1_steps = 0, defl_k = 0;
    bool rank_reduced = false, pencil_shifted = false, breakdown = false;
    bool all_converged = true;
    int first_failure = -1;
};

// krylov.cpp:400-463 (X in original variables, N x nshift)
void solve_family(const Geom& g, const Vec& b, const Vec& sig, const Vec& sigp, const Config& cfg, double* X,
                  std::vector<Stats>& stats, Vec& p1relres, FamilyOut& out) {
    const int ns = int(sig.size());
    if (ns == 0) throw std::invalid_argument("solve_family: no shifts");
    double sbar = 0.0;
    if (cfg.center_shifts) sbar = std::accumulate(sigp.begin(), sigp.end(), 0.0) / ns;
    Family fam = transform_family(g, sbar);
    const int64_t N = g.N();
    Vec bs(static_cast<size_t>(N));
    for (int64_t i = 0; i < N; ++i) bs[size_t(i)] = fam.minv_sqrt[size_t(i)] * b[size_t(i)];
    Multishift p1 = multishift_gmres(fam.Ks, bs, sig, cfg.arnoldi_steps, cfg.tol);
    out.phase1_steps = p1.a.steps;
    out.breakdown = p1.a.breakdown;
    p1relres = p1.relres;
    Deflation basis;
    if (cfg.deflation_dim > 0) {
        const int k = std::min(cfg.deflation_dim, p1.a.steps);
        HarmonicRitz hr = harmonic_ritz(p1.a.T, p1.a.steps, k);
        out.pencil_shifted = hr.pencil_shifted;
        basis = build_deflation_basis(fam, p1.a, hr.Z);
    }
    out.defl_k = basis.k;
    out.rank_reduced = basis.rank_reduced;
    Vec jd;
    if (cfg.jacobi) {
        const double ms = std::accumulate(sig.begin(), sig.end(), 0.0) / ns;
        const double msp = std::accumulate(sigp.begin(), sigp.end(), 0.0) / ns - sbar;
        jd.resize(static_cast<size_t>(N));
        for (int64_t i = 0; i < N; ++i)
            jd[size_t(i)] = std::max(std::abs((fam.Ks.diag(i) + ms) + msp * fam.Rs.diag(i)), 1e-300);
    }
    stats.assign(static_cast<size_t>(ns), Stats{});
    auto work = [&](int j) {
        const double sp = sigp[size_t(j)] - sbar;
        Shifted defl;
        if (basis.k > 0) defl = Shifted(basis, sig[size_t(j)], sp, cfg.explicit_qr_update);
        Vec x0(p1.X.col(j), p1.X.col(j) + N);
        Vec xs = augmented_gmres(fam, sig[size_t(j)], sp, bs, defl, x0, cfg.restart, cfg.tol, cfg.max_restarts,
                                 stats[size_t(j)], cfg.jacobi ? &jd : nullptr);
        for (int64_t i = 0; i < N; ++i) X[int64_t(j) * N + i] = fam.minv_sqrt[size_t(i)] * xs[size_t(i)];
    };
    const int T = std::max(1, std::min(cfg.threads, ns));
    if (T == 1) {
        for (int j = 0; j < ns; ++j) work(j);
    } else {
        std::vector<std::thread> ts;
        for (int t = 0; t < T; ++t)
            ts.emplace_back([&, t] {
                for (int j = t; j < ns; j += T) work(j);
            });
        for (auto& th : ts) th.join();
    }
    for (int j = 0; j < ns; ++j)
        if (!stats[size_t(j)].converged) {
            out.all_converged = false;
            if (out.first_failure < 0) out.first_failure = j;
        }
}

Config make_cfg(const int* ci, double tol) {
    Config c;
    c.arnoldi_steps = ci[0];
    c.deflation_dim = ci[1];
    c.restart = ci[2];
    c.max_restarts = ci[3];
    c.center_shifts = ci[4] != 0;
    c.jacobi = ci[5] != 0;
    c.explicit_qr_update = ci[6] != 0;
    c.threads = ci[7];
    c.tol = tol;
    return c;
}

}  // namespace krylov_oracle

using namespace krylov_oracle;

namespace {
thread_local std::string g_kerr;
template <class F>
int kguard(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_kerr = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_kerr = e.what();
        return 2;
    }
}
void to_mat(Mat& M, const double* p, int64_t r, int64_t c) {
    M = Mat(r, c);
    std::copy(p, p + r * c, M.d.begin());
}
}  // namespace

extern "C" {

const char* oracle_krylov_last_error() { return g_kerr.c_str(); }

// fam.apply(sigma, sp, x) (which = 0) or Rs x (which = 1) of transform_family(K, M, R, sbar)
int oracle_krylov_apply(int nx, int ny, int nz, double Lx, double Ly, double Lz, double sbar, int which,
                        double sigma, double sp, const double* x, double* y, double* minv_sqrt) {
    return kguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        Family f = transform_family(g, sbar);
        if (which == 0)
            f.apply(sigma, sp, x, y);
        else
            f.Rs.mv(x, y);
        if (minv_sqrt) std::copy(f.minv_sqrt.begin(), f.minv_sqrt.end(), minv_sqrt);
    });
}

// phase 1 on transform_family(sbar) with the transformed rhs M^-1/2 b.
// V: N x (n+1), T: (n+1) x n buffers (leading parts filled); info = {steps, breakdown}
int oracle_krylov_multishift(int nx, int ny, int nz, double Lx, double Ly, double Lz, double sbar,
                             const double* b, int nshift, const double* sig, int n, double tol, double* X,
                             double* relres, double* V, double* T, int* info) {
    return kguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        Family f = transform_family(g, sbar);
        const int64_t N = g.N();
        Vec bs(static_cast<size_t>(N));
        for (int64_t i = 0; i < N; ++i) bs[size_t(i)] = f.minv_sqrt[size_t(i)] * b[i];
        Multishift r = multishift_gmres(f.Ks, bs, Vec(sig, sig + nshift), n, tol);
        std::copy(r.X.d.begin(), r.X.d.end(), X);
        std::copy(r.relres.begin(), r.relres.end(), relres);
        const int s = r.a.steps;
        std::copy(r.a.V.d.begin(), r.a.V.d.end(), V);
        for (int j = 0; j < s; ++j)
            for (int i = 0; i <= s; ++i) T[size_t(i + j * (n + 1))] = r.a.T(i, j);
        info[0] = s;
        info[1] = r.a.breakdown ? 1 : 0;
    });
}

// T: (n+1) x n; Z: n x k; info = {pencil_shifted}
int oracle_krylov_harmonic_ritz(int n, const double* T, int k, double* Z, double* theta, int* info) {
    return kguard([&] {
        Mat Tb;
        to_mat(Tb, T, n + 1, n);
        HarmonicRitz hr = harmonic_ritz(Tb, n, k);
        std::copy(hr.Z.d.begin(), hr.Z.d.end(), Z);
        std::copy(hr.theta.begin(), hr.theta.end(), theta);
        info[0] = hr.pencil_shifted ? 1 : 0;
    });
}

// build_deflation_basis from an Arnoldi (V: N x (s+1), T: (s+1) x s) and Z (s x k).
// U, C, RU: N x k buffers; info = {k_out, rank_reduced}
int oracle_krylov_deflation(int nx, int ny, int nz, double Lx, double Ly, double Lz, double sbar, int s,
                            const double* V, const double* T, int k, const double* Z, double* U, double* C,
                            double* RU, int* info) {
    return kguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        Family f = transform_family(g, sbar);
        Arnoldi a;
        to_mat(a.V, V, g.N(), s + 1);
        to_mat(a.T, T, s + 1, s);
        a.steps = s;
        Mat Zm;
        to_mat(Zm, Z, s, k);
        Deflation d = build_deflation_basis(f, a, Zm);
        info[0] = d.k;
        info[1] = d.rank_reduced ? 1 : 0;
        if (d.k > 0) {
            std::copy(d.U.d.begin(), d.U.d.end(), U);
            std::copy(d.C.d.begin(), d.C.d.end(), C);
            std::copy(d.RU.d.begin(), d.RU.d.end(), RU);
        }
    });
}

// dense C_j, U_j of ShiftedDeflation(basis(U, C, RU), sigma, sp, force_qr); info = {cholesky_failed}
int oracle_krylov_shifted_dense(int64_t N, int k, const double* U, const double* C, const double* RU, double sigma,
                                double sp, int force_qr, double* Cj, double* Uj, int* info) {
    return kguard([&] {
        Deflation d;
        to_mat(d.U, U, N, k);
        to_mat(d.C, C, N, k);
        to_mat(d.RU, RU, N, k);
        d.k = k;
        d.UtC = tmul(d.U, d.C);
        d.CtRU = tmul(d.C, d.RU);
        d.RUtU = tmul(d.RU, d.U);
        d.UtU = tmul(d.U, d.U);
        d.RUtRU = tmul(d.RU, d.RU);
        Shifted s(d, sigma, sp, force_qr != 0);
        for (int j = 0; j < k; ++j) {
            Vec e(static_cast<size_t>(k), 0.0);
            e[size_t(j)] = 1.0;
            std::fill(Cj + int64_t(j) * N, Cj + int64_t(j + 1) * N, 0.0);
            std::fill(Uj + int64_t(j) * N, Uj + int64_t(j + 1) * N, 0.0);
            s.add_C(e, Cj + int64_t(j) * N, 1.0);
            s.add_U(e, Uj + int64_t(j) * N, 1.0);
        }
        info[0] = s.chol_failed ? 1 : 0;
    });
}

// solve_family for one right-hand side b (N).  cfgi = {arnoldi_steps,
// deflation_dim, restart, max_restarts, center_shifts, jacobi,
// explicit_qr_update, threads}.  X: N x nshift; info = {phase1_steps, defl_k,
// rank_reduced, pencil_shifted, breakdown, all_converged, first_failure}
int oracle_krylov_solve_family(int nx, int ny, int nz, double Lx, double Ly, double Lz, const double* b,
                               int nshift, const double* sig, const double* sigp, const int* cfgi, double tol,
                               double* X, int* iters, int* matvecs, double* relres, int* converged,
                               double* p1relres, int* info) {
    return kguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        Config cfg = make_cfg(cfgi, tol);
        std::vector<Stats> st;
        Vec p1;
        FamilyOut o;
        solve_family(g, Vec(b, b + g.N()), Vec(sig, sig + nshift), Vec(sigp, sigp + nshift), cfg, X, st, p1, o);
        for (int j = 0; j < nshift; ++j) {
            iters[j] = st[size_t(j)].iterations;
            matvecs[j] = st[size_t(j)].matvecs;
            relres[j] = st[size_t(j)].relres;
            converged[j] = st[size_t(j)].converged ? 1 : 0;
            p1relres[j] = p1[size_t(j)];
        }
        info[0] = o.phase1_steps;
        info[1] = o.defl_k;
        info[2] = o.rank_reduced;
        info[3] = o.pencil_shifted;
        info[4] = o.breakdown;
        info[5] = o.all_converged;
        info[6] = o.first_failure;
    });
}

}  // extern "C"
