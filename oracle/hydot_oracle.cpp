// hydot_oracle.cpp -- CPU ORACLE (test infrastructure only).
//
// A plain C++ restatement of the reference hot path in
// /root/reference/proj (arXiv 1410.0986, "hydot"), used ONLY by tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// as the checker and the CPU baseline.  The product (paper_1410_0986_b200/)
// never links, loads or calls this file.
//
// Parity status: the reference itself cannot be built here (it needs Eigen
// 3.4, absent from the image), and it ships no golden numeric
// vectors.  This restatement is pinned by (a) the reference's own
// known-answer tests (cluster-tree fixtures test_lowrank.cpp:139-174,
// tolerance formula :246-256, measurement ordering test_born.cpp:73-81),
// (b) the C++ standard's known answer for mt19937_64 ([rand.predef]:
// the 10000th output of a default-seeded engine is 9981545732273789042),
// (c) the reference's bound/determinism tests restated in tests/, and
// (d) by construction: the Gaussian stream is produced by the very libstdc++
// 13 <random> code the reference calls (lowrank.cpp:136-143).  Eigen's
// HouseholderQR/BDCSVD are replaced by LAPACK dgeqrf/dorgqr/dgesdd from the
// scipy-bundled OpenBLAS (same algorithms up to rounding) -- those numerics
// are "parity pinned by bounds", not bitwise.
//
// Every function cites the reference file:line it follows.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

extern "C" {
void scipy_dgemm_(const char*, const char*, const int*, const int*, const int*,
                  const double*, const double*, const int*, const double*,
                  const int*, const double*, double*, const int*);
void scipy_dgeqrf_(const int*, const int*, double*, const int*, double*,
                   double*, const int*, int*);
void scipy_dorgqr_(const int*, const int*, const int*, double*, const int*,
                   const double*, double*, const int*, int*);
void scipy_dgesdd_(const char*, const int*, const int*, double*, const int*,
                   double*, double*, const int*, double*, const int*, double*,
                   const int*, int*, int*);
void scipy_openblas_set_num_threads(int);
}

namespace oracle {

// ---------------------------------------------------------------- Mat ------
// Column-major dense matrix (Eigen::MatrixXd stand-in, grid.hpp:12-14).
struct Mat {
    int64_t r = 0, c = 0;
    std::vector<double> d;
    Mat() = default;
    Mat(int64_t rows, int64_t cols) : r(rows), c(cols), d(size_t(rows * cols), 0.0) {}
    double& operator()(int64_t i, int64_t j) { return d[size_t(i + j * r)]; }
    double operator()(int64_t i, int64_t j) const { return d[size_t(i + j * r)]; }
    double* col(int64_t j) { return d.data() + j * r; }
    const double* col(int64_t j) const { return d.data() + j * r; }
    static Mat identity(int64_t n) {
        Mat I(n, n);
        for (int64_t i = 0; i < n; ++i) I(i, i) = 1.0;
        return I;
    }
    Mat transpose() const {
        Mat t(c, r);
        for (int64_t j = 0; j < c; ++j)
            for (int64_t i = 0; i < r; ++i) t(j, i) = (*this)(i, j);
        return t;
    }
    Mat leftCols(int64_t k) const {
        Mat o(r, k);
        std::copy(d.begin(), d.begin() + r * k, o.d.begin());
        return o;
    }
    Mat rows_range(int64_t i0, int64_t n) const {
        Mat o(n, c);
        for (int64_t j = 0; j < c; ++j)
            for (int64_t i = 0; i < n; ++i) o(i, j) = (*this)(i0 + i, j);
        return o;
    }
    double norm() const {  // Frobenius, Eigen .norm()
        double s = 0.0;
        for (double v : d) s += v * v;
        return std::sqrt(s);
    }
};

static int I32(int64_t v) {
    if (v > INT32_MAX) throw std::invalid_argument("dimension exceeds LAPACK int");
    return int(v);
}

// C = op(A) * op(B) via dgemm (Eigen A*B).
static Mat matmul(const Mat& A, bool ta, const Mat& B, bool tb) {
    int64_t m = ta ? A.c : A.r, k = ta ? A.r : A.c;
    int64_t k2 = tb ? B.c : B.r, n = tb ? B.r : B.c;
    if (k != k2) throw std::invalid_argument("matmul: inner dimension mismatch");
    Mat C(m, n);
    if (m == 0 || n == 0) return C;
    if (k == 0) return C;
    int M = I32(m), N = I32(n), K = I32(k);
    int lda = std::max(1, I32(A.r)), ldb = std::max(1, I32(B.r)), ldc = std::max(1, M);
    double one = 1.0, zero = 0.0;
    scipy_dgemm_(ta ? "T" : "N", tb ? "T" : "N", &M, &N, &K, &one, A.d.data(), &lda,
                 B.d.data(), &ldb, &zero, C.d.data(), &ldc);
    return C;
}

// ------------------------------------------------------------- ledger ------
// FlopLedger (lowrank.hpp:38-52) and charge() (lowrank.cpp:20-28).
struct Ledger {
    double leaf = 0, agglomeration = 0, recompress = 0, other = 0, kernel_tally = 0;
};
enum Cat { LEAF = 0, AGGLOMERATION = 1, RECOMPRESS = 2, OTHER = 3 };
static void charge(Ledger* l, int cat, double f) {
    if (!l) return;
    switch (cat) {
        case LEAF: l->leaf += f; break;
        case AGGLOMERATION: l->agglomeration += f; break;
        case RECOMPRESS: l->recompress += f; break;
        default: l->other += f; break;
    }
}
static void tally(Ledger* l, int cat, double f) {
    if (l) l->kernel_tally += f;
    charge(l, cat, f);
}

// gemm with ledger (lowrank.cpp:31-36)
static Mat gemm(const Mat& A, bool ta, const Mat& B, bool tb, Ledger* l, int cat) {
    double rows = ta ? A.c : A.r, inner = ta ? A.r : A.c, cols = tb ? B.r : B.c;
    tally(l, cat, 2.0 * rows * cols * inner);
    return matmul(A, ta, B, tb);
}
static double svd_flops(double m, double n) {  // lowrank.cpp:38-41
    double mn = std::min(m, n), mx = std::max(m, n);
    return 14.0 * mx * mn * mn;
}
static double qr_flops(double m, double n) { return 2.0 * m * n * n; }  // :51

struct ThinSVD {
    Mat U;
    std::vector<double> s;
    Mat V;
};

// Plain thin SVD (Eigen::BDCSVD ComputeThinU|ThinV, lowrank.cpp:43-49) via
// LAPACK dgesdd (divide and conquer as well).
static ThinSVD lapack_svd(const Mat& A0) {
    ThinSVD out;
    int64_t m = A0.r, n = A0.c, k = std::min(m, n);
    out.U = Mat(m, k);
    out.V = Mat(n, k);
    out.s.assign(size_t(k), 0.0);
    if (k == 0) return out;
    Mat A = A0;
    Mat VT(k, n);
    int M = I32(m), N = I32(n), lda = M, ldu = M, ldvt = I32(k), info = 0, lwork = -1;
    std::vector<int> iwork(size_t(8 * k));
    double wq = 0;
    scipy_dgesdd_("S", &M, &N, A.d.data(), &lda, out.s.data(), out.U.d.data(), &ldu,
                  VT.d.data(), &ldvt, &wq, &lwork, iwork.data(), &info);
    lwork = int(wq) + 1;
    std::vector<double> work(static_cast<size_t>(lwork));
    scipy_dgesdd_("S", &M, &N, A.d.data(), &lda, out.s.data(), out.U.d.data(), &ldu,
                  VT.d.data(), &ldvt, work.data(), &lwork, iwork.data(), &info);
    if (info != 0) throw std::runtime_error("dgesdd failed, info=" + std::to_string(info));
    out.V = VT.transpose();
    return out;
}

static ThinSVD thin_svd(const Mat& A, Ledger* l, int cat) {  // lowrank.cpp:43-49
    tally(l, cat, svd_flops(double(A.r), double(A.c)));
    return lapack_svd(A);
}

// Householder QR (Eigen::HouseholderQR) -> R (n x n upper) and thin Q (m x n).
struct QR {
    Mat R, Q;
};
static QR householder_qr(const Mat& A0) {
    int64_t m = A0.r, n = A0.c;
    QR out;
    Mat A = A0;
    int64_t k = std::min(m, n);
    std::vector<double> tau(size_t(std::max<int64_t>(k, 1)));
    int M = I32(m), N = I32(n), lda = std::max(1, M), info = 0, lwork = -1;
    double wq = 0;
    if (k > 0) {
        scipy_dgeqrf_(&M, &N, A.d.data(), &lda, tau.data(), &wq, &lwork, &info);
        lwork = std::max(1, int(wq));
        std::vector<double> work(static_cast<size_t>(lwork));
        scipy_dgeqrf_(&M, &N, A.d.data(), &lda, tau.data(), work.data(), &lwork, &info);
        if (info != 0) throw std::runtime_error("dgeqrf failed");
    }
    out.R = Mat(k, n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i <= std::min<int64_t>(j, k - 1); ++i) out.R(i, j) = A(i, j);
    // thin Q = Q * I(m, k)
    out.Q = A.leftCols(k);
    if (k > 0) {
        int K = I32(k);
        lwork = -1;
        scipy_dorgqr_(&M, &K, &K, out.Q.d.data(), &lda, tau.data(), &wq, &lwork, &info);
        lwork = std::max(1, int(wq));
        std::vector<double> work(static_cast<size_t>(lwork));
        scipy_dorgqr_(&M, &K, &K, out.Q.d.data(), &lda, tau.data(), work.data(), &lwork, &info);
        if (info != 0) throw std::runtime_error("dorgqr failed");
    }
    return out;
}

// fast_thin_svd (lowrank.cpp:62-93): QR of the long dimension first.
static ThinSVD fast_thin_svd(const Mat& A, Ledger* l, int cat) {
    const int64_t m = A.r, n = A.c;
    ThinSVD out;
    if (n >= 2 * m && m > 0) {  // :66-72
        ThinSVD t = fast_thin_svd(A.transpose(), l, cat);
        out.U = std::move(t.V);
        out.s = std::move(t.s);
        out.V = std::move(t.U);
        return out;
    }
    if (m >= 2 * n && n > 0) {  // :73-87
        tally(l, cat, 2.0 * qr_flops(double(m), double(n)) + svd_flops(double(n), double(n)));
        QR qr = householder_qr(A);
        ThinSVD s = lapack_svd(qr.R);  // R is n x n
        out.U = matmul(qr.Q, false, s.U, false);  // Q * [U; 0]
        out.s = s.s;
        out.V = s.V;
        return out;
    }
    ThinSVD s = thin_svd(A, l, cat);  // :88-92
    return s;
}

// ------------------------------------------------------ Gaussian stream ----
// libstdc++ std::mt19937_64 + std::normal_distribution<double>, one
// distribution object per randsvd call, filled column-major
// (lowrank.cpp:136-143).
struct Gaussian {
    std::mt19937_64 rng;
    std::normal_distribution<double> gauss{0.0, 1.0};
    explicit Gaussian(uint64_t seed) : rng(seed) {}
    Mat draw(int64_t rows, int64_t cols) {
        Mat G(rows, cols);
        for (int64_t j = 0; j < cols; ++j)
            for (int64_t i = 0; i < rows; ++i) G(i, j) = gauss(rng);
        return G;
    }
};

// ------------------------------------------------------------- factor ------
enum Method { M_NONE = 0, M_RANDSVD = 1, M_ACA_FULL = 2, M_ACA_PARTIAL = 3,
              M_AGGLOMERATE = 4, M_RECURSIVE = 5, M_RECOMPRESS = 6 };

struct Factor {  // LowRankFactor (lowrank.hpp:25-36)
    Mat U, V;
    double tol = 0.0;
    int method = M_NONE;
    bool flagged = false;
    int64_t rank() const { return U.c; }
};

// randsvd (lowrank.cpp:131-199) on a dense operator (dense_op, :111-120).
static Factor randsvd(const Mat& A, double eps, int p, int kprobe, uint64_t seed,
                      Ledger* l, int cat, int r0) {
    const int64_t m = A.r, n = A.c;
    const int64_t nmax = std::min(m, n);
    Gaussian g(seed);
    Factor f;
    f.tol = eps;
    f.method = M_RANDSVD;
    if (m == 0 || n == 0) {
        f.U = Mat(m, 0);
        f.V = Mat(n, 0);
        return f;
    }
    int64_t r = std::clamp<int64_t>(r0, 1, nmax);
    Mat Q;
    double sigma_top = 0.0;
    bool identity = false;
    while (true) {
        int64_t rs = std::min<int64_t>(r + p, nmax);
        if (rs >= nmax && m <= n) {  // :159-164
            identity = true;
            break;
        }
        Mat Omega1 = g.draw(n, rs);
        tally(l, cat, 2.0 * double(m) * double(n) * double(rs));  // apply_mm :97-99
        Mat Y = matmul(A, false, Omega1, false);
        ThinSVD svdY = fast_thin_svd(Y, l, cat);
        int64_t qcols = std::min<int64_t>(r, svdY.U.c);
        Q = svdY.U.leftCols(qcols);
        sigma_top = svdY.s[0];

        Mat Omega2 = g.draw(n, kprobe);
        tally(l, cat, 2.0 * double(m) * double(n) * double(kprobe));
        Mat P = matmul(A, false, Omega2, false);
        Mat QtP = gemm(Q, true, P, false, l, cat);
        Mat QQtP = gemm(Q, false, QtP, false, l, cat);
        double er2 = 0.0;
        for (size_t i = 0; i < P.d.size(); ++i) {
            double dlt = P.d[i] - QQtP.d[i];
            er2 += dlt * dlt;
        }
        double er = std::sqrt(er2);
        if (er <= eps * sigma_top) break;  // :176
        if (r >= nmax) {                   // :177-180
            f.flagged = true;
            break;
        }
        r = std::min<int64_t>(2 * r, nmax);  // :181
    }
    int64_t qc = identity ? m : Q.c;
    tally(l, cat, 2.0 * double(m) * double(n) * double(qc));  // apply_mm adjoint :184
    Mat B = identity ? A : matmul(Q, true, A, false);  // (A^T Q)^T = Q^T A
    ThinSVD svdB = fast_thin_svd(B, l, cat);
    const std::vector<double>& s = svdB.s;
    double s1 = s.empty() ? 0.0 : s[0];
    int64_t keep = 0;
    for (size_t i = 0; i < s.size(); ++i)
        if (s[i] > eps * s1 && s[i] > 0) keep = int64_t(i) + 1;  // :187-190
    Mat Uk = svdB.U.leftCols(keep);
    if (identity) {
        tally(l, cat, 2.0 * double(m) * double(keep) * double(m));  // gemm(I, U)
        f.U = Uk;
    } else {
        f.U = gemm(Q, false, Uk, false, l, cat);  // :191
    }
    f.V = svdB.V.leftCols(keep);  // :192
    for (int64_t j = 0; j < keep; ++j)
        for (int64_t i = 0; i < n; ++i) f.V(i, j) *= s[size_t(j)];
    tally(l, cat, 1.0 * double(n) * double(keep));  // :193-197
    return f;
}

// agglomerate (lowrank.cpp:321-359)
static Factor agglomerate(const Factor& f1, const Factor& f2, double eps, uint64_t seed,
                          Ledger* l, int rank_hint, int p, int kprobe) {
    if (f1.V.r != f2.V.r) throw std::invalid_argument("agglomerate: column dimension mismatch");
    const int64_t n = f1.V.r, r1 = f1.rank(), r2 = f2.rank();
    const int64_t m1 = f1.U.r, m2 = f2.U.r;
    Factor out;
    out.tol = eps;
    out.method = M_AGGLOMERATE;
    if (r1 + r2 == 0) {
        out.U = Mat(m1 + m2, 0);
        out.V = Mat(n, 0);
        return out;
    }
    Mat W(r1 + r2, n);  // [V1^T; V2^T]  :339-341
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < r1; ++j) W(j, i) = f1.V(i, j);
        for (int64_t j = 0; j < r2; ++j) W(r1 + j, i) = f2.V(i, j);
    }
    int hint = int(std::max<int64_t>({r1, r2, int64_t(rank_hint)}));
    Factor inner = randsvd(W, eps, p, kprobe, seed, l, AGGLOMERATION, hint);  // :344-346
    int64_t rp = inner.rank();
    out.U = Mat(m1 + m2, rp);
    out.V = inner.V;
    if (rp > 0) {
        Mat top = gemm(f1.U, false, inner.U.rows_range(0, r1), false, l, AGGLOMERATION);
        Mat bot = gemm(f2.U, false, inner.U.rows_range(r1, r2), false, l, AGGLOMERATION);
        for (int64_t j = 0; j < rp; ++j) {
            for (int64_t i = 0; i < m1; ++i) out.U(i, j) = top(i, j);
            for (int64_t i = 0; i < m2; ++i) out.U(m1 + i, j) = bot(i, j);
        }
    }
    out.flagged = f1.flagged || f2.flagged || inner.flagged;  // :357
    return out;
}

// -------------------------------------------------------- cluster tree -----
// ClusterTree / build_cluster_tree / depth / leaf_order (lowrank.cpp:361-438)
struct Node {
    std::vector<int> idx;
    int left = -1, right = -1;
    std::vector<double> lo, hi;
    bool is_leaf() const { return left < 0; }
};
struct Tree {
    std::vector<Node> nodes;
    int root = 0;
    int depth() const {
        std::function<int(int)> go = [&](int v) -> int {
            const Node& nd = nodes[size_t(v)];
            if (nd.is_leaf()) return 0;
            return 1 + std::max(go(nd.left), go(nd.right));
        };
        return nodes.empty() ? 0 : go(root);
    }
    std::vector<int> leaf_order() const {
        std::vector<int> order;
        std::function<void(int)> go = [&](int v) {
            const Node& nd = nodes[size_t(v)];
            if (nd.is_leaf()) {
                order.insert(order.end(), nd.idx.begin(), nd.idx.end());
                return;
            }
            go(nd.left);
            go(nd.right);
        };
        if (!nodes.empty()) go(root);
        return order;
    }
};

static Tree build_cluster_tree(const Mat& pos, const std::vector<double>& lo,
                               const std::vector<double>& hi) {
    const int d = int(pos.c);
    if (pos.r < 1) throw std::invalid_argument("build_cluster_tree: no sources");
    if (int(lo.size()) != d || int(hi.size()) != d)
        throw std::invalid_argument("build_cluster_tree: box dimension");
    Tree tree;
    std::function<int(std::vector<int>, std::vector<double>, std::vector<double>)> split =
        [&](std::vector<int> idx, std::vector<double> a, std::vector<double> b) -> int {
        int me = int(tree.nodes.size());
        tree.nodes.push_back({});
        tree.nodes[size_t(me)].idx = idx;
        tree.nodes[size_t(me)].lo = a;
        tree.nodes[size_t(me)].hi = b;
        if (idx.size() <= 2) return me;  // :401
        int jmax = 0;
        for (int j = 1; j < d; ++j)
            if (b[size_t(j)] - a[size_t(j)] > b[size_t(jmax)] - a[size_t(jmax)]) jmax = j;  // :403-405
        double gamma = 0.5 * (a[size_t(jmax)] + b[size_t(jmax)]);
        std::vector<int> t1, t2;
        for (int i : idx) (pos(i, jmax) <= gamma ? t1 : t2).push_back(i);  // :409
        std::vector<double> b1 = b, a2 = a;
        b1[size_t(jmax)] = gamma;
        a2[size_t(jmax)] = gamma;
        if (t1.empty() || t2.empty()) {  // :413-425 median fallback
            std::vector<int> sorted = idx;
            std::stable_sort(sorted.begin(), sorted.end(),
                             [&](int x, int y) { return pos(x, jmax) < pos(y, jmax); });
            size_t half = sorted.size() / 2;
            t1.assign(sorted.begin(), sorted.begin() + long(half));
            t2.assign(sorted.begin() + long(half), sorted.end());
            b1 = b;
            a2 = a;
        }
        int lft = split(std::move(t1), a, b1);
        int rgt = split(std::move(t2), a2, b);
        tree.nodes[size_t(me)].left = lft;
        tree.nodes[size_t(me)].right = rgt;
        return me;
    };
    std::vector<int> all(size_t(pos.r));
    for (size_t i = 0; i < all.size(); ++i) all[i] = int(i);
    tree.root = split(all, lo, hi);
    return tree;
}

// ---------------------------------------------------- recursive_lowrank ----
struct RecResult {
    Factor factor;
    std::vector<int> source_order, row_perm, node_rank, node_depth;
    Ledger ledger;
};

// recursive_lowrank + leaf_compress + node_hint (lowrank.cpp:442-521).
// block(s) returns the rows_per_source x cols block of source s.
// Sharded replay (the multi-GPU schedule): source_ids maps local source i
// to its global id and node_offset is the subtree root's global pre-order id,
// so seeds and row_perm use global ids (identity when unsharded).
static RecResult recursive_lowrank(const Tree& tree, double eps, int rows_per, int64_t cols,
                                   const std::function<Mat(int)>& block, uint64_t seed, int p,
                                   int kprobe, const int* source_ids = nullptr,
                                   int node_offset = 0) {
    (void)cols;
    auto gs = [&](int s) { return source_ids ? source_ids[s] : s; };
    RecResult res;
    res.node_rank.assign(tree.nodes.size(), -1);
    res.node_depth.assign(tree.nodes.size(), 0);
    int leaf_hint = -1;
    std::map<int, int> depth_hint;
    auto node_hint = [&](int depth) {  // :452-455
        auto it = depth_hint.find(depth);
        return it == depth_hint.end() ? -1 : it->second + 2;
    };
    std::function<Factor(int, int)> go = [&](int v, int depth) -> Factor {
        const Node& nd = tree.nodes[size_t(v)];
        res.node_depth[size_t(v)] = depth;
        Factor f;
        try {
            if (nd.is_leaf()) {
                std::vector<Factor> parts;
                for (int s : nd.idx) {
                    Mat blk = block(s);
                    parts.push_back(randsvd(blk, eps, p, kprobe,
                                            seed + 0x9e3779b97f4a7c15ULL * uint64_t(gs(s) + 1),
                                            &res.ledger, LEAF, std::max(1, leaf_hint + 2)));
                    leaf_hint = int(parts.back().rank());
                }
                if (parts.empty()) throw std::runtime_error("empty leaf cluster");
                f = parts[0];
                for (size_t i = 1; i < parts.size(); ++i)
                    f = agglomerate(f, parts[i], eps,
                                    seed + 0x517cc1b727220a95ULL * uint64_t(node_offset + v + 1),
                                    &res.ledger, node_hint(depth), p, kprobe);
            } else {
                Factor fl = go(nd.left, depth + 1);
                Factor fr = go(nd.right, depth + 1);
                f = agglomerate(fl, fr, eps, seed + 0x2545f4914f6cdd1dULL * uint64_t(node_offset + v + 1),
                                &res.ledger, node_hint(depth), p, kprobe);
            }
        } catch (const std::exception& e) {
            throw std::runtime_error("recursive_lowrank at node " + std::to_string(v) + ": " +
                                     e.what());
        }
        res.node_rank[size_t(v)] = int(f.rank());
        depth_hint[depth] = int(f.rank());
        return f;
    };
    res.factor = go(tree.root, 0);
    res.factor.method = M_RECURSIVE;
    res.factor.tol = eps;
    res.source_order = tree.leaf_order();
    for (int s : res.source_order)
        for (int q = 0; q < rows_per; ++q) res.row_perm.push_back(gs(s) * rows_per + q);
    return res;
}

// tolerance_schedule (lowrank.cpp:540-545)
static double tolerance_schedule(double eps_d, int L, int N_r) {
    if (eps_d <= 0 || L < 0 || N_r < 1)
        throw std::invalid_argument("tolerance_schedule: bad arguments");
    return eps_d / (std::pow(2.0, 0.5 * L) * (L + 1) * std::sqrt(double(N_r)));
}

// recompress (lowrank.cpp:547-587)
static Factor recompress(const Factor& f, double eps, int rank, Ledger* l) {
    const int64_t r = f.rank();
    Factor out;
    out.tol = eps;
    out.method = M_RECOMPRESS;
    out.flagged = f.flagged;
    if (r == 0) {
        out.U = Mat(f.U.r, 0);
        out.V = Mat(f.V.r, 0);
        return out;
    }
    tally(l, RECOMPRESS, qr_flops(double(f.U.r), double(r)) + qr_flops(double(f.V.r), double(r)));
    QR qu = householder_qr(f.U), qv = householder_qr(f.V);
    Mat core = gemm(qu.R, false, qv.R, true, l, RECOMPRESS);
    ThinSVD svd = thin_svd(core, l, RECOMPRESS);
    const std::vector<double>& s = svd.s;
    double s1 = s.empty() ? 0.0 : s[0];
    int64_t keep;
    if (rank >= 0) {
        keep = std::min<int64_t>(rank, int64_t(s.size()));
    } else {
        keep = 0;
        for (size_t i = 0; i < s.size(); ++i)
            if (s[i] > eps * s1 && s[i] > 0) keep = int64_t(i) + 1;
    }
    out.U = gemm(qu.Q, false, svd.U.leftCols(keep), false, l, RECOMPRESS);
    Mat Vs = svd.V.leftCols(keep);
    for (int64_t j = 0; j < keep; ++j)
        for (int64_t i = 0; i < Vs.r; ++i) Vs(i, j) *= s[size_t(j)];
    out.V = gemm(qv.Q, false, Vs, false, l, RECOMPRESS);
    return out;
}

// ------------------------------------------------------------- fields ------
// 7-point vertex-centred finite-volume operator (BASELINE.json configs; the
// reference's K + sigma M + sigma' R form, grid.cpp:112-174, with the FEM
// stencil replaced by the 7-point one per SURVEY Appendix A #1):
//   unknowns: vertices with 0<ix<nx-1, 0<iy<ny-1 (side faces Dirichlet,
//   grid.hpp:42-45); zext = h (interior) or h/2 (iz = 0 or nz-1);
//   lateral link weight zext, vertical link weight h, V = h^2 zext,
//   S = h^2 on z faces.  (A x)_i = diag_i x_i - sum_j w_ij x_j with
//   diag_i = sum_j w_ij + sigma V_i + sigma' S_i.  Dirichlet rows: identity.
struct Grid7 {
    int nx, ny, nz;
    double h;
    int64_t N() const { return int64_t(nx) * ny * nz; }
    bool dirichlet(int ix, int iy) const { return ix == 0 || ix == nx - 1 || iy == 0 || iy == ny - 1; }
};

// mu (optional): the nonlinear forward model's perturbed medium, absorption
// sigma + dsig mu_i per vertex (experiments.cpp:154-206, w = nu (mu_bg + dmu mu) / D)
static void apply7(const Grid7& g, double sigma, double sigmap, const double* x, double* y,
                   const double* mu = nullptr, double dsig = 0.0) {
    const double h = g.h;
    for (int iz = 0; iz < g.nz; ++iz) {
        const bool zb = (iz == 0 || iz == g.nz - 1);
        const double zext = zb ? 0.5 * h : h;
        const double V = h * h * zext, S = zb ? h * h : 0.0;
        for (int iy = 0; iy < g.ny; ++iy)
            for (int ix = 0; ix < g.nx; ++ix) {
                int64_t i = ix + int64_t(g.nx) * (iy + int64_t(g.ny) * iz);
                if (g.dirichlet(ix, iy)) {
                    y[i] = x[i];
                    continue;
                }
                // neighbour sum in fixed order: -x, +x, -y, +y, -z, +z
                double wsum = 4.0 * zext;
                // Dirichlet neighbours are eliminated symmetrically
                // (grid.cpp:121-130): their link stays on the diagonal only.
                double xm = ix - 1 > 0 ? x[i - 1] : 0.0;
                double xp = ix + 1 < g.nx - 1 ? x[i + 1] : 0.0;
                double ym = iy - 1 > 0 ? x[i - g.nx] : 0.0;
                double yp = iy + 1 < g.ny - 1 ? x[i + g.nx] : 0.0;
                double nb = zext * xm;
                nb = nb + zext * xp;
                nb = nb + zext * ym;
                nb = nb + zext * yp;
                int64_t plane = int64_t(g.nx) * g.ny;
                if (iz > 0) {
                    wsum = wsum + h;
                    nb = nb + h * x[i - plane];
                }
                if (iz < g.nz - 1) {
                    wsum = wsum + h;
                    nb = nb + h * x[i + plane];
                }
                const double sg = mu ? sigma + dsig * mu[i] : sigma;
                double diag = wsum + sg * V + sigmap * S;
                y[i] = diag * x[i] - nb;
            }
    }
}

// Batched CG (replaces krylov::solve_family, krylov.cpp:400-463,
// by CG on the SPD system).  Returns iterations used.  If fixed_iters > 0,
// runs exactly that many iterations (parity mode).
static int cg_solve(const Grid7& g, double sigma, double sigmap, const double* b, double* x,
                    double tol, int max_iter, int fixed_iters, double* relres_out,
                    const double* mu = nullptr, double dsig = 0.0) {
    const int64_t N = g.N();
    std::vector<double> r(b, b + N), p(b, b + N), q(static_cast<size_t>(N));
    std::fill(x, x + N, 0.0);
    auto dot = [&](const double* a, const double* c) {
        double s = 0.0;
        for (int64_t i = 0; i < N; ++i) s += a[i] * c[i];
        return s;
    };
    double rr = dot(r.data(), r.data());
    double bnorm = std::sqrt(rr);
    int it = 0;
    double relres = bnorm > 0 ? 1.0 : 0.0;
    if (bnorm == 0.0) {
        if (relres_out) *relres_out = 0.0;
        return 0;
    }
    int limit = fixed_iters > 0 ? fixed_iters : max_iter;
    for (it = 0; it < limit;) {
        apply7(g, sigma, sigmap, p.data(), q.data(), mu, dsig);
        double pq = dot(p.data(), q.data());
        double alpha = rr / pq;
        for (int64_t i = 0; i < N; ++i) {
            x[i] = x[i] + alpha * p[i];
            r[i] = r[i] - alpha * q[i];
        }
        double rr_new = dot(r.data(), r.data());
        ++it;
        relres = std::sqrt(rr_new) / bnorm;
        if (fixed_iters <= 0 && relres <= tol) break;
        double beta = rr_new / rr;
        for (int64_t i = 0; i < N; ++i) p[i] = r[i] + beta * p[i];
        rr = rr_new;
    }
    if (relres_out) *relres_out = relres;
    return it;
}

}  // namespace oracle

// ===================================================================== C ABI
// Flat C interface used by oracle/oracle.py (ctypes).  Matrices are
// column-major doubles.  Errors return nonzero and set oracle_last_error().
using namespace oracle;

static thread_local std::string g_err;

struct oracle_factor {
    Factor f;
    std::vector<int> row_perm, node_rank, node_depth;
    Ledger ledger;
};

template <class F>
static int guard(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

static Mat from_ptr(const double* a, int64_t rows, int64_t cols, int64_t ld) {
    Mat m(rows, cols);
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) m(i, j) = a[i + j * ld];
    return m;
}

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }
void oracle_set_threads(int n) { scipy_openblas_set_num_threads(n); }

// libstdc++ normal stream (lowrank.cpp:136-143): the first `count` deviates
// of a fresh (engine(seed), normal_distribution) pair.
int oracle_gaussian(uint64_t seed, int64_t count, double* out) {
    return guard([&] {
        Gaussian g(seed);
        for (int64_t i = 0; i < count; ++i) out[i] = g.gauss(g.rng);
    });
}
// raw engine outputs (tempered u64)
int oracle_mt19937_64(uint64_t seed, int64_t count, uint64_t* out) {
    return guard([&] {
        std::mt19937_64 e(seed);
        for (int64_t i = 0; i < count; ++i) out[i] = e();
    });
}

// assemble_H_block (born.cpp:82-98): out row-major (rows d*nl+l, N cols):
// out[(d*nl+l)*N + v] = (-nu) * ((phi_d[v,l] * phi_s[v,l]) * w[v]).
int oracle_born_block(int64_t N, int nl, const double* incident, const double* const* adjoint,
                      int nd, const double* w, double nu, double* out) {
    return guard([&] {
        for (int d = 0; d < nd; ++d)
            for (int l = 0; l < nl; ++l) {
                const double* pd = adjoint[d] + int64_t(l) * N;
                const double* ps = incident + int64_t(l) * N;
                double* o = out + (int64_t(d) * nl + l) * N;
                for (int64_t v = 0; v < N; ++v) o[v] = (-nu) * ((pd[v] * ps[v]) * w[v]);
            }
    });
}

int oracle_apply7(int nx, int ny, int nz, double h, double sigma, double sigmap, const double* x,
                  double* y) {
    return guard([&] { apply7(Grid7{nx, ny, nz, h}, sigma, sigmap, x, y); });
}

// Fields for n_rhs unit-vertex sources x n_lambda shifts; out is
// N x (n_rhs*nl), column k*nl+l, scaled by inv_D[l] (born.cpp:54-65).
// dsig / mu non-null: the perturbed medium sigma_l + dsig_l mu(v) (the
// nonlinear forward model's fields, experiments.cpp:154-206)
int oracle_fields_var(int nx, int ny, int nz, double h, int nl, const double* sigma, const double* sigmap,
                      const double* inv_D, const double* dsig, const double* mu, const int64_t* rhs_vertex,
                      int n_rhs, double tol, int max_iter, int fixed_iters, int threads, double* out, int* iters,
                      double* relres);

int oracle_fields(int nx, int ny, int nz, double h, int nl, const double* sigma,
                  const double* sigmap, const double* inv_D, const int64_t* rhs_vertex, int n_rhs,
                  double tol, int max_iter, int fixed_iters, int threads, double* out, int* iters,
                  double* relres) {
    return oracle_fields_var(nx, ny, nz, h, nl, sigma, sigmap, inv_D, nullptr, nullptr, rhs_vertex, n_rhs, tol,
                             max_iter, fixed_iters, threads, out, iters, relres);
}

int oracle_fields_var(int nx, int ny, int nz, double h, int nl, const double* sigma, const double* sigmap,
                      const double* inv_D, const double* dsig, const double* mu, const int64_t* rhs_vertex,
                      int n_rhs, double tol, int max_iter, int fixed_iters, int threads, double* out, int* iters,
                      double* relres) {
    return guard([&] {
        Grid7 g{nx, ny, nz, h};
        const int64_t N = g.N();
        int total = n_rhs * nl;
        std::vector<std::string> errs(size_t(std::max(1, threads)));
        auto work = [&](int t) {
            try {
                std::vector<double> b(static_cast<size_t>(N));
                for (int k = t; k < total; k += std::max(1, threads)) {
                    int s = k / nl, l = k % nl;
                    std::fill(b.begin(), b.end(), 0.0);
                    int64_t v = rhs_vertex[s];
                    if (v < 0 || v >= N) throw std::invalid_argument("rhs vertex out of range");
                    int ix = int(v % nx), iy = int((v / nx) % ny);
                    if (g.dirichlet(ix, iy))
                        throw std::invalid_argument(
                            "source support falls entirely on the Dirichlet boundary");
                    b[size_t(v)] = 1.0;
                    double* x = out + int64_t(k) * N;
                    double rr;
                    int it = cg_solve(g, sigma[l], sigmap[l], b.data(), x, tol, max_iter,
                                      fixed_iters, &rr, mu, dsig ? dsig[l] : 0.0);
                    for (int64_t i = 0; i < N; ++i) x[i] *= inv_D[l];
                    if (iters) iters[k] = it;
                    if (relres) relres[k] = rr;
                }
            } catch (const std::exception& e) {
                errs[size_t(t)] = e.what();
            }
        };
        if (threads <= 1) {
            work(0);
        } else {
            std::vector<std::thread> ts;
            for (int t = 0; t < threads; ++t) ts.emplace_back(work, t);
            for (auto& th : ts) th.join();
        }
        for (auto& e : errs)
            if (!e.empty()) throw std::invalid_argument(e);
    });
}

double oracle_tolerance_schedule(double eps_d, int L, int N_r) {
    double v = -1.0;
    if (guard([&] { v = tolerance_schedule(eps_d, L, N_r); }) != 0) return -1.0;
    return v;
}

// ---- factor handles
void oracle_factor_free(oracle_factor* f) { delete f; }
void oracle_factor_info(const oracle_factor* f, int64_t* rows, int64_t* cols, int64_t* rank,
                        double* tol, int* method, int* flagged) {
    *rows = f->f.U.r;
    *cols = f->f.V.r;
    *rank = f->f.rank();
    *tol = f->f.tol;
    *method = f->f.method;
    *flagged = f->f.flagged ? 1 : 0;
}
void oracle_factor_get(const oracle_factor* f, double* U, double* V) {
    std::copy(f->f.U.d.begin(), f->f.U.d.end(), U);
    std::copy(f->f.V.d.begin(), f->f.V.d.end(), V);
}
void oracle_factor_meta(const oracle_factor* f, int* row_perm, int* node_rank, int* node_depth,
                        double* ledger5) {
    if (row_perm) std::copy(f->row_perm.begin(), f->row_perm.end(), row_perm);
    if (node_rank) std::copy(f->node_rank.begin(), f->node_rank.end(), node_rank);
    if (node_depth) std::copy(f->node_depth.begin(), f->node_depth.end(), node_depth);
    if (ledger5) {
        ledger5[0] = f->ledger.leaf;
        ledger5[1] = f->ledger.agglomeration;
        ledger5[2] = f->ledger.recompress;
        ledger5[3] = f->ledger.other;
        ledger5[4] = f->ledger.kernel_tally;
    }
}
int64_t oracle_factor_perm_len(const oracle_factor* f) { return int64_t(f->row_perm.size()); }

oracle_factor* oracle_factor_make(const double* U, const double* V, int64_t rows, int64_t cols,
                                  int64_t rank, double tol, int method, int flagged) {
    auto* f = new oracle_factor;
    f->f.U = from_ptr(U, rows, rank, rows);
    f->f.V = from_ptr(V, cols, rank, cols);
    f->f.tol = tol;
    f->f.method = method;
    f->f.flagged = flagged != 0;
    return f;
}

int oracle_randsvd(const double* A, int64_t m, int64_t n, int64_t lda, double eps, int p,
                   int kprobe, uint64_t seed, int cat, int r0, oracle_factor** out) {
    return guard([&] {
        auto* f = new oracle_factor;
        std::unique_ptr<oracle_factor> hold(f);
        Mat Am = from_ptr(A, m, n, lda);
        f->f = randsvd(Am, eps, p, kprobe, seed, &f->ledger, cat, r0);
        *out = hold.release();
    });
}

int oracle_agglomerate(const oracle_factor* f1, const oracle_factor* f2, double eps,
                       uint64_t seed, int rank_hint, int p, int kprobe, oracle_factor** out) {
    return guard([&] {
        std::unique_ptr<oracle_factor> f(new oracle_factor);
        f->f = agglomerate(f1->f, f2->f, eps, seed, &f->ledger, rank_hint, p, kprobe);
        *out = f.release();
    });
}

int oracle_recompress(const oracle_factor* in, double eps, int rank, oracle_factor** out) {
    return guard([&] {
        std::unique_ptr<oracle_factor> f(new oracle_factor);
        f->f = recompress(in->f, eps, rank, &f->ledger);
        f->row_perm = in->row_perm;
        *out = f.release();
    });
}

// ---- tree
struct oracle_tree {
    Tree t;
};
int oracle_build_cluster_tree(const double* pos, int n, int d, const double* lo, const double* hi,
                              oracle_tree** out) {
    return guard([&] {
        Mat P = from_ptr(pos, n, d, n);
        std::unique_ptr<oracle_tree> t(new oracle_tree);
        t->t = build_cluster_tree(P, std::vector<double>(lo, lo + d), std::vector<double>(hi, hi + d));
        *out = t.release();
    });
}
void oracle_tree_free(oracle_tree* t) { delete t; }
int oracle_tree_num_nodes(const oracle_tree* t) { return int(t->t.nodes.size()); }
int oracle_tree_root(const oracle_tree* t) { return t->t.root; }
int oracle_tree_depth(const oracle_tree* t) { return t->t.depth(); }
void oracle_tree_node(const oracle_tree* t, int v, int* left, int* right, int* nidx) {
    const Node& nd = t->t.nodes[size_t(v)];
    *left = nd.left;
    *right = nd.right;
    *nidx = int(nd.idx.size());
}
void oracle_tree_node_idx(const oracle_tree* t, int v, int* idx) {
    const Node& nd = t->t.nodes[size_t(v)];
    std::copy(nd.idx.begin(), nd.idx.end(), idx);
}
void oracle_tree_leaf_order(const oracle_tree* t, int* out) {
    auto o = t->t.leaf_order();
    std::copy(o.begin(), o.end(), out);
}

// recursive_lowrank over a dense stacked H (rows source-major, column-major
// M x N, ldh) -- the compress_H BlockProvider (experiments.cpp:235-240).
int oracle_recursive_lowrank(const oracle_tree* t, double eps, const double* H, int64_t M,
                             int64_t N, int64_t ldh, int rows_per, uint64_t seed, int p,
                             int kprobe, oracle_factor** out) {
    return guard([&] {
        auto block = [&](int s) { return from_ptr(H + int64_t(s) * rows_per, rows_per, N, ldh); };
        (void)M;
        RecResult r = recursive_lowrank(t->t, eps, rows_per, N, block, seed, p, kprobe);
        std::unique_ptr<oracle_factor> f(new oracle_factor);
        f->f = std::move(r.factor);
        f->row_perm = r.row_perm;
        f->node_rank = r.node_rank;
        f->node_depth = r.node_depth;
        f->ledger = r.ledger;
        *out = f.release();
    });
}

// Same, with the Born blocks formed from fields on demand (the device
// provider's semantics): incident[s] N x nl, adjoint[s*nd+d] N x nl.
int oracle_recursive_lowrank_born(const oracle_tree* t, double eps, int64_t N, int nl, int nd,
                                  const double* const* incident, const double* const* adjoint,
                                  const double* w, double nu, uint64_t seed, int p, int kprobe,
                                  const int* source_ids, int node_offset, oracle_factor** out) {
    return guard([&] {
        int rows_per = nd * nl;
        auto block = [&](int s) {
            Mat b(rows_per, N);
            for (int d = 0; d < nd; ++d)
                for (int l = 0; l < nl; ++l) {
                    const double* pd = adjoint[int64_t(s) * nd + d] + int64_t(l) * N;
                    const double* ps = incident[s] + int64_t(l) * N;
                    int row = d * nl + l;
                    for (int64_t v = 0; v < N; ++v) b(row, v) = (-nu) * ((pd[v] * ps[v]) * w[v]);
                }
            return b;
        };
        RecResult r = recursive_lowrank(t->t, eps, rows_per, N, block, seed, p, kprobe, source_ids,
                                        node_offset);
        std::unique_ptr<oracle_factor> f(new oracle_factor);
        f->f = std::move(r.factor);
        f->row_perm = r.row_perm;
        f->node_rank = r.node_rank;
        f->node_depth = r.node_depth;
        f->ledger = r.ledger;
        *out = f.release();
    });
}

// lr_matvec / lr_rmatvec (lowrank.cpp:589-599) on b columns, plain.
int oracle_lr_matmat(const oracle_factor* f, int trans, int b, const double* X, double* Y) {
    return guard([&] {
        const Mat& U = f->f.U;
        const Mat& V = f->f.V;
        if (!trans) {
            Mat Xm = from_ptr(X, V.r, b, V.r);
            Mat Z = matmul(V, true, Xm, false);
            Mat R = matmul(U, false, Z, false);
            std::copy(R.d.begin(), R.d.end(), Y);
        } else {
            Mat Ym = from_ptr(X, U.r, b, U.r);
            Mat Z = matmul(U, true, Ym, false);
            Mat R = matmul(V, false, Z, false);
            std::copy(R.d.begin(), R.d.end(), Y);
        }
    });
}

// J~ products with the chromophore axis:
//  trans=0: X is (N*nc) x b (chromophore-major blocks of N), Y is M x b;
//    y[row_perm[i]] = sum_c eps_c[l(row_perm[i])] * (U V^T x_c)[i]
//    with l(r) = r % nl (born.cpp:118-127, experiments.cpp:255-262).
//  trans=1: Y given (M x b) -> X (N*nc) x b: x_c = V U^T (gather_perm(E_c y)).
int oracle_j_matmat(const oracle_factor* f, int trans, int b, const int* row_perm,
                    const double* eps_c, int nl, int nc, const double* in, double* out) {
    return guard([&] {
        const Mat& U = f->f.U;
        const Mat& V = f->f.V;
        const int64_t M = U.r, N = V.r;
        if (!trans) {
            Mat Y(M, b);
            for (int c = 0; c < nc; ++c) {
                Mat Xc(N, b);
                for (int j = 0; j < b; ++j)
                    for (int64_t i = 0; i < N; ++i) Xc(i, j) = in[int64_t(c) * N + i + int64_t(j) * N * nc];
                Mat T = matmul(U, false, matmul(V, true, Xc, false), false);
                for (int j = 0; j < b; ++j)
                    for (int64_t i = 0; i < M; ++i) {
                        int r = row_perm[i];
                        Y(r, j) += eps_c[(r % nl) + int64_t(c) * nl] * T(i, j);
                    }
            }
            std::copy(Y.d.begin(), Y.d.end(), out);
        } else {
            for (int c = 0; c < nc; ++c) {
                Mat G(M, b);
                for (int j = 0; j < b; ++j)
                    for (int64_t i = 0; i < M; ++i) {
                        int r = row_perm[i];
                        G(i, j) = eps_c[(r % nl) + int64_t(c) * nl] * in[r + int64_t(j) * M];
                    }
                Mat Xc = matmul(V, false, matmul(U, true, G, false), false);
                for (int j = 0; j < b; ++j)
                    for (int64_t i = 0; i < N; ++i) out[int64_t(c) * N + i + int64_t(j) * N * nc] = Xc(i, j);
            }
        }
    });
}

// Thin SVD via the oracle's fast_thin_svd (for kernel-level parity tests).
int oracle_fast_thin_svd(const double* A, int64_t m, int64_t n, double* U, double* s, double* V) {
    return guard([&] {
        ThinSVD t = fast_thin_svd(from_ptr(A, m, n, m), nullptr, OTHER);
        std::copy(t.U.d.begin(), t.U.d.end(), U);
        std::copy(t.s.begin(), t.s.end(), s);
        std::copy(t.V.d.begin(), t.V.d.end(), V);
    });
}

// Factor file (lowrank.cpp:601-655): {M,N,r:i64, tol:f64, method:i64,
// plen:i64, perm:i64[plen], U row-major, V row-major}.
int oracle_save_factor(const char* path, const oracle_factor* f, const int* perm, int64_t plen) {
    return guard([&] {
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::runtime_error(std::string("cannot write factor: ") + path);
        auto wi = [&](int64_t v) { out.write(reinterpret_cast<const char*>(&v), 8); };
        auto wf = [&](double v) { out.write(reinterpret_cast<const char*>(&v), 8); };
        wi(f->f.U.r);
        wi(f->f.V.r);
        wi(f->f.rank());
        wf(f->f.tol);
        wi(f->f.method);
        wi(plen);
        for (int64_t i = 0; i < plen; ++i) wi(perm[i]);
        for (int64_t i = 0; i < f->f.U.r; ++i)
            for (int64_t j = 0; j < f->f.rank(); ++j) wf(f->f.U(i, j));
        for (int64_t i = 0; i < f->f.V.r; ++i)
            for (int64_t j = 0; j < f->f.rank(); ++j) wf(f->f.V(i, j));
    });
}

}  // extern "C"
