// lowrank.cpp -- host drivers of the device compression path: randsvd,
// agglomerate, recursive_lowrank, recompress (lowrank.cpp:131-199, 321-359,
// 385-521, 540-587 of the reference).  All matrices stay in HBM; the host
// only sees singular values, the probe error and ranks (one small D2H read
// per decision, exactly the quantities the reference branches on).
#include "lowrank.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <string>

namespace hydot {

namespace {
double svd_flops(double m, double n) {  // lowrank.cpp:38-41
    double mn = std::min(m, n), mx = std::max(m, n);
    return 14.0 * mx * mn * mn;
}
double qr_flops(double m, double n) { return 2.0 * m * n * n; }  // lowrank.cpp:51
void charge(Ledger* l, int cat, double f) {
    if (l) l->charge(cat, f);
}

// materialise L = S^T (S stored n x m) as column-major m x n
DBuf materialise_t(Ctx& c, const double* S, int64_t ld, int64_t m, int64_t n) {
    DBuf t = dalloc(c, size_t(std::max<int64_t>(m * n, 1)));
    transpose(c, n, m, S, ld, t.d(), m);
    return t;
}

// Thin SVD of X (m x n, m >= n) by QR-preconditioned one-sided Jacobi
// (the dgejsv idea): X = Q1 R1, R1^T = Q2 R2, Jacobi on L = R2^T gives
// L = Ux S Vx^T, hence X = (Q1 Ux) S (Q2 Vx)^T.  Jacobi on the twice
// QR-factored triangle needs ~4x fewer sweeps than on X itself (measured
// 8-10 vs 28-41 on graded 300x300 cores).  `upper`: X is already the n x n
// triangle R1 (Q1 = I).
// SVD of an n x n upper triangle R1 that came from the QR of norm-ordered
// columns: R1^T = Q2 R2, Jacobi on L = R2^T = Ux S Vx^T, so R1 = Ux S (Q2 Vx)^T.
// Ux -> U (n x n), Q2 Vx -> V (n x n).
void svd_of_sorted_r(Ctx& c, int64_t n, const double* R1, double* U, std::vector<double>& s, double* V) {
    QRFact q2;
    DBuf T = dalloc(c, size_t(n * n)), R2 = dalloc(c, size_t(n * n));
    transpose(c, n, n, R1, n, T.d(), n);  // R1^T
    geqrf(c, n, n, T.d(), n, q2);
    extract_upper(c, n, q2.a.d(), n, R2.d(), n);
    transpose(c, n, n, R2.d(), n, T.d(), n);  // L = R2^T
    jacobi_svd(c, n, n, T.d(), n, U, n, s, V, n);
    apply_q(c, q2, false, n, V, n);  // Q2 Vx
}

void jacobi_precond(Ctx& c, int64_t m, int64_t n, const double* X, int64_t ldx, bool upper,
                    double* U, int64_t ldu, std::vector<double>& s, double* V, int64_t ldv) {
    if (n <= 48) {  // the single-CTA shared-memory driver is already cheap
        jacobi_svd(c, m, n, X, ldx, U, ldu, s, V, ldv);
        return;
    }
    (void)upper;
    // 1. order columns by decreasing norm (X P), 2. X P = Q1 R1, 3. R1^T =
    // Q2 R2, 4. Jacobi on L = R2^T:  X = (Q1 Ul) S (P Q2 Vl)^T.
    // Measured on the config-1 pipeline: total Jacobi time 1.73 s with
    // norm-ordering + two QRs, 3.17 s with norm-ordering + one QR, 3.40 s
    // with two QRs only.
    constexpr bool qrqr = true;
    DBuf nrm = dalloc(c, size_t(n));
    col_norms(c, m, n, X, ldx, nrm.d());
    std::vector<double> hn(static_cast<size_t>(n));
    c.d2h(hn.data(), nrm.d(), size_t(n));
    std::vector<int> perm(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) perm[size_t(j)] = int(j);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return hn[size_t(a)] > hn[size_t(b)]; });
    DBuf dperm(c, size_t(n) * sizeof(int));
    HYDOT_CUDA(cudaMemcpyAsync(dperm.as<void>(), perm.data(), size_t(n) * sizeof(int),
                               cudaMemcpyHostToDevice, c.stream));
    DBuf Xp = dalloc(c, size_t(m * n));
    gather_cols(c, m, n, X, ldx, dperm.as<int>(), Xp.d(), m);
    QRFact q1, q2;
    geqrf(c, m, n, Xp.d(), m, q1);
    Xp.release();
    DBuf R1 = dalloc(c, size_t(n * n));
    extract_upper(c, n, q1.a.d(), m, R1.d(), n);
    DBuf Ux = dalloc(c, size_t(n * n));
    DBuf Vx = dalloc(c, size_t(n * n));
    if (qrqr) {
        DBuf T = dalloc(c, size_t(n * n));
        transpose(c, n, n, R1.d(), n, T.d(), n);  // R1^T
        geqrf(c, n, n, T.d(), n, q2);
        extract_upper(c, n, q2.a.d(), n, R1.d(), n);  // R2
        transpose(c, n, n, R1.d(), n, T.d(), n);      // L = R2^T
        jacobi_svd(c, n, n, T.d(), n, Ux.d(), n, s, Vx.d(), n);
        apply_q(c, q2, false, n, Vx.d(), n);  // Q2 Vx
    } else {
        jacobi_svd(c, n, n, R1.d(), n, Ux.d(), n, s, Vx.d(), n);
    }
    scatter_rows(c, n, n, Vx.d(), n, dperm.as<int>(), V, ldv);  // V = P Vr
    fill(c, m, n, 0.0, U, ldu);
    copy2d(c, n, n, Ux.d(), n, U, ldu);
    apply_q(c, q1, false, n, U, ldu, n);  // U = Q1 [Ur; 0]
    c.sync();  // host perm vector goes out of scope
}

// plain thin SVD of L (m x n) by Jacobi on the taller orientation
SVDd direct_svd(Ctx& c, const double* S, int64_t ld, bool trans, int64_t m, int64_t n) {
    SVDd o;
    o.m = m;
    o.n = n;
    o.k = std::min(m, n);
    o.U = dalloc(c, size_t(std::max<int64_t>(m * o.k, 1)));
    o.V = dalloc(c, size_t(std::max<int64_t>(n * o.k, 1)));
    if (o.k == 0) return o;
    if (m >= n) {
        // need L column-major (m x n)
        DBuf tmp;
        const double* Lp = S;
        int64_t ldl = ld;
        if (trans) {
            tmp = materialise_t(c, S, ld, m, n);
            Lp = tmp.d();
            ldl = m;
        }
        jacobi_precond(c, m, n, Lp, ldl, false, o.U.d(), m, o.s, o.V.d(), n);
    } else {
        // Jacobi on L^T (n x m): L^T = U' S V'^T  =>  L = V' S U'^T
        DBuf tmp;
        const double* Lt = S;
        int64_t ldt = ld;
        if (!trans) {
            tmp = materialise_t(c, S, ld, n, m);  // L^T as n x m
            Lt = tmp.d();
            ldt = n;
        }
        jacobi_precond(c, n, m, Lt, ldt, false, o.V.d(), n, o.s, o.U.d(), m);
    }
    return o;
}
}  // namespace

SVDd thin_svd(Ctx& c, const double* S, int64_t ld, bool trans, int64_t m, int64_t n, Ledger* l,
              int cat) {
    charge(l, cat, svd_flops(double(m), double(n)));  // lowrank.cpp:43-49
    return direct_svd(c, S, ld, trans, m, n);
}

namespace {
// The presorted tall QR of the Q = I branch, started speculatively (see
// randsvd).  Its buffers are allocated on c.stream; the side stream fills
// them; `ev` marks completion.  Unused, it makes c.stream wait for `ev`
// before its buffers are released.
struct TallSpec {
    Ctx* c = nullptr;
    const double* src = nullptr;
    int64_t ld = 0, m = 0, n = 0;
    std::vector<int> perm;
    DBuf dperm;
    QRFact qf;
    cudaEvent_t ev = nullptr;
    bool used = false;
    ~TallSpec() {
        if (ev) {
            if (!used && c) cudaStreamWaitEvent(c->stream, ev, 0);
            cudaEventDestroy(ev);
        }
    }
};

// column order by decreasing norm of the m x n matrix L
void presort_perm(Ctx& c, int64_t m, int64_t n, const double* Lp, int64_t ldl, std::vector<int>& perm) {
    DBuf nrm = dalloc(c, size_t(n));
    col_norms(c, m, n, Lp, ldl, nrm.d());
    std::vector<double> hn(static_cast<size_t>(n));
    c.d2h(hn.data(), nrm.d(), size_t(n));
    perm.resize(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) perm[size_t(j)] = int(j);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return hn[size_t(a)] > hn[size_t(b)]; });
}
}  // namespace

namespace {
// lazyU / lazyV: the caller accepts U (resp. V) as Q [Ur; 0] when the tall
// branch produces it (the request is forwarded through the transposed
// recursion); the SVDd's U (V) is then left empty.
SVDd fast_thin_svd_impl(Ctx& c, const double* S, int64_t ld, bool trans, int64_t m, int64_t n,
                        Ledger* l, int cat, LazyV* lazyU, LazyV* lazyV, TallSpec* spec = nullptr) {
    if (n >= 2 * m && m > 0) {  // lowrank.cpp:66-72
        SVDd t = fast_thin_svd_impl(c, S, ld, !trans, n, m, l, cat, lazyV, lazyU, spec);
        SVDd o;
        o.m = m;
        o.n = n;
        o.k = t.k;
        o.U = std::move(t.V);
        o.V = std::move(t.U);
        o.s = std::move(t.s);
        return o;
    }
    if (m >= 2 * n && n > 0) {  // lowrank.cpp:73-87
        charge(l, cat, 2.0 * qr_flops(double(m), double(n)) + svd_flops(double(n), double(n)));
        DBuf tmp;
        const double* Lp = S;
        int64_t ldl = ld;
        if (trans) {
            tmp = materialise_t(c, S, ld, m, n);
            Lp = tmp.d();
            ldl = m;
        }
        SVDd o;
        o.m = m;
        o.n = n;
        o.k = n;
        o.V = dalloc(c, size_t(n * n));
        DBuf Ur = dalloc(c, size_t(n * n));
        QRFact qf;
        if (n <= 48) {
            geqrf(c, m, n, Lp, ldl, qf);
            tmp.release();
            DBuf R = dalloc(c, size_t(n * n));
            extract_upper(c, n, qf.a.d(), m, R.d(), n);
            jacobi_precond(c, n, n, R.d(), n, true, Ur.d(), n, o.s, o.V.d(), n);
        } else {
            // norm-order the tall columns first: QR(A P) = Q R1 is the
            // preconditioner's first QR, so only R1^T's QR remains
            // (A = (Q Ux) S (P Q2 Vx)^T) -- one n x n QR and one n x n
            // Q-application fewer than sorting R afterwards
            std::vector<int> perm;
            DBuf dperm;
            if (spec && spec->ev && !trans && spec->src == Lp && spec->ld == ldl && spec->m == m &&
                spec->n == n) {  // started speculatively on the side stream
                HYDOT_CUDA(cudaStreamWaitEvent(c.stream, spec->ev, 0));
                spec->used = true;
                perm = std::move(spec->perm);
                dperm = std::move(spec->dperm);
                qf = std::move(spec->qf);
                if (!geqrf_verify(c, qf)) {  // a CholeskyQR panel was left: Householder panels
                    DBuf As = dalloc(c, size_t(m * n));
                    gather_cols(c, m, n, Lp, ldl, dperm.as<int>(), As.d(), m);
                    geqrf(c, m, n, As.d(), m, qf, QRCheck::Safe);
                }
            } else {
                presort_perm(c, m, n, Lp, ldl, perm);
                dperm = DBuf(c, size_t(n) * sizeof(int));
                HYDOT_CUDA(cudaMemcpyAsync(dperm.as<void>(), perm.data(), size_t(n) * sizeof(int),
                                           cudaMemcpyHostToDevice, c.stream));
                DBuf As = dalloc(c, size_t(m * n));
                gather_cols(c, m, n, Lp, ldl, dperm.as<int>(), As.d(), m);
                tmp.release();
                geqrf(c, m, n, As.d(), m, qf);
            }
            tmp.release();
            DBuf R1 = dalloc(c, size_t(n * n)), Vr = dalloc(c, size_t(n * n));
            extract_upper(c, n, qf.a.d(), m, R1.d(), n);
            svd_of_sorted_r(c, n, R1.d(), Ur.d(), o.s, Vr.d());
            scatter_rows(c, n, n, Vr.d(), n, dperm.as<int>(), o.V.d(), n);  // V = P (Q2 Vx)
            c.sync();  // host perm vector goes out of scope
        }
        // U = Q [Ur; 0]
        if (lazyU) {
            lazyU->q = std::move(qf);
            lazyU->Z = std::move(Ur);
            lazyU->zr = n;
            lazyU->set = true;
            return o;
        }
        o.U = dalloc(c, size_t(m * n));
        fill(c, m, n, 0.0, o.U.d(), m);
        copy2d(c, n, n, Ur.d(), n, o.U.d(), m);
        apply_q(c, qf, false, n, o.U.d(), m, n);
        return o;
    }
    return thin_svd(c, S, ld, trans, m, n, l, cat);  // lowrank.cpp:88-92
}
}  // namespace

SVDd fast_thin_svd(Ctx& c, const double* S, int64_t ld, bool trans, int64_t m, int64_t n,
                   Ledger* l, int cat) {
    return fast_thin_svd_impl(c, S, ld, trans, m, n, l, cat, nullptr, nullptr);
}

void wait_v(Ctx& c, const Factor& f) {
    if (!f.pending) return;
    HYDOT_CUDA(cudaStreamWaitEvent(c.stream, f.pending->ev, 0));
    f.pending->waited = true;
    f.pending.reset();  // the held inputs are released in c.stream order
}

void materialize_v(Ctx& c, Factor& f) {
    wait_v(c, f);
    if (!f.lazy) return;
    const LazyV& L = *f.lazy;
    f.V = dalloc(c, size_t(std::max<int64_t>(f.cols * f.rank, 1)));
    if (f.rank > 0) {
        fill(c, f.cols, f.rank, 0.0, f.V.d(), f.cols);
        copy2d(c, L.zr, f.rank, L.Z.d(), L.zr, f.V.d(), f.cols);
        apply_q(c, L.q, false, f.rank, f.V.d(), f.cols, L.zr);
    }
    c.sync();
    f.lazy.reset();
}

// HYDOT_SPECULATE=0: no speculative Q = I branch QR
bool speculate_on() {
    static const bool on = [] {
        const char* e = std::getenv("HYDOT_SPECULATE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// HYDOT_ASYNC_V=0 forms every non-root V in line
bool async_v_on() {
    static const bool on = [] {
        const char* e = std::getenv("HYDOT_ASYNC_V");
        return !(e && e[0] == '0');
    }();
    return on;
}

// V = Q [Z; 0] on the side stream: the next node only needs this node's
// rank (host), so its sketch / QR / Jacobi overlap the Q application (the
// small-core Jacobi leaves most SMs idle).  f.V is allocated on c.stream
// (freed in its order); the side stream starts after everything c.stream
// has issued and its temporaries live and die on the side stream; the
// Householder factor and Z stay held until a consumer waits (wait_v).
void materialize_v_async(Ctx& c, Factor& f) {
    if (!f.lazy) return;
    if (!async_v_on() || f.rank == 0) {
        materialize_v(c, f);
        return;
    }
    const std::shared_ptr<LazyV> L = f.lazy;
    f.V = dalloc(c, size_t(f.cols * f.rank));
    cudaEvent_t start = nullptr;
    HYDOT_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    HYDOT_CUDA(cudaEventRecord(start, c.stream));
    cudaStream_t main = c.stream, side = c.side_stream();
    HYDOT_CUDA(cudaStreamWaitEvent(side, start, 0));
    cudaEventDestroy(start);  // released once recorded work completes
    auto pend = std::make_shared<Factor::Pending>();
    pend->hold = L;
    c.stream = side;
    try {
        fill(c, f.cols, f.rank, 0.0, f.V.d(), f.cols);
        copy2d(c, L->zr, f.rank, L->Z.d(), L->zr, f.V.d(), f.cols);
        apply_q(c, L->q, false, f.rank, f.V.d(), f.cols, L->zr);
        HYDOT_CUDA(cudaEventCreateWithFlags(&pend->ev, cudaEventDisableTiming));
        HYDOT_CUDA(cudaEventRecord(pend->ev, side));
    } catch (...) {
        c.stream = main;
        throw;
    }
    c.stream = main;
    f.lazy.reset();
    f.pending = pend;
}

// HYDOT_TRACE_RANDSVD=1: one stderr line per sketch pass / Q = I decision
bool trace_randsvd() {
    const char* e = std::getenv("HYDOT_TRACE_RANDSVD");
    return e && e[0] == '1';
}

namespace {
Factor randsvd_impl(Ctx& c, int64_t m, int64_t n, const double* At, int64_t lda, const LinOpDev* op,
                    double eps, int p, int kprobe, uint64_t seed, Ledger* l, int cat, int r0,
                    bool lazy_v);

// what fast_thin_svd charges for an m x n matrix (lowrank.cpp:62-93)
double fast_thin_svd_flops(double m, double n) {
    if (n >= 2 * m && m > 0) return fast_thin_svd_flops(n, m);
    if (m >= 2 * n && n > 0) return 2.0 * qr_flops(m, n) + svd_flops(n, n);
    return svd_flops(m, n);
}

// HYDOT_REJECT_BOUND=0: every sketch pass is evaluated in full (read per
// call: the parity test runs both ways in one process)
bool reject_bound_on() {
    const char* e = std::getenv("HYDOT_REJECT_BOUND");
    return !(e && e[0] == '0');
}
// candidate ranks from which the bound is tried: below, the p extra columns
// of Y capture too much of the residual for the bound to decide
constexpr int64_t kRejectBoundMinRank = 600;
constexpr double kRejectMargin = 1.05;
constexpr int kPowerIters = 40;

// A sketch pass that will be rejected, decided without the SVD of Y.  The
// reference tests er = |P - Q Q^T P|_F against eps sigma_1(Y) with Q the r
// leading left singular vectors of Y (lowrank.cpp:167-176).  range(Q) lies in
// range(Y), so with the Householder QR Y = Q_Y R
//     er >= lb = |(Q_Y^T P)[rs:m, :]|_F,
// and sigma_1(Y) comes from a power iteration on Y^T Y (|Y^T Y x| with unit
// x, a lower estimate that must have settled to 2e-3).  The caller rejects
// when lb > 1.05 eps sigma_est: the same decision as the reference's, at the
// cost of one QR instead of the QR + Jacobi SVD + two Q applications.  A
// pass the bound cannot decide is evaluated in full.
bool sketch_lower_bound(Ctx& c, int64_t m, int64_t rs, int kprobe, const double* YP, double& lb, double& sig) {
    StageTimer _t(c, "reject_bound", m, rs);
    if (m <= rs) return false;
    QRFact qf;
    geqrf(c, m, rs, YP, m, qf);
    DBuf Pc = dalloc(c, size_t(m * kprobe));
    copy2d(c, m, kprobe, YP + m * rs, m, Pc.d(), m);
    apply_q(c, qf, true, kprobe, Pc.d(), m);
    DBuf zero = dalloc(c, size_t((m - rs) * kprobe));
    fill(c, m - rs, kprobe, 0.0, zero.d(), m - rs);
    DBuf x = dalloc(c, size_t(rs)), y = dalloc(c, size_t(m)), hist = dalloc(c, size_t(kPowerIters));
    fill(c, rs, 1, 1.0, x.d(), rs);
    for (int it = 0; it < kPowerIters; ++it) {
        skinny_nn(c, m, rs, 1, YP, m, x.d(), rs, y.d(), m);   // y = Y x
        skinny_tn(c, m, rs, 1, YP, m, y.d(), m, x.d(), rs);   // x = Y^T y
        normalize(c, rs, x.d(), hist.d() + it);               // |Y^T Y x_it| -> sigma_1^2 from below
    }
    lb = frob_diff(c, m - rs, kprobe, Pc.d() + rs, m, zero.d(), m - rs);
    std::vector<double> h(static_cast<size_t>(kPowerIters));
    c.d2h(h.data(), hist.d(), h.size());
    const double last = h.back(), before = h[size_t(kPowerIters - 9)];
    if (!(last > 0.0) || !std::isfinite(last) || !std::isfinite(lb)) return false;
    if (last > before * (1.0 + 2e-3)) return false;  // not settled
    sig = std::sqrt(last);
    return true;
}
}

Factor randsvd(Ctx& c, int64_t m, int64_t n, const double* At, int64_t lda, double eps, int p,
               int kprobe, uint64_t seed, Ledger* l, int cat, int r0, bool lazy_v) {
    return randsvd_impl(c, m, n, At, lda, nullptr, eps, p, kprobe, seed, l, cat, r0, lazy_v);
}

Factor randsvd(Ctx& c, const LinOpDev& A, double eps, int p, int kprobe, uint64_t seed, Ledger* l,
               int cat, int r0) {
    if (A.rows > 0 && A.cols > 0 && (!A.mm || !A.rmm))
        throw std::invalid_argument("randsvd: operator without products");
    return randsvd_impl(c, A.rows, A.cols, nullptr, 0, &A, eps, p, kprobe, seed, l, cat, r0, false);
}

namespace {
// At != nullptr: dense operator (row-major A); else the callbacks of *op
Factor randsvd_impl(Ctx& c, int64_t m, int64_t n, const double* At, int64_t lda, const LinOpDev* op,
                    double eps, int p, int kprobe, uint64_t seed, Ledger* l, int cat, int r0,
                    bool lazy_v) {
    Factor f;
    f.rows = m;
    f.cols = n;
    f.tol = eps;
    f.method = HYDOT_METHOD_RANDSVD;
    if (m == 0 || n == 0) return f;  // lowrank.cpp:148-152
    if (p < 0 || kprobe < 1) throw std::invalid_argument("randsvd: p >= 0 and kprobe >= 1 required");
    const int64_t nmax = std::min(m, n);
    int64_t r = std::clamp<int64_t>(r0, 1, nmax);
    std::unique_ptr<RngStream> rng;
    SVDd svdY;
    DBuf YP;
    int64_t qc = 0;
    bool identity = false;
    // Speculation: when the first sketch pass will be followed, if rejected,
    // by Q = I (the doubled rank reaches nmax) -- nearly every call of the
    // path -- the Q = I branch's presorted tall QR of A^T starts now on the
    // side stream, beside the sketch pass.  An accepted pass discards it.
    std::unique_ptr<TallSpec> spec;
    {
        const int64_t r1 = r, rs1 = std::min<int64_t>(r1 + p, nmax);
        const int64_t r2 = std::min<int64_t>(2 * r1, nmax), rs2 = std::min<int64_t>(r2 + p, nmax);
        // the speculative copy + factor hold 2 n m doubles beside the pass:
        // capped at 16 GB (config 1's root needs 3.8 GB); cudaMemGetInfo is
        // not used here -- it cost 2 % of the step and most of the e2e overlap
        const bool small = double(n) * double(m) * 16.0 <= 16.0 * double(1ull << 30);
        if (At && !(rs1 >= nmax && m <= n) && rs2 >= nmax && m <= n && n >= 2 * m && m > 48 && small &&
            async_v_on() && speculate_on()) {
            // speculation is optional: if its buffers do not fit, run without it
            try {
                spec.reset(new TallSpec());
                spec->c = &c;
                spec->src = At;
                spec->ld = lda;
                spec->m = n;
                spec->n = m;
                presort_perm(c, n, m, At, lda, spec->perm);
                spec->dperm = DBuf(c, size_t(m) * sizeof(int));
                HYDOT_CUDA(cudaMemcpyAsync(spec->dperm.as<void>(), spec->perm.data(), size_t(m) * sizeof(int),
                                           cudaMemcpyHostToDevice, c.stream));
                spec->qf.a = dalloc(c, size_t(n * m));  // on c.stream: freed in its order
                spec->qf.tau = dalloc(c, size_t(m));
                spec->qf.T = dalloc(c, size_t(kQRBlock) * size_t(m));
            } catch (const std::bad_alloc&) {
                spec.reset();  // no event yet: nothing was issued on the side stream
            }
        }
        if (spec) {
            cudaEvent_t start;
            HYDOT_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
            HYDOT_CUDA(cudaEventRecord(start, c.stream));
            cudaStream_t main = c.stream, side = c.side_stream();
            HYDOT_CUDA(cudaStreamWaitEvent(side, start, 0));
            cudaEventDestroy(start);
            c.stream = side;
            try {
                DBuf As = dalloc(c, size_t(n * m));
                gather_cols(c, n, m, At, lda, spec->dperm.as<int>(), As.d(), n);
                geqrf(c, n, m, As.d(), n, spec->qf, QRCheck::Deferred);  // verified by the consumer
                HYDOT_CUDA(cudaEventCreateWithFlags(&spec->ev, cudaEventDisableTiming));
                HYDOT_CUDA(cudaEventRecord(spec->ev, side));
            } catch (const std::bad_alloc&) {
                // the side stream may still write spec's buffers (allocated in
                // c.stream order): finish it before they are released
                c.stream = main;
                cudaStreamSynchronize(side);
                spec.reset();
            } catch (...) {
                c.stream = main;
                cudaStreamSynchronize(side);
                throw;
            }
            c.stream = main;
        }
    }
    while (true) {
        const int64_t rs = std::min<int64_t>(r + p, nmax);
        if (rs >= nmax && m <= n) {  // lowrank.cpp:159-164: Q = I_m
            if (trace_randsvd())
                fprintf(stderr, "[randsvd] m=%lld n=%lld r=%lld identity\n", (long long)m, (long long)n,
                        (long long)r);
            identity = true;
            break;
        }
        if (!rng) rng.reset(new RngStream(c, seed));
        const int64_t w = rs + kprobe;
        const double* Om = rng->take(n * w);  // [Omega1 | Omega2], n x (rs+k)
        YP = dalloc(c, size_t(m * w));
        if (At)
            dgemm(c, true, false, m, w, n, 1.0, At, lda, Om, n, 0.0, YP.d(), m);
        else
            op->mm(w, Om, YP.d());  // [Y | P] = A [Omega1 | Omega2]
        charge(l, cat, 2.0 * double(m) * double(n) * double(rs));      // apply_mm Y
        charge(l, cat, 2.0 * double(m) * double(n) * double(kprobe));  // apply_mm P
        if (r < nmax && r >= kRejectBoundMinRank && reject_bound_on()) {
            double lb = 0.0, sig = 0.0;
            const bool ok = sketch_lower_bound(c, m, rs, kprobe, YP.d(), lb, sig);
            const bool reject = ok && lb > kRejectMargin * eps * sig;
            if (trace_randsvd())
                fprintf(stderr, "[randsvd] m=%lld n=%lld r=%lld rs=%lld er>=%.3e thr~%.3e %s\n", (long long)m,
                        (long long)n, (long long)r, (long long)rs, lb, eps * sig,
                        reject ? "reject (bound)" : "undecided");
            if (reject) {
                // the reference's pass: SVD of Y, Q^T P, Q (Q^T P) (lowrank.cpp:167-175)
                const double q = double(std::min<int64_t>(r, rs));
                charge(l, cat, fast_thin_svd_flops(double(m), double(rs)));
                charge(l, cat, 2.0 * q * double(kprobe) * double(m));
                charge(l, cat, 2.0 * double(m) * double(kprobe) * q);
                r = std::min<int64_t>(2 * r, nmax);  // :181
                continue;
            }
        }
        svdY = fast_thin_svd(c, YP.d(), m, false, m, rs, l, cat);
        qc = std::min<int64_t>(r, svdY.k);
        const double sigma_top = svdY.s.empty() ? 0.0 : svdY.s[0];
        const double* Q = svdY.U.d();
        const double* P = YP.d() + m * rs;
        DBuf QtP = dalloc(c, size_t(std::max<int64_t>(qc * kprobe, 1)));
        DBuf QQtP = dalloc(c, size_t(m * kprobe));
        dgemm(c, true, false, qc, kprobe, m, 1.0, Q, m, P, m, 0.0, QtP.d(), qc);
        charge(l, cat, 2.0 * double(qc) * double(kprobe) * double(m));
        dgemm(c, false, false, m, kprobe, qc, 1.0, Q, m, QtP.d(), qc, 0.0, QQtP.d(), m);
        charge(l, cat, 2.0 * double(m) * double(kprobe) * double(qc));
        const double er = frob_diff(c, m, kprobe, P, m, QQtP.d(), m);
        if (trace_randsvd())
            fprintf(stderr, "[randsvd] m=%lld n=%lld r=%lld rs=%lld er=%.3e thr=%.3e %s\n", (long long)m,
                    (long long)n, (long long)r, (long long)rs, er, eps * sigma_top,
                    er <= eps * sigma_top ? "accept" : "reject");
        if (er <= eps * sigma_top) break;  // lowrank.cpp:176
        if (r >= nmax) {                   // :177-180
            f.flagged = true;
            break;
        }
        r = std::min<int64_t>(2 * r, nmax);  // :181
    }
    // B = (A^T Q)^T (lowrank.cpp:184), held as B^T (n x qc)
    DBuf Bt;
    const double* Btp;
    int64_t ldb;
    if (identity && At) {
        qc = m;
        Btp = At;  // A^T I = A^T (exact)
        ldb = lda;
    } else if (identity) {
        qc = m;
        DBuf I = dalloc(c, size_t(m * m));
        set_identity(c, m, m, I.d(), m);
        Bt = dalloc(c, size_t(n * m));
        op->rmm(m, I.d(), Bt.d());  // apply_mm(A, I, true)
        Btp = Bt.d();
        ldb = n;
    } else {
        Bt = dalloc(c, size_t(n * qc));
        if (At)
            dgemm(c, false, false, n, qc, m, 1.0, At, lda, svdY.U.d(), m, 0.0, Bt.d(), n);
        else
            op->rmm(qc, svdY.U.d(), Bt.d());
        Btp = Bt.d();
        ldb = n;
    }
    charge(l, cat, 2.0 * double(m) * double(n) * double(qc));
    // V of the tall branch always comes back implicit (Q [Ur; 0]): only the
    // kept columns are then formed (or, with lazy_v, none until first use)
    auto lz = std::make_shared<LazyV>();
    SVDd svdB = fast_thin_svd_impl(c, Btp, ldb, true, qc, n, l, cat, nullptr, lz.get(), identity ? spec.get() : nullptr);
    const std::vector<double>& s = svdB.s;
    const double s1 = s.empty() ? 0.0 : s[0];
    int64_t keep = 0;
    for (size_t i = 0; i < s.size(); ++i)
        if (s[i] > eps * s1 && s[i] > 0) keep = int64_t(i) + 1;  // :187-190
    f.rank = keep;
    f.U = dalloc(c, size_t(std::max<int64_t>(m * keep, 1)));
    if (!lz->set) f.V = dalloc(c, size_t(std::max<int64_t>(n * keep, 1)));
    if (keep > 0) {
        if (identity) {
            copy2d(c, m, keep, svdB.U.d(), qc, f.U.d(), m);  // I * U (exact)
        } else {
            dgemm(c, false, false, m, keep, qc, 1.0, svdY.U.d(), m, svdB.U.d(), qc, 0.0, f.U.d(),
                  m);  // :191
        }
        DBuf sd = dalloc(c, size_t(keep));
        HYDOT_CUDA(cudaMemcpyAsync(sd.d(), s.data(), size_t(keep) * 8, cudaMemcpyHostToDevice,
                                   c.stream));
        if (lz->set) {  // V = Q [Ur[:, :keep] S; 0], kept implicit
            DBuf Z = dalloc(c, size_t(lz->zr * keep));
            copy2d(c, lz->zr, keep, lz->Z.d(), lz->zr, Z.d(), lz->zr);
            scale_cols(c, lz->zr, keep, Z.d(), lz->zr, sd.d());
            lz->Z = std::move(Z);
            f.lazy = lz;
        } else {
            copy2d(c, n, keep, svdB.V.d(), n, f.V.d(), n);  // :192
            scale_cols(c, n, keep, f.V.d(), n, sd.d());
        }
        c.sync();
    } else if (lz->set) {
        f.V = dalloc(c, 1);
    }
    charge(l, cat, 2.0 * double(m) * double(keep) * double(qc));
    charge(l, cat, 1.0 * double(n) * double(keep));  // :193-197
    if (!lazy_v) materialize_v_async(c, f);
    return f;
}
}  // namespace

Factor agglomerate(Ctx& c, const Factor& f1, const Factor& f2, double eps, uint64_t seed,
                   Ledger* l, int rank_hint, int p, int kprobe, bool lazy_v) {
    if (f1.lazy || f2.lazy) throw std::runtime_error("agglomerate: factor V not materialised");
    if (f1.cols != f2.cols)
        throw std::invalid_argument("agglomerate: column dimension mismatch");  // :324-325
    const int64_t n = f1.cols, r1 = f1.rank, r2 = f2.rank, m1 = f1.rows, m2 = f2.rows;
    Factor out;
    out.rows = m1 + m2;
    out.cols = n;
    out.tol = eps;
    out.method = HYDOT_METHOD_AGGLOMERATE;
    if (r1 + r2 == 0) {  // :333-337 (the reference returns flagged = false here)
        return out;
    }
    wait_v(c, f1);
    wait_v(c, f2);
    // W = [V1^T; V2^T] held as W^T = [V1 V2] (n x (r1+r2))  :339-341
    DBuf Wt = dalloc(c, size_t(n * (r1 + r2)));
    copy2d(c, n, r1, f1.V.d(), n, Wt.d(), n);
    copy2d(c, n, r2, f2.V.d(), n, Wt.d() + n * r1, n);
    const int hint = int(std::max<int64_t>({r1, r2, int64_t(rank_hint)}));
    Factor inner = randsvd(c, r1 + r2, n, Wt.d(), n, eps, p, kprobe, seed, l,
                           HYDOT_CAT_AGGLOMERATION, hint, lazy_v);  // :344-346
    Wt.release();
    const int64_t rp = inner.rank;
    out.rank = rp;
    out.U = dalloc(c, size_t(std::max<int64_t>((m1 + m2) * rp, 1)));
    if (rp > 0) {  // :349-356
        dgemm(c, false, false, m1, rp, r1, 1.0, f1.U.d(), m1, inner.U.d(), r1 + r2, 0.0, out.U.d(),
              m1 + m2);
        charge(l, HYDOT_CAT_AGGLOMERATION, 2.0 * double(m1) * double(rp) * double(r1));
        dgemm(c, false, false, m2, rp, r2, 1.0, f2.U.d(), m2, inner.U.d() + r1, r1 + r2, 0.0,
              out.U.d() + m1, m1 + m2);
        charge(l, HYDOT_CAT_AGGLOMERATION, 2.0 * double(m2) * double(rp) * double(r2));
    }
    out.V = std::move(inner.V);
    out.lazy = std::move(inner.lazy);
    out.pending = std::move(inner.pending);
    out.flagged = f1.flagged || f2.flagged || inner.flagged;  // :357
    return out;
}

Factor recompress(Ctx& c, const Factor& f, double eps, int rank, Ledger* l) {
    const int64_t r = f.rank, M = f.rows, N = f.cols;
    Factor out;
    out.rows = M;
    out.cols = N;
    out.tol = eps;
    out.method = HYDOT_METHOD_RECOMPRESS;
    out.flagged = f.flagged;
    if (r == 0) return out;  // :554-558
    if (M < r || N < r) throw std::invalid_argument("recompress: rank exceeds a factor dimension");
    charge(l, HYDOT_CAT_RECOMPRESS, qr_flops(double(M), double(r)) + qr_flops(double(N), double(r)));
    // V = Q_W [Z; 0] (lazy root): QR(V) = Q_W blkdiag(Q_Z, I) [R_Z; 0], so
    // only the small zr x r Z is factored and Q_W is applied once at the end
    wait_v(c, f);
    const LazyV* lv = f.lazy.get();
    QRFact qu, qv;
    // the two QRs are independent and latency-bound: QR(U) runs on the side
    // stream next to QR(V) (or QR(Z)); `side_done` orders the frees of qu
    // (allocated on the side stream) after every use on c.stream
    cudaStream_t main = c.stream;
    // the first attempt of either QR launches no cooperative kernel (tall
    // panels by CholeskyQR, short ones in one CTA); a Householder redo runs
    // on the main stream after the join (qu) or beside ordinary kernels (qv)
    const bool overlap = async_v_on();
    struct SideJoin {
        Ctx& c;
        cudaStream_t main;
        bool on;
        ~SideJoin() {
            if (!on) return;
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
                cudaEventRecord(e, main);
                cudaStreamWaitEvent(c.side, e, 0);
                cudaEventDestroy(e);
            }
        }
    } side_done{c, main, overlap};
    cudaEvent_t ev_u = nullptr;
    struct Unchain {
        Ctx& c;
        bool prev;
        Unchain(Ctx& cc, bool on) : c(cc), prev(cc.coop_unchained) { c.coop_unchained = prev || on; }
        ~Unchain() { c.coop_unchained = prev; }
    } unchain{c, overlap};  // both panel grids fit the device together (checked above)
    if (overlap) {
        cudaEvent_t ev0;
        HYDOT_CUDA(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
        HYDOT_CUDA(cudaEventRecord(ev0, main));
        HYDOT_CUDA(cudaStreamWaitEvent(c.side_stream(), ev0, 0));
        cudaEventDestroy(ev0);
        c.stream = c.side;
        try {
            geqrf(c, M, r, f.U.d(), M, qu, QRCheck::Deferred);  // :564 (verified after the join)
        } catch (...) {
            c.stream = main;
            throw;
        }
        HYDOT_CUDA(cudaEventCreateWithFlags(&ev_u, cudaEventDisableTiming));
        HYDOT_CUDA(cudaEventRecord(ev_u, c.side));
        c.stream = main;
    } else {
        geqrf(c, M, r, f.U.d(), M, qu);  // :564
    }
    if (lv)
        geqrf(c, lv->zr, r, lv->Z.d(), lv->zr, qv);
    else
        geqrf(c, N, r, f.V.d(), N, qv);
    if (ev_u) {
        HYDOT_CUDA(cudaStreamWaitEvent(main, ev_u, 0));
        cudaEventDestroy(ev_u);
        if (!geqrf_verify(c, qu)) geqrf(c, M, r, f.U.d(), M, qu, QRCheck::Safe);
    }
    c.coop_unchained = unchain.prev;  // later cooperative launches chain again
    const int64_t vm = lv ? lv->zr : N;
    DBuf Ru = dalloc(c, size_t(r * r)), Rv = dalloc(c, size_t(r * r)), core = dalloc(c, size_t(r * r));
    extract_upper(c, r, qu.a.d(), M, Ru.d(), r);
    extract_upper(c, r, qv.a.d(), vm, Rv.d(), r);
    dgemm(c, false, true, r, r, r, 1.0, Ru.d(), r, Rv.d(), r, 0.0, core.d(), r);  // :567
    charge(l, HYDOT_CAT_RECOMPRESS, 2.0 * double(r) * double(r) * double(r));
    // The core of a factor whose U / V columns are already orthogonal (every
    // factor the recursion produces) is diagonal to rounding: Jacobi then
    // converges in 1-2 sweeps on it directly and the QR preconditioning
    // (sort + two r x r QRs) is skipped.  General cores keep it.
    SVDd svd;
    if (r > 48 && offdiag_ratio(c, r, core.d(), r) < 1e-8) {
        charge(l, HYDOT_CAT_RECOMPRESS, svd_flops(double(r), double(r)));  // as thin_svd
        svd.m = svd.n = svd.k = r;
        svd.U = dalloc(c, size_t(r * r));
        svd.V = dalloc(c, size_t(r * r));
        jacobi_svd(c, r, r, core.d(), r, svd.U.d(), r, svd.s, svd.V.d(), r);
    } else {
        svd = thin_svd(c, core.d(), r, false, r, r, l, HYDOT_CAT_RECOMPRESS);  // :568
    }
    const std::vector<double>& s = svd.s;
    const double s1 = s.empty() ? 0.0 : s[0];
    int64_t keep;
    if (rank >= 0) {
        keep = std::min<int64_t>(rank, int64_t(s.size()));
    } else {
        keep = 0;
        for (size_t i = 0; i < s.size(); ++i)
            if (s[i] > eps * s1 && s[i] > 0) keep = int64_t(i) + 1;
    }
    out.rank = keep;
    // U = Q_U [U~_k; 0], V = Q_V [V~_k S_k; 0]  (:579-585)
    out.U = dalloc(c, size_t(std::max<int64_t>(M * keep, 1)));
    out.V = dalloc(c, size_t(std::max<int64_t>(N * keep, 1)));
    if (keep > 0) {
        fill(c, M, keep, 0.0, out.U.d(), M);
        copy2d(c, r, keep, svd.U.d(), r, out.U.d(), M);
        apply_q(c, qu, false, keep, out.U.d(), M, r);
        DBuf sd = dalloc(c, size_t(keep));
        HYDOT_CUDA(cudaMemcpyAsync(sd.d(), s.data(), size_t(keep) * 8, cudaMemcpyHostToDevice,
                                   c.stream));
        if (lv) {
            DBuf small = dalloc(c, size_t(vm * keep));  // Q_Z [V~_k S_k; 0]
            fill(c, vm, keep, 0.0, small.d(), vm);
            copy2d(c, r, keep, svd.V.d(), r, small.d(), vm);
            scale_cols(c, r, keep, small.d(), vm, sd.d());
            apply_q(c, qv, false, keep, small.d(), vm, r);
            fill(c, N, keep, 0.0, out.V.d(), N);
            copy2d(c, vm, keep, small.d(), vm, out.V.d(), N);
            apply_q(c, lv->q, false, keep, out.V.d(), N, vm);
        } else {
            fill(c, N, keep, 0.0, out.V.d(), N);
            copy2d(c, r, keep, svd.V.d(), r, out.V.d(), N);
            scale_cols(c, r, keep, out.V.d(), N, sd.d());
            apply_q(c, qv, false, keep, out.V.d(), N, r);
        }
        c.sync();
    }
    charge(l, HYDOT_CAT_RECOMPRESS, 2.0 * double(M) * double(keep) * double(r));
    charge(l, HYDOT_CAT_RECOMPRESS, 2.0 * double(N) * double(keep) * double(r));
    return out;
}

// ------------------------------------------------------------------ tree --
int Tree::depth() const {  // lowrank.cpp:361-368
    std::function<int(int)> go = [&](int v) -> int {
        const TreeNode& nd = nodes[size_t(v)];
        return nd.is_leaf() ? 0 : 1 + std::max(go(nd.left), go(nd.right));
    };
    return nodes.empty() ? 0 : go(root);
}

std::vector<int> Tree::leaf_order() const {  // lowrank.cpp:370-383
    std::vector<int> out;
    std::function<void(int)> go = [&](int v) {
        const TreeNode& nd = nodes[size_t(v)];
        if (nd.is_leaf()) {
            out.insert(out.end(), nd.idx.begin(), nd.idx.end());
        } else {
            go(nd.left);
            go(nd.right);
        }
    };
    if (!nodes.empty()) go(root);
    return out;
}

// geometric bisection (lowrank.cpp:385-438): widest extent (ties -> lowest
// axis), "<= midpoint" goes left, <= 2 sources per leaf, median fallback.
Tree build_cluster_tree(const double* pos, int n, int d, const double* lo, const double* hi) {
    if (n < 1) throw std::invalid_argument("build_cluster_tree: no sources");
    if (d < 1) throw std::invalid_argument("build_cluster_tree: box dimension");
    Tree t;
    auto P = [&](int i, int j) { return pos[i + int64_t(j) * n]; };
    std::function<int(std::vector<int>, std::vector<double>, std::vector<double>)> rec =
        [&](std::vector<int> idx, std::vector<double> a, std::vector<double> b) -> int {
        const int me = int(t.nodes.size());
        t.nodes.push_back(TreeNode{idx, -1, -1, a, b});
        if (idx.size() <= 2) return me;
        int ax = 0;
        for (int j = 1; j < d; ++j)
            if (b[size_t(j)] - a[size_t(j)] > b[size_t(ax)] - a[size_t(ax)]) ax = j;
        const double mid = 0.5 * (a[size_t(ax)] + b[size_t(ax)]);
        std::vector<int> left, right;
        for (int i : idx) {
            if (P(i, ax) <= mid) left.push_back(i);
            else right.push_back(i);
        }
        std::vector<double> bl = b, ar = a;
        bl[size_t(ax)] = mid;
        ar[size_t(ax)] = mid;
        if (left.empty() || right.empty()) {
            std::vector<int> srt = idx;
            std::stable_sort(srt.begin(), srt.end(), [&](int x, int y) { return P(x, ax) < P(y, ax); });
            const size_t h = srt.size() / 2;
            left.assign(srt.begin(), srt.begin() + long(h));
            right.assign(srt.begin() + long(h), srt.end());
            bl = b;
            ar = a;
        }
        const int lc = rec(std::move(left), a, bl);
        const int rc = rec(std::move(right), ar, b);
        t.nodes[size_t(me)].left = lc;
        t.nodes[size_t(me)].right = rc;
        return me;
    };
    std::vector<int> all(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) all[size_t(i)] = i;
    t.root = rec(all, std::vector<double>(lo, lo + d), std::vector<double>(hi, hi + d));
    return t;
}

double tolerance_schedule(double eps_d, int L, int N_r) {  // lowrank.cpp:540-545
    if (eps_d <= 0 || L < 0 || N_r < 1)
        throw std::invalid_argument("tolerance_schedule: bad arguments");
    return eps_d / (std::pow(2.0, 0.5 * L) * (L + 1) * std::sqrt(double(N_r)));
}

// recursive_lowrank (lowrank.cpp:459-521) with the reference's warm-start
// chains (leaf_hint across leaves in DFS order, depth_hint per depth).
RecOut recursive_lowrank(Ctx& c, const Tree& t, double eps, int rows_per, int64_t cols,
                         const BlockFn& block, uint64_t seed, int p, int kprobe,
                         const std::vector<int>& source_ids, int node_offset, bool lazy_root) {
    auto gsrc = [&](int s) { return source_ids.empty() ? s : source_ids[size_t(s)]; };
    RecOut res;
    res.node_rank.assign(t.nodes.size(), -1);
    res.node_depth.assign(t.nodes.size(), 0);
    int leaf_hint = -1;
    std::map<int, int> depth_hint;
    auto node_hint = [&](int depth) {
        auto it = depth_hint.find(depth);
        return it == depth_hint.end() ? -1 : it->second + 2;
    };
    DBuf blk = dalloc(c, size_t(rows_per) * size_t(cols));
    std::function<Factor(int, int)> go = [&](int v, int depth) -> Factor {
        const TreeNode& nd = t.nodes[size_t(v)];
        res.node_depth[size_t(v)] = depth;
        Factor f;
        try {
            if (nd.is_leaf()) {
                std::vector<Factor> parts;
                const bool lazy_here = lazy_root && v == t.root;
                for (int s : nd.idx) {
                    block(s, blk.d(), cols);
                    parts.push_back(randsvd(c, rows_per, cols, blk.d(), cols, eps, p, kprobe,
                                            seed + 0x9e3779b97f4a7c15ULL * uint64_t(gsrc(s) + 1),
                                            &res.ledger, HYDOT_CAT_LEAF,
                                            std::max(1, leaf_hint + 2), lazy_here && nd.idx.size() == 1));
                    leaf_hint = int(parts.back().rank);
                }
                if (parts.empty()) throw std::runtime_error("empty leaf cluster");
                f = std::move(parts[0]);
                for (size_t i = 1; i < parts.size(); ++i)
                    f = agglomerate(c, f, parts[i], eps,
                                    seed + 0x517cc1b727220a95ULL * uint64_t(node_offset + v + 1), &res.ledger,
                                    node_hint(depth), p, kprobe, lazy_here && i + 1 == parts.size());
            } else {
                Factor fl = go(nd.left, depth + 1);
                Factor fr = go(nd.right, depth + 1);
                f = agglomerate(c, fl, fr, eps, seed + 0x2545f4914f6cdd1dULL * uint64_t(node_offset + v + 1),
                                &res.ledger, node_hint(depth), p, kprobe, lazy_root && v == t.root);
            }
        } catch (const CudaError&) {
            throw;
        } catch (const std::bad_alloc&) {
            throw;
        } catch (const std::exception& e) {
            throw std::runtime_error("recursive_lowrank at node " + std::to_string(v) + ": " +
                                     e.what());
        }
        res.node_rank[size_t(v)] = int(f.rank);
        depth_hint[depth] = int(f.rank);
        return f;
    };
    res.factor = go(t.root, 0);
    res.factor.method = HYDOT_METHOD_RECURSIVE;
    res.factor.tol = eps;
    res.source_order = t.leaf_order();
    for (int s : res.source_order)
        for (int q = 0; q < rows_per; ++q) res.row_perm.push_back(gsrc(s) * rows_per + q);
    return res;
}

}  // namespace hydot
