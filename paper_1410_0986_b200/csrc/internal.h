// internal.h -- shared host-side declarations of the B200 hydot library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hydot_b200.h"

namespace hydot {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define HYDOT_CUDA(call)                                                                   \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw ::hydot::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct RngTables;

// Function attributes (cudaFuncSetAttribute) are per device: a call site
// sets them once for every device a context of this process uses, under a
// lock (contexts on several GPUs may run on different host threads).
struct AttrGate {
    std::mutex mu;
    uint64_t done = 0;
};
template <class F>
void attr_once(AttrGate& g, int device, F&& set) {
    std::lock_guard<std::mutex> lk(g.mu);
    const uint64_t bit = 1ull << (device & 63);
    if (!(g.done & bit)) {
        set();
        g.done |= bit;
    }
}

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    // side stream for work whose result is consumed later (the V of a
    // finished node while the next node's decisions run); created on demand
    cudaStream_t side = nullptr;
    cudaStream_t side_stream() {
        if (!side) HYDOT_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        return side;
    }
    // High-priority streams for the panel chain of a look-ahead QR (qr.cu):
    // [1] serves a factorisation issued on the side stream, [0] any other,
    // so that the two factorisations that may be in flight at once (the
    // speculative tall QR beside the main stream's) never queue behind each
    // other.  Created on demand.
    cudaStream_t hp[2] = {nullptr, nullptr};
    cudaStream_t hp_stream(int which) {
        if (!hp[which]) {
            int least = 0, greatest = 0;
            HYDOT_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            HYDOT_CUDA(cudaStreamCreateWithPriority(&hp[which], cudaStreamNonBlocking, greatest));
        }
        return hp[which];
    }
    // Memory pools.  By default every stream allocates from the device's
    // default pool.  HYDOT_STREAM_POOLS=1 gives the side stream and the
    // high-priority streams pools of their own: a block freed in one stream's
    // order can serve another stream only once that free has completed, and
    // separate pools take that cross-stream reuse (and the waits it can
    // insert when the device memory is exhausted) out of the picture.
    // Measured on the config-2 step: no effect on the step time (the default
    // pool's high-water mark is 82 GB either way, the side pool adds 6.7 GB),
    // so it stays off: config 2 with its 55 GB of fields leaves little room.
    cudaMemPool_t side_pool = nullptr, hp_pool = nullptr;
    cudaMemPool_t make_pool() {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t p = nullptr;
        HYDOT_CUDA(cudaMemPoolCreate(&p, &props));
        uint64_t thr = UINT64_MAX;  // keep freed memory cached
        HYDOT_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr));
        return p;
    }
    // the pool that serves allocations ordered on s (nullptr: the default pool)
    cudaMemPool_t pool_for(cudaStream_t s) {
        static const bool on = [] {
            const char* e = std::getenv("HYDOT_STREAM_POOLS");
            return e && e[0] == '1';
        }();
        if (!on || !s) return nullptr;
        if (s == side) {
            if (!side_pool) side_pool = make_pool();
            return side_pool;
        }
        if (s == hp[0] || s == hp[1]) {
            if (!hp_pool) hp_pool = make_pool();
            return hp_pool;
        }
        return nullptr;
    }
    // Cooperative launches of both streams form one chain (each waits for
    // the previous one to finish): a cooperative grid then only ever shares
    // the GPU with ordinary kernels, which always complete, so two partially
    // resident grids can never wait on each other.  coop_unchained: the
    // caller has proven that the grids in flight fit the device together.
    cudaEvent_t coop_ev = nullptr;
    bool coop_recorded = false;
    bool coop_unchained = false;
    void coop_launch(const void* kern, dim3 grid, dim3 block, void** args, size_t smem) {
        if (!coop_unchained && coop_recorded) HYDOT_CUDA(cudaStreamWaitEvent(stream, coop_ev, 0));
        HYDOT_CUDA(cudaLaunchCooperativeKernel(kern, grid, block, args, smem, stream));
        if (!coop_unchained) {
            if (!coop_ev) HYDOT_CUDA(cudaEventCreateWithFlags(&coop_ev, cudaEventDisableTiming));
            HYDOT_CUDA(cudaEventRecord(coop_ev, stream));
            coop_recorded = true;
        }
    }
    std::string err;
    int64_t launches = 0;
    int num_sms = 148;
    // host-pinned scratch for small D2H reads
    double* pinned = nullptr;
    size_t pinned_len = 0;
    // MT19937-64 jump polynomials on the device (rng.cu)
    uint64_t* jump_dev = nullptr;
    int64_t jump_n = 0;
    // live per-stage timing with CUDA events on the context stream (no
    // synchronisation; hydot_ctx_timing_report resolves them)
    bool timing = false;
    std::vector<std::string> timing_filter;  // empty = every stage
    bool timed(const char* name) const {
        if (!timing) return false;
        if (timing_filter.empty()) return true;
        for (const auto& f : timing_filter)
            if (f == name) return true;
        return false;
    }
    struct TRec {
        const char* name;
        cudaEvent_t a, b;
        double flops, bytes;
    };
    std::vector<TRec> trecs;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t take_event() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        HYDOT_CUDA(cudaEventCreate(&e));
        return e;
    }
    void count(int64_t n = 1) { launches += n; }
    void check_launch() {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw CudaError(std::string("kernel launch: ") + cudaGetErrorString(e));
        ++launches;
    }
    void sync() { HYDOT_CUDA(cudaStreamSynchronize(stream)); }
    // copy n doubles device->host through pinned scratch (synchronises)
    void d2h(double* dst, const double* src, size_t n);
};

// Stream-ordered device buffer (cudaMallocAsync / cudaFreeAsync pool).
class DBuf {
   public:
    DBuf() = default;
    DBuf(Ctx& c, size_t bytes) { alloc(c, bytes); }
    ~DBuf() { release(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept { *this = std::move(o); }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            s_ = o.s_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void alloc(Ctx& c, size_t bytes) {
        release();
        s_ = c.stream;
        n_ = bytes;
        if (bytes) {
            cudaMemPool_t pool = c.pool_for(s_);
            cudaError_t e = pool ? cudaMallocFromPoolAsync(&p_, bytes, pool, s_) : cudaMallocAsync(&p_, bytes, s_);
            if (e != cudaSuccess) {
                p_ = nullptr;
                cudaGetLastError();  // do not leave the failed allocation as the sticky last error
                throw std::bad_alloc();
            }
        }
    }
    void release() {
        if (p_) cudaFreeAsync(p_, s_);
        p_ = nullptr;
        n_ = 0;
    }
    template <class T = double>
    T* as() const {
        return static_cast<T*>(p_);
    }
    double* d() const { return static_cast<double*>(p_); }
    size_t bytes() const { return n_; }

   private:
    void* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

inline DBuf dalloc(Ctx& c, size_t n_doubles) { return DBuf(c, n_doubles * sizeof(double)); }

// Optional stage timer (HYDOT_PROFILE=1): synchronises around each scoped
// stage and accumulates wall time per name; report via hydot_profile_dump().
struct StageTimer {
    StageTimer(Ctx& c, const char* name, int64_t a = -1, int64_t b = -1, int64_t k = -1,
               double flops = 0.0, double bytes = 0.0);
    ~StageTimer();
    Ctx& c_;
    const char* name_;
    int64_t a_, b_, k_;
    double t0_ = 0;
    bool on_ = false;
    double flops_, bytes_;
    cudaEvent_t ea_ = nullptr;
};

// ---------------------------------------------------------------- ledger --
struct Ledger {
    double leaf = 0, agglomeration = 0, recompress = 0, other = 0, kernel_tally = 0;
    void charge(int cat, double f) {
        kernel_tally += f;
        switch (cat) {
            case HYDOT_CAT_LEAF: leaf += f; break;
            case HYDOT_CAT_AGGLOMERATION: agglomeration += f; break;
            case HYDOT_CAT_RECOMPRESS: recompress += f; break;
            default: other += f; break;
        }
    }
};

// --------------------------------------------------------------- kernels --
// gemm.cu
void dgemm(Ctx& c, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
           const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
           int64_t ldc);

// util.cu
void copy2d(Ctx& c, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
            int64_t ldd);
void transpose(Ctx& c, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
               int64_t ldd);  // dst (cols x rows) = src^T
void fill(Ctx& c, int64_t rows, int64_t cols, double v, double* dst, int64_t ldd);
void set_identity(Ctx& c, int64_t rows, int64_t cols, double* dst, int64_t ldd);
void scale_cols(Ctx& c, int64_t rows, int64_t cols, double* A, int64_t lda,
                const double* s_dev);  // A(:,j) *= s[j]
void extract_upper(Ctx& c, int64_t n, const double* A, int64_t lda, double* R,
                   int64_t ldr);  // R = triu(A[0:n,0:n])
void gather_cols(Ctx& c, int64_t rows, int64_t cols, const double* src, int64_t lds,
                 const int* idx_dev, double* dst, int64_t ldd);
double frob_diff(Ctx& c, int64_t rows, int64_t cols, const double* A, int64_t lda,
                 const double* B, int64_t ldb);  // ||A - B||_F (synchronises)
void col_norms(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* out_dev);
void normalize(Ctx& c, int64_t n, double* x, double* nrm_dev);  // x /= ||x||, *nrm_dev = ||x||
// ||offdiag(A)||_F / ||A||_F of an n x n matrix (synchronises)
double offdiag_ratio(Ctx& c, int64_t n, const double* A, int64_t lda);
void scatter_rows(Ctx& c, int64_t rows, int64_t cols, const double* src, int64_t lds,
                  const int* idx_dev, double* dst, int64_t ldd);  // dst[idx[i],:] = src[i,:]

// born.cu
// y[(s nd + d) nl + l] = F[s][l][det[s nd + d]] (F: ns x nl x N, device det)
void gather_measure(Ctx& c, int ns, int nd, int nl, int64_t N, const double* F, const int64_t* det_dev, double* y);
void born_block(Ctx& c, int64_t N, int nl, const double* inc, const double* const* adj_h, int nd,
                const double* w, double nu, double* out, int64_t ld);

// qr.cu : blocked Householder QR (LAPACK dgeqrf/dorgqr semantics)
struct QRFact {
    int64_t m = 0, n = 0;
    DBuf a;    // m x n: R in the upper triangle, Householder vectors below
    DBuf tau;  // n
    DBuf T;    // kQRBlock x n : block reflector triangles
    DBuf flag;  // device int: raised when a CholeskyQR panel had to be left (see geqrf)
    bool unverified = false;  // flag not read yet (QRCheck::Deferred)
};
constexpr int kQRBlock = 128;  // block-reflector width (qr.cu)
// Tall panels are factored by CholeskyQR + Householder reconstruction, which
// leaves a panel it cannot orthonormalise and raises f.flag; the
// factorisation is then redone with Householder panels (Safe).
//   Now:      the flag is read at the end (one stream synchronisation) and the redo happens inside
//   Deferred: no synchronisation; the caller must call geqrf_verify after joining the stream and,
//             when it returns false, redo with geqrf(..., QRCheck::Safe)
//   Safe:     Householder panels only
enum class QRCheck { Now, Deferred, Safe };
void geqrf(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, QRFact& f, QRCheck chk = QRCheck::Now);
bool geqrf_verify(Ctx& c, QRFact& f);  // synchronises c.stream
// Y (m x k) := Q Y (trans=false) or Q^T Y.  nz_rows >= 0 (Q Y only): Y's
// rows >= nz_rows are zero on entry (the Q [Z; 0] products).
void apply_q(Ctx& c, const QRFact& f, bool trans, int64_t k, double* Y, int64_t ldy, int64_t nz_rows = -1);

// While alive, Jacobi SVDs accumulate V for every column (full BDCSVD
// contract, e.g. hydot_thin_svd); otherwise the large driver recovers V
// from one GEMM, exact for every singular triple the path can keep.
struct StrictSVD {
    StrictSVD();
    ~StrictSVD();
    bool prev_;
};
// svd.cu : one-sided Jacobi thin SVD of X (m x n, m >= n); s descending.
void jacobi_svd(Ctx& c, int64_t m, int64_t n, const double* X, int64_t ldx, double* U,
                int64_t ldu, std::vector<double>& s, double* V, int64_t ldv);

// bjacobi.cu: block one-sided Jacobi (DMMA Gram + pair eigen-solve + DMMA
// update) to convergence on U (m x n, ld m); returns the sweep count
int bjacobi_converge(Ctx& c, int64_t m, int64_t n, double* U, double tol);
int64_t bjacobi_min_n();

// cg.cu
struct CGStats {
    std::vector<int> iters;
    std::vector<double> relres;
};
void fields_solve(Ctx& c, const hydot_grid7& g, int nl, const double* sigma,
                  const double* sigmap, const double* inv_D, const int64_t* rhs_vertex, int n_rhs,
                  double tol, int max_iter, int fixed_iters, double* out, CGStats* stats);
void apply7(Ctx& c, const hydot_grid7& g, double sigma, double sigmap, const double* x,
            double* y);
// the perturbed medium of the nonlinear forward model: per-vertex absorption
// sigma_l + dsig_l mu(v) (dsig_dev: n_lambda, mu_dev: N)
void fields_solve_var(Ctx& c, const hydot_grid7& g, int nl, const double* sigma, const double* sigmap,
                      const double* inv_D, const double* dsig_dev, const double* mu_dev, const int64_t* rhs_vertex,
                      int n_rhs, double tol, int max_iter, int fixed_iters, double* out, CGStats* stats);
// the reference's trilinear-FEM operator K + sigma M + sigma' R (grid.cpp)
void apply_fem(Ctx& c, const hydot_grid_geom& g, double sigma, double sigmap, const double* x, double* y);
void fields_solve_fem(Ctx& c, const hydot_grid_geom& g, int nl, const double* sigma, const double* sigmap,
                      const double* inv_D, const double* points, int n_pts, double tol, int max_iter,
                      int fixed_iters, double* out, CGStats* stats);

// the 8 trilinear (vertex, weight) pairs of each FEM point source (born.cpp:27-35)
void fem_point_weights(const hydot_grid_geom& g, const double* points, int n_pts, std::vector<int64_t>& ridx,
                       std::vector<double>& rw, std::vector<double>& b2);
// gmres.cu: krylov::solve_family (krylov.cpp:400-463) on the FEM operator for
// n_rhs device right-hand sides b_dev (n_rhs x N); X (original variables,
// times mult[shift] when given) at X_dev + (r * nsh + j) * x_stride
void solve_family_fem(Ctx& c, const hydot_grid_geom& g, int nsh, const double* sigma, const double* sigmap,
                      const double* b_dev, int n_rhs, const hydot_krylov_config& cfg, const double* mult,
                      double* X_dev, int64_t x_stride, hydot_krylov_stats* stats, hydot_krylov_family* fam);
// compute_fields (born.cpp:39-80) with the reference's solver on its operator
void fields_solve_fem_gmres(Ctx& c, const hydot_grid_geom& g, int nl, const double* sigma, const double* sigmap,
                            const double* inv_D, const double* points, int n_pts, const hydot_krylov_config& cfg,
                            double* out, hydot_krylov_stats* stats, hydot_krylov_family* fam);

// forward.cpp: full_diffusion_forward (experiments.cpp:154-206) for the
// 7-point operator; outputs ns x nd x nl measurements (device)
void full_forward(Ctx& c, const hydot_grid7& g, int nl, const double* sigma, const double* sigmap,
                  const double* inv_D, const double* dsigma, const double* mu_dev, const int64_t* src_h, int ns,
                  const int64_t* det_h, int nd, double tol, int max_iter, int fixed_iters, double* y_tot,
                  double* y_inc, int* iters_max);

// matmat.cu
void j_combine(Ctx& c, int64_t M, int b, int nc, int nl, const double* T, int64_t ldt,
               const int* row_perm, const double* eps_c, double* Y, int64_t ldy);
void j_gather_scale(Ctx& c, int64_t M, int b, int nc, int nl, const double* X, int64_t ldx,
                    const int* row_perm, const double* eps_c, double* G, int64_t ldg);
void j_matmat(Ctx& c, const double* U, const double* V, int64_t M, int64_t N, int64_t R, bool trans, int b,
              const int* row_perm, const double* eps_c, int nl, int nc, const double* X, int64_t ldx, double* Y,
              int64_t ldy);
void kron_conc(Ctx& c, int64_t N, int b, int nc, const double* conc_dev, const double* D, int64_t ldd,
               double* X, int64_t ldx);
void wsq_rows(Ctx& c, int64_t M, int b, const double* w, const double* X, int64_t ldx, double* Y, int64_t ldy);
// tall-skinny products for q <= 16 right-hand sides (HBM streams):
// Z (R x q) = A^T X with A K x R;  Y (M x q) = A Z with A M x R
bool skinny_ok(int q);
void skinny_tn(Ctx& c, int64_t K, int64_t R, int q, const double* A, int64_t lda, const double* X,
               int64_t ldx, double* Z, int64_t ldz);
void skinny_nn(Ctx& c, int64_t M, int64_t R, int q, const double* A, int64_t lda, const double* Z,
               int64_t ldz, double* Y, int64_t ldy);

// rng.cu
class RngStream {
   public:
    RngStream(Ctx& c, uint64_t seed);
    ~RngStream();
    // pointer to the next `count` normals of the libstdc++ stream (valid until
    // the next take()); advances the stream.
    const double* take(int64_t count);
    // fill out with normals [offset, offset+count) (random access)
    void fill(int64_t offset, int64_t count, double* out);
    void raw(int64_t offset, int64_t count, uint64_t* out);

   private:
    void ensure_normals(int64_t upto);
    void generate_chunks(int64_t c_end);
    Ctx& c_;
    uint64_t seed_;
    DBuf prefix_;       // z_0 .. z_{kPrefix-1}
    DBuf normals_;      // all normals generated so far
    int64_t n_chunks_ = 0;
    int64_t n_normals_ = 0;
    int64_t consumed_ = 0;
    DBuf total_;  // accepted pairs of all chunks so far (device; the host keeps a lower bound)
};
bool rng_selftest_host();

}  // namespace hydot
