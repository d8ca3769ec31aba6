// util.cu -- small data-movement kernels used between the hot-path stages
// (copies, transposes, column scaling, triangle extraction, norms).
#include "internal.h"

namespace hydot {
namespace {

inline int grid_for(Ctx& c, int64_t n, int threads = 256) {
    int64_t b = (n + threads - 1) / threads;
    return int(std::max<int64_t>(1, std::min<int64_t>(b, int64_t(c.num_sms) * 16)));
}

__global__ void copy2d_k(int64_t rows, int64_t cols, const double* __restrict__ s, int64_t lds,
                         double* __restrict__ d, int64_t ldd) {
    int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % rows, j = e / rows;
        d[i + j * ldd] = s[i + j * lds];
    }
}

// 32x32 tiled transpose through shared memory
__global__ void transpose_k(int64_t rows, int64_t cols, const double* __restrict__ s, int64_t lds,
                            double* __restrict__ d, int64_t ldd) {
    __shared__ double tile[32][33];
    int64_t i0 = int64_t(blockIdx.x) * 32, j0 = int64_t(blockIdx.y) * 32;
    for (int jj = threadIdx.y; jj < 32; jj += blockDim.y) {
        int64_t i = i0 + threadIdx.x, j = j0 + jj;
        if (i < rows && j < cols) tile[jj][threadIdx.x] = s[i + j * lds];
    }
    __syncthreads();
    for (int ii = threadIdx.y; ii < 32; ii += blockDim.y) {
        int64_t j = j0 + threadIdx.x, i = i0 + ii;
        if (i < rows && j < cols) d[j + i * ldd] = tile[threadIdx.x][ii];
    }
}

__global__ void fill_k(int64_t rows, int64_t cols, double v, double* d, int64_t ldd, int ident) {
    int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % rows, j = e / rows;
        d[i + j * ldd] = ident ? (i == j ? 1.0 : 0.0) : v;
    }
}

__global__ void scale_cols_k(int64_t rows, int64_t cols, double* A, int64_t lda,
                             const double* __restrict__ s) {
    int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % rows, j = e / rows;
        A[i + j * lda] *= s[j];
    }
}

__global__ void upper_k(int64_t n, const double* __restrict__ A, int64_t lda, double* R,
                        int64_t ldr) {
    int64_t total = n * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % n, j = e / n;
        R[i + j * ldr] = i <= j ? A[i + j * lda] : 0.0;
    }
}

__global__ void gather_cols_k(int64_t rows, int64_t cols, const double* __restrict__ s,
                              int64_t lds, const int* __restrict__ idx, double* __restrict__ d,
                              int64_t ldd) {
    int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % rows, j = e / rows;
        d[i + j * ldd] = s[i + int64_t(idx[j]) * lds];
    }
}

// per-block partial sums of (A-B)^2 in fixed order; final sum on one block
// sum of squares of the off-diagonal (off = 1) or diagonal (off = 0) part
__global__ void part2_partial(int64_t n, const double* __restrict__ A, int64_t lda, int off,
                              double* __restrict__ part) {
    __shared__ double sh[256];
    double acc = 0.0;
    const int64_t total = n * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e % n, j = e / n;
        if ((i != j) == (off != 0)) {
            const double v = A[i + j * lda];
            acc += v * v;
        }
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void diff2_partial(int64_t rows, int64_t cols, const double* __restrict__ A,
                              int64_t lda, const double* __restrict__ B, int64_t ldb,
                              double* __restrict__ part) {
    __shared__ double sh[256];
    double acc = 0.0;
    int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % rows, j = e / rows;
        double dlt = A[i + j * lda] - (B ? B[i + j * ldb] : 0.0);
        acc += dlt * dlt;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void sum_partials(int n, const double* __restrict__ part, double* out) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// x <- x / ||x||_2 (one CTA), the norm stored to *nrm
__global__ void __launch_bounds__(1024) normalize_k(int64_t n, double* __restrict__ x, double* __restrict__ nrm) {
    __shared__ double sh[32];
    __shared__ double tot;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += x[i] * x[i];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) tot = sqrt(v);
    }
    __syncthreads();
    const double t = tot, inv = t > 0.0 ? 1.0 / t : 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] *= inv;
    if (threadIdx.x == 0) *nrm = t;
}

}  // namespace

void normalize(Ctx& c, int64_t n, double* x, double* nrm_dev) {
    normalize_k<<<1, 1024, 0, c.stream>>>(n, x, nrm_dev);
    c.check_launch();
}

void Ctx::d2h(double* dst, const double* src, size_t n) {
    if (pinned_len < n) {
        if (pinned) cudaFreeHost(pinned);
        size_t want = std::max<size_t>(n, 4096);
        HYDOT_CUDA(cudaMallocHost(&pinned, want * sizeof(double)));
        pinned_len = want;
    }
    HYDOT_CUDA(cudaMemcpyAsync(pinned, src, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    sync();
    std::copy(pinned, pinned + n, dst);
}

void copy2d(Ctx& c, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
            int64_t ldd) {
    if (rows <= 0 || cols <= 0) return;
    if (lds == rows && ldd == rows) {
        HYDOT_CUDA(cudaMemcpyAsync(dst, src, size_t(rows * cols) * 8, cudaMemcpyDeviceToDevice,
                                   c.stream));
        return;
    }
    copy2d_k<<<grid_for(c, rows * cols), 256, 0, c.stream>>>(rows, cols, src, lds, dst, ldd);
    c.check_launch();
}

void transpose(Ctx& c, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
               int64_t ldd) {
    StageTimer _t(c, "transpose");
    if (rows <= 0 || cols <= 0) return;
    dim3 grid = dim3(unsigned((rows + 31) / 32), unsigned((cols + 31) / 32));
    if (grid.y > 65535) throw std::invalid_argument("transpose: too many columns");
    transpose_k<<<grid, dim3(32, 8), 0, c.stream>>>(rows, cols, src, lds, dst, ldd);
    c.check_launch();
}

void fill(Ctx& c, int64_t rows, int64_t cols, double v, double* dst, int64_t ldd) {
    if (rows <= 0 || cols <= 0) return;
    fill_k<<<grid_for(c, rows * cols), 256, 0, c.stream>>>(rows, cols, v, dst, ldd, 0);
    c.check_launch();
}

void set_identity(Ctx& c, int64_t rows, int64_t cols, double* dst, int64_t ldd) {
    if (rows <= 0 || cols <= 0) return;
    fill_k<<<grid_for(c, rows * cols), 256, 0, c.stream>>>(rows, cols, 0.0, dst, ldd, 1);
    c.check_launch();
}

void scale_cols(Ctx& c, int64_t rows, int64_t cols, double* A, int64_t lda, const double* s) {
    if (rows <= 0 || cols <= 0) return;
    scale_cols_k<<<grid_for(c, rows * cols), 256, 0, c.stream>>>(rows, cols, A, lda, s);
    c.check_launch();
}

void extract_upper(Ctx& c, int64_t n, const double* A, int64_t lda, double* R, int64_t ldr) {
    if (n <= 0) return;
    upper_k<<<grid_for(c, n * n), 256, 0, c.stream>>>(n, A, lda, R, ldr);
    c.check_launch();
}

void gather_cols(Ctx& c, int64_t rows, int64_t cols, const double* src, int64_t lds,
                 const int* idx, double* dst, int64_t ldd) {
    if (rows <= 0 || cols <= 0) return;
    gather_cols_k<<<grid_for(c, rows * cols), 256, 0, c.stream>>>(rows, cols, src, lds, idx, dst,
                                                                   ldd);
    c.check_launch();
}

double offdiag_ratio(Ctx& c, int64_t n, const double* A, int64_t lda) {
    if (n <= 1) return 0.0;
    const int blocks = std::min(grid_for(c, n * n), 256);
    DBuf part = dalloc(c, 2 * (size_t(blocks) + 1));
    double v[2];
    for (int off = 0; off < 2; ++off) {
        double* pp = part.d() + off * (blocks + 1);
        part2_partial<<<blocks, 256, 0, c.stream>>>(n, A, lda, off, pp);
        c.check_launch();
        sum_partials<<<1, 256, 0, c.stream>>>(blocks, pp, pp + blocks);
        c.check_launch();
    }
    c.d2h(&v[0], part.d() + blocks, 1);
    c.d2h(&v[1], part.d() + (blocks + 1) + blocks, 1);
    const double tot = v[0] + v[1];
    return tot > 0.0 ? std::sqrt(v[1] / tot) : 0.0;
}

double frob_diff(Ctx& c, int64_t rows, int64_t cols, const double* A, int64_t lda,
                 const double* B, int64_t ldb) {
    StageTimer _t(c, "probe_norm");
    if (rows <= 0 || cols <= 0) return 0.0;
    int blocks = std::min(grid_for(c, rows * cols), 256);
    DBuf part = dalloc(c, size_t(blocks) + 1);
    diff2_partial<<<blocks, 256, 0, c.stream>>>(rows, cols, A, lda, B, ldb, part.d());
    c.check_launch();
    sum_partials<<<1, 256, 0, c.stream>>>(blocks, part.d(), part.d() + blocks);
    c.check_launch();
    double v = 0;
    c.d2h(&v, part.d() + blocks, 1);
    return std::sqrt(v);
}

}  // namespace hydot

// ------------------------------------------------------------ profiling --
#include <array>
#include <chrono>
#include <cstdlib>
#include <map>
#include <mutex>

namespace hydot {
namespace {
std::mutex g_prof_mu;
std::map<std::string, std::pair<double, long>>& prof_table() {
    static std::map<std::string, std::pair<double, long>> t;
    return t;
}
bool prof_on() {
    static int on = [] {
        const char* e = std::getenv("HYDOT_PROFILE");
        return (e && (e[0] == '1' || e[0] == '2')) ? (e[0] - '0') : 0;
    }();
    return on != 0;
}
int prof_level() {
    const char* e = std::getenv("HYDOT_PROFILE");
    return (e && e[0] == '2') ? 2 : 1;
}
double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
thread_local int g_depth = 0;
}  // namespace

StageTimer::StageTimer(Ctx& c, const char* name, int64_t a, int64_t b, int64_t k, double flops,
                       double bytes)
    : c_(c), name_(name), a_(a), b_(b), k_(k), flops_(flops), bytes_(bytes) {
    if (c_.timed(name)) {
        ea_ = c_.take_event();
        cudaEventRecord(ea_, c_.stream);
    }
    on_ = prof_on() && g_depth == 0;
    ++g_depth;
    if (on_) {
        c_.sync();
        t0_ = now_s();
    }
}
StageTimer::~StageTimer() {
    --g_depth;
    if (ea_) {
        cudaEvent_t eb = c_.take_event();
        cudaEventRecord(eb, c_.stream);
        c_.trecs.push_back(Ctx::TRec{name_, ea_, eb, flops_, bytes_});
    }
    if (!on_) return;
    cudaStreamSynchronize(c_.stream);
    double dt = now_s() - t0_;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    auto& e = prof_table()[name_];
    e.first += dt;
    e.second += 1;
    if (prof_level() == 2 && dt > 1e-3)
        fprintf(stderr, "[stage] %s %lld %lld %lld ms=%.3f\n", name_, (long long)a_, (long long)b_,
                (long long)k_, dt * 1e3);
}
}  // namespace hydot

// resolve the event records of a context: JSON {name: [ms, calls, flops, bytes]}
std::string timing_report(hydot::Ctx& c) {
    cudaStreamSynchronize(c.stream);
    std::map<std::string, std::array<double, 4>> agg;
    for (auto& r : c.trecs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto& e = agg[r.name];
        e[0] += ms;
        e[1] += 1;
        e[2] += r.flops;
        e[3] += r.bytes;
        c.ev_pool.push_back(r.a);
        c.ev_pool.push_back(r.b);
    }
    c.trecs.clear();
    std::string s = "{";
    bool first = true;
    for (auto& kv : agg) {
        char tmp[320];
        snprintf(tmp, sizeof tmp, "%s\"%s\": [%.6f, %.0f, %.6e, %.6e]", first ? "" : ", ", kv.first.c_str(),
                 kv.second[0], kv.second[1], kv.second[2], kv.second[3]);
        s += tmp;
        first = false;
    }
    return s + "}";
}

extern "C" int hydot_profile_dump(char* buf, int len) {
    std::lock_guard<std::mutex> lk(hydot::g_prof_mu);
    std::string s = "{";
    bool first = true;
    for (auto& kv : hydot::prof_table()) {
        char tmp[256];
        snprintf(tmp, sizeof tmp, "%s\"%s\": [%.6f, %ld]", first ? "" : ", ", kv.first.c_str(),
                 kv.second.first, kv.second.second);
        s += tmp;
        first = false;
    }
    s += "}";
    hydot::prof_table().clear();
    if (buf && len > 0) {
        snprintf(buf, size_t(len), "%s", s.c_str());
    }
    return int(s.size());
}

// ---------------------------------------------------- column utilities --
namespace hydot {
namespace {
__global__ void colnorm2_k(int64_t m, const double* __restrict__ A, int64_t lda,
                           double* __restrict__ out) {
    __shared__ double sh[8];
    const double* a = A + int64_t(blockIdx.x) * lda;
    double s = 0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s += a[i] * a[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
        out[blockIdx.x] = sqrt(t);
    }
}
// dst[idx[i], j] = src[i, j]
__global__ void scatter_rows_k(int64_t rows, int64_t cols, const double* __restrict__ s,
                               int64_t lds, const int* __restrict__ idx, double* __restrict__ d,
                               int64_t ldd) {
    int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % rows, j = e / rows;
        d[int64_t(idx[i]) + j * ldd] = s[i + j * lds];
    }
}
}  // namespace

void col_norms(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* out_dev) {
    if (n <= 0) return;
    colnorm2_k<<<unsigned(n), 256, 0, c.stream>>>(m, A, lda, out_dev);
    c.check_launch();
}

void scatter_rows(Ctx& c, int64_t rows, int64_t cols, const double* src, int64_t lds,
                  const int* idx, double* dst, int64_t ldd) {
    if (rows <= 0 || cols <= 0) return;
    int blocks = int(std::max<int64_t>(1, std::min<int64_t>((rows * cols + 255) / 256, int64_t(c.num_sms) * 16)));
    scatter_rows_k<<<blocks, 256, 0, c.stream>>>(rows, cols, src, lds, idx, dst, ldd);
    c.check_launch();
}
}  // namespace hydot
