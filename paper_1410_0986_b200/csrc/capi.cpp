// capi.cpp -- the C ABI (include/hydot_b200.h) over the device drivers.
// Status mapping keeps the reference's exception classes:
// std::invalid_argument -> HYDOT_EINVAL, std::runtime_error -> HYDOT_ERUNTIME.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "lowrank.h"
#include "pals.h"

using namespace hydot;

std::string timing_report(hydot::Ctx& c);  // util.cu

struct hydot_ctx_s {
    std::shared_ptr<Ctx> c;
};
struct hydot_factor_s {
    std::shared_ptr<Ctx> owner;
    Factor f;
};
struct hydot_tree_s {
    Tree t;
};

namespace {
thread_local std::string g_err;

template <class F>
hydot_status guard(Ctx* c, F&& fn) {
    std::string msg;
    hydot_status st = HYDOT_OK;
    try {
        if (c) HYDOT_CUDA(cudaSetDevice(c->device));
        fn();
    } catch (const CudaError& e) {
        msg = e.what();
        st = HYDOT_ECUDA;
    } catch (const std::bad_alloc&) {
        msg = "out of device memory";
        st = HYDOT_ENOMEM;
    } catch (const std::invalid_argument& e) {
        msg = e.what();
        st = HYDOT_EINVAL;
    } catch (const std::exception& e) {
        msg = e.what();
        st = HYDOT_ERUNTIME;
    }
    if (st != HYDOT_OK) {
        if (c) c->err = msg;
        g_err = msg;
    }
    return st;
}

Ctx& ctx_of(hydot_ctx ctx) {
    if (!ctx || !ctx->c) throw std::invalid_argument("null hydot_ctx");
    return *ctx->c;
}

void ledger_out(const Ledger& l, hydot_ledger* out) {
    if (!out) return;
    out->leaf += l.leaf;
    out->agglomeration += l.agglomeration;
    out->recompress += l.recompress;
    out->other += l.other;
    out->kernel_tally += l.kernel_tally;
}

// the factor with V materialised (a lazy root V is formed on first use)
Factor& dense(Ctx& c, hydot_factor f) {
    materialize_v(c, f->f);
    return f->f;
}

// recursive_lowrank keeps the root's V implicit for recompress
// (HYDOT_LAZY_ROOT=0 materialises it at once)
bool lazy_root_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("HYDOT_LAZY_ROOT");
        return !(e && e[0] == '0');
    }();
    return on;
}

hydot_factor wrap(const std::shared_ptr<Ctx>& owner, Factor&& f) {
    auto* h = new hydot_factor_s;
    h->owner = owner;
    h->f = std::move(f);
    return h;
}
}  // namespace

// shared with comm.cpp: the context behind a handle, and the status of an
// exception (the same mapping as guard)
hydot::Ctx& hydot_ctx_ref(hydot_ctx ctx) { return ctx_of(ctx); }
hydot_status hydot_guard_status(const std::exception& e, hydot::Ctx* c) {
    hydot_status st = HYDOT_ERUNTIME;
    if (dynamic_cast<const CudaError*>(&e)) st = HYDOT_ECUDA;
    else if (dynamic_cast<const std::bad_alloc*>(&e)) st = HYDOT_ENOMEM;
    else if (dynamic_cast<const std::invalid_argument*>(&e)) st = HYDOT_EINVAL;
    const std::string msg = st == HYDOT_ENOMEM ? std::string("out of device memory") : std::string(e.what());
    if (c) c->err = msg;
    g_err = msg;
    return st;
}

extern "C" {

int hydot_version(void) { return 1; }

hydot_status hydot_ctx_create(int device, hydot_ctx* out) {
    if (!out) return HYDOT_EINVAL;
    *out = nullptr;
    return guard(nullptr, [&] {
        auto c = std::make_shared<Ctx>();
        c->device = device;
        HYDOT_CUDA(cudaSetDevice(device));
        HYDOT_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        int sms = 0;
        HYDOT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        c->num_sms = sms;
        // keep freed pool memory cached (the path allocates per node)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            // map a working reserve once per device so the GB-sized per-node
            // buffers of the merges never wait for the pool to grow
            // (HYDOT_POOL_RESERVE_GB, default 48 -- config 1 measured 2.42 s
            // per step with 16 GB (the pool kept growing under fragmentation)
            // and 2.06 s with 48 GB; capped at a third of the free memory;
            // 0 disables)
            static bool reserved[64] = {};
            const char* e = std::getenv("HYDOT_POOL_RESERVE_GB");
            const double gb = e ? std::atof(e) : 48.0;
            if (gb > 0 && device >= 0 && device < 64 && !reserved[device]) {
                reserved[device] = true;
                size_t fr = 0, tot = 0;
                HYDOT_CUDA(cudaMemGetInfo(&fr, &tot));
                const size_t want = std::min(size_t(gb * double(1ull << 30)), fr / 3);
                void* p = nullptr;
                if (want > 0 && cudaMallocAsync(&p, want, c->stream) == cudaSuccess) {
                    HYDOT_CUDA(cudaFreeAsync(p, c->stream));
                    HYDOT_CUDA(cudaStreamSynchronize(c->stream));
                } else {
                    cudaGetLastError();
                }
            }
        }
        auto* h = new hydot_ctx_s;
        h->c = c;
        *out = h;
    });
}

hydot_status hydot_ctx_destroy(hydot_ctx ctx) {
    if (!ctx) return HYDOT_OK;
    hydot_status st = guard(ctx->c.get(), [&] {
        Ctx& c = *ctx->c;
        c.sync();
        if (c.side) {
            cudaStreamSynchronize(c.side);
            cudaStreamDestroy(c.side);
            c.side = nullptr;
        }
        for (auto& h : c.hp)
            if (h) {
                cudaStreamSynchronize(h);
                cudaStreamDestroy(h);
                h = nullptr;
            }
        if (const char* e = std::getenv("HYDOT_POOL_STATS"); e && e[0] == '1') {
            // high-water marks of the pools (reserved = mapped from the device, used = handed out)
            auto report = [](const char* name, cudaMemPool_t p) {
                if (!p) return;
                uint64_t rh = 0, uh = 0, rc = 0;
                cudaMemPoolGetAttribute(p, cudaMemPoolAttrReservedMemHigh, &rh);
                cudaMemPoolGetAttribute(p, cudaMemPoolAttrUsedMemHigh, &uh);
                cudaMemPoolGetAttribute(p, cudaMemPoolAttrReservedMemCurrent, &rc);
                fprintf(stderr, "[pool] %s reserved_high=%.2f GB used_high=%.2f GB reserved_now=%.2f GB\n", name,
                        double(rh) / double(1ull << 30), double(uh) / double(1ull << 30),
                        double(rc) / double(1ull << 30));
            };
            cudaMemPool_t def = nullptr;
            if (cudaDeviceGetDefaultMemPool(&def, c.device) == cudaSuccess) report("default", def);
            report("side", c.side_pool);
            report("hp", c.hp_pool);
        }
        for (cudaMemPool_t* p : {&c.side_pool, &c.hp_pool})
            if (*p) {
                cudaMemPoolDestroy(*p);
                *p = nullptr;
            }
        if (c.coop_ev) cudaEventDestroy(c.coop_ev);
        c.coop_ev = nullptr;
        if (c.pinned) cudaFreeHost(c.pinned);
        c.pinned = nullptr;
        if (c.jump_dev) cudaFree(c.jump_dev);
        c.jump_dev = nullptr;
    });
    delete ctx;
    return st;
}

const char* hydot_last_error(hydot_ctx ctx) {
    if (ctx && ctx->c && !ctx->c->err.empty()) return ctx->c->err.c_str();
    return g_err.c_str();
}

hydot_status hydot_ctx_set_stream(hydot_ctx ctx, void* s) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        c.sync();
        c.stream = static_cast<cudaStream_t>(s);  // NULL = the legacy default stream
    });
}

hydot_status hydot_ctx_synchronize(hydot_ctx ctx) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] { ctx_of(ctx).sync(); });
}

int64_t hydot_ctx_launch_count(hydot_ctx ctx) { return ctx && ctx->c ? ctx->c->launches : -1; }

hydot_status hydot_ctx_set_timing(hydot_ctx ctx, int on) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] { ctx_of(ctx).timing = on != 0; });
}

hydot_status hydot_ctx_set_timing_filter(hydot_ctx ctx, const char* names) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        c.timing_filter.clear();
        if (!names) return;
        std::string s(names), cur;
        for (char ch : s + ",") {
            if (ch == ',') {
                if (!cur.empty()) c.timing_filter.push_back(cur);
                cur.clear();
            } else if (ch != ' ') {
                cur += ch;
            }
        }
    });
}

int hydot_ctx_timing_report(hydot_ctx ctx, char* buf, int len) {
    if (!ctx || !ctx->c) return -1;
    std::string s = timing_report(*ctx->c);
    if (buf && len > 0) snprintf(buf, size_t(len), "%s", s.c_str());
    return int(s.size());
}

// ------------------------------------------------------------- fields ----
hydot_status hydot_fields_solve(hydot_ctx ctx, const hydot_grid7* grid, int n_lambda,
                                const double* sigma_h, const double* sigma_prime_h,
                                const double* inv_D_h, const int64_t* rhs_vertex_h, int n_rhs,
                                double tol, int max_iter, int fixed_iters, double* out_dev,
                                int* iters_h, double* relres_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!grid || !sigma_h || !sigma_prime_h || !inv_D_h || !rhs_vertex_h || !out_dev)
            throw std::invalid_argument("hydot_fields_solve: null argument");
        CGStats st;
        fields_solve(c, *grid, n_lambda, sigma_h, sigma_prime_h, inv_D_h, rhs_vertex_h, n_rhs, tol,
                     max_iter, fixed_iters, out_dev, &st);
        const int total = n_rhs * n_lambda;
        if (iters_h) std::memcpy(iters_h, st.iters.data(), size_t(total) * sizeof(int));
        if (relres_h) std::memcpy(relres_h, st.relres.data(), size_t(total) * sizeof(double));
        if (fixed_iters <= 0)
            for (int k = 0; k < total; ++k)
                if (!(st.relres[size_t(k)] <= tol))
                    throw std::runtime_error("field solve failed at rhs " + std::to_string(k / n_lambda) +
                                             ", wavelength index " + std::to_string(k % n_lambda));
    });
}

hydot_status hydot_full_forward(hydot_ctx ctx, const hydot_grid7* grid, int n_lambda, const double* sigma_h,
                                const double* sigma_prime_h, const double* inv_D_h, const double* dsigma_h,
                                const double* mu_dev, const int64_t* source_vertex_h, int n_sources,
                                const int64_t* detector_vertex_h, int n_det, double tol, int max_iter,
                                int fixed_iters, double* y_total_dev, double* y_incident_dev, int* iters_max_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!grid || !sigma_h || !sigma_prime_h || !inv_D_h || !dsigma_h || !mu_dev || !source_vertex_h ||
            !detector_vertex_h || !y_total_dev || !y_incident_dev)
            throw std::invalid_argument("full_forward: null argument");
        full_forward(c, *grid, n_lambda, sigma_h, sigma_prime_h, inv_D_h, dsigma_h, mu_dev, source_vertex_h,
                     n_sources, detector_vertex_h, n_det, tol, max_iter, fixed_iters, y_total_dev, y_incident_dev,
                     iters_max_h);
    });
}

hydot_status hydot_apply_fem(hydot_ctx ctx, const hydot_grid_geom* geom, double sigma, double sigma_prime,
                             const double* x_dev, double* y_dev) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!geom || !x_dev || !y_dev) throw std::invalid_argument("hydot_apply_fem: null argument");
        apply_fem(c, *geom, sigma, sigma_prime, x_dev, y_dev);
    });
}

hydot_status hydot_fields_solve_fem(hydot_ctx ctx, const hydot_grid_geom* geom, int n_lambda,
                                    const double* sigma_h, const double* sigma_prime_h, const double* inv_D_h,
                                    const double* points_h, int n_points, double tol, int max_iter,
                                    int fixed_iters, double* out_dev, int* iters_h, double* relres_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!geom || !sigma_h || !sigma_prime_h || !inv_D_h || !points_h || !out_dev)
            throw std::invalid_argument("hydot_fields_solve_fem: null argument");
        CGStats st;
        fields_solve_fem(c, *geom, n_lambda, sigma_h, sigma_prime_h, inv_D_h, points_h, n_points, tol, max_iter,
                         fixed_iters, out_dev, &st);
        const int total = n_points * n_lambda;
        for (int k = 0; k < total; ++k) {
            if (iters_h) iters_h[k] = st.iters[size_t(k)];
            if (relres_h) relres_h[k] = st.relres[size_t(k)];
        }
        if (fixed_iters <= 0)
            for (int k = 0; k < total; ++k)
                if (!(st.relres[size_t(k)] <= tol))
                    throw std::runtime_error("field solve failed at point " + std::to_string(k / n_lambda) +
                                             ", wavelength index " + std::to_string(k % n_lambda));
    });
}

void hydot_krylov_config_default(hydot_krylov_config* cfg) {
    if (!cfg) return;
    *cfg = hydot_krylov_config{80, 10, 50, 1e-8, 40, 1, 0, 0};  // krylov.hpp:13-23
}

hydot_status hydot_solve_family_fem(hydot_ctx ctx, const hydot_grid_geom* geom, int n_shifts,
                                    const double* sigma_h, const double* sigma_prime_h, const double* b_dev,
                                    int n_rhs, const hydot_krylov_config* cfg, double* X_dev,
                                    hydot_krylov_stats* stats_h, hydot_krylov_family* fam_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!geom || !sigma_h || !sigma_prime_h || !b_dev || !cfg || !X_dev)
            throw std::invalid_argument("hydot_solve_family_fem: null argument");
        const int64_t N = int64_t(geom->nx) * geom->ny * geom->nz;
        solve_family_fem(c, *geom, n_shifts, sigma_h, sigma_prime_h, b_dev, n_rhs, *cfg, nullptr, X_dev, N, stats_h,
                         fam_h);
    });
}

hydot_status hydot_fields_solve_fem_gmres(hydot_ctx ctx, const hydot_grid_geom* geom, int n_lambda,
                                          const double* sigma_h, const double* sigma_prime_h,
                                          const double* inv_D_h, const double* points_h, int n_points,
                                          const hydot_krylov_config* cfg, double* out_dev,
                                          hydot_krylov_stats* stats_h, hydot_krylov_family* fam_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!geom || !sigma_h || !sigma_prime_h || !inv_D_h || !points_h || !cfg || !out_dev)
            throw std::invalid_argument("hydot_fields_solve_fem_gmres: null argument");
        fields_solve_fem_gmres(c, *geom, n_lambda, sigma_h, sigma_prime_h, inv_D_h, points_h, n_points, *cfg,
                               out_dev, stats_h, fam_h);
    });
}

hydot_status hydot_apply7(hydot_ctx ctx, const hydot_grid7* grid, double sigma,
                          double sigma_prime, const double* x_dev, double* y_dev) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!grid || !x_dev || !y_dev) throw std::invalid_argument("hydot_apply7: null argument");
        apply7(c, *grid, sigma, sigma_prime, x_dev, y_dev);
        c.sync();
    });
}

// --------------------------------------------------------------- born ----
hydot_status hydot_born_block(hydot_ctx ctx, int64_t N, int n_lambda, const double* incident_dev,
                              const double* const* adjoint_dev_h, int n_det, const double* w_dev,
                              double nu, double* out_dev, int64_t ld) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (N < 0 || n_lambda < 0 || n_det < 0) throw std::invalid_argument("assemble_H_block: negative size");
        if (!incident_dev || !adjoint_dev_h || !w_dev || !out_dev)
            throw std::invalid_argument("assemble_H_block: null argument");
        born_block(c, N, n_lambda, incident_dev, adjoint_dev_h, n_det, w_dev, nu, out_dev, ld);
        c.sync();
    });
}

// ---------------------------------------------------------- generator ----
hydot_status hydot_gaussian(hydot_ctx ctx, uint64_t seed, int64_t offset, int64_t count,
                            double* out_dev) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (offset < 0 || count < 0) throw std::invalid_argument("hydot_gaussian: negative range");
        if (count == 0) return;
        RngStream rs(c, seed);
        rs.fill(offset, count, out_dev);
        c.sync();
    });
}

hydot_status hydot_mt19937_64(hydot_ctx ctx, uint64_t seed, int64_t offset, int64_t count,
                              uint64_t* out_dev) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (offset < 0 || count < 0) throw std::invalid_argument("hydot_mt19937_64: negative range");
        RngStream rs(c, seed);
        rs.raw(offset, count, out_dev);
        c.sync();
    });
}

hydot_status hydot_rng_selftest(void) {
    return guard(nullptr, [&] {
        if (!rng_selftest_host()) throw std::runtime_error("MT19937-64 jump-ahead self test failed");
    });
}

// ------------------------------------------------------------- factor ----
hydot_status hydot_factor_create(hydot_ctx ctx, int64_t rows, int64_t cols, int64_t rank,
                                 const double* U, int64_t ldu, const double* V, int64_t ldv,
                                 int from_host, double tol, int method, int flagged,
                                 hydot_factor* out) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!out || rows < 0 || cols < 0 || rank < 0 || rank > std::min(rows, cols) ||
            (rank > 0 && (!U || !V || ldu < rows || ldv < cols)))
            throw std::invalid_argument("hydot_factor_create: bad dimensions");
        Factor f;
        f.rows = rows;
        f.cols = cols;
        f.rank = rank;
        f.tol = tol;
        f.method = method;
        f.flagged = flagged != 0;
        f.U = dalloc(c, size_t(std::max<int64_t>(rows * rank, 1)));
        f.V = dalloc(c, size_t(std::max<int64_t>(cols * rank, 1)));
        auto kind = from_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        if (rank > 0) {
            HYDOT_CUDA(cudaMemcpy2DAsync(f.U.d(), size_t(rows) * 8, U, size_t(ldu) * 8,
                                         size_t(rows) * 8, size_t(rank), kind, c.stream));
            HYDOT_CUDA(cudaMemcpy2DAsync(f.V.d(), size_t(cols) * 8, V, size_t(ldv) * 8,
                                         size_t(cols) * 8, size_t(rank), kind, c.stream));
        }
        c.sync();
        *out = wrap(ctx->c, std::move(f));
    });
}

hydot_status hydot_factor_info(hydot_factor f, int64_t* rows, int64_t* cols, int64_t* rank,
                               double* tol, int* method, int* flagged) {
    if (!f) return HYDOT_EINVAL;
    if (rows) *rows = f->f.rows;
    if (cols) *cols = f->f.cols;
    if (rank) *rank = f->f.rank;
    if (tol) *tol = f->f.tol;
    if (method) *method = f->f.method;
    if (flagged) *flagged = f->f.flagged ? 1 : 0;
    return HYDOT_OK;
}

hydot_status hydot_factor_download(hydot_ctx ctx, hydot_factor f, double* U, double* V,
                                   int to_host) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!f) throw std::invalid_argument("null factor");
        auto kind = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        if (V) dense(c, f);
        if (f->f.rank > 0) {
            if (U)
                HYDOT_CUDA(cudaMemcpyAsync(U, f->f.U.d(), size_t(f->f.rows * f->f.rank) * 8, kind,
                                           c.stream));
            if (V)
                HYDOT_CUDA(cudaMemcpyAsync(V, f->f.V.d(), size_t(f->f.cols * f->f.rank) * 8, kind,
                                           c.stream));
        }
        c.sync();
    });
}

hydot_status hydot_factor_device_ptrs(hydot_factor f, const double** U_dev, const double** V_dev) {
    if (!f) return HYDOT_EINVAL;
    if (V_dev && (f->f.lazy || f->f.pending)) {
        if (!f->owner) return HYDOT_ERUNTIME;
        hydot_status st = guard(f->owner.get(), [&] {
            cudaSetDevice(f->owner->device);
            dense(*f->owner, f);
        });
        if (st != HYDOT_OK) return st;
    }
    if (U_dev) *U_dev = f->f.U.d();
    if (V_dev) *V_dev = f->f.V.d();
    return HYDOT_OK;
}

void hydot_factor_free(hydot_factor f) {
    if (!f) return;
    if (f->owner) cudaSetDevice(f->owner->device);
    delete f;
}

// ------------------------------------------------------------ lowrank ----
hydot_status hydot_randsvd(hydot_ctx ctx, int64_t m, int64_t n, const double* a_dev, int64_t lda,
                           double eps, int p, int kprobe, uint64_t seed, int category, int r0,
                           hydot_factor* out, hydot_ledger* ledger_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!out || m < 0 || n < 0 || (m > 0 && n > 0 && (!a_dev || lda < n)))
            throw std::invalid_argument("randsvd: bad operator");
        Ledger l;
        Factor f = randsvd(c, m, n, a_dev, lda, eps, p, kprobe, seed, &l, category, r0);
        c.sync();
        ledger_out(l, ledger_h);
        *out = wrap(ctx->c, std::move(f));
    });
}

hydot_status hydot_randsvd_linop(hydot_ctx ctx, const hydot_linop* A, double eps, int p, int kprobe,
                                 uint64_t seed, int category, int r0, hydot_factor* out,
                                 hydot_ledger* ledger_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!out || !A || A->rows < 0 || A->cols < 0)
            throw std::invalid_argument("randsvd: bad operator");
        const bool empty = A->rows == 0 || A->cols == 0;
        if (!empty && ((!A->mm && !A->mv) || (!A->rmm && !A->rmv)))
            throw std::invalid_argument("randsvd: operator without products");
        LinOpDev op;
        op.rows = A->rows;
        op.cols = A->cols;
        // apply_mm (lowrank.cpp:95-107): the block form if present, else by columns
        auto product = [&c, A](hydot_mm_fn blk, hydot_mv_fn col, int64_t in_rows, int64_t out_rows) {
            return [&c, A, blk, col, in_rows, out_rows](int64_t k, const double* X, double* Y) {
                int rc = 0;
                if (blk) {
                    rc = blk(A->user, k, X, in_rows, Y, out_rows, c.stream);
                } else {
                    for (int64_t j = 0; j < k && rc == 0; ++j)
                        rc = col(A->user, X + j * in_rows, Y + j * out_rows, c.stream);
                }
                if (rc != 0) throw std::runtime_error("randsvd: operator callback failed");
            };
        };
        op.mm = product(A->mm, A->mv, A->cols, A->rows);
        op.rmm = product(A->rmm, A->rmv, A->rows, A->cols);
        Ledger l;
        Factor f = randsvd(c, op, eps, p, kprobe, seed, &l, category, r0);
        c.sync();
        ledger_out(l, ledger_h);
        *out = wrap(ctx->c, std::move(f));
    });
}

hydot_status hydot_agglomerate(hydot_ctx ctx, hydot_factor f1, hydot_factor f2, double eps,
                               uint64_t seed, int rank_hint, int p, int kprobe, hydot_factor* out,
                               hydot_ledger* ledger_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!f1 || !f2 || !out) throw std::invalid_argument("agglomerate: null factor");
        Ledger l;
        Factor f = agglomerate(c, dense(c, f1), dense(c, f2), eps, seed, &l, rank_hint, p, kprobe);
        c.sync();
        ledger_out(l, ledger_h);
        *out = wrap(ctx->c, std::move(f));
    });
}

hydot_status hydot_tolerance_schedule(double eps_d, int L, int N_r, double* out) {
    return guard(nullptr, [&] {
        if (!out) throw std::invalid_argument("tolerance_schedule: null output");
        *out = tolerance_schedule(eps_d, L, N_r);
    });
}

hydot_status hydot_tree_build(const double* positions_h, int n, int d, const double* lo_h,
                              const double* hi_h, hydot_tree* out) {
    if (out) *out = nullptr;
    return guard(nullptr, [&] {
        if (!positions_h || !lo_h || !hi_h || !out)
            throw std::invalid_argument("build_cluster_tree: null argument");
        auto* t = new hydot_tree_s;
        try {
            t->t = build_cluster_tree(positions_h, n, d, lo_h, hi_h);
        } catch (...) {
            delete t;
            throw;
        }
        *out = t;
    });
}
int hydot_tree_num_nodes(hydot_tree t) { return t ? int(t->t.nodes.size()) : -1; }
int hydot_tree_root(hydot_tree t) { return t ? t->t.root : -1; }
int hydot_tree_depth(hydot_tree t) { return t ? t->t.depth() : -1; }
hydot_status hydot_tree_node(hydot_tree t, int v, int* left, int* right, int* n_idx, int* idx_h) {
    if (!t || v < 0 || v >= int(t->t.nodes.size())) return HYDOT_EINVAL;
    const TreeNode& nd = t->t.nodes[size_t(v)];
    if (left) *left = nd.left;
    if (right) *right = nd.right;
    if (n_idx) *n_idx = int(nd.idx.size());
    if (idx_h) std::memcpy(idx_h, nd.idx.data(), nd.idx.size() * sizeof(int));
    return HYDOT_OK;
}
hydot_status hydot_tree_leaf_order(hydot_tree t, int* order_h) {
    if (!t || !order_h) return HYDOT_EINVAL;
    auto o = t->t.leaf_order();
    std::memcpy(order_h, o.data(), o.size() * sizeof(int));
    return HYDOT_OK;
}
hydot_status hydot_tree_node_box(hydot_tree t, int v, double* lo_h, double* hi_h) {
    if (!t || v < 0 || v >= int(t->t.nodes.size())) return HYDOT_EINVAL;
    const TreeNode& nd = t->t.nodes[size_t(v)];
    if (lo_h) std::memcpy(lo_h, nd.lo.data(), nd.lo.size() * sizeof(double));
    if (hi_h) std::memcpy(hi_h, nd.hi.data(), nd.hi.size() * sizeof(double));
    return HYDOT_OK;
}
void hydot_tree_free(hydot_tree t) { delete t; }

hydot_status hydot_recursive_lowrank(hydot_ctx ctx, hydot_tree tree, double eps,
                                     const hydot_provider* provider, const hydot_born_fields* born,
                                     const hydot_rec_opts* opts, hydot_factor* out,
                                     int* row_perm_h, int* node_rank_h, int* node_depth_h,
                                     hydot_ledger* ledger_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!tree || !out || (!provider == !born))
            throw std::invalid_argument("recursive_lowrank: need a tree and exactly one provider");
        hydot_rec_opts o{0, 20, 10, 0, nullptr, 0};
        if (opts) o = *opts;
        if (o.hint_mode != 0) throw std::invalid_argument("recursive_lowrank: unknown hint_mode");
        std::vector<int> src_ids;
        int nsrc = 0;
        for (const auto& nd : tree->t.nodes)
            for (int s : nd.idx) nsrc = std::max(nsrc, s + 1);
        src_ids.resize(size_t(nsrc));
        for (int s = 0; s < nsrc; ++s) src_ids[size_t(s)] = o.source_ids ? o.source_ids[s] : s;
        int rows_per;
        int64_t cols;
        BlockFn fn;
        if (provider) {
            rows_per = provider->rows_per_source;
            cols = provider->cols;
            if (!provider->block) throw std::invalid_argument("BlockProvider: null block function");
            fn = [&](int s, double* dst, int64_t ld) {
                if (provider->block(provider->user, s, dst, ld) != 0)
                    throw std::runtime_error("BlockProvider failed for source " + std::to_string(s));
            };
        } else {
            rows_per = born->n_det * born->n_lambda;
            cols = born->N;
            fn = [&](int s, double* dst, int64_t ld) {
                if (s < 0 || s >= born->n_sources) throw std::invalid_argument("source out of range");
                if (born->ready_events_h && born->ready_events_h[s])
                    HYDOT_CUDA(cudaStreamWaitEvent(c.stream, static_cast<cudaEvent_t>(born->ready_events_h[s]), 0));
                born_block(c, born->N, born->n_lambda, born->incident_dev_h[s],
                           born->adjoint_dev_h + int64_t(s) * born->n_det, born->n_det, born->w_dev,
                           born->nu, dst, ld);
            };
        }
        RecOut r = recursive_lowrank(c, tree->t, eps, rows_per, cols, fn, o.seed, o.p, o.kprobe,
                                     src_ids, o.node_offset, lazy_root_enabled());
        c.sync();
        if (row_perm_h) std::memcpy(row_perm_h, r.row_perm.data(), r.row_perm.size() * sizeof(int));
        if (node_rank_h) std::memcpy(node_rank_h, r.node_rank.data(), r.node_rank.size() * sizeof(int));
        if (node_depth_h)
            std::memcpy(node_depth_h, r.node_depth.data(), r.node_depth.size() * sizeof(int));
        ledger_out(r.ledger, ledger_h);
        *out = wrap(ctx->c, std::move(r.factor));
    });
}

hydot_status hydot_recompress(hydot_ctx ctx, hydot_factor f, double eps, int rank,
                              hydot_factor* out, hydot_ledger* ledger_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!f || !out) throw std::invalid_argument("recompress: null factor");
        Ledger l;
        Factor g = recompress(c, f->f, eps, rank, &l);
        c.sync();
        ledger_out(l, ledger_h);
        *out = wrap(ctx->c, std::move(g));
    });
}

hydot_status hydot_lr_matmat(hydot_ctx ctx, hydot_factor f, int trans, int b, const double* X_dev,
                             int64_t ldx, double* Y_dev, int64_t ldy) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!f) throw std::invalid_argument("lr_matvec: null factor");
        const Factor& F = dense(c, f);
        const int64_t in_rows = trans ? F.rows : F.cols, out_rows = trans ? F.cols : F.rows;
        if (b < 0 || ldx < in_rows || ldy < out_rows)
            throw std::invalid_argument(trans ? "lr_rmatvec: dimension mismatch"
                                              : "lr_matvec: dimension mismatch");
        if (b == 0) return;
        if (F.rank == 0) {
            fill(c, out_rows, b, 0.0, Y_dev, ldy);
            c.sync();
            return;
        }
        DBuf Z = dalloc(c, size_t(F.rank) * size_t(b));
        const double* A1 = trans ? F.U.d() : F.V.d();  // contract against X
        const double* A2 = trans ? F.V.d() : F.U.d();
        if (skinny_ok(b)) {
            skinny_tn(c, in_rows, F.rank, b, A1, in_rows, X_dev, ldx, Z.d(), F.rank);
            skinny_nn(c, out_rows, F.rank, b, A2, out_rows, Z.d(), F.rank, Y_dev, ldy);
        } else {
            dgemm(c, true, false, F.rank, b, in_rows, 1.0, A1, in_rows, X_dev, ldx, 0.0, Z.d(), F.rank);
            dgemm(c, false, false, out_rows, b, F.rank, 1.0, A2, out_rows, Z.d(), F.rank, 0.0, Y_dev, ldy);
        }
        c.sync();
    });
}

hydot_status hydot_j_matmat(hydot_ctx ctx, hydot_factor f, int trans, int b, const int* row_perm_dev,
                            const double* eps_c_dev, int n_lambda, int n_c, const double* X_dev,
                            int64_t ldx, double* Y_dev, int64_t ldy) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!f || !row_perm_dev || !eps_c_dev || n_lambda < 1 || n_c < 1 || b < 0)
            throw std::invalid_argument("J matmat: bad arguments");
        const Factor& F = dense(c, f);
        j_matmat(c, F.U.d(), F.V.d(), F.rows, F.cols, F.rank, trans != 0, b, row_perm_dev, eps_c_dev, n_lambda, n_c,
                 X_dev, ldx, Y_dev, ldy);
        c.sync();
    });
}

hydot_status hydot_thin_svd(hydot_ctx ctx, int64_t m, int64_t n, const double* a_dev, int64_t lda,
                            double* U_dev, double* s_h, double* V_dev) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (m < 0 || n < 0 || lda < m) throw std::invalid_argument("thin_svd: bad dimensions");
        // full orthonormal U, V like Eigen::BDCSVD; HYDOT_THIN_SVD_PATH=1
        // runs the path's own (lazy-V) variant instead, for profiling
        const bool path_mode = [] {
            const char* e = std::getenv("HYDOT_THIN_SVD_PATH");
            return e && e[0] == '1';
        }();
        std::unique_ptr<StrictSVD> strict;
        if (!path_mode) strict.reset(new StrictSVD());
        SVDd s = fast_thin_svd(c, a_dev, lda, false, m, n, nullptr, HYDOT_CAT_OTHER);
        const int64_t k = s.k;
        if (k > 0) {
            HYDOT_CUDA(cudaMemcpyAsync(U_dev, s.U.d(), size_t(m * k) * 8, cudaMemcpyDeviceToDevice, c.stream));
            HYDOT_CUDA(cudaMemcpyAsync(V_dev, s.V.d(), size_t(n * k) * 8, cudaMemcpyDeviceToDevice, c.stream));
            std::memcpy(s_h, s.s.data(), size_t(k) * 8);
        }
        c.sync();
    });
}

hydot_status hydot_householder_qr(hydot_ctx ctx, int64_t m, int64_t n, const double* a_dev,
                                  int64_t lda, double* R_dev, double* Q_dev) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (m < n || n < 0 || lda < m) throw std::invalid_argument("householder_qr: needs m >= n");
        QRFact qf;
        geqrf(c, m, n, a_dev, lda, qf);
        if (R_dev) extract_upper(c, n, qf.a.d(), m, R_dev, n);
        if (Q_dev) {
            fill(c, m, n, 0.0, Q_dev, m);
            set_identity(c, n, n, Q_dev, m);
            apply_q(c, qf, false, n, Q_dev, m);
        }
        c.sync();
    });
}

hydot_status hydot_dgemm(hydot_ctx ctx, int transa, int transb, int64_t m, int64_t n, int64_t k,
                         double alpha, const double* A_dev, int64_t lda, const double* B_dev,
                         int64_t ldb, double beta, double* C_dev, int64_t ldc) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (m < 0 || n < 0 || k < 0 || ldc < m) throw std::invalid_argument("dgemm: bad dimensions");
        dgemm(c, transa != 0, transb != 0, m, n, k, alpha, A_dev, lda, B_dev, ldb, beta, C_dev, ldc);
        c.sync();
    });
}

// ------------------------------------------------------------------ pals --
namespace {
hydot::pals::Hop hop_of(Ctx& c, const hydot_hop* op) {
    if (!op || !op->H) throw std::invalid_argument("PaLS: null operator");
    hydot::pals::Hop h;
    h.f = &dense(c, op->H);
    h.perm = op->row_perm_dev;
    return h;
}
hydot::pals::Geom geom_of(const hydot_grid_geom* g) {
    if (!g) throw std::invalid_argument("PaLS: null grid");
    return hydot::pals::Geom::make(*g);
}
hydot::pals::Params params_of(const hydot_pals_params* p) {
    if (!p) throw std::invalid_argument("PaLS: null parameters");
    return hydot::pals::Params::from(*p);
}
}  // namespace

hydot_status hydot_pals_eval(hydot_ctx ctx, int which, const hydot_grid_geom* geom,
                             const hydot_pals_params* p, double* out_dev, int64_t ldo) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        hydot::pals::Geom g = geom_of(geom);
        if (which < 0 || which > 2 || !out_dev || ldo < g.N()) throw std::invalid_argument("pals_eval: bad arguments");
        hydot::pals::eval(c, which, g, params_of(p), out_dev, ldo);
        c.sync();
    });
}

hydot_status hydot_pals_hmv(hydot_ctx ctx, const hydot_hop* op, int b, const double* X_dev, int64_t ldx,
                            double* Y_dev, int64_t ldy) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (b < 0) throw std::invalid_argument("Hmv: negative column count");
        hydot::pals::hmv(c, hop_of(c, op), b, X_dev, ldx, Y_dev, ldy);
        c.sync();
    });
}

hydot_status hydot_pals_solve_concentrations(hydot_ctx ctx, const hydot_hop* op, const double* mu_dev,
                                             const double* w_dev, const double* y_dev, const double* ext_h,
                                             int n_lambda, int n_species, double* c_h, int* flagged_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!mu_dev || !w_dev || !y_dev || !ext_h || !c_h) throw std::invalid_argument("solve_concentrations: null argument");
        hydot::pals::Conc r =
            hydot::pals::solve_concentrations(c, hop_of(c, op), mu_dev, w_dev, y_dev, ext_h, n_lambda, n_species);
        std::copy(r.c.begin(), r.c.end(), c_h);
        if (flagged_h) *flagged_h = r.flagged ? 1 : 0;
    });
}

hydot_status hydot_pals_lm_step(hydot_ctx ctx, int64_t M, int n, const double* J_dev, int64_t ldj,
                                const double* eps_dev, double nu, double* dp_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (M < 0 || n < 0 || !dp_h) throw std::invalid_argument("lm_step: bad arguments");
        std::vector<double> dp = hydot::pals::lm_step(c, M, n, J_dev, ldj, eps_dev, nu);
        std::copy(dp.begin(), dp.end(), dp_h);
    });
}

hydot_status hydot_pals_metrics(hydot_ctx ctx, int64_t n, const double* mu_true_dev, const double* mu_hat_dev,
                                double threshold, double* l2_rel_h, double* dice_h, int* flagged_h) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (n < 0) throw std::invalid_argument("metrics: length mismatch");
        hydot::pals::Metrics m = hydot::pals::metrics(c, n, mu_true_dev, mu_hat_dev, threshold);
        if (l2_rel_h) *l2_rel_h = m.l2_rel;
        if (dice_h) *dice_h = m.dice;
        if (flagged_h) *flagged_h = m.flagged ? 1 : 0;
    });
}

hydot_status hydot_pals_reconstruct(hydot_ctx ctx, const hydot_hop* op, const hydot_grid_geom* geom,
                                    const double* ext_h, int n_lambda, int n_species, const double* y_dev,
                                    const double* w_dev, const hydot_pals_params* init, double noise_norm,
                                    const hydot_recon_config* cfg, const double* mu_truth_dev,
                                    hydot_recon_result* out) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!ext_h || !y_dev || !w_dev || !cfg || !out || n_lambda < 1 || n_species < 0)
            throw std::invalid_argument("reconstruct: bad arguments");
        hydot::pals::Params p0 = params_of(init);
        if (out->p.np != p0.np() || (p0.np() > 0 && (!out->p.alpha || !out->p.beta || !out->p.centers)) ||
            (n_species > 0 && !out->c_h) || (out->trace_cap > 0 && !out->trace_h))
            throw std::invalid_argument("reconstruct: result arrays");
        hydot::pals::ReconCfg rc;
        rc.max_outer = cfg->max_outer;
        rc.max_inner = cfg->max_inner;
        rc.max_retries = cfg->max_retries;
        rc.gamma = cfg->gamma;
        rc.nu0 = cfg->nu0;
        rc.stagnation_tol = cfg->stagnation_tol;
        if (cfg->fixed_c_h) rc.fixed_c.assign(cfg->fixed_c_h, cfg->fixed_c_h + n_species);
        if (cfg->normal_blocks < 0) throw std::invalid_argument("reconstruct: normal_blocks < 0");
        rc.normal_blocks = cfg->normal_blocks;
        hydot::pals::Recon r = hydot::pals::reconstruct(c, hop_of(c, op), geom_of(geom), ext_h, n_lambda, n_species,
                                                        y_dev, w_dev, p0, noise_norm, rc, mu_truth_dev);
        std::copy(r.p.alpha.begin(), r.p.alpha.end(), out->p.alpha);
        std::copy(r.p.beta.begin(), r.p.beta.end(), out->p.beta);
        std::copy(r.p.centers.begin(), r.p.centers.end(), out->p.centers);
        out->p.tau_level = r.p.tau_level;
        out->p.eps_H = r.p.eps_H;
        out->p.nu_norm = r.p.nu_norm;
        std::copy(r.c.begin(), r.c.end(), out->c_h);
        out->trace_len = int(r.trace.size());
        for (int i = 0; i < std::min(out->trace_len, out->trace_cap); ++i) {
            const auto& t = r.trace[size_t(i)];
            out->trace_h[i] = hydot_trace_row{t.outer, t.inner, t.resnorm, t.nu, t.accepted ? 1 : 0, t.dice};
        }
        out->resnorm = r.resnorm;
        out->converged = r.converged ? 1 : 0;
        out->flagged = r.flagged ? 1 : 0;
        out->hmv_calls = r.hmv_calls;
        out->hmv_columns = r.hmv_columns;
        out->normal_columns = r.normal_columns;
    });
}

// --------------------------------------------------------------- file I/O --
hydot_status hydot_factor_save(hydot_ctx ctx, hydot_factor f, const int* row_perm_h, int64_t plen,
                               const char* path) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!f || !path || plen < 0 || (plen > 0 && !row_perm_h))
            throw std::invalid_argument("save_factor: bad arguments");
        save_factor_file(c, path, dense(c, f), row_perm_h, plen);
    });
}

hydot_status hydot_factor_file_info(const char* path, int64_t* rows, int64_t* cols, int64_t* rank,
                                    int64_t* plen) {
    return guard(nullptr, [&] {
        if (!path) throw std::invalid_argument("load_factor: null path");
        int64_t m, n, r, p;
        factor_file_info(path, m, n, r, p);
        if (rows) *rows = m;
        if (cols) *cols = n;
        if (rank) *rank = r;
        if (plen) *plen = p;
    });
}

hydot_status hydot_factor_load(hydot_ctx ctx, const char* path, hydot_factor* out, int* row_perm_h,
                               int64_t perm_cap) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!out || !path) throw std::invalid_argument("load_factor: bad arguments");
        std::vector<int> perm;
        Factor f = load_factor_file(c, path, perm);
        if (row_perm_h) {
            if (perm_cap < int64_t(perm.size())) throw std::invalid_argument("load_factor: row_perm buffer too small");
            std::copy(perm.begin(), perm.end(), row_perm_h);
        }
        c.sync();
        *out = wrap(ctx->c, std::move(f));
    });
}

hydot_status hydot_block_save(hydot_ctx ctx, const double* block_dev, int64_t rows, int64_t cols,
                              int64_t ld, const char* path) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!path || rows < 0 || cols < 0 || (rows > 0 && (!block_dev || ld < cols)))
            throw std::invalid_argument("save_block: bad arguments");
        save_block_file(c, path, block_dev, rows, cols, ld);
    });
}

hydot_status hydot_block_file_info(const char* path, int64_t* rows, int64_t* cols) {
    return guard(nullptr, [&] {
        if (!path) throw std::invalid_argument("load_block: null path");
        int64_t r, k;
        block_file_info(path, r, k);
        if (rows) *rows = r;
        if (cols) *cols = k;
    });
}

hydot_status hydot_block_load(hydot_ctx ctx, const char* path, double* block_dev, int64_t ld, int64_t rows_cap,
                              int64_t* rows, int64_t* cols) {
    return guard(ctx ? ctx->c.get() : nullptr, [&] {
        Ctx& c = ctx_of(ctx);
        if (!path || !block_dev) throw std::invalid_argument("load_block: bad arguments");
        int64_t r = 0, k = 0;
        if (rows_cap < 0) throw std::invalid_argument("load_block: bad arguments");
        load_block_file(c, path, block_dev, ld, rows_cap, r, k);
        if (rows) *rows = r;
        if (cols) *cols = k;
    });
}

}  // extern "C"
