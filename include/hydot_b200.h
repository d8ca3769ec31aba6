/* hydot_b200.h -- C ABI of the B200-native hydot hot path.
 *
 * Drop-in boundary for the reference's Born -> low-rank -> matvec path
 * (/root/reference/proj, arXiv 1410.0986).  Every entry point names the
 * reference interface it replaces (file:line, relative to /root/reference).
 * Plain pointers and sizes only: no Eigen, no torch types.
 *
 * Conventions
 *  - Matrices are column-major doubles with an explicit leading dimension,
 *    like Eigen::MatrixXd (proj/include/hydot/grid.hpp:12-14), unless a
 *    parameter says "row-major".
 *  - "_dev" pointers are device (cudaMalloc) memory on the context's GPU;
 *    "_h" pointers are host memory.  No borrowed pointer is retained after a
 *    call returns.
 *  - Every call is stream-ordered on the context's stream and synchronous
 *    from the caller's view for its host outputs.  Internally the context
 *    also uses one side stream (a node's V formed while the next node
 *    decides); it is joined to the context's stream by events before any
 *    result is handed out, so callers only ever see the context's stream.
 *  - Errors: a status code; hydot_last_error(ctx) returns the message.
 *    HYDOT_EINVAL  <-> std::invalid_argument in the reference,
 *    HYDOT_ERUNTIME<-> std::runtime_error (messages keep the reference
 *    prefixes, e.g. "recursive_lowrank at node v: ", lowrank.cpp:503-506).
 */
#ifndef HYDOT_B200_H
#define HYDOT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HYDOT_OK = 0,
    HYDOT_EINVAL = 1,   /* std::invalid_argument */
    HYDOT_ERUNTIME = 2, /* std::runtime_error */
    HYDOT_ENOMEM = 3,
    HYDOT_ECUDA = 4,
    HYDOT_ENCCL = 5
} hydot_status;

typedef struct hydot_ctx_s* hydot_ctx;
typedef struct hydot_factor_s* hydot_factor;
typedef struct hydot_tree_s* hydot_tree;

/* lowrank::Method (proj/include/hydot/lowrank.hpp:14-22) */
enum {
    HYDOT_METHOD_NONE = 0,
    HYDOT_METHOD_RANDSVD = 1,
    HYDOT_METHOD_ACA_FULL = 2,
    HYDOT_METHOD_ACA_PARTIAL = 3,
    HYDOT_METHOD_AGGLOMERATE = 4,
    HYDOT_METHOD_RECURSIVE = 5,
    HYDOT_METHOD_RECOMPRESS = 6
};

/* lowrank::FlopCategory (lowrank.hpp:54) */
enum { HYDOT_CAT_LEAF = 0, HYDOT_CAT_AGGLOMERATION = 1, HYDOT_CAT_RECOMPRESS = 2, HYDOT_CAT_OTHER = 3 };

/* lowrank::FlopLedger (lowrank.hpp:38-52) */
typedef struct {
    double leaf, agglomeration, recompress, other, kernel_tally;
} hydot_ledger;

/* ------------------------------------------------------------ context -- */
int hydot_version(void);
hydot_status hydot_ctx_create(int device, hydot_ctx* out);
hydot_status hydot_ctx_destroy(hydot_ctx ctx);
const char* hydot_last_error(hydot_ctx ctx);
/* run on a caller-owned cudaStream_t (NULL = the legacy default stream, e.g.
 * torch's default stream); the context starts on its own stream. */
hydot_status hydot_ctx_set_stream(hydot_ctx ctx, void* cuda_stream);
hydot_status hydot_ctx_synchronize(hydot_ctx ctx);
/* number of kernels this context launched so far (evidence counter) */
int64_t hydot_ctx_launch_count(hydot_ctx ctx);
/* per-stage wall times recorded when HYDOT_PROFILE=1 (JSON written into buf,
 * then cleared); returns the JSON length */
int hydot_profile_dump(char* buf, int len);
/* live per-stage timing with CUDA events on the context stream (no extra
 * synchronisation while on); the report resolves and clears the records:
 * JSON {stage: [ms, calls, algorithmic flops, algorithmic bytes]} */
hydot_status hydot_ctx_set_timing(hydot_ctx ctx, int on);
/* restrict the live timing to the stages named in a comma-separated list
 * (NULL or "" = all stages): lets a benchmark time one kernel class inside
 * its timed region without paying an event pair per stage everywhere. */
hydot_status hydot_ctx_set_timing_filter(hydot_ctx ctx, const char* names);
int hydot_ctx_timing_report(hydot_ctx ctx, char* buf, int len);

/* ------------------------------------------------------------- fields -- */
/* 7-point vertex-centred FV operator on an nx*ny*nz vertex grid (spacing h,
 * x-fastest n = ix + nx*(iy + ny*iz), grid.hpp:22-28); side faces Dirichlet,
 * z faces Robin (grid.hpp:18-21).  Replaces the FEM K/M/R of
 * grid.cpp:112-174 per BASELINE.json. */
typedef struct {
    int nx, ny, nz;
    double h;
} hydot_grid7;

/* Fields for unit-vertex sources: replaces born::compute_fields
 * (born.hpp:54-56, born.cpp:39-80; solver krylov::solve_family,
 * krylov.cpp:400-463) by batched matrix-free CG on the SPD systems
 * (K + sigma_l M + sigma'_l R) x = e_v, then x *= inv_D[l] (born.cpp:62-63).
 * out_dev: N x (n_rhs*n_lambda), column k*n_lambda + l, ld = N.
 * fixed_iters > 0 runs exactly that many iterations (parity mode).
 * iters_h / relres_h (optional): per system. */
hydot_status hydot_fields_solve(hydot_ctx ctx, const hydot_grid7* grid, int n_lambda,
                                const double* sigma_h, const double* sigma_prime_h,
                                const double* inv_D_h, const int64_t* rhs_vertex_h, int n_rhs,
                                double tol, int max_iter, int fixed_iters, double* out_dev,
                                int* iters_h, double* relres_h);

/* experiments::full_diffusion_forward (experiments.cpp:154-206; the
 * nonlinear forward model) for the 7-point operator: per wavelength l and
 * source s, x_tot solves (K + (sigma_l + dsigma_l mu(v)) M + sigma'_l R) x =
 * e_{source_vertex[s]} and x_inc the same with mu = 0;
 * y_total[(s*n_det + d)*n_lambda + l] = inv_D_l x_tot(detector_vertex[s*n_det + d]),
 * y_incident likewise (y_scattered = y_total - y_incident).  dsigma_l =
 * (sum_c c_pert_c eps_c(lambda_l)) nu / D_l; mu_dev: N vertex values
 * (pals::shape).  Both solves use the same batched CG, so mu = 0 gives
 * y_total == y_incident bitwise.  Outputs are device arrays. */
hydot_status hydot_full_forward(hydot_ctx ctx, const hydot_grid7* grid, int n_lambda, const double* sigma_h,
                                const double* sigma_prime_h, const double* inv_D_h, const double* dsigma_h,
                                const double* mu_dev, const int64_t* source_vertex_h, int n_sources,
                                const int64_t* detector_vertex_h, int n_det, double tol, int max_iter,
                                int fixed_iters, double* y_total_dev, double* y_incident_dev, int* iters_max_h);

/* y = A_l x for one shift (the operator the CG applies; for tests). */
hydot_status hydot_apply7(hydot_ctx ctx, const hydot_grid7* grid, double sigma,
                          double sigma_prime, const double* x_dev, double* y_dev);

/* grid::build_grid (grid.cpp:94-110): vertices on [-Lx,Lx]x[-Ly,Ly]x[0,Lz],
 * x-fastest, h = 2L/(n-1) laterally and Lz/(nz-1) vertically. */
typedef struct hydot_grid_geom {
    int nx, ny, nz;
    double Lx, Ly, Lz;
} hydot_grid_geom;

/* The reference's own operator, for reference fixtures: trilinear-FEM
 * stiffness K with the Dirichlet side vertices eliminated (unit diagonal),
 * row-lumped mass M and the bilinear face mass R on z = 0 and z = Lz
 * (grid.cpp:112-174; element matrices by its 2x2x2 Gauss rule), applied
 * matrix-free: y = (K + sigma M + sigma' R) x. */
hydot_status hydot_apply_fem(hydot_ctx ctx, const hydot_grid_geom* geom, double sigma,
                             double sigma_prime, const double* x_dev, double* y_dev);
/* compute_fields (born.cpp:39-80) with that operator and the reference's
 * point sources: points_h (n_points x 3, x y z) give the trilinear
 * point_source_vector (grid.cpp:212-237) with Dirichlet entries zeroed
 * (born.cpp:27-35); same batched CG, output layout as hydot_fields_solve. */
hydot_status hydot_fields_solve_fem(hydot_ctx ctx, const hydot_grid_geom* geom, int n_lambda,
                                    const double* sigma_h, const double* sigma_prime_h,
                                    const double* inv_D_h, const double* points_h, int n_points,
                                    double tol, int max_iter, int fixed_iters, double* out_dev,
                                    int* iters_h, double* relres_h);

/* ------------------------------------------------------------ krylov -- */
/* The reference's recycled shifted-family solver (krylov.hpp, krylov.cpp:
 * 21-463) on the FEM operator above.  hydot_krylov_config is
 * krylov::SolverConfig (krylov.hpp:13-23) without `threads` (the device
 * solves every shift of every right-hand side of a batch together);
 * hydot_krylov_config_default gives the reference defaults (80, 10, 50,
 * 1e-8, 40, center, no Jacobi, Gram/Cholesky update). */
typedef struct hydot_krylov_config {
    int arnoldi_steps;      /* phase-1 basis size n (<= 200) */
    int deflation_dim;      /* k harmonic Ritz vectors (<= 32) */
    int restart;            /* m, augmented GMRES cycle length (<= 200) */
    double tol;             /* relative residual target */
    int max_restarts;
    int center_shifts;      /* sbar' = mean sigma' folded into Ks */
    int jacobi;             /* fixed diagonal right preconditioner */
    int explicit_qr_update; /* bypass the Gram/Cholesky basis update */
} hydot_krylov_config;
void hydot_krylov_config_default(hydot_krylov_config* cfg);

/* krylov::IterationStats (krylov.hpp:109-114) per (rhs, shift), plus the
 * phase-1 least-squares residual of that shift (MultishiftResult::relres). */
typedef struct hydot_krylov_stats {
    int iterations; /* inner Arnoldi steps of phase 2 */
    int matvecs;
    double relres;
    int converged;
    double phase1_relres;
} hydot_krylov_stats;

/* Per right-hand side: FamilyResult (krylov.hpp:128-134) summary and the
 * phase-1 / deflation facts (ArnoldiData::steps, breakdown, HarmonicRitz::
 * pencil_shifted, DeflationBasis::k / rank_reduced, ShiftedDeflation::
 * cholesky_failed count). */
typedef struct hydot_krylov_family {
    int phase1_steps;
    int deflation_k;
    int rank_reduced;
    int pencil_shifted;
    int breakdown;
    int cholesky_failed;
    int all_converged;
    int first_failure; /* shift index, -1 if none */
} hydot_krylov_family;

/* krylov::solve_family (krylov.hpp:137-141, krylov.cpp:400-463) for n_rhs
 * right-hand sides b_dev (n_rhs x N, device) and the shifts (sigma_j,
 * sigma'_j): X_dev[(r*n_shifts + j)*N + v] = x_{r,j} in the original
 * variables.  stats_h: n_rhs*n_shifts entries, fam_h: n_rhs (both nullable).
 * Like the reference, unconverged systems are reported, not raised;
 * b = 0 is HYDOT_EINVAL ("multishift_gmres: b must be nonzero"). */
hydot_status hydot_solve_family_fem(hydot_ctx ctx, const hydot_grid_geom* geom, int n_shifts,
                                    const double* sigma_h, const double* sigma_prime_h, const double* b_dev,
                                    int n_rhs, const hydot_krylov_config* cfg, double* X_dev,
                                    hydot_krylov_stats* stats_h, hydot_krylov_family* fam_h);
/* born::compute_fields (born.cpp:39-80) with that solver: the point sources
 * of hydot_fields_solve_fem, X scaled by inv_D per wavelength, same output
 * layout; an unconverged system raises HYDOT_ERUNTIME ("field solve failed
 * at point p, wavelength index l", born.cpp:58-61). */
hydot_status hydot_fields_solve_fem_gmres(hydot_ctx ctx, const hydot_grid_geom* geom, int n_lambda,
                                          const double* sigma_h, const double* sigma_prime_h,
                                          const double* inv_D_h, const double* points_h, int n_points,
                                          const hydot_krylov_config* cfg, double* out_dev,
                                          hydot_krylov_stats* stats_h, hydot_krylov_family* fam_h);

/* --------------------------------------------------------------- born -- */
/* born::assemble_H_block (born.hpp:61-62, born.cpp:82-98):
 *   out[(d*n_lambda + l)*ld + v] = (-nu) * ((phi_d[v,l] * phi_s[v,l]) * w[v])
 * i.e. the (n_det*n_lambda) x N block stored ROW-major (rows contiguous over
 * voxels; the save_block file order, born.cpp:156-167).
 * incident_dev: N x n_lambda (ld N); adjoint_dev_h: host array of n_det
 * device pointers, each N x n_lambda. */
hydot_status hydot_born_block(hydot_ctx ctx, int64_t N, int n_lambda, const double* incident_dev,
                              const double* const* adjoint_dev_h, int n_det, const double* w_dev,
                              double nu, double* out_dev, int64_t ld);

/* --------------------------------------------------------- generator -- */
/* The Gaussian stream of randsvd (lowrank.cpp:136-143): deviates
 * [offset, offset+count) of std::normal_distribution<double> (libstdc++
 * polar method) driven by std::mt19937_64(seed), generated on the GPU with
 * MT19937-64 jump-ahead. */
hydot_status hydot_gaussian(hydot_ctx ctx, uint64_t seed, int64_t offset, int64_t count,
                            double* out_dev);
/* raw tempered engine outputs [offset, offset+count) */
hydot_status hydot_mt19937_64(hydot_ctx ctx, uint64_t seed, int64_t offset, int64_t count,
                              uint64_t* out_dev);
/* host-only self check of the jump-ahead tables against a sequential
 * engine (no GPU needed); returns HYDOT_OK when they agree. */
hydot_status hydot_rng_selftest(void);

/* ------------------------------------------------------------- factor -- */
/* lowrank::LowRankFactor (lowrank.hpp:25-36), device resident: U rows x r,
 * V cols x r (column-major), singular values folded into V. */
hydot_status hydot_factor_create(hydot_ctx ctx, int64_t rows, int64_t cols, int64_t rank,
                                 const double* U, int64_t ldu, const double* V, int64_t ldv,
                                 int from_host, double tol, int method, int flagged,
                                 hydot_factor* out);
hydot_status hydot_factor_info(hydot_factor f, int64_t* rows, int64_t* cols, int64_t* rank,
                               double* tol, int* method, int* flagged);
/* copy U (rows x r) and V (cols x r) out; to_host selects host/device dst */
hydot_status hydot_factor_download(hydot_ctx ctx, hydot_factor f, double* U, double* V,
                                   int to_host);
/* device pointers of U and V.  A factor returned by
 * hydot_recursive_lowrank holds its V implicitly (Householder Q of the root
 * merge times a small matrix) until first use: asking for V here (or
 * downloading it, or any product / save / agglomerate) forms it on the
 * owning context's stream; hydot_recompress consumes the implicit form
 * directly.  HYDOT_LAZY_ROOT=0 forms it at once. */
hydot_status hydot_factor_device_ptrs(hydot_factor f, const double** U_dev, const double** V_dev);
void hydot_factor_free(hydot_factor f);

/* ------------------------------------------------------------ lowrank -- */
/* lowrank::randsvd (lowrank.hpp:70-72, lowrank.cpp:131-199) on a dense
 * device operator A (dense_op, lowrank.cpp:111-120) of m x n stored
 * ROW-major (a_dev[i*lda + j]; lda >= n).  category: HYDOT_CAT_*. */
hydot_status hydot_randsvd(hydot_ctx ctx, int64_t m, int64_t n, const double* a_dev, int64_t lda,
                           double eps, int p, int kprobe, uint64_t seed, int category, int r0,
                           hydot_factor* out, hydot_ledger* ledger_h);

/* lowrank::LinOp (lowrank.hpp:56-63): a matrix-free operator given by
 * callbacks on DEVICE operands (column-major, unit column stride).  mv / rmv
 * are A x and A^T y; mm / rmm are the optional block forms A X (X cols x k,
 * ldx; Y rows x k, ldy) and A^T Y -- when NULL the columns go through mv /
 * rmv one by one, as apply_mm does (lowrank.cpp:95-107).  A callback must
 * enqueue its work on `stream` (a cudaStream_t: its inputs are ready there
 * and its output is consumed there) and return 0; any other value aborts
 * the call with HYDOT_ERUNTIME. */
typedef int (*hydot_mv_fn)(void* user, const double* x_dev, double* y_dev, void* stream);
typedef int (*hydot_mm_fn)(void* user, int64_t k, const double* X_dev, int64_t ldx, double* Y_dev,
                           int64_t ldy, void* stream);
typedef struct {
    int64_t rows, cols;
    hydot_mv_fn mv, rmv;
    hydot_mm_fn mm, rmm;
    void* user;
} hydot_linop;

/* lowrank::randsvd (lowrank.hpp:70-72, lowrank.cpp:131-199) on a LinOp: the
 * same sketch passes, Gaussian stream, accept / double / Q = I decisions and
 * ledger as hydot_randsvd; the Q = I branch takes A^T as rmm(I_rows) like
 * the reference (lowrank.cpp:159-164, 184).  With the dense products as
 * callbacks it returns hydot_randsvd's factor. */
hydot_status hydot_randsvd_linop(hydot_ctx ctx, const hydot_linop* A, double eps, int p, int kprobe,
                                 uint64_t seed, int category, int r0, hydot_factor* out,
                                 hydot_ledger* ledger_h);

/* lowrank::agglomerate (lowrank.hpp:98-100, lowrank.cpp:321-359); the
 * reference hard-codes p=20, kprobe=10 (lowrank.cpp:344). */
hydot_status hydot_agglomerate(hydot_ctx ctx, hydot_factor f1, hydot_factor f2, double eps,
                               uint64_t seed, int rank_hint, int p, int kprobe,
                               hydot_factor* out, hydot_ledger* ledger_h);

/* lowrank::tolerance_schedule (lowrank.cpp:540-545) */
hydot_status hydot_tolerance_schedule(double eps_d, int L, int N_r, double* out);

/* lowrank::build_cluster_tree / ClusterTree (lowrank.hpp:103-119,
 * lowrank.cpp:361-438).  positions_h: n x d column-major. */
hydot_status hydot_tree_build(const double* positions_h, int n, int d, const double* lo_h,
                              const double* hi_h, hydot_tree* out);
int hydot_tree_num_nodes(hydot_tree t);
int hydot_tree_root(hydot_tree t);
int hydot_tree_depth(hydot_tree t);
/* node v: children (-1 for a leaf) and source count; idx_h may be NULL */
hydot_status hydot_tree_node(hydot_tree t, int v, int* left, int* right, int* n_idx, int* idx_h);
hydot_status hydot_tree_leaf_order(hydot_tree t, int* order_h);
/* bounding box of node v (ClusterTree::Node::lo / hi, d values each) */
hydot_status hydot_tree_node_box(hydot_tree t, int v, double* lo_h, double* hi_h);
void hydot_tree_free(hydot_tree t);

/* lowrank::BlockProvider (lowrank.hpp:122-126): fills the rows_per_source x
 * cols block of source s ROW-major into out_dev (ld >= cols); returns 0 on
 * success. */
typedef int (*hydot_block_fn)(void* user, int source, double* out_dev, int64_t ld);
typedef struct {
    int rows_per_source;
    int64_t cols;
    hydot_block_fn block;
    void* user;
} hydot_provider;

/* Built-in device provider forming Born blocks from resident fields
 * (compress_H's provider, experiments.cpp:235-240, without a dense H):
 * incident_dev_h[s] (N x n_lambda), adjoint_dev_h[s*n_det + d].
 * ready_events_h (optional, n_sources cudaEvent_t or NULL): the context
 * stream waits on source s's event before forming its blocks, so a caller
 * can stream the fields in on another stream while earlier leaves compress. */
typedef struct {
    int64_t N;
    int n_lambda, n_sources, n_det;
    const double* const* incident_dev_h;
    const double* const* adjoint_dev_h;
    const double* w_dev;
    double nu;
    void* const* ready_events_h;
} hydot_born_fields;

/* RecursiveOptions (lowrank.hpp:128-131) + knobs the reference hard-codes
 * (p=20, kprobe=10, lowrank.cpp:344,448).  hint_mode 0 = the reference's
 * sequential warm-start chains (lowrank.cpp:466-471). */
typedef struct {
    uint64_t seed;
    int p;
    int kprobe;
    int hint_mode;
    /* Sharded execution (multi-GPU): the tree is a subtree of a global tree
     * whose pre-order node ids start at node_offset, and local source i is
     * global source source_ids[i].  Seeds (lowrank.cpp:485,494,500) and
     * row_perm use the global ids, so a shard reproduces the global run's
     * per-node seeds.  source_ids NULL / node_offset 0 = unsharded. */
    const int* source_ids;
    int node_offset;
} hydot_rec_opts;

/* lowrank::recursive_lowrank (lowrank.hpp:142-144, lowrank.cpp:459-521).
 * Exactly one of provider / born must be non-NULL.  Outputs: factor (rows
 * in leaf order), row_perm_h (M), node_rank_h / node_depth_h (num_nodes),
 * ledger_h; any output pointer may be NULL. */
hydot_status hydot_recursive_lowrank(hydot_ctx ctx, hydot_tree tree, double eps,
                                     const hydot_provider* provider, const hydot_born_fields* born,
                                     const hydot_rec_opts* opts, hydot_factor* out,
                                     int* row_perm_h, int* node_rank_h, int* node_depth_h,
                                     hydot_ledger* ledger_h);

/* lowrank::recompress (lowrank.hpp:157-158, lowrank.cpp:547-587) */
hydot_status hydot_recompress(hydot_ctx ctx, hydot_factor f, double eps, int rank,
                              hydot_factor* out, hydot_ledger* ledger_h);

/* lowrank::lr_matvec / lr_rmatvec (lowrank.cpp:589-599) on b columns:
 * trans=0: Y (rows x b) = U (V^T X), X cols x b;  trans=1: Y = V (U^T X). */
hydot_status hydot_lr_matmat(hydot_ctx ctx, hydot_factor f, int trans, int b, const double* X_dev,
                             int64_t ldx, double* Y_dev, int64_t ldy);

/* J~ = [E_1 H~, ..., E_nc H~] products with the measurement permutation
 * (permuted_matvec, experiments.cpp:255-262) and the chromophore scaling
 * (forward_measure, born.cpp:118-127; pals.cpp:124-135):
 *  trans=0: X_dev (N*n_c) x b (chromophore-major blocks of N) ->
 *           Y_dev (M x b): y[row_perm[i]] = sum_c eps_c[l, c] (U V^T x_c)[i],
 *           l = row_perm[i] % n_lambda;
 *  trans=1: X_dev (M x b) -> Y_dev (N*n_c) x b: y_c = V U^T gather(E_c x).
 * row_perm_dev: M ints; eps_c_dev: n_lambda x n_c (column-major). */
hydot_status hydot_j_matmat(hydot_ctx ctx, hydot_factor f, int trans, int b, const int* row_perm_dev,
                            const double* eps_c_dev, int n_lambda, int n_c, const double* X_dev,
                            int64_t ldx, double* Y_dev, int64_t ldy);

/* Thin SVD of a dense device matrix (m x n column-major) by the path of
 * fast_thin_svd (lowrank.cpp:62-93); U m x k, s k (host), V n x k,
 * k = min(m,n).  Exposed for kernel-level parity tests. */
hydot_status hydot_thin_svd(hydot_ctx ctx, int64_t m, int64_t n, const double* a_dev, int64_t lda,
                            double* U_dev, double* s_h, double* V_dev);

/* Householder QR (Eigen::HouseholderQR as used at lowrank.cpp:77-83,
 * 564-566): R (n x n upper, device, ld n) and thin Q (m x n, device) of a
 * device m x n matrix, m >= n. */
hydot_status hydot_householder_qr(hydot_ctx ctx, int64_t m, int64_t n, const double* a_dev,
                                  int64_t lda, double* R_dev, double* Q_dev);

/* C = alpha op(A) op(B) + beta C, FP64 DMMA tensor-core GEMM (column-major;
 * transa/transb 0 or 1).  The kernel behind every GEMM of the path. */
hydot_status hydot_dgemm(hydot_ctx ctx, int transa, int transb, int64_t m, int64_t n, int64_t k,
                         double alpha, const double* A_dev, int64_t lda, const double* B_dev,
                         int64_t ldb, double beta, double* C_dev, int64_t ldc);

/* ------------------------------------------------------------ file I/O -- */
/* save_factor / load_factor (lowrank.hpp:165-167, lowrank.cpp:601-655): the
 * reference's binary factor file -- int64 rows, cols, rank; float64 tol;
 * int64 method; int64 plen and plen int64 row_perm; U then V row-major.
 * Errors: HYDOT_ERUNTIME with "cannot write factor: ", "cannot read
 * factor: ", "corrupt factor file: ", "truncated factor file: " + path. */
hydot_status hydot_factor_save(hydot_ctx ctx, hydot_factor f, const int* row_perm_h, int64_t plen,
                               const char* path);
hydot_status hydot_factor_file_info(const char* path, int64_t* rows, int64_t* cols, int64_t* rank,
                                    int64_t* plen);
/* row_perm_h (perm_cap ints, may be NULL) receives the stored permutation */
hydot_status hydot_factor_load(hydot_ctx ctx, const char* path, hydot_factor* out, int* row_perm_h,
                               int64_t perm_cap);
/* save_block / load_block (born.hpp:85-86, born.cpp:156-185): float64 rows,
 * cols, then the block row-major.  The device block is row-major with row
 * stride ld (the layout hydot_born_block writes). */
hydot_status hydot_block_save(hydot_ctx ctx, const double* block_dev, int64_t rows, int64_t cols,
                              int64_t ld, const char* path);
hydot_status hydot_block_file_info(const char* path, int64_t* rows, int64_t* cols);
/* rows_cap: rows the device buffer holds (row stride ld >= cols); a file
 * whose header exceeds rows_cap x ld is rejected (HYDOT_EINVAL) before any
 * device write. */
hydot_status hydot_block_load(hydot_ctx ctx, const char* path, double* block_dev, int64_t ld,
                              int64_t rows_cap, int64_t* rows, int64_t* cols);

/* ----------------------------------------------------------- multi-GPU -- */
/* One process per GPU; an NCCL communicator bound to a context (SURVEY
 * 8(b)/(e)).  Rank 0 calls hydot_comm_unique_id and hands the bytes to every
 * rank (e.g. over torch.distributed); each rank then calls
 * hydot_comm_create with its own context.  NCCL is loaded at run time
 * (libnccl.so.2); without it the calls return HYDOT_ENCCL. */
#define HYDOT_COMM_ID_BYTES 128
typedef struct hydot_comm_s* hydot_comm;
hydot_status hydot_comm_unique_id(unsigned char id_out[HYDOT_COMM_ID_BYTES]);
hydot_status hydot_comm_create(hydot_ctx ctx, int world, int rank, const unsigned char id[HYDOT_COMM_ID_BYTES],
                               hydot_comm* out);
hydot_status hydot_comm_destroy(hydot_comm comm);
hydot_status hydot_comm_info(hydot_comm comm, int* world, int* rank);
/* in-place sum over ranks of n doubles on the context's stream */
hydot_status hydot_comm_allreduce(hydot_ctx ctx, hydot_comm comm, double* buf_dev, int64_t n);
/* hydot_j_matmat under voxel-sharded V (lr_matvec / lr_rmatvec,
 * lowrank.cpp:589-599, + permuted_matvec, experiments.cpp:255-262): U (M x R)
 * replicated, V_loc = this rank's Nloc voxel rows of V.  trans=0: X_dev is
 * the rank's rows of each chromophore block ((Nloc*n_c) x b), Y_dev (M x b)
 * complete on every rank after one R x (b n_c) all-reduce of V^T X;
 * trans=1: X_dev (M x b) replicated, Y_dev the rank's (Nloc*n_c) x b rows
 * (no communication). */
hydot_status hydot_j_matmat_voxel(hydot_ctx ctx, hydot_comm comm, int trans, int b, const double* U_dev,
                                  int64_t M, const double* Vloc_dev, int64_t Nloc, int64_t R,
                                  const int* row_perm_dev, const double* eps_c_dev, int n_lambda, int n_c,
                                  const double* X_dev, int64_t ldx, double* Y_dev, int64_t ldy);

/* ---------------------------------------------------------------- pals -- */
/* Parametric level-set reconstruction, the caller of the compressed
 * operator: proj/include/hydot/pals.hpp, src/pals.cpp.
 * N- and M-length arrays are device pointers; parameters, spectra and
 * concentrations are host arrays. */

/* PaLSParams (pals.hpp:16-32): n_p RBF weights, widths, centres. */
typedef struct hydot_pals_params {
    int np;
    double* alpha;    /* n_p */
    double* beta;     /* n_p, > 0 */
    double* centers;  /* n_p x 3, column-major */
    double tau_level, eps_H, nu_norm;
} hydot_pals_params;

/* The measurement operator handed to the loop (the reference's Hmv,
 * experiments.cpp:255-262): y[row_perm[i]] = (U V^T x)[i]. */
typedef struct hydot_hop {
    hydot_factor H;
    const int* row_perm_dev; /* M ints; NULL = identity order */
} hydot_hop;

enum { HYDOT_PALS_LEVEL_SET = 0, HYDOT_PALS_SHAPE = 1, HYDOT_PALS_JACOBIAN = 2 };

/* level_set / shape / shape_jacobian (pals.cpp:74-119): which selects phi
 * (N), mu = H_eps(phi - tau) (N) or dmu/dp (N x 5 n_p, columns
 * [d/dalpha | d/dbeta | d/dcx | d/dcy | d/dcz], ld ldo). */
hydot_status hydot_pals_eval(hydot_ctx ctx, int which, const hydot_grid_geom* geom,
                             const hydot_pals_params* p, double* out_dev, int64_t ldo);

/* Hmv on b columns: Y (M x b) = P U V^T X, X N x b. */
hydot_status hydot_pals_hmv(hydot_ctx ctx, const hydot_hop* op, int b, const double* X_dev,
                            int64_t ldx, double* Y_dev, int64_t ldy);

/* solve_concentrations (pals.cpp:139-156): c = (W D(p))^+ (W y), D columns
 * E_i H mu; ext_h n_lambda x n_species (extinction at the setup
 * wavelengths, column-major); flagged = rank-deficient system. */
hydot_status hydot_pals_solve_concentrations(hydot_ctx ctx, const hydot_hop* op, const double* mu_dev,
                                             const double* w_dev, const double* y_dev,
                                             const double* ext_h, int n_lambda, int n_species,
                                             double* c_h, int* flagged_h);

/* lm_step (pals.cpp:158-169): dp minimising ||[J; sqrt(nu) I] dp + [eps; 0]||
 * (J M x n on the device, dp n on the host). */
hydot_status hydot_pals_lm_step(hydot_ctx ctx, int64_t M, int n, const double* J_dev, int64_t ldj,
                                const double* eps_dev, double nu, double* dp_h);

/* metrics (pals.cpp:307-329). */
hydot_status hydot_pals_metrics(hydot_ctx ctx, int64_t n, const double* mu_true_dev,
                                const double* mu_hat_dev, double threshold, double* l2_rel_h,
                                double* dice_h, int* flagged_h);

/* ReconConfig (pals.hpp:67-75). */
typedef struct hydot_recon_config {
    int max_outer, max_inner, max_retries;
    double gamma, nu0, stagnation_tol;
    const double* fixed_c_h; /* n_species, or NULL to solve for c */
    /* BASELINE config 4 benchmark knob (0 = the reference loop): after each
     * Gauss-Newton step's Jacobian, normal_blocks J~x products on the step's
     * chromophore-expanded shape-Jacobian columns and as many J~^T y on
     * y = W^2 J~x (E_c axis from ext_h, the operator's row permutation). */
    int normal_blocks;
} hydot_recon_config;

/* TraceRow (pals.hpp:77-84). */
typedef struct hydot_trace_row {
    int outer, inner;
    double resnorm, nu;
    int accepted;
    double dice;
} hydot_trace_row;

/* ReconResult (pals.hpp:86-93); arrays are caller-allocated: p.alpha /
 * p.beta (n_p), p.centers (3 n_p), c_h (n_species), trace_h (trace_cap).
 * trace_len is the full trace length (rows beyond trace_cap dropped);
 * hmv_calls / hmv_columns count the operator products issued. */
typedef struct hydot_recon_result {
    hydot_pals_params p;
    double* c_h;
    hydot_trace_row* trace_h;
    int trace_cap, trace_len;
    double resnorm;
    int converged, flagged;
    int64_t hmv_calls, hmv_columns;
    int64_t normal_columns; /* J~x columns issued by normal_blocks (as many J~^T y) */
} hydot_recon_result;

/* reconstruct (pals.cpp:193-295): alternating concentration / shape
 * reconstruction with Levenberg-Marquardt shape updates on the device;
 * mu_truth_dev (N) optional, for the dice column of the trace. */
hydot_status hydot_pals_reconstruct(hydot_ctx ctx, const hydot_hop* op, const hydot_grid_geom* geom,
                                    const double* ext_h, int n_lambda, int n_species,
                                    const double* y_dev, const double* w_dev,
                                    const hydot_pals_params* init, double noise_norm,
                                    const hydot_recon_config* cfg, const double* mu_truth_dev,
                                    hydot_recon_result* out);

#ifdef __cplusplus
}
#endif
#endif /* HYDOT_B200_H */
