// pals.h -- device PaLS reconstruction: the caller of the
// compressed operator, restating proj/src/pals.cpp with every N- and
// M-sized array resident on the GPU.  Only n_p-, n_species- and
// 5n_p x 5n_p-sized quantities touch the host.
#pragma once

#include <vector>

#include "internal.h"
#include "lowrank.h"

namespace hydot {
namespace pals {

// grid::Grid / build_grid (grid.hpp:22-45, grid.cpp:94-110)
struct Geom {
    int nx = 0, ny = 0, nz = 0;
    double Lx = 0, Ly = 0, Lz = 0, hx = 0, hy = 0, hz = 0;
    static Geom make(const hydot_grid_geom& g);
    int64_t N() const { return int64_t(nx) * ny * nz; }
};

// PaLSParams (pals.hpp:16-32); centers n_p x 3 column-major
struct Params {
    std::vector<double> alpha, beta, centers;
    double tau_level = 0.1, eps_H = 0.05, nu_norm = 1e-3;
    int np() const { return int(alpha.size()); }
    std::vector<double> to_vector() const;                       // pals.cpp:14-23
    Params with_vector(const std::vector<double>& v) const;      // pals.cpp:25-36
    static Params from(const hydot_pals_params& p);
};

// the reference's Hmv (experiments.cpp:255-262): y[perm[i]] = (U V^T x)[i]
struct Hop {
    const Factor* f = nullptr;
    const int* perm = nullptr;  // device, M entries; null = identity
};

enum { EVAL_LEVEL_SET = 0, EVAL_SHAPE = 1, EVAL_JACOBIAN = 2 };

// ---- pals.cu: kernels
// level_set / shape / shape_jacobian (pals.cpp:74-119) into out (ld ldo)
void eval(Ctx& c, int which, const Geom& g, const Params& p, double* out, int64_t ldo);
// eps = w .* (y - D(hmu) cvec), D(m,i) = ext[m % nl, i] * hmu[m] (pals.cpp:180-188)
void residual(Ctx& c, int64_t M, int nl, int nsp, const double* ext_dev, const double* c_dev,
              const double* y, const double* w, const double* hmu, double* eps);
// J(m, j) = -w[m] * ebar[m % nl] * HJ(m, j) (pals.cpp:252-256)
void jscale(Ctx& c, int64_t M, int ncols, int nl, const double* w, const double* ebar_dev,
            const double* HJ, int64_t ldh, double* J, int64_t ldj);
// ||x||_2 (deterministic two-level reduction; synchronises)
double norm2(Ctx& c, int64_t n, const double* x);
// A = [J; sqrt(nu) I] ((M+n) x n), rhs = [-eps; 0]
void stack_damped(Ctx& c, int64_t M, int n, const double* J, int64_t ldj, const double* eps,
                  double nu, double* A, double* rhs);
// sums for metrics(): {sum (a-b)^2, sum a^2, sum b^2, #a>thr, #b>thr, #both}
void metric_sums(Ctx& c, int64_t N, const double* a, const double* b, double thr, double out[6]);

// ---- pals_loop.cpp: host logic over the device pieces
void hmv(Ctx& c, const Hop& h, int b, const double* X, int64_t ldx, double* Y, int64_t ldy);

struct Conc {
    std::vector<double> c;
    bool flagged = false;
};
// solve_concentrations (pals.cpp:139-156)
Conc solve_concentrations(Ctx& c, const Hop& h, const double* mu, const double* w, const double* y,
                          const double* ext_h, int nl, int nsp);
// lm_step (pals.cpp:158-169): device Householder QR of the stacked system
std::vector<double> lm_step(Ctx& c, int64_t M, int n, const double* J, int64_t ldj, const double* eps,
                            double nu);

struct Metrics {
    double l2_rel = 0.0, dice = 0.0;
    bool flagged = false;
};
Metrics metrics(Ctx& c, int64_t N, const double* a, const double* b, double thr);  // pals.cpp:307-329

struct TraceRow {
    int outer = 0, inner = 0;
    double resnorm = 0.0, nu = 0.0;
    bool accepted = false;
    double dice = -1.0;
};
struct ReconCfg {  // ReconConfig (pals.hpp:67-75)
    int max_outer = 30, max_inner = 5, max_retries = 8;
    double gamma = 1.2, nu0 = 1.0, stagnation_tol = 1e-6;
    std::vector<double> fixed_c;
    // BASELINE config 4's per-step work (a benchmark knob, not part of
    // pals.cpp): after each Gauss-Newton step's Jacobian, `normal_blocks`
    // J~x products on the step's chromophore-expanded shape-Jacobian columns
    // x_k = c (x) dmu/dp_k and as many J~^T y products on y = W^2 J~ x (the
    // normal-equation products of the step); 0 = off
    int normal_blocks = 0;
};
struct Recon {  // ReconResult (pals.hpp:86-93)
    Params p;
    std::vector<double> c;
    std::vector<TraceRow> trace;
    double resnorm = 0.0;
    bool converged = false, flagged = false;
    int64_t hmv_calls = 0, hmv_columns = 0;
    int64_t normal_columns = 0;  // J~x (and as many J~^T y) columns of normal_blocks
};
// reconstruct (pals.cpp:193-295)
Recon reconstruct(Ctx& c, const Hop& h, const Geom& g, const double* ext_h, int nl, int nsp,
                  const double* y, const double* w, const Params& init, double noise_norm,
                  const ReconCfg& cfg, const double* mu_truth);

}  // namespace pals
}  // namespace hydot
