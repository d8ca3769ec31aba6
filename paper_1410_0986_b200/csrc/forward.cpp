// forward.cpp -- the nonlinear (full diffusion) forward model on the device,
// experiments::full_diffusion_forward (experiments.cpp:154-206; SURVEY 8(f)
// #4): per wavelength, the fields of the perturbed medium
//   (K + M_w + sigma'_l R) x = e_src,  w = sigma_l + dsig_l mu(v)
// and of the background (mu = 0), detector values scaled by 1/D_l
// (born.cpp:62-63), y_scattered = y_total - y_incident.  Both solves run the
// same variable-coefficient batched CG (fields_solve_var), so mu = 0 gives
// bit-identical totals and incidents (test_harness.cpp:125-136).  Sources
// are solved in batches that keep one batch's fields under ~16 GB.
#include <algorithm>
#include <vector>

#include "internal.h"

namespace hydot {

void full_forward(Ctx& c, const hydot_grid7& g, int nl, const double* sigma, const double* sigmap,
                  const double* inv_D, const double* dsigma, const double* mu_dev, const int64_t* src_h, int ns,
                  const int64_t* det_h, int nd, double tol, int max_iter, int fixed_iters, double* y_tot,
                  double* y_inc, int* iters_max) {
    if (ns < 1 || nd < 1 || nl < 1) throw std::invalid_argument("full_forward: empty setup");
    const int64_t N = int64_t(g.nx) * g.ny * g.nz;
    for (int k = 0; k < ns * nd; ++k)
        if (det_h[k] < 0 || det_h[k] >= N) throw std::invalid_argument("full_forward: detector outside domain");
    DBuf dsig = dalloc(c, size_t(nl)), zero = dalloc(c, size_t(nl));
    HYDOT_CUDA(cudaMemcpyAsync(dsig.d(), dsigma, size_t(nl) * 8, cudaMemcpyHostToDevice, c.stream));
    fill(c, nl, 1, 0.0, zero.d(), nl);
    const int64_t per_src = int64_t(nl) * N;
    const int batch = int(std::max<int64_t>(1, std::min<int64_t>(ns, (int64_t(16) << 30) / (8 * per_src))));
    DBuf F = dalloc(c, size_t(batch) * size_t(per_src));
    DBuf det = DBuf(c, size_t(ns) * nd * sizeof(int64_t));
    HYDOT_CUDA(cudaMemcpyAsync(det.as<void>(), det_h, size_t(ns) * nd * sizeof(int64_t), cudaMemcpyHostToDevice,
                               c.stream));
    int imax = 0;
    for (int s0 = 0; s0 < ns; s0 += batch) {
        const int nb = std::min(batch, ns - s0);
        for (int pass = 0; pass < 2; ++pass) {
            CGStats st;
            fields_solve_var(c, g, nl, sigma, sigmap, inv_D, pass == 0 ? dsig.d() : zero.d(), mu_dev, src_h + s0, nb,
                             tol, max_iter, fixed_iters, F.d(), &st);
            for (int it : st.iters) imax = std::max(imax, it);
            gather_measure(c, nb, nd, nl, N, F.d(), det.as<int64_t>() + int64_t(s0) * nd,
                           (pass == 0 ? y_tot : y_inc) + int64_t(s0) * nd * nl);
        }
    }
    c.sync();
    if (iters_max) *iters_max = imax;
}

}  // namespace hydot
