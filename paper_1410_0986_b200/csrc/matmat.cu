// matmat.cu -- epilogues of the low-rank J~ products.
//
// J~ X = P [E_1 U, ..., E_nc U] (V^T X_c): the two GEMMs run on the DMMA
// kernel; these kernels apply the chromophore scaling E_c (forward_measure,
// born.cpp:118-127: row m scaled by sum_c c_c eps_c(lambda_{m mod nl})) and
// the measurement permutation (permuted_matvec, experiments.cpp:255-262:
// out[row_perm[i]] = tmp[i]).
#include "internal.h"

namespace hydot {
namespace {

// Y[row_perm[i], j] = sum_c eps_c[l, c] * T[i, j*nc + c],  l = row_perm[i] % nl
__global__ void j_combine_k(int64_t M, int b, int nc, int nl, const double* __restrict__ T,
                            int64_t ldt, const int* __restrict__ rp, const double* __restrict__ eps,
                            double* __restrict__ Y, int64_t ldy) {
    int64_t total = M * b;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % M;
        int j = int(e / M);
        int row = rp[i];
        int l = row % nl;
        double s = 0.0;
        for (int c = 0; c < nc; ++c) s += eps[l + c * nl] * T[i + int64_t(j * nc + c) * ldt];
        Y[row + int64_t(j) * ldy] = s;
    }
}

// G[i, j*nc + c] = eps_c[l, c] * X[row_perm[i], j]
__global__ void j_gather_scale_k(int64_t M, int b, int nc, int nl, const double* __restrict__ X,
                                 int64_t ldx, const int* __restrict__ rp,
                                 const double* __restrict__ eps, double* __restrict__ G,
                                 int64_t ldg) {
    int64_t total = M * b;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = e % M;
        int j = int(e / M);
        int row = rp[i];
        int l = row % nl;
        double x = X[row + int64_t(j) * ldx];
        for (int c = 0; c < nc; ++c) G[i + int64_t(j * nc + c) * ldg] = eps[l + c * nl] * x;
    }
}

}  // namespace

void j_combine(Ctx& c, int64_t M, int b, int nc, int nl, const double* T, int64_t ldt,
               const int* row_perm, const double* eps_c, double* Y, int64_t ldy) {
    int blocks = int(std::max<int64_t>(1, std::min<int64_t>((M * b + 255) / 256, int64_t(c.num_sms) * 8)));
    j_combine_k<<<blocks, 256, 0, c.stream>>>(M, b, nc, nl, T, ldt, row_perm, eps_c, Y, ldy);
    c.check_launch();
}

void j_gather_scale(Ctx& c, int64_t M, int b, int nc, int nl, const double* X, int64_t ldx,
                    const int* row_perm, const double* eps_c, double* G, int64_t ldg) {
    int blocks = int(std::max<int64_t>(1, std::min<int64_t>((M * b + 255) / 256, int64_t(c.num_sms) * 8)));
    j_gather_scale_k<<<blocks, 256, 0, c.stream>>>(M, b, nc, nl, X, ldx, row_perm, eps_c, G, ldg);
    c.check_launch();
}

}  // namespace hydot
