// born.cu -- per-(source, detector) Born block assembly.
//
// Replaces born::assemble_H_block (born.cpp:82-98):
//   row (d*nl + l), voxel v  =  (-nu) * ((phi_d[v,l] * phi_s[v,l]) * w[v])
// evaluated with exactly the reference's multiplication order (no adds, so
// the result is bitwise identical to the CPU).  HBM-bound: each thread moves
// 128-bit vectors (double2) along the voxel axis, which is contiguous both in
// the fields (each wavelength column is voxel-contiguous, born.hpp:45-50) and
// in the row-major output block, so every load and store is coalesced.
#include "internal.h"

namespace hydot {
namespace {

__global__ void born_block_k(int64_t N, int nl, const double* __restrict__ inc,
                             const double* const* __restrict__ adj, const double* __restrict__ w,
                             double nu, double* __restrict__ out, int64_t ld, int vec2) {
    const int row = blockIdx.y;
    const int d = row / nl, l = row - d * nl;
    const double* __restrict__ pd = adj[d] + int64_t(l) * N;
    const double* __restrict__ ps = inc + int64_t(l) * N;
    double* __restrict__ o = out + int64_t(row) * ld;
    const double mnu = -nu;
    if (vec2) {
        const int64_t n2 = N >> 1;
        for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2;
             i += int64_t(gridDim.x) * blockDim.x) {
            double2 a = __ldg(reinterpret_cast<const double2*>(pd) + i);
            double2 b = __ldg(reinterpret_cast<const double2*>(ps) + i);
            double2 c = __ldg(reinterpret_cast<const double2*>(w) + i);
            double2 r;
            r.x = __dmul_rn(mnu, __dmul_rn(__dmul_rn(a.x, b.x), c.x));
            r.y = __dmul_rn(mnu, __dmul_rn(__dmul_rn(a.y, b.y), c.y));
            __stcs(reinterpret_cast<double2*>(o) + i, r);
        }
        if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
            int64_t v = N - 1;
            o[v] = __dmul_rn(mnu, __dmul_rn(__dmul_rn(pd[v], ps[v]), w[v]));
        }
    } else {
        for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < N;
             v += int64_t(gridDim.x) * blockDim.x)
            o[v] = __dmul_rn(mnu, __dmul_rn(__dmul_rn(pd[v], ps[v]), w[v]));
    }
}

// y[(s nd + d) nl + l] = F[s][l][det[s nd + d]]: detector values of point
// fields (interpolate at a vertex, grid.cpp; measurement_index order
// born.hpp:35-37)
__global__ void gather_measure_k(int ns, int nd, int nl, int64_t N, const double* __restrict__ F,
                                 const int64_t* __restrict__ det, double* __restrict__ y) {
    const int total = ns * nd * nl;
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < total; m += gridDim.x * blockDim.x) {
        const int l = m % nl, sd = m / nl, s = sd / nd;
        y[m] = F[(int64_t(s) * nl + l) * N + det[sd]];
    }
}

}  // namespace

void gather_measure(Ctx& c, int ns, int nd, int nl, int64_t N, const double* F, const int64_t* det_dev, double* y) {
    const int total = ns * nd * nl;
    const int blocks = std::max(1, std::min((total + 255) / 256, c.num_sms * 4));
    gather_measure_k<<<blocks, 256, 0, c.stream>>>(ns, nd, nl, N, F, det_dev, y);
    c.check_launch();
}

void born_block(Ctx& c, int64_t N, int nl, const double* inc, const double* const* adj_h, int nd,
                const double* w, double nu, double* out, int64_t ld) {
    StageTimer _t(c, "born_block", N, nl, nd, 0.0, 8.0 * double(N) * (2.0 * nd * nl + nl + 1));
    if (N <= 0 || nl <= 0 || nd <= 0) return;
    if (ld < N) throw std::invalid_argument("assemble_H_block: ld < N");
    int rows = nd * nl;
    if (rows > 65535) throw std::invalid_argument("assemble_H_block: too many rows");
    DBuf ptrs(c, sizeof(double*) * size_t(nd));
    HYDOT_CUDA(cudaMemcpyAsync(ptrs.as<void>(), adj_h, sizeof(double*) * size_t(nd),
                               cudaMemcpyHostToDevice, c.stream));
    bool al = ((reinterpret_cast<uintptr_t>(inc) | reinterpret_cast<uintptr_t>(w) |
                reinterpret_cast<uintptr_t>(out)) & 15) == 0 && (N % 2 == 0) && (ld % 2 == 0);
    for (int d = 0; d < nd && al; ++d)
        if (reinterpret_cast<uintptr_t>(adj_h[d]) & 15) al = false;
    int64_t work = al ? N / 2 : N;
    int bx = int(std::min<int64_t>((work + 255) / 256, std::max<int64_t>(1, (int64_t(c.num_sms) * 8 + rows - 1) / rows * 4)));
    bx = std::max(bx, 1);
    dim3 grid = dim3(unsigned(bx), unsigned(rows));
    born_block_k<<<grid, 256, 0, c.stream>>>(N, nl, inc, ptrs.as<const double*>(), w, nu, out, ld,
                                             al ? 1 : 0);
    c.check_launch();
}

}  // namespace hydot
