// fem_oracle.cpp -- CPU ORACLE (test infrastructure only).
//
// Restatement of the reference's own field operator and point sources
// (/root/reference/proj/src/grid.cpp:12-174, 212-237; born.cpp:27-35):
// trilinear-element stiffness K (Dirichlet side vertices eliminated, unit
// diagonal), row-lumped mass M and the bilinear z-face mass R, element
// matrices by the same 2x2x2 / 2x2 Gauss rule.  Two forms:
//   * fem_dense: the reference's triplet assembly, literally (cells in
//     (cz, cy, cx) order, local a then b, duplicates summed in insertion
//     order) -> a dense K + sigma M + sigma' R for tiny grids.  It pins the
//     matrix-free form below to the reference's assembly semantics.
//   * fem_apply: matrix-free, in the device kernel's operation order (cells
//     (cz, cy, cx) ascending, local vertex b inner), so device parity is
//     bitwise.
// Used only by tests/ as the checker of csrc/cg.cu's FEM mode.
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fem_oracle.h"

namespace fem_oracle {

constexpr double kGaussPt = 0.57735026918962576451;  // grid.cpp:14

// element_matrices (grid.cpp:39-64), face_mass (:67-88)
void element(double hx, double hy, double hz, double Ke[64], double Me[64], double Re[16]) {
    for (int e = 0; e < 64; ++e) Ke[e] = Me[e] = 0.0;
    for (int e = 0; e < 16; ++e) Re[e] = 0.0;
    const double detJ = hx * hy * hz / 8.0;
    const double ih[3] = {2.0 / hx, 2.0 / hy, 2.0 / hz};
    for (int qx = 0; qx < 2; ++qx)
        for (int qy = 0; qy < 2; ++qy)
            for (int qz = 0; qz < 2; ++qz) {
                const double xi = qx ? kGaussPt : -kGaussPt, eta = qy ? kGaussPt : -kGaussPt,
                             zeta = qz ? kGaussPt : -kGaussPt;
                double Nv[8], G[8][3];
                for (int a = 0; a < 8; ++a) {
                    const double sx = (a & 1) ? 1.0 : -1.0, sy = (a & 2) ? 1.0 : -1.0, sz = (a & 4) ? 1.0 : -1.0;
                    Nv[a] = 0.125 * (1 + sx * xi) * (1 + sy * eta) * (1 + sz * zeta);
                    G[a][0] = 0.125 * sx * (1 + sy * eta) * (1 + sz * zeta) * ih[0];
                    G[a][1] = 0.125 * sy * (1 + sx * xi) * (1 + sz * zeta) * ih[1];
                    G[a][2] = 0.125 * sz * (1 + sx * xi) * (1 + sy * eta) * ih[2];
                }
                for (int a = 0; a < 8; ++a)
                    for (int b = 0; b < 8; ++b) {
                        const double dot = G[a][0] * G[b][0] + G[a][1] * G[b][1] + G[a][2] * G[b][2];
                        Ke[a * 8 + b] += detJ * dot;
                        Me[a * 8 + b] += detJ * Nv[a] * Nv[b];
                    }
            }
    const double detF = hx * hy / 4.0;
    for (int qx = 0; qx < 2; ++qx)
        for (int qy = 0; qy < 2; ++qy) {
            const double xi = qx ? kGaussPt : -kGaussPt, eta = qy ? kGaussPt : -kGaussPt;
            for (int a = 0; a < 4; ++a) {
                const double Na = 0.25 * (1 + ((a & 1) ? 1.0 : -1.0) * xi) * (1 + ((a & 2) ? 1.0 : -1.0) * eta);
                for (int b = 0; b < 4; ++b) {
                    const double Nb =
                        0.25 * (1 + ((b & 1) ? 1.0 : -1.0) * xi) * (1 + ((b & 2) ? 1.0 : -1.0) * eta);
                    Re[a * 4 + b] += detF * Na * Nb;
                }
            }
        }
}

// matrix-free y = (K + sigma M + sigma' R) x in the device order
void apply(const Geom& g, const double* E, double sigma, double sigmap, const double* x, double* y) {
    const double *Ke = E, *Me = E + 64, *Re = E + 128;
    for (int iz = 0; iz < g.nz; ++iz)
        for (int iy = 0; iy < g.ny; ++iy)
            for (int ix = 0; ix < g.nx; ++ix) {
                const int64_t i = g.idx(ix, iy, iz);
                const bool di = g.dir(ix, iy);
                double kx = 0.0, m = 0.0;
                for (int oz = -1; oz <= 0; ++oz) {
                    const int cz = iz + oz;
                    if (cz < 0 || cz > g.nz - 2) continue;
                    for (int oy = -1; oy <= 0; ++oy) {
                        const int cy = iy + oy;
                        if (cy < 0 || cy > g.ny - 2) continue;
                        for (int ox = -1; ox <= 0; ++ox) {
                            const int cx = ix + ox;
                            if (cx < 0 || cx > g.nx - 2) continue;
                            const int a = (ox ? 1 : 0) | (oy ? 2 : 0) | (oz ? 4 : 0);
                            for (int b = 0; b < 8; ++b) {
                                const int jx = cx + (b & 1), jy = cy + ((b >> 1) & 1), jz = cz + ((b >> 2) & 1);
                                m = m + Me[a * 8 + b];
                                if (!di && !g.dir(jx, jy)) kx = kx + Ke[a * 8 + b] * x[g.idx(jx, jy, jz)];
                            }
                        }
                    }
                }
                double v = di ? x[i] : kx;
                v = v + sigma * (m * x[i]);
                if (iz == 0 || iz == g.nz - 1) {
                    double rx = 0.0;
                    for (int oy = -1; oy <= 0; ++oy) {
                        const int cy = iy + oy;
                        if (cy < 0 || cy > g.ny - 2) continue;
                        for (int ox = -1; ox <= 0; ++ox) {
                            const int cx = ix + ox;
                            if (cx < 0 || cx > g.nx - 2) continue;
                            const int a = (ox ? 1 : 0) | (oy ? 2 : 0);
                            for (int b = 0; b < 4; ++b)
                                rx = rx + Re[a * 4 + b] * x[g.idx(cx + (b & 1), cy + ((b >> 1) & 1), iz)];
                        }
                    }
                    v = v + sigmap * rx;
                }
                y[i] = v;
            }
}

// the reference's triplet assembly (grid.cpp:112-174), dense, duplicates
// summed in insertion order: K, M (lumped), R, then A = K + sigma M + sigma' R
void dense(const Geom& g, double sigma, double sigmap, double* A) {
    const int64_t N = g.N();
    double Ke[64], Me[64], Re[16];
    element(g.hx, g.hy, g.hz, Ke, Me, Re);
    std::vector<double> K(size_t(N * N), 0.0), M(size_t(N * N), 0.0), R(size_t(N * N), 0.0);
    auto at = [&](std::vector<double>& T, int64_t r, int64_t c) -> double& { return T[size_t(r + c * N)]; };
    for (int cz = 0; cz < g.nz - 1; ++cz)
        for (int cy = 0; cy < g.ny - 1; ++cy)
            for (int cx = 0; cx < g.nx - 1; ++cx) {
                int64_t v[8];
                bool d[8];
                for (int a = 0; a < 8; ++a) {
                    const int jx = cx + (a & 1), jy = cy + ((a >> 1) & 1), jz = cz + ((a >> 2) & 1);
                    v[a] = g.idx(jx, jy, jz);
                    d[a] = g.dir(jx, jy);
                }
                for (int a = 0; a < 8; ++a) {
                    if (d[a]) continue;
                    for (int b = 0; b < 8; ++b) {
                        if (d[b]) continue;
                        at(K, v[a], v[b]) += Ke[a * 8 + b];  // assemble_stiffness
                    }
                }
                for (int a = 0; a < 8; ++a)
                    for (int b = 0; b < 8; ++b) at(M, v[a], v[a]) += Me[a * 8 + b];  // lumped mass
            }
    for (int iy = 0; iy < g.ny; ++iy)
        for (int ix = 0; ix < g.nx; ++ix)
            for (int iz = 0; iz < g.nz; ++iz)
                if (g.dir(ix, iy)) at(K, g.idx(ix, iy, iz), g.idx(ix, iy, iz)) += 1.0;
    for (int iz : {0, g.nz - 1})
        for (int cy = 0; cy < g.ny - 1; ++cy)
            for (int cx = 0; cx < g.nx - 1; ++cx) {
                int64_t v[4];
                for (int a = 0; a < 4; ++a) v[a] = g.idx(cx + (a & 1), cy + ((a >> 1) & 1), iz);
                for (int a = 0; a < 4; ++a)
                    for (int b = 0; b < 4; ++b) at(R, v[a], v[b]) += Re[a * 4 + b];  // assemble_robin
            }
    for (int64_t e = 0; e < N * N; ++e) A[e] = K[size_t(e)] + sigma * M[size_t(e)] + sigmap * R[size_t(e)];
}

// source_rhs (born.cpp:27-35) over point_source_vector (grid.cpp:212-237)
std::vector<double> point_source(const Geom& g, const double r[3]) {
    if (!(r[0] >= -g.Lx && r[0] <= g.Lx && r[1] >= -g.Ly && r[1] <= g.Ly && r[2] >= 0.0 && r[2] <= g.Lz))
        throw std::invalid_argument("point_source_vector: point outside domain");
    auto clamp_cell = [](double t, int ncells) {
        int c = static_cast<int>(std::floor(t));
        if (c < 0) c = 0;
        if (c > ncells - 1) c = ncells - 1;
        return c;
    };
    const double tx = (r[0] + g.Lx) / g.hx, ty = (r[1] + g.Ly) / g.hy, tz = r[2] / g.hz;
    const int cx = clamp_cell(tx, g.nx - 1), cy = clamp_cell(ty, g.ny - 1), cz = clamp_cell(tz, g.nz - 1);
    const double xi = 2 * (tx - cx) - 1, eta = 2 * (ty - cy) - 1, zeta = 2 * (tz - cz) - 1;
    std::vector<double> b(static_cast<size_t>(g.N()), 0.0);
    double n2 = 0.0;
    for (int a = 0; a < 8; ++a) {
        const int jx = cx + (a & 1), jy = cy + ((a >> 1) & 1), jz = cz + ((a >> 2) & 1);
        const double sx = (a & 1) ? 1.0 : -1.0, sy = (a & 2) ? 1.0 : -1.0, sz = (a & 4) ? 1.0 : -1.0;
        double w = 0.125 * (1 + sx * xi) * (1 + sy * eta) * (1 + sz * zeta);
        if (g.dir(jx, jy)) w = 0.0;
        b[size_t(g.idx(jx, jy, jz))] = w;
        n2 += w * w;
    }
    if (n2 == 0.0) throw std::invalid_argument("source support falls entirely on the Dirichlet boundary");
    return b;
}

// CG on the FEM operator (same recurrences as the 7-point oracle CG)
int cg(const Geom& g, const double* E, double sigma, double sigmap, const double* b, double* x, double tol,
       int max_iter, int fixed_iters, double* relres_out) {
    const int64_t N = g.N();
    std::vector<double> r(b, b + N), p(b, b + N), q(static_cast<size_t>(N));
    std::fill(x, x + N, 0.0);
    auto dot = [&](const double* a, const double* c) {
        double s = 0.0;
        for (int64_t i = 0; i < N; ++i) s += a[i] * c[i];
        return s;
    };
    double rr = dot(r.data(), r.data());
    const double bnorm = std::sqrt(rr);
    int it = 0;
    double relres = bnorm > 0 ? 1.0 : 0.0;
    const int limit = fixed_iters > 0 ? fixed_iters : max_iter;
    for (it = 0; it < limit;) {
        apply(g, E, sigma, sigmap, p.data(), q.data());
        const double alpha = rr / dot(p.data(), q.data());
        for (int64_t i = 0; i < N; ++i) {
            x[i] = x[i] + alpha * p[i];
            r[i] = r[i] - alpha * q[i];
        }
        const double rr_new = dot(r.data(), r.data());
        ++it;
        relres = std::sqrt(rr_new) / bnorm;
        if (fixed_iters <= 0 && relres <= tol) break;
        const double beta = rr_new / rr;
        for (int64_t i = 0; i < N; ++i) p[i] = r[i] + beta * p[i];
        rr = rr_new;
    }
    if (relres_out) *relres_out = relres;
    return it;
}

}  // namespace fem_oracle

using namespace fem_oracle;

namespace {
thread_local std::string g_ferr;
template <class F>
int fguard(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_ferr = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_ferr = e.what();
        return 2;
    }
}
}  // namespace

extern "C" {

const char* oracle_fem_last_error() { return g_ferr.c_str(); }

int oracle_fem_element(double hx, double hy, double hz, double* Ke, double* Me, double* Re) {
    return fguard([&] { element(hx, hy, hz, Ke, Me, Re); });
}

int oracle_fem_apply(int nx, int ny, int nz, double Lx, double Ly, double Lz, double sigma, double sigmap,
                     const double* x, double* y) {
    return fguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        double E[144];
        element(g.hx, g.hy, g.hz, E, E + 64, E + 128);
        apply(g, E, sigma, sigmap, x, y);
    });
}

int oracle_fem_dense(int nx, int ny, int nz, double Lx, double Ly, double Lz, double sigma, double sigmap,
                     double* A) {
    return fguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        if (g.N() > 4096) throw std::invalid_argument("fem_dense: grid too large");
        dense(g, sigma, sigmap, A);
    });
}

int oracle_fem_point_source(int nx, int ny, int nz, double Lx, double Ly, double Lz, const double* r, double* b) {
    return fguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        std::vector<double> v = point_source(g, r);
        std::copy(v.begin(), v.end(), b);
    });
}

int oracle_fem_fields(int nx, int ny, int nz, double Lx, double Ly, double Lz, int nl, const double* sigma,
                      const double* sigmap, const double* inv_D, const double* points, int n_pts, double tol,
                      int max_iter, int fixed_iters, int threads, double* out, int* iters, double* relres) {
    return fguard([&] {
        Geom g(nx, ny, nz, Lx, Ly, Lz);
        double E[144];
        element(g.hx, g.hy, g.hz, E, E + 64, E + 128);
        const int64_t N = g.N();
        const int total = n_pts * nl;
        std::vector<std::vector<double>> rhs;
        for (int s = 0; s < n_pts; ++s) rhs.push_back(point_source(g, points + 3 * s));
        const int T = std::max(1, threads);
        auto work = [&](int t) {
            for (int k = t; k < total; k += T) {
                const int s = k / nl, l = k % nl;
                double* x = out + int64_t(k) * N;
                double rr;
                const int it = cg(g, E, sigma[l], sigmap[l], rhs[size_t(s)].data(), x, tol, max_iter, fixed_iters, &rr);
                for (int64_t i = 0; i < N; ++i) x[i] *= inv_D[l];
                if (iters) iters[k] = it;
                if (relres) relres[k] = rr;
            }
        };
        if (T == 1) {
            work(0);
        } else {
            std::vector<std::thread> ts;
            for (int t = 0; t < T; ++t) ts.emplace_back(work, t);
            for (auto& th : ts) th.join();
        }
    });
}

}  // extern "C"
