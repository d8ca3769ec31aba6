// fem_oracle.h -- CPU ORACLE (test infrastructure only): the grid geometry
// of grid::build_grid (grid.cpp:94-110) shared by fem_oracle.cpp and
// krylov_oracle.cpp.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace fem_oracle {

struct Geom {
    int nx, ny, nz;
    double Lx, Ly, Lz, hx, hy, hz;
    Geom(int x, int y, int z, double lx, double ly, double lz) : nx(x), ny(y), nz(z), Lx(lx), Ly(ly), Lz(lz) {
        if (nx < 3 || ny < 3 || nz < 2) throw std::invalid_argument("fields_solve: bad grid");
        if (Lx <= 0 || Ly <= 0 || Lz <= 0) throw std::invalid_argument("build_grid: extents must be positive");
        hx = 2 * Lx / (nx - 1);  // grid.cpp:106-108
        hy = 2 * Ly / (ny - 1);
        hz = Lz / (nz - 1);
    }
    int64_t N() const { return int64_t(nx) * ny * nz; }
    int64_t idx(int ix, int iy, int iz) const { return (int64_t(iz) * ny + iy) * nx + ix; }
    bool dir(int ix, int iy) const { return ix == 0 || ix == nx - 1 || iy == 0 || iy == ny - 1; }
};

// element_matrices / face_mass (grid.cpp:39-88)
void element(double hx, double hy, double hz, double Ke[64], double Me[64], double Re[16]);
// source_rhs over point_source_vector (born.cpp:27-35, grid.cpp:212-237)
std::vector<double> point_source(const Geom& g, const double r[3]);

}  // namespace fem_oracle
