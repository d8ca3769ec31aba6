// fileio.cpp -- the reference's factor / block file formats
// for device-resident data:
//   save_factor / load_factor (lowrank.cpp:601-655): int64 rows, cols, rank;
//     float64 tol; int64 method; int64 plen; plen x int64 row_perm; U
//     row-major (rows x rank); V row-major (cols x rank); native endianness.
//   save_block / load_block (born.cpp:156-185): float64 rows, cols; the
//     block row-major.
// Device matrices are column-major: they cross the bus in row chunks of
// <= 64 MB through a device transpose, so a many-GB V never needs a full
// host copy.  Errors keep the reference's runtime_error messages.
#include <cstdio>
#include <memory>
#include <string>

#include "internal.h"
#include "lowrank.h"

namespace hydot {
namespace {

constexpr size_t kChunkBytes = size_t(64) << 20;

struct File {
    FILE* f = nullptr;
    File(const std::string& p, const char* mode) : f(std::fopen(p.c_str(), mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

// write a column-major device matrix (rows x cols, ld) row-major
void write_rowmajor(Ctx& c, FILE* out, const double* A, int64_t rows, int64_t cols, int64_t ld,
                    const std::string& path) {
    if (rows <= 0 || cols <= 0) return;
    const int64_t chunk = std::max<int64_t>(1, int64_t(kChunkBytes / 8) / cols);
    DBuf t = dalloc(c, size_t(std::min(rows, chunk) * cols));
    std::unique_ptr<double[]> h(new double[size_t(std::min(rows, chunk) * cols)]);
    for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
        const int64_t nr = std::min(chunk, rows - r0);
        transpose(c, nr, cols, A + r0, ld, t.d(), cols);  // (cols x nr) col-major = rows row-major
        c.d2h(h.get(), t.d(), size_t(nr * cols));
        if (std::fwrite(h.get(), 8, size_t(nr * cols), out) != size_t(nr * cols))
            throw std::runtime_error("cannot write factor: " + path);
    }
}

// read rows x cols row-major values into a column-major device matrix
bool read_rowmajor(Ctx& c, FILE* in, double* A, int64_t rows, int64_t cols, int64_t ld) {
    if (rows <= 0 || cols <= 0) return true;
    const int64_t chunk = std::max<int64_t>(1, int64_t(kChunkBytes / 8) / cols);
    DBuf t = dalloc(c, size_t(std::min(rows, chunk) * cols));
    std::unique_ptr<double[]> h(new double[size_t(std::min(rows, chunk) * cols)]);
    for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
        const int64_t nr = std::min(chunk, rows - r0);
        if (std::fread(h.get(), 8, size_t(nr * cols), in) != size_t(nr * cols)) return false;
        HYDOT_CUDA(cudaMemcpyAsync(t.d(), h.get(), size_t(nr * cols) * 8, cudaMemcpyHostToDevice, c.stream));
        transpose(c, cols, nr, t.d(), cols, A + r0, ld);  // row-major chunk -> column-major rows
        c.sync();  // h is reused
    }
    return true;
}

}  // namespace

void save_factor_file(Ctx& c, const std::string& path, const Factor& f, const int* perm, int64_t plen) {
    File out(path, "wb");
    if (!out.f) throw std::runtime_error("cannot write factor: " + path);
    const int64_t hdr[3] = {f.rows, f.cols, f.rank};
    const double tol = f.tol;
    const int64_t meth = f.method, pl = plen;
    bool ok = std::fwrite(hdr, 8, 3, out.f) == 3 && std::fwrite(&tol, 8, 1, out.f) == 1 &&
              std::fwrite(&meth, 8, 1, out.f) == 1 && std::fwrite(&pl, 8, 1, out.f) == 1;
    for (int64_t i = 0; ok && i < plen; ++i) {
        const int64_t p = perm[i];
        ok = std::fwrite(&p, 8, 1, out.f) == 1;
    }
    if (!ok) throw std::runtime_error("cannot write factor: " + path);
    write_rowmajor(c, out.f, f.U.d(), f.rows, f.rank, f.rows, path);
    write_rowmajor(c, out.f, f.V.d(), f.cols, f.rank, f.cols, path);
}

bool factor_file_info(const std::string& path, int64_t& rows, int64_t& cols, int64_t& rank, int64_t& plen) {
    File in(path, "rb");
    if (!in.f) throw std::runtime_error("cannot read factor: " + path);
    int64_t hdr[3];
    double tol;
    int64_t meth;
    if (std::fread(hdr, 8, 3, in.f) != 3 || std::fread(&tol, 8, 1, in.f) != 1 ||
        std::fread(&meth, 8, 1, in.f) != 1 || std::fread(&plen, 8, 1, in.f) != 1)
        throw std::runtime_error("corrupt factor file: " + path);
    rows = hdr[0];
    cols = hdr[1];
    rank = hdr[2];
    if (rows < 0 || cols < 0 || rank < 0 || rank > std::min(rows, cols) || plen < 0)
        throw std::runtime_error("corrupt factor file: " + path);
    return true;
}

Factor load_factor_file(Ctx& c, const std::string& path, std::vector<int>& perm) {
    File in(path, "rb");
    if (!in.f) throw std::runtime_error("cannot read factor: " + path);
    int64_t hdr[3], meth = 0, plen = 0;
    double tol = 0.0;
    if (std::fread(hdr, 8, 3, in.f) != 3 || std::fread(&tol, 8, 1, in.f) != 1 ||
        std::fread(&meth, 8, 1, in.f) != 1 || std::fread(&plen, 8, 1, in.f) != 1)
        throw std::runtime_error("corrupt factor file: " + path);
    const int64_t m = hdr[0], n = hdr[1], r = hdr[2];
    if (m < 0 || n < 0 || r < 0 || r > std::min(m, n) || plen < 0)
        throw std::runtime_error("corrupt factor file: " + path);
    perm.assign(size_t(plen), 0);
    for (int64_t i = 0; i < plen; ++i) {
        int64_t p;
        if (std::fread(&p, 8, 1, in.f) != 1) throw std::runtime_error("truncated factor file: " + path);
        perm[size_t(i)] = int(p);
    }
    Factor f;
    f.rows = m;
    f.cols = n;
    f.rank = r;
    f.tol = tol;
    f.method = int(meth);
    f.U = dalloc(c, size_t(std::max<int64_t>(m * r, 1)));
    f.V = dalloc(c, size_t(std::max<int64_t>(n * r, 1)));
    if (!read_rowmajor(c, in.f, f.U.d(), m, r, m) || !read_rowmajor(c, in.f, f.V.d(), n, r, n))
        throw std::runtime_error("truncated factor file: " + path);
    return f;
}

void save_block_file(Ctx& c, const std::string& path, const double* block, int64_t rows, int64_t cols,
                     int64_t ld) {
    File out(path, "wb");
    if (!out.f) throw std::runtime_error("cannot write block: " + path);
    const double hdr[2] = {double(rows), double(cols)};
    if (std::fwrite(hdr, 8, 2, out.f) != 2) throw std::runtime_error("cannot write block: " + path);
    // the device block is row-major with row stride ld: rows go out as they are
    if (rows <= 0 || cols <= 0) return;
    const int64_t chunk = std::max<int64_t>(1, int64_t(kChunkBytes / 8) / cols);
    std::unique_ptr<double[]> h(new double[size_t(std::min(rows, chunk) * cols)]);
    for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
        const int64_t nr = std::min(chunk, rows - r0);
        HYDOT_CUDA(cudaMemcpy2DAsync(h.get(), size_t(cols) * 8, block + r0 * ld, size_t(ld) * 8,
                                     size_t(cols) * 8, size_t(nr), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (std::fwrite(h.get(), 8, size_t(nr * cols), out.f) != size_t(nr * cols))
            throw std::runtime_error("cannot write block: " + path);
    }
}

void block_file_info(const std::string& path, int64_t& rows, int64_t& cols) {
    File in(path, "rb");
    if (!in.f) throw std::runtime_error("cannot read block: " + path);
    double hdr[2];
    if (std::fread(hdr, 8, 2, in.f) != 2 || hdr[0] < 0 || hdr[1] < 0)
        throw std::runtime_error("corrupt block file: " + path);
    rows = int64_t(hdr[0]);
    cols = int64_t(hdr[1]);
}

void load_block_file(Ctx& c, const std::string& path, double* block, int64_t ld, int64_t rows_cap, int64_t& rows,
                     int64_t& cols) {
    File in(path, "rb");
    if (!in.f) throw std::runtime_error("cannot read block: " + path);
    double hdr[2];
    if (std::fread(hdr, 8, 2, in.f) != 2 || hdr[0] < 0 || hdr[1] < 0)
        throw std::runtime_error("corrupt block file: " + path);
    rows = int64_t(hdr[0]);
    cols = int64_t(hdr[1]);
    if (ld < cols) throw std::invalid_argument("load_block: leading dimension smaller than the block");
    if (rows > rows_cap) throw std::invalid_argument("load_block: block has more rows than the buffer holds");
    if (rows <= 0 || cols <= 0) return;
    const int64_t chunk = std::max<int64_t>(1, int64_t(kChunkBytes / 8) / cols);
    std::unique_ptr<double[]> h(new double[size_t(std::min(rows, chunk) * cols)]);
    for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
        const int64_t nr = std::min(chunk, rows - r0);
        if (std::fread(h.get(), 8, size_t(nr * cols), in.f) != size_t(nr * cols))
            throw std::runtime_error("truncated block file: " + path);
        HYDOT_CUDA(cudaMemcpy2DAsync(block + r0 * ld, size_t(ld) * 8, h.get(), size_t(cols) * 8,
                                     size_t(cols) * 8, size_t(nr), cudaMemcpyHostToDevice, c.stream));
        c.sync();
    }
}

}  // namespace hydot
