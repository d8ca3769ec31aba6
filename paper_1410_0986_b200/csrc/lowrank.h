// lowrank.h -- device-resident low-rank factors and the compression drivers.
#pragma once

#include <functional>
#include <memory>

#include "internal.h"

namespace hydot {

// V held implicitly as Q [Z; 0]: Q the (cols x zr) Householder QR of the
// last tall factorisation, Z zr x rank (ld zr).  The root of the recursion
// keeps its V this way so that recompress can factor the small Z instead of
// the tall V (one cols x r QR and one Q application fewer); any other use
// materialises V first (materialize_v).
struct LazyV {
    QRFact q;
    DBuf Z;
    int64_t zr = 0;
    bool set = false;
};

// lowrank::LowRankFactor (lowrank.hpp:25-36) with U, V in device memory.
struct Factor {
    int64_t rows = 0, cols = 0, rank = 0;
    DBuf U, V;  // rows x rank (ld rows), cols x rank (ld cols)
    double tol = 0.0;
    int method = HYDOT_METHOD_NONE;
    bool flagged = false;
    std::shared_ptr<LazyV> lazy;  // non-null: V is Q [Z; 0] (V itself empty)
    // non-null: V is being formed on the side stream; valid once `ev` has
    // completed; `hold` keeps the inputs of that work alive until then
    struct Pending {
        cudaEvent_t ev = nullptr;
        std::shared_ptr<LazyV> hold;
        bool waited = false;  // a stream waits on ev (wait_v)
        ~Pending() {
            // a factor dropped before any consumer waited: V (freed in
            // c.stream order) may still be written on the side stream
            if (ev && !waited) cudaEventSynchronize(ev);
            if (ev) cudaEventDestroy(ev);
        }
    };
    // declared last: destroyed (and, if never waited on, synchronised) before
    // the buffers above are released
    mutable std::shared_ptr<Pending> pending;
};
// V := Q [Z; 0] in place (no-op for a dense factor); waits for a pending V
void materialize_v(Ctx& c, Factor& f);
// start forming V on the side stream (returns at once; consumers call wait_v)
void materialize_v_async(Ctx& c, Factor& f);
// make V (dense or pending) usable on c.stream
void wait_v(Ctx& c, const Factor& f);

// thin SVD result: U m x k, s (host), V n x k
struct SVDd {
    int64_t m = 0, n = 0, k = 0;
    DBuf U, V;
    std::vector<double> s;
};

// fast_thin_svd (lowrank.cpp:62-93) of the logical matrix L (m x n):
// trans=false: L = S (column-major m x n, ld); trans=true: L = S^T with S
// stored n x m.
SVDd fast_thin_svd(Ctx& c, const double* S, int64_t ld, bool trans, int64_t m, int64_t n,
                   Ledger* l, int cat);
SVDd thin_svd(Ctx& c, const double* S, int64_t ld, bool trans, int64_t m, int64_t n, Ledger* l,
              int cat);

// randsvd (lowrank.cpp:131-199) on A (m x n) given row-major: A(i,j) =
// At[j + i*lda].
// lazy_v: the result may keep V as Q [Z; 0] (see LazyV)
Factor randsvd(Ctx& c, int64_t m, int64_t n, const double* At, int64_t lda, double eps, int p,
               int kprobe, uint64_t seed, Ledger* l, int cat, int r0, bool lazy_v = false);

// LinOp (lowrank.hpp:56-63) with device operands: mm forms Y (m x k, ld m)
// = A X from X (n x k, ld n), rmm forms X (n x k, ld n) = A^T Y; both
// column-major, enqueued on c.stream.
struct LinOpDev {
    int64_t rows = 0, cols = 0;
    std::function<void(int64_t k, const double* X, double* Y)> mm, rmm;
};
// randsvd on a matrix-free operator: the same branch structure, stream and
// ledger; the Q = I branch obtains A^T as rmm(I_m) like the reference's
// apply_mm(A, Q, true) with Q = I (lowrank.cpp:159-164, 184)
Factor randsvd(Ctx& c, const LinOpDev& A, double eps, int p, int kprobe, uint64_t seed, Ledger* l,
               int cat, int r0);

Factor agglomerate(Ctx& c, const Factor& f1, const Factor& f2, double eps, uint64_t seed,
                   Ledger* l, int rank_hint, int p, int kprobe, bool lazy_v = false);

Factor recompress(Ctx& c, const Factor& f, double eps, int rank, Ledger* l);

// ClusterTree (lowrank.hpp:103-119)
struct TreeNode {
    std::vector<int> idx;
    int left = -1, right = -1;
    std::vector<double> lo, hi;
    bool is_leaf() const { return left < 0; }
};
struct Tree {
    std::vector<TreeNode> nodes;
    int root = 0;
    int depth() const;
    std::vector<int> leaf_order() const;
};
Tree build_cluster_tree(const double* pos, int n, int d, const double* lo, const double* hi);
double tolerance_schedule(double eps_d, int L, int N_r);

struct RecOut {
    Factor factor;
    std::vector<int> source_order, row_perm, node_rank, node_depth;
    Ledger ledger;
};
// block(s, out, ld): fill rows_per x cols block of source s row-major
using BlockFn = std::function<void(int, double*, int64_t)>;
RecOut recursive_lowrank(Ctx& c, const Tree& t, double eps, int rows_per, int64_t cols,
                         const BlockFn& block, uint64_t seed, int p, int kprobe,
                         const std::vector<int>& source_ids = {}, int node_offset = 0,
                         bool lazy_root = false);

// fileio.cpp: the reference's factor / block file formats
void save_factor_file(Ctx& c, const std::string& path, const Factor& f, const int* perm, int64_t plen);
bool factor_file_info(const std::string& path, int64_t& rows, int64_t& cols, int64_t& rank, int64_t& plen);
Factor load_factor_file(Ctx& c, const std::string& path, std::vector<int>& perm);
void save_block_file(Ctx& c, const std::string& path, const double* block, int64_t rows, int64_t cols,
                     int64_t ld);
void block_file_info(const std::string& path, int64_t& rows, int64_t& cols);
// rows_cap: rows the caller's buffer holds (row stride ld); a larger file is
// rejected before any device write
void load_block_file(Ctx& c, const std::string& path, double* block, int64_t ld, int64_t rows_cap, int64_t& rows,
                     int64_t& cols);

}  // namespace hydot
