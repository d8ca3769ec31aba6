// comm.cpp -- the multi-GPU handle of the C ABI: an NCCL
// communicator bound to one context (one process per GPU, NVLink /
// NVSwitch), plus the products whose only exchange is the R x (b n_c)
// all-reduce of V^T X under voxel-sharded V (lowrank.cpp:589-599,
// experiments.cpp:255-262).  NCCL is loaded at run time (libnccl.so.2), so
// the library itself has no link dependency on it; inside a PyTorch process
// the already-loaded NCCL of the same SONAME is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "internal.h"

namespace hydot {
namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
                 api.GetErrorString;
        if (!api.ok) api.why = "libnccl.so.2 lacks an expected symbol";
    });
    return api;
}

}  // namespace

struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define HYDOT_NCCL(call)                                                                         \
    do {                                                                                         \
        ncclResult_t r_ = (call);                                                                \
        if (r_ != ncclSuccess)                                                                   \
            throw ::hydot::NcclError(std::string(#call) + ": " + nccl().GetErrorString(r_));      \
    } while (0)

struct Comm {
    int world = 1, rank = 0, device = 0;
    ncclComm_t nc = nullptr;
    ~Comm() {
        if (nc && nccl().ok) nccl().CommDestroy(nc);
    }
    void allreduce_sum(Ctx& c, double* buf, int64_t n) {
        if (world == 1 || n == 0) return;
        HYDOT_NCCL(nccl().AllReduce(buf, buf, size_t(n), ncclDouble, ncclSum, nc, c.stream));
    }
};

}  // namespace hydot

using hydot::Comm;
using hydot::Ctx;
using hydot::DBuf;
using hydot::nccl;

struct hydot_comm_s {
    std::unique_ptr<Comm> c;
};

// from capi.cpp
hydot::Ctx& hydot_ctx_ref(hydot_ctx ctx);
hydot_status hydot_guard_status(const std::exception& e, hydot::Ctx* c);

namespace {
template <class F>
hydot_status comm_guard(Ctx* c, F&& fn) {
    try {
        if (c) HYDOT_CUDA(cudaSetDevice(c->device));
        fn();
        return HYDOT_OK;
    } catch (const hydot::NcclError& e) {
        if (c) c->err = e.what();
        return HYDOT_ENCCL;
    } catch (const std::exception& e) {
        return hydot_guard_status(e, c);
    }
}
}  // namespace

extern "C" {

hydot_status hydot_comm_unique_id(unsigned char id_out[HYDOT_COMM_ID_BYTES]) {
    return comm_guard(nullptr, [&] {
        if (!id_out) throw std::invalid_argument("comm: null id buffer");
        if (!nccl().ok) throw hydot::NcclError(nccl().why);
        static_assert(sizeof(ncclUniqueId) == HYDOT_COMM_ID_BYTES, "NCCL unique id size");
        ncclUniqueId id;
        HYDOT_NCCL(nccl().GetUniqueId(&id));
        std::memcpy(id_out, &id, sizeof id);
    });
}

hydot_status hydot_comm_create(hydot_ctx ctx, int world, int rank, const unsigned char id[HYDOT_COMM_ID_BYTES],
                               hydot_comm* out) {
    if (out) *out = nullptr;
    Ctx* cp = ctx ? &hydot_ctx_ref(ctx) : nullptr;
    return comm_guard(cp, [&] {
        if (!ctx || !out || !id || world < 1 || rank < 0 || rank >= world)
            throw std::invalid_argument("comm: bad arguments");
        auto c = std::make_unique<Comm>();
        c->world = world;
        c->rank = rank;
        c->device = cp->device;
        if (world > 1) {
            if (!nccl().ok) throw hydot::NcclError(nccl().why);
            ncclUniqueId uid;
            std::memcpy(&uid, id, sizeof uid);
            HYDOT_NCCL(nccl().CommInitRank(&c->nc, world, uid, rank));
        }
        *out = new hydot_comm_s{std::move(c)};
    });
}

hydot_status hydot_comm_destroy(hydot_comm comm) {
    delete comm;
    return HYDOT_OK;
}

hydot_status hydot_comm_info(hydot_comm comm, int* world, int* rank) {
    if (!comm) return HYDOT_EINVAL;
    if (world) *world = comm->c->world;
    if (rank) *rank = comm->c->rank;
    return HYDOT_OK;
}

hydot_status hydot_comm_allreduce(hydot_ctx ctx, hydot_comm comm, double* buf_dev, int64_t n) {
    Ctx* cp = ctx ? &hydot_ctx_ref(ctx) : nullptr;
    return comm_guard(cp, [&] {
        if (!ctx || !comm || (n > 0 && !buf_dev) || n < 0) throw std::invalid_argument("comm: bad arguments");
        comm->c->allreduce_sum(*cp, buf_dev, n);
        cp->sync();
    });
}

hydot_status hydot_j_matmat_voxel(hydot_ctx ctx, hydot_comm comm, int trans, int b, const double* U_dev,
                                  int64_t M, const double* Vloc_dev, int64_t Nloc, int64_t R,
                                  const int* row_perm_dev, const double* eps_c_dev, int n_lambda, int n_c,
                                  const double* X_dev, int64_t ldx, double* Y_dev, int64_t ldy) {
    Ctx* cp = ctx ? &hydot_ctx_ref(ctx) : nullptr;
    return comm_guard(cp, [&] {
        Ctx& c = *cp;
        if (!ctx || !comm || !row_perm_dev || !eps_c_dev || n_lambda < 1 || n_c < 1 || b < 0 || M < 0 || Nloc < 0 ||
            R < 0)
            throw std::invalid_argument("J matmat (voxel): bad arguments");
        if (b == 0) return;
        const int64_t q = int64_t(b) * n_c;
        if (!trans) {
            // Z = sum_g V_g^T X_g (R x b n_c): local product + all-reduce; Y = P E (U Z)
            if (ldx != Nloc * n_c || ldy < M) throw std::invalid_argument("J matvec (voxel): dimension mismatch");
            DBuf Z = hydot::dalloc(c, size_t(std::max<int64_t>(R * q, 1)));
            if (R > 0) {
                if (Nloc > 0)
                    hydot::dgemm(c, true, false, R, q, Nloc, 1.0, Vloc_dev, Nloc, X_dev, Nloc, 0.0, Z.d(), R);
                else
                    hydot::fill(c, R, q, 0.0, Z.d(), R);
                comm->c->allreduce_sum(c, Z.d(), R * q);
            }
            DBuf T = hydot::dalloc(c, size_t(std::max<int64_t>(M * q, 1)));
            if (R > 0)
                hydot::dgemm(c, false, false, M, q, R, 1.0, U_dev, M, Z.d(), R, 0.0, T.d(), M);
            else
                hydot::fill(c, M, q, 0.0, T.d(), M);
            hydot::j_combine(c, M, b, n_c, n_lambda, T.d(), M, row_perm_dev, eps_c_dev, Y_dev, ldy);
        } else {
            // the rank's voxel rows of J~^T Y = V_loc (U^T G): no communication
            if (ldx < M || ldy != Nloc * n_c) throw std::invalid_argument("J rmatvec (voxel): dimension mismatch");
            DBuf G = hydot::dalloc(c, size_t(std::max<int64_t>(M * q, 1)));
            DBuf W = hydot::dalloc(c, size_t(std::max<int64_t>(R * q, 1)));
            hydot::j_gather_scale(c, M, b, n_c, n_lambda, X_dev, ldx, row_perm_dev, eps_c_dev, G.d(), M);
            if (R > 0 && Nloc > 0) {
                hydot::dgemm(c, true, false, R, q, M, 1.0, U_dev, M, G.d(), M, 0.0, W.d(), R);
                hydot::dgemm(c, false, false, Nloc, q, R, 1.0, Vloc_dev, Nloc, W.d(), R, 0.0, Y_dev, Nloc);
            } else if (Nloc > 0) {
                hydot::fill(c, Nloc, q, 0.0, Y_dev, Nloc);
            }
        }
        c.sync();
    });
}

}  // extern "C"
