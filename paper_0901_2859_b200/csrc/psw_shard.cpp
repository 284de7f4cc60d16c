// Multi-GPU row sharding (psw_shard_*): rank r of `world` owns the blocks
// [r*P/world, (r+1)*P/world) of one global partition (the paper's data
// decomposition with PEs = GPUs) and the rows of those
// blocks. The dichotomy combination is linear in the betas
// (combine_matrix), so every rank forms its share of ALL boundary values,
//   V_r = sum_{t in rank r} MR[:, t] right_t + ML[:, t] left_t,
// one all-reduce(sum) of p values per RHS gives V, and each rank finishes
// its own blocks. This is the only exchange of the solve; the reference
// only counts it (runtime/run.hpp:93-94). The device work is the RESWEEP
// kernels over the rank's own segments (psw_resweep.cu).
//
// NCCL is loaded at run time (dlopen libnccl.so.2): the library stays
// loadable on hosts without NCCL, and a process that already mapped NCCL
// (torch does) shares that copy.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "psw_internal.h"

struct psw_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
};

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // PSW_NCCL_LIB: another NCCL build, or the tests' host-staged stand-in
        // (tests/cpp/fake_nccl.cpp) that lets several ranks share one GPU
        const char* lib = std::getenv("PSW_NCCL_LIB");
        if (!lib || !*lib) lib = "libnccl.so.2";
        void* h = dlopen(lib, RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string(lib) + " not loadable: " + dlerror();
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce &&
                 api.GetErrorString;
        if (!api.ok) api.why = std::string(lib) + " lacks the expected symbols";
    });
    return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
    const NcclApi& api = nccl();
    psw::set_error(PSW_NCCL_ERROR, std::string(what) + ": " +
                                       (api.GetErrorString ? api.GetErrorString(r) : "nccl error"));
    return PSW_NCCL_ERROR;
}

int need_nccl() {
    const NcclApi& api = nccl();
    if (api.ok) return PSW_OK;
    psw::set_error(PSW_NCCL_ERROR, api.why);
    return PSW_NCCL_ERROR;
}

int check_shard(const psw_plan* plan, const void* F, int64_t ldf, int64_t nrhs) {
    if (!plan || nrhs < 0 || (nrhs > 0 && !F) || ldf < nrhs) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid shard solve arguments");
        return PSW_INVALID_ARGUMENT;
    }
    if (!plan->d_rs_group) {
        psw::set_error(PSW_NOT_SUPPORTED, "plan has no shard tables");
        return PSW_NOT_SUPPORTED;
    }
    return PSW_OK;
}

// runs `body` on the plan's device and restores the caller's device
template <typename Fn>
int on_device(int dev, Fn&& body) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != dev) {
        const cudaError_t e = cudaSetDevice(dev);
        if (e != cudaSuccess) return psw::cuda_fail(e, "cudaSetDevice");
    }
    const int rc = body();
    if (prev != dev) cudaSetDevice(prev);
    return rc;
}

}  // namespace

namespace psw {
int build_plan(psw_plan** out, int64_t n, const double* sub, const double* diag,
               const double* sup, int64_t p, const int64_t* bnd, int dtype, int device,
               int rank, int world, std::vector<double>* cmat_host, bool shard, int strategy,
               int flags);
}  // namespace psw

extern "C" {
int psw_shard_plan_create(psw_plan** out, int64_t n, const double* sub, const double* diag,
                          const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                          int device, int rank, int world) {
    return psw::build_plan(out, n, sub, diag, sup, p, boundaries, dtype, device, rank, world,
                           nullptr, true, PSW_GROW_AUTO, 0);
}
int64_t psw_shard_partials_count(const psw_plan* plan) { return plan ? plan->p : -1; }
int64_t psw_shard_row_offset(const psw_plan* plan) { return plan ? plan->row0 : -1; }
int64_t psw_shard_rows(const psw_plan* plan) { return plan ? plan->row1 - plan->row0 : -1; }
int64_t psw_shard_workspace_bytes(const psw_plan* plan, int64_t nrhs) {
    if (!plan || nrhs < 0) return -1;
    return psw::shard_workspace_bytes(plan, nrhs);
}

int psw_shard_forward(const psw_plan* plan, const void* F, int64_t ldf, int64_t nrhs,
                      void* workspace, double* partials, void* stream) {
    psw::clear_error();
    psw::reset_launches();
    if (int rc = check_shard(plan, F, ldf, nrhs)) return rc;
    if (nrhs > 0 && (!workspace || (plan->p > 0 && !partials))) {
        psw::set_error(PSW_INVALID_ARGUMENT, "null workspace or partials");
        return PSW_INVALID_ARGUMENT;
    }
    if (nrhs == 0) return PSW_OK;
    return on_device(plan->device, [&] {
        return psw::shard_forward(plan, F, ldf, nrhs, workspace, partials, nrhs,
                                  static_cast<cudaStream_t>(stream));
    });
}

int psw_shard_backward(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                       int64_t nrhs, void* workspace, const double* partials, void* stream) {
    psw::clear_error();
    psw::reset_launches();
    if (int rc = check_shard(plan, F, ldf, nrhs)) return rc;
    if (nrhs > 0 && (!X || ldx < nrhs || !workspace || (plan->p > 0 && !partials))) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid solution, workspace or partials buffer");
        return PSW_INVALID_ARGUMENT;
    }
    if (nrhs == 0) return PSW_OK;
    return on_device(plan->device, [&] {
        return psw::shard_backward(plan, F, ldf, X, ldx, nrhs, workspace, partials, nrhs,
                                   static_cast<cudaStream_t>(stream));
    });
}

int psw_comm_unique_id(void* id_out) {
    psw::clear_error();
    if (!id_out) {
        psw::set_error(PSW_INVALID_ARGUMENT, "null id buffer");
        return PSW_INVALID_ARGUMENT;
    }
    if (int rc = need_nccl()) return rc;
    ncclUniqueId id;
    if (ncclResult_t r = nccl().GetUniqueId(&id)) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id_out, &id, sizeof(id));
    return PSW_OK;
}

int psw_comm_create(psw_comm** out, int nranks, int rank, const void* id, int device) {
    psw::clear_error();
    if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid communicator arguments");
        return PSW_INVALID_ARGUMENT;
    }
    *out = nullptr;
    if (int rc = need_nccl()) return rc;
    auto* c = new psw_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    const int rc = on_device(device, [&] {
        if (ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, uid, rank))
            return nccl_fail(r, "ncclCommInitRank");
        return int(PSW_OK);
    });
    if (rc != PSW_OK) {
        delete c;
        return rc;
    }
    *out = c;
    return PSW_OK;
}

int psw_comm_destroy(psw_comm* comm) {
    psw::clear_error();
    if (!comm) return PSW_OK;
    int rc = PSW_OK;
    if (comm->comm && nccl().ok)
        if (ncclResult_t r = nccl().CommDestroy(comm->comm)) rc = nccl_fail(r, "ncclCommDestroy");
    delete comm;
    return rc;
}

int psw_shard_solve(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                    int64_t nrhs, psw_comm* comm, void* stream) {
    psw::clear_error();
    psw::reset_launches();
    if (int rc = check_shard(plan, F, ldf, nrhs)) return rc;
    if (nrhs > 0 && (!X || ldx < nrhs)) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid solution buffer");
        return PSW_INVALID_ARGUMENT;
    }
    if ((plan->world > 1 && !comm) ||
        (comm && (comm->nranks != plan->world || comm->rank != plan->rank ||
                  comm->device != plan->device))) {
        psw::set_error(PSW_INVALID_ARGUMENT,
                       "communicator does not match the plan's rank, world and device");
        return PSW_INVALID_ARGUMENT;
    }
    if (nrhs == 0) return PSW_OK;
    auto s = static_cast<cudaStream_t>(stream);
    return on_device(plan->device, [&]() -> int {
        const int64_t p = plan->p;
        const size_t ws = (size_t(psw::shard_workspace_bytes(plan, nrhs)) + 255) & ~size_t(255);
        // boundary values at a pitch of whole 64-RHS chunks (the TMA solve
        // kernel copies them chunk by chunk); the padding rides along in the sum
        const int64_t ldv = (nrhs + 63) / 64 * 64;
        const size_t vb = sizeof(double) * size_t(p > 0 ? p : 1) * size_t(ldv);
        void* mem = nullptr;
        PSW_CUDA_TRY(psw::scratch_alloc(&mem, ws + vb, plan->device, s));
        double* V = reinterpret_cast<double*>(static_cast<char*>(mem) + ws);
        int rc = psw::shard_forward(plan, F, ldf, nrhs, mem, V, ldv, s);
        // the exchange (a 1-rank communicator still runs NCCL's in-place sum)
        if (rc == PSW_OK && p > 0 && comm) {
            if (ncclResult_t r = nccl().AllReduce(V, V, size_t(p) * size_t(ldv), ncclFloat64,
                                                  ncclSum, comm->comm, s))
                rc = nccl_fail(r, "ncclAllReduce");
        }
        if (rc == PSW_OK) rc = psw::shard_backward(plan, F, ldf, X, ldx, nrhs, mem, V, ldv, s);
        psw::scratch_free(mem, s);
        return rc;
    });
}
}  // extern "C"
