// Multi-GPU row sharding (psw_shard_*): rank r of `world` owns the blocks
// [r*P/world, (r+1)*P/world) of one global partition (the paper's data
// decomposition with PEs = GPUs) and the rows of those
// blocks. The dichotomy combination is linear in the betas
// (combine_matrix), so every rank forms its share of ALL boundary values,
//   V_r = sum_{t in rank r} MR[:, t] right_t + ML[:, t] left_t,
// one all-reduce(sum) of p values per RHS gives V, and each rank finishes
// its own blocks. This is the only exchange of the solve; the reference
// only counts it (runtime/run.hpp:93-94).
#include "psw_internal.h"

namespace psw {

int build_shard_tables(psw_plan* pl, const std::vector<double>& cmat) {
    const int64_t Ploc = pl->P / pl->world;
    pl->blk0 = pl->rank * Ploc;
    pl->blk1 = pl->blk0 + Ploc;
    pl->row0 = pl->blk[2 * pl->blk0];
    pl->row1 = pl->blk[2 * (pl->blk1 - 1) + 1];
    pl->npartials = pl->p;
    if (!cmat.empty() && !pl->d_cmat) {
        PSW_CUDA_TRY(cudaMalloc(&pl->d_cmat, sizeof(double) * cmat.size()));
        PSW_CUDA_TRY(cudaMemcpy(pl->d_cmat, cmat.data(), sizeof(double) * cmat.size(),
                                cudaMemcpyHostToDevice));
        pl->info.device_bytes += int64_t(sizeof(double) * cmat.size());
    }
    return PSW_OK;
}

int build_plan(psw_plan** out, int64_t n, const double* sub, const double* diag,
               const double* sup, int64_t p, const int64_t* bnd, int dtype, int device,
               int rank, int world, std::vector<double>* cmat_host, bool shard, int strategy);

}  // namespace psw

namespace {
int check_shard(const psw_plan* plan, const void* X, int64_t ldx, int64_t nrhs,
                const void* partials) {
    if (!plan || nrhs < 0 || (nrhs > 0 && (!X || !partials)) || ldx < nrhs) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid shard solve arguments");
        return PSW_INVALID_ARGUMENT;
    }
    return PSW_OK;
}
}  // namespace

extern "C" {
int psw_shard_plan_create(psw_plan** out, int64_t n, const double* sub, const double* diag,
                          const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                          int device, int rank, int world) {
    return psw::build_plan(out, n, sub, diag, sup, p, boundaries, dtype, device, rank, world,
                           nullptr, true, PSW_GROW_AUTO);
}
int64_t psw_shard_partials_count(const psw_plan* plan) { return plan ? plan->p : -1; }
int64_t psw_shard_row_offset(const psw_plan* plan) { return plan ? plan->row0 : -1; }
int64_t psw_shard_rows(const psw_plan* plan) {
    if (!plan) return -1;
    return plan->row1 - plan->row0;
}
int psw_shard_forward(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                      int64_t nrhs, double* partials, void* stream) {
    psw::clear_error();
    psw::reset_launches();
    if (int rc = check_shard(plan, X, ldx, nrhs, partials)) return rc;
    if (!F || ldf < nrhs) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid right-hand-side buffer");
        return PSW_INVALID_ARGUMENT;
    }
    if (nrhs == 0) return PSW_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != plan->device) PSW_CUDA_TRY(cudaSetDevice(plan->device));
    const int rc = psw::shard_forward(plan, F, ldf, X, ldx, nrhs, partials,
                                      static_cast<cudaStream_t>(stream));
    if (prev != plan->device) cudaSetDevice(prev);
    return rc;
}
int psw_shard_backward(const psw_plan* plan, void* X, int64_t ldx, int64_t nrhs,
                       const double* partials, void* stream) {
    psw::clear_error();
    psw::reset_launches();
    if (int rc = check_shard(plan, X, ldx, nrhs, partials)) return rc;
    if (nrhs == 0) return PSW_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != plan->device) PSW_CUDA_TRY(cudaSetDevice(plan->device));
    const int rc = psw::shard_backward(plan, X, ldx, nrhs, partials,
                                       static_cast<cudaStream_t>(stream));
    if (prev != plan->device) cudaSetDevice(prev);
    return rc;
}
}
