// Multi-GPU row sharding (psw_shard_*). Placeholder: full implementation in
// progress; entry points exist so the ABI is complete.
#include "psw_internal.h"

namespace psw {
int build_shard_tables(psw_plan*) {
    set_error(PSW_NOT_SUPPORTED, "row sharding not available yet");
    return PSW_NOT_SUPPORTED;
}
int build_plan(psw_plan** out, int64_t n, const double* sub, const double* diag,
               const double* sup, int64_t p, const int64_t* bnd, int dtype, int device,
               int rank, int world);
}  // namespace psw

extern "C" {
int psw_shard_plan_create(psw_plan** out, int64_t n, const double* sub, const double* diag,
                          const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                          int device, int rank, int world) {
    return psw::build_plan(out, n, sub, diag, sup, p, boundaries, dtype, device, rank, world);
}
int64_t psw_shard_partials_count(const psw_plan* plan) { return plan ? plan->npartials : -1; }
int64_t psw_shard_row_offset(const psw_plan* plan) { return plan ? plan->row0 : -1; }
int64_t psw_shard_rows(const psw_plan* plan) { return plan ? plan->row1 - plan->row0 : -1; }
int psw_shard_forward(const psw_plan*, const void*, int64_t, void*, int64_t, int64_t, double*,
                      void*) {
    psw::set_error(PSW_NOT_SUPPORTED, "row sharding not available yet");
    return PSW_NOT_SUPPORTED;
}
int psw_shard_backward(const psw_plan*, void*, int64_t, int64_t, const double*, void*) {
    psw::set_error(PSW_NOT_SUPPORTED, "row sharding not available yet");
    return PSW_NOT_SUPPORTED;
}
}
