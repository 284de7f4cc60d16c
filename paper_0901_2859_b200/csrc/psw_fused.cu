// FUSED solve path (single read of F, on-chip forward intermediates).
// Placeholder until the cluster-resident kernel lands: reports unsupported,
// so AUTO routes every shape to the STAGED path.
#include "psw_internal.h"

namespace psw {

bool fused_supported(const psw_plan*, int, int64_t) { return false; }

int solve_fused(const psw_plan*, const void*, int64_t, void*, int64_t, int64_t, int, cudaStream_t,
                void**, int) {
    set_error(PSW_NOT_SUPPORTED, "fused path not available");
    return PSW_NOT_SUPPORTED;
}

}  // namespace psw
