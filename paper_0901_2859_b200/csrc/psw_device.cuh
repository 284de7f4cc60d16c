// Device helpers shared by the STAGED and FUSED paths.
#pragma once

#include <cstdint>

#include "psw_internal.h"

namespace psw {

// Reference-rounded multiply-add (no contraction): s + a*b. Used for the
// betas and the dichotomy combination so their rounding is the reference's
// (betas.hpp:48,54 and boundary_solve.hpp:48-53 compiled without FP
// contraction).
__device__ __forceinline__ double madd_rn(double s, double a, double b) {
    return __dadd_rn(s, __dmul_rn(a, b));
}

// boundary_solve.hpp:42-55 (segment_particular). bl/br point at block 0 of
// this RHS; block t is at [t * stride].
__device__ __forceinline__ double seg_sum(const double* bl, const double* br, int64_t stride,
                                          const double* __restrict__ zr,
                                          const double* __restrict__ zl, int p, int kl, int kr,
                                          int e) {
    double s = 0.0;
    for (int t = kl + 1; t <= e; ++t) s = madd_rn(s, br[int64_t(t) * stride], zr[t * p + e]);
    for (int t = e + 1; t <= kr; ++t) s = madd_rn(s, bl[int64_t(t) * stride], zl[(t - 1) * p + e]);
    return s;
}

// One dichotomy item (segment_component, boundary_solve.hpp:61-88, with the
// 2x2 endpoint match): V[i * vstride] from the betas and the already-known
// V[kl], V[kr]. Items of one level are independent (boundary_solve.hpp:106).
// The (up to) three segment sums S(kl,kr,i), S(kl,kr,kl), S(kl,kr,kr) run in
// one pass over t = kl+1..kr with three independent accumulators; each one
// still adds its terms in ascending t exactly like segment_particular
// (:48-53), so the result is bitwise the serial evaluation.
__device__ __forceinline__ void combine_item(const CombineItem it, int p, const double* bl,
                                             const double* br, int64_t stride,
                                             const double* __restrict__ zr,
                                             const double* __restrict__ zl, double* V,
                                             int64_t vstride) {
    {
        const int i = it.i, kl = it.kl, kr = it.kr;
        const bool lk = kl >= 0, rk = kr < p;
        double vi = 0.0, sl = 0.0, sr = 0.0;
        for (int t = kl + 1; t <= kr; ++t) {
            const double bR = br[int64_t(t) * stride], bL = bl[int64_t(t) * stride];
            const bool right = t <= i;
            vi = madd_rn(vi, right ? bR : bL, right ? zr[t * p + i] : zl[(t - 1) * p + i]);
            if (lk) sl = madd_rn(sl, bL, zl[(t - 1) * p + kl]);  // e = kl < t
            if (rk) sr = madd_rn(sr, bR, zr[t * p + kr]);        // e = kr >= t
        }
        double v;
        if (lk && rk) {
            const double b1 = __dsub_rn(V[int64_t(kl) * vstride], sl);
            const double b2 = __dsub_rn(V[int64_t(kr) * vstride], sr);
            const double m12 = zl[kr * p + kl];
            const double m21 = zr[kl * p + kr];
            const double det = __dsub_rn(1.0, __dmul_rn(m12, m21));
            const double cl = __ddiv_rn(__dsub_rn(b1, __dmul_rn(m12, b2)), det);
            const double cr = __ddiv_rn(__dsub_rn(b2, __dmul_rn(m21, b1)), det);
            v = madd_rn(madd_rn(vi, cl, zr[kl * p + i]), cr, zl[kr * p + i]);
        } else if (rk) {
            const double cr = __dsub_rn(V[int64_t(kr) * vstride], sr);
            v = madd_rn(vi, cr, zl[kr * p + i]);
        } else if (lk) {
            const double cl = __dsub_rn(V[int64_t(kl) * vstride], sl);
            v = madd_rn(vi, cl, zr[kl * p + i]);
        } else {
            v = vi;
        }
        V[int64_t(i) * vstride] = v;
    }
}

// boundary_solve.hpp:96-121 for one RHS: every item in level order.
__device__ __forceinline__ void combine_rhs(const CombineItem* __restrict__ items, int p,
                                            const double* bl, const double* br, int64_t stride,
                                            const double* __restrict__ zr,
                                            const double* __restrict__ zl, double* V,
                                            int64_t vstride) {
    for (int w = 0; w < p; ++w) combine_item(items[w], p, bl, br, stride, zr, zl, V, vstride);
}

}  // namespace psw
