// ADI line-sweep consumer (poisson/adi.hpp): the
// Peaceman-Rachford half-step right-hand sides and the convergence norms.
//
// A half step along direction 1 solves, for every interior line j,
//   (T - (h1^2/tau) I) u+ = -h1^2 (u/tau + L2 u + f)      (adi.hpp:143-158)
// and along direction 2, for every interior line i,
//   (T - (h2^2/tau) I) u' = -h2^2 (u+/tau + L1 u+ + f)    (adi.hpp:160-175).
// The grid is the reference's Grid2D: (n1+1) x (n2+1) nodes, row-major with
// j contiguous, zero Dirichlet boundary. Direction-1 systems run along i, so
// their right-hand sides are written RHS-contiguous (layout R: row i - 1,
// RHS j - 1) and solved straight into the interior of the half-step grid;
// direction-2 systems run along j (layout S: system i - 1 contiguous). The
// stencil arithmetic is the reference's, operation for operation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "parsweep_b200.h"
#include "psw_internal.h"

namespace psw {
namespace {

// x / d for a divisor shared by the whole grid: q = x * (1/d) refined by one
// FMA residual step, the correctly rounded quotient except in rare ties (the
// reference divides, adi.hpp:148-150, 165-167; an IEEE division per node is
// what made this pass compute-bound)
__device__ __forceinline__ double div_by(double x, double d, double r) {
    const double q = x * r;
    return fma(fma(-q, d, x), r, q);
}

__global__ void adi_rhs_kernel(const double* __restrict__ u, int64_t ldu,
                               const double* __restrict__ f, int64_t ldf,
                               double* __restrict__ rhs, int64_t ldr, int64_t n1, int64_t n2,
                               double h1, double h2, double tau, double rt, double rh, int dir) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x + 1;
    const int64_t i = int64_t(blockIdx.y) + 1;
    if (j >= n2 || i >= n1) return;
    const int64_t ld = ldu;
    const int64_t c = i * ld + j;
    const double uc = u[c];
    double lam, hs;  // rt = 1 / tau, rh = 1 / h^2 of the direction (host, IEEE)
    if (dir == 1) {  // adi.hpp:148-150
        const double hh = __dmul_rn(h2, h2);
        lam = div_by(__dadd_rn(__dsub_rn(u[c + 1], __dmul_rn(2.0, uc)), u[c - 1]), hh, rh);
        hs = __dmul_rn(-h1, h1);
    } else {  // adi.hpp:165-167
        const double hh = __dmul_rn(h1, h1);
        lam = div_by(__dadd_rn(__dsub_rn(u[c + ld], __dmul_rn(2.0, uc)), u[c - ld]), hh, rh);
        hs = __dmul_rn(-h2, h2);
    }
    rhs[(i - 1) * ldr + (j - 1)] =
        __dmul_rn(hs, __dadd_rn(__dadd_rn(div_by(uc, tau, rt), lam), f[i * ldf + j]));
}

// out[0] = max |a - b|, out[1] = max |b| (non-negative doubles order like
// their bit patterns, so an integer atomicMax reduces them exactly)
__global__ void max_abs_diff_kernel(const double* __restrict__ a, int64_t lda,
                                    const double* __restrict__ b, int64_t ldb, int64_t rows,
                                    int64_t cols, unsigned long long* out) {
    double md = 0.0, mb = 0.0;
    const int64_t count = rows * cols;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
         k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = k / cols, c = k - r * cols;
        const double bv = b[r * ldb + c];
        md = fmax(md, fabs(a[r * lda + c] - bv));
        mb = fmax(mb, fabs(bv));
    }
    for (int o = 16; o > 0; o >>= 1) {
        md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
        mb = fmax(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(md)));
        atomicMax(out + 1, static_cast<unsigned long long>(__double_as_longlong(mb)));
    }
}

}  // namespace

int adi_rhs(int dir, const double* u, int64_t ldu, const double* f, int64_t ldf, double* rhs,
            int64_t ldr, int64_t n1, int64_t n2, double h1, double h2, double tau, cudaStream_t s) {
    if (n1 < 2 || n2 < 2) return PSW_OK;
    const dim3 grid(unsigned((n2 - 1 + 127) / 128), unsigned(n1 - 1));
    const double hh = dir == 1 ? h2 * h2 : h1 * h1;
    adi_rhs_kernel<<<grid, 128, 0, s>>>(u, ldu, f, ldf, rhs, ldr, n1, n2, h1, h2, tau, 1.0 / tau,
                                        1.0 / hh, dir);
    PSW_CUDA_TRY(cudaGetLastError());
    note_launches(1);
    return PSW_OK;
}

int grid_max_abs_diff(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t rows,
                      int64_t cols, double* out2, cudaStream_t s) {
    PSW_CUDA_TRY(cudaMemsetAsync(out2, 0, 2 * sizeof(double), s));
    const int64_t count = rows * cols;
    if (count <= 0) return PSW_OK;
    const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 8);
    max_abs_diff_kernel<<<unsigned(blocks), 256, 0, s>>>(
        a, lda, b, ldb, rows, cols, reinterpret_cast<unsigned long long*>(out2));
    PSW_CUDA_TRY(cudaGetLastError());
    note_launches(1);
    return PSW_OK;
}

}  // namespace psw

extern "C" {

int psw_adi_rhs(int dir, const double* u, int64_t ldu, const double* f, int64_t ldf, double* rhs,
                int64_t ldr, int64_t n1, int64_t n2, double h1, double h2, double tau,
                void* stream) {
    psw::clear_error();
    psw::reset_launches();
    if ((dir != 1 && dir != 2) || !u || !f || !rhs || ldr < n2 - 1 || ldu < n2 + 1 ||
        ldf < n2 + 1 || !(tau > 0.0)) {
        psw::set_error(PSW_INVALID_ARGUMENT, "psw_adi_rhs: invalid arguments");
        return PSW_INVALID_ARGUMENT;
    }
    return psw::adi_rhs(dir, u, ldu, f, ldf, rhs, ldr, n1, n2, h1, h2, tau,
                        static_cast<cudaStream_t>(stream));
}

int psw_grid_max_abs_diff(const double* a, int64_t lda, const double* b, int64_t ldb,
                          int64_t rows, int64_t cols, double* out2, void* stream) {
    psw::clear_error();
    psw::reset_launches();
    if (!a || !b || !out2 || rows < 0 || cols < 0 || lda < cols || ldb < cols) {
        psw::set_error(PSW_INVALID_ARGUMENT, "psw_grid_max_abs_diff: invalid arguments");
        return PSW_INVALID_ARGUMENT;
    }
    return psw::grid_max_abs_diff(a, lda, b, ldb, rows, cols, out2,
                                  static_cast<cudaStream_t>(stream));
}

}  // extern "C"
