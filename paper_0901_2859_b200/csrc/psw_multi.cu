// Multi-matrix batched solve (psw_solve_multi): right-hand side k (column k
// of a layout-R series) is solved with its own plan, plans[k]. This is the
// per-harmonic loop of the reference Fourier solver (poisson/fourier.hpp:
// 157-164 over FourierWorkspace::solve_harmonic, :75-86: one matrix
// B_l = tri(1, -(2 + d_l), 1) and one right-hand side per harmonic) as one
// three-kernel pass over all harmonics instead of one solve per harmonic.
//
// The kernels are the STAGED path's (psw_staged.cu) with per-RHS plan
// tables: one thread per (rhs k, block t) for the forward sweep with both
// beta dot products and the backward sweep, one thread per rhs for the
// level-order dichotomy with that rhs' Z samples. Every right-hand side
// therefore gets bitwise the betas, boundary values and solution of a
// single-plan STAGED solve, i.e. the reference's betas and boundary values.
// All plans share the partition (the workspace's, fourier.hpp:47-51).
#include <algorithm>
#include <string>
#include <vector>

#include "psw_device.cuh"
#include "psw_internal.h"

namespace psw {
namespace {

constexpr int kThreads = 128;

template <typename T>
__global__ void __launch_bounds__(kThreads) multi_fwd_kernel(
    const T* F, int64_t ldf, T* X, int64_t ldx, int64_t N, const int32_t* __restrict__ blk,
    const FwdCoef<T>* const* __restrict__ cfs, double* __restrict__ bl_out,
    double* __restrict__ br_out, int p) {
    const int t = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (k >= N) return;
    const FwdCoef<T>* cf = cfs[k];
    const int s = blk[2 * t], e = blk[2 * t + 1];
    T d = T(0);
    double br = 0.0, bl = 0.0;
    for (int q = s; q < e; ++q) {
        const FwdCoef<T> c = cf[q];
        const T fv = F[int64_t(q) * ldf + k];
        d = fma(c.ma, d, fv * c.rp);
        br = madd_rn(br, double(fv), double(c.gr));
        bl = madd_rn(bl, double(fv), double(c.gl));
        X[int64_t(q) * ldx + k] = d;
    }
    if (t < p) br_out[int64_t(t) * N + k] = br;
    if (t > 0) bl_out[int64_t(t) * N + k] = bl;
}

__global__ void __launch_bounds__(kThreads) multi_combine_kernel(
    const double* __restrict__ bl, const double* __restrict__ br, int64_t N, int p,
    const CombineItem* __restrict__ items, const double* const* __restrict__ zrs,
    const double* const* __restrict__ zls, double* __restrict__ V) {
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (k >= N) return;
    combine_rhs(items, p, bl + k, br + k, N, zrs[k], zls[k], V + k, N);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) multi_bwd_kernel(
    T* X, int64_t ldx, int64_t N, const int32_t* __restrict__ blk,
    const BwdCoef<T>* const* __restrict__ cbs, const double* __restrict__ V, int p) {
    const int t = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (k >= N) return;
    const BwdCoef<T>* cb = cbs[k];
    const int s = blk[2 * t], e = blk[2 * t + 1];
    const T xl = t > 0 ? T(V[int64_t(t - 1) * N + k]) : T(0);
    T xn = t < p ? T(V[int64_t(t) * N + k]) : T(0);
    for (int q = e - 1; q >= s; --q) {
        const BwdCoef<T> c = cb[q];
        xn = fma(c.al, xn, fma(xl, c.w, X[int64_t(q) * ldx + k]));
        X[int64_t(q) * ldx + k] = xn;
    }
}

template <typename T>
int launch_multi(const psw_plan* const* plans, int64_t N, const void* Fv, int64_t ldf, void* Xv,
                 int64_t ldx, cudaStream_t s) {
    const psw_plan* p0 = plans[0];
    const int P = int(p0->P), p = int(p0->p);
    // per-RHS table pointers (device), then betas and boundary values
    std::vector<const void*> tab(size_t(4) * N);
    for (int64_t k = 0; k < N; ++k) {
        tab[k] = plans[k]->d_fwd;
        tab[N + k] = plans[k]->d_bwd;
        tab[2 * N + k] = plans[k]->d_zr;
        tab[3 * N + k] = plans[k]->d_zl;
    }
    const size_t tab_b = sizeof(void*) * tab.size();
    const size_t need = tab_b + sizeof(double) * size_t(N) * (2 * size_t(P) + size_t(p > 0 ? p : 1));
    void* scratch = nullptr;
    PSW_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&scratch), need, p0->device, s));
    PSW_CUDA_TRY(cudaMemcpyAsync(scratch, tab.data(), tab_b, cudaMemcpyHostToDevice, s));
    PSW_CUDA_TRY(cudaStreamSynchronize(s));  // the host table goes out of scope
    auto** dtab = static_cast<const void**>(scratch);
    double* bl = reinterpret_cast<double*>(static_cast<char*>(scratch) + tab_b);
    double* br = bl + size_t(P) * N;
    double* V = br + size_t(P) * N;
    const dim3 grid(unsigned((N + kThreads - 1) / kThreads), unsigned(P));
    multi_fwd_kernel<T><<<grid, kThreads, 0, s>>>(
        static_cast<const T*>(Fv), ldf, static_cast<T*>(Xv), ldx, N, p0->d_blk,
        reinterpret_cast<const FwdCoef<T>* const*>(dtab), bl, br, p);
    int64_t launches = 1;
    if (p > 0) {
        multi_combine_kernel<<<grid.x, kThreads, 0, s>>>(
            bl, br, N, p, p0->d_items, reinterpret_cast<const double* const*>(dtab + 2 * N),
            reinterpret_cast<const double* const*>(dtab + 3 * N), V);
        ++launches;
    }
    multi_bwd_kernel<T><<<grid, kThreads, 0, s>>>(
        static_cast<T*>(Xv), ldx, N, p0->d_blk, reinterpret_cast<const BwdCoef<T>* const*>(dtab + N),
        V, p);
    ++launches;
    cudaError_t e = cudaGetLastError();
    scratch_free(scratch, s);
    if (e != cudaSuccess) return cuda_fail(e, "multi-plan kernels");
    note_launches(launches);
    return PSW_OK;
}

}  // namespace
}  // namespace psw

// ---------------------------------------------------------------- bundles
// psw_multi_create gathers the plans' per-row sweep tables once into
// interleaved arrays ([row][rhs]: a warp's 32 right-hand sides read one
// contiguous 1 KB / 512 B piece per row) and keeps the Z-sample pointer
// table on the device; psw_multi_solve then runs the same three kernels with
// coalesced coefficient loads, rows in register batches, no host sync.
namespace psw {
namespace {

constexpr int kMB = 16;  // rows per register batch

template <typename T>
__global__ void multi_gather_kernel(const FwdCoef<T>* const* __restrict__ cfs,
                                    const BwdCoef<T>* const* __restrict__ cbs, int64_t n, int64_t N,
                                    FwdCoef<T>* __restrict__ fo, BwdCoef<T>* __restrict__ bo) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= N) return;
    for (int64_t q = blockIdx.y; q < n; q += gridDim.y) {
        fo[q * N + k] = cfs[k][q];
        bo[q * N + k] = cbs[k][q];
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) bundle_fwd_kernel(
    const T* __restrict__ F, int64_t ldf, T* __restrict__ X, int64_t ldx, int64_t N,
    const int32_t* __restrict__ blk, const FwdCoef<T>* __restrict__ cf, double* __restrict__ bl_out,
    double* __restrict__ br_out, int p) {
    const int t = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (k >= N) return;
    const int s = blk[2 * t], e = blk[2 * t + 1];
    T d = T(0);
    double br = 0.0, bl = 0.0;
    for (int q0 = s; q0 < e; q0 += kMB) {
        T fv[kMB];
        FwdCoef<T> c[kMB];
#pragma unroll
        for (int u = 0; u < kMB; ++u)
            if (q0 + u < e) {
                fv[u] = F[int64_t(q0 + u) * ldf + k];
                c[u] = cf[int64_t(q0 + u) * N + k];
            }
#pragma unroll
        for (int u = 0; u < kMB; ++u)
            if (q0 + u < e) {
                d = fma(c[u].ma, d, fv[u] * c[u].rp);
                br = madd_rn(br, double(fv[u]), double(c[u].gr));
                bl = madd_rn(bl, double(fv[u]), double(c[u].gl));
                X[int64_t(q0 + u) * ldx + k] = d;
            }
    }
    if (t < p) br_out[int64_t(t) * N + k] = br;
    if (t > 0) bl_out[int64_t(t) * N + k] = bl;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) bundle_bwd_kernel(
    T* __restrict__ X, int64_t ldx, int64_t N, const int32_t* __restrict__ blk,
    const BwdCoef<T>* __restrict__ cb, const double* __restrict__ V, int p) {
    const int t = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (k >= N) return;
    const int s = blk[2 * t], e = blk[2 * t + 1];
    const T xl = t > 0 ? T(V[int64_t(t - 1) * N + k]) : T(0);
    T xn = t < p ? T(V[int64_t(t) * N + k]) : T(0);
    for (int q1 = e - 1; q1 >= s; q1 -= kMB) {
        T dv[kMB];
        BwdCoef<T> c[kMB];
#pragma unroll
        for (int u = 0; u < kMB; ++u)
            if (q1 - u >= s) {
                dv[u] = X[int64_t(q1 - u) * ldx + k];
                c[u] = cb[int64_t(q1 - u) * N + k];
            }
#pragma unroll
        for (int u = 0; u < kMB; ++u)
            if (q1 - u >= s) {
                xn = fma(c[u].al, xn, fma(xl, c[u].w, dv[u]));
                X[int64_t(q1 - u) * ldx + k] = xn;
            }
    }
}

}  // namespace
}  // namespace psw

struct psw_multi {
    int64_t n = 0, N = 0, P = 1, p = 0;
    int dtype = PSW_F64, device = 0;
    const psw_plan* p0 = nullptr;  // partition, level items (shared by every plan)
    psw_plan* own_p0 = nullptr;    // psw_multi_create_systems: the bundle's own copy of p0
    void* fwd = nullptr;           // FwdCoef<T>[n][N]
    void* bwd = nullptr;           // BwdCoef<T>[n][N]
    void* zptr = nullptr;          // const double*[2][N]: every plan's ZR, ZL samples
    double* zall = nullptr;        // psw_multi_create_systems: [2][N][p p + 2] samples
};

namespace psw {
int build_plan(psw_plan** out, int64_t n, const double* sub, const double* diag, const double* sup,
               int64_t p, const int64_t* bnd, int dtype, int device, int rank, int world,
               std::vector<double>* cmat_host, bool shard, int strategy, int flags);
void destroy_plan(psw_plan* pl);
size_t device_setup_batch_bytes(int64_t n, int64_t N, int64_t p);
int device_setup_batch(int64_t n, int64_t N, const double* sub, const double* diag,
                       const double* sup, int64_t p, const int64_t* bnd,
                       const std::vector<int32_t>& blk, int dtype, void* fwd, void* bwd, double* zr,
                       double* zl, int64_t& bad_sys, int64_t& bad_row);
}  // namespace psw

// The bundle of nsys symmetric systems sharing one partition, built directly
// on the device (psw_prelim.cu device_setup_batch: preliminary sweeps and
// block sweep coefficients of all systems in [row][system] layout) instead of
// one plan per system gathered afterwards: the once-per-mesh phase of the
// Fourier consumer (fourier.hpp:41-105). sub / diag / sup are host arrays
// [nsys][n-1] / [nsys][n] / [nsys][n-1] with sub == sup (the DirectSymmetric
// route, preliminary.hpp:111-112; anything else answers PSW_NOT_SUPPORTED and
// the caller creates plans one by one). The tables are bitwise those of
// psw_multi_create over per-system plans.
extern "C" int psw_multi_create_systems(psw_multi** out, int64_t n, int64_t nsys, const double* sub,
                                        const double* diag, const double* sup, int64_t p,
                                        const int64_t* boundaries, int dtype, int device) {
    psw::clear_error();
    if (!out || n < 2 || nsys <= 0 || !sub || !diag || !sup || p < 0 || (p > 0 && !boundaries) ||
        (dtype != PSW_F64 && dtype != PSW_F32)) {
        psw::set_error(PSW_INVALID_ARGUMENT, "psw_multi_create_systems: invalid arguments");
        return PSW_INVALID_ARGUMENT;
    }
    *out = nullptr;
    if (int rc = psw_partition_validate(n, p, boundaries)) return rc;
    for (int64_t k = 0; k < nsys; ++k)
        for (int64_t i = 0; i + 1 < n; ++i)
            if (!(sub[k * (n - 1) + i] == sup[k * (n - 1) + i])) {
                psw::set_error(PSW_NOT_SUPPORTED,
                               "psw_multi_create_systems takes symmetric systems (sub == super) only");
                return PSW_NOT_SUPPORTED;
            }
    const size_t scratch = psw::device_setup_batch_bytes(n, nsys, p);
    if (scratch > (size_t(32) << 30)) {
        psw::set_error(PSW_NOT_SUPPORTED, "psw_multi_create_systems: batch too large for one pass");
        return PSW_NOT_SUPPORTED;
    }
    // system 0 as an ordinary (lean) plan: validation of the matrix layout,
    // the partition's block table and the level-ordered combination items
    psw_plan* p0 = nullptr;
    if (int rc = psw::build_plan(&p0, n, sub, diag, sup, p, boundaries, dtype, device, 0, 1, nullptr,
                                 false, PSW_GROW_DIRECT_SYMMETRIC, PSW_PLAN_STAGED_ONLY))
        return rc;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    auto* m = new psw_multi();
    m->n = n;
    m->N = nsys;
    m->P = p + 1;
    m->p = p;
    m->dtype = dtype;
    m->device = device;
    m->p0 = m->own_p0 = p0;
    const size_t es = dtype == PSW_F64 ? 8 : 4;
    const size_t fb = 4 * es * size_t(n) * size_t(nsys), bb = 16 * size_t(n) * size_t(nsys);
    const size_t zs = size_t(p) * size_t(p) + 2;
    cudaError_t e = cudaMalloc(&m->fwd, fb);
    if (e == cudaSuccess) e = cudaMalloc(&m->bwd, bb);
    if (e == cudaSuccess) e = cudaMalloc(&m->zptr, sizeof(void*) * 2 * size_t(nsys));
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&m->zall), 8 * 2 * zs * size_t(nsys));
    int rc = PSW_OK;
    int64_t bad_sys = -1, bad_row = -1;
    if (e == cudaSuccess) {
        std::vector<const double*> zp(2 * size_t(nsys));
        for (int64_t k = 0; k < nsys; ++k) {
            zp[size_t(k)] = m->zall + size_t(k) * zs;
            zp[size_t(nsys + k)] = m->zall + (size_t(nsys) + size_t(k)) * zs;
        }
        e = cudaMemcpy(m->zptr, zp.data(), sizeof(void*) * zp.size(), cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            rc = psw::device_setup_batch(n, nsys, sub, diag, sup, p, boundaries, p0->blk, dtype,
                                         m->fwd, m->bwd, m->zall, m->zall + size_t(nsys) * zs,
                                         bad_sys, bad_row);
    }
    cudaSetDevice(prev);
    if (e != cudaSuccess) rc = psw::cuda_fail(e, "psw_multi_create_systems");
    if (rc == PSW_PIVOT_BREAKDOWN)
        psw::set_error(PSW_PIVOT_BREAKDOWN,
                       "pivot breakdown during forward elimination at row " +
                           std::to_string(bad_row) + " (system " + std::to_string(bad_sys) + ")",
                       bad_row);
    if (rc != PSW_OK) {
        psw_multi_destroy(m);
        return rc;
    }
    *out = m;
    return PSW_OK;
}

extern "C" int psw_multi_create(psw_multi** out, const psw_plan* const* plans, int64_t nplans) {
    psw::clear_error();
    if (!out || nplans <= 0 || !plans) {
        psw::set_error(PSW_INVALID_ARGUMENT, "psw_multi_create: invalid arguments");
        return PSW_INVALID_ARGUMENT;
    }
    *out = nullptr;
    const psw_plan* p0 = plans[0];
    for (int64_t k = 0; k < nplans; ++k) {
        const psw_plan* q = plans[k];
        if (!q || q->world != 1 || q->n != p0->n || q->P != p0->P || q->dtype != p0->dtype ||
            q->device != p0->device || q->bnd != p0->bnd) {
            psw::set_error(PSW_INVALID_ARGUMENT,
                           "psw_multi_create: plans must share order, partition, dtype and device");
            return PSW_INVALID_ARGUMENT;
        }
    }
    int prev = 0;
    cudaGetDevice(&prev);
    PSW_CUDA_TRY(cudaSetDevice(p0->device));
    auto* m = new psw_multi();
    m->n = p0->n;
    m->N = nplans;
    m->P = p0->P;
    m->p = p0->p;
    m->dtype = p0->dtype;
    m->device = p0->device;
    m->p0 = p0;
    const size_t es = p0->dtype == PSW_F64 ? 8 : 4;
    const size_t fb = sizeof(double) * 4 * size_t(m->n) * size_t(nplans) / (8 / es);
    const size_t bb = 16 * size_t(m->n) * size_t(nplans);
    std::vector<const void*> tab(size_t(4) * nplans);
    for (int64_t k = 0; k < nplans; ++k) {
        tab[size_t(k)] = plans[k]->d_fwd;
        tab[size_t(nplans + k)] = plans[k]->d_bwd;
        tab[size_t(2 * nplans + k)] = plans[k]->d_zr;
        tab[size_t(3 * nplans + k)] = plans[k]->d_zl;
    }
    void* dtab = nullptr;
    cudaError_t e = cudaMalloc(&m->fwd, fb);
    if (e == cudaSuccess) e = cudaMalloc(&m->bwd, bb);
    if (e == cudaSuccess) e = cudaMalloc(&m->zptr, sizeof(void*) * 2 * size_t(nplans));
    if (e == cudaSuccess) e = cudaMalloc(&dtab, sizeof(void*) * tab.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(dtab, tab.data(), sizeof(void*) * tab.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(m->zptr, tab.data() + 2 * nplans, sizeof(void*) * 2 * size_t(nplans),
                       cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        const dim3 grid(unsigned((nplans + 127) / 128), unsigned(std::min<int64_t>(m->n, 4096)));
        auto** dt = static_cast<const void**>(dtab);
        if (p0->dtype == PSW_F64)
            psw::multi_gather_kernel<double><<<grid, 128>>>(
                reinterpret_cast<const psw::FwdCoef<double>* const*>(dt),
                reinterpret_cast<const psw::BwdCoef<double>* const*>(dt + nplans), m->n, nplans,
                static_cast<psw::FwdCoef<double>*>(m->fwd), static_cast<psw::BwdCoef<double>*>(m->bwd));
        else
            psw::multi_gather_kernel<float><<<grid, 128>>>(
                reinterpret_cast<const psw::FwdCoef<float>* const*>(dt),
                reinterpret_cast<const psw::BwdCoef<float>* const*>(dt + nplans), m->n, nplans,
                static_cast<psw::FwdCoef<float>*>(m->fwd), static_cast<psw::BwdCoef<float>*>(m->bwd));
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    if (dtab) cudaFree(dtab);
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        psw_multi_destroy(m);
        return psw::cuda_fail(e, "psw_multi_create");
    }
    *out = m;
    return PSW_OK;
}

extern "C" void psw_multi_destroy(psw_multi* m) {
    if (!m) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    for (void* q : {m->fwd, m->bwd, m->zptr, static_cast<void*>(m->zall)})
        if (q) cudaFree(q);
    cudaSetDevice(prev);
    if (m->own_p0) psw::destroy_plan(m->own_p0);
    delete m;
}

namespace psw {
namespace {
template <typename T>
int bundle_solve(const psw_multi* m, const void* Fv, int64_t ldf, void* Xv, int64_t ldx,
                 cudaStream_t s) {
    const int64_t N = m->N;
    const int P = int(m->P), p = int(m->p);
    void* scratch = nullptr;
    const size_t need = sizeof(double) * size_t(N) * (2 * size_t(P) + size_t(p > 0 ? p : 1));
    PSW_CUDA_TRY(scratch_alloc(&scratch, need, m->device, s));
    double* bl = static_cast<double*>(scratch);
    double* br = bl + size_t(P) * N;
    double* V = br + size_t(P) * N;
    const dim3 grid(unsigned((N + kThreads - 1) / kThreads), unsigned(P));
    bundle_fwd_kernel<T><<<grid, kThreads, 0, s>>>(static_cast<const T*>(Fv), ldf,
                                                   static_cast<T*>(Xv), ldx, N, m->p0->d_blk,
                                                   static_cast<const FwdCoef<T>*>(m->fwd), bl, br, p);
    int64_t launches = 1;
    if (p > 0) {
        const double* const* zp = static_cast<const double* const*>(m->zptr);
        multi_combine_kernel<<<grid.x, kThreads, 0, s>>>(bl, br, N, p, m->p0->d_items, zp, zp + N, V);
        ++launches;
    }
    bundle_bwd_kernel<T><<<grid, kThreads, 0, s>>>(static_cast<T*>(Xv), ldx, N, m->p0->d_blk,
                                                   static_cast<const BwdCoef<T>*>(m->bwd), V, p);
    ++launches;
    cudaError_t e = cudaGetLastError();
    scratch_free(scratch, s);
    if (e != cudaSuccess) return cuda_fail(e, "multi-plan bundle kernels");
    note_launches(launches);
    return PSW_OK;
}
}  // namespace
}  // namespace psw

extern "C" int psw_multi_solve(const psw_multi* m, const void* F, int64_t ldf, void* X, int64_t ldx,
                               void* stream) {
    psw::clear_error();
    psw::reset_launches();
    if (!m || !F || !X || ldf < m->N || ldx < m->N) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid arguments to psw_multi_solve");
        return PSW_INVALID_ARGUMENT;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != m->device) PSW_CUDA_TRY(cudaSetDevice(m->device));
    auto s = static_cast<cudaStream_t>(stream);
    const int rc = m->dtype == PSW_F64 ? psw::bundle_solve<double>(m, F, ldf, X, ldx, s)
                                       : psw::bundle_solve<float>(m, F, ldf, X, ldx, s);
    if (prev != m->device) cudaSetDevice(prev);
    return rc;
}

extern "C" int psw_solve_multi(const psw_plan* const* plans, int64_t nplans, const void* F,
                               int64_t ldf, void* X, int64_t ldx, void* stream) {
    psw::clear_error();
    psw::reset_launches();
    if (nplans < 0 || (nplans > 0 && (!plans || !F || !X)) || ldf < nplans || ldx < nplans) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid arguments to psw_solve_multi");
        return PSW_INVALID_ARGUMENT;
    }
    if (nplans == 0) return PSW_OK;
    const psw_plan* p0 = plans[0];
    for (int64_t k = 0; k < nplans; ++k) {
        const psw_plan* q = plans[k];
        if (!q || q->world != 1 || q->n != p0->n || q->P != p0->P || q->dtype != p0->dtype ||
            q->device != p0->device || q->bnd != p0->bnd) {
            psw::set_error(PSW_INVALID_ARGUMENT,
                           "psw_solve_multi: plans must share order, partition, dtype and device");
            return PSW_INVALID_ARGUMENT;
        }
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != p0->device) PSW_CUDA_TRY(cudaSetDevice(p0->device));
    auto s = static_cast<cudaStream_t>(stream);
    const int rc = p0->dtype == PSW_F64 ? psw::launch_multi<double>(plans, nplans, F, ldf, X, ldx, s)
                                        : psw::launch_multi<float>(plans, nplans, F, ldf, X, ldx, s);
    if (prev != p0->device) cudaSetDevice(prev);
    return rc;
}
