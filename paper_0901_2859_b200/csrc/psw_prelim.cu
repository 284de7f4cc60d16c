// GPU-side preliminary for the DirectSymmetric route:
// the p boundaries' three Thomas solves of compute_preliminary
// (preliminary.hpp:171-199: g_j = inv(A) e_{r_j} (:139-143), z_left (:29-37)
// and z_right (:41-49)) as 3p independent device threads, one sequential
// sweep each, instead of the host's worker threads.
//
// Every operation is the host restatement's (psw_plan.cpp thomas(), compiled
// without FP contraction): separately rounded products, sums and IEEE
// divisions (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn), the same pivot
// floor, the same loop order. The results are therefore bitwise the host
// setup's (and so the reference's): inverse-row restrictions, Z samples,
// the largest |z| and the first pivot breakdown in the serial executor's
// order (boundary, then g, z_left, z_right).
#include <algorithm>
#include <vector>

#include "psw_internal.h"

namespace psw {
namespace {

constexpr double kFloor = 1e-300;  // core/thomas.hpp:14

struct PrelimArgs {
    int64_t n, p;
    const double *sub, *diag, *sup;
    const int64_t* bnd;   // 1-based boundaries
    const int32_t* blk;   // [2t] = s_t, [2t+1] = e_t (0-based owned rows)
    double *gr, *gl;      // n each: inverse rows restricted to blocks j, j+1
    double *zr, *zl;      // p x p samples
    double* zmax;         // per (task, j)
    int64_t* fail;        // per (task, j): breakdown row or -1
    double* scratch;      // per (task, j): al[n], be[n]
};

// The host thomas() on one system given by accessor functions; keeps al/be in
// scratch, then runs the backward sweep calling visit(i, x_i) from i = n-1
// down to `stop` (inclusive). Returns the breakdown row or -1.
// The coefficient loads of kB rows are issued together ahead of their
// dependent chain (a single thread otherwise waits a full memory latency per
// row), and so are the backward sweep's al/be reloads.
constexpr int kB = 32;

template <typename Sub, typename Diag, typename Sup, typename Rhs, typename Visit>
__device__ int64_t thomas_dev(int64_t n, Sub sub, Diag diag, Sup sup, Rhs f, double* al,
                              double* be, int64_t stop, Visit visit) {
    double piv = diag(0);
    if (fabs(piv) < kFloor) return 0;
    double alp = n > 1 ? __ddiv_rn(-sup(0), piv) : 0.0;
    double bep = __ddiv_rn(f(0), piv);
    al[0] = alp;
    be[0] = bep;
    for (int64_t i0 = 1; i0 < n; i0 += kB) {
        double vs[kB], vd[kB], vu[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + u;
            if (i < n) {
                vs[u] = sub(i - 1);
                vd[u] = diag(i);
                vu[u] = i + 1 < n ? sup(i) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + u;
            if (i < n) {
                piv = __dadd_rn(vd[u], __dmul_rn(vs[u], alp));
                if (fabs(piv) < kFloor) return i;
                alp = i + 1 < n ? __ddiv_rn(-vu[u], piv) : 0.0;
                bep = __ddiv_rn(__dsub_rn(f(i), __dmul_rn(vs[u], bep)), piv);
                al[i] = alp;
                be[i] = bep;
            }
        }
    }
    double x = be[n - 1];
    visit(n - 1, x);
    for (int64_t i1 = n - 2; i1 >= stop; i1 -= kB) {
        double va[kB], vb[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i1 - u;
            if (i >= stop) {
                va[u] = al[i];
                vb[u] = be[i];
            }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i1 - u;
            if (i >= stop) {
                x = __dadd_rn(vb[u], __dmul_rn(va[u], x));
                visit(i, x);
            }
        }
    }
    return -1;
}

// the backward sweep again from stored al/be (z_left samples)
template <typename Visit>
__device__ void thomas_back(int64_t n, const double* al, const double* be, Visit visit) {
    double x = be[n - 1];
    visit(n - 1, x);
    for (int64_t i1 = n - 2; i1 >= 0; i1 -= kB) {
        double va[kB], vb[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (i1 - u >= 0) {
                va[u] = al[i1 - u];
                vb[u] = be[i1 - u];
            }
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (i1 - u >= 0) {
                x = __dadd_rn(vb[u], __dmul_rn(va[u], x));
                visit(i1 - u, x);
            }
    }
}

__global__ void prelim_kernel(PrelimArgs a) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int task = blockIdx.y;  // 0: g row, 1: z_left, 2: z_right
    if (j >= a.p) return;
    const int64_t n = a.n, p = a.p, r = a.bnd[j];
    const int64_t slot = int64_t(task) * p + j;
    double* al = a.scratch + size_t(slot) * 2 * size_t(n);
    double* be = al + n;
    double mz = 0.0;
    int64_t bad = -1;
    if (task == 0) {
        // g_j: A e_{r-1}; rows of blocks j and j+1 only (betas.hpp:46-55)
        const int64_t lo = a.blk[2 * j], mid = a.blk[2 * j + 1], hi = a.blk[2 * (j + 1) + 1];
        bad = thomas_dev(
            n, [&](int64_t i) { return a.sub[i]; }, [&](int64_t i) { return a.diag[i]; },
            [&](int64_t i) { return a.sup[i]; },
            [&](int64_t i) { return i == r - 1 ? 1.0 : 0.0; }, al, be, lo,
            [&](int64_t i, double x) {
                if (i >= lo && i < mid) a.gr[i] = x;
                else if (i >= mid && i < hi) a.gl[i] = x;
            });
    } else if (task == 1) {
        // z_left: rows 0..r-1, the last one a unit row, rhs e_last
        bad = thomas_dev(
            r, [&](int64_t i) { return i == r - 2 ? 0.0 : a.sub[i]; },
            [&](int64_t i) { return i == r - 1 ? 1.0 : a.diag[i]; },
            [&](int64_t i) { return a.sup[i]; },
            [&](int64_t i) { return i == r - 1 ? 1.0 : 0.0; }, al, be, 0,
            [&](int64_t i, double x) { mz = fmax(mz, fabs(x)); });
        if (bad < 0) {  // samples ZL[j][i] = z_left[r_i - 1], i <= j (preliminary.hpp:85-96)
            int64_t next = j;  // boundaries are increasing: walk them down with a second sweep
            thomas_back(r, al, be, [&](int64_t i, double x) {
                while (next >= 0 && a.bnd[next] - 1 == i) {
                    a.zl[j * p + next] = x;
                    --next;
                }
            });
        }
    } else {
        // z_right: rows r-1..n-1, the first one a unit row, rhs e_first
        const int64_t m = n - r + 1;
        int64_t nq = p - 1;
        bad = thomas_dev(
            m, [&](int64_t i) { return a.sub[r - 1 + i]; },
            [&](int64_t i) { return i == 0 ? 1.0 : a.diag[r - 1 + i]; },
            [&](int64_t i) { return i == 0 ? 0.0 : a.sup[r - 1 + i]; },
            [&](int64_t i) { return i == 0 ? 1.0 : 0.0; }, al, be, 0,
            [&](int64_t i, double x) {
                mz = fmax(mz, fabs(x));
                // ZR[j][q] = z_right[r_q - r], q >= j (preliminary.hpp:85-96): the
                // sweep runs downwards, so walk the boundaries from the last one
                while (nq >= j && a.bnd[nq] - r == i) {
                    a.zr[j * p + nq] = x;
                    --nq;
                }
            });
    }
    a.zmax[slot] = mz;
    a.fail[slot] = bad;
}

}  // namespace

// Device preliminary of a DirectSymmetric plan: fills gr, gl (n), zr, zl
// (p x p), max_z; returns PSW_OK or PSW_PIVOT_BREAKDOWN with *bad_row (the
// serial executor's first failure) or a CUDA error.
int device_preliminary(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* bnd, const std::vector<int32_t>& blk,
                       std::vector<double>& gr, std::vector<double>& gl, std::vector<double>& zr,
                       std::vector<double>& zl, double& max_z, int64_t& bad_row) {
    const size_t nn = size_t(n), pp = size_t(p);
    size_t bytes = sizeof(double) * (3 * nn + 2 * nn + 2 * pp * pp + 3 * pp) +
                   sizeof(int64_t) * (pp + 3 * pp) + sizeof(int32_t) * blk.size() +
                   sizeof(double) * 3 * pp * 2 * nn + 16 * 256;  // + carve alignment
    char* d = nullptr;
    PSW_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&d), bytes));
    auto carve = [&](size_t b) {
        char* q = d;
        d += (b + 255) & ~size_t(255);
        return q;
    };
    char* base = d;
    PrelimArgs a;
    a.n = n;
    a.p = p;
    double* dsub = reinterpret_cast<double*>(carve(sizeof(double) * nn));
    double* ddiag = reinterpret_cast<double*>(carve(sizeof(double) * nn));
    double* dsup = reinterpret_cast<double*>(carve(sizeof(double) * nn));
    int64_t* dbnd = reinterpret_cast<int64_t*>(carve(sizeof(int64_t) * pp));
    int32_t* dblk = reinterpret_cast<int32_t*>(carve(sizeof(int32_t) * blk.size()));
    a.gr = reinterpret_cast<double*>(carve(sizeof(double) * nn));
    a.gl = reinterpret_cast<double*>(carve(sizeof(double) * nn));
    a.zr = reinterpret_cast<double*>(carve(sizeof(double) * pp * pp));
    a.zl = reinterpret_cast<double*>(carve(sizeof(double) * pp * pp));
    a.zmax = reinterpret_cast<double*>(carve(sizeof(double) * 3 * pp));
    a.fail = reinterpret_cast<int64_t*>(carve(sizeof(int64_t) * 3 * pp));
    a.scratch = reinterpret_cast<double*>(carve(sizeof(double) * 3 * pp * 2 * nn));
    a.sub = dsub;
    a.diag = ddiag;
    a.sup = dsup;
    a.bnd = dbnd;
    a.blk = dblk;
    int rc = PSW_OK;
    auto fail = [&](cudaError_t e, const char* what) {
        rc = cuda_fail(e, what);
        cudaFree(base);
        return rc;
    };
    cudaError_t e;
    if ((e = cudaMemcpy(dsub, sub, sizeof(double) * (nn - 1), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(ddiag, diag, sizeof(double) * nn, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dsup, sup, sizeof(double) * (nn - 1), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dbnd, bnd, sizeof(int64_t) * pp, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dblk, blk.data(), sizeof(int32_t) * blk.size(), cudaMemcpyHostToDevice)) ||
        (e = cudaMemset(a.gr, 0, sizeof(double) * nn)) || (e = cudaMemset(a.gl, 0, sizeof(double) * nn)) ||
        (e = cudaMemset(a.zr, 0, sizeof(double) * pp * pp)) ||
        (e = cudaMemset(a.zl, 0, sizeof(double) * pp * pp)))
        return fail(e, "device preliminary upload");
    prelim_kernel<<<dim3(unsigned((p + 31) / 32), 3), 32>>>(a);
    if ((e = cudaGetLastError()) || (e = cudaDeviceSynchronize())) return fail(e, "device preliminary");
    std::vector<double> zmax(3 * pp);
    std::vector<int64_t> fails(3 * pp);
    gr.assign(nn, 0.0);
    gl.assign(nn, 0.0);
    zr.assign(pp * pp, 0.0);
    zl.assign(pp * pp, 0.0);
    if ((e = cudaMemcpy(gr.data(), a.gr, sizeof(double) * nn, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(gl.data(), a.gl, sizeof(double) * nn, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(zr.data(), a.zr, sizeof(double) * pp * pp, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(zl.data(), a.zl, sizeof(double) * pp * pp, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(zmax.data(), a.zmax, sizeof(double) * 3 * pp, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(fails.data(), a.fail, sizeof(int64_t) * 3 * pp, cudaMemcpyDeviceToHost)))
        return fail(e, "device preliminary download");
    cudaFree(base);
    bad_row = -1;
    for (size_t j = 0; j < pp && bad_row < 0; ++j)  // boundary order, then g, z_left, z_right
        for (int task = 0; task < 3 && bad_row < 0; ++task)
            if (fails[task * pp + j] >= 0) bad_row = fails[task * pp + j];
    if (bad_row >= 0) return PSW_PIVOT_BREAKDOWN;
    max_z = 0.0;
    for (size_t j = 0; j < pp; ++j) max_z = std::max({max_z, zmax[pp + j], zmax[2 * pp + j]});
    return PSW_OK;
}

}  // namespace psw
