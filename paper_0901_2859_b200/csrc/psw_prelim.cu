// GPU-side preliminary for the DirectSymmetric route:
// the p boundaries' three Thomas solves of compute_preliminary
// (preliminary.hpp:171-199: g_j = inv(A) e_{r_j} (:139-143), z_left (:29-37)
// and z_right (:41-49)) on the device, bitwise the host restatement
// (psw_plan.cpp thomas(), itself bitwise the reference).
//
// Every value is produced by the host's operations in the host's order
// (separately rounded __dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn, the same
// pivot floor), so nothing is re-associated. What makes it fast is that most
// of the 3p sweeps' 6 p n row steps are provably redundant, and which ones is
// decided by exact (bit) comparisons, never by a tolerance:
//
// 1. One pivot chain instead of 2p + 1. The forward eliminations of all g_j
//    and of every z_left run over rows of A itself, so their pivots and
//    alphas are those of ONE chain over A ("global chain": pv_i, al_i). A
//    z_right system starts with a unit row at r_j; its chain al' is computed
//    row by row until al'_i has the same bits as al_i — from there on both
//    chains apply the same operations to the same state and stay identical,
//    so the global values are used. Strictly dominant matrices merge within
//    a few dozen rows; a chain that never merges simply runs to the end.
// 2. The global chain itself is cut into chunks of L rows, each started W
//    rows early from an arbitrary state (the row taken as a first row). A
//    chunk is accepted iff the alpha it computed for the row before its
//    first row has the bits of the alpha its predecessor stored there
//    (induction from chunk 0, which starts at row 0). If any chunk is
//    refused, one thread recomputes the whole chain serially (the slow, always
//    exact path: non-contractive matrices such as (-1, 2, -1)).
// 3. Unit right-hand sides make beta chains that are exactly zero outside a
//    window: before the unit entry beta_i = (+0)/pv_i, after it the chain
//    beta_i = (0 - s beta_{i-1})/pv_i decays and, once a beta is exactly
//    zero, every later one is (+0)/pv_i again. The serial division chain
//    stops there. In such a zero region the back substitution
//    x_i = beta_i + al_i x_{i+1} only produces signed zeros, and
//    (+0) + (+-0) = +0 restarts the sign at every row with a positive pivot:
//    the value at any row follows from the nearest such row above it
//    ("anchor"), not from the whole chain.
//
// Scratch holds a window of kWin rows per chain; a chain that needs more (a
// matrix whose betas do not decay) reports overflow and the caller runs the
// host setup instead.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "psw_internal.h"

namespace psw {
namespace {

constexpr double kFloor = 1e-300;  // core/thomas.hpp:14
constexpr int kB = 16;             // rows whose loads are issued together

struct PrelimArgs {
    int64_t n, p;
    int64_t L, W, nchunk, win;
    const double *sub, *diag, *sup;
    const int64_t* bnd;   // 1-based boundaries
    const int32_t* blk;   // [2t] = s_t, [2t+1] = e_t (0-based owned rows)
    double *al, *pv;      // the global chain (n each)
    long long* spec;      // per chunk: bits of the alpha computed for row cL - 1
    int64_t* brk;         // per chunk: first stored row with |pivot| < floor, or -1
    int32_t* neg;         // per chunk: 1 if some row's pivot is not > 0 (conservative)
    int64_t* status;      // [0] global breakdown row or -1, [1] serial path taken, [2] window overflow
    double *gr, *gl;      // n each: inverse rows restricted to blocks j, j+1
    double *zr, *zl;      // p x p samples
    double* zmax;         // [2][p]
    int64_t* fail;        // per j: z_right breakdown (local row) or -1
    double *bg, *az, *bz; // p x win windows: g betas, z_right alphas and betas
};

__device__ __forceinline__ long long bits(double v) { return __double_as_longlong(v); }
__device__ __forceinline__ double zero_like(double pv) { return copysign(0.0, pv); }  // (+0)/pv

// ---- the global chain, speculative chunks ---------------------------------
__global__ void pivot_chunks_kernel(PrelimArgs a) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= a.nchunk) return;
    const int64_t n = a.n, start = c * a.L, end = min(n, start + a.L);
    const int64_t w0 = max(int64_t(0), start - a.W);
    double piv = a.diag[w0];
    double alp = w0 + 1 < n ? __ddiv_rn(-a.sup[w0], piv) : 0.0;
    int64_t brk = -1;
    bool warm_bad = false, anyneg = false;
    if (w0 >= start) {
        if (fabs(piv) < kFloor) brk = w0;
        anyneg = !(piv > 0.0);
        a.al[w0] = alp;
        a.pv[w0] = piv;
    } else if (fabs(piv) < kFloor) {
        warm_bad = true;
    }
    if (w0 == start - 1) a.spec[c] = bits(alp);
    for (int64_t i0 = w0 + 1; i0 < end; i0 += kB) {
        double vs[kB], vd[kB], vu[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + u;
            if (i < end) {
                vs[u] = a.sub[i - 1];
                vd[u] = a.diag[i];
                vu[u] = i + 1 < n ? a.sup[i] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + u;
            if (i < end) {
                piv = __dadd_rn(vd[u], __dmul_rn(vs[u], alp));
                alp = i + 1 < n ? __ddiv_rn(-vu[u], piv) : 0.0;
                if (i >= start) {
                    if (brk < 0 && fabs(piv) < kFloor) brk = i;
                    anyneg |= !(piv > 0.0);
                    a.al[i] = alp;
                    a.pv[i] = piv;
                } else {
                    if (fabs(piv) < kFloor) warm_bad = true;
                    if (i == start - 1) a.spec[c] = bits(alp);
                }
            }
        }
    }
    // a floor hit while warming up came from a state that may not be the true
    // one: refuse the chunk (0x7ff8... with a payload no division produces)
    if (warm_bad) a.spec[c] = 0x7ff8dead0000beefLL;
    a.brk[c] = brk;
    a.neg[c] = anyneg ? 1 : 0;
}

// accept the chunks (parallel) or recompute the whole chain with one thread
__global__ void pivot_accept_kernel(PrelimArgs a) {
    __shared__ int s_bad;
    __shared__ unsigned long long s_brk;
    if (threadIdx.x == 0) {
        s_bad = 0;
        s_brk = ~0ull;
    }
    __syncthreads();
    int bad = 0;
    unsigned long long first = ~0ull;
    for (int64_t c = threadIdx.x; c < a.nchunk; c += blockDim.x) {
        if (c > 0 && bits(a.al[c * a.L - 1]) != a.spec[c]) bad = 1;
        if (a.brk[c] >= 0) first = min(first, (unsigned long long)a.brk[c]);
    }
    if (bad) atomicOr(&s_bad, 1);
    if (first != ~0ull) atomicMin(&s_brk, first);
    __syncthreads();
    if (s_bad)  // the chunks' flags describe refused values: walk every row
        for (int64_t c = threadIdx.x; c < a.nchunk; c += blockDim.x) a.neg[c] = 1;
    if (threadIdx.x != 0) return;
    a.status[1] = s_bad;
    if (!s_bad) {
        a.status[0] = s_brk == ~0ull ? -1 : int64_t(s_brk);
        return;
    }
    // the always-exact path: the host loop, one thread
    const int64_t n = a.n;
    double piv = a.diag[0];
    int64_t brk = -1;
    if (fabs(piv) < kFloor) brk = 0;
    double alp = n > 1 ? __ddiv_rn(-a.sup[0], piv) : 0.0;
    a.al[0] = alp;
    a.pv[0] = piv;
    for (int64_t i0 = 1; i0 < n && brk < 0; i0 += kB) {
        double vs[kB], vd[kB], vu[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + u;
            if (i < n) {
                vs[u] = a.sub[i - 1];
                vd[u] = a.diag[i];
                vu[u] = i + 1 < n ? a.sup[i] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + u;
            if (i < n && brk < 0) {
                piv = __dadd_rn(vd[u], __dmul_rn(vs[u], alp));
                if (fabs(piv) < kFloor) brk = i;
                alp = i + 1 < n ? __ddiv_rn(-vu[u], piv) : 0.0;
                a.al[i] = alp;
                a.pv[i] = piv;
            }
        }
    }
    a.status[0] = brk;
}

// ---- the 3p boundary sweeps -------------------------------------------------
// Row-indexed arrays are reached through views so that the same sweeps run
// on one system (Lin: contiguous rows) and on a batch of systems laid out
// [row][system] (Str: thread k strides by the number of systems, a warp's 32
// systems read one contiguous piece per row).
template <typename T>
struct Lin {
    T* p;
    __device__ __forceinline__ T& operator[](int64_t i) const { return p[i]; }
    __device__ __forceinline__ Lin at(int64_t i) const { return Lin{p + i}; }
};
template <typename T>
struct Str {
    T* p;
    int64_t s;
    __device__ __forceinline__ T& operator[](int64_t i) const { return p[i * s]; }
    __device__ __forceinline__ Str at(int64_t i) const { return Str{p + i * s, s}; }
};

template <template <typename> class V>
struct SweepView {
    int64_t n, p, L, win;
    V<const double> sub, diag, sup, al, pv;  // A and its global chain
    V<const int32_t> neg;                    // per chunk of L rows: some pivot is not > 0
    V<double> gr, gl;                        // g_j on blocks j / j+1
    V<double> bg, az, bz;                    // windows of all p chains (chain j at j * win)
    const int64_t* bnd;                      // 1-based boundaries
    const int32_t* blk;                      // [2t] = s_t, [2t+1] = e_t
    double *zr, *zl;                         // p x p samples
    double* zmax;                            // [2][p]
    int64_t* fail;                           // per j: z_right breakdown (local row) or -1
    int64_t* overflow;                       // set to 1 when a chain outgrows its window
};

// first row k >= q of a zero region whose value is known without looking
// further: a positive pivot ((+0) + (+-0) = +0) or the region's last row
template <typename PV>
__device__ __forceinline__ int64_t anchor(const PV& pv, int64_t q, int64_t last) {
    int64_t k = q;
    while (k < last && !(pv[k] > 0.0)) ++k;
    return k;
}

// x_i = be(i) + al[i] x_{i+1} from row hi - 1 down to lo with batched loads
template <typename Be, typename Al, typename Visit>
__device__ __forceinline__ void back_chain(int64_t hi, int64_t lo, double& x, Be be, Al al,
                                           Visit visit) {
    for (int64_t i1 = hi - 1; i1 >= lo; i1 -= kB) {
        double va[kB], vb[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (i1 - u >= lo) {
                va[u] = al(i1 - u);
                vb[u] = be(i1 - u);
            }
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (i1 - u >= lo) {
                x = __dadd_rn(vb[u], __dmul_rn(va[u], x));
                visit(i1 - u, x);
            }
    }
}

// Rows b-1 .. lo of a zero region (betas (+0)/pv, x_b = x a signed zero): a
// chunk whose pivots are all positive holds +0 everywhere, which the tables
// were initialised to, and hands +0 on; other chunks are walked row by row.
template <template <typename> class V, typename Keep>
__device__ __forceinline__ void zero_walk(const SweepView<V>& a, int64_t lo, int64_t b, double& x,
                                          Keep keep) {
    int64_t i = b - 1;
    while (i >= lo) {
        const int64_t c = i / a.L, first = max(lo, c * a.L);
        if (!a.neg[c]) {
            x = 0.0;
        } else {
            back_chain(i + 1, first, x, [&](int64_t q) { return zero_like(a.pv[q]); },
                       [&](int64_t q) { return a.al[q]; }, keep);
        }
        i = first - 1;
    }
}

template <template <typename> class V>
__device__ __forceinline__ void sweep_task(const SweepView<V>& a, int64_t j, int task) {
    const int64_t n = a.n, p = a.p, r = a.bnd[j], win = a.win;
    const auto &al = a.al, &pv = a.pv, &sub = a.sub;
    auto zal = [&](int64_t i) { return al[i]; };
    auto zbe = [&](int64_t i) { return zero_like(pv[i]); };
    if (task == 0) {
        // g_j = inv(A) e_{r-1}: betas are (+0)/pv before row r-1, 1/pv_{r-1}
        // there, then the decaying chain; rows of blocks j and j+1 are kept
        // (betas.hpp:46-55)
        const int64_t lo = a.blk[2 * j], mid = a.blk[2 * j + 1], hi = a.blk[2 * (j + 1) + 1];
        const auto bg = a.bg.at(j * win);
        double be = __ddiv_rn(1.0, pv[r - 1]);
        bg[0] = be;
        int64_t fend = r - 1;
        for (int64_t i = r; i < n && be != 0.0; ++i) {
            if (i - (r - 1) >= win) {
                *a.overflow = 1;
                return;
            }
            be = __ddiv_rn(__dsub_rn(0.0, __dmul_rn(sub[i - 1], be)), pv[i]);
            bg[i - (r - 1)] = be;
            fend = i;
        }
        auto keep = [&](int64_t i, double x) {
            if (i >= lo && i < mid) a.gr[i] = x;
            else if (i >= mid && i < hi) a.gl[i] = x;
        };
        // x belongs to row cur; rows above fend hold signed zeros
        const int64_t s0 = max(fend, hi - 1);
        int64_t cur;
        double x;
        if (s0 == n - 1) {
            x = fend == n - 1 ? double(bg[fend - (r - 1)]) : zero_like(pv[n - 1]);
            cur = n - 1;
            keep(cur, x);
        } else {
            const int64_t k = anchor(pv, s0 + 1, n - 1);
            x = zero_like(pv[k]);
            back_chain(k, s0 + 1, x, zbe, zal, [&](int64_t, double) {});
            cur = s0 + 1;  // >= hi: not kept
        }
        if (cur > fend + 1) {  // stored rows of block j+1 beyond the betas' decay
            zero_walk(a, fend + 1, cur, x, keep);
            cur = fend + 1;
        }
        back_chain(cur, r - 1, x, [&](int64_t i) { return double(bg[i - (r - 1)]); }, zal, keep);
        cur = r - 1;
        // below the unit entry the betas are (+0)/pv again: x decays to an exact zero
        while (cur > lo && x != 0.0) {
            const int64_t stop = max(lo, cur - 64);
            back_chain(cur, stop, x, zbe, zal, keep);
            cur = stop;
        }
        zero_walk(a, lo, cur, x, keep);
    } else if (task == 1) {
        // z_left: rows 0..r-1 of A with a unit last row and rhs e_last: the
        // global chain up to row r-2, betas (+0)/pv, x_{r-1} = 1
        // samples ZL[j][i] = z_left[r_i - 1], i <= j (preliminary.hpp:85-96)
        int64_t next = j;
        double mz = 0.0, x = 1.0;
        int64_t row = r - 1;  // the row x belongs to
        auto visit = [&](int64_t i, double v) {
            mz = fmax(mz, fabs(v));
            while (next >= 0 && a.bnd[next] - 1 == i) {
                a.zl[j * p + next] = v;
                --next;
            }
        };
        visit(row, x);
        // the decaying part, in pieces, until the value is an exact zero
        while (row > 0 && x != 0.0) {
            const int64_t lo = max(int64_t(0), row - 256);
            int64_t stop = row;  // first row (from above) holding an exact zero
            bool hit = false;
            for (int64_t i1 = row - 1; i1 >= lo && !hit; i1 -= kB) {
                double va[kB], vp[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u)
                    if (i1 - u >= lo) {
                        va[u] = al[i1 - u];
                        vp[u] = pv[i1 - u];
                    }
#pragma unroll
                for (int u = 0; u < kB; ++u)
                    if (i1 - u >= lo && !hit) {
                        x = __dadd_rn(zero_like(vp[u]), __dmul_rn(va[u], x));
                        visit(i1 - u, x);
                        stop = i1 - u;
                        hit = x == 0.0;
                    }
            }
            row = stop;
        }
        // zero region below `row` (x_row = +-0 known): the remaining samples
        while (next >= 0) {
            const int64_t q = a.bnd[next] - 1;  // q < row
            const int64_t k = anchor(pv, q, row);
            double v = k == row ? x : zero_like(pv[k]);
            back_chain(k, q, v, zbe, zal, [&](int64_t, double) {});
            a.zl[j * p + next] = v;
            // the next sample lies below q, whose value is now known
            row = q;
            x = v;
            --next;
        }
        a.zmax[j] = mz;
    } else {
        // z_right: rows r-1..n-1 of A with a unit first row and rhs e_first;
        // local row i is global row r-1+i
        const int64_t m = n - r + 1, g0 = r - 1;
        const auto az = a.az.at(j * win), bz = a.bz.at(j * win);
        double alp = m > 1 ? __ddiv_rn(-0.0, 1.0) : 0.0;
        double be = __ddiv_rn(1.0, 1.0);
        az[0] = alp;
        bz[0] = be;
        bool merged = false;
        int64_t fend = 0;
        for (int64_t i = 1; i < m && !(merged && be == 0.0); ++i) {
            if (i >= win) {
                *a.overflow = 1;
                return;
            }
            const int64_t g = g0 + i;
            double piv;
            if (!merged) {
                piv = __dadd_rn(a.diag[g], __dmul_rn(sub[g - 1], alp));
                if (fabs(piv) < kFloor) {
                    a.fail[j] = i;
                    return;
                }
                alp = i + 1 < m ? __ddiv_rn(-a.sup[g], piv) : 0.0;
                merged = bits(alp) == bits(al[g]);
            } else {
                piv = pv[g];
                alp = al[g];
            }
            be = __ddiv_rn(__dsub_rn(0.0, __dmul_rn(sub[g - 1], be)), piv);
            az[i] = alp;
            bz[i] = be;
            fend = i;
        }
        // rows beyond fend (if any): merged, betas (+0)/pv — a zero region up
        // to the last row. Samples ZR[j][q] = z_right[r_q - r], q >= j.
        int64_t nq = p - 1;
        while (nq >= j && a.bnd[nq] - r > fend) {
            const int64_t q = g0 + (a.bnd[nq] - r);
            const int64_t k = anchor(pv, q, n - 1);
            double v = zero_like(pv[k]);
            back_chain(k, q, v, zbe, zal, [&](int64_t, double) {});
            a.zr[j * p + nq] = v;
            --nq;
        }
        double mz = 0.0, x;
        auto visit = [&](int64_t i, double v) {
            mz = fmax(mz, fabs(v));
            while (nq >= j && a.bnd[nq] - r == i) {
                a.zr[j * p + nq] = v;
                --nq;
            }
        };
        if (fend == m - 1) {
            x = bz[fend];
        } else {  // x_{fend+1}: a signed zero from its anchor
            const int64_t q = g0 + fend + 1;
            const int64_t k = anchor(pv, q, n - 1);
            double v = zero_like(pv[k]);
            back_chain(k, q, v, zbe, zal, [&](int64_t, double) {});
            x = __dadd_rn(bz[fend], __dmul_rn(az[fend], v));
        }
        visit(fend, x);
        back_chain(fend, 0, x, [&](int64_t i) { return double(bz[i]); },
                   [&](int64_t i) { return double(az[i]); }, visit);
        a.zmax[p + j] = mz;
    }
}

__global__ void sweeps_kernel(PrelimArgs a) {
    if (threadIdx.x != 0 || a.status[0] >= 0) return;
    SweepView<Lin> v{a.n, a.p, a.L, a.win, {a.sub}, {a.diag}, {a.sup}, {a.al}, {a.pv}, {a.neg},
                     {a.gr}, {a.gl}, {a.bg}, {a.az}, {a.bz}, a.bnd, a.blk, a.zr, a.zl, a.zmax,
                     a.fail, a.status + 2};
    sweep_task(v, blockIdx.x, blockIdx.y);
}

int64_t env_i64(const char* name, int64_t dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoll(e) : dflt;
}

}  // namespace

// Device preliminary of a DirectSymmetric plan: fills gr, gl (n), zr, zl
// (p x p), max_z. Returns PSW_OK, PSW_PIVOT_BREAKDOWN with *bad_row (the
// serial executor's first failure: boundary, then g, z_left, z_right), a CUDA
// error, or PSW_NOT_SUPPORTED when a chain outgrew its scratch window or the
// scratch could not be allocated (the caller then runs the host setup).
// *serial = 1 if the global chain took the one-thread path.
int device_preliminary(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* bnd, const std::vector<int32_t>& blk,
                       std::vector<double>& gr, std::vector<double>& gl, std::vector<double>& zr,
                       std::vector<double>& zl, double& max_z, int64_t& bad_row, int* serial) {
    const size_t nn = size_t(n), pp = size_t(p);
    PrelimArgs a{};
    a.n = n;
    a.p = p;
    a.L = std::max<int64_t>(8, env_i64("PSW_PRELIM_CHUNK", 512));
    a.W = std::max<int64_t>(0, env_i64("PSW_PRELIM_WARM", 256));
    a.nchunk = (n + a.L - 1) / a.L;
    a.win = std::min<int64_t>(n, std::max<int64_t>(64, env_i64("PSW_PRELIM_WINDOW", 1 << 16)));
    const size_t nc = size_t(a.nchunk), win = size_t(a.win);
    auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t bytes = 7 * up(8 * nn) + up(8 * pp) + up(4 * blk.size()) + 2 * up(8 * nc) + up(4 * nc) +
                         up(8 * 4) + 2 * up(8 * pp * pp) + up(8 * 2 * pp) + up(8 * pp) +
                         3 * up(8 * pp * win);
    char* base = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&base), bytes) != cudaSuccess) {
        cudaGetLastError();  // no room for the device sweeps' scratch: the host runs them
        return PSW_NOT_SUPPORTED;
    }
    char* d = base;
    auto carve = [&](size_t b) {
        char* q = d;
        d += up(b);
        return q;
    };
    double* dsub = reinterpret_cast<double*>(carve(8 * nn));
    double* ddiag = reinterpret_cast<double*>(carve(8 * nn));
    double* dsup = reinterpret_cast<double*>(carve(8 * nn));
    a.al = reinterpret_cast<double*>(carve(8 * nn));
    a.pv = reinterpret_cast<double*>(carve(8 * nn));
    a.gr = reinterpret_cast<double*>(carve(8 * nn));
    a.gl = reinterpret_cast<double*>(carve(8 * nn));
    int64_t* dbnd = reinterpret_cast<int64_t*>(carve(8 * pp));
    int32_t* dblk = reinterpret_cast<int32_t*>(carve(4 * blk.size()));
    a.spec = reinterpret_cast<long long*>(carve(8 * nc));
    a.brk = reinterpret_cast<int64_t*>(carve(8 * nc));
    a.neg = reinterpret_cast<int32_t*>(carve(4 * nc));
    a.status = reinterpret_cast<int64_t*>(carve(8 * 4));
    a.zr = reinterpret_cast<double*>(carve(8 * pp * pp));
    a.zl = reinterpret_cast<double*>(carve(8 * pp * pp));
    a.zmax = reinterpret_cast<double*>(carve(8 * 2 * pp));
    a.fail = reinterpret_cast<int64_t*>(carve(8 * pp));
    a.bg = reinterpret_cast<double*>(carve(8 * pp * win));
    a.az = reinterpret_cast<double*>(carve(8 * pp * win));
    a.bz = reinterpret_cast<double*>(carve(8 * pp * win));
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
    if ((e = cudaMemcpy(dsub, sub, 8 * (nn - 1), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(ddiag, diag, 8 * nn, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dsup, sup, 8 * (nn - 1), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dbnd, bnd, 8 * pp, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dblk, blk.data(), 4 * blk.size(), cudaMemcpyHostToDevice)) ||
        (e = cudaMemsetAsync(a.gr, 0, 8 * nn)) || (e = cudaMemsetAsync(a.gl, 0, 8 * nn)) ||
        (e = cudaMemsetAsync(a.zr, 0, 8 * pp * pp)) || (e = cudaMemsetAsync(a.zl, 0, 8 * pp * pp)) ||
        (e = cudaMemsetAsync(a.status, 0, 8 * 4)) || (e = cudaMemsetAsync(a.spec, 0xff, 8 * nc)) || (e = cudaMemsetAsync(a.fail, 0xff, 8 * pp)))
        return fail(e, "device preliminary upload");
    const bool verbose = env_i64("PSW_SETUP_VERBOSE", 0) != 0;
    cudaEvent_t ev[4] = {};
    if (verbose)
        for (auto& q : ev) cudaEventCreate(&q);
    if (verbose) cudaEventRecord(ev[0]);
    pivot_chunks_kernel<<<unsigned((a.nchunk + 31) / 32), 32>>>(a);
    if (verbose) cudaEventRecord(ev[1]);
    pivot_accept_kernel<<<1, 256>>>(a);
    if (verbose) cudaEventRecord(ev[2]);
    sweeps_kernel<<<dim3(unsigned(p), 3), 32>>>(a);
    if (verbose) cudaEventRecord(ev[3]);
    if ((e = cudaGetLastError()) || (e = cudaDeviceSynchronize())) return fail(e, "device preliminary");
    if (verbose) {
        float t[3] = {};
        for (int k = 0; k < 3; ++k) cudaEventElapsedTime(&t[k], ev[k], ev[k + 1]);
        std::fprintf(stderr, "psw device preliminary: pivot chunks %.3f ms, accept %.3f ms, sweeps %.3f ms\n",
                     t[0], t[1], t[2]);
        for (auto& q : ev) cudaEventDestroy(q);
    }
    int64_t status[4];
    std::vector<double> zmax(2 * pp);
    std::vector<int64_t> fails(pp);
    if ((e = cudaMemcpy(status, a.status, sizeof(status), cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(zmax.data(), a.zmax, 8 * 2 * pp, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(fails.data(), a.fail, 8 * pp, cudaMemcpyDeviceToHost)))
        return fail(e, "device preliminary download");
    if (serial) *serial = int(status[1]);
    bad_row = status[0];  // the global chain: boundary 0's g row fails first
    for (size_t j = 0; j < pp && bad_row < 0; ++j)
        if (fails[j] >= 0) bad_row = fails[j];
    if (bad_row >= 0) {
        cudaFree(base);
        return PSW_PIVOT_BREAKDOWN;
    }
    if (status[2]) {  // a chain outgrew its window: not an error, the host does it
        cudaFree(base);
        return PSW_NOT_SUPPORTED;
    }
    gr.resize(nn);
    gl.resize(nn);
    zr.resize(pp * pp);
    zl.resize(pp * pp);
    if ((e = cudaMemcpy(gr.data(), a.gr, 8 * nn, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(gl.data(), a.gl, 8 * nn, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(zr.data(), a.zr, 8 * pp * pp, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(zl.data(), a.zl, 8 * pp * pp, cudaMemcpyDeviceToHost)))
        return fail(e, "device preliminary download");
    cudaFree(base);
    max_z = 0.0;
    for (size_t j = 0; j < 2 * pp; ++j) max_z = std::max(max_z, zmax[j]);
    return PSW_OK;
}

// ---------------------------------------------------------------------------
// Batched setup: N systems that share one partition (the Fourier consumer's
// harmonics, fourier.hpp:41-105: one matrix B_l per harmonic), every table of
// the multi-matrix bundle (psw_multi.cu) built on the device in [row][system]
// layout, one thread per system / (system, block) / (system, boundary, sweep).
// The arithmetic is the single-system setup's, operation for operation: the
// global pivot chain (serial per system here: the systems are the parallel
// axis), sweep_task for the 3p boundary sweeps, and build_plan's per-block
// sweep coefficients (local_solve.hpp:25-50 hoisted out of the RHS loop).
namespace {

struct BatchArgs {
    int64_t n, N, p, L, nchunk, win;
    const double *sub, *diag, *sup;  // [row][sys]
    double *al, *pv;                 // global chain [row][sys]
    int32_t* neg;                    // [chunk][sys]
    int64_t* brk;                    // [sys] first pivot breakdown of the global chain or -1
    double *rp, *ma, *w, *alb;       // block sweep coefficients [row][sys]
    double *gr, *gl;                 // [row][sys]
    double *bg, *az, *bz;            // [p * win][sys]
    const int64_t* bnd;
    const int32_t* blk;
    double *zr, *zl;                 // [sys][p * p + 2]
    double* zmax;                    // [sys][2 p]
    int64_t* fail;                   // [sys][p]
    int64_t* overflow;
};

// in[sys][len] -> out[len][sys]
__global__ void interleave_kernel(const double* __restrict__ in, double* __restrict__ out,
                                  int64_t N, int64_t len) {
    __shared__ double tile[32][33];
    const int64_t k0 = int64_t(blockIdx.x) * 32, i0 = int64_t(blockIdx.y) * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t k = k0 + r, i = i0 + threadIdx.x;
        if (k < N && i < len) tile[r][threadIdx.x] = in[k * len + i];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r, k = k0 + threadIdx.x;
        if (k < N && i < len) out[i * N + k] = tile[threadIdx.x][r];
    }
}

__global__ void batch_chain_kernel(BatchArgs a) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= a.N) return;
    const int64_t n = a.n, N = a.N;
    double piv = a.diag[k];
    int64_t brk = fabs(piv) < kFloor ? 0 : -1;
    double alp = n > 1 ? __ddiv_rn(-a.sup[k], piv) : 0.0;
    a.al[k] = alp;
    a.pv[k] = piv;
    bool anyneg = !(piv > 0.0);
    for (int64_t i0 = 1; i0 < n && brk < 0; i0 += kB) {
        double vs[kB], vd[kB], vu[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + u;
            if (i < n) {
                vs[u] = a.sub[(i - 1) * N + k];
                vd[u] = a.diag[i * N + k];
                vu[u] = i + 1 < n ? a.sup[i * N + k] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + u;
            if (i < n && brk < 0) {
                if (i % a.L == 0) {
                    a.neg[(i / a.L - 1) * N + k] = anyneg ? 1 : 0;
                    anyneg = false;
                }
                piv = __dadd_rn(vd[u], __dmul_rn(vs[u], alp));
                if (fabs(piv) < kFloor) brk = i;
                alp = i + 1 < n ? __ddiv_rn(-vu[u], piv) : 0.0;
                anyneg |= !(piv > 0.0);
                a.al[i * N + k] = alp;
                a.pv[i * N + k] = piv;
            }
        }
    }
    a.neg[((n - 1) / a.L) * N + k] = anyneg ? 1 : 0;
    a.brk[k] = brk;
}

// build_plan's per-row sweep coefficients of block t (psw_plan.cpp; the
// unit-row block systems of local_solve.hpp:25-50)
__global__ void batch_block_kernel(BatchArgs a) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t t = blockIdx.y;
    if (k >= a.N) return;
    const int64_t n = a.n, N = a.N, p = a.p;
    const int64_t s = a.blk[2 * t], e = a.blk[2 * t + 1];
    const int64_t h = t == p ? n - 1 : e;  // closed block end
    double alpha_prev, wprev;
    if (t > 0) {  // unit first row carrying x_{t-1}
        a.rp[s * N + k] = 0.0;
        a.ma[s * N + k] = 0.0;
        a.w[s * N + k] = 1.0;
        a.alb[s * N + k] = 0.0;
        alpha_prev = 0.0;
        wprev = 1.0;
    } else {
        const double piv = a.diag[k];
        alpha_prev = h > s ? __ddiv_rn(-a.sup[k], piv) : 0.0;
        a.rp[s * N + k] = __ddiv_rn(1.0, piv);
        a.ma[s * N + k] = 0.0;
        a.w[s * N + k] = 0.0;
        a.alb[s * N + k] = alpha_prev;
        wprev = 0.0;
    }
    const int64_t last = t == p ? n : e;
    for (int64_t q0 = s + 1; q0 < last; q0 += kB) {
        double vs[kB], vd[kB], vu[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t q = q0 + u;
            if (q < last) {
                vs[u] = a.sub[(q - 1) * N + k];
                vd[u] = a.diag[q * N + k];
                vu[u] = q < h ? a.sup[q * N + k] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t q = q0 + u;
            if (q < last) {
                const double piv = __dadd_rn(vd[u], __dmul_rn(vs[u], alpha_prev));
                const double al = q < h ? __ddiv_rn(-vu[u], piv) : 0.0;
                const double ma = __ddiv_rn(-vs[u], piv);
                wprev = t > 0 ? __dmul_rn(ma, wprev) : 0.0;
                a.rp[q * N + k] = __ddiv_rn(1.0, piv);
                a.ma[q * N + k] = ma;
                a.w[q * N + k] = wprev;
                a.alb[q * N + k] = al;
                alpha_prev = al;
            }
        }
    }
}

__global__ void batch_sweeps_kernel(BatchArgs a) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= a.N || a.brk[k] >= 0) return;
    const int64_t N = a.N, p = a.p;
    SweepView<Str> v{a.n, p, a.L, a.win,
                     {a.sub + k, N}, {a.diag + k, N}, {a.sup + k, N}, {a.al + k, N}, {a.pv + k, N},
                     {a.neg + k, N}, {a.gr + k, N}, {a.gl + k, N}, {a.bg + k, N}, {a.az + k, N},
                     {a.bz + k, N}, a.bnd, a.blk, a.zr + k * (p * p + 2), a.zl + k * (p * p + 2),
                     a.zmax + k * 2 * p, a.fail + k * p, a.overflow};
    sweep_task(v, blockIdx.y, blockIdx.z);
}

template <typename T>
__global__ void batch_assemble_kernel(BatchArgs a, FwdCoef<T>* __restrict__ fo,
                                      BwdCoef<T>* __restrict__ bo) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= a.N) return;
    for (int64_t q = blockIdx.y; q < a.n; q += gridDim.y) {
        const int64_t o = q * a.N + k;
        fo[o] = {T(a.rp[o]), T(a.ma[o]), T(a.gr[o]), T(a.gl[o])};
        bo[o] = {T(a.w[o]), T(a.alb[o])};
    }
}

}  // namespace

size_t device_setup_batch_bytes(int64_t n, int64_t N, int64_t p) {
    return sizeof(double) * size_t(n) * size_t(N) * (3 + 2 + 4 + 2 + 3 * size_t(p));
}

// sub / diag / sup: host arrays [N][n-1] / [N][n] / [N][n-1]. fwd / bwd: device
// FwdCoef<T> / BwdCoef<T> [n][N]; zr / zl: device [N][p p + 2] (zeroed here).
// PSW_PIVOT_BREAKDOWN reports the first failing system and its row in the
// serial executor's order.
int device_setup_batch(int64_t n, int64_t N, const double* sub, const double* diag,
                       const double* sup, int64_t p, const int64_t* bnd,
                       const std::vector<int32_t>& blk, int dtype, void* fwd, void* bwd, double* zr,
                       double* zl, int64_t& bad_sys, int64_t& bad_row) {
    const size_t nn = size_t(n), NN = size_t(N), pp = size_t(p);
    BatchArgs a{};
    a.n = n;
    a.N = N;
    a.p = p;
    a.L = 512;
    a.nchunk = (n + a.L - 1) / a.L;
    a.win = n;
    auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t plane = up(8 * nn * NN);
    const size_t bytes = (11 + 3 * pp) * plane + up(8 * (nn - 1) * NN) * 0 + up(4 * size_t(a.nchunk) * NN) +
                         up(8 * NN) + up(8 * pp) + up(4 * blk.size()) + up(8 * 2 * pp * NN + 8) +
                         up(8 * pp * NN + 8) + 256;
    char* base = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&base), bytes) != cudaSuccess) {
        cudaGetLastError();
        set_error(PSW_NOT_SUPPORTED, "batched setup: no room for " + std::to_string(bytes >> 20) +
                                         " MB of device scratch (create the plans one by one)");
        return PSW_NOT_SUPPORTED;
    }
    char* d = base;
    auto carve = [&](size_t b) {
        char* q = d;
        d += up(b);
        return q;
    };
    auto dplane = [&]() { return reinterpret_cast<double*>(carve(8 * nn * NN)); };
    double *tsub = dplane(), *tdiag = dplane(), *tsup = dplane();
    a.al = dplane();
    a.pv = dplane();
    a.rp = dplane();
    a.ma = dplane();
    a.w = dplane();
    a.alb = dplane();
    a.gr = dplane();
    a.gl = dplane();
    a.bg = reinterpret_cast<double*>(carve(plane * pp));
    a.az = reinterpret_cast<double*>(carve(plane * pp));
    a.bz = reinterpret_cast<double*>(carve(plane * pp));
    a.neg = reinterpret_cast<int32_t*>(carve(4 * size_t(a.nchunk) * NN));
    a.brk = reinterpret_cast<int64_t*>(carve(8 * NN));
    int64_t* dbnd = reinterpret_cast<int64_t*>(carve(8 * pp));
    int32_t* dblk = reinterpret_cast<int32_t*>(carve(4 * blk.size()));
    a.zmax = reinterpret_cast<double*>(carve(8 * 2 * pp * NN + 8));
    a.fail = reinterpret_cast<int64_t*>(carve(8 * pp * NN + 8));
    a.overflow = reinterpret_cast<int64_t*>(carve(8));
    a.sub = tsub;
    a.diag = tdiag;
    a.sup = tsup;
    a.bnd = dbnd;
    a.blk = dblk;
    a.zr = zr;
    a.zl = zl;
    int rc = PSW_OK;
    auto fail = [&](cudaError_t e, const char* what) {
        rc = cuda_fail(e, what);
        cudaFree(base);
        return rc;
    };
    cudaError_t e;
    // the host arrays go through the (not yet used) gr / gl / rp planes
    double* stage[3] = {a.gr, a.gl, a.rp};
    const double* host[3] = {sub, diag, sup};
    const size_t len[3] = {nn - 1, nn, nn - 1};
    double* dst[3] = {tsub, tdiag, tsup};
    for (int q = 0; q < 3; ++q) {
        if (len[q] == 0) continue;
        if ((e = cudaMemcpy(stage[q], host[q], 8 * len[q] * NN, cudaMemcpyHostToDevice)))
            return fail(e, "batched setup upload");
        const dim3 grid(unsigned((N + 31) / 32), unsigned((len[q] + 31) / 32));
        interleave_kernel<<<grid, dim3(32, 8)>>>(stage[q], dst[q], N, int64_t(len[q]));
    }
    if ((e = cudaMemcpy(dbnd, bnd, 8 * pp, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dblk, blk.data(), 4 * blk.size(), cudaMemcpyHostToDevice)) ||
        (e = cudaMemsetAsync(a.gr, 0, 8 * nn * NN)) || (e = cudaMemsetAsync(a.gl, 0, 8 * nn * NN)) ||
        (e = cudaMemsetAsync(zr, 0, 8 * (pp * pp + 2) * NN)) ||
        (e = cudaMemsetAsync(zl, 0, 8 * (pp * pp + 2) * NN)) ||
        (e = cudaMemsetAsync(a.overflow, 0, 8)) || (e = cudaMemsetAsync(a.fail, 0xff, 8 * pp * NN + 8)))
        return fail(e, "batched setup init");
    const unsigned gx = unsigned((N + 127) / 128);
    batch_chain_kernel<<<gx, 128>>>(a);
    batch_block_kernel<<<dim3(gx, unsigned(p + 1)), 128>>>(a);
    if (p > 0) batch_sweeps_kernel<<<dim3(gx, unsigned(p), 3), 128>>>(a);
    const dim3 ga(gx, unsigned(std::min<int64_t>(n, 1024)));
    if (dtype == PSW_F64)
        batch_assemble_kernel<double><<<ga, 128>>>(a, static_cast<FwdCoef<double>*>(fwd),
                                                   static_cast<BwdCoef<double>*>(bwd));
    else
        batch_assemble_kernel<float><<<ga, 128>>>(a, static_cast<FwdCoef<float>*>(fwd),
                                                  static_cast<BwdCoef<float>*>(bwd));
    if ((e = cudaGetLastError()) || (e = cudaDeviceSynchronize())) return fail(e, "batched setup");
    std::vector<int64_t> brk(NN), fails(pp * NN + 1);
    if ((e = cudaMemcpy(brk.data(), a.brk, 8 * NN, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(fails.data(), a.fail, 8 * pp * NN, cudaMemcpyDeviceToHost)))
        return fail(e, "batched setup download");
    cudaFree(base);
    bad_sys = bad_row = -1;
    for (size_t k = 0; k < NN && bad_row < 0; ++k) {
        if (brk[k] >= 0) bad_row = brk[k];
        for (size_t j = 0; j < pp && bad_row < 0; ++j)
            if (fails[k * pp + j] >= 0) bad_row = fails[k * pp + j];
        if (bad_row >= 0) bad_sys = int64_t(k);
    }
    return bad_row >= 0 ? PSW_PIVOT_BREAKDOWN : PSW_OK;
}

}  // namespace psw
