// RESWEEP solve path: F is read twice and X written once (3 s bytes per
// unknown instead of the STAGED path's 4 s); nothing of size n x N besides F
// and X touches HBM. Any partition; both layouts.
//
// Every block is cut into segments of kSegLen rows (the last one of a block
// takes the rest, build_fused_tables). In the affine form of the unit-row
// block sweep (psw_internal.h; local_solve.hpp:39-48 + thomas.hpp:31-44)
//   forward   d_q = f_q rp_q + ma_q d_{q-1}
//   backward  x_q = d_q + x_l w_q + al_q x_{q+1}
// a segment [a, b) swept from a zero carry (d~) is exact after
// d_q = d~_q + mu_q D_{a-1}, and its back substitution after the carry
// x_a = Lam~ + D_{a-1} K1 + x_l K2 + nu x_b (Lam~ = sum lam_q d~_q).
//
//   K1 part     one thread per (rhs k, segment): the segment's F rows (all
//               loads in flight), d~ from zero, Lam~ and the two beta dot
//               products of the segment (betas.hpp:42-57 split by segment).
//   K2 comb     per (rhs k, block t): forward fold of the segment partials
//               (exact carries D_{a-1}, block betas), boundary values V
//               (P <= 64: the tabulated combination matrix, psw_plan.cpp
//               combine_matrix; otherwise the STAGED level-order dichotomy,
//               boundary_solve.hpp:96-121), backward fold (x_b per segment).
//   K3 solve    one thread per (rhs k, segment): F rows read again, forward
//               sweep from the exact carry, back substitution from the exact
//               x_b, X streamed out.
// K3 walks the segments in the reverse of K1's order: the F rows K1 read
// last are still in L2 when K3 starts (C1: F = 128 MB, L2 = 126 MB).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "psw_device.cuh"
#include "psw_internal.h"

namespace psw {
namespace {

constexpr int kThreads = 128;
constexpr int kSegMax = kSegLen + 1;

// Scratch per (segment s, rhs k), [s * N + k]:
//   pd  K1: d~ at the segment end      -> K2: D_{a-1} (exact carry into s)
//   px  K1: Lam~                       -> K2: Lam~ + D_{a-1} K1
//   pr  K1: segment right-beta partial -> K2: x_b (x at the row after s)
//   pl  K1: segment left-beta partial
template <typename T>
struct Scratch {
    T* pd;
    T* px;
    T* pr;  // partial sums accumulated in double, stored in the solve precision
    T* pl;
    int64_t ld;  // row pitch (>= N, a multiple of 32)
};

// ------------------------------------------------------------------ K1
template <typename T>
__global__ void __launch_bounds__(kThreads) rs_part_kernel(
    const T* __restrict__ F, int64_t ldf, int64_t N, const SegDesc* __restrict__ desc,
    const FusedFwd<T>* __restrict__ ff, Scratch<T> sc) {
    __shared__ FusedFwd<T> cs[kSegMax];
    const int s = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    const bool kv = k < N;
    const SegDesc sd = desc[s];
    const int a = sd.a, len = sd.b - sd.a;
    const T* fp = F + int64_t(a) * ldf + (kv ? k : 0);
    // segments of >= 31 rows (every segment of a uniform partition) run
    // their first 31 rows unpredicated: a fully predicated 33-row sweep is
    // several times slower
    T d = T(0), lx = T(0);
    double br = 0.0, bl = 0.0;
    auto sweep = [&](auto full) {
        constexpr bool FULL = decltype(full)::value;
        T v[kSegMax];
        if (kv) {
#pragma unroll
            for (int r = 0; r < kSegMax; ++r)
                if ((FULL && r < kSegLen - 1) || r < len) v[r] = fp[int64_t(r) * ldf];
        }
        for (int i = threadIdx.x; i < len; i += kThreads) cs[i] = ff[a + i];
        __syncthreads();
        if (!kv) return;
#pragma unroll
        for (int r = 0; r < kSegMax; ++r) {
            if ((FULL && r < kSegLen - 1) || r < len) {
                const FusedFwd<T> c = cs[r];
                d = fma(c.ma, d, v[r] * c.rp);
                br = fma(double(v[r]), double(c.gr), br);
                bl = fma(double(v[r]), double(c.gl), bl);
                lx = fma(c.lam, d, lx);
            }
        }
    };
    if (len >= kSegLen - 1)
        sweep(std::true_type{});
    else
        sweep(std::false_type{});
    if (!kv) return;
    const int64_t o = int64_t(s) * sc.ld + k;
    sc.pd[o] = d;
    sc.px[o] = lx;
    sc.pr[o] = T(br);
    sc.pl[o] = T(bl);
}

// ------------------------------------------------------------------ K2
// Forward fold of block t for rhs k: exact carries and block betas.
template <typename T, int U = 8>
__device__ __forceinline__ void fold_fwd(const Scratch<T>& sc, const SegCoef* __restrict__ segc,
                                         int s0, int s1, int64_t N, int64_t k, double& R,
                                         double& L) {
    // U segments' partials in flight per thread
    double D = 0.0;
    R = 0.0;
    L = 0.0;
    for (int lo = s0; lo < s1; lo += U) {
        T dv[U], xv[U], rv[U], lv[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (lo + u < s1) {
                const int64_t o = int64_t(lo + u) * sc.ld + k;
                dv[u] = sc.pd[o];
                xv[u] = sc.px[o];
                rv[u] = sc.pr[o];
                lv[u] = sc.pl[o];
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (lo + u < s1) {
                const SegCoef c = segc[lo + u];
                const int64_t o = int64_t(lo + u) * sc.ld + k;
                sc.pd[o] = T(D);
                sc.px[o] = T(fma(D, c.k1, double(xv[u])));
                R += double(rv[u]);
                L += double(lv[u]);
                D = fma(c.mu_end, D, double(dv[u]));
            }
    }
}

// Backward fold of block t for rhs k from x at row e_t: x_b of every segment.
template <typename T>
__device__ __forceinline__ void fold_bwd(const Scratch<T>& sc, const SegCoef* __restrict__ segc,
                                         int s0, int s1, int64_t N, int64_t k, double xl,
                                         double xb) {
    constexpr int U = 8;
    for (int hi = s1; hi > s0; hi -= U) {
        T av[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (hi - 1 - u >= s0) av[u] = sc.px[int64_t(hi - 1 - u) * sc.ld + k];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int sg = hi - 1 - u;
            if (sg >= s0) {
                const SegCoef c = segc[sg];
                sc.pr[int64_t(sg) * sc.ld + k] = T(xb);
                xb = fma(c.nu, xb, fma(xl, c.k2, double(av[u])));
            }
        }
    }
}

// P <= kCombMaxP with a combination matrix: one CTA per 32 RHS, warp w
// handles blocks w, w + kCombWarps, ... in both phases; the block betas of
// the CTA's RHS meet in shared memory.
constexpr int kCombWarps = 16;
constexpr int kCombMaxP = 64;

// one boundary value: row m of the combination matrix times the betas
__device__ __forceinline__ double cmat_row(const double* __restrict__ m,
                                           const double (*sb)[32], int len, int lane) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int u = 0;
    for (; u + 4 <= len; u += 4) {
        a0 = fma(m[u], sb[u][lane], a0);
        a1 = fma(m[u + 1], sb[u + 1][lane], a1);
        a2 = fma(m[u + 2], sb[u + 2][lane], a2);
        a3 = fma(m[u + 3], sb[u + 3][lane], a3);
    }
    for (; u < len; ++u) a0 = fma(m[u], sb[u][lane], a0);
    return (a0 + a1) + (a2 + a3);
}

template <typename T>
__global__ void __launch_bounds__(kCombWarps * 32) rs_comb_kernel(
    int64_t N, int P, int p, const int32_t* __restrict__ segoff, const SegCoef* __restrict__ segc,
    const double* __restrict__ gcmat, Scratch<T> sc, double* __restrict__ V) {
    __shared__ double sb[2 * kCombMaxP][32];  // [u] right_u, [P + u] left_u
    extern __shared__ double cmat[];           // p x 2P combination matrix
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < p * 2 * P; i += blockDim.x) cmat[i] = gcmat[i];
    const int64_t k = int64_t(blockIdx.x) * 32 + lane;
    const bool kv = k < N;
    for (int t = warp; t < P; t += kCombWarps) {
        double R = 0.0, L = 0.0;
        if (kv) fold_fwd(sc, segc, segoff[t], segoff[t + 1], N, k, R, L);
        sb[t][lane] = t < p ? R : 0.0;      // betas.hpp:46-49
        sb[P + t][lane] = t > 0 ? L : 0.0;  // betas.hpp:51-55
    }
    __syncthreads();
    if (!kv) return;
    for (int t = warp; t < P; t += kCombWarps) {
        const double xl = t > 0 ? cmat_row(cmat + int64_t(t - 1) * 2 * P, sb, 2 * P, lane) : 0.0;
        const double xb = t < p ? cmat_row(cmat + int64_t(t) * 2 * P, sb, 2 * P, lane) : 0.0;
        if (t < p) V[int64_t(t) * sc.ld + k] = xb;
        fold_bwd(sc, segc, segoff[t], segoff[t + 1], N, k, xl, xb);
    }
}

// General P: the folds one thread per (rhs k, block t) around the STAGED
// combination kernel.
template <typename T>
__global__ void __launch_bounds__(kThreads) rs_fold_kernel(
    int64_t N, int p, const int32_t* __restrict__ segoff, const SegCoef* __restrict__ segc,
    Scratch<T> sc, double* __restrict__ bl, double* __restrict__ br) {
    const int t = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (k >= N) return;
    double R, L;
    // fp32: 16 segments in flight (the split fold is latency-bound: C2 comb
    // 1.39 -> 1.08 ms); fp64 keeps 8 (16 costs occupancy: C3 comb 0.47 -> 0.60 ms)
    fold_fwd<T, sizeof(T) == 4 ? 16 : 8>(sc, segc, segoff[t], segoff[t + 1], N, k, R, L);
    if (t < p) br[int64_t(t) * sc.ld + k] = R;
    if (t > 0) bl[int64_t(t) * sc.ld + k] = L;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) rs_carry_kernel(
    int64_t N, int p, const int32_t* __restrict__ segoff, const SegCoef* __restrict__ segc,
    Scratch<T> sc, const double* __restrict__ V) {
    const int t = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (k >= N) return;
    const double xl = t > 0 ? V[int64_t(t - 1) * sc.ld + k] : 0.0;
    const double xb = t < p ? V[int64_t(t) * sc.ld + k] : 0.0;
    fold_bwd(sc, segc, segoff[t], segoff[t + 1], N, k, xl, xb);
}

// Boundary values from the combination matrix, one thread per (rhs k,
// boundary j): V[j] = sum_u MR[j][u] right_u + ML[j][u] left_u
// (right_p and left_0 do not exist, betas.hpp:46-55).
__global__ void __launch_bounds__(kThreads) rs_vmat_kernel(
    int64_t N, int64_t ld, int P, int p, const double* __restrict__ cmat,
    const double* __restrict__ bl, const double* __restrict__ br, double* __restrict__ V) {
    const int j = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (k >= N) return;
    const double* m = cmat + int64_t(j) * 2 * P;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
    for (int u = 0; u < P; ++u) {
        if (u < p) a0 = fma(m[u], br[int64_t(u) * ld + k], a0);
        if (u > 0) a1 = fma(m[P + u], bl[int64_t(u) * ld + k], a1);
    }
    V[int64_t(j) * ld + k] = a0 + a1;
}

// ------------------------------------------------------------------ K3
template <typename T>
__global__ void __launch_bounds__(kThreads, 4) rs_solve_kernel(
    const T* F, int64_t ldf, T* X, int64_t ldx, int64_t N, const SegDesc* __restrict__ desc,
    const FwdCoef<T>* __restrict__ cf, const BwdCoef<T>* __restrict__ cb, Scratch<T> sc,
    const double* __restrict__ V, int NS) {
    __shared__ FwdCoef<T> csf[kSegMax];
    __shared__ BwdCoef<T> csb[kSegMax];
    const int s = NS - 1 - int(blockIdx.y);  // reverse of K1's order (L2 reuse)
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    const bool kv = k < N;
    const SegDesc sd = desc[s];
    const int a = sd.a, len = sd.b - sd.a, t = sd.t;
    const T* fp = F + int64_t(a) * ldf + (kv ? k : 0);
    auto sweep = [&](auto full) {
        constexpr bool FULL = decltype(full)::value;
        T v[kSegMax];
        if (kv) {
#pragma unroll
            for (int r = 0; r < kSegMax; ++r)
                if ((FULL && r < kSegLen - 1) || r < len) v[r] = __ldcs(fp + int64_t(r) * ldf);
        }
        for (int i = threadIdx.x; i < len; i += kThreads) {
            csf[i] = cf[a + i];
            csb[i] = cb[a + i];
        }
        __syncthreads();
        if (!kv) return;
        const int64_t o = int64_t(s) * sc.ld + k;
        T d = sc.pd[o];
        T xn = T(sc.pr[o]);
        const T xl = t > 0 ? T(V[int64_t(t - 1) * sc.ld + k]) : T(0);
#pragma unroll
        for (int r = 0; r < kSegMax; ++r) {
            if ((FULL && r < kSegLen - 1) || r < len) {
                d = fma(csf[r].ma, d, v[r] * csf[r].rp);
                v[r] = d;
            }
        }
        T* xp = X + int64_t(a) * ldx + k;
#pragma unroll
        for (int r = kSegMax - 1; r >= 0; --r) {
            if ((FULL && r < kSegLen - 1) || r < len) {
                xn = fma(csb[r].al, xn, fma(xl, csb[r].w, v[r]));
                __stcs(xp + int64_t(r) * ldx, xn);
            }
        }
    };
    if (len >= kSegLen - 1)
        sweep(std::true_type{});
    else
        sweep(std::false_type{});
}

// ------------------------------------------------------------ layout S
// F[k * ldf + i]: every RHS is contiguous. One warp per (32 RHS, segment):
// the segment's rows of its 32 RHS are loaded coalesced (cp.async, 256
// contiguous bytes per instruction) into a [rhs][row] shared tile with an
// odd row pitch (conflict-free per-lane sweeps), lane r sweeps RHS r. Four
// warps of a CTA share one segment (its coefficient rows are staged once).
constexpr int kSWarps = 4;
constexpr int kSPitch = kSegMax;  // 33: odd pitch, conflict-free column access

template <typename T>
__device__ __forceinline__ void s_tile_load(T (*tile)[kSPitch], const T* src, int64_t ld, int len,
                                            int nk, int lane) {
    // rows 0..31 by lane, row 32 (a 33-row segment) by lane = rhs
#pragma unroll 4
    for (int j = 0; j < 32; ++j)
        if (j < nk && lane < len) {
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tile[j][lane]));
            asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst),
                         "l"(src + int64_t(j) * ld + lane), "n"(sizeof(T))
                         : "memory");
        }
    if (len > 32 && lane < nk) {
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tile[lane][32]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst),
                     "l"(src + int64_t(lane) * ld + 32), "n"(sizeof(T))
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <typename T>
__global__ void __launch_bounds__(kSWarps * 32) rs_part_s_kernel(
    const T* __restrict__ F, int64_t ldf, int64_t N, const SegDesc* __restrict__ desc,
    const FusedFwd<T>* __restrict__ ff, Scratch<T> sc) {
    __shared__ T tiles[kSWarps][32][kSPitch];
    __shared__ FusedFwd<T> cs[kSegMax];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.y;
    const int64_t k0 = (int64_t(blockIdx.x) * kSWarps + warp) * 32;
    const int nk = k0 < N ? int(N - k0 < 32 ? N - k0 : 32) : 0;
    const SegDesc sd = desc[s];
    const int a = sd.a, len = sd.b - sd.a;
    if (nk > 0) s_tile_load(tiles[warp], F + k0 * ldf + a, ldf, len, nk, lane);
    for (int i = threadIdx.x; i < len; i += kSWarps * 32) cs[i] = ff[a + i];
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (lane >= nk) return;
    const T* col = tiles[warp][lane];
    T d = T(0), lx = T(0);
    double br = 0.0, bl = 0.0;
    auto sweep = [&](auto full) {
        constexpr bool FULL = decltype(full)::value;
#pragma unroll
        for (int r = 0; r < kSegMax; ++r) {
            if ((FULL && r < kSegLen - 1) || r < len) {
                const FusedFwd<T> c = cs[r];
                const T f = col[r];
                d = fma(c.ma, d, f * c.rp);
                br = fma(double(f), double(c.gr), br);
                bl = fma(double(f), double(c.gl), bl);
                lx = fma(c.lam, d, lx);
            }
        }
    };
    if (len >= kSegLen - 1)
        sweep(std::true_type{});
    else
        sweep(std::false_type{});
    const int64_t o = int64_t(s) * sc.ld + k0 + lane;
    sc.pd[o] = d;
    sc.px[o] = lx;
    sc.pr[o] = T(br);
    sc.pl[o] = T(bl);
}

template <typename T>
__global__ void __launch_bounds__(kSWarps * 32) rs_solve_s_kernel(
    const T* F, int64_t ldf, T* X, int64_t ldx, int64_t N, const SegDesc* __restrict__ desc,
    const FwdCoef<T>* __restrict__ cf, const BwdCoef<T>* __restrict__ cb, Scratch<T> sc,
    const double* __restrict__ V, int NS) {
    __shared__ T tiles[kSWarps][32][kSPitch];
    __shared__ FwdCoef<T> csf[kSegMax];
    __shared__ BwdCoef<T> csb[kSegMax];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = NS - 1 - int(blockIdx.y);  // reverse of K1's order (L2 reuse)
    const int64_t k0 = (int64_t(blockIdx.x) * kSWarps + warp) * 32;
    const int nk = k0 < N ? int(N - k0 < 32 ? N - k0 : 32) : 0;
    const SegDesc sd = desc[s];
    const int a = sd.a, len = sd.b - sd.a, t = sd.t;
    if (nk > 0) s_tile_load(tiles[warp], F + k0 * ldf + a, ldf, len, nk, lane);
    for (int i = threadIdx.x; i < len; i += kSWarps * 32) {
        csf[i] = cf[a + i];
        csb[i] = cb[a + i];
    }
    T d = T(0), xn = T(0), xl = T(0);
    if (lane < nk) {  // the carries' loads overlap the tile's
        const int64_t o = int64_t(s) * sc.ld + k0 + lane;
        d = sc.pd[o];
        xn = T(sc.pr[o]);
        if (t > 0) xl = T(V[int64_t(t - 1) * sc.ld + k0 + lane]);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (nk == 0) return;
    T* col = tiles[warp][lane];
    auto sweep = [&](auto full) {
        constexpr bool FULL = decltype(full)::value;
#pragma unroll
        for (int r = 0; r < kSegMax; ++r) {
            if ((FULL && r < kSegLen - 1) || r < len) {
                d = fma(csf[r].ma, d, col[r] * csf[r].rp);
                col[r] = d;
            }
        }
#pragma unroll
        for (int r = kSegMax - 1; r >= 0; --r) {
            if ((FULL && r < kSegLen - 1) || r < len) {
                xn = fma(csb[r].al, xn, fma(xl, csb[r].w, col[r]));
                col[r] = xn;
            }
        }
    };
    if (lane < nk) {
        if (len >= kSegLen - 1)
            sweep(std::true_type{});
        else
            sweep(std::false_type{});
    }
    __syncwarp();
    // coalesced write-back: RHS j's rows by lane (row 32 by lane = rhs)
    T* dst = X + k0 * ldx + a;
#pragma unroll 4
    for (int j = 0; j < 32; ++j)
        if (j < nk && lane < len) __stcs(dst + int64_t(j) * ldx + lane, tiles[warp][j][lane]);
    if (len > 32 && lane < nk) __stcs(dst + int64_t(lane) * ldx + 32, tiles[warp][lane][32]);
}

template <typename T>
int launch_resweep(const psw_plan* pl, const void* Fv, int64_t ldf, void* Xv, int64_t ldx,
                   int64_t N, int layout, cudaStream_t s, void** ev, int nev) {
    const T* F = static_cast<const T*>(Fv);
    T* X = static_cast<T*>(Xv);
    const int P = int(pl->P), p = int(pl->p);
    const int NS = pl->seg_off.back();
    const int64_t ld = (N + 31) / 32 * 32;  // scratch row pitch
    const size_t sn = size_t(NS) * size_t(ld);
    const size_t need = sn * 4 * sizeof(T) +
                        sizeof(double) * size_t(ld) * (2 * size_t(P) + size_t(std::max(p, 1))) + 256;
    void* scratch = nullptr;
    PSW_CUDA_TRY(cudaMallocAsync(&scratch, need, s));
    char* c = static_cast<char*>(scratch);
    Scratch<T> sc;
    sc.ld = ld;
    double* bl = reinterpret_cast<double*>(c);
    double* br = bl + size_t(P) * ld;
    double* V = br + size_t(P) * ld;
    sc.pr = reinterpret_cast<T*>(V + size_t(std::max(p, 1)) * ld);
    sc.pl = sc.pr + sn;
    sc.pd = sc.pl + sn;
    sc.px = sc.pd + sn;
    const unsigned gx = unsigned((N + kThreads - 1) / kThreads);
    const auto* desc = pl->d_segdesc;
    const unsigned gs = unsigned((N + kSWarps * 32 - 1) / (kSWarps * 32));
    mark(ev, nev, 0, s);
    if (layout == PSW_LAYOUT_S)
        rs_part_s_kernel<T><<<dim3(gs, unsigned(NS)), kSWarps * 32, 0, s>>>(
            F, ldf, N, desc, static_cast<const FusedFwd<T>*>(pl->d_ffwd), sc);
    else
        rs_part_kernel<T><<<dim3(gx, unsigned(NS)), kThreads, 0, s>>>(
            F, ldf, N, desc, static_cast<const FusedFwd<T>*>(pl->d_ffwd), sc);
    mark(ev, nev, 1, s);
    int64_t launches = 1;
    // fused fold + combination + carries when there are enough 32-RHS CTAs
    // to fill the GPU, otherwise one kernel per step over (rhs, block) threads
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pl->device);
    const bool cm = pl->d_cmat && P <= kCombMaxP;
    static const int fused_comb = [] {  // PSW_RESWEEP_COMB=0: always the split kernels
        const char* e = std::getenv("PSW_RESWEEP_COMB");
        return e ? std::atoi(e) : 1;
    }();
    if (cm && fused_comb && (N + 31) / 32 >= nsm / 2 && int64_t(NS) * 4 <= 512) {
        const size_t cmb = sizeof(double) * size_t(p) * 2 * P;
        PSW_CUDA_TRY(cudaFuncSetAttribute(rs_comb_kernel<T>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(cmb)));
        rs_comb_kernel<T><<<unsigned((N + 31) / 32), kCombWarps * 32, cmb, s>>>(
            N, P, p, pl->d_segoff, pl->d_seg, pl->d_cmat, sc, V);
        ++launches;
    } else {
        rs_fold_kernel<T><<<dim3(gx, unsigned(P)), kThreads, 0, s>>>(N, p, pl->d_segoff,
                                                                     pl->d_seg, sc, bl, br);
        ++launches;
        if (p > 0 && cm) {
            rs_vmat_kernel<<<dim3(gx, unsigned(p)), kThreads, 0, s>>>(N, ld, P, p, pl->d_cmat, bl,
                                                                      br, V);
            ++launches;
        } else if (p > 0) {
            // the combination runs over the padded pitch (columns >= N unused)
            int rc = launch_combine(pl, bl, br, ld, V, s);
            if (rc != PSW_OK) {
                cudaFreeAsync(scratch, s);
                return rc;
            }
            ++launches;
        }
        rs_carry_kernel<T><<<dim3(gx, unsigned(P)), kThreads, 0, s>>>(N, p, pl->d_segoff,
                                                                      pl->d_seg, sc, V);
        ++launches;
    }
    mark(ev, nev, 2, s);
    if (layout == PSW_LAYOUT_S)
        rs_solve_s_kernel<T><<<dim3(gs, unsigned(NS)), kSWarps * 32, 0, s>>>(
            F, ldf, X, ldx, N, desc, static_cast<const FwdCoef<T>*>(pl->d_fwd),
            static_cast<const BwdCoef<T>*>(pl->d_bwd), sc, V, NS);
    else
        rs_solve_kernel<T><<<dim3(gx, unsigned(NS)), kThreads, 0, s>>>(
            F, ldf, X, ldx, N, desc, static_cast<const FwdCoef<T>*>(pl->d_fwd),
            static_cast<const BwdCoef<T>*>(pl->d_bwd), sc, V, NS);
    ++launches;
    mark(ev, nev, 3, s);
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(scratch, s);
    if (e != cudaSuccess) return cuda_fail(e, "resweep kernels");
    note_launches(launches);
    return PSW_OK;
}

}  // namespace

bool resweep_supported(const psw_plan* pl, int layout, int64_t N) {
    if (pl->world != 1 || (layout != PSW_LAYOUT_R && layout != PSW_LAYOUT_S) || N < 1) return false;
    if (!pl->d_segdesc || !pl->d_ffwd || pl->seg_off.empty()) return false;
    return pl->seg_off.back() < 65536 && pl->P < 65536;  // grid.y
}

int solve_resweep(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                  int layout, cudaStream_t s, void** ev, int nev) {
    return pl->dtype == PSW_F64 ? launch_resweep<double>(pl, F, ldf, X, ldx, N, layout, s, ev, nev)
                                : launch_resweep<float>(pl, F, ldf, X, ldx, N, layout, s, ev, nev);
}

}  // namespace psw
