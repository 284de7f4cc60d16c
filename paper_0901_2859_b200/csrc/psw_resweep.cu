// RESWEEP solve path: F is read twice and X written once (3 s bytes per
// unknown; the intermediates are a few aggregates per 256 rows), any
// partition, both layouts. The same kernels serve three drivers:
//   solve_resweep   all RHS at once (the 2^20-row config C3: one 16-RHS
//                   column of F is 128 MB, no single-read scheme fits on chip)
//   shard_forward / shard_backward   a rank's own blocks of a row-sharded
//                   solve (psw_shard.cpp), around one all-reduce
//
// Every block is cut into segments of kSegLen rows (the last one of a block
// takes the rest, build_fused_tables). In the affine form of the unit-row
// block sweep (psw_internal.h; local_solve.hpp:39-48 + thomas.hpp:31-44)
//   forward   d_q = f_q rp_q + ma_q d_{q-1}
//   backward  x_q = d_q + x_l w_q + al_q x_{q+1}
// a segment [a, b) swept from a zero carry (d~) is exact after
// d_q = d~_q + mu_q D_{a-1}, and its back substitution after the carry
// x_a = Lam~ + D_{a-1} K1 + x_l K2 + nu x_b (Lam~ = sum lam_q d~_q).
// A CTA ("group") takes kRsSeg consecutive segments x 32 RHS (warp = segment,
// lane = RHS); the part of a group inside one block is a "run", whose
// segments compose into one affine map of the same form (run SegCoef).
//
//   K1 part    the group's F rows (all loads in flight), d~ from zero, Lam~
//              and the two beta dot products per segment (betas.hpp:42-57
//              split by segment); one warp per run folds its segments:
//              run d~ end, run Lam, run beta partials -> scratch.
//   K2         per (RHS, block): forward fold over the block's runs (exact
//              run carries D_in, block betas), boundary values V (P <= 64:
//              the tabulated combination matrix, psw_plan.cpp
//              combine_matrix; otherwise the STAGED level-order dichotomy,
//              boundary_solve.hpp:96-121), backward fold (x at every run's end).
//   K3 solve   F rows read again, d~ from zero, one warp per run rebuilds
//              the exact segment carries from the run's (D_in, x_B), back
//              substitution, X streamed out. Groups in the reverse of K1's
//              order (the rows K1 read last are the likeliest L2 hits).
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "psw_device.cuh"
#include "psw_internal.h"
#include "psw_tma.cuh"

namespace psw {
namespace {

constexpr int kRsThreads = kRsSeg * 32;
constexpr int kRsMinBlocks = 512 / kRsThreads;  // 16 warps per SM
constexpr int kSegMax = kSegLen + 1;
constexpr int kRsRows = kRsSeg * kSegMax;  // coefficient rows staged per group (bound)
constexpr int kSPitch = kSegMax;           // layout S tile pitch (odd: conflict-free columns)
constexpr int kTmaRows = 256;              // rows per group at most (one TMA stage)

// Per (run r, rhs k), [r * ld + k], all fp64:
//   dt   K1: run d~ end (zero carry)  -> K2: D_in (exact carry into the run)
//   lam  K1: run Lam (zero D_in, x_l, x_B)
//   br   K1: run right-beta partial   -> K2: x_B (x at the row after the run)
//   bl   K1: run left-beta partial
struct RsScratch {
    double* dt;
    double* lam;
    double* br;
    double* bl;
    int64_t ld;
};

template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
    return __ldcs(p);
}

// layout S: the rows [a, a+len) of RHS k0..k0+nk-1 into tile[rhs][row]
// (cp.async, 32 consecutive rows of one RHS per instruction)
template <typename T>
__device__ __forceinline__ void s_tile_load(T (*tile)[kSPitch], const T* src, int64_t ld, int len,
                                            int nk, int lane) {
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

// row r of a segment of length len is swept: the first kSegLen - 1 rows
// unpredicated when the segment is full length (every segment of a uniform
// partition: 31, 32 or 33 rows), else row by row
template <bool FULL>
__device__ __forceinline__ bool row_on(int r, int len) {
    return (FULL && r < kSegLen - 1) || r < len;
}

// ------------------------------------------------------------------ K1
template <typename T, bool LS>
__global__ void __launch_bounds__(kRsThreads, kRsMinBlocks) rs_part_kernel(
    const T* __restrict__ F, int64_t ldf, int64_t N, int32_t row0,
    const RsGroup* __restrict__ groups, const RsRun* __restrict__ runs,
    const SegDesc* __restrict__ desc, const SegCoef* __restrict__ segc,
    const FusedFwd<T>* __restrict__ ff, RsScratch sc) {
    __shared__ FusedFwd<T> cs[kRsRows];
    __shared__ SegCoef s_sc[kRsSeg];
    __shared__ double s_d[kRsSeg][32], s_l[kRsSeg][32], s_r[kRsSeg][32], s_b[kRsSeg][32];
    extern __shared__ __align__(16) unsigned char dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const RsGroup g = groups[blockIdx.y];
    const int64_t k0 = int64_t(blockIdx.x) * 32;
    const int64_t k = k0 + lane;
    const int nk = int(N - k0 < 32 ? N - k0 : 32);
    const bool kv = lane < nk;
    const int sg = g.s0 + warp;
    const bool sv = sg < g.s1;
    int a = g.ra, len = 0;
    if (sv) {
        const SegDesc d = desc[sg];
        a = d.a;
        len = d.b - d.a;
    }
    T v[kSegMax];
    T(*tile)[kSPitch] = reinterpret_cast<T(*)[kSPitch]>(dyn) + warp * 32;
    if constexpr (LS) {
        if (sv) s_tile_load(tile, F + k0 * ldf + (a - row0), ldf, len, nk, lane);
    } else if (kv && sv) {
        const T* fp = F + int64_t(a - row0) * ldf + k;
        if (len >= kSegLen - 1) {
#pragma unroll
            for (int r = 0; r < kSegMax; ++r)
                if (row_on<true>(r, len)) v[r] = fp[int64_t(r) * ldf];
        } else {
#pragma unroll
            for (int r = 0; r < kSegMax; ++r)
                if (row_on<false>(r, len)) v[r] = fp[int64_t(r) * ldf];
        }
    }
    for (int i = threadIdx.x; i < g.rb - g.ra; i += kRsThreads) cs[i] = ff[g.ra + i];
    if (threadIdx.x < g.s1 - g.s0) s_sc[threadIdx.x] = segc[g.s0 + threadIdx.x];
    if constexpr (LS) asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    T d = T(0), lx = T(0);
    double br = 0.0, bl = 0.0;
    if (kv && sv) {
        const FusedFwd<T>* c = cs + (a - g.ra);
        auto sweep = [&](auto full) {
            constexpr bool FULL = decltype(full)::value;
#pragma unroll
            for (int r = 0; r < kSegMax; ++r) {
                if (row_on<FULL>(r, len)) {
                    const FusedFwd<T> q = c[r];
                    const T f = LS ? tile[lane][r] : v[r];
                    d = fma(q.ma, d, f * q.rp);
                    br = fma(double(f), double(q.gr), br);
                    bl = fma(double(f), double(q.gl), bl);
                    lx = fma(q.lam, d, lx);
                }
            }
        };
        if (len >= kSegLen - 1)
            sweep(std::true_type{});
        else
            sweep(std::false_type{});
    }
    s_d[warp][lane] = double(d);
    s_l[warp][lane] = double(lx);
    s_r[warp][lane] = br;
    s_b[warp][lane] = bl;
    __syncthreads();
    const int run = g.r0 + warp;
    if (run < g.r1 && kv) {
        const RsRun rr = runs[run];
        double D = 0.0, lam = 0.0, nupre = 1.0, R = 0.0, L = 0.0;
        for (int s = rr.s0; s < rr.s1; ++s) {
            const int j = s - g.s0;
            const SegCoef q = s_sc[j];
            lam = fma(nupre, fma(D, q.k1, s_l[j][lane]), lam);
            D = fma(q.mu_end, D, s_d[j][lane]);
            nupre *= q.nu;
            R += s_r[j][lane];
            L += s_b[j][lane];
        }
        const int64_t o = int64_t(run) * sc.ld + k;
        sc.dt[o] = D;
        sc.lam[o] = lam;
        sc.br[o] = R;
        sc.bl[o] = L;
    }
}

// ------------------------------------------------------------------ K2
// Forward fold of one block's runs [r0, r1) for rhs k: the exact carry into
// every run (stored in place of its d~ end) and the block betas.
__device__ __forceinline__ void fold_fwd(const RsScratch& sc, const SegCoef* __restrict__ rc,
                                         int r0, int r1, int64_t k, double& R, double& L) {
    constexpr int U = 8;  // runs' partials in flight per thread
    double D = 0.0;
    R = 0.0;
    L = 0.0;
    for (int lo = r0; lo < r1; lo += U) {
        double dv[U], rv[U], lv[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (lo + u < r1) {
                const int64_t o = int64_t(lo + u) * sc.ld + k;
                dv[u] = sc.dt[o];
                rv[u] = sc.br[o];
                lv[u] = sc.bl[o];
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (lo + u < r1) {
                sc.dt[int64_t(lo + u) * sc.ld + k] = D;
                R += rv[u];
                L += lv[u];
                D = fma(rc[lo + u].mu_end, D, dv[u]);
            }
    }
}

// Backward fold of one block's runs from x at the block's closing row (x_b)
// with the block's left boundary value xl: x at the end of every run.
__device__ __forceinline__ void fold_bwd(const RsScratch& sc, const SegCoef* __restrict__ rc,
                                         int r0, int r1, int64_t k, double xl, double xb) {
    constexpr int U = 8;
    for (int hi = r1; hi > r0; hi -= U) {
        double lv[U], dv[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (hi - 1 - u >= r0) {
                const int64_t o = int64_t(hi - 1 - u) * sc.ld + k;
                lv[u] = sc.lam[o];
                dv[u] = sc.dt[o];
            }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = hi - 1 - u;
            if (r >= r0) {
                const SegCoef q = rc[r];
                sc.br[int64_t(r) * sc.ld + k] = xb;
                xb = fma(q.nu, xb, fma(xl, q.k2, fma(dv[u], q.k1, lv[u])));
            }
        }
    }
}

// P <= kCombMaxP with a combination matrix (whole-system plans): one CTA per
// 32 RHS, warp w handles blocks w, w + kCombWarps, ... in both phases; the
// block betas of the CTA's RHS meet in shared memory.
constexpr int kCombWarps = 16;
constexpr int kCombMaxP = 64;

__device__ __forceinline__ double cmat_row(const double* __restrict__ m, const double (*sb)[32],
                                           int len, int lane) {
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

__global__ void __launch_bounds__(kCombWarps * 32) rs_comb_kernel(
    int64_t N, int P, int p, const int32_t* __restrict__ runoff, const SegCoef* __restrict__ rc,
    const double* __restrict__ gcmat, RsScratch sc, double* __restrict__ V, int64_t ldv) {
    __shared__ double sb[2 * kCombMaxP][32];  // [u] right_u, [P + u] left_u
    extern __shared__ double cmat[];           // p x 2P combination matrix
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < p * 2 * P; i += blockDim.x) cmat[i] = gcmat[i];
    const int64_t k = int64_t(blockIdx.x) * 32 + lane;
    const bool kv = k < N;
    for (int t = warp; t < P; t += kCombWarps) {
        double R = 0.0, L = 0.0;
        if (kv) fold_fwd(sc, rc, runoff[t], runoff[t + 1], k, R, L);
        sb[t][lane] = t < p ? R : 0.0;      // betas.hpp:46-49
        sb[P + t][lane] = t > 0 ? L : 0.0;  // betas.hpp:51-55
    }
    __syncthreads();
    if (!kv) return;
    for (int t = warp; t < P; t += kCombWarps) {
        const double xl = t > 0 ? cmat_row(cmat + int64_t(t - 1) * 2 * P, sb, 2 * P, lane) : 0.0;
        const double xb = t < p ? cmat_row(cmat + int64_t(t) * 2 * P, sb, 2 * P, lane) : 0.0;
        if (t < p) V[int64_t(t) * ldv + k] = xb;
        fold_bwd(sc, rc, runoff[t], runoff[t + 1], k, xl, xb);
    }
}

// General P and row shards: the folds one thread per (rhs k, own block tl)
// around the combination. Betas land at [tl * ld + k].
__global__ void __launch_bounds__(128) rs_fold_kernel(int64_t N, const int32_t* __restrict__ runoff,
                                                      const SegCoef* __restrict__ rc, RsScratch sc,
                                                      double* __restrict__ bl,
                                                      double* __restrict__ br) {
    const int tl = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * 128 + threadIdx.x;
    pdl_trigger();
    pdl_wait();  // K1's run aggregates
    if (k >= N) return;
    double R, L;
    fold_fwd(sc, rc, runoff[tl], runoff[tl + 1], k, R, L);
    br[int64_t(tl) * sc.ld + k] = R;
    bl[int64_t(tl) * sc.ld + k] = L;
}

__global__ void __launch_bounds__(128) rs_carry_kernel(int64_t N, int p, int t0,
                                                       const int32_t* __restrict__ runoff,
                                                       const SegCoef* __restrict__ rc,
                                                       RsScratch sc, const double* __restrict__ V,
                                                       int64_t ldv) {
    const int tl = blockIdx.y, t = t0 + tl;
    const int64_t k = int64_t(blockIdx.x) * 128 + threadIdx.x;
    pdl_trigger();
    pdl_wait();  // the boundary values
    if (k >= N) return;
    const double xl = t > 0 ? V[int64_t(t - 1) * ldv + k] : 0.0;
    const double xb = t < p ? V[int64_t(t) * ldv + k] : 0.0;
    fold_bwd(sc, rc, runoff[tl], runoff[tl + 1], k, xl, xb);
}

// Whole-system boundary values V = MR right + ML left (P <= kCombMaxP): CTA
// (x, y) forms rows 32y .. 32y + 31 of V for 64 RHS. The CTA's betas and its
// 32 combination-matrix rows are staged in shared memory first (all loads in
// flight); warp w then forms rows 32y + 4w .. 32y + 4w + 3 for RHS k0 + lane
// and k0 + 32 + lane, each beta loaded once for the warp's four rows and each
// matrix quadruple (one broadcast 32-byte load) once for its two RHS: 16
// shared loads per 32 FMAs (cmat_row's one per FMA made the kernel
// shared-load bound, 266 us on C2). Every V entry is summed exactly as
// cmat_row sums it (four interleaved partial sums over u, (a0 + a1) + (a2 + a3)).
constexpr int kVmatRows = 32;
constexpr int kVmatRhs = 64;
__global__ void __launch_bounds__(256) rs_vmat_kernel(int64_t N, int64_t ld, int P, int p,
                                                      const double* __restrict__ gcmat,
                                                      const double* __restrict__ bl,
                                                      const double* __restrict__ br,
                                                      double* __restrict__ V, int64_t ldv) {
    extern __shared__ __align__(16) double sbv[];  // [2P][64] betas: right_u, left_u; [32][2P] rows
    double* sm = sbv + 2 * P * kVmatRhs;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t k0 = int64_t(blockIdx.x) * kVmatRhs;
    const int j0 = int(blockIdx.y) * kVmatRows;
    const int nj = min(kVmatRows, p - j0);
    const int len = 2 * P;
    for (int i = threadIdx.x; i < kVmatRows * len; i += blockDim.x)
        sm[i] = i < nj * len ? gcmat[int64_t(j0) * len + i] : 0.0;
    pdl_trigger();
    pdl_wait();  // the folds' block betas
    for (int i = threadIdx.x; i < len * kVmatRhs; i += blockDim.x) {
        const int u = i / kVmatRhs, l = i % kVmatRhs;
        const int64_t k = k0 + l;
        double v = 0.0;
        if (k < N) {
            if (u < P)
                v = u < p ? br[int64_t(u) * ld + k] : 0.0;  // betas.hpp:46-49
            else
                v = u - P > 0 ? bl[int64_t(u - P) * ld + k] : 0.0;  // betas.hpp:51-55
        }
        sbv[i] = v;
    }
    __syncthreads();
    double acc[4][2][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[r][c][q] = 0.0;
    const double* mrow = sm + (4 * warp) * len;
    int u = 0;
    for (; u + 4 <= len; u += 4) {
        double b[2][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            b[0][q] = sbv[(u + q) * kVmatRhs + lane];
            b[1][q] = sbv[(u + q) * kVmatRhs + 32 + lane];
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double2 m01 = *reinterpret_cast<const double2*>(mrow + r * len + u);
            const double2 m23 = *reinterpret_cast<const double2*>(mrow + r * len + u + 2);
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                acc[r][c][0] = fma(m01.x, b[c][0], acc[r][c][0]);
                acc[r][c][1] = fma(m01.y, b[c][1], acc[r][c][1]);
                acc[r][c][2] = fma(m23.x, b[c][2], acc[r][c][2]);
                acc[r][c][3] = fma(m23.y, b[c][3], acc[r][c][3]);
            }
        }
    }
    for (; u < len; ++u)  // len % 4 == 2 (odd P): the tail into the first partial sum
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c)
                acc[r][c][0] = fma(mrow[r * len + u], sbv[u * kVmatRhs + 32 * c + lane], acc[r][c][0]);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int jj = 4 * warp + r;
        if (jj >= nj) break;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int64_t k = k0 + 32 * c + lane;
            if (k < N)
                V[int64_t(j0 + jj) * ldv + k] = (acc[r][c][0] + acc[r][c][1]) + (acc[r][c][2] + acc[r][c][3]);
        }
    }
}

// Row shards: the rank's share of every boundary value, one thread per
// (rhs k, boundary j): V_r[j] = sum over own blocks t of MR[j][t] right_t +
// ML[j][t] left_t (right_p and left_0 do not exist, betas.hpp:46-55).
__global__ void __launch_bounds__(128) rs_vpart_kernel(int64_t N, int64_t ld, int P, int p, int t0,
                                                       int nb, const double* __restrict__ cmat,
                                                       const double* __restrict__ bl,
                                                       const double* __restrict__ br,
                                                       double* __restrict__ out, int64_t ldo) {
    const int j = blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * 128 + threadIdx.x;
    if (k >= N) return;
    const double* m = cmat + int64_t(j) * 2 * P;
    double a0 = 0.0, a1 = 0.0;
    for (int tl = 0; tl < nb; ++tl) {
        const int t = t0 + tl;
        if (t < p) a0 = fma(m[t], br[int64_t(tl) * ld + k], a0);
        if (t > 0) a1 = fma(m[P + t], bl[int64_t(tl) * ld + k], a1);
    }
    out[int64_t(j) * ldo + k] = a0 + a1;
}

// ------------------------------------------------------------------ K3
template <typename T, bool LS, bool STREAM>
__global__ void __launch_bounds__(kRsThreads, kRsMinBlocks) rs_solve_kernel(
    const T* F, int64_t ldf, T* X, int64_t ldx, int64_t N, int32_t row0, int ngroups,
    const RsGroup* __restrict__ groups, const RsRun* __restrict__ runs,
    const SegDesc* __restrict__ desc, const SegCoef* __restrict__ segc,
    const SolveCoef<T>* __restrict__ sco, const CarryW* __restrict__ cw, RsScratch sc,
    const double* __restrict__ V, int64_t ldv) {
    __shared__ SolveCoef<T> cs[kRsRows];
    __shared__ CarryW s_cw[kRsSeg];
    __shared__ double s_d[kRsSeg][32], s_l[kRsSeg][32];
    extern __shared__ __align__(16) unsigned char dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = ngroups - 1 - int(blockIdx.y);  // reverse of K1's order
    const RsGroup g = groups[gi];
    const int64_t k0 = int64_t(blockIdx.x) * 32;
    const int64_t k = k0 + lane;
    const int nk = int(N - k0 < 32 ? N - k0 : 32);
    const bool kv = lane < nk;
    const int sg = g.s0 + warp;
    const bool sv = sg < g.s1;
    int a = g.ra, len = 0, t = 0;
    if (sv) {
        const SegDesc d = desc[sg];
        a = d.a;
        len = d.b - d.a;
        t = d.t;
    }
    // everything the carry phase needs is requested before F: the run's
    // (D_in, x_B) and left boundary value (= this segment's x_l)
    double rD = 0.0, rx = 0.0, rxl = 0.0;
    if (sv && kv) {
        const int64_t o = int64_t(g.r0 + (t - g.t0)) * sc.ld + k;
        rD = sc.dt[o];
        rx = sc.br[o];
        rxl = t > 0 ? V[int64_t(t - 1) * ldv + k] : 0.0;
    }
    const T xl = T(rxl);
    T v[kSegMax];
    T(*tile)[kSPitch] = reinterpret_cast<T(*)[kSPitch]>(dyn) + warp * 32;
    if constexpr (LS) {
        if (sv) s_tile_load(tile, F + k0 * ldf + (a - row0), ldf, len, nk, lane);
    } else if (kv && sv) {
        const T* fp = F + int64_t(a - row0) * ldf + k;
        if (len >= kSegLen - 1) {
#pragma unroll
            for (int r = 0; r < kSegMax; ++r)
                if (row_on<true>(r, len)) v[r] = STREAM ? ld_stream(fp + int64_t(r) * ldf) : fp[int64_t(r) * ldf];
        } else {
#pragma unroll
            for (int r = 0; r < kSegMax; ++r)
                if (row_on<false>(r, len)) v[r] = STREAM ? ld_stream(fp + int64_t(r) * ldf) : fp[int64_t(r) * ldf];
        }
    }
    for (int i = threadIdx.x; i < g.rb - g.ra; i += kRsThreads) cs[i] = sco[g.ra + i];
    for (int i = threadIdx.x; i < (g.s1 - g.s0) * int(sizeof(CarryW) / 8); i += kRsThreads)
        reinterpret_cast<double*>(s_cw)[i] = reinterpret_cast<const double*>(cw + int64_t(gi) * kRsSeg)[i];
    if constexpr (LS) asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const SolveCoef<T>* c = cs + (a - g.ra);
    const bool on = kv && sv;
    // forward from a zero carry, d~ in place of f
    T d = T(0), lx = T(0);
    auto fwd = [&](auto full) {
        constexpr bool FULL = decltype(full)::value;
#pragma unroll
        for (int r = 0; r < kSegMax; ++r) {
            if (row_on<FULL>(r, len)) {
                const SolveCoef<T> q = c[r];
                const T f = LS ? tile[lane][r] : v[r];
                d = fma(q.ma, d, f * q.rp);
                lx = fma(q.lam, d, lx);
                if (LS)
                    tile[lane][r] = d;
                else
                    v[r] = d;
            }
        }
    };
    if (on) {
        if (len >= kSegLen - 1)
            fwd(std::true_type{});
        else
            fwd(std::false_type{});
    }
    s_d[warp][lane] = double(d);
    s_l[warp][lane] = double(lx);
    __syncthreads();
    // the segment's exact carries in closed form over its run (CarryW, as
    // rs_solve_tma: both kernels round alike)
    double dc = 0.0, xc = 0.0;
    if (on) {
        const CarryW& q = s_cw[warp];
        const int ns = g.s1 - g.s0;
        dc = q.P * rD;
        xc = fma(q.Q, rx, fma(q.K2, rxl, q.K1 * rD));
#pragma unroll
        for (int i = 0; i < kRsSeg; ++i)
            if (i < ns) {
                const double dd = s_d[i][lane];
                dc = fma(q.A[i], dd, dc);
                xc = fma(q.C[i], dd, fma(q.B[i], s_l[i][lane], xc));
            }
    }
    if (on) {
        const T D = T(dc);
        T x = T(xc);
        T* xp = X + int64_t(a - row0) * ldx + k;
        auto bwd = [&](auto full) {
            constexpr bool FULL = decltype(full)::value;
#pragma unroll
            for (int r = kSegMax - 1; r >= 0; --r) {
                if (row_on<FULL>(r, len)) {
                    const SolveCoef<T> q = c[r];
                    const T dq = fma(q.mu, D, LS ? tile[lane][r] : v[r]);
                    x = fma(q.al, x, fma(xl, q.w, dq));
                    if (LS)
                        tile[lane][r] = x;
                    else
                        __stcs(xp + int64_t(r) * ldx, x);
                }
            }
        };
        if (len >= kSegLen - 1)
            bwd(std::true_type{});
        else
            bwd(std::false_type{});
    }
    if constexpr (LS) {
        __syncwarp();
        if (sv) {  // coalesced write-back: RHS j's rows by lane (row 32 by lane = rhs)
            T* dst = X + k0 * ldx + (a - row0);
#pragma unroll 4
            for (int j = 0; j < 32; ++j)
                if (j < nk && lane < len) __stcs(dst + int64_t(j) * ldx + lane, tile[j][lane]);
            if (len > 32 && lane < nk) __stcs(dst + int64_t(lane) * ldx + 32, tile[lane][32]);
        }
    }
}

// ------------------------------------------------------------------ host
struct Work {
    RsScratch sc;
    double* bl;  // own blocks x ld
    double* br;
    double* V;   // p x ldv (whole-system solves; shards pass their own)
    int64_t ldv;
};

int64_t pad64(int64_t N) { return (N + 63) / 64 * 64; }  // a whole TMA chunk of fp32 RHS

size_t work_bytes(const psw_plan* pl, int64_t N, bool withV) {
    const int64_t ld = pad64(N);
    const int64_t nb = pl->blk1 - pl->blk0;
    size_t b = sizeof(double) * size_t(ld) * (4 * size_t(pl->rs_nruns) + 2 * size_t(nb));
    if (withV) b += sizeof(double) * size_t(ld) * size_t(std::max<int64_t>(pl->p, 1));
    return b + 256;
}

Work carve(const psw_plan* pl, int64_t N, void* mem, bool withV) {
    const int64_t ld = pad64(N);
    const int64_t nb = pl->blk1 - pl->blk0;
    double* c = static_cast<double*>(mem);
    Work w;
    w.sc.ld = ld;
    const size_t rn = size_t(pl->rs_nruns) * size_t(ld);
    w.sc.dt = c;
    w.sc.lam = c + rn;
    w.sc.br = c + 2 * rn;
    w.sc.bl = c + 3 * rn;
    w.bl = c + 4 * rn;
    w.br = w.bl + size_t(nb) * size_t(ld);
    w.V = withV ? w.br + size_t(nb) * size_t(ld) : nullptr;
    w.ldv = ld;
    return w;
}

#include "psw_rs_tma.cuh"

template <typename T, bool LS>
size_t tile_smem() {
    return LS ? sizeof(T) * kRsSeg * 32 * kSPitch : 0;
}

template <typename T, bool LS>
int launch_part(const psw_plan* pl, const T* F, int64_t ldf, int64_t N, const Work& w,
                cudaStream_t s) {
    if constexpr (!LS) {
        int rc = PSW_OK;
        if (launch_part_tma<T>(pl, F, ldf, N, w.sc, s, rc)) return rc;
    }
    const size_t dyn = tile_smem<T, LS>();
    auto kern = rs_part_kernel<T, LS>;
    if (dyn > 0) {
        static std::once_flag once;
        cudaError_t e = cudaSuccess;
        std::call_once(once, [&] {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
        });
        PSW_CUDA_TRY(e);
    }
    const dim3 grid(unsigned((N + 31) / 32), unsigned(pl->rs_ngroups));
    kern<<<grid, kRsThreads, dyn, s>>>(F, ldf, N, int32_t(pl->row0), pl->d_rs_group, pl->d_rs_run,
                                      pl->d_segdesc, pl->d_seg,
                                      static_cast<const FusedFwd<T>*>(pl->d_ffwd), w.sc);
    return PSW_OK;
}

template <typename T, bool LS, bool STREAM>
int launch_solve_t(const psw_plan* pl, const T* F, int64_t ldf, T* X, int64_t ldx, int64_t N,
                   const Work& w, const double* V, int64_t ldv, cudaStream_t s) {
    const size_t dyn = tile_smem<T, LS>();
    auto kern = rs_solve_kernel<T, LS, STREAM>;
    if (dyn > 0) {
        static std::once_flag once;
        cudaError_t e = cudaSuccess;
        std::call_once(once, [&] {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
        });
        PSW_CUDA_TRY(e);
    }
    const dim3 grid(unsigned((N + 31) / 32), unsigned(pl->rs_ngroups));
    kern<<<grid, kRsThreads, dyn, s>>>(F, ldf, X, ldx, N, int32_t(pl->row0), pl->rs_ngroups,
                                      pl->d_rs_group, pl->d_rs_run, pl->d_segdesc, pl->d_seg,
                                      static_cast<const SolveCoef<T>*>(pl->d_scoef), pl->d_rs_cw, w.sc,
                                      V, ldv);
    return PSW_OK;
}

template <typename T, bool LS>
int launch_solve(const psw_plan* pl, const T* F, int64_t ldf, T* X, int64_t ldx, int64_t N,
                 const Work& w, const double* V, int64_t ldv, bool stream_loads, cudaStream_t s) {
    if constexpr (!LS) {
        int rc = PSW_OK;
        if (launch_solve_tma<T>(pl, F, ldf, X, ldx, N, w.sc, V, ldv, s, rc)) return rc;
    }
    return stream_loads ? launch_solve_t<T, LS, true>(pl, F, ldf, X, ldx, N, w, V, ldv, s)
                        : launch_solve_t<T, LS, false>(pl, F, ldf, X, ldx, N, w, V, ldv, s);
}

// K2 of a whole-system plan: boundary values into w.V, run carries in place.
// fold (one thread per RHS and block) -> V (the combination matrix for
// P <= kCombMaxP, else the STAGED dichotomy) -> carry (RHS x block), each a
// programmatic dependent launch of the one before. PSW_RESWEEP_COMB=1: the
// single-kernel rs_comb_kernel (one CTA per 32 RHS).
int launch_comb(const psw_plan* pl, int64_t N, const Work& w, cudaStream_t s, int64_t& launches) {
    const int P = int(pl->P), p = int(pl->p);
    const unsigned gx = unsigned((N + 127) / 128);
    static const int single = [] {
        const char* e = std::getenv("PSW_RESWEEP_COMB");
        return e ? std::atoi(e) : 0;
    }();
    if (single == 1 && pl->d_cmat && P <= kCombMaxP) {
        const size_t cmb = sizeof(double) * size_t(std::max(p, 1)) * 2 * P;
        static std::once_flag once;
        cudaError_t e = cudaSuccess;
        std::call_once(once, [&] {
            e = cudaFuncSetAttribute(rs_comb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(double) * (kCombMaxP - 1) * 2 * kCombMaxP));
        });
        PSW_CUDA_TRY(e);
        rs_comb_kernel<<<unsigned((N + 31) / 32), kCombWarps * 32, cmb, s>>>(
            N, P, p, pl->d_rs_runoff, pl->d_rs_runcoef, pl->d_cmat, w.sc, w.V, w.ldv);
        ++launches;
        return PSW_OK;
    }
    PSW_CUDA_TRY(launch_pdl(rs_fold_kernel, dim3(gx, unsigned(P)), dim3(128), 0, s, N,
                            pl->d_rs_runoff, pl->d_rs_runcoef, w.sc, w.bl, w.br));
    ++launches;
    if (p > 0) {
        if (pl->d_cmat && P <= kCombMaxP) {
            const size_t vsm = sizeof(double) * 2 * P * (kVmatRhs + kVmatRows);
            static std::once_flag once;
            cudaError_t ea = cudaSuccess;
            std::call_once(once, [&] {
                ea = cudaFuncSetAttribute(rs_vmat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(sizeof(double) * 2 * kCombMaxP * (kVmatRhs + kVmatRows)));
            });
            PSW_CUDA_TRY(ea);
            PSW_CUDA_TRY(launch_pdl(rs_vmat_kernel,
                                    dim3(unsigned((N + kVmatRhs - 1) / kVmatRhs),
                                         unsigned((p + kVmatRows - 1) / kVmatRows)),
                                    dim3(256), vsm, s, N, w.sc.ld, P, p, pl->d_cmat, w.bl, w.br, w.V,
                                    w.ldv));
        } else {
            // the combination runs over the padded pitch (columns >= N unused)
            if (int rc = launch_combine(pl, w.bl, w.br, w.sc.ld, w.V, s)) return rc;
        }
        ++launches;
    }
    PSW_CUDA_TRY(launch_pdl(rs_carry_kernel, dim3(gx, unsigned(P)), dim3(128), 0, s, N, p, 0,
                            pl->d_rs_runoff, pl->d_rs_runcoef, w.sc, w.V, w.ldv));
    ++launches;
    return PSW_OK;
}

template <typename T>
int solve_all(const psw_plan* pl, const void* Fv, int64_t ldf, void* Xv, int64_t ldx, int64_t N,
              int layout, const Work& w, bool stream_loads, cudaStream_t s, void** ev, int nev,
              int64_t& launches) {
    const T* F = static_cast<const T*>(Fv);
    T* X = static_cast<T*>(Xv);
    mark(ev, nev, 0, s);
    int rc = layout == PSW_LAYOUT_S ? launch_part<T, true>(pl, F, ldf, N, w, s)
                                    : launch_part<T, false>(pl, F, ldf, N, w, s);
    if (rc) return rc;
    ++launches;
    mark(ev, nev, 1, s);
    if ((rc = launch_comb(pl, N, w, s, launches))) return rc;
    mark(ev, nev, 2, s);
    rc = layout == PSW_LAYOUT_S
             ? launch_solve<T, true>(pl, F, ldf, X, ldx, N, w, w.V, w.ldv, stream_loads, s)
             : launch_solve<T, false>(pl, F, ldf, X, ldx, N, w, w.V, w.ldv, stream_loads, s);
    if (rc) return rc;
    ++launches;
    mark(ev, nev, 3, s);
    return PSW_OK;
}

int solve_all_dt(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                 int layout, const Work& w, bool stream_loads, cudaStream_t s, void** ev, int nev,
                 int64_t& launches) {
    return pl->dtype == PSW_F64
               ? solve_all<double>(pl, F, ldf, X, ldx, N, layout, w, stream_loads, s, ev, nev, launches)
               : solve_all<float>(pl, F, ldf, X, ldx, N, layout, w, stream_loads, s, ev, nev, launches);
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

}  // namespace

// ------------------------------------------------------------------ tables
int build_rs_tables(psw_plan* pl, const std::vector<SegDesc>& desc,
                    const std::vector<SegCoef>& seg, const std::vector<FusedFwd<double>>& ff,
                    const std::vector<FusedBwd<double>>& fb) {
    const int s_begin = pl->seg_off[size_t(pl->blk0)], s_end = pl->seg_off[size_t(pl->blk1)];
    std::vector<RsGroup> groups;
    std::vector<RsRun> runs;
    std::vector<SegCoef> rcoef;
    std::vector<int32_t> runoff(size_t(pl->blk1 - pl->blk0) + 1, 0);
    for (int g0 = s_begin, g1 = 0; g0 < s_end; g0 = g1) {
        // kRsSeg segments, at most kTmaRows rows (one TMA stage)
        g1 = g0 + 1;
        while (g1 < s_end && g1 - g0 < kRsSeg && desc[size_t(g1)].b - desc[size_t(g0)].a <= kTmaRows)
            ++g1;
        RsGroup g{g0, g1, int32_t(runs.size()), 0, desc[size_t(g0)].a, desc[size_t(g1 - 1)].b,
                  desc[size_t(g0)].t, 0};
        for (int s = g0; s < g1;) {
            const int t = desc[size_t(s)].t;
            int e = s;
            while (e < g1 && desc[size_t(e)].t == t) ++e;
            // compose the segments' affine maps (psw_internal.h): with
            // D_{a-1} = Drel + MUpre D_in along the run and x_a(s) = Lam~_s +
            // D_{a-1} K1_s + x_l K2_s + nu_s x_b(s)
            double mu = 1.0, k1 = 0.0, k2 = 0.0, nu = 1.0;
            for (int q = s; q < e; ++q) {
                const SegCoef& c = seg[size_t(q)];
                k1 += nu * mu * c.k1;
                k2 += nu * c.k2;
                mu *= c.mu_end;
                nu *= c.nu;
            }
            runs.push_back({s, e, t, int32_t(t - pl->blk0)});
            rcoef.push_back({mu, k1, k2, nu});
            s = e;
        }
        g.r1 = int32_t(runs.size());
        pl->rs_maxruns = std::max(pl->rs_maxruns, int(g.r1 - g.r0));
        for (int q = g0; q < g1; ++q) {
            const int len = desc[size_t(q)].b - desc[size_t(q)].a;
            pl->rs_minseg = pl->rs_minseg ? std::min(pl->rs_minseg, len) : len;
        }
        groups.push_back(g);
    }
    static_assert(kRsSeg <= 8, "CarryW holds 8 slots");
    // closed-form carry weights per group slot (CarryW, psw_internal.h)
    std::vector<CarryW> cw(groups.size() * kRsSeg, CarryW{});
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        const RsGroup& g = groups[gi];
        const int ns = g.s1 - g.s0;
        for (int w = 0; w < ns; ++w) {
            const int t = desc[size_t(g.s0 + w)].t;
            int lo = w, hi = w + 1;  // the run's slots [lo, hi)
            while (lo > 0 && desc[size_t(g.s0 + lo - 1)].t == t) --lo;
            while (hi < ns && desc[size_t(g.s0 + hi)].t == t) ++hi;
            auto sc = [&](int i) -> const SegCoef& { return seg[size_t(g.s0 + i)]; };
            // Pr[j] = prod mu over [lo, j); Am[j][i] = prod mu over (i, j)
            double Pr[8], Am[8][8] = {};
            for (int j = lo; j < hi; ++j) {
                Pr[j] = 1.0;
                for (int l = lo; l < j; ++l) Pr[j] *= sc(l).mu_end;
                for (int i = lo; i < j; ++i) {
                    double a = 1.0;
                    for (int l = i + 1; l < j; ++l) a *= sc(l).mu_end;
                    Am[j][i] = a;
                }
            }
            CarryW& c = cw[gi * kRsSeg + size_t(w)];
            c.P = Pr[w];
            for (int i = lo; i < w; ++i) c.A[i] = Am[w][i];
            c.Q = 1.0;
            for (int l = w + 1; l < hi; ++l) c.Q *= sc(l).nu;
            for (int j = w + 1; j < hi; ++j) {
                double b = 1.0;  // prod nu over (w, j)
                for (int l = w + 1; l < j; ++l) b *= sc(l).nu;
                c.B[j] = b;
                c.K2 += b * sc(j).k2;
                c.K1 += b * sc(j).k1 * Pr[j];
                for (int i = lo; i < j; ++i) c.C[i] += b * sc(j).k1 * Am[j][i];
            }
        }
    }
    for (size_t r = 0; r < runs.size(); ++r) runoff[size_t(runs[r].tl) + 1] = int32_t(r + 1);
    for (size_t i = 1; i < runoff.size(); ++i) runoff[i] = std::max(runoff[i], runoff[i - 1]);
    pl->rs_ngroups = int(groups.size());
    pl->rs_nruns = int(runs.size());
    // per-row solve coefficients (rp, ma, lam from the forward table, mu, w,
    // al from the backward one)
    const int64_t n = pl->n;
    const size_t es = pl->dtype == PSW_F64 ? sizeof(SolveCoef<double>) : sizeof(SolveCoef<float>);
    std::vector<unsigned char> sco(size_t(n) * es);
    for (int64_t q = 0; q < n; ++q) {
        const FusedFwd<double>& a = ff[size_t(q)];
        const FusedBwd<double>& b = fb[size_t(q)];
        if (pl->dtype == PSW_F64)
            reinterpret_cast<SolveCoef<double>*>(sco.data())[q] = {a.rp, a.ma, a.lam, b.mu, b.w, b.al};
        else
            reinterpret_cast<SolveCoef<float>*>(sco.data())[q] = {
                float(a.rp), float(a.ma), float(a.lam), float(b.mu), float(b.w), float(b.al)};
    }
    auto up = [&](void** dst, const void* src, size_t bytes) -> int {
        PSW_CUDA_TRY(cudaMalloc(dst, std::max<size_t>(bytes, 16)));
        if (bytes) PSW_CUDA_TRY(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
        pl->info.device_bytes += int64_t(bytes);
        return PSW_OK;
    };
    if (int rc = up(reinterpret_cast<void**>(&pl->d_rs_group), groups.data(), sizeof(RsGroup) * groups.size())) return rc;
    if (int rc = up(reinterpret_cast<void**>(&pl->d_rs_run), runs.data(), sizeof(RsRun) * runs.size())) return rc;
    if (int rc = up(reinterpret_cast<void**>(&pl->d_rs_runcoef), rcoef.data(), sizeof(SegCoef) * rcoef.size())) return rc;
    if (int rc = up(reinterpret_cast<void**>(&pl->d_rs_runoff), runoff.data(), sizeof(int32_t) * runoff.size())) return rc;
    if (int rc = up(reinterpret_cast<void**>(&pl->d_rs_cw), cw.data(), sizeof(CarryW) * cw.size())) return rc;
    return up(&pl->d_scoef, sco.data(), sco.size());
}

// ------------------------------------------------------------------ drivers
bool resweep_supported(const psw_plan* pl, int layout, int64_t N) {
    if (pl->world != 1 || (layout != PSW_LAYOUT_R && layout != PSW_LAYOUT_S) || N < 1) return false;
    return pl->d_rs_group && pl->rs_ngroups > 0 && pl->rs_ngroups < 65536 && pl->P < 65536 &&
           (N + 31) / 32 < (int64_t{1} << 31);
}

int solve_resweep(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                  int layout, cudaStream_t s, void** ev, int nev) {
    void* mem = nullptr;
    PSW_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&mem), work_bytes(pl, N, true), pl->device, s));
    const Work w = carve(pl, N, mem, true);
    int64_t launches = 0;
    int rc = solve_all_dt(pl, F, ldf, X, ldx, N, layout, w, true, s, ev, nev, launches);
    cudaError_t e = cudaGetLastError();
    scratch_free(mem, s);
    if (rc != PSW_OK) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "resweep kernels");
    note_launches(launches);
    return PSW_OK;
}

// ------------------------------------------------------------------ shards
int64_t shard_workspace_bytes(const psw_plan* pl, int64_t N) {
    return int64_t(work_bytes(pl, N, false));
}

int shard_forward(const psw_plan* pl, const void* Fv, int64_t ldf, int64_t N, void* ws,
                  double* partials, int64_t ldv, cudaStream_t s) {
    const Work w = carve(pl, N, ws, false);
    const int nb = int(pl->blk1 - pl->blk0), p = int(pl->p);
    int rc = pl->dtype == PSW_F64
                 ? launch_part<double, false>(pl, static_cast<const double*>(Fv), ldf, N, w, s)
                 : launch_part<float, false>(pl, static_cast<const float*>(Fv), ldf, N, w, s);
    if (rc) return rc;
    const unsigned gx = unsigned((N + 127) / 128);
    rs_fold_kernel<<<dim3(gx, unsigned(nb)), 128, 0, s>>>(N, pl->d_rs_runoff, pl->d_rs_runcoef,
                                                          w.sc, w.bl, w.br);
    int64_t launches = 2;
    if (p > 0) {
        rs_vpart_kernel<<<dim3(gx, unsigned(p)), 128, 0, s>>>(N, w.sc.ld, int(pl->P), p,
                                                              int(pl->blk0), nb, pl->d_cmat, w.bl,
                                                              w.br, partials, ldv);
        ++launches;
    }
    PSW_CUDA_TRY(cudaGetLastError());
    note_launches(launches);
    return PSW_OK;
}

int shard_backward(const psw_plan* pl, const void* Fv, int64_t ldf, void* Xv, int64_t ldx,
                   int64_t N, void* ws, const double* V, int64_t ldv, cudaStream_t s) {
    const Work w = carve(pl, N, ws, false);
    const int nb = int(pl->blk1 - pl->blk0), p = int(pl->p);
    const unsigned gx = unsigned((N + 127) / 128);
    rs_carry_kernel<<<dim3(gx, unsigned(nb)), 128, 0, s>>>(N, p, int(pl->blk0), pl->d_rs_runoff,
                                                           pl->d_rs_runcoef, w.sc, V, ldv);
    int rc = pl->dtype == PSW_F64
                 ? launch_solve<double, false>(pl, static_cast<const double*>(Fv), ldf,
                                               static_cast<double*>(Xv), ldx, N, w, V, ldv, true, s)
                 : launch_solve<float, false>(pl, static_cast<const float*>(Fv), ldf,
                                              static_cast<float*>(Xv), ldx, N, w, V, ldv, true, s);
    if (rc) return rc;
    PSW_CUDA_TRY(cudaGetLastError());
    note_launches(2);
    return PSW_OK;
}

}  // namespace psw
