// CLUSTER solve path: one persistent kernel, F read once and X written once
// (the minimum traffic of SURVEY §8(d)), one CTA per SM holding a whole
// 128-byte-wide RHS strip of G blocks in shared memory.
//
// Layout R, uniform partition (n = P m), P = C G:
//   * an RHS tile = W right-hand sides (128 contiguous bytes of every row:
//     the write granularity that keeps HBM writes at full speed);
//   * a thread-block cluster of C CTAs owns a tile; CTA c owns blocks
//     [cG, cG + G) = G m rows (+1 for the last block) and keeps them in a
//     shared-memory slab filled by TMA (W x 32-row boxes, one mbarrier per
//     box). Clusters are persistent and walk the tiles;
//   * one thread per (block, 32-row segment, rhs): forward sweep of the
//     segment from a zero carry with d~ in registers, beta dot products
//     (betas.hpp:42-57 split by segment) and Lam~ (psw_internal.h); the slab
//     is handed to TMA for the next tile as soon as every thread swept it;
//   * a block scan folds the segment partials into exact carries and block
//     betas, which are pushed to every CTA of the cluster with st.async
//     (DSMEM stores completing on the receiver's mbarrier);
//   * each CTA evaluates the G + 1 boundary values it needs from the
//     combination matrix (psw_plan.cpp combine_matrix: the reference
//     dichotomy, boundary_solve.hpp:96-121, is linear in the betas);
//   * a backward block fold gives every segment its exact x_b, and the back
//     substitution streams X out of registers.
// Compared with the FUSED path (psw_fused.cu: 16-CTA clusters of one block
// each, three CTAs per SM), a CTA here holds four blocks (C1: 128 KB of F in
// flight per SM, four CTAs per exchange) and the sweep coefficients live in
// bank-padded structure-of-arrays tables next to the slab.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cooperative_groups.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "psw_device.cuh"
#include "psw_internal.h"
#include "psw_tma.cuh"

namespace cg = cooperative_groups;

namespace psw {
namespace {

constexpr int kMaxThreads = 512;
constexpr int kMaxC = 16;                   // cluster size (> 8 needs the non-portable opt-in)
constexpr size_t kSmemTwoPerSm = 115712 - 512;  // two CTAs per SM (228 KB, 1 KB reserved each)
constexpr size_t kSmemMax = 232448;         // 227 KB per CTA (sm_100)
constexpr int kSegMax = kSegLen + 1;
constexpr int kMaxBox = 256;                // TMA box height limit

__device__ __forceinline__ void bar_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

__device__ __forceinline__ void st_async_2(uint32_t raddr, double a, double b, uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
            raddr),
        "d"(a), "d"(b), "r"(rbar)
        : "memory");
}

// optional phase trace (PSW_CLUSTER_TRACE=1): clock64 at 8 points of tile 2
// for every CTA, dumped by the host after the launch
constexpr int kTraceSlots = 8;
__device__ unsigned long long g_ctrace[1024 * kTraceSlots];
__device__ unsigned long long g_gtrace[1024 * 2];  // globaltimer: push, exchange complete
__device__ unsigned long long g_btrace[1024 * 8];  // globaltimer: push of every block (G <= 8)
__device__ unsigned long long g_etrace[1024 * 4];  // globaltimer: entry, tables ready, first tile done, exit

struct CGeom {
    int n, P, p, m, G, C, S, H, trace;  // H: TMA box height (divides m)
    int64_t N, ldx, ntiles;
};

// Coefficients of slab row q: two 4-vectors {rp, ma, gr, gl}, {lam, mu, w, al}
// (64 B for fp64), 16 bytes of padding every 32 rows so that rows q and
// q + 32 (two segments read by one warp) land in different banks.
template <typename T>
struct alignas(4 * sizeof(T)) Quad {
    T x, y, z, w;
};
template <typename T>
__host__ __device__ __forceinline__ size_t coff(int q) {
    return size_t(q) * 8 * sizeof(T) + size_t(q >> 5) * 16;
}

// Coefficient row a + r from the segment's first row a: segments start at
// slab rows a = 0 or 1 mod 32 (uniform partitions, m % 32 == 0), so with
// AC = a mod 32 known at compile time every row is a constant offset from
// coff(a) (AC < 0: computed).
template <typename T, int AC>
__device__ __forceinline__ const unsigned char* crow(const unsigned char* co, const unsigned char* cb,
                                                     int a, int r) {
    if constexpr (AC < 0)
        return co + coff<T>(a + r);
    else
        return cb + size_t(r) * 8 * sizeof(T) + size_t((AC + r) >> 5) * 16;
}

// Shared-memory carve-up (bytes), identical on host and device.
template <typename T, int W, int NSLAB, bool LS = false>
struct CLayout {
    int ra;
    size_t slab_b, coef, seg, allx, vals, cm, segc, bars, total;
    __host__ __device__ CLayout(int G, int m, int S, int P, int nth) {
        auto up = [](size_t x) { return (x + 127) & ~size_t(127); };
        ra = G * m + 1;               // slab rows of the last CTA
        // layout S: G*m/16 swizzled 16-row boxes (1024-aligned) + a 2-row tail
        slab_b = LS ? up(size_t(G * m) * W * sizeof(T) + size_t(2) * W * sizeof(T))
                    : up(size_t(ra) * W * sizeof(T));
        coef = NSLAB * slab_b;
        seg = up(coef + coff<T>(ra) + 16);
        // sd, sx per thread; the beta partials per pair of segments when a warp
        // holds two segments of one block (W = 16), else per thread
        allx = up(seg + size_t(W == 16 ? 3 : 4) * nth * sizeof(double));
        vals = up(allx + size_t(2) * P * W * 2 * sizeof(double));
        cm = up(vals + size_t(G + 1) * W * sizeof(double));
        segc = up(cm + size_t(G + 1) * 2 * P * sizeof(double));
        bars = up(segc + size_t(G) * S * sizeof(SegCoef));
        total = bars + size_t(NSLAB * G + 3) * sizeof(uint64_t);
    }
};

// forward rows of one segment from a zero carry: d~ into dr, partials to
// the thread's slots (betas.hpp:42-57 split by segment; Lam~, psw_internal.h)
// Layout S slab (fp64, W = 16): 16-row TMA boxes with the 128-byte swizzle,
// box c = rows 16c..16c+15 of all W right-hand sides, rhs l's rows in the
// 128-byte line l of the box, 16-byte chunk (q/2) XOR (l mod 8).
template <typename T, int W>
__device__ __forceinline__ int s_index(int q, int l) {
    return ((q >> 4) * W + l) * 16 + ((((q & 15) >> 1) ^ (l & 7)) << 1) + (q & 1);
}

__device__ __forceinline__ void st_v4(double* p, double a, double b, double c, double d) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
                 : "memory");
}

__device__ __forceinline__ void st_v2(double* p, double a, double b) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

// Layout S backward (fp64): a right-hand side's rows are contiguous, so each
// thread writes its segment as whole 32-byte sectors (256-bit stores) once
// the segment is solved; AL = the segment's first global row mod 4 (0 for
// the first block's segments, 3 for the others: blocks start at t*m - 1).
// Rows 31, 32 exist when len > 31, > 32.
template <int AL>
__device__ __forceinline__ void bwd_v4(const unsigned char* co, int a, int len,
                                       double (&dr)[kSegMax], double D, double xl, double xn,
                                       double* xp) {
    const unsigned char* cb = co + coff<double>(a);
#pragma unroll
    for (int r = kSegMax - 1; r >= 0; --r) {
        if (r < kSegLen - 1 || r < len) {
            const Quad<double> c1 = reinterpret_cast<const Quad<double>*>(crow<double, AL == 0 ? 1 : 0>(co, cb, a, r))[1];
            xn = fma(c1.w, xn, fma(xl, c1.z, fma(c1.y, D, dr[r])));
            dr[r] = xn;
        }
    }
    constexpr int r0 = AL == 0 ? 0 : 4 - AL;  // first 32-byte aligned row
    if constexpr (AL == 3) __stcs(xp, dr[0]);
    // full groups inside rows 0..30
#pragma unroll
    for (int r = r0; r + 4 <= kSegLen - 1; r += 4) st_v4(xp + r, dr[r], dr[r + 1], dr[r + 2], dr[r + 3]);
    // the last group starts at rt and runs to len
    constexpr int rt = r0 + ((kSegLen - 1 - r0) / 4) * 4;
    const int nt = len - rt;  // 1..5
    if (nt >= 4) {
        st_v4(xp + rt, dr[rt], dr[rt + 1], dr[rt + 2], dr[rt + 3]);
        if constexpr (rt + 4 < kSegMax)
            if (nt == 5) __stcs(xp + rt + 4, dr[rt + 4]);
    } else {
        if (nt >= 2) st_v2(xp + rt, dr[rt], dr[rt + 1]);
        if (nt == 1) __stcs(xp + rt, dr[rt]);
        if (nt == 3) __stcs(xp + rt + 2, dr[rt + 2]);
    }
}

// 4 x 4 transpose of 32-byte chunks among the four lanes 4g .. 4g+3: lane a
// enters with chunks c[0..3] (16 consecutive rows) of its own right-hand
// side and leaves with chunk a of the right-hand sides of lanes 4g + s in
// c[s] (two butterfly stages, selects with compile-time register indices).
__device__ __forceinline__ void chunk_transpose4(double (&c)[4][4], int lane) {
    const bool a1 = lane & 2, a0 = lane & 1;
#pragma unroll
    for (int s0 = 0; s0 < 2; ++s0)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double send = a1 ? c[s0][e] : c[s0 + 2][e];
            const double recv = __shfl_xor_sync(0xffffffffu, send, 2);
            if (a1) c[s0][e] = recv; else c[s0 + 2][e] = recv;
        }
#pragma unroll
    for (int s0 = 0; s0 < 4; s0 += 2)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double send = a0 ? c[s0][e] : c[s0 + 1][e];
            const double recv = __shfl_xor_sync(0xffffffffu, send, 1);
            if (a0) c[s0][e] = recv; else c[s0 + 1][e] = recv;
        }
}

// Layout S backward with whole-line stores (fp64): as bwd_v4, but the four
// lanes of a group exchange their 32-byte chunks first, so that a group's
// store instruction writes 128 contiguous bytes (16 rows) of ONE right-hand
// side instead of four separate sectors: a warp store touches 8 lines, not
// 32. The arithmetic and the values are bwd_v4's. Every lane of the warp
// runs it (shuffles); `kk0` = the group's first right-hand side, stores to
// right-hand sides >= N are dropped. ga = the segment's first global row.
template <int AL>
__device__ __forceinline__ void bwd_v4t(const unsigned char* co, int a, int len,
                                        double (&dr)[kSegMax], double D, double xl, double xn,
                                        double* X, int64_t ldx, int64_t kk, int64_t N, int ga,
                                        int lane) {
    const unsigned char* cb = co + coff<double>(a);
#pragma unroll
    for (int r = kSegMax - 1; r >= 0; --r) {
        if (r < kSegLen - 1 || r < len) {
            const Quad<double> c1 = reinterpret_cast<const Quad<double>*>(crow<double, AL == 0 ? 1 : 0>(co, cb, a, r))[1];
            xn = fma(c1.w, xn, fma(xl, c1.z, fma(c1.y, D, dr[r])));
            dr[r] = xn;
        } else {
            dr[r] = 0.0;
        }
    }
    constexpr int o0 = AL == 0 ? 0 : 1;  // first row of the first whole line
    const int aa = lane & 3;
    const int64_t k0 = kk - aa;
    if constexpr (AL == 3)
        if (kk < N) __stcs(X + kk * ldx + ga, dr[0]);
    if constexpr (o0 + 32 < kSegMax)
        if (kk < N && len > o0 + 32) __stcs(X + kk * ldx + ga + o0 + 32, dr[o0 + 32]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double c[4][4];
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
            for (int e = 0; e < 4; ++e) c[s][e] = dr[o0 + 16 * h + 4 * s + e];
        chunk_transpose4(c, lane);
        // rows of this lane's chunk that exist (the segment may end inside it)
        const int nt = len - (o0 + 16 * h + 4 * aa);
        double* xp = X + k0 * ldx + ga + o0 + 16 * h + 4 * aa;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            double* q = xp + int64_t(s) * ldx;
            if (k0 + s < N) {
                if (nt >= 4) {
                    st_v4(q, c[s][0], c[s][1], c[s][2], c[s][3]);
                } else {
                    if (nt >= 2) st_v2(q, c[s][0], c[s][1]);
                    if (nt == 1) __stcs(q, c[s][0]);
                    if (nt == 3) __stcs(q + 2, c[s][2]);
                }
            }
        }
    }
}

template <typename T, int W, int NMAX, bool EXACT = (NMAX <= kSegLen), bool LS = false, int DL = 0,
          int AC = -1>
__device__ __forceinline__ void fwd(const T* slab, const unsigned char* co, int a, int lane,
                                    int len, T (&dr)[kSegMax], double* sd, double* sx, double* sr,
                                    double* sl, int tid, int gm = 0) {
    const T* col = slab + size_t(a) * W + lane;
    // layout S: physical row a + 1 + r = q16 + DL + r with q16 a multiple of 16
    // (DL = (a + 1) mod 16, compile time), so box, chunk and half of every row
    // are constants and only the lane's XOR term is a register
    const int q16 = a + 1 - DL;
    const T* lb = slab + q16 * 16 + lane * 16;
    const int x2 = (lane & 7) << 1;
    T fn = T(0);  // the second row of a 16-byte chunk (layout S)
    const unsigned char* cb = co + coff<T>(a);
    T d = T(0), lx = T(0);
    double br = 0.0, bl = 0.0;
#pragma unroll
    for (int r = 0; r < NMAX; ++r) {
        if (EXACT || r < kSegLen - 1 || r < len) {
            const Quad<T>* c = reinterpret_cast<const Quad<T>*>(crow<T, AC>(co, cb, a, r));
            const Quad<T> c0 = c[0];
            const T lam = c[1].x;
            T f;
            if constexpr (LS) {  // physical row a + r + 1; rows >= gm in the tail box
                // rows 0..30 two at a time (one 16-byte chunk: conflict-free for
                // 16 lanes), rows 31, 32 one at a time (they may be in the tail box)
                const int j = DL + r;  // a constant after unrolling
                const int o = ((j >> 4) << 8) + (x2 ^ (((j & 15) >> 1) << 1));
                if (r >= kSegLen - 1) {
                    const int q = a + r + 1;
                    f = q >= gm ? slab[gm * W + lane * 2 + (q - gm)] : lb[o + (j & 1)];
                } else if ((j & 1) == 0 && r + 1 <= kSegLen - 2) {
                    const double2 v = *reinterpret_cast<const double2*>(lb + o);
                    f = v.x;
                    fn = v.y;
                } else if ((j & 1) == 1 && r >= 1) {
                    f = fn;
                } else {
                    f = lb[o + (j & 1)];
                }
            } else {
                f = col[r * W];
            }
            d = fma(c0.y, d, f * c0.x);
            br = fma(double(f), double(c0.z), br);
            bl = fma(double(f), double(c0.w), bl);
            lx = fma(lam, d, lx);
            dr[r] = d;
        }
    }
    sd[tid] = double(d);
    sx[tid] = double(lx);
    if constexpr (W == 16) {  // lanes 16..31 sweep the next segment of the same block
        br += __shfl_down_sync(0xffffffffu, br, 16);
        bl += __shfl_down_sync(0xffffffffu, bl, 16);
        if ((tid & 31) < 16) {
            sr[(tid >> 5) * 16 + (tid & 15)] = br;
            sl[(tid >> 5) * 16 + (tid & 15)] = bl;
        }
    } else {
        sr[tid] = br;
        sl[tid] = bl;
    }
}

// back substitution of one segment from the exact carries, last row first
template <typename T, int NMAX, bool EXACT = (NMAX <= kSegLen), int AC = -1>
__device__ __forceinline__ void bwd(const unsigned char* co, int a, int len,
                                    const T (&dr)[kSegMax], T D, T xl, T xn, T* xp, int64_t ldx) {
    const unsigned char* cb = co + coff<T>(a);
#pragma unroll
    for (int r = NMAX - 1; r >= 0; --r) {
        if (EXACT || r < kSegLen - 1 || r < len) {
            const Quad<T> c1 = reinterpret_cast<const Quad<T>*>(crow<T, AC>(co, cb, a, r))[1];
            xn = fma(c1.w, xn, fma(xl, c1.z, fma(c1.y, D, dr[r])));
            __stcs(xp + int64_t(r) * ldx, xn);
        }
    }
}

template <typename T, int W, int NSLAB, bool LS = false, int V4 = 0>
__global__ void __launch_bounds__(kMaxThreads / NSLAB) cluster_kernel(
    const __grid_constant__ CUtensorMap tmF, const __grid_constant__ CUtensorMap tmF1,
    const __grid_constant__ CUtensorMap tmF2, const T* F, int64_t ldf, T* X, CGeom g, const FusedFwd<T>* __restrict__ gff, const FusedBwd<T>* __restrict__ gfb,
    const SegCoef* __restrict__ gsegc, const SegDesc* __restrict__ gdesc,
    const double* __restrict__ gcmat, const unsigned char* __restrict__ gtab, int64_t tab_stride) {
    extern __shared__ __align__(1024) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    auto etrace = [&](int slot) {
        if (g.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            g_etrace[blockIdx.x * 4 + slot] = t;
        }
    };
    etrace(0);
    const int C = g.C, G = g.G, S = g.S, P = g.P, p = g.p, m = g.m;
    const int crank = int(cluster.block_rank());
    const int64_t cid = blockIdx.x / C, ncl = gridDim.x / C;
    // units of W right-hand sides; with two slabs a cluster takes them in
    // adjacent pairs (2q, 2q + 1), so the two 64-byte halves of every 128-byte
    // X line are written back to back and merge in L2
    const int64_t ngroups = (g.ntiles + NSLAB - 1) / NSLAB;
    const int64_t ntl = ngroups > cid ? NSLAB * ((ngroups - cid + ncl - 1) / ncl) : 0;
    auto unit = [&](int64_t k) { return (cid + (k / NSLAB) * ncl) * NSLAB + (k % NSLAB); };
    const int nth = G * S * W;
    const int tid = threadIdx.x;
    const CLayout<T, W, NSLAB, LS> L(G, m, S, P, nth);
    // slab row 0 is global row crank*G*m - 1 (row -1 of CTA 0 is outside F:
    // TMA zero-fills it)
    const int base = crank * G * m - 1;
    const int nrows = crank == C - 1 ? G * m + 1 : G * m;
    const bool last_cta = crank == C - 1;
    unsigned char* co = smem + L.coef;  // coefficient rows (coff)
    double* sd = reinterpret_cast<double*>(smem + L.seg);  // d~ end -> carry D
    double* sx = sd + nth;                                 // Lam~ -> Lam~ + D K1
    double* sr = sx + nth;                                 // right partials
    double* sl = sr + (W == 16 ? nth / 2 : nth);           // left partials
    double* allx = reinterpret_cast<double*>(smem + L.allx);  // [2][P][W][R, L]
    double* vals = reinterpret_cast<double*>(smem + L.vals);  // [G + 1][W]
    double* cm = reinterpret_cast<double*>(smem + L.cm);      // [G + 1][2P]
    SegCoef* segc = reinterpret_cast<SegCoef*>(smem + L.segc);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* xbar = bars + NSLAB * G;

    const int lane = tid % W, h = tid / W, j = h / S;
    const int t = crank * G + j;
    const SegDesc sgd = gdesc[t * S + h % S];
    const int a = sgd.a - base, len = sgd.b - sgd.a;  // slab rows [a, a + len)
    const bool first_seg = (h % S) == 0;

    auto slab_of = [&](int64_t k) {
        return reinterpret_cast<T*>(smem + size_t(k % NSLAB) * L.slab_b);
    };
    auto bars_of = [&](int64_t k) { return bars + (k % NSLAB) * G; };
    // rows of block jb of unit k into the slab: m / H boxes (+ the n-th row
    // for the last block of the last CTA); one mbarrier per block
    auto issue_block = [&](int64_t k, int jb) {
        const int k0 = int(unit(k) * W);
        T* slab = slab_of(k);
        uint64_t* bar = &bars_of(k)[jb];
        const bool extra = last_cta && jb == G - 1;
        if constexpr (LS) {
            // the whole slab on the first barrier (boxes straddle blocks): G*m/16
            // boxes of 16 rows from global row base - 1 (even, so every box
            // starts on 16 bytes: TMA rejects an odd fp64 row) and a 2-row tail
            // box (tmF1, unswizzled); physical slab row = slab row + 1; row -2
            // of CTA 0 and rows past n are zero-filled
            if (jb != 0) return;
            const int nb = G * m / 16;
            mbar_expect_tx(bar, uint32_t((nb * 16 + 2) * W * sizeof(T)));
            for (int c = 0; c < nb; ++c)
                tma_load_2d(slab + size_t(c) * 16 * W, &tmF, base - 1 + 16 * c, k0, bar);
            tma_load_2d(slab + size_t(nb) * 16 * W, &tmF1, base - 1 + 16 * nb, k0, bar);
            return;
        }
        if (crank == 0 && jb == 0) {
            // global rows [0, m - 1) into slab rows [1, m): no box reaches row -1
            // (a box partly outside F is slow to complete)
            mbar_expect_tx(bar, uint32_t((m - 1) * W * sizeof(T)));
            for (int r = 0; r + g.H < m; r += g.H)
                tma_load_2d(slab + size_t(r + 1) * W, &tmF, k0, r, bar);
            tma_load_2d(slab + size_t(m - g.H + 1) * W, &tmF2, k0, m - g.H, bar);
            return;
        }
        mbar_expect_tx(bar, uint32_t((m + (extra ? 1 : 0)) * W * sizeof(T)));
        for (int r = jb * m; r < (jb + 1) * m; r += g.H)
            tma_load_2d(slab + size_t(r) * W, &tmF, k0, base + r, bar);
        if (extra) {  // row n - 1: one 128-byte bulk copy unless the tile is ragged
            const int64_t row = base + G * m;
            if (int64_t(k0) + W <= g.N)
                bulk_load(slab + size_t(G * m) * W, F + row * ldf + k0, uint32_t(W * sizeof(T)), bar);
            else
                tma_load_2d(slab + size_t(G * m) * W, &tmF1, k0, int(row), bar);
        }
    };
    if (tid == 0) {
        for (int i = 0; i < NSLAB * G; ++i) mbar_init(&bars[i], 1);
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        mbar_init(&xbar[2], 1);  // coefficient tables
        fence_mbar_init();
        // this rank's coefficient tables (prebuilt in the shared-memory layout)
        const uint32_t tb = uint32_t(coff<T>(nrows) + 16 + 15) & ~15u;
        mbar_expect_tx(&xbar[2], tb);
        for (uint32_t o = 0; o < tb; o += 32768)
            bulk_load(co + o, gtab + size_t(crank) * size_t(tab_stride) + o,
                      tb - o < 32768u ? tb - o : 32768u, &xbar[2]);
        // the first units stream in while the coefficient tables are copied
        for (int64_t k = 0; k < NSLAB && k < ntl; ++k)
            for (int jb = 0; jb < G; ++jb) issue_block(k, jb);
    }
    for (int i = tid; i < G * S; i += nth) segc[i] = gsegc[crank * G * S + i];
    for (int i = tid; i < (G + 1) * 2 * P; i += nth) {  // rows of boundaries crank*G - 1 + r
        const int bi = crank * G - 1 + i / (2 * P);
        cm[i] = (bi >= 0 && bi < p) ? gcmat[int64_t(bi) * 2 * P + i % (2 * P)] : 0.0;
    }
    __syncthreads();
    cluster.sync();  // every CTA's exchange barrier is initialised before any push
    mbar_wait(&xbar[2], 0);
    etrace(1);

    // each block's last thread (not a scan thread when S > 1) streams the
    // block's rows of the next unit in as soon as the block has swept them
    const bool block_issuer = (h % S) == S - 1 && lane == W - 1;
    T dr[kSegMax];
    auto stamp = [&](int64_t k, int slot) {
        if (g.trace && k == 2 && tid == 0 && blockIdx.x < 1024)
            g_ctrace[blockIdx.x * kTraceSlots + slot] = clock64();
    };
    for (int64_t k = 0; k < ntl; ++k) {
        const int buf = int(k & 1);
        stamp(k, 0);
        if (tid == 0) mbar_expect_tx(&xbar[buf], uint32_t(P * W * 2 * sizeof(double)));
        T* slab = slab_of(k);
        mbar_wait(&bars_of(k)[LS ? 0 : j], uint32_t((k / NSLAB) & 1));
        stamp(k, 1);
        // ---- forward sweep of the segment, d~ in registers
        // one instruction stream for every lane: segments are 31, 32 or 33 rows
        // (m % 32 == 0), and the two segments a warp sweeps may differ in length;
        // rows 0..30 unpredicated, the last two under a predicate
        if constexpr (LS) {  // a + 1 = 1 or 2 mod 16 (uniform partition, m % 32 == 0)
            if (((a + 1) & 15) == 1)
                fwd<T, W, kSegMax, false, LS, 1, 0>(slab, co, a, lane, len, dr, sd, sx, sr, sl, tid, G * m);
            else
                fwd<T, W, kSegMax, false, LS, 2, 1>(slab, co, a, lane, len, dr, sd, sx, sr, sl, tid, G * m);
        } else {  // a = 0 or 1 mod 32
            if ((a & 31) == 0)
                fwd<T, W, kSegMax, false, LS, 0, 0>(slab, co, a, lane, len, dr, sd, sx, sr, sl, tid, G * m);
            else
                fwd<T, W, kSegMax, false, LS, 0, 1>(slab, co, a, lane, len, dr, sd, sx, sr, sl, tid, G * m);
        }
        bar_sync(2 + j, S * W);  // the block's rows swept, its partials visible
        if (g.trace > 2 && tid == 0) {  // force the deferred barrier wait before the stamp
            volatile double* vs = sd;
            if (vs[nth - 1] == 1.2345e300) sd[0] = 0.0;
        }
        stamp(k, 2);
        if constexpr (LS) {  // the last warp refills once every block has swept
            if (k + NSLAB < ntl) {
                if (tid >= nth - 32) {  // bar.sync/arrive count whole warps
                    bar_sync(15, nth);
                    if (tid == nth - 1) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        issue_block(k + NSLAB, 0);
                    }
                } else {
                    bar_arrive(15, nth);
                }
            }
        } else if (block_issuer && k + NSLAB < ntl) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_block(k + NSLAB, j);
        }
        // ---- block scan: exact carries, block betas, pushed to every CTA
        if (first_seg) {
            double D = 0.0, R = 0.0, Lb = 0.0;
            for (int q = 0; q < S; ++q) {
                const int id = (j * S + q) * W + lane;
                const SegCoef sc = segc[j * S + q];
                const double dend = sd[id];
                sd[id] = D;
                sx[id] = fma(D, sc.k1, sx[id]);
                // the beta partials of segment pairs (W = 16) or segments
                if (W != 16 || (q & 1) == 0) {
                    const int bid = W == 16 ? ((j * S + q) >> 1) * 16 + lane : id;
                    R += sr[bid];
                    Lb += sl[bid];
                }
                D = fma(sc.mu_end, D, dend);
            }
            stamp(k, 7);
            if (t >= p) R = 0.0;   // right_t exists for t < p (betas.hpp:46-49)
            if (t == 0) Lb = 0.0;  // left_t for t > 0 (betas.hpp:51-55)
            double* dst = allx + (size_t(buf) * P + t) * W * 2 + lane * 2;
            const uint32_t src = smem_u32(dst), bar = smem_u32(&xbar[buf]);
            if (g.trace && k == 2 && lane == 0 && blockIdx.x < 1024 && j < 8) {
                unsigned long long tt;
                asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tt));
                g_btrace[blockIdx.x * 8 + j] = tt;
            }
            for (int c = 0; c < C; ++c) st_async_2(mapa_u32(src, c), R, Lb, mapa_u32(bar, c));
        }
        stamp(k, 3);
        if (g.trace && k == 2 && tid == 0 && blockIdx.x < 1024) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            g_gtrace[blockIdx.x * 2] = t;
        }
        // only the warps evaluating boundary values wait on the exchange (the
        // others would spin on the barrier and starve the scan's shared loads)
        const bool comb = tid < (G + 1) * W;
        if (tid < ((G + 1) * W + 31) / 32 * 32) mbar_wait(&xbar[buf], uint32_t((k >> 1) & 1));
        stamp(k, 4);
        if (g.trace && k == 2 && tid == 0 && blockIdx.x < 1024) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            g_gtrace[blockIdx.x * 2 + 1] = t;
        }
        // ---- the G + 1 boundary values of this CTA's blocks
        if (comb) {
            const int r = tid / W, ln = tid % W;
            const int bi = crank * G - 1 + r;
            double v = 0.0;
            if (bi >= 0 && bi < p) {
                const double* mr = cm + r * 2 * P;
                const double* ax = allx + size_t(buf) * P * W * 2 + ln * 2;
                double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
                int u = 0;
                for (; u + 2 <= P; u += 2) {
                    v0 = fma(mr[u], ax[u * W * 2], v0);
                    v1 = fma(mr[P + u], ax[u * W * 2 + 1], v1);
                    v2 = fma(mr[u + 1], ax[(u + 1) * W * 2], v2);
                    v3 = fma(mr[P + u + 1], ax[(u + 1) * W * 2 + 1], v3);
                }
                for (; u < P; ++u) {
                    v0 = fma(mr[u], ax[u * W * 2], v0);
                    v1 = fma(mr[P + u], ax[u * W * 2 + 1], v1);
                }
                v = (v0 + v2) + (v1 + v3);
            }
            vals[tid] = v;
        }
        bar_sync(1, nth);
        // ---- backward block fold: x_b of every segment
        const double xl = vals[j * W + lane];  // boundary t - 1 (0 for t = 0)
        if (first_seg) {
            double xb = vals[(j + 1) * W + lane];  // boundary t (0 for t = p)
            for (int q = S - 1; q >= 0; --q) {
                const int id = (j * S + q) * W + lane;
                const SegCoef sc = segc[j * S + q];
                const double A = sx[id];
                sx[id] = xb;  // sx: Lam~ + D K1 -> x_b
                xb = fma(sc.nu, xb, fma(xl, sc.k2, A));
            }
        }
        bar_sync(1, nth);
        stamp(k, 5);
        // ---- back substitution from the exact carries, X streamed out
        const int64_t kk = unit(k) * W + lane;
        const T D = T(sd[tid]), xlt = T(xl);
        T xn = T(sx[tid]);
        if constexpr (LS) {
            // layout S: the rhs' rows are contiguous; 32-byte stores when X and
            // its pitch are 32-byte aligned (V4; segments start at rows = 0 or 3
            // mod 4, choose_t). One store variant per instantiation: a third
            // one drives ptxas to 64 registers and 0.8 KB of spills (171 vs
            // 110 us on C4).
            if constexpr (V4 == 2) {  // whole-line stores: the warp's lanes exchange chunks
                double* xb = reinterpret_cast<double*>(X);
                if ((sgd.a & 3) == 0)
                    bwd_v4t<0>(co, a, len, dr, D, xlt, xn, xb, g.ldx, kk, g.N, sgd.a, lane);
                else
                    bwd_v4t<3>(co, a, len, dr, D, xlt, xn, xb, g.ldx, kk, g.N, sgd.a, lane);
            } else if (kk < g.N) {
                if constexpr (V4 == 1) {
                    double* xp = reinterpret_cast<double*>(X) + kk * g.ldx + sgd.a;
                    if ((sgd.a & 3) == 0)
                        bwd_v4<0>(co, a, len, dr, D, xlt, xn, xp);
                    else
                        bwd_v4<3>(co, a, len, dr, D, xlt, xn, xp);
                } else {
                    bwd<T, kSegMax, false>(co, a, len, dr, D, xlt, xn, X + kk * g.ldx + sgd.a, 1);
                }
            }
        } else if (kk < g.N) {
            T* xp = X + int64_t(sgd.a) * g.ldx + kk;
            if ((a & 31) == 0)
                bwd<T, kSegMax, false, 0>(co, a, len, dr, D, xlt, xn, xp, g.ldx);
            else
                bwd<T, kSegMax, false, 1>(co, a, len, dr, D, xlt, xn, xp, g.ldx);
        }
        stamp(k, 6);
        if (k == 0) etrace(2);
    }
    cluster.sync();  // no CTA leaves while a peer may still push into it
    etrace(3);
}

// ---------------------------------------------------------------- host side
struct CChoice {
    int W = 0, G = 0, C = 0, nslab = 1;
    size_t smem = 0;
};

template <typename T, int W, int NSLAB, bool LS = false>
CChoice choose_t(const psw_plan* pl) {
    CChoice ch;
    if (!pl->uniform || pl->world != 1 || !pl->d_ffwd || !pl->d_cmat || pl->nseg <= 0) return ch;
    const int P = int(pl->P), m = int(pl->m), S = pl->nseg;
    if (S * kSegLen < m - 1 || S * kSegLen > m + kSegLen || m % 32) return ch;
    if (W == 16 && S % 2) return ch;  // a warp's two segments must share a block
    static const int force_g = [] {
        const char* e = std::getenv("PSW_CLUSTER_G");  // tuning override
        return e ? std::atoi(e) : 0;
    }();
    // Two CTAs per SM when a CTA fits half the shared memory (two independent
    // tile chains per SM; C1: G = 2, C = 8 -> 63.9 us vs G = 4, C = 4 -> 68.1
    // us), else one; within each, the fewest CTAs per tile first.
    for (int pass = 0; pass < 2 && ch.G == 0; ++pass) {
        for (int G = P; G >= 1; --G) {
            if (P % G) continue;
            const int C = P / G;
            if (C > kMaxC) break;
            if (force_g > 0 && G != force_g) continue;
            // layout S needs G >= 2: the forward reads row 30 of a segment from
            // the swizzled boxes, but with G = 1 CTA 0's only block is the short
            // first block, whose row 30 is the CTA's last row, in the tail box.
            // A tail check on row 30 costs registers (spills, C4 88 -> 95 us).
            if (LS && G == 1) continue;
            const int nth = G * S * W;
            if (nth > kMaxThreads / NSLAB || nth % 32) continue;
            const size_t smem = CLayout<T, W, NSLAB, LS>(G, m, S, P, nth).total;
            if (smem > (pass == 0 && force_g == 0 ? kSmemTwoPerSm : kSmemMax)) continue;
            ch.nslab = NSLAB;
            ch.W = W;
            ch.G = G;
            ch.C = C;
            ch.smem = smem;
            break;
        }
    }
    return ch;
}

// One 128-byte slab per CTA. (A two-slab variant with 64-byte rows, so the
// next unit streams in during the whole current one, measured slower on C1 —
// 129 vs 89 us before the segment fix — and was removed.)
CChoice choose(const psw_plan* pl, int layout = PSW_LAYOUT_R) {
    if (layout == PSW_LAYOUT_S)  // fp64 only: 16 rows = one 128-byte swizzle line
        return pl->dtype == PSW_F64 ? choose_t<double, 16, 1, true>(pl) : CChoice{};
    return pl->dtype == PSW_F64 ? choose_t<double, 16, 1>(pl) : choose_t<float, 32, 1>(pl);
}

int box_height(int m) {
    for (int h = kMaxBox; h >= 32; h /= 2)
        if (m % h == 0) return h;
    return 32;
}

// layout S: rows are the contiguous dimension; 16-row boxes of W right-hand
// sides with the 128-byte swizzle (s_index)
bool encode_s(CUtensorMap* tm, CUtensorMap* tm1, const void* F, int64_t N, int64_t n, int64_t ldf,
              int es, int W, int tail) {
    auto enc = tensor_map_encoder();
    if (!enc) {
        set_error(PSW_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        return false;
    }
    const cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(N)};
    const cuuint64_t strides[1] = {cuuint64_t(ldf) * cuuint64_t(es)};
    const cuuint32_t box[2] = {cuuint32_t(128 / es), cuuint32_t(W)};
    const cuuint32_t estr[2] = {1, 1};
    const auto dt = es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const cuuint32_t box1[2] = {cuuint32_t(tail), cuuint32_t(W)};  // the tail rows, unswizzled
    CUresult r = enc(tm, dt, 2, const_cast<void*>(F), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
        r = enc(tm1, dt, 2, const_cast<void*>(F), dims, strides, box1, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error(PSW_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
        return false;
    }
    return true;
}

bool encode(CUtensorMap* tm, CUtensorMap* tm1, CUtensorMap* tm2, const void* F, int64_t N,
            int64_t n, int64_t ldf, int es, int W, int H) {
    auto enc = tensor_map_encoder();
    if (!enc) {
        set_error(PSW_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        return false;
    }
    const cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(n)};
    const cuuint64_t strides[1] = {cuuint64_t(ldf) * cuuint64_t(es)};
    const cuuint32_t box[2] = {cuuint32_t(W), cuuint32_t(H)};
    const cuuint32_t box1[2] = {cuuint32_t(W), 1};
    const cuuint32_t box2[2] = {cuuint32_t(W), cuuint32_t(H - 1)};
    const cuuint32_t estr[2] = {1, 1};
    const auto dt = es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r = enc(tm, dt, 2, const_cast<void*>(F), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
        r = enc(tm1, dt, 2, const_cast<void*>(F), dims, strides, box1, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
        r = enc(tm2, dt, 2, const_cast<void*>(F), dims, strides, box2, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error(PSW_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
        return false;
    }
    return true;
}

// Coefficient tables of every cluster rank in the kernel's shared-memory
// layout (coff), built with the plan for the configuration each layout picks:
// the kernel fetches its rank's table with one bulk copy instead of
// scattering rows, and a solve never writes to the plan.
template <typename T>
int cluster_tables(psw_plan* pl, const CChoice& ch, int layout,
                   const std::vector<FusedFwd<double>>& ff,
                   const std::vector<FusedBwd<double>>& fb) {
    const int G = ch.G, C = ch.C, m = int(pl->m);
    const int ra = G * m + 1;
    const size_t stride = ((coff<T>(ra) + 16 + 127) / 128) * 128;
    std::vector<unsigned char> host(stride * C, 0);
    for (int c = 0; c < C; ++c) {
        const int base = c * G * m - 1;
        const int nrows = c == C - 1 ? G * m + 1 : G * m;
        for (int i = 0; i < nrows; ++i) {
            const int q = base + i;
            if (q < 0 || q >= pl->n) continue;
            Quad<T>* o = reinterpret_cast<Quad<T>*>(host.data() + size_t(c) * stride + coff<T>(i));
            o[0] = {T(ff[q].rp), T(ff[q].ma), T(ff[q].gr), T(ff[q].gl)};
            o[1] = {T(ff[q].lam), T(fb[q].mu), T(fb[q].w), T(fb[q].al)};
        }
    }
    void* d = nullptr;
    PSW_CUDA_TRY(cudaMalloc(&d, host.size()));
    pl->d_ctab[layout] = d;
    pl->ctab_stride[layout] = int64_t(stride);
    PSW_CUDA_TRY(cudaMemcpy(d, host.data(), host.size(), cudaMemcpyHostToDevice));
    pl->info.device_bytes += int64_t(host.size());
    return PSW_OK;
}

template <typename T, int W, int NSLAB, bool LS = false, int V4 = 0>
int launch(const psw_plan* pl, const CChoice& ch, const void* F, int64_t ldf, void* X, int64_t ldx,
           int64_t N, cudaStream_t s, void** ev, int nev) {
    const int lay = LS ? PSW_LAYOUT_S : PSW_LAYOUT_R;
    if (!pl->d_ctab[lay]) {
        set_error(PSW_NOT_SUPPORTED, "cluster tables missing for this layout");
        return PSW_NOT_SUPPORTED;
    }
    CUtensorMap tm, tm1, tm2;
    const int H = box_height(int(pl->m));
    if (LS) {
        // F: 16-row swizzled boxes + the 2-row tail
        if (!encode_s(&tm, &tm1, F, N, pl->n, ldf, int(sizeof(T)), W, 2)) return PSW_CUDA_ERROR;
        tm2 = tm;
    } else if (!encode(&tm, &tm1, &tm2, F, N, pl->n, ldf, int(sizeof(T)), W, H)) {
        return PSW_CUDA_ERROR;
    }
    CGeom g;
    g.n = int(pl->n);
    g.P = int(pl->P);
    g.p = int(pl->p);
    g.m = int(pl->m);
    g.G = ch.G;
    g.C = ch.C;
    g.S = pl->nseg;
    g.H = H;
    g.trace = std::getenv("PSW_CLUSTER_TRACE") ? std::atoi(std::getenv("PSW_CLUSTER_TRACE")) : 0;
    g.N = N;
    g.ldx = ldx;
    g.ntiles = (N + W - 1) / W;
    auto kern = cluster_kernel<T, W, NSLAB, LS, V4>;
    PSW_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ch.smem)));
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(unsigned(ch.G * g.S * W), 1, 1);
    cfg.dynamicSmemBytes = ch.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(ch.C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (ch.C > 8)
        PSW_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    static std::mutex mu;
    static std::vector<std::pair<std::array<int64_t, 5>, int>> cache;
    const std::array<int64_t, 5> key = {int64_t(sizeof(T)) + 16 * NSLAB + 64 * int64_t(LS) + 128 * int64_t(V4), ch.G, ch.C,
                                        int64_t(ch.smem), pl->device};
    int maxc = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (auto& kv : cache)
            if (kv.first == key) maxc = kv.second;
        if (maxc == 0) {
            cfg.gridDim = dim3(unsigned(ch.C), 1, 1);
            PSW_CUDA_TRY(cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg));
            if (maxc < 1) maxc = 1;
            cache.push_back({key, maxc});
        }
    }
    int64_t ncl = std::min<int64_t>((g.ntiles + NSLAB - 1) / NSLAB, maxc);
    if (const char* e = std::getenv("PSW_CLUSTER_CLUSTERS"))  // tuning override
        ncl = std::max<int64_t>(1, std::min<int64_t>(ncl, std::atoll(e)));
    cfg.gridDim = dim3(unsigned(ncl * ch.C), 1, 1);
    if (std::getenv("PSW_CLUSTER_VERBOSE"))
        std::fprintf(stderr, "cluster: W=%d slabs=%d G=%d C=%d S=%d threads=%d smem=%zu max_clusters=%d clusters=%lld\n",
                     W, NSLAB, ch.G, ch.C, g.S, ch.G * g.S * W, ch.smem, maxc, (long long)ncl);
    mark(ev, nev, 0, s);
    PSW_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tm, tm1, tm2, static_cast<const T*>(F), ldf,
                                    static_cast<T*>(X), g,
                                    static_cast<const FusedFwd<T>*>(pl->d_ffwd),
                                    static_cast<const FusedBwd<T>*>(pl->d_fbwd), pl->d_seg,
                                    pl->d_segdesc, pl->d_cmat,
                                    static_cast<const unsigned char*>(pl->d_ctab[lay]),
                                    pl->ctab_stride[lay]));
    mark(ev, nev, 1, s);
    note_launches(1);
    if (g.trace) {
        std::vector<unsigned long long> tr(1024 * kTraceSlots);
        cudaStreamSynchronize(s);
        cudaMemcpyFromSymbol(tr.data(), g_ctrace, sizeof(unsigned long long) * tr.size());
        const char* names[] = {"slab wait", "forward+B1", "scan+push", "exchange wait",
                               "combine+B2+fold+B3", "backward", "  (scan)", "  (push)"};
        const int nb = int(std::min<int64_t>(1024, ncl * ch.C));
        for (int r = 0; r < ch.C && g.trace > 1; ++r) {  // per cluster rank, phases 0..5
            std::fprintf(stderr, "cluster trace rank %d:", r);
            for (int ph = 0; ph < 6; ++ph) {
                std::vector<long long> v;
                for (int b = r; b < nb; b += ch.C)
                    v.push_back((long long)(tr[b * kTraceSlots + ph + 1] - tr[b * kTraceSlots + ph]));
                std::sort(v.begin(), v.end());
                std::fprintf(stderr, " %s %lld |", names[ph], v[v.size() / 2]);
            }
            std::fprintf(stderr, "\n");
        }
        for (int ph = 0; ph < 8; ++ph) {
            // phases: slots 0-1-2-(7)-3-4-5-6; ph 6 = scan (2 -> 7), ph 7 = push (7 -> 3)
            const int a0 = ph == 6 ? 2 : ph == 7 ? 7 : ph, a1 = ph == 6 ? 7 : ph == 7 ? 3 : ph + 1;
            std::vector<long long> v;
            for (int b = 0; b < nb; ++b)
                v.push_back((long long)(tr[b * kTraceSlots + a1] - tr[b * kTraceSlots + a0]));
            std::sort(v.begin(), v.end());
            std::fprintf(stderr, "cluster trace %-22s min %7lld median %7lld  p90 %7lld cycles\n", names[ph],
                         v[0], v[v.size() / 2], v[v.size() * 9 / 10]);
        }
        std::vector<unsigned long long> gt(1024 * 2);
        cudaMemcpyFromSymbol(gt.data(), g_gtrace, sizeof(unsigned long long) * gt.size());
        std::vector<long long> lat, skew;
        for (int c0 = 0; c0 + ch.C <= nb; c0 += ch.C) {
            unsigned long long mx = 0, mn = ~0ull;
            for (int r = 0; r < ch.C; ++r) {
                mx = std::max(mx, gt[(c0 + r) * 2]);
                mn = std::min(mn, gt[(c0 + r) * 2]);
            }
            skew.push_back((long long)(mx - mn));
            for (int r = 0; r < ch.C; ++r) lat.push_back((long long)(gt[(c0 + r) * 2 + 1]) - (long long)mx);
        }
        std::vector<std::vector<long long>> byrank(ch.C);
        for (int c0 = 0; c0 + ch.C <= nb; c0 += ch.C) {
            unsigned long long mn = ~0ull;
            for (int r = 0; r < ch.C; ++r) mn = std::min(mn, gt[(c0 + r) * 2]);
            for (int r = 0; r < ch.C; ++r) byrank[r].push_back((long long)(gt[(c0 + r) * 2] - mn));
        }
        for (int r = 0; r < ch.C; ++r) {
            std::sort(byrank[r].begin(), byrank[r].end());
            std::fprintf(stderr, "cluster trace rank %d push offset (ns): median %lld\n", r,
                         byrank[r][byrank[r].size() / 2]);
        }
        {
            std::vector<unsigned long long> bt(1024 * 8);
            cudaMemcpyFromSymbol(bt.data(), g_btrace, sizeof(unsigned long long) * bt.size());
            std::vector<std::vector<long long>> off(ch.C * ch.G);
            for (int c0 = 0; c0 + ch.C <= nb; c0 += ch.C) {
                unsigned long long mn = ~0ull;
                for (int r = 0; r < ch.C; ++r)
                    for (int jb = 0; jb < ch.G; ++jb) mn = std::min(mn, bt[(c0 + r) * 8 + jb]);
                for (int r = 0; r < ch.C; ++r)
                    for (int jb = 0; jb < ch.G; ++jb)
                        off[r * ch.G + jb].push_back((long long)(bt[(c0 + r) * 8 + jb] - mn));
            }
            std::fprintf(stderr, "cluster trace block push offsets (ns, median) rank x block:");
            for (size_t i = 0; i < off.size(); ++i) {
                std::sort(off[i].begin(), off[i].end());
                std::fprintf(stderr, "%s%lld", i % ch.G ? " " : " | ", off[i][off[i].size() / 2]);
            }
            std::fprintf(stderr, "\n");
        }
        {
            std::vector<unsigned long long> et(1024 * 4);
            cudaMemcpyFromSymbol(et.data(), g_etrace, sizeof(unsigned long long) * et.size());
            unsigned long long t0 = ~0ull;
            for (int b = 0; b < nb; ++b) t0 = std::min(t0, et[b * 4]);
            long long mx[4] = {0, 0, 0, 0}, mnv[4] = {1LL << 60, 1LL << 60, 1LL << 60, 1LL << 60};
            for (int b = 0; b < nb; ++b)
                for (int q = 0; q < 4; ++q) {
                    const long long v = (long long)(et[b * 4 + q] - t0);
                    mx[q] = std::max(mx[q], v);
                    mnv[q] = std::min(mnv[q], v);
                }
            std::fprintf(stderr, "cluster trace timeline (ns from the first CTA): entry %lld..%lld, "
                         "tables ready %lld..%lld, first tile done %lld..%lld, exit %lld..%lld\n",
                         mnv[0], mx[0], mnv[1], mx[1], mnv[2], mx[2], mnv[3], mx[3]);
        }
        std::sort(lat.begin(), lat.end());
        std::sort(skew.begin(), skew.end());
        std::fprintf(stderr, "cluster trace push skew in cluster (ns): median %lld p90 %lld; "
                     "exchange complete after the last push (ns): min %lld median %lld p90 %lld\n",
                     skew[skew.size() / 2], skew[skew.size() * 9 / 10], lat[0], lat[lat.size() / 2],
                     lat[lat.size() * 9 / 10]);
    }
    return PSW_OK;
}

}  // namespace

int build_cluster_tables(psw_plan* pl, const std::vector<FusedFwd<double>>& ff,
                         const std::vector<FusedBwd<double>>& fb) {
    for (int lay : {PSW_LAYOUT_R, PSW_LAYOUT_S}) {
        const CChoice ch = choose(pl, lay);
        if (ch.G <= 0) continue;
        const int rc = pl->dtype == PSW_F64 ? cluster_tables<double>(pl, ch, lay, ff, fb)
                                            : cluster_tables<float>(pl, ch, lay, ff, fb);
        if (rc != PSW_OK) return rc;
    }
    return PSW_OK;
}

bool cluster_supported(const psw_plan* pl, int layout, int64_t N, const void* F, int64_t ldf) {
    if ((layout != PSW_LAYOUT_R && layout != PSW_LAYOUT_S) || N < 1 || N > (int64_t{1} << 31))
        return false;
    const int es = pl->dtype == PSW_F64 ? 8 : 4;
    if ((reinterpret_cast<uintptr_t>(F) & 15) || ((size_t(ldf) * es) & 15)) return false;
    return choose(pl, layout).G > 0;
}

int solve_cluster(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                  int layout, cudaStream_t s, void** ev, int nev) {
    if (!cluster_supported(pl, layout, N, F, ldf)) {
        set_error(PSW_NOT_SUPPORTED,
                  "cluster path needs a uniform partition whose blocks fit a cluster, 16-byte "
                  "aligned F / row pitch, and fp64 for layout S");
        return PSW_NOT_SUPPORTED;
    }
    const CChoice ch = choose(pl, layout);
    if (layout == PSW_LAYOUT_S) {
        if ((reinterpret_cast<uintptr_t>(X) & 31) || ((size_t(ldx) * sizeof(double)) & 31))
            return launch<double, 16, 1, true, 0>(pl, ch, F, ldf, X, ldx, N, s, ev, nev);
        // PSW_CLUSTER_ST=1: per-lane 32-byte stores instead of the whole-line stores
        static const int st = [] {
            const char* e = std::getenv("PSW_CLUSTER_ST");
            return e && *e ? std::atoi(e) : 2;
        }();
        return st == 1 ? launch<double, 16, 1, true, 1>(pl, ch, F, ldf, X, ldx, N, s, ev, nev)
                       : launch<double, 16, 1, true, 2>(pl, ch, F, ldf, X, ldx, N, s, ev, nev);
    }
    return pl->dtype == PSW_F64 ? launch<double, 16, 1>(pl, ch, F, ldf, X, ldx, N, s, ev, nev)
                                : launch<float, 32, 1>(pl, ch, F, ldf, X, ldx, N, s, ev, nev);
}

}  // namespace psw
