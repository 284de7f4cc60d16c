// PIPE solve path: one persistent kernel for any partition with P <= 64
// blocks, both layouts and both dtypes, whose forward intermediates stay in
// L2.
//
// Every block of the partition is cut into segments of <= 33 rows
// (psw_fused.cu build_fused_tables; psw_internal.h FusedFwd/FusedBwd/SegCoef
// give the exact affine carries between segments). RHS are processed in
// chunks of Nc right-hand sides sized so that a chunk's forward
// intermediates (parked in X) stay in L2 next to the streams of F and X: HBM
// sees F read once and X written once, the minimum traffic of SURVEY §8(d).
//
// Work items, one warp each, 32 RHS = one per lane ("group" g of chunk c):
//   A(c,g,s)  forward sweep of segment s from a zero carry (local_solve.hpp:
//             39-48 in the affine form of psw_internal.h): d~ -> X, and the
//             segment partials d~_end, Lam = sum lam d~, the two beta partial
//             dot products (betas.hpp:42-57) -> scratch. The warp finishing
//             the last segment of block t sums the block's betas; the warp
//             finishing the last block of the group runs the dichotomy
//             combination (boundary_solve.hpp:96-121, exact level order) and
//             publishes the boundary values ("last arriver", acq_rel counters);
//   C(c,g,s)  the segment's exact carries (forward fold of D over the
//             block's earlier segments, backward fold of x from x_r down),
//             then the back substitution
//             x_q = d~_q + mu_q D + x_l w_q + al_q x_{q+1} -> X.
// A global ticket counter hands items out in the order
//   round r:  A(r,*)  C(r-L,*)      (lag L >= 1, >= L + 1 scratch slots)
// so every item depends only on items with smaller tickets, held by warps
// that are already running: the persistent grid cannot deadlock. Items are
// short (one segment: <= 33 rows x 32 RHS, all loads in flight at once).
//
// Row movement: layout R (F[i*ld + k]) loads a lane's rows straight into
// registers (each row of a group is one coalesced 256-byte segment); layout S
// (one system per row) goes through a padded shared-memory transpose per warp.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "psw_device.cuh"
#include "psw_internal.h"
#include "psw_tma.cuh"

namespace psw {
namespace {

constexpr int kLanes = 32;             // RHS per group
constexpr int kSegMax = kSegLen + 1;   // rows per segment (max)
constexpr int kTileLd = kSegMax + 2;   // odd row pitch of the S transpose tile
constexpr int kWarps = 8;              // warps per CTA
constexpr int kMaxBlocks = 64;         // block betas / values staged in shared memory
constexpr int kMaxFold = 64;           // segments per block (carry fold scratch)
constexpr int kCoefBytes = kSegMax * 48;  // per-warp staged coefficients (FusedFwd<double> rows)

struct PipeGeom {
    int P, p, NS, NG, nchunks, lag, nslots;
    int tables;    // Z samples + items copied to shared memory (p <= 64)
    int tab_off, bscr_off, lock_off, tile_off, tile_bytes, coef_off;  // shared-memory carve-up (bytes)
    int64_t N, Nc, ldf, ldx, total;
};

struct PipeBuf {
    unsigned long long* head;
    int* blkcnt;    // [nchunks * NG][P] finished A items per block
    int* grpcnt;    // [nchunks * NG] blocks with their betas summed
    int* flagB;     // [nchunks * NG] boundary values ready
    int* doneC;     // [nchunks * NG] finished C items
    double* part;   // [nslots][NS][4][Nc]: d~_end, Lam, beta_R, beta_L
    double* bb;     // [nslots][P][2][Nc]: block betas left, right
    double* V;      // [nslots][max(p, 1)][Nc]
};

struct PipeTabs {
    const SegDesc* desc;    // [NS] rows [a, b) of block t
    const int32_t* segoff;  // [P + 1]
    const SegCoef* segc;    // [NS]
    const void* ff;         // FusedFwd<T>[n]
    const void* fb;         // FusedBwd<T>[n]
    const CombineItem* items;
    const double* zr;
    const double* zl;
};

// Optional item trace (psw_debug_trace): 8 x u64 per ticket = start, ready
// (dependencies met), end (%globaltimer ns), (type << 32 | smid).
__device__ unsigned long long* g_pipe_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Lane 0 polls with relaxed loads (an acquire per poll would invalidate the
// SM's L1 on every iteration and stall the other warps' traffic), then one
// acquire fence; __syncwarp extends the ordering to the other lanes.
__device__ __forceinline__ void wait_geq(const int* flag, int target, int lane) {
    if (lane == 0) {
        if (ld_relaxed_gpu(flag) < target) {
            int ns = 32;
            while (ld_relaxed_gpu(flag) < target) {
                __nanosleep(ns);
                ns = ns < 512 ? 2 * ns : ns;
            }
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncwarp();
}

__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
                 : "memory");
    return old;
}

// ---- row movement: a segment of the group's RHS <-> the lanes' registers --
// Layout R: lane = RHS, rows at stride ld (coalesced across the warp).
template <typename T>
__device__ __forceinline__ void load_r(const T* src, int64_t ld, int len, bool kv,
                                       T (&v)[kSegMax], bool streaming) {
#pragma unroll
    for (int r = 0; r < kSegMax; ++r)
        v[r] = (kv && r < len) ? (streaming ? __ldcs(src + r * ld) : __ldcg(src + r * ld)) : T(0);
}
// Layout S: lanes along the rows of one RHS at a time into the warp's tile,
// then each lane takes its RHS' column (odd pitch: conflict-free).
template <typename T>
__device__ __forceinline__ void load_s(const T* src, int64_t ld, int len, int nk, int lane,
                                       T* tile, T (&v)[kSegMax], bool streaming) {
#pragma unroll 8
    for (int j = 0; j < kLanes; ++j) {
        if (j < nk) {
            const T* col = src + int64_t(j) * ld;
            if (lane < len)
                tile[j * kTileLd + lane] = streaming ? __ldcs(col + lane) : __ldcg(col + lane);
            if (lane + kLanes < len)
                tile[j * kTileLd + lane + kLanes] =
                    streaming ? __ldcs(col + lane + kLanes) : __ldcg(col + lane + kLanes);
        }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kSegMax; ++r) v[r] = tile[lane * kTileLd + r];
    __syncwarp();
}
template <typename T>
__device__ __forceinline__ void store_s(T* dst, int64_t ld, int len, int nk, int lane, T* tile,
                                        const T (&v)[kSegMax], bool streaming) {
#pragma unroll
    for (int r = 0; r < kSegMax; ++r) tile[lane * kTileLd + r] = v[r];
    __syncwarp();
#pragma unroll 8
    for (int j = 0; j < kLanes; ++j) {
        if (j < nk) {
            T* col = dst + int64_t(j) * ld;
            if (lane < len) {
                if (streaming) __stcs(col + lane, tile[j * kTileLd + lane]);
                else col[lane] = tile[j * kTileLd + lane];
            }
            if (lane + kLanes < len) {
                if (streaming) __stcs(col + lane + kLanes, tile[j * kTileLd + lane + kLanes]);
                else col[lane + kLanes] = tile[j * kTileLd + lane + kLanes];
            }
        }
    }
    __syncwarp();
}

// A segment's sweep coefficients into the warp's shared scratch, one row per
// lane (16-byte pieces, one round trip for all rows): the recurrences then
// read them as conflict-free broadcasts instead of dependent cached loads.
template <typename C>
__device__ __forceinline__ const C* stage_coef(const C* src, int len, int lane, C* dst) {
    static_assert(sizeof(C) % 16 == 0, "16-byte rows");
    constexpr int kPieces = int(sizeof(C) / 16);
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int row = lane; row < len; row += kLanes) {
#pragma unroll
        for (int k = 0; k < kPieces; ++k) d[row * kPieces + k] = __ldg(s + row * kPieces + k);
    }
    return dst;
}

template <typename T, int LAYOUT>
__global__ void __launch_bounds__(kWarps * 32, 2) pipe_kernel(const T* F, T* X, const PipeGeom g,
                                                              const PipeBuf b, PipeTabs tb) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int P = g.P, p = g.p, NG = g.NG, NS = g.NS;
    const CombineItem* items = tb.items;
    const double* zr = tb.zr;
    const double* zl = tb.zl;
    if (g.tables) {
        // combination tables once per CTA in shared memory: the combination
        // never waits on global loads behind the saturated streams
        double* szr = reinterpret_cast<double*>(smem + g.tab_off);
        double* szl = szr + p * p;
        CombineItem* sit = reinterpret_cast<CombineItem*>(szl + p * p);
        for (int i = threadIdx.x; i < p * p; i += blockDim.x) {
            szr[i] = zr[i];
            szl[i] = zl[i];
        }
        for (int i = threadIdx.x; i < p; i += blockDim.x) sit[i] = items[i];
        zr = szr;
        zl = szl;
        items = sit;
    }
    int* const block_lock = reinterpret_cast<int*>(smem + g.lock_off);
    if (threadIdx.x == 0) *block_lock = 0;
    // per-warp scratch: the S transpose tile, reused for the carry fold
    T* const tile = reinterpret_cast<T*>(smem + g.tile_off + size_t(warp) * g.tile_bytes);
    double* const dfold = reinterpret_cast<double*>(tile);
    unsigned char* const coef_s = smem + g.coef_off + size_t(warp) * kCoefBytes;
    __syncthreads();
    const auto* ffw = static_cast<const FusedFwd<T>*>(tb.ff);
    const auto* fbw = static_cast<const FusedBwd<T>*>(tb.fb);
    const int64_t RS = int64_t(NG) * 2 * int64_t(NS);
    const int64_t Nc = g.Nc;
    const int L = g.lag, NSL = g.nslots;

    long long it = 0;
    if (lane == 0) it = static_cast<long long>(atomicAdd(b.head, 1ULL));
    it = __shfl_sync(0xffffffffu, it, 0);
    unsigned long long* const trace = g_pipe_trace;
    while (it < g.total) {
        long long nxt = 0;
        unsigned long long* tr = trace && lane == 0 ? trace + 8 * it : nullptr;
        if (tr) tr[0] = gtimer_ns();
        if (lane == 0) nxt = static_cast<long long>(atomicAdd(b.head, 1ULL));
        const int r = int(it / RS);
        const int64_t pos = it % RS;
        if (pos < int64_t(NG) * NS) {
            // ---------------- A(r, g, s): forward sweep of one segment
            // segment-major: the groups of a chunk read the same rows together,
            // so DRAM sees Nc * s contiguous bytes per row instead of 256
            const int c = r, grp = int(pos % NG), s = int(pos / NG);
            const int64_t k0 = int64_t(c) * Nc + int64_t(grp) * kLanes;
            if (c < g.nchunks && k0 < g.N) {
                const int q = c * NG + grp, slot = c % NSL;
                if (c >= NSL) wait_geq(b.doneC + (q - NSL * NG), NS, lane);  // slot drained
                if (tr) tr[1] = gtimer_ns(), tr[3] = (0ull << 32) | smid();
                const SegDesc sd = tb.desc[s];
                const int len = sd.b - sd.a, t = sd.t;
                const bool kv = k0 + lane < g.N;
                const int nk = g.N - k0 < kLanes ? int(g.N - k0) : kLanes;
                const int64_t kl = int64_t(grp) * kLanes + lane;
                T v[kSegMax];
                if constexpr (LAYOUT == PSW_LAYOUT_R)
                    load_r(F + int64_t(sd.a) * g.ldf + k0 + lane, g.ldf, len, kv, v, true);
                else
                    load_s(F + k0 * g.ldf + sd.a, g.ldf, len, nk, lane, tile, v, true);
                const FusedFwd<T>* cf =
                    stage_coef(ffw + sd.a, len, lane, reinterpret_cast<FusedFwd<T>*>(coef_s));
                __syncwarp();
                T d = T(0);
                double sR = 0.0, sL = 0.0, sX = 0.0;
#pragma unroll
                for (int rr = 0; rr < kSegMax; ++rr) {
                    if (rr < len) {
                        const FusedFwd<T> cc = cf[rr];
                        const T f = v[rr];
                        d = fma(cc.ma, d, f * cc.rp);
                        sR = fma(double(f), double(cc.gr), sR);
                        sL = fma(double(f), double(cc.gl), sL);
                        sX = fma(double(cc.lam), double(d), sX);
                        v[rr] = d;
                    }
                }
                if constexpr (LAYOUT == PSW_LAYOUT_R) {
                    if (kv) {
                        T* xp = X + int64_t(sd.a) * g.ldx + k0 + lane;
#pragma unroll
                        for (int rr = 0; rr < kSegMax; ++rr)
                            if (rr < len) xp[rr * g.ldx] = v[rr];
                    }
                } else {
                    store_s(X + k0 * g.ldx + sd.a, g.ldx, len, nk, lane, tile, v, false);
                }
                double* part = b.part + int64_t(slot) * NS * 4 * Nc + kl;
                if (kv) {
                    double* ps = part + int64_t(s) * 4 * Nc;
                    ps[0] = double(d);
                    ps[Nc] = sX;
                    ps[2 * Nc] = sR;
                    ps[3 * Nc] = sL;
                }
                // the last segment of block t to finish sums the block betas;
                // the last block of the group to finish runs the combination
                int last = 0;
                __syncwarp();
                if (lane == 0) {
                    const int s0 = tb.segoff[t], s1 = tb.segoff[t + 1];
                    last = atom_add_acq_rel(b.blkcnt + int64_t(q) * P + t, 1) == s1 - s0 - 1;
                }
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    const int s0 = tb.segoff[t], s1 = tb.segoff[t + 1];
                    double bR = 0.0, bL = 0.0;
                    if (kv) {
#pragma unroll 8
                        for (int sg = s0; sg < s1; ++sg) {
                            bR += __ldcg(part + int64_t(sg) * 4 * Nc + 2 * Nc);
                            bL += __ldcg(part + int64_t(sg) * 4 * Nc + 3 * Nc);
                        }
                        double* bb = b.bb + (int64_t(slot) * 2 * P + 2 * t) * Nc + kl;
                        bb[0] = bL;
                        bb[Nc] = bR;
                    }
                    __syncwarp();
                    int lastb = 0;
                    if (lane == 0) lastb = atom_add_acq_rel(b.grpcnt + q, 1) == P - 1;
                    lastb = __shfl_sync(0xffffffffu, lastb, 0);
                    if (lastb) {
                        // the group's combination in the CTA's shared scratch
                        // (one at a time per CTA): betas staged with all loads in
                        // flight, exact level-order dichotomy, values -> V
                        if (lane == 0)
                            while (atomicCAS(block_lock, 0, 1) != 0) __nanosleep(64);
                        __syncwarp();
                        double* sl = reinterpret_cast<double*>(smem + g.bscr_off) + lane;
                        double* sr = sl + P * kLanes;
                        double* sv = sr + P * kLanes;
                        if (kv && p > 0) {
                            const double* bb = b.bb + int64_t(slot) * 2 * P * Nc + kl;
#pragma unroll 8
                            for (int tt = 0; tt < P; ++tt) {
                                sl[tt * kLanes] = __ldcg(bb + int64_t(2 * tt) * Nc);
                                sr[tt * kLanes] = __ldcg(bb + int64_t(2 * tt + 1) * Nc);
                            }
                            combine_rhs(items, p, sl, sr, kLanes, zr, zl, sv, kLanes);
                            double* V = b.V + int64_t(slot) * p * Nc + kl;
                            for (int j = 0; j < p; ++j) V[int64_t(j) * Nc] = sv[j * kLanes];
                        }
                        __syncwarp();
                        if (lane == 0) {
                            atomicExch(block_lock, 0);
                            red_release_add(b.flagB + q, 1);
                        }
                    }
                }
            }
        } else {
            // ---------------- C(r-L, g, s): back substitution of one segment
            const int64_t idx = pos - int64_t(NG) * NS;
            const int c = r - L, grp = int(idx % NG), s = int(idx / NG);
            const int64_t k0 = int64_t(c) * Nc + int64_t(grp) * kLanes;
            if (c >= 0 && k0 < g.N) {
                const int q = c * NG + grp, slot = c % NSL;
                wait_geq(b.flagB + q, 1, lane);
                if (tr) tr[1] = gtimer_ns(), tr[3] = (2ull << 32) | smid();
                const SegDesc sd = tb.desc[s];
                const int len = sd.b - sd.a, t = sd.t;
                const int s0 = tb.segoff[t], s1 = tb.segoff[t + 1];
                const bool kv = k0 + lane < g.N;
                const int nk = g.N - k0 < kLanes ? int(g.N - k0) : kLanes;
                const int64_t kl = int64_t(grp) * kLanes + lane;
                // d~ of the segment in flight first, then the carries
                T v[kSegMax];
                if constexpr (LAYOUT == PSW_LAYOUT_R)
                    load_r(X + int64_t(sd.a) * g.ldx + k0 + lane, g.ldx, len, kv, v, false);
                else
                    load_s(X + k0 * g.ldx + sd.a, g.ldx, len, nk, lane, tile, v, false);
                // exact carries (psw_internal.h): forward fold over the block's
                // segments D_{a-1}, backward fold from x_r down to this segment
                double D = 0.0, x = 0.0, xl = 0.0;
                if (kv) {
                    const double* part = b.part + int64_t(slot) * NS * 4 * Nc + kl;
                    const double* V = b.V + int64_t(slot) * max(p, 1) * Nc + kl;
                    xl = t > 0 ? __ldcg(V + int64_t(t - 1) * Nc) : 0.0;
                    x = t < p ? __ldcg(V + int64_t(t) * Nc) : 0.0;
                    double Dc = 0.0;
#pragma unroll 8
                    for (int sg = s0; sg < s1; ++sg) {
                        if (sg == s) D = Dc;
                        if (sg > s) dfold[(sg - s0) * kLanes + lane] = Dc;
                        Dc = fma(tb.segc[sg].mu_end, Dc, __ldcg(part + int64_t(sg) * 4 * Nc));
                    }
#pragma unroll 4
                    for (int sg = s1 - 1; sg > s; --sg) {
                        const SegCoef sc = tb.segc[sg];
                        const double lam = __ldcg(part + int64_t(sg) * 4 * Nc + Nc);
                        x = fma(sc.nu, x, fma(xl, sc.k2, fma(dfold[(sg - s0) * kLanes + lane], sc.k1, lam)));
                    }
                }
                __syncwarp();
                const T Dt = T(D), xlt = T(xl);
                T xn = T(x);
                const FusedBwd<T>* cb =
                    stage_coef(fbw + sd.a, len, lane, reinterpret_cast<FusedBwd<T>*>(coef_s));
                __syncwarp();
#pragma unroll
                for (int rr = kSegMax - 1; rr >= 0; --rr) {
                    if (rr < len) {
                        const FusedBwd<T> cc = cb[rr];
                        const T cq = fma(xlt, cc.w, fma(cc.mu, Dt, v[rr]));
                        xn = fma(cc.al, xn, cq);
                        v[rr] = xn;
                    }
                }
                if constexpr (LAYOUT == PSW_LAYOUT_R) {
                    if (kv) {
                        T* xp = X + int64_t(sd.a) * g.ldx + k0 + lane;
#pragma unroll
                        for (int rr = 0; rr < kSegMax; ++rr)
                            if (rr < len) __stcs(xp + rr * g.ldx, v[rr]);
                    }
                } else {
                    store_s(X + k0 * g.ldx + sd.a, g.ldx, len, nk, lane, tile, v, true);
                }
                __syncwarp();
                if (lane == 0) red_release_add(b.doneC + q, 1);
            }
        }
        if (tr) tr[2] = gtimer_ns();
        it = __shfl_sync(0xffffffffu, nxt, 0);
    }
}

// ------------------------------------------------------------- host
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

struct PipeConfig {
    int lag = 1, nslots = 2;
    bool tables = false;
    int tab_off = 0, bscr_off = 0, lock_off = 0, tile_off = 0, tile_bytes = 0, coef_off = 0;
    size_t smem = 0;
    int64_t Nc = 0;
};

int max_segments_per_block(const psw_plan* pl) {
    int mx = 0;
    for (size_t t = 0; t + 1 < pl->seg_off.size(); ++t)
        mx = std::max(mx, pl->seg_off[t + 1] - pl->seg_off[t]);
    return mx;
}

template <typename T, int LAYOUT>
PipeConfig pipe_config(const psw_plan* pl, int64_t N) {
    PipeConfig c;
    const int64_t P = pl->P, p = pl->p;
    // shared memory: [combination tables][block betas + values][lock][per-warp scratch]
    size_t off = 0;
    c.tables = p > 0 && p <= kMaxBlocks;
    c.tab_off = 0;
    if (c.tables) off += size_t(2 * p * p) * sizeof(double) + size_t(p) * sizeof(CombineItem);
    off = (off + 127) & ~size_t(127);
    c.bscr_off = int(off);
    off += size_t(3 * P) * kLanes * sizeof(double);
    c.lock_off = int(off);
    off = (off + 16 + 127) & ~size_t(127);
    c.tile_off = int(off);
    // per warp: the S transpose tile and the carry fold (S_t doubles per lane)
    const size_t tile = LAYOUT == PSW_LAYOUT_S ? size_t(kLanes) * kTileLd * sizeof(T) : 0;
    const size_t fold = size_t(max_segments_per_block(pl)) * kLanes * sizeof(double);
    c.tile_bytes = int((std::max(tile, fold) + 127) & ~size_t(127));
    off += size_t(kWarps) * c.tile_bytes;
    c.coef_off = int(off);
    off += size_t(kWarps) * kCoefBytes;
    c.smem = off;
    c.lag = std::max(1, std::min(4, env_int("PSW_PIPE_LAG", 1)));
    c.nslots = std::max(c.lag + 1, env_int("PSW_PIPE_SLOTS", 3));
    // chunk: forward intermediates of Nc RHS (n * Nc * s bytes) resident in L2
    const double mb = std::max(1, env_int("PSW_PIPE_CHUNK_MB", 16));
    const int64_t per_rhs = pl->n * int64_t(sizeof(T));
    int64_t nc = int64_t(mb * 1048576.0 / double(per_rhs)) / kLanes * kLanes;
    nc = std::max<int64_t>(kLanes, nc);
    nc = std::min<int64_t>(nc, (N + kLanes - 1) / kLanes * kLanes);
    c.Nc = nc;
    return c;
}

template <typename T, int LAYOUT>
int launch_pipe(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                cudaStream_t s, void** ev, int nev) {
    const PipeConfig pc = pipe_config<T, LAYOUT>(pl, N);
    const int64_t NS = pl->seg_off.back();
    PipeGeom g;
    g.P = int(pl->P);
    g.p = int(pl->p);
    g.NS = int(NS);
    g.NG = int(pc.Nc / kLanes);
    g.nchunks = int((N + pc.Nc - 1) / pc.Nc);
    g.lag = pc.lag;
    g.nslots = pc.nslots;
    g.tables = pc.tables ? 1 : 0;
    g.tab_off = pc.tab_off;
    g.bscr_off = pc.bscr_off;
    g.lock_off = pc.lock_off;
    g.tile_off = pc.tile_off;
    g.tile_bytes = pc.tile_bytes;
    g.coef_off = pc.coef_off;
    g.N = N;
    g.Nc = pc.Nc;
    g.ldf = ldf;
    g.ldx = ldx;
    g.total = int64_t(g.nchunks + g.lag) * g.NG * 2 * NS;
    PipeTabs tb;
    tb.desc = pl->d_segdesc;
    tb.segoff = pl->d_segoff;
    tb.segc = pl->d_seg;
    tb.ff = pl->d_ffwd;
    tb.fb = pl->d_fbwd;
    tb.items = pl->d_items;
    tb.zr = pl->d_zr;
    tb.zl = pl->d_zl;

    // scratch: ticket + counters (zeroed) | segment partials | block betas | values
    const size_t ncnt = size_t(g.nchunks) * g.NG;
    const size_t cnt_bytes = (8 + (ncnt * (3 + size_t(g.P))) * sizeof(int) + 255) & ~size_t(255);
    const size_t part_bytes = sizeof(double) * g.nslots * size_t(NS) * 4 * pc.Nc;
    const size_t bb_bytes = sizeof(double) * g.nslots * size_t(g.P) * 2 * pc.Nc;
    const size_t v_bytes = sizeof(double) * g.nslots * size_t(std::max(g.p, 1)) * pc.Nc;
    void* scratch = nullptr;
    PSW_CUDA_TRY(cudaMallocAsync(&scratch, cnt_bytes + part_bytes + bb_bytes + v_bytes, s));
    char* cp = static_cast<char*>(scratch);
    PipeBuf b;
    b.head = reinterpret_cast<unsigned long long*>(cp);
    b.blkcnt = reinterpret_cast<int*>(cp + 8);
    b.grpcnt = b.blkcnt + ncnt * g.P;
    b.flagB = b.grpcnt + ncnt;
    b.doneC = b.flagB + ncnt;
    b.part = reinterpret_cast<double*>(cp + cnt_bytes);
    b.bb = reinterpret_cast<double*>(cp + cnt_bytes + part_bytes);
    b.V = reinterpret_cast<double*>(cp + cnt_bytes + part_bytes + bb_bytes);
    int rc = PSW_OK;
    mark(ev, nev, 0, s);
    cudaError_t e = cudaMemsetAsync(scratch, 0, cnt_bytes, s);
    if (e == cudaSuccess) {
        auto kern = pipe_kernel<T, LAYOUT>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pc.smem));
        int dev = 0, nsm = 0, occ = 0;
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWarps * 32, pc.smem);
        if (e == cudaSuccess && occ < 1) e = cudaErrorInvalidConfiguration;
        if (e == cudaSuccess) {
            if (const int eo = env_int("PSW_PIPE_CTAS_PER_SM", 0)) occ = std::min(occ, eo);
            const int64_t grid =
                std::min<int64_t>(int64_t(nsm) * occ, (g.total + kWarps - 1) / kWarps);
            kern<<<unsigned(grid), unsigned(kWarps * 32), pc.smem, s>>>(
                static_cast<const T*>(F), static_cast<T*>(X), g, b, tb);
            e = cudaGetLastError();
            mark(ev, nev, 1, s);
        }
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "pipe_kernel launch");
    else note_launches(1);
    cudaFreeAsync(scratch, s);
    return rc;
}

}  // namespace

int set_pipe_trace(void* buf) {
    unsigned long long* q = static_cast<unsigned long long*>(buf);
    PSW_CUDA_TRY(cudaMemcpyToSymbol(g_pipe_trace, &q, sizeof(q)));
    return PSW_OK;
}

bool pipe_supported(const psw_plan* pl, int layout, int64_t N, const void*, int64_t,
                    const void*, int64_t) {
    if (pl->world != 1 || N < 1 || N >= (int64_t{1} << 31) || pl->n >= (int64_t{1} << 31))
        return false;
    if (!pl->d_segdesc || pl->seg_off.empty() || pl->P > kMaxBlocks) return false;
    // the carry fold keeps a block's forward carries in the warp's scratch
    if (max_segments_per_block(pl) > kMaxFold) return false;
    return layout == PSW_LAYOUT_R || layout == PSW_LAYOUT_S;
}

int solve_pipe(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
               int layout, cudaStream_t s, void** ev, int nev) {
    if (pl->dtype == PSW_F64)
        return layout == PSW_LAYOUT_R
                   ? launch_pipe<double, PSW_LAYOUT_R>(pl, F, ldf, X, ldx, N, s, ev, nev)
                   : launch_pipe<double, PSW_LAYOUT_S>(pl, F, ldf, X, ldx, N, s, ev, nev);
    return layout == PSW_LAYOUT_R
               ? launch_pipe<float, PSW_LAYOUT_R>(pl, F, ldf, X, ldx, N, s, ev, nev)
               : launch_pipe<float, PSW_LAYOUT_S>(pl, F, ldf, X, ldx, N, s, ev, nev);
}

}  // namespace psw
