// PIPE solve path: one persistent kernel for any partition, both layouts and
// both dtypes, whose forward intermediates stay in L2.
//
// The STAGED algorithm (psw_staged.cu: block forward sweep + betas, the exact
// dichotomy combination, block back substitution; bitwise the same
// arithmetic) is cut into work items over RHS chunks of Nc right-hand sides
// sized so that a chunk's forward intermediates d (parked in X, like STAGED)
// fit in L2 next to the streams of F and X. HBM then sees F read once and X
// written once (the d round trip is served by L2), i.e. the minimum traffic
// of SURVEY §8(d), without the on-chip capacity limit of the FUSED kernel.
//
// Items (one warp each, 32 RHS = one per lane, "group" g of chunk c):
//   A(c,g,t)  forward sweep of block t (local_solve.hpp:39-48 in the affine
//             form of psw_internal.h) + both beta dot products
//             (betas.hpp:42-57), d -> X, betas -> scratch;
//   B(c,g)    dichotomy combination for the group's RHS
//             (boundary_solve.hpp:96-121) once all P blocks' A items are in;
//   C(c,g,t)  back substitution of block t once B(c,g) is in, x -> X.
// A global ticket counter hands items out in the order
//   round r:  B(r-1,*)  A(r,*)  C(r-1,*)
// so each item depends only on items with smaller tickets, held by warps
// that are already running: the persistent grid cannot deadlock, and a
// chunk's combination runs while the next chunk's forward sweeps stream.
// Completion is published with release/acquire counters in global memory.
//
// Rows move by TMA: 32-row x 32-RHS boxes (layout R: 32 x 32 rows of one
// group; layout S: 128-byte-swizzled boxes along the system so the per-lane
// column reads are conflict-free) plus a bulk copy of the 32 rows' sweep
// coefficients, K stages deep per warp, one mbarrier per stage. Results are
// stored with coalesced generic stores (layout S through the tile).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "psw_device.cuh"
#include "psw_internal.h"
#include "psw_tma.cuh"

namespace psw {
namespace {

constexpr int kRows = 32;         // rows per stage (one box)
constexpr int kLanes = 32;        // RHS per group
constexpr int kCoefBytes = 1024;  // coefficient slot per stage (32 rows x <= 32 B)
constexpr int kMaxWarps = 8;
constexpr int kLayoutSPlain = 2;  // layout S, unswizzled tiles (diagnostic, PSW_PIPE_PLAIN_S)

struct PipeGeom {
    int P, p, NG, K, nchunks, warp_bytes, stage_b;
    int64_t N, Nc, ldx, total;
};

struct PipeBuf {
    unsigned long long* head;
    int* doneA;   // [nchunks * NG] finished A items
    int* flagB;   // [nchunks * NG] B item finished
    int* doneC;   // [nchunks * NG] finished C items
    double* bet;  // [2 slots][2: left, right][P][Nc]
    double* V;    // [2 slots][max(p, 1)][Nc]
};

template <typename T, int LAYOUT>
struct TileMap {
    static constexpr int kBytes = kRows * kLanes * int(sizeof(T));
    static constexpr int kQB = 128 / int(sizeof(T));  // rows per 128-byte swizzle row (S)
    static constexpr int kE = 16 / int(sizeof(T));
    static constexpr int kBoxes = LAYOUT == PSW_LAYOUT_S ? kRows / kQB : 1;
    // element (rhs j, row r) of a stage tile
    __device__ __forceinline__ static T* at(unsigned char* tile, int j, int r) {
        if constexpr (LAYOUT == PSW_LAYOUT_R) {
            return reinterpret_cast<T*>(tile) + r * kLanes + j;
        } else if constexpr (LAYOUT == kLayoutSPlain) {
            return reinterpret_cast<T*>(tile) + j * kRows + r;
        } else {
            const int off = (r / kQB) * (kLanes * 128) + j * 128 +
                            ((((r % kQB) / kE) ^ (j & 7)) << 4) + (r % kE) * int(sizeof(T));
            return reinterpret_cast<T*>(tile + off);
        }
    }
    // lane 0: stage load of rows [q0, q0 + 32) x RHS [k0, k0 + 32) + coefficients
    __device__ __forceinline__ static void issue(unsigned char* tile, void* coef, const void* csrc,
                                                 uint32_t cbytes, uint64_t* bar,
                                                 const CUtensorMap* map, int64_t k0, int q0,
                                                 uint64_t pol) {
        mbar_expect_tx(bar, uint32_t(kBytes) + cbytes);
        if constexpr (LAYOUT == PSW_LAYOUT_R) {
            tma_load_2d_hint(tile, map, int(k0), q0, bar, pol);
        } else if constexpr (LAYOUT == kLayoutSPlain) {
            tma_load_2d_hint(tile, map, q0, int(k0), bar, pol);
        } else {
#pragma unroll
            for (int b = 0; b < kBoxes; ++b)
                tma_load_2d_hint(tile + b * (kLanes * 128), map, q0 + b * kQB, int(k0), bar, pol);
        }
        bulk_load(coef, csrc, cbytes, bar);
    }
};

// Optional item trace (psw_debug_trace): 4 x u64 per ticket = start, ready
// (dependencies met), end (%globaltimer ns) and (type << 32 | smid).
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

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// every lane spins (each lane's own acquire orders its later loads)
__device__ __forceinline__ void wait_geq(const int* flag, int target) {
    while (ld_acquire_gpu(flag) < target) __nanosleep(32);
}

// publish this warp's global writes, then bump the counter
__device__ __forceinline__ void publish(int* counter, int lane) {
    __threadfence();
    __syncwarp();
    if (lane == 0) red_release_add(counter, 1);
}

template <typename T, int LAYOUT>
struct PipeWarp {
    using TM = TileMap<T, LAYOUT>;
    unsigned char* tiles;
    unsigned char* coefs;
    uint64_t* bars;
    uint32_t seq;  // stages consumed so far (ring position and parity)
    int K, lane;

    __device__ __forceinline__ unsigned char* tile(uint32_t sq) const {
        return tiles + (sq % K) * TM::kBytes;
    }
    __device__ __forceinline__ unsigned char* coef(uint32_t sq) const {
        return coefs + (sq % K) * kCoefBytes;
    }
    __device__ __forceinline__ uint64_t* bar(uint32_t sq) const { return bars + (sq % K); }
    __device__ __forceinline__ void wait(uint32_t sq) const { mbar_wait(bar(sq), (sq / K) & 1); }

    // tile rows [lo, hi) -> X rows q0 + r, coalesced: for each RHS j of the
    // group the lanes write consecutive rows of its system (layout S)
    __device__ __forceinline__ void store_s(unsigned char* tl, T* X, int64_t ldx, int64_t k0,
                                            int64_t N, int q0, int lo, int hi, bool stream) const {
        if (lane >= lo && lane < hi) {
#pragma unroll 4
            for (int j = 0; j < kLanes; ++j) {
                if (k0 + j >= N) break;
                T* dst = X + (k0 + j) * ldx + q0 + lane;
                const T v = *TM::at(tl, j, lane);
                if (stream) __stcs(dst, v);
                else *dst = v;
            }
        }
    }

    // Stage grid of block rows [s, e): stage i holds rows [sa + 32 i, +32)
    // with sa = s rounded down to 16 bytes (TMA needs 16-byte aligned starts
    // along the contiguous dimension, which is the row index in layout S).
    static constexpr int kAlign = LAYOUT == PSW_LAYOUT_R ? 1 : 16 / int(sizeof(T));

    // A(c, g, t): forward sweep + betas of block rows [s, e)
    __device__ __forceinline__ void fwd(const CUtensorMap* tmF, T* X, int64_t ldx, int64_t N,
                                        int64_t k0, int s, int e, const FwdCoef<T>* cf,
                                        uint64_t pol, double& br, double& bl) {
        const int sa = s - s % kAlign;
        const int nst = (e - sa + kRows - 1) / kRows;
        const uint32_t cb = uint32_t(kRows * sizeof(FwdCoef<T>));
        if (lane == 0)
            for (int i = 0; i < nst && i < K; ++i)
                TM::issue(tile(seq + i), coef(seq + i), cf + sa + i * kRows, cb, bar(seq + i),
                          tmF, k0, sa + i * kRows, pol);
        const bool kv = k0 + lane < N;
        T d = T(0);
        br = 0.0;
        bl = 0.0;
        for (int i = 0; i < nst; ++i) {
            const uint32_t sq = seq + i;
            wait(sq);
            unsigned char* tl = tile(sq);
            const FwdCoef<T>* cs = reinterpret_cast<const FwdCoef<T>*>(coef(sq));
            const int q0 = sa + i * kRows;
            const int lo = i == 0 ? s - sa : 0;
            const int hi = min(kRows, e - q0);
            T* xr = X + int64_t(q0) * ldx + k0 + lane;
            auto step = [&](int r) {
                T* slot = TM::at(tl, lane, r);
                const T fv = *slot;
                const FwdCoef<T> c = cs[r];
                d = fma(c.ma, d, fv * c.rp);
                br = madd_rn(br, double(fv), double(c.gr));
                bl = madd_rn(bl, double(fv), double(c.gl));
                if constexpr (LAYOUT == PSW_LAYOUT_R) {
                    if (kv) xr[int64_t(r) * ldx] = d;
                } else {
                    *slot = d;
                }
            };
            if (lo == 0 && hi == kRows) {
#pragma unroll
                for (int r = 0; r < kRows; ++r) step(r);
            } else {
                for (int r = lo; r < hi; ++r) step(r);
            }
            __syncwarp();
            if constexpr (LAYOUT != PSW_LAYOUT_R) {
                store_s(tl, X, ldx, k0, N, q0, lo, hi, false);
                __syncwarp();
            }
            if (lane == 0 && i + K < nst) {
                fence_proxy_async_smem();
                TM::issue(tile(sq), coef(sq), cf + sa + (i + K) * kRows, cb, bar(sq), tmF, k0,
                          sa + (i + K) * kRows, pol);
            }
        }
        seq += nst;
    }

    // C(c, g, t): back substitution of block rows [s, e) from x_r, with x_l
    __device__ __forceinline__ void bwd(const CUtensorMap* tmX, T* X, int64_t ldx, int64_t N,
                                        int64_t k0, int s, int e, const BwdCoef<T>* cbw, T xl,
                                        T x, uint64_t pol) {
        const int sa = s - s % kAlign;
        const int nst = (e - sa + kRows - 1) / kRows;
        const uint32_t cb = uint32_t(kRows * sizeof(BwdCoef<T>));
        if (lane == 0)
            for (int i = 0; i < nst && i < K; ++i) {
                const int bs = nst - 1 - i;
                TM::issue(tile(seq + i), coef(seq + i), cbw + sa + bs * kRows, cb, bar(seq + i),
                          tmX, k0, sa + bs * kRows, pol);
            }
        const bool kv = k0 + lane < N;
        for (int i = 0; i < nst; ++i) {
            const uint32_t sq = seq + i;
            wait(sq);
            unsigned char* tl = tile(sq);
            const BwdCoef<T>* cs = reinterpret_cast<const BwdCoef<T>*>(coef(sq));
            const int bs = nst - 1 - i;
            const int q0 = sa + bs * kRows;
            const int lo = bs == 0 ? s - sa : 0;
            const int hi = min(kRows, e - q0);
            T* xr = X + int64_t(q0) * ldx + k0 + lane;
            auto step = [&](int r) {
                T* slot = TM::at(tl, lane, r);
                const BwdCoef<T> c = cs[r];
                x = fma(c.al, x, fma(xl, c.w, *slot));
                if constexpr (LAYOUT == PSW_LAYOUT_R) {
                    if (kv) __stcs(xr + int64_t(r) * ldx, x);
                } else {
                    *slot = x;
                }
            };
            if (lo == 0 && hi == kRows) {
#pragma unroll
                for (int r = kRows - 1; r >= 0; --r) step(r);
            } else {
                for (int r = hi - 1; r >= lo; --r) step(r);
            }
            __syncwarp();
            if constexpr (LAYOUT != PSW_LAYOUT_R) {
                store_s(tl, X, ldx, k0, N, q0, lo, hi, true);
                __syncwarp();
            }
            if (lane == 0 && i + K < nst) {
                const int bs2 = nst - 1 - (i + K);
                fence_proxy_async_smem();
                TM::issue(tile(sq), coef(sq), cbw + sa + bs2 * kRows, cb, bar(sq), tmX, k0,
                          sa + bs2 * kRows, pol);
            }
        }
        seq += nst;
    }
};

template <typename T, int LAYOUT>
__global__ void __launch_bounds__(kMaxWarps * 32) pipe_kernel(
    const __grid_constant__ CUtensorMap tmF, const __grid_constant__ CUtensorMap tmX, T* X,
    const PipeGeom g, const PipeBuf b, const int32_t* __restrict__ blk,
    const FwdCoef<T>* __restrict__ cf, const BwdCoef<T>* __restrict__ cbw,
    const CombineItem* __restrict__ items, const double* __restrict__ zr,
    const double* __restrict__ zl) {
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* base = reinterpret_cast<unsigned char*>(
                              (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023)) +
                          size_t(warp) * g.warp_bytes;
    PipeWarp<T, LAYOUT> w;
    w.K = g.K;
    w.lane = lane;
    w.seq = 0;
    w.tiles = base;
    w.coefs = base + g.K * TileMap<T, LAYOUT>::kBytes;
    w.bars = reinterpret_cast<uint64_t*>(base + g.warp_bytes - 8 * g.K);
    if (lane == 0) {
        for (int i = 0; i < g.K; ++i) mbar_init(&w.bars[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t pol_first = policy_evict_first();
    const int P = g.P, p = g.p, NG = g.NG;
    const int64_t RS = int64_t(NG) * (1 + 2 * P);
    const int64_t Nc = g.Nc;

    long long it = 0;
    if (lane == 0) it = static_cast<long long>(atomicAdd(b.head, 1ULL));
    it = __shfl_sync(0xffffffffu, it, 0);
    unsigned long long* const trace = g_pipe_trace;
    while (it < g.total) {
        long long nxt = 0;
        unsigned long long* tr = trace && lane == 0 ? trace + 4 * it : nullptr;
        if (tr) tr[0] = gtimer_ns();
        if (lane == 0) nxt = static_cast<long long>(atomicAdd(b.head, 1ULL));
        const int r = int(it / RS);
        const int pos = int(it % RS);
        if (pos < NG) {
            // ---- B(r-1, pos): combination
            const int c = r - 1, grp = pos;
            const int64_t k0 = int64_t(c) * Nc + int64_t(grp) * kLanes;
            if (c >= 0 && k0 < g.N) {
                const int q = c * NG + grp, slot = c & 1;
                wait_geq(b.doneA + q, P);
                if (c >= 2) wait_geq(b.doneC + (q - 2 * NG), P);  // V slot drained
                if (tr) tr[1] = gtimer_ns(), tr[3] = (1ull << 32) | smid();
                const int64_t kl = int64_t(grp) * kLanes + lane;
                const bool kv = k0 + lane < g.N;
                const double* bl = b.bet + (int64_t(slot) * 2 + 0) * P * Nc + kl;
                const double* br = b.bet + (int64_t(slot) * 2 + 1) * P * Nc + kl;
                double* V = b.V + int64_t(slot) * p * Nc + kl;
                if (p > 0 && g.stage_b) {
                    // betas and values of the group in this warp's (idle) stage
                    // buffers: all loads in flight at once, then the combination
                    // from shared memory (same arithmetic, so bitwise STAGED)
                    double* sl = reinterpret_cast<double*>(w.tiles);
                    double* sr = sl + P * kLanes;
                    double* sv = sr + P * kLanes;
                    if (kv) {
#pragma unroll 8
                        for (int t = 0; t < P; ++t) {
                            sl[t * kLanes + lane] = bl[int64_t(t) * Nc];
                            sr[t * kLanes + lane] = br[int64_t(t) * Nc];
                        }
                        combine_rhs(items, p, sl + lane, sr + lane, kLanes, zr, zl, sv + lane,
                                    kLanes);
                        for (int j = 0; j < p; ++j) V[int64_t(j) * Nc] = sv[j * kLanes + lane];
                    }
                    __syncwarp();
                } else if (p > 0 && kv) {
                    combine_rhs(items, p, bl, br, Nc, zr, zl, V, Nc);
                }
                publish(b.flagB + q, lane);
            }
        } else if (pos < NG * (1 + P)) {
            // ---- A(r, g, t): forward sweep
            const int idx = pos - NG, c = r, grp = idx / P, t = idx % P;
            const int64_t k0 = int64_t(c) * Nc + int64_t(grp) * kLanes;
            if (c < g.nchunks && k0 < g.N) {
                const int q = c * NG + grp, slot = c & 1;
                if (c >= 2) wait_geq(b.flagB + (q - 2 * NG), 1);  // beta slot drained
                if (tr) tr[1] = gtimer_ns(), tr[3] = (0ull << 32) | smid();
                double br, bl;
                w.fwd(&tmF, X, g.ldx, g.N, k0, blk[2 * t], blk[2 * t + 1], cf, pol_first, br, bl);
                if (k0 + lane < g.N) {
                    const int64_t kl = int64_t(grp) * kLanes + lane;
                    if (t > 0) b.bet[((int64_t(slot) * 2 + 0) * P + t) * Nc + kl] = bl;
                    if (t < p) b.bet[((int64_t(slot) * 2 + 1) * P + t) * Nc + kl] = br;
                }
                publish(b.doneA + q, lane);
            }
        } else {
            // ---- C(r-1, g, t): back substitution
            const int idx = pos - NG * (1 + P), c = r - 1, grp = idx / P, t = idx % P;
            const int64_t k0 = int64_t(c) * Nc + int64_t(grp) * kLanes;
            if (c >= 0 && k0 < g.N) {
                const int q = c * NG + grp, slot = c & 1;
                wait_geq(b.flagB + q, 1);
                if (tr) tr[1] = gtimer_ns(), tr[3] = (2ull << 32) | smid();
                if (lane == 0) fence_proxy_async_global();  // d (generic stores) -> TMA reads
                T xl = T(0), xr = T(0);
                if (k0 + lane < g.N) {
                    const double* V = b.V + int64_t(slot) * p * Nc + int64_t(grp) * kLanes + lane;
                    if (t > 0) xl = T(V[int64_t(t - 1) * Nc]);
                    if (t < p) xr = T(V[int64_t(t) * Nc]);
                }
                w.bwd(&tmX, X, g.ldx, g.N, k0, blk[2 * t], blk[2 * t + 1], cbw, xl, xr, pol_first);
                publish(b.doneC + q, lane);
            }
        }
        if (tr) tr[2] = gtimer_ns();
        it = __shfl_sync(0xffffffffu, nxt, 0);
    }
}

struct PipeConfig {
    int K = 0, warps = 0;
    bool stage_b = false;
    size_t area = 0;
    int64_t Nc = 0;
    size_t warp_bytes = 0, smem = 0;
};

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

template <typename T>
PipeConfig pipe_config(const psw_plan* pl, int64_t N) {
    PipeConfig c;
    c.K = std::max(2, std::min(8, env_int("PSW_PIPE_STAGES", 4)));
    const size_t tile = size_t(kRows) * kLanes * sizeof(T);
    // stage buffers (reused by the combination items for the group's betas
    // and boundary values when they fit: (3P - 1) x 32 doubles, P <= 64)
    size_t area = size_t(c.K) * (tile + kCoefBytes);
    const size_t bscratch = size_t(3 * pl->P - 1) * kLanes * sizeof(double);
    c.stage_b = pl->P <= 64;
    if (c.stage_b) area = std::max(area, bscratch);
    c.area = area;
    c.warp_bytes = (area + 8 * c.K + 1023) & ~size_t(1023);
    const size_t budget = 226 * 1024 - 1024;
    c.warps = int(std::min<size_t>(kMaxWarps, budget / c.warp_bytes));
    if (const int ew = env_int("PSW_PIPE_WARPS", 0)) c.warps = std::max(1, std::min(c.warps, ew));
    c.smem = c.warps * c.warp_bytes + 1024;
    // chunk: forward intermediates of Nc RHS (n * Nc * s bytes) resident in L2
    const double mb = std::max(1, env_int("PSW_PIPE_CHUNK_MB", 24));
    const int64_t per_rhs = pl->n * int64_t(sizeof(T));
    int64_t nc = int64_t(mb * 1048576.0 / double(per_rhs)) / kLanes * kLanes;
    nc = std::max<int64_t>(kLanes, nc);
    nc = std::min<int64_t>(nc, (N + kLanes - 1) / kLanes * kLanes);
    c.Nc = nc;
    return c;
}

bool encode_map(CUtensorMap* tm, const void* base, int64_t inner, int64_t outer, int64_t ld,
                int es, uint32_t box0, bool swizzle) {
    auto encode = tensor_map_encoder();
    if (!encode) {
        set_error(PSW_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        return false;
    }
    const cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
    const cuuint64_t strides[1] = {cuuint64_t(ld) * cuuint64_t(es)};
    const cuuint32_t box[2] = {box0, cuuint32_t(kRows)};
    const cuuint32_t estr[2] = {1, 1};
    const auto dt = es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const CUresult r =
        encode(tm, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE,
               swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error(PSW_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
        return false;
    }
    return true;
}

template <typename T, int LAYOUT>
int launch_pipe(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                cudaStream_t s, void** ev, int nev) {
    const int es = int(sizeof(T));
    const PipeConfig pc = pipe_config<T>(pl, N);
    CUtensorMap tmF, tmX;
    const bool sw = LAYOUT == PSW_LAYOUT_S;
    const uint32_t box0 = sw ? uint32_t(128 / es) : uint32_t(kRows);
    if (LAYOUT == PSW_LAYOUT_R) {
        if (!encode_map(&tmF, F, N, pl->n, ldf, es, box0, false) ||
            !encode_map(&tmX, X, N, pl->n, ldx, es, box0, false))
            return PSW_CUDA_ERROR;
    } else {
        if (!encode_map(&tmF, F, pl->n, N, ldf, es, box0, sw) ||
            !encode_map(&tmX, X, pl->n, N, ldx, es, box0, sw))
            return PSW_CUDA_ERROR;
    }
    PipeGeom g;
    g.P = int(pl->P);
    g.p = int(pl->p);
    g.NG = int(pc.Nc / kLanes);
    g.K = pc.K;
    g.nchunks = int((N + pc.Nc - 1) / pc.Nc);
    g.warp_bytes = int(pc.warp_bytes);
    g.stage_b = pc.stage_b ? 1 : 0;
    g.N = N;
    g.Nc = pc.Nc;
    g.ldx = ldx;
    g.total = int64_t(g.nchunks + 1) * g.NG * (1 + 2 * g.P);

    // scratch: ticket + counters (zeroed) | betas | boundary values
    const size_t ncnt = size_t(g.nchunks) * g.NG;
    const size_t cnt_bytes = (8 + 3 * ncnt * sizeof(int) + 255) & ~size_t(255);
    const size_t bet_bytes = sizeof(double) * 2 * 2 * size_t(g.P) * pc.Nc;
    const size_t v_bytes = sizeof(double) * 2 * size_t(std::max(g.p, 1)) * pc.Nc;
    void* scratch = nullptr;
    PSW_CUDA_TRY(cudaMallocAsync(&scratch, cnt_bytes + bet_bytes + v_bytes, s));
    char* cp = static_cast<char*>(scratch);
    PipeBuf b;
    b.head = reinterpret_cast<unsigned long long*>(cp);
    b.doneA = reinterpret_cast<int*>(cp + 8);
    b.flagB = b.doneA + ncnt;
    b.doneC = b.flagB + ncnt;
    b.bet = reinterpret_cast<double*>(cp + cnt_bytes);
    b.V = reinterpret_cast<double*>(cp + cnt_bytes + bet_bytes);
    int rc = PSW_OK;
    mark(ev, nev, 0, s);
    if (cudaMemsetAsync(scratch, 0, cnt_bytes, s) != cudaSuccess) {
        rc = cuda_fail(cudaGetLastError(), "cudaMemsetAsync");
    } else {
        auto kern = pipe_kernel<T, LAYOUT>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(pc.smem));
        int dev = 0, nsm = 0, occ = 0;
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, pc.warps * 32, pc.smem);
        if (e == cudaSuccess && occ < 1) e = cudaErrorInvalidConfiguration;
        if (e == cudaSuccess) {
            const int64_t grid = std::min<int64_t>(int64_t(nsm) * occ,
                                                   (g.total + pc.warps - 1) / pc.warps);
            kern<<<unsigned(grid), unsigned(pc.warps * 32), pc.smem, s>>>(
                tmF, tmX, static_cast<T*>(X), g, b, pl->d_blk,
                static_cast<const FwdCoef<T>*>(pl->d_fwd), static_cast<const BwdCoef<T>*>(pl->d_bwd),
                pl->d_items, pl->d_zr, pl->d_zl);
            e = cudaGetLastError();
            mark(ev, nev, 1, s);
        }
        if (e != cudaSuccess) rc = cuda_fail(e, "pipe_kernel launch");
        else note_launches(1);
    }
    cudaFreeAsync(scratch, s);
    return rc;
}

}  // namespace

int set_pipe_trace(void* buf) {
    unsigned long long* q = static_cast<unsigned long long*>(buf);
    PSW_CUDA_TRY(cudaMemcpyToSymbol(g_pipe_trace, &q, sizeof(q)));
    return PSW_OK;
}

bool pipe_supported(const psw_plan* pl, int layout, int64_t N, const void* F, int64_t ldf,
                    const void* X, int64_t ldx) {
    if (pl->world != 1 || N < 1 || N >= (int64_t{1} << 31) || pl->n >= (int64_t{1} << 31))
        return false;
    if (layout != PSW_LAYOUT_R && layout != PSW_LAYOUT_S) return false;
    const int es = pl->dtype == PSW_F64 ? 8 : 4;
    // TMA: 16-byte aligned bases and row pitches
    if ((reinterpret_cast<uintptr_t>(F) & 15) || (reinterpret_cast<uintptr_t>(X) & 15)) return false;
    if (((size_t(ldf) * es) & 15) || ((size_t(ldx) * es) & 15)) return false;
    return true;
}

int solve_pipe(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
               int layout, cudaStream_t s, void** ev, int nev) {
    if (pl->dtype == PSW_F64)
        return layout == PSW_LAYOUT_R
                   ? launch_pipe<double, PSW_LAYOUT_R>(pl, F, ldf, X, ldx, N, s, ev, nev)
                   : std::getenv("PSW_PIPE_PLAIN_S")
                         ? launch_pipe<double, kLayoutSPlain>(pl, F, ldf, X, ldx, N, s, ev, nev)
                         : launch_pipe<double, PSW_LAYOUT_S>(pl, F, ldf, X, ldx, N, s, ev, nev);
    return layout == PSW_LAYOUT_R
               ? launch_pipe<float, PSW_LAYOUT_R>(pl, F, ldf, X, ldx, N, s, ev, nev)
               : std::getenv("PSW_PIPE_PLAIN_S")
                         ? launch_pipe<float, kLayoutSPlain>(pl, F, ldf, X, ldx, N, s, ev, nev)
                         : launch_pipe<float, PSW_LAYOUT_S>(pl, F, ldf, X, ldx, N, s, ev, nev);
}

}  // namespace psw
