// TILE solve path: one CTA per RHS tile, two passes over the tile's rows, no
// cross-CTA exchange.
//
// A tile is W right-hand sides x all n rows (layout R: 128 contiguous bytes
// per row; layout S: W systems). Every block of the partition is cut into
// segments of <= 33 rows (psw_fused.cu build_fused_tables; the exact affine
// carries of psw_internal.h). One CTA owns a tile:
//   pass 1  every (segment, RHS) thread sweeps its rows forward from a zero
//           carry (local_solve.hpp:39-48 in affine form) and keeps only the
//           segment partials d~_end, Lam and the two beta dot products
//           (betas.hpp:42-57) in shared memory;
//   scans   per (block, RHS): forward carries D and block betas, the
//           boundary values through the tabulated dichotomy combination
//           (boundary_solve.hpp:96-121 as a linear map, psw_plan.cpp
//           combine_matrix), backward carries x at every segment end;
//   pass 2  every (segment, RHS) thread re-reads its rows (an L2 hit: the
//           tile was read moments ago and at most ~#SM tiles are live),
//           sweeps forward from the exact carry D and back from the exact
//           carry x_b, and streams X.
// HBM sees F once and X once; nothing waits on another CTA.
// The number of co-resident tiles is capped so their rows fit in L2.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <type_traits>

#include "psw_device.cuh"
#include "psw_internal.h"

namespace psw {
namespace {

constexpr int kSegMax = kSegLen + 1;
constexpr int kMaxThreads = 512;

struct TileGeom {
    int n, P, p, NS, W, NW;
    int part_smem;  // 1: segment partials in shared memory, 0: per-CTA global scratch
    int coef_off;   // per-worker coefficient staging (bytes into shared memory)
    int prefetch;   // L2 prefetch of the worker's next segment in pass 1
    int64_t N, ldf, ldx, ntiles;
};

struct TileTabs {
    const SegDesc* desc;
    const int32_t* segoff;
    const SegCoef* segc;
    const void* ff;  // FusedFwd<T>[n]
    const void* fb;  // FusedBwd<T>[n]
    const double* cmat;  // [p][2P]
    double* gpart;       // [gridDim.x][NS][W][4] when the partials do not fit in smem
};

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
template <typename T>
__device__ __forceinline__ T ld_hint(const T* p, uint64_t pol);
template <>
__device__ __forceinline__ double ld_hint<double>(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
template <>
__device__ __forceinline__ float ld_hint<float>(const float* p, uint64_t pol) {
    float v;
    asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ void prefetch_l2(const void* q) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
}

// a segment's rows of this thread's RHS into registers
// (FULL: the segment has >= kSegLen - 1 rows, only the last two are predicated)
template <typename T, int LAYOUT, bool FULL = false>
__device__ __forceinline__ void load_seg(const T* F, int64_t ldf, int64_t k, int a, int len,
                                         bool kv, uint64_t pol, T (&v)[kSegMax]) {
    const T* src = LAYOUT == PSW_LAYOUT_R ? F + int64_t(a) * ldf + k : F + k * ldf + a;
    const int64_t step = LAYOUT == PSW_LAYOUT_R ? ldf : 1;
#pragma unroll
    for (int r = 0; r < kSegMax; ++r)
        v[r] = (kv && ((FULL && r < kSegLen - 1) || r < len)) ? ld_hint(src + r * step, pol) : T(0);
}

// A segment's coefficient rows into the worker's shared staging area, the
// worker's W lanes copying 16-byte pieces (all in flight with the row loads);
// the sweeps then read conflict-free broadcasts.
template <typename C>
__device__ __forceinline__ const C* stage(const C* src, int len, int lane, int W, C* dst) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    const int pieces = len * int(sizeof(C) / 16);
    for (int i = lane; i < pieces; i += W) d[i] = __ldg(s + i);
    return dst;
}

template <typename T>
constexpr int coef_stage_bytes() {
    return kSegMax * int(sizeof(FusedFwd<T>) + sizeof(FusedBwd<T>));
}

template <typename T, int LAYOUT>
__global__ void __launch_bounds__(kMaxThreads) tile_kernel(const T* F, T* X, const TileGeom g,
                                                           const TileTabs tb) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int W = g.W, NW = g.NW, P = g.P, p = g.p, NS = g.NS;
    const int nthr = W * NW;
    const int tid = threadIdx.x;
    const int lane = tid % W, worker = tid / W;
    // shared memory: block betas [P][W][2], values [p][W], partials [NS][W][4]
    double* bb = reinterpret_cast<double*>(smem);
    double* vals = bb + size_t(P) * W * 2;
    double* part = g.part_smem ? vals + size_t(max(p, 1)) * W
                               : tb.gpart + size_t(blockIdx.x) * NS * W * 4;
    const auto* ffw = static_cast<const FusedFwd<T>*>(tb.ff);
    const auto* fbw = static_cast<const FusedBwd<T>*>(tb.fb);
    const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
    // the worker's lanes within its warp (W = 16: half warps)
    const unsigned wmask = W >= 32 ? 0xffffffffu : (((1u << W) - 1u) << (tid % 32 / W * W));
    FusedFwd<T>* const sff =
        reinterpret_cast<FusedFwd<T>*>(smem + g.coef_off + size_t(worker) * coef_stage_bytes<T>());
    FusedBwd<T>* const sfb = reinterpret_cast<FusedBwd<T>*>(sff + kSegMax);

    for (int64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
        const int64_t k = tile * W + lane;
        const bool kv = k < g.N;
        // ---- pass 1: segment partials (rows kept in L2 for pass 2)
        for (int s = worker; s < NS; s += NW) {
            const SegDesc sd = tb.desc[s];
            const int len = sd.b - sd.a;
            T d = T(0);
            double sR = 0.0, sL = 0.0, sX = 0.0;
            // one instruction stream for segments of >= 31 rows (both workers
            // of a warp), rows 0..30 unpredicated
            auto pass1 = [&](auto full) {
                constexpr bool FULL = decltype(full)::value;
                T v[kSegMax];
                load_seg<T, LAYOUT, FULL>(F, g.ldf, k, sd.a, len, kv, keep, v);
                if (g.prefetch && s + NW < NS) {
                    // the worker's next segment into L2 while this one is in flight
                    const SegDesc sn = tb.desc[s + NW];
                    if (LAYOUT == PSW_LAYOUT_R) {
                        if (lane == 0)
                            for (int r = 0; r < sn.b - sn.a; ++r)
                                prefetch_l2(F + int64_t(sn.a + r) * g.ldf + tile * W);
                    } else if (kv) {
                        for (int r = 0; r < sn.b - sn.a; r += 16) prefetch_l2(F + k * g.ldf + sn.a + r);
                    }
                }
                const FusedFwd<T>* cf = stage(ffw + sd.a, len, lane, W, sff);
                __syncwarp(wmask);
#pragma unroll
                for (int r = 0; r < kSegMax; ++r) {
                    if ((FULL && r < kSegLen - 1) || r < len) {
                        const FusedFwd<T> c = cf[r];
                        d = fma(c.ma, d, v[r] * c.rp);
                        sR = fma(double(v[r]), double(c.gr), sR);
                        sL = fma(double(v[r]), double(c.gl), sL);
                        sX = fma(double(c.lam), double(d), sX);
                    }
                }
            };
            if (len >= kSegLen - 1)
                pass1(std::true_type{});
            else
                pass1(std::false_type{});
            double* ps = part + (size_t(s) * W + lane) * 4;
            ps[0] = double(d);
            ps[1] = sX;
            ps[2] = sR;
            ps[3] = sL;
            __syncwarp(wmask);  // staging area reused by the next segment
        }
        __syncthreads();
        // ---- forward carries and block betas, per (block, RHS)
        for (int i = tid; i < P * W; i += nthr) {
            const int t = i / W, ln = i % W;
            const int s0 = tb.segoff[t], s1 = tb.segoff[t + 1];
            double D = 0.0, bR = 0.0, bL = 0.0;
            for (int s = s0; s < s1; ++s) {
                double* ps = part + (size_t(s) * W + ln) * 4;
                const double dend = ps[0];
                ps[0] = D;  // carry into the segment: D_{a-1}
                D = fma(tb.segc[s].mu_end, D, dend);
                bR += ps[2];
                bL += ps[3];
            }
            bb[(t * W + ln) * 2] = bR;
            bb[(t * W + ln) * 2 + 1] = bL;
        }
        __syncthreads();
        // ---- boundary values: V_j = MR_j . right + ML_j . left
        for (int i = tid; i < p * W; i += nthr) {
            const int j = i / W, ln = i % W;
            const double* M = tb.cmat + size_t(j) * 2 * P;
            double v = 0.0;
            for (int t = 0; t < P; ++t) {
                v = fma(M[t], bb[(t * W + ln) * 2], v);
                v = fma(M[P + t], bb[(t * W + ln) * 2 + 1], v);
            }
            vals[j * W + ln] = v;
        }
        __syncthreads();
        // ---- backward carries: x at the row after every segment
        for (int i = tid; i < P * W; i += nthr) {
            const int t = i / W, ln = i % W;
            const int s0 = tb.segoff[t], s1 = tb.segoff[t + 1];
            const double xl = t > 0 ? vals[(t - 1) * W + ln] : 0.0;
            double x = t < p ? vals[t * W + ln] : 0.0;
            for (int s = s1 - 1; s >= s0; --s) {
                double* ps = part + (size_t(s) * W + ln) * 4;
                const SegCoef sc = tb.segc[s];
                const double lam = ps[1];
                ps[1] = x;
                x = fma(sc.nu, x, fma(xl, sc.k2, fma(ps[0], sc.k1, lam)));
            }
        }
        __syncthreads();
        // ---- pass 2: exact sweeps from the carries, X streamed out
        for (int s = worker; s < NS; s += NW) {
            const SegDesc sd = tb.desc[s];
            const int len = sd.b - sd.a, t = sd.t;
            auto pass2 = [&](auto full) {
                constexpr bool FULL = decltype(full)::value;
                T v[kSegMax];
                load_seg<T, LAYOUT, FULL>(F, g.ldf, k, sd.a, len, kv, drop, v);
                const FusedFwd<T>* cf = stage(ffw + sd.a, len, lane, W, sff);
                const FusedBwd<T>* cb = stage(fbw + sd.a, len, lane, W, sfb);
                const double* ps = part + (size_t(s) * W + lane) * 4;
                const T D = T(ps[0]);
                T x = T(ps[1]);
                const T xl = t > 0 ? T(vals[(t - 1) * W + lane]) : T(0);
                __syncwarp(wmask);
                T d = D;
#pragma unroll
                for (int r = 0; r < kSegMax; ++r) {
                    if ((FULL && r < kSegLen - 1) || r < len) {
                        const FusedFwd<T> c = cf[r];
                        d = fma(c.ma, d, v[r] * c.rp);
                        v[r] = d;
                    }
                }
#pragma unroll
                for (int r = kSegMax - 1; r >= 0; --r) {
                    if ((FULL && r < kSegLen - 1) || r < len) {
                        const FusedBwd<T> c = cb[r];
                        x = fma(c.al, x, fma(xl, c.w, v[r]));
                        v[r] = x;
                    }
                }
                if (kv) {
                    T* dst = LAYOUT == PSW_LAYOUT_R ? X + int64_t(sd.a) * g.ldx + k : X + k * g.ldx + sd.a;
                    const int64_t step = LAYOUT == PSW_LAYOUT_R ? g.ldx : 1;
#pragma unroll
                    for (int r = 0; r < kSegMax; ++r)
                        if ((FULL && r < kSegLen - 1) || r < len) __stcs(dst + r * step, v[r]);
                }
            };
            if (len >= kSegLen - 1)
                pass2(std::true_type{});
            else
                pass2(std::false_type{});
            __syncwarp(wmask);
        }
        __syncthreads();
    }
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

template <typename T, int LAYOUT>
int launch_tile(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                cudaStream_t s, void** ev, int nev) {
    TileGeom g;
    g.n = int(pl->n);
    g.P = int(pl->P);
    g.p = int(pl->p);
    g.NS = int(pl->seg_off.back());
    // layout R: 128 contiguous bytes of a row per tile; layout S: 32 systems
    g.W = LAYOUT == PSW_LAYOUT_R ? 128 / int(sizeof(T)) : 32;
    const int threads = std::max(g.W, std::min(kMaxThreads, env_int("PSW_TILE_THREADS", 512)) /
                                          g.W * g.W);
    g.NW = threads / g.W;
    g.N = N;
    g.ldf = ldf;
    g.ldx = ldx;
    g.ntiles = (N + g.W - 1) / g.W;
    g.prefetch = env_int("PSW_TILE_PREFETCH", 0);  // measured neutral on C1
    const size_t fixed = (size_t(g.P) * g.W * 2 + size_t(std::max(g.p, 1)) * g.W) * sizeof(double);
    const size_t partb = size_t(g.NS) * g.W * 4 * sizeof(double);
    constexpr size_t kSmemCap = 227 * 1024;
    // fewer workers when the per-worker coefficient staging does not fit
    while (g.NW > 1 && fixed + size_t(g.NW) * coef_stage_bytes<T>() > kSmemCap) g.NW /= 2;
    const size_t coefb = size_t(g.NW) * coef_stage_bytes<T>();
    if (fixed + coefb > kSmemCap) {
        set_error(PSW_NOT_SUPPORTED, "tile path: too many blocks for shared memory");
        return PSW_NOT_SUPPORTED;
    }
    g.part_smem = fixed + partb + coefb <=
                          std::min(kSmemCap, size_t(env_int("PSW_TILE_SMEM_KB", 200)) * 1024)
                      ? 1
                      : 0;
    g.coef_off = int((fixed + (g.part_smem ? partb : 0) + 15) & ~size_t(15));
    const size_t smem = size_t(g.coef_off) + coefb;

    const int nthreads = g.NW * g.W;
    auto kern = tile_kernel<T, LAYOUT>;
    PSW_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int dev = 0, nsm = 0, occ = 0;
    PSW_CUDA_TRY(cudaGetDevice(&dev));
    PSW_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    PSW_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nthreads, smem));
    if (occ < 1) {
        set_error(PSW_NOT_SUPPORTED, "tile path: kernel does not fit on an SM");
        return PSW_NOT_SUPPORTED;
    }
    // co-resident tiles: their rows must stay in L2 between the two passes
    const double tile_bytes = double(g.n) * g.W * sizeof(T);
    const double l2 = double(env_int("PSW_TILE_L2_MB", 64)) * 1048576.0;
    int64_t grid = std::min<int64_t>(int64_t(nsm) * occ, g.ntiles);
    grid = std::max<int64_t>(1, std::min<int64_t>(grid, int64_t(l2 / tile_bytes)));
    if (const int ec = env_int("PSW_TILE_CTAS", 0)) grid = std::max(1, std::min<int>(int(grid), ec));
    TileTabs tb;
    tb.desc = pl->d_segdesc;
    tb.segoff = pl->d_segoff;
    tb.segc = pl->d_seg;
    tb.ff = pl->d_ffwd;
    tb.fb = pl->d_fbwd;
    tb.cmat = pl->d_cmat;
    tb.gpart = nullptr;
    void* scratch = nullptr;
    if (!g.part_smem) {
        PSW_CUDA_TRY(cudaMallocAsync(&scratch, size_t(grid) * partb, s));
        tb.gpart = static_cast<double*>(scratch);
    }
    if (std::getenv("PSW_TILE_VERBOSE"))
        std::fprintf(stderr, "tile: W=%d NW=%d NS=%d smem=%zu part_smem=%d occ=%d grid=%lld tiles=%lld\n",
                     g.W, g.NW, g.NS, smem, g.part_smem, occ, (long long)grid, (long long)g.ntiles);
    mark(ev, nev, 0, s);
    kern<<<unsigned(grid), unsigned(nthreads), smem, s>>>(static_cast<const T*>(F),
                                                         static_cast<T*>(X), g, tb);
    const cudaError_t e = cudaGetLastError();
    mark(ev, nev, 1, s);
    if (scratch) cudaFreeAsync(scratch, s);
    if (e != cudaSuccess) return cuda_fail(e, "tile_kernel launch");
    note_launches(1);
    return PSW_OK;
}

}  // namespace

bool tile_supported(const psw_plan* pl, int layout, int64_t N) {
    if (pl->world != 1 || N < 1 || N >= (int64_t{1} << 31) || pl->n >= (int64_t{1} << 31))
        return false;
    if (!pl->d_segdesc || pl->seg_off.empty() || (pl->p > 0 && !pl->d_cmat) || pl->P > 256)
        return false;
    return layout == PSW_LAYOUT_R || layout == PSW_LAYOUT_S;
}

int solve_tile(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
               int layout, cudaStream_t s, void** ev, int nev) {
    if (pl->dtype == PSW_F64)
        return layout == PSW_LAYOUT_R
                   ? launch_tile<double, PSW_LAYOUT_R>(pl, F, ldf, X, ldx, N, s, ev, nev)
                   : launch_tile<double, PSW_LAYOUT_S>(pl, F, ldf, X, ldx, N, s, ev, nev);
    return layout == PSW_LAYOUT_R
               ? launch_tile<float, PSW_LAYOUT_R>(pl, F, ldf, X, ldx, N, s, ev, nev)
               : launch_tile<float, PSW_LAYOUT_S>(pl, F, ldf, X, ldx, N, s, ev, nev);
}

}  // namespace psw
