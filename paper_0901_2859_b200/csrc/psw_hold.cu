// HOLD solve path: F is read once and X written once (2 s bytes per unknown)
// for systems too long for a cluster (CLUSTER / FUSED: a 128-byte RHS tile of
// every row must fit 16 CTAs) but short enough that one RHS tile of all n
// rows fits the shared memory of the WHOLE grid: the fp32 config C2
// (n = 65536: a 32-RHS tile is 8 MB, 57 KB on each of 147 SMs, three tiles in
// flight). RESWEEP reads F twice there (3 s).
//
// One persistent cooperative launch, one CTA per SM. CTA c keeps the same
// contiguous rows (<= kHdSeg segments of the plan's segment table) of every
// tile; tile i = RHS columns [32 i, 32 i + 32). The per-row coefficients of
// the CTA's rows are loaded into shared memory once. Warp roles:
//   sweep warps (one per segment, lane = RHS)
//       A(i): forward sweep from a zero carry out of the TMA-filled slab,
//             d~ written in place, Lam~ and the two beta partials per segment
//             (betas.hpp:42-57 split by segment);
//       C(i): back substitution from the segment's exact carries, x in place,
//             the segment's rows stored with cp.async.bulk.tensor; the slab
//             stage goes back to the producer once the store has read it.
//       Order C(i - S + 1), A(i): S tiles are in flight per CTA.
//   producer   TMA loads of the CTA's rows of tile i into stage i % S.
//   fold       the CTA's segments folded into run aggregates (run = the part
//              of the CTA inside one block; the affine composition of
//              psw_resweep.cu), published to the exchange scratch.
//   owner      for the blocks this CTA owns: forward fold over the block's
//              runs (exact carry into every run, block betas), published.
//   V warps    for the boundary values this CTA owns: row j of the
//              combination matrix (psw_plan.cpp combine_matrix = the
//              dichotomy of boundary_solve.hpp:96-121 as a linear map) times
//              all block betas, published.
//   carry      per own run: backward fold over the block's later runs from
//              V_t, then the exact carries of the run's segments -> sweep
//              warps (shared memory + mbarrier).
// The exchange goes through L2 in flag-in-data words ({lo32, flag, hi32,
// flag}, one 16-byte store per double; the reader polls the word itself, flag
// = tile index + 1), so a hop costs one store-to-poll latency (0.84 us
// measured, tools/hopbench.cu) and no fences. The scratch has 2 S slots per
// quantity: a word of tile i is rewritten for tile i + 2 S only after every
// reader of tile i has passed (sweep order C(i - S + 1), A(i) and in-order
// exchange warps). All CTAs must be co-resident
// (cooperative launch); a poll that does not complete within ~2 s traps.
//
// Summation orders are fixed (no atomics): results are run-to-run bitwise
// reproducible. Supported: fp32 plans, layout R, whole-system plans with a
// combination matrix and P <= kHoldMaxP, TMA-addressable F and X.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "psw_internal.h"
#include "psw_tma.cuh"

namespace psw {
namespace {

constexpr int kHdSeg = 14;   // sweep warps = segments per CTA at most
constexpr int kHdVW = 4;     // V warps
constexpr int kWProd = kHdSeg, kWFold = kHdSeg + 1, kWOwn = kHdSeg + 2, kWCarry = kHdSeg + 3,
              kWV0 = kHdSeg + 4;
constexpr int kHdWarps = kHdSeg + 4 + kHdVW;
constexpr int kHdThreads = kHdWarps * 32;
constexpr int kHdMaxStages = 4;
constexpr int kHdW = 32;     // RHS per tile (lane = RHS)
constexpr int kHoldMaxP = 64;
constexpr int kSegMax = kSegLen + 1;

template <typename T>
struct alignas(16) HoldCoef {
    T rp, ma, gr, gl, lam, mu, w, al;
};

struct HoldMeta {
    RsGroup g;
    SegDesc desc[kHdSeg];
    SegCoef seg[kHdSeg];
    RsRun run[kHdSeg];
    SegCoef rc[kHdSeg];
};

struct HoldArgs {
    int64_t N;
    int ntiles, stages, depth;
    int P, p, ncta, nruns, maxrows, hs;
    uint32_t slab_bytes;  // one stage
    uint32_t slotw;       // uint4 words per exchange slot
    const RsGroup* cta;
    const RsRun* runs;
    const SegCoef* rcoef;
    const int32_t* runoff;
    const SegDesc* desc;
    const SegCoef* segc;
    const void* coef;
    const double* cmat;
    uint4* xch;
};

// ---- flag-in-data exchange words
__device__ __forceinline__ void ll_store(uint4* p, double v, uint32_t flag) {
    const uint64_t b = uint64_t(__double_as_longlong(v));
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(uint32_t(b)),
                 "r"(flag), "r"(uint32_t(b >> 32)), "r"(flag)
                 : "memory");
}
__device__ __forceinline__ uint4 ll_ld(const uint4* p) {
    uint4 w;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                 : "l"(p)
                 : "memory");
    return w;
}
__device__ __forceinline__ double ll_val(const uint4& w) {
    return __longlong_as_double((long long)((uint64_t(w.z) << 32) | w.x));
}
__device__ __noinline__ void ll_spin(const uint4* p, uint32_t flag, uint4& w) {
    const long long t0 = clock64();
    int n = 0;
    do {
        w = ll_ld(p);
        if ((++n & 1023) == 0 && clock64() - t0 > 4000000000LL) __trap();  // ~2 s: a lost word
    } while (w.y != flag || w.w != flag);
}
// K words requested together (one L2 latency when they are all there)
template <int K>
__device__ __forceinline__ void ll_wait(const uint4* const (&p)[K], const bool (&on)[K],
                                        uint32_t flag, double (&v)[K]) {
    uint4 w[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (on[k]) w[k] = ll_ld(p[k]);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        v[k] = 0.0;
        if (on[k]) {
            if (w[k].y != flag || w[k].w != flag) ll_spin(p[k], flag, w[k]);
            v[k] = ll_val(w[k]);
        }
    }
}
__device__ __forceinline__ double ll_wait1(const uint4* p, uint32_t flag) {
    uint4 w = ll_ld(p);
    if (w.y != flag || w.w != flag) ll_spin(p, flag, w);
    return ll_val(w);
}

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void st_tma_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_group() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
template <bool FULL>
__device__ __forceinline__ bool hd_row_on(int r, int len) {
    return (FULL && r < kSegLen - 1) || r < len;
}

// exchange scratch addressing (uint4 words; lane added by the caller)
struct Xch {
    uint4* base;
    int nruns, P;
    __device__ __forceinline__ uint4* run(int r, int q) const { return base + (size_t(r) * 4 + q) * 32; }
    __device__ __forceinline__ uint4* din(int r) const { return base + (size_t(nruns) * 4 + r) * 32; }
    __device__ __forceinline__ uint4* beta(int u) const { return base + (size_t(nruns) * 5 + u) * 32; }
    __device__ __forceinline__ uint4* v(int j) const {
        return base + (size_t(nruns) * 5 + 2 * size_t(P) + j) * 32;
    }
};

template <typename T>
__global__ void __launch_bounds__(kHdThreads, 1) hold_kernel(
    const __grid_constant__ CUtensorMap f32m, const __grid_constant__ CUtensorMap f1m,
    const __grid_constant__ CUtensorMap x32m, const __grid_constant__ CUtensorMap x1m,
    const HoldArgs A) {
    extern __shared__ __align__(1024) unsigned char dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x, S = A.stages;
    unsigned char* slab0 = dyn;
    HoldCoef<T>* coef = reinterpret_cast<HoldCoef<T>*>(dyn + size_t(S) * A.slab_bytes);
    HoldMeta* mt = reinterpret_cast<HoldMeta*>(coef + A.maxrows);
    T* lamt = reinterpret_cast<T*>(mt + 1);                 // [S][kHdSeg][32]
    T* rl = lamt + size_t(S) * kHdSeg * 32;                 // [S][kHdSeg][2][32]
    T* car = rl + size_t(S) * kHdSeg * 2 * 32;              // [S][kHdSeg][3][32]
    double* dsc = reinterpret_cast<double*>(car + size_t(S) * kHdSeg * 3 * 32);  // [kHdSeg][32]
    double* vred = dsc + kHdSeg * 32;                       // [2][kHdVW][32]
    uint64_t* full = reinterpret_cast<uint64_t*>(vred + 2 * kHdVW * 32);
    uint64_t* empty = full + kHdMaxStages;
    uint64_t* agg = empty + kHdMaxStages;
    uint64_t* carr = agg + kHdMaxStages;
    uint64_t* cbar = carr + kHdMaxStages;

    const RsGroup g = A.cta[b];
    const int ns = g.s1 - g.s0, nr = g.r1 - g.r0, rows = g.rb - g.ra;
    if (threadIdx.x < ns) {
        mt->desc[threadIdx.x] = A.desc[g.s0 + threadIdx.x];
        mt->seg[threadIdx.x] = A.segc[g.s0 + threadIdx.x];
    }
    if (threadIdx.x < nr) {
        mt->run[threadIdx.x] = A.runs[g.r0 + threadIdx.x];
        mt->rc[threadIdx.x] = A.rcoef[g.r0 + threadIdx.x];
    }
    if (threadIdx.x == 0) {
        mt->g = g;
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], ns);
            mbar_init(&agg[s], ns);
            mbar_init(&carr[s], 1);
        }
        mbar_init(cbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int ntiles = A.ntiles;

    // ------------------------------------------------------------ sweep warps
    if (warp < kHdSeg) {
        if (warp >= ns) return;
        const SegDesc sd = mt->desc[warp];
        const int a = sd.a - g.ra, len = sd.b - sd.a;
        const bool full_len = len >= kSegLen - 1;
        const HoldCoef<T>* c = coef + a;
        mbar_wait(cbar, 0);
        int pend = -1;
        for (int i = 0; i < ntiles + S - 1; ++i) {
            if (i >= S - 1) {  // C(k): back substitution of tile k
                const int k = i - (S - 1), st = k % S;
                mbar_wait(&carr[st], uint32_t((k / S) & 1));
                T* f = reinterpret_cast<T*>(slab0 + size_t(st) * A.slab_bytes) + a * kHdW + lane;
                const T* cv = car + (size_t(st) * kHdSeg + warp) * 3 * 32;
                const T D = cv[lane], xl = cv[64 + lane];
                T x = cv[32 + lane];
                auto bwd = [&](auto full_) {
                    constexpr bool FULL = decltype(full_)::value;
#pragma unroll
                    for (int r = kSegMax - 1; r >= 0; --r) {
                        if (hd_row_on<FULL>(r, len)) {
                            const HoldCoef<T> q = c[r];
                            const T dq = fma(q.mu, D, f[r * kHdW]);
                            x = fma(q.al, x, fma(xl, q.w, dq));
                            f[r * kHdW] = x;
                        }
                    }
                };
                if (full_len)
                    bwd(std::true_type{});
                else
                    bwd(std::false_type{});
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const int col = k * kHdW, n32 = len >> 5;
                    const T* src = f - lane;
                    for (int j = 0; j < n32; ++j) st_tma_2d(&x32m, col, sd.a + 32 * j, src + size_t(j) * 32 * kHdW);
                    for (int r = n32 * 32; r < len; ++r) st_tma_2d(&x1m, col, sd.a + r, src + size_t(r) * kHdW);
                    bulk_commit_group();
                }
                pend = st;
            }
            if (i < ntiles) {  // A(i): forward sweep of tile i
                const int st = i % S;
                mbar_wait(&full[st], uint32_t((i / S) & 1));
                T* f = reinterpret_cast<T*>(slab0 + size_t(st) * A.slab_bytes) + a * kHdW + lane;
                T d = T(0), lx = T(0), br = T(0), bl = T(0);
                auto fwd = [&](auto full_) {
                    constexpr bool FULL = decltype(full_)::value;
#pragma unroll
                    for (int r = 0; r < kSegMax; ++r) {
                        if (hd_row_on<FULL>(r, len)) {
                            const HoldCoef<T> q = c[r];
                            const T fv = f[r * kHdW];
                            d = fma(q.ma, d, fv * q.rp);
                            br = fma(fv, q.gr, br);
                            bl = fma(fv, q.gl, bl);
                            lx = fma(q.lam, d, lx);
                            f[r * kHdW] = d;
                        }
                    }
                };
                if (full_len)
                    fwd(std::true_type{});
                else
                    fwd(std::false_type{});
                lamt[(size_t(st) * kHdSeg + warp) * 32 + lane] = lx;
                T* rp = rl + (size_t(st) * kHdSeg + warp) * 64;
                rp[lane] = br;
                rp[32 + lane] = bl;
                __syncwarp();
                if (lane == 0) mbar_arrive_cta(&agg[st]);
            }
            if (pend >= 0 && lane == 0) {  // the store of C(k) has read its stage
                bulk_wait_read0();
                mbar_arrive_cta(&empty[pend]);
            }
            pend = -1;
        }
        if (lane == 0) bulk_wait0();
        return;
    }

    // ------------------------------------------------------------ producer
    if (warp == kWProd) {
        if (lane != 0) return;
        mbar_expect_tx(cbar, uint32_t(rows) * uint32_t(sizeof(HoldCoef<T>)));
        bulk_load(coef, static_cast<const HoldCoef<T>*>(A.coef) + g.ra,
                  uint32_t(rows) * uint32_t(sizeof(HoldCoef<T>)), cbar);
        const int n32 = rows >> 5;
        for (int i = 0; i < ntiles; ++i) {
            const int st = i % S;
            if (i >= S) mbar_wait(&empty[st], uint32_t((i / S - 1) & 1));
            unsigned char* stage = slab0 + size_t(st) * A.slab_bytes;
            mbar_expect_tx(&full[st], uint32_t(rows) * kHdW * uint32_t(sizeof(T)));
            const int col = i * kHdW;
            for (int j = 0; j < n32; ++j)
                tma_load_2d(stage + size_t(j) * 32 * kHdW * sizeof(T), &f32m, col, g.ra + 32 * j, &full[st]);
            for (int r = n32 * 32; r < rows; ++r)
                tma_load_2d(stage + size_t(r) * kHdW * sizeof(T), &f1m, col, g.ra + r, &full[st]);
        }
        return;
    }

    Xch X{nullptr, A.nruns, A.P};
    // ------------------------------------------------------------ fold: segments -> runs
    if (warp == kWFold) {
        for (int i = 0; i < ntiles; ++i) {
            const int st = i % S;
            mbar_wait(&agg[st], uint32_t((i / S) & 1));
            const T* slab = reinterpret_cast<const T*>(slab0 + size_t(st) * A.slab_bytes);
            X.base = A.xch + size_t(i % A.depth) * A.slotw;
            const uint32_t flag = uint32_t(i + 1);
            for (int j = 0; j < nr; ++j) {
                const RsRun rr = mt->run[j];
                double D = 0.0, lam = 0.0, nupre = 1.0, R = 0.0, L = 0.0;
                for (int s = rr.s0; s < rr.s1; ++s) {
                    const int ls = s - g.s0;
                    const SegCoef q = mt->seg[ls];
                    const double dd = double(slab[(mt->desc[ls].b - 1 - g.ra) * kHdW + lane]);
                    const double lm = double(lamt[(size_t(st) * kHdSeg + ls) * 32 + lane]);
                    const T* rp = rl + (size_t(st) * kHdSeg + ls) * 64;
                    lam = fma(nupre, fma(D, q.k1, lm), lam);
                    D = fma(q.mu_end, D, dd);
                    nupre *= q.nu;
                    R += double(rp[lane]);
                    L += double(rp[32 + lane]);
                }
                const int r = g.r0 + j;
                ll_store(X.run(r, 0) + lane, D, flag);
                ll_store(X.run(r, 1) + lane, lam, flag);
                ll_store(X.run(r, 2) + lane, R, flag);
                ll_store(X.run(r, 3) + lane, L, flag);
            }
        }
        return;
    }

    // ------------------------------------------------------------ owner: runs -> block betas, run carries
    if (warp == kWOwn) {
        const int tlo = (b * A.P + A.ncta - 1) / A.ncta, thi = ((b + 1) * A.P + A.ncta - 1) / A.ncta;
        if (tlo >= thi) return;
        for (int i = 0; i < ntiles; ++i) {
            X.base = A.xch + size_t(i % A.depth) * A.slotw;
            const uint32_t flag = uint32_t(i + 1);
            for (int t = tlo; t < thi; ++t) {
                const int r0 = A.runoff[t], r1 = A.runoff[t + 1];
                double D = 0.0, R = 0.0, L = 0.0;
                for (int lo = r0; lo < r1; lo += 4) {
                    const uint4* ptr[12];
                    bool on[12];
                    double v[12];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int r = min(lo + u, r1 - 1);
                        ptr[3 * u] = X.run(r, 0) + lane;
                        ptr[3 * u + 1] = X.run(r, 2) + lane;
                        ptr[3 * u + 2] = X.run(r, 3) + lane;
                        on[3 * u] = on[3 * u + 1] = on[3 * u + 2] = lo + u < r1;
                    }
                    ll_wait<12>(ptr, on, flag, v);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (lo + u < r1) {
                            ll_store(X.din(lo + u) + lane, D, flag);
                            R += v[3 * u + 1];
                            L += v[3 * u + 2];
                            D = fma(A.rcoef[lo + u].mu_end, D, v[3 * u]);
                        }
                }
                ll_store(X.beta(t) + lane, t < A.p ? R : 0.0, flag);       // betas.hpp:46-49
                ll_store(X.beta(A.P + t) + lane, t > 0 ? L : 0.0, flag);   // betas.hpp:51-55
            }
        }
        return;
    }

    // ------------------------------------------------------------ V warps: betas -> boundary values
    if (warp >= kWV0) {
        const int q = warp - kWV0;
        const int parts = A.p * A.hs;
        const int elo = (b * parts + A.ncta - 1) / A.ncta, ehi = ((b + 1) * parts + A.ncta - 1) / A.ncta;
        if (elo >= ehi) return;
        const int hs = A.hs, width = 32 / hs, sub = lane / width, nU = 2 * A.P;
        const int niter = (nU + hs - 1) / hs;
        int par = 0;
        for (int i = 0; i < ntiles; ++i) {
            X.base = A.xch + size_t(i % A.depth) * A.slotw;
            const uint32_t flag = uint32_t(i + 1);
            for (int e = elo; e < ehi; ++e) {
                const int j = e / hs, h = e - j * hs;
                const int rhs = h * width + (lane - sub * width);
                const double* m = A.cmat + size_t(j) * nU;
                double acc = 0.0;
                for (int i0 = q; i0 < niter; i0 += kHdVW * 8) {
                    const uint4* ptr[8];
                    bool on[8];
                    double v[8];
                    double mc[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int u = (i0 + k * kHdVW) * hs + sub;
                        on[k] = u < nU;
                        ptr[k] = X.beta(on[k] ? u : 0) + rhs;
                        mc[k] = on[k] ? m[u] : 0.0;
                    }
                    ll_wait<8>(ptr, on, flag, v);
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc = fma(mc[k], v[k], acc);
                }
                if (hs == 2) acc += __shfl_xor_sync(0xffffffffu, acc, 16);
                double* vr = vred + size_t(par) * kHdVW * 32;
                vr[q * 32 + lane] = acc;
                asm volatile("bar.sync 2, %0;" ::"n"(kHdVW * 32) : "memory");
                if (q == 0 && lane < width) {
                    const double vj = (vr[lane] + vr[32 + lane]) + (vr[64 + lane] + vr[96 + lane]);
                    ll_store(X.v(j) + h * width + lane, vj, flag);
                }
                par ^= 1;
            }
        }
        return;
    }

    // ------------------------------------------------------------ carry: exact carries of the own segments
    if (warp == kWCarry) {
        for (int i = 0; i < ntiles; ++i) {
            const int st = i % S;
            mbar_wait(&agg[st], uint32_t((i / S) & 1));
            const T* slab = reinterpret_cast<const T*>(slab0 + size_t(st) * A.slab_bytes);
            X.base = A.xch + size_t(i % A.depth) * A.slotw;
            const uint32_t flag = uint32_t(i + 1);
            for (int j = 0; j < nr; ++j) {
                const RsRun rr = mt->run[j];
                const int t = rr.t, r = g.r0 + j, rend = A.runoff[t + 1];
                double xl, xb, D;
                {
                    const uint4* ptr[3] = {X.v(t > 0 ? t - 1 : 0) + lane, X.v(t < A.p ? t : 0) + lane,
                                           X.din(r) + lane};
                    const bool on[3] = {t > 0, t < A.p, true};
                    double v[3];
                    ll_wait<3>(ptr, on, flag, v);
                    xl = v[0];
                    xb = v[1];
                    D = v[2];
                }
                // backward over the block's later runs: x at the row after this run
                for (int hi = rend; hi > r + 1; hi -= 4) {
                    const uint4* ptr[8];
                    bool on[8];
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int q = hi - 1 - u;
                        on[2 * u] = on[2 * u + 1] = q > r;
                        ptr[2 * u] = X.run(q > r ? q : r, 1) + lane;
                        ptr[2 * u + 1] = X.din(q > r ? q : r) + lane;
                    }
                    ll_wait<8>(ptr, on, flag, v);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int q = hi - 1 - u;
                        if (q > r) {
                            const SegCoef c = A.rcoef[q];
                            xb = fma(c.nu, xb, fma(xl, c.k2, fma(v[2 * u + 1], c.k1, v[2 * u])));
                        }
                    }
                }
                // the run's own segments (serial affine fold, psw_internal.h)
                for (int s = rr.s0; s < rr.s1; ++s) {
                    const int ls = s - g.s0;
                    dsc[ls * 32 + lane] = D;
                    car[((size_t(st) * kHdSeg + ls) * 3 + 0) * 32 + lane] = T(D);
                    const double dd = double(slab[(mt->desc[ls].b - 1 - g.ra) * kHdW + lane]);
                    D = fma(mt->seg[ls].mu_end, D, dd);
                }
                double x = xb;
                for (int s = rr.s1 - 1; s >= rr.s0; --s) {
                    const int ls = s - g.s0;
                    const SegCoef c = mt->seg[ls];
                    car[((size_t(st) * kHdSeg + ls) * 3 + 1) * 32 + lane] = T(x);
                    car[((size_t(st) * kHdSeg + ls) * 3 + 2) * 32 + lane] = T(xl);
                    const double lm = double(lamt[(size_t(st) * kHdSeg + ls) * 32 + lane]);
                    x = fma(c.nu, x, fma(xl, c.k2, fma(dsc[ls * 32 + lane], c.k1, lm)));
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_cta(&carr[st]);
        }
        return;
    }
}

// ------------------------------------------------------------------ host
size_t hold_fixed_smem(int maxrows, int stages, size_t es) {
    return size_t(maxrows) * 8 * es + sizeof(HoldMeta) + size_t(stages) * kHdSeg * 32 * es * 6 +
           sizeof(double) * (kHdSeg * 32 + 2 * kHdVW * 32) + 8 * (4 * kHdMaxStages + 1) + 64;
}

template <typename T>
bool hold_encode(const void* base, int64_t ld, int64_t N, int64_t rows, CUtensorMap* m32,
                 CUtensorMap* m1) {
    const auto enc = tensor_map_encoder();
    constexpr int es = int(sizeof(T));
    if (!enc || (reinterpret_cast<uintptr_t>(base) & 15) || (ld * es) % 16 || N < kHdW || rows < 1 ||
        ld < N)
        return false;
    cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(ld) * es};
    cuuint32_t box32[2] = {cuuint32_t(kHdW), 32}, box1[2] = {cuuint32_t(kHdW), 1}, one[2] = {1, 1};
    const CUtensorMapDataType dt =
        es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    for (int k = 0; k < 2; ++k)
        if (enc(k ? m1 : m32, dt, 2, const_cast<void*>(base), dims, strides, k ? box1 : box32, one,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    return true;
}

int hold_env(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// stages that fit one SM (0: the path does not apply)
int hold_stages(const psw_plan* pl, size_t& smem, size_t& slab_bytes) {
    int maxs = 0;
    cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, pl->device);
    const size_t es = 4;
    slab_bytes = (size_t(pl->hd_maxrows) * kHdW * es + 127) / 128 * 128;
    int S = std::min(hold_env("PSW_HOLD_STAGES", 3), kHdMaxStages);
    for (; S >= 1; --S) {
        smem = size_t(S) * slab_bytes + hold_fixed_smem(pl->hd_maxrows, S, es);
        if (smem <= size_t(maxs)) return S;
    }
    return 0;
}

}  // namespace

int build_hold_tables(psw_plan* pl, const std::vector<SegDesc>& desc, const std::vector<SegCoef>& seg,
                      const std::vector<FusedFwd<double>>& ff,
                      const std::vector<FusedBwd<double>>& fb) {
    pl->hd_ncta = 0;
    if (pl->dtype != PSW_F32 || pl->world != 1 || !pl->d_cmat || pl->P > kHoldMaxP) return PSW_OK;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pl->device);
    const int nseg = int(desc.size());
    if (nsm < 1 || nseg < 1) return PSW_OK;
    const int NS = (nseg + nsm - 1) / nsm;
    if (NS > kHdSeg) return PSW_OK;
    std::vector<RsGroup> ctas;
    std::vector<RsRun> runs;
    std::vector<SegCoef> rcoef;
    std::vector<int32_t> runoff(size_t(pl->P) + 1, 0);
    int maxrows = 0;
    for (int g0 = 0; g0 < nseg; g0 += NS) {
        const int g1 = std::min(nseg, g0 + NS);
        RsGroup g{g0, g1, int32_t(runs.size()), 0, desc[size_t(g0)].a, desc[size_t(g1 - 1)].b,
                  desc[size_t(g0)].t, 0};
        for (int s = g0; s < g1;) {
            const int t = desc[size_t(s)].t;
            int e = s;
            while (e < g1 && desc[size_t(e)].t == t) ++e;
            // the segments' affine maps composed (as build_rs_tables)
            double mu = 1.0, k1 = 0.0, k2 = 0.0, nu = 1.0;
            for (int q = s; q < e; ++q) {
                const SegCoef& c = seg[size_t(q)];
                k1 += nu * mu * c.k1;
                k2 += nu * c.k2;
                mu *= c.mu_end;
                nu *= c.nu;
            }
            runs.push_back({s, e, t, t});
            rcoef.push_back({mu, k1, k2, nu});
            s = e;
        }
        g.r1 = int32_t(runs.size());
        maxrows = std::max(maxrows, int(g.rb - g.ra));
        ctas.push_back(g);
    }
    for (size_t r = 0; r < runs.size(); ++r) runoff[size_t(runs[r].t) + 1] = int32_t(r + 1);
    for (size_t i = 1; i < runoff.size(); ++i) runoff[i] = std::max(runoff[i], runoff[i - 1]);
    const int64_t n = pl->n;
    std::vector<HoldCoef<float>> co(static_cast<size_t>(n));
    for (int64_t q = 0; q < n; ++q) {
        const FusedFwd<double>& a = ff[size_t(q)];
        const FusedBwd<double>& c = fb[size_t(q)];
        co[size_t(q)] = {float(a.rp), float(a.ma), float(a.gr), float(a.gl),
                         float(a.lam), float(c.mu), float(c.w), float(c.al)};
    }
    auto up = [&](void** dst, const void* src, size_t bytes) -> int {
        PSW_CUDA_TRY(cudaMalloc(dst, std::max<size_t>(bytes, 16)));
        if (bytes) PSW_CUDA_TRY(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
        pl->info.device_bytes += int64_t(bytes);
        return PSW_OK;
    };
    if (int rc = up(reinterpret_cast<void**>(&pl->d_hd_cta), ctas.data(), sizeof(RsGroup) * ctas.size())) return rc;
    if (int rc = up(reinterpret_cast<void**>(&pl->d_hd_run), runs.data(), sizeof(RsRun) * runs.size())) return rc;
    if (int rc = up(reinterpret_cast<void**>(&pl->d_hd_runcoef), rcoef.data(), sizeof(SegCoef) * rcoef.size())) return rc;
    if (int rc = up(reinterpret_cast<void**>(&pl->d_hd_runoff), runoff.data(), sizeof(int32_t) * runoff.size())) return rc;
    if (int rc = up(&pl->d_hd_coef, co.data(), sizeof(HoldCoef<float>) * co.size())) return rc;
    pl->hd_ncta = int(ctas.size());
    pl->hd_nruns = int(runs.size());
    pl->hd_maxrows = maxrows;
    return PSW_OK;
}

bool hold_supported(const psw_plan* pl, int layout, int64_t N, const void* F, int64_t ldf,
                    const void* X, int64_t ldx) {
    if (layout != PSW_LAYOUT_R || pl->hd_ncta < 1 || pl->dtype != PSW_F32 || N < kHdW ||
        N > (int64_t{1} << 30))
        return false;
    if ((reinterpret_cast<uintptr_t>(F) & 15) || (ldf * 4) % 16 || ldf < N) return false;
    if ((reinterpret_cast<uintptr_t>(X) & 15) || (ldx * 4) % 16 || ldx < N) return false;
    size_t smem, slab;
    return hold_stages(pl, smem, slab) >= 2 && tensor_map_encoder() != nullptr;
}

int solve_hold(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
               int layout, cudaStream_t s, void** ev, int nev) {
    if (!hold_supported(pl, layout, N, F, ldf, X, ldx)) {
        set_error(PSW_NOT_SUPPORTED, "hold path does not support this plan/shape");
        return PSW_NOT_SUPPORTED;
    }
    using T = float;
    CUtensorMap f32m, f1m, x32m, x1m;
    if (!hold_encode<T>(F, ldf, N, pl->n, &f32m, &f1m) || !hold_encode<T>(X, ldx, N, pl->n, &x32m, &x1m)) {
        set_error(PSW_NOT_SUPPORTED, "hold path: tensor map encoding failed");
        return PSW_NOT_SUPPORTED;
    }
    HoldArgs A{};
    size_t smem, slab;
    A.stages = hold_stages(pl, smem, slab);
    A.slab_bytes = uint32_t(slab);
    A.N = N;
    A.ntiles = int((N + kHdW - 1) / kHdW);
    A.depth = 2 * A.stages;
    A.P = int(pl->P);
    A.p = int(pl->p);
    A.ncta = pl->hd_ncta;
    A.nruns = pl->hd_nruns;
    A.maxrows = pl->hd_maxrows;
    A.hs = (A.p * 2 <= A.ncta) ? 2 : 1;
    A.slotw = uint32_t((5 * size_t(A.nruns) + 2 * size_t(A.P) + size_t(std::max(A.p, 1))) * 32);
    A.cta = pl->d_hd_cta;
    A.runs = pl->d_hd_run;
    A.rcoef = pl->d_hd_runcoef;
    A.runoff = pl->d_hd_runoff;
    A.desc = pl->d_segdesc;
    A.segc = pl->d_seg;
    A.coef = pl->d_hd_coef;
    A.cmat = pl->d_cmat;
    const size_t xbytes = size_t(A.depth) * A.slotw * sizeof(uint4);
    void* mem = nullptr;
    PSW_CUDA_TRY(scratch_alloc(&mem, xbytes, pl->device, s));
    A.xch = static_cast<uint4*>(mem);
    auto kern = hold_kernel<T>;
    {
        static std::mutex mu;
        static size_t set = 0;
        std::lock_guard<std::mutex> lk(mu);
        if (smem > set) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            if (e != cudaSuccess) {
                scratch_free(mem, s);
                return cuda_fail(e, "hold_kernel attribute");
            }
            set = smem;
        }
    }
    cudaError_t e = cudaMemsetAsync(mem, 0, xbytes, s);
    mark(ev, nev, 0, s);
    if (e == cudaSuccess) {
        void* args[] = {&f32m, &f1m, &x32m, &x1m, &A};
        e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(unsigned(A.ncta)),
                                        dim3(kHdThreads), args, smem, s);
    }
    mark(ev, nev, 1, s);
    scratch_free(mem, s);
    if (e != cudaSuccess) return cuda_fail(e, "hold_kernel launch");
    note_launches(1);
    return PSW_OK;
}

}  // namespace psw
