// STAGED solve path: three kernels, any partition, any shape, both layouts.
//
//   K1 fwd      one thread per (rhs k, block t): forward sweep of the block's
//               unit-row system (local_solve.hpp:39-48 + thomas.hpp:31-41 in
//               the affine form of psw_internal.h) fused with both beta dot
//               products (betas.hpp:42-57) on the same read of F; the forward
//               intermediate d0 is parked in X.
//   K2 combine  one thread per rhs: the dichotomy combination in level order
//               (boundary_solve.hpp:96-121) -> boundary values V.
//   K3 bwd      one thread per (rhs k, block t): back substitution with the
//               boundary values, x = d0 + x_l w + al x_next, in place in X.
//
// HBM traffic: F read once, X written twice and read once (d0 round trip):
// 4 s bytes / unknown; the FUSED path (psw_fused.cu) removes the round trip.
// Betas and the combination use separately rounded products and sums in the
// reference's summation order, so betas and boundary values are bitwise the
// reference's (compiled without FP contraction) for the same inputs.
#include "psw_device.cuh"
#include "psw_internal.h"

namespace psw {
namespace {

constexpr int kThreads = 128;
constexpr int kCoefChunk = 256;  // block rows whose coefficients are staged in shared memory

// rows per register batch: the next batch is loaded while the current one is
// swept, so 2 * kBatch rows per thread are in flight or in registers
template <typename T>
constexpr int kBatch = 16;

template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
    return __ldcs(p);  // F is read exactly once: evict-first
}

// L2 prefetch distance (rows) of the forward sweep's F stream: the HBM
// latency-bandwidth product is covered by fire-and-forget prefetches instead
// of registers (measured: fwd C1 64 -> 59 us, C2 7.74 -> 6.84 ms; the same in
// the backward sweep, whose d0 rows are recent writes, was a loss)
constexpr int kPrefetch = 64;
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Cooperative copy of coefficient rows [c0, c1) into shared memory.
template <typename C>
__device__ __forceinline__ void stage_rows(C* dst, const C* __restrict__ src, int c0, int c1) {
    __syncthreads();
    for (int i = threadIdx.x; i < c1 - c0; i += blockDim.x) dst[i] = src[c0 + i];
    __syncthreads();
}

// ---------------------------------------------------------------- layout R
// One thread per (rhs k, block t0 + blockIdx.y). F/X row 0 is global row
// row_off (row shards, psw_shard.cpp); betas land at [(t - t0) * N + k].
// The block's sweep coefficients are staged in shared memory (warp-uniform
// broadcasts), F rows stream through double-buffered register batches.
template <typename T>
__global__ void __launch_bounds__(kThreads) fwd_r_kernel(
    const T* F, int64_t ldf, T* X, int64_t ldx, int64_t N, const int32_t* __restrict__ blk,
    const FwdCoef<T>* __restrict__ cf, double* __restrict__ bl_out, double* __restrict__ br_out,
    int p, int t0, int row_off) {
    constexpr int U = kBatch<T>;
    __shared__ FwdCoef<T> cs[kCoefChunk];
    const int t = t0 + blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    const bool kv = k < N;
    const int s = blk[2 * t], e = blk[2 * t + 1];
    const T* f = F + (kv ? k : 0) - int64_t(row_off) * ldf;  // f[q * ldf] = global row q
    T* x = X + (kv ? k : 0) - int64_t(row_off) * ldx;
    T d = T(0);
    double br = 0.0, bl = 0.0;
    for (int c0 = s; c0 < e; c0 += kCoefChunk) {
        const int c1 = min(e, c0 + kCoefChunk);
        stage_rows(cs, cf, c0, c1);
        if (!kv) continue;
        const int nb = (c1 - c0) / U;
        T cur[U], nxt[U];
        if (nb > 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) cur[u] = ld_stream(f + int64_t(c0 + u) * ldf);
        }
        int q = c0;
        for (int bi = 0; bi < nb; ++bi, q += U) {
            if (bi + 1 < nb) {
#pragma unroll
                for (int u = 0; u < U; ++u) nxt[u] = ld_stream(f + int64_t(q + U + u) * ldf);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (q + kPrefetch + u < e) prefetch_l2(f + int64_t(q + kPrefetch + u) * ldf);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const FwdCoef<T> c = cs[q - c0 + u];
                d = fma(c.ma, d, cur[u] * c.rp);
                br = madd_rn(br, double(cur[u]), double(c.gr));
                bl = madd_rn(bl, double(cur[u]), double(c.gl));
                x[int64_t(q + u) * ldx] = d;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) cur[u] = nxt[u];
        }
        for (; q < c1; ++q) {
            const T fv = ld_stream(f + int64_t(q) * ldf);
            const FwdCoef<T> c = cs[q - c0];
            d = fma(c.ma, d, fv * c.rp);
            br = madd_rn(br, double(fv), double(c.gr));
            bl = madd_rn(bl, double(fv), double(c.gl));
            x[int64_t(q) * ldx] = d;
        }
    }
    if (kv) {
        if (t < p) br_out[int64_t(t - t0) * N + k] = br;
        if (t > 0) bl_out[int64_t(t - t0) * N + k] = bl;
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) bwd_r_kernel(
    T* X, int64_t ldx, int64_t N, const int32_t* __restrict__ blk,
    const BwdCoef<T>* __restrict__ cb, const double* __restrict__ V, int p, int t0, int row_off) {
    constexpr int U = kBatch<T>;
    __shared__ BwdCoef<T> cs[kCoefChunk];
    const int t = t0 + blockIdx.y;
    const int64_t k = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    const bool kv = k < N;
    const int s = blk[2 * t], e = blk[2 * t + 1];
    T xl = T(0), xn = T(0);
    if (kv) {
        xl = t > 0 ? T(V[int64_t(t - 1) * N + k]) : T(0);
        xn = t < p ? T(V[int64_t(t) * N + k]) : T(0);
    }
    T* x = X + (kv ? k : 0) - int64_t(row_off) * ldx;
    for (int c1 = e; c1 > s; c1 -= kCoefChunk) {
        const int c0 = max(s, c1 - kCoefChunk);
        stage_rows(cs, cb, c0, c1);
        if (!kv) continue;
        const int nb = (c1 - c0) / U;
        T cur[U], nxt[U];
        if (nb > 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) cur[u] = x[int64_t(c1 - 1 - u) * ldx];
        }
        int q = c1 - 1;  // rows q, q-1, ..., q-U+1 form the current batch
        for (int bi = 0; bi < nb; ++bi, q -= U) {
            if (bi + 1 < nb) {
#pragma unroll
                for (int u = 0; u < U; ++u) nxt[u] = x[int64_t(q - U - u) * ldx];
            }

#pragma unroll
            for (int u = 0; u < U; ++u) {
                const BwdCoef<T> c = cs[q - u - c0];
                xn = fma(c.al, xn, fma(xl, c.w, cur[u]));
                __stcs(x + int64_t(q - u) * ldx, xn);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) cur[u] = nxt[u];
        }
        for (; q >= c0; --q) {
            const BwdCoef<T> c = cs[q - c0];
            xn = fma(c.al, xn, fma(xl, c.w, x[int64_t(q) * ldx]));
            __stcs(x + int64_t(q) * ldx, xn);
        }
    }
}

// ---------------------------------------------------------------- layout S
// One warp per (32 RHS, block): chunks of 32 rows are read coalesced along
// the system (each RHS contiguous), transposed through shared memory so each
// lane sweeps its own RHS, and written back the same way. Two tiles per warp:
// the next chunk's loads are in flight while the current one is swept.
constexpr int kWarps = kThreads / 32;

// Asynchronous tile load (cp.async: global -> shared without a register
// round trip), so a warp can sweep one tile while the next is in flight.
template <typename T>
__device__ __forceinline__ void tile_load(T (*tile)[33], const T* src, int64_t ld, int cnt,
                                          int nk, int lane, bool /*streaming*/) {
    if (lane < cnt) {
        const T* p = src + lane;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nk) {
                const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tile[j][lane]));
                asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst),
                             "l"(p + int64_t(j) * ld), "n"(sizeof(T))
                             : "memory");
            }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
// wait until at most `pending` of this thread's tile loads are outstanding
template <int pending>
__device__ __forceinline__ void tile_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(pending) : "memory");
    __syncwarp();
}

template <typename T>
__device__ __forceinline__ void tile_store(T (*tile)[33], T* dst, int64_t ld, int cnt, int nk,
                                           int lane, bool streaming) {
    if (lane < cnt) {
        T* p = dst + lane;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nk) {
                if (streaming) __stcs(p + int64_t(j) * ld, tile[j][lane]);
                else p[int64_t(j) * ld] = tile[j][lane];
            }
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) fwd_s_kernel(
    const T* F, int64_t ldf, T* X, int64_t ldx, int64_t N, const int32_t* __restrict__ blk,
    const FwdCoef<T>* __restrict__ cf, double* __restrict__ bl_out, double* __restrict__ br_out,
    int p) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    FwdCoef<T>* cs = reinterpret_cast<FwdCoef<T>*>(s_raw);
    auto tiles = reinterpret_cast<T(*)[2][32][33]>(s_raw + kCoefChunk * sizeof(FwdCoef<T>));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.y;
    const int64_t k0 = (int64_t(blockIdx.x) * kWarps + warp) * 32;
    const bool wv = k0 < N;
    const int nk = wv ? int(N - k0 < 32 ? N - k0 : 32) : 0;
    const int s = blk[2 * t], e = blk[2 * t + 1];
    const T* src = F + (wv ? k0 : 0) * ldf;
    T* dst = X + (wv ? k0 : 0) * ldx;
    T d = T(0);
    double br = 0.0, bl = 0.0;
    for (int c0 = s; c0 < e; c0 += kCoefChunk) {
        const int c1 = min(e, c0 + kCoefChunk);
        stage_rows(cs, cf, c0, c1);
        if (!wv) continue;
        int buf = 0;
        tile_load(tiles[warp][0], src + c0, ldf, min(32, c1 - c0), nk, lane, true);
        for (int q0 = c0; q0 < c1; q0 += 32, buf ^= 1) {
            const int cnt = min(32, c1 - q0);
            if (q0 + 32 < c1) {  // next chunk in flight while this one is swept
                tile_load(tiles[warp][buf ^ 1], src + q0 + 32, ldf, min(32, c1 - q0 - 32), nk,
                          lane, true);
                // the chunk after that into L2 (no shared memory needed)
                if (q0 + 64 + lane < e) {
#pragma unroll 8
                    for (int j = 0; j < 32; ++j)
                        if (j < nk) prefetch_l2(src + int64_t(j) * ldf + q0 + 64 + lane);
                }
                tile_wait<1>();
            } else {
                tile_wait<0>();
            }
            T(*tile)[33] = tiles[warp][buf];
            if (lane < nk) {
                auto row = [&](int r) {
                    const FwdCoef<T> c = cs[q0 - c0 + r];
                    const T fv = tile[lane][r];
                    d = fma(c.ma, d, fv * c.rp);
                    br = madd_rn(br, double(fv), double(c.gr));
                    bl = madd_rn(bl, double(fv), double(c.gl));
                    tile[lane][r] = d;
                };
                if (cnt == 32) {
#pragma unroll
                    for (int r = 0; r < 32; ++r) row(r);
                } else {
                    for (int r = 0; r < cnt; ++r) row(r);
                }
            }
            __syncwarp();
            tile_store(tile, dst + q0, ldx, cnt, nk, lane, false);
            __syncwarp();
        }
    }
    if (wv && lane < nk) {
        if (t < p) br_out[int64_t(t) * N + k0 + lane] = br;
        if (t > 0) bl_out[int64_t(t) * N + k0 + lane] = bl;
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) bwd_s_kernel(
    T* X, int64_t ldx, int64_t N, const int32_t* __restrict__ blk,
    const BwdCoef<T>* __restrict__ cb, const double* __restrict__ V, int p) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    BwdCoef<T>* cs = reinterpret_cast<BwdCoef<T>*>(s_raw);
    auto tiles = reinterpret_cast<T(*)[2][32][33]>(s_raw + kCoefChunk * sizeof(BwdCoef<T>));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.y;
    const int64_t k0 = (int64_t(blockIdx.x) * kWarps + warp) * 32;
    const bool wv = k0 < N;
    const int nk = wv ? int(N - k0 < 32 ? N - k0 : 32) : 0;
    const int s = blk[2 * t], e = blk[2 * t + 1];
    T* xs = X + (wv ? k0 : 0) * ldx;
    T xl = T(0), xn = T(0);
    if (wv && lane < nk) {
        if (t > 0) xl = T(V[int64_t(t - 1) * N + k0 + lane]);
        if (t < p) xn = T(V[int64_t(t) * N + k0 + lane]);
    }
    for (int c1 = e; c1 > s; c1 -= kCoefChunk) {
        const int c0 = max(s, c1 - kCoefChunk);
        stage_rows(cs, cb, c0, c1);
        if (!wv) continue;
        int buf = 0;
        {
            const int q0 = max(c0, c1 - 32);
            tile_load(tiles[warp][0], xs + q0, ldx, c1 - q0, nk, lane, false);
        }
        for (int q1 = c1; q1 > c0; q1 -= 32, buf ^= 1) {
            const int q0 = max(c0, q1 - 32);
            const int cnt = q1 - q0;
            if (q0 > c0) {
                const int n0 = max(c0, q0 - 32);
                tile_load(tiles[warp][buf ^ 1], xs + n0, ldx, q0 - n0, nk, lane, false);
                // the chunk after that into L2 (no shared memory needed)
                const int p0 = max(c0, n0 - 32);
                if (p0 < n0 && lane < n0 - p0) {
#pragma unroll 8
                    for (int j = 0; j < 32; ++j)
                        if (j < nk) prefetch_l2(xs + int64_t(j) * ldx + p0 + lane);
                }
                tile_wait<1>();
            } else {
                tile_wait<0>();
            }
            T(*tile)[33] = tiles[warp][buf];
            if (lane < nk) {
                auto row = [&](int r) {
                    const BwdCoef<T> c = cs[q0 - c0 + r];
                    xn = fma(c.al, xn, fma(xl, c.w, tile[lane][r]));
                    tile[lane][r] = xn;
                };
                if (cnt == 32) {
#pragma unroll
                    for (int r = 31; r >= 0; --r) row(r);
                } else {
                    for (int r = cnt - 1; r >= 0; --r) row(r);
                }
            }
            __syncwarp();
            tile_store(tile, xs + q0, ldx, cnt, nk, lane, true);
            __syncwarp();
        }
    }
}

template <typename T, typename C>
constexpr size_t s_smem() {
    return kCoefChunk * sizeof(C) + size_t(kWarps) * 2 * 32 * 33 * sizeof(T);
}

// --------------------------------------------------------------- combine
// One thread per RHS, 32 RHS per CTA. For P <= kStageP the CTA first stages
// its RHS' betas (coalesced, all loads in flight) and keeps the boundary
// values in shared memory; larger P reads betas from global/L2.
constexpr int kCombineThreads = 32;
constexpr int kStageP = 96;
constexpr int kStageTables = 40;  // Z samples + items in shared memory up to this P

__global__ void __launch_bounds__(kCombineThreads) combine_kernel(
    const double* __restrict__ bl, const double* __restrict__ br, int64_t N, int p,
    const CombineItem* __restrict__ items, const double* __restrict__ zr,
    const double* __restrict__ zl, double* __restrict__ V) {
    extern __shared__ double sh[];  // [2][P][32] betas + [p][32] values (+ tables)
    const int lane = threadIdx.x;
    const int64_t k0 = int64_t(blockIdx.x) * kCombineThreads;
    const int64_t k = k0 + lane;
    const int P = p + 1;
    if (P <= kStageP) {
        double* sl = sh;
        double* sr = sh + P * kCombineThreads;
        double* sv = sh + 2 * P * kCombineThreads;
        if (P <= kStageTables) {
            // the Z samples and the items as well: the level-order recurrence
            // then never waits on a cached global load
            double* szr = sv + p * kCombineThreads;
            double* szl = szr + p * p;
            CombineItem* sit = reinterpret_cast<CombineItem*>(szl + p * p);
            for (int i = lane; i < p * p; i += kCombineThreads) {
                szr[i] = zr[i];
                szl[i] = zl[i];
            }
            for (int i = lane; i < p; i += kCombineThreads) sit[i] = items[i];
            zr = szr;
            zl = szl;
            items = sit;
        }
        for (int t = 0; t < P; ++t) {
            sl[t * kCombineThreads + lane] = k < N ? bl[int64_t(t) * N + k] : 0.0;
            sr[t * kCombineThreads + lane] = k < N ? br[int64_t(t) * N + k] : 0.0;
        }
        __syncwarp();
        if (k < N) combine_rhs(items, p, sl + lane, sr + lane, kCombineThreads, zr, zl, sv + lane,
                               kCombineThreads);
        __syncwarp();
        if (k < N)
            for (int j = 0; j < p; ++j) V[int64_t(j) * N + k] = sv[j * kCombineThreads + lane];
    } else if (k < N) {
        combine_rhs(items, p, bl + k, br + k, N, zr, zl, V + k, N);
    }
}

size_t combine_smem(int64_t P) {
    if (P > kStageP) return 0;
    size_t b = sizeof(double) * kCombineThreads * (3 * P - 1);
    if (P <= kStageTables)
        b += sizeof(double) * 2 * size_t(P - 1) * size_t(P - 1) + sizeof(CombineItem) * size_t(P - 1);
    return b;
}

// beyond 48 KB of dynamic shared memory (P in 37..40 with staged tables)
// the kernel must opt in
int combine_prepare(int64_t P) {
    const size_t b = combine_smem(P);
    if (b > 48 * 1024)
        PSW_CUDA_TRY(cudaFuncSetAttribute(combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(b)));
    return PSW_OK;
}

template <typename T>
int launch_staged(const psw_plan* pl, const void* Fv, int64_t ldf, void* Xv, int64_t ldx,
                  int64_t N, int layout, cudaStream_t s, double* bl, double* br, double* V,
                  void** ev, int nev) {
    const T* F = static_cast<const T*>(Fv);
    T* X = static_cast<T*>(Xv);
    const int p = int(pl->p);
    const auto* cf = static_cast<const FwdCoef<T>*>(pl->d_fwd);
    const auto* cb = static_cast<const BwdCoef<T>*>(pl->d_bwd);
    int64_t launches = 0;
    if (layout == PSW_LAYOUT_R) {
        dim3 grid(unsigned((N + kThreads - 1) / kThreads), unsigned(pl->P));
        mark(ev, nev, 0, s);
        fwd_r_kernel<T><<<grid, kThreads, 0, s>>>(F, ldf, X, ldx, N, pl->d_blk, cf, bl, br, p, 0, 0);
        ++launches;
        mark(ev, nev, 1, s);
        if (p > 0) {
            if (int rc = combine_prepare(pl->P)) return rc;
            combine_kernel<<<unsigned((N + kCombineThreads - 1) / kCombineThreads), kCombineThreads,
                             combine_smem(pl->P), s>>>(bl, br, N, p, pl->d_items, pl->d_zr, pl->d_zl, V);
            ++launches;
        }
        mark(ev, nev, 2, s);
        bwd_r_kernel<T><<<grid, kThreads, 0, s>>>(X, ldx, N, pl->d_blk, cb, V, p, 0, 0);
        ++launches;
        mark(ev, nev, 3, s);
    } else {
        dim3 grid(unsigned((N + 32 * kWarps - 1) / (32 * kWarps)), unsigned(pl->P));
        constexpr size_t sf = s_smem<T, FwdCoef<T>>(), sb = s_smem<T, BwdCoef<T>>();
        PSW_CUDA_TRY(cudaFuncSetAttribute(fwd_s_kernel<T>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(sf)));
        PSW_CUDA_TRY(cudaFuncSetAttribute(bwd_s_kernel<T>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(sb)));
        mark(ev, nev, 0, s);
        fwd_s_kernel<T><<<grid, kThreads, sf, s>>>(F, ldf, X, ldx, N, pl->d_blk, cf, bl, br, p);
        ++launches;
        mark(ev, nev, 1, s);
        if (p > 0) {
            if (int rc = combine_prepare(pl->P)) return rc;
            combine_kernel<<<unsigned((N + kCombineThreads - 1) / kCombineThreads), kCombineThreads,
                             combine_smem(pl->P), s>>>(
                bl, br, N, p, pl->d_items, pl->d_zr, pl->d_zl, V);
            ++launches;
        }
        mark(ev, nev, 2, s);
        bwd_s_kernel<T><<<grid, kThreads, sb, s>>>(X, ldx, N, pl->d_blk, cb, V, p);
        ++launches;
        mark(ev, nev, 3, s);
    }
    PSW_CUDA_TRY(cudaGetLastError());
    note_launches(launches);
    return PSW_OK;
}

}  // namespace

int launch_combine(const psw_plan* pl, const double* bl, const double* br, int64_t N, double* V,
                   cudaStream_t s) {
    const int p = int(pl->p);
    if (p <= 0) return PSW_OK;
    if (int rc = combine_prepare(pl->P)) return rc;
    combine_kernel<<<unsigned((N + kCombineThreads - 1) / kCombineThreads), kCombineThreads,
                     combine_smem(pl->P), s>>>(bl, br, N, p, pl->d_items, pl->d_zr, pl->d_zl, V);
    PSW_CUDA_TRY(cudaGetLastError());
    return PSW_OK;
}

int solve_staged(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                 int layout, cudaStream_t s, double* ext_bl, double* ext_br, double* ext_v,
                 void** events, int nevents) {
    const int64_t P = pl->P, p = pl->p;
    // scratch: betas (P x N each) and boundary values (p x N), stream-ordered
    double* bl = ext_bl;
    double* br = ext_br;
    double* V = ext_v;
    void* scratch = nullptr;
    size_t need = 0;
    if (!bl) need += sizeof(double) * P * N;
    if (!br) need += sizeof(double) * P * N;
    if (!V) need += sizeof(double) * (p > 0 ? p : 1) * N;
    if (need) {
        PSW_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&scratch), need, pl->device, s));
        char* c = static_cast<char*>(scratch);
        if (!bl) { bl = reinterpret_cast<double*>(c); c += sizeof(double) * P * N; }
        if (!br) { br = reinterpret_cast<double*>(c); c += sizeof(double) * P * N; }
        if (!V) { V = reinterpret_cast<double*>(c); }
    }
    int rc = pl->dtype == PSW_F64
                 ? launch_staged<double>(pl, F, ldf, X, ldx, N, layout, s, bl, br, V, events, nevents)
                 : launch_staged<float>(pl, F, ldf, X, ldx, N, layout, s, bl, br, V, events, nevents);
    if (scratch) scratch_free(scratch, s);
    return rc;
}

// ------------------------------------------------------------ data fill
namespace {
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ double unit53(uint64_t seed, uint64_t idx) {
    return __dmul_rn(double(splitmix64(seed ^ idx) >> 11), 1.0 / 9007199254740992.0);
}

template <typename T>
__global__ void fill_uniform_kernel(T* out, int64_t count, uint64_t seed, uint64_t offset,
                                    double lo, double span) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = T(__dadd_rn(lo, __dmul_rn(span, unit53(seed, offset + uint64_t(i)))));
}

template <typename T>
__global__ void fill_normal_kernel(T* out, int64_t count, uint64_t seed, uint64_t offset) {
    const int64_t pairs = (count + 1) / 2;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < pairs;
         i += int64_t(gridDim.x) * blockDim.x) {
        const double u1 = 1.0 - unit53(seed, offset + 2 * uint64_t(i));  // (0, 1]
        const double u2 = unit53(seed, offset + 2 * uint64_t(i) + 1);
        const double r = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        out[2 * i] = T(r * cs);
        if (2 * i + 1 < count) out[2 * i + 1] = T(r * sn);
    }
}
}  // namespace

int fill_uniform(void* dst, int dtype, int64_t count, uint64_t seed, uint64_t offset, double lo,
                 double hi, cudaStream_t s) {
    if (!dst || count < 0) {
        set_error(PSW_INVALID_ARGUMENT, "invalid fill buffer");
        return PSW_INVALID_ARGUMENT;
    }
    if (count == 0) return PSW_OK;
    const unsigned blocks = 148 * 16;
    if (dtype == PSW_F64)
        fill_uniform_kernel<double><<<blocks, 256, 0, s>>>(static_cast<double*>(dst), count, seed, offset, lo, hi - lo);
    else
        fill_uniform_kernel<float><<<blocks, 256, 0, s>>>(static_cast<float*>(dst), count, seed, offset, lo, hi - lo);
    PSW_CUDA_TRY(cudaGetLastError());
    note_launches(1);
    return PSW_OK;
}

int fill_normal(void* dst, int dtype, int64_t count, uint64_t seed, uint64_t offset,
                cudaStream_t s) {
    if (!dst || count < 0) {
        set_error(PSW_INVALID_ARGUMENT, "invalid fill buffer");
        return PSW_INVALID_ARGUMENT;
    }
    if (count == 0) return PSW_OK;
    const unsigned blocks = 148 * 16;
    if (dtype == PSW_F64)
        fill_normal_kernel<double><<<blocks, 256, 0, s>>>(static_cast<double*>(dst), count, seed, offset);
    else
        fill_normal_kernel<float><<<blocks, 256, 0, s>>>(static_cast<float*>(dst), count, seed, offset);
    PSW_CUDA_TRY(cudaGetLastError());
    note_launches(1);
    return PSW_OK;
}

int l2_flush(void* scratch, int64_t bytes, cudaStream_t s) {
    PSW_CUDA_TRY(cudaMemsetAsync(scratch, 0, size_t(bytes), s));
    return PSW_OK;
}

}  // namespace psw
