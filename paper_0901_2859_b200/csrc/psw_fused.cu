// FUSED solve path: one persistent kernel, F read once, X written once (the
// minimum traffic of SURVEY §8(d)); forward intermediates never leave the chip.
//
// Work decomposition (layout R, uniform partition n = P*m):
//   * an RHS tile = W right-hand sides (128 contiguous bytes per row by
//     default, 256 with PSW_FUSED_ROW_BYTES=256);
//   * one thread-block CLUSTER of C CTAs owns a tile; CTA c owns G
//     consecutive blocks (P = C*G): rows [c*G*m - 1, (c+1)*G*m - 1), the
//     reference's half-open blocks (partition.hpp:26-29). Clusters are
//     persistent and walk the tiles cluster_id, cluster_id + nclusters, ...;
//   * TMA streams the CTA's rows (box W x 32 rows, one mbarrier per box) into
//     a shared-memory slab; the plan tables (sweep coefficients, segment
//     constants, rows of the combination matrix) arrive once by bulk copy;
//   * every block is cut into S segments of kSegLen rows, one thread per
//     (block, segment, rhs): the forward sweep and both beta dot products
//     (betas.hpp:42-57) run S-wide with d~ kept in registers, segment carries
//     are exact affine scans (psw_internal.h, FusedFwd/FusedBwd). The slab is
//     refilled with the next tile as soon as the sweep has read it;
//   * block betas are pushed to every CTA of the cluster with st.async
//     (DSMEM stores that complete bytes on the receiver's mbarrier: no
//     cluster-wide barrier per tile);
//   * the dichotomy combination (boundary_solve.hpp:96-121) is linear in the
//     betas; the plan tabulates it (combination matrix, psw_plan.cpp
//     combine_matrix) and each CTA evaluates only its own boundary values;
//   * the backward sweep starts from exact segment carries and streams X with
//     evict-first stores.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cooperative_groups.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "psw_device.cuh"
#include "psw_internal.h"
#include "psw_tma.cuh"

namespace cg = cooperative_groups;

namespace psw {
namespace {

constexpr int kChunk = 32;                 // rows per TMA box / mbarrier
constexpr int kMaxCluster = 16;
constexpr int kMaxThreads = 256;  // threads per CTA
constexpr size_t kSmemTarget = 110 * 1024;  // >= 2 CTAs per SM
constexpr size_t kSmemMax = 200 * 1024;

// Optional per-CTA phase trace (psw_debug_trace): 16 slots per CTA and
// iteration 0, clock64() at phase boundaries, %globaltimer at start/end.
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PSW_TRACE(k)                                                                  \
    do {                                                                              \
        if (trace && it == 1 && threadIdx.x == 0) trace[blockIdx.x * 16 + (k)] = clock64(); \
    } while (0)

// shared::cluster address of `addr` (own CTA) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

// 16-byte remote store that completes its bytes on the remote mbarrier
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double a, double b, uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
            raddr),
        "d"(a), "d"(b), "r"(rbar)
        : "memory");
}


// CTA-wide named barrier (id 1)
__device__ __forceinline__ void cta_sync(int nc) {
    asm volatile("bar.sync 1, %0;" ::"r"(nc) : "memory");
}

struct FusedGeom {
    int n, P, p, m, G, C, S, rows_alloc, nchunks, prefetch;
    int64_t N, ldx, ntiles;
};

// Shared-memory carve-up (bytes), identical on host and device: the slab
// (TMA landing zone, handed back to the producer right after the forward
// sweep), the plan tables loaded once, per-tile-parity scan buffers and beta
// exchange buffers.
struct FusedLayout {
    size_t slab_b, ff, fb, segc, cm, seg0, seg_b, part, all0, all_b, vals, bars, total;
    int nslab, nall;
    __host__ __device__ FusedLayout(int rows_alloc, int nchunks, int G, int S, int P, int W,
                                    int es, bool lag, bool gc) {
        auto up = [](size_t x) { return (x + 127) & ~size_t(127); };
        // LAG: two slabs (tile k+1 loads while tile k is swept and its d~
        // parked in place) and four exchange buffers (a peer may run up to
        // three tiles ahead of a CTA's combination, see FusedTile::step_lag)
        nslab = lag ? 2 : 1;
        nall = lag ? 4 : 2;
        slab_b = up(size_t(rows_alloc) * W * es);
        // GC: the sweep coefficients are read from global memory (L1-resident)
        // instead of being copied here, leaving shared memory to the slabs
        ff = nslab * slab_b;                                                     // FusedFwd rows
        fb = up(ff + (gc ? 0 : size_t(rows_alloc) * (es == 8 ? 48 : 32)));      // FusedBwd rows
        segc = up(fb + (gc ? 0 : size_t(rows_alloc) * (es == 8 ? 32 : 16)));    // G*S SegCoef
        cm = up(segc + size_t(G) * S * sizeof(SegCoef));            // (G+1) x 2P doubles
        seg0 = up(cm + size_t(G + 1) * 2 * P * sizeof(double));     // 3 x G*S*W doubles / parity
        seg_b = up(size_t(3) * G * S * W * sizeof(double));
        part = seg0 + 2 * seg_b;                                    // 2 x G*S*W beta partials
        all0 = up(part + size_t(2) * G * S * W * sizeof(double));   // P x W x (R,L) / buffer
        all_b = up(size_t(2) * P * W * sizeof(double));
        vals = all0 + nall * all_b;                                 // P x W doubles
        bars = up(vals + size_t(P) * W * sizeof(double));           // slab chunks, plan, exchange
        total = bars + size_t(nslab * nchunks + 1 + nall) * sizeof(uint64_t);
    }
};

constexpr int kSegMax = kSegLen + 1;  // the last block owns m + 1 rows

// Forward rows of one segment, d~ kept in registers. NMAX is a compile-time
// bound (fully unrolled); rows q >= len are skipped (only when NMAX > len).
template <typename T, int W, int NMAX, bool UNI = false>
__device__ __forceinline__ void fwd_rows(const FusedFwd<T>* __restrict__ cf,
                                         const T* __restrict__ col, T (&dr)[kSegMax], T& d,
                                         T& sr, T& sl, T& sx, int len) {
#pragma unroll
    for (int q = 0; q < NMAX; ++q) {
        if (NMAX == kSegLen || (UNI && q < kSegLen - 1) || q < len) {
            const FusedFwd<T> c = cf[q];
            const T f = col[q * W];
            d = fma(c.ma, d, f * c.rp);
            sr = fma(f, c.gr, sr);
            sl = fma(f, c.gl, sl);
            sx = fma(c.lam, d, sx);
            dr[q] = d;
        }
    }
}

// Forward rows of one segment, d~ written back over f in the slab.
template <typename T, int W, int NMAX, bool UNI = false>
__device__ __forceinline__ void fwd_rows_smem(const FusedFwd<T>* __restrict__ cf, T* col, T& d,
                                              T& sr, T& sl, T& sx, int len) {
#pragma unroll
    for (int q = 0; q < NMAX; ++q) {
        if (NMAX == kSegLen || (UNI && q < kSegLen - 1) || q < len) {
            const FusedFwd<T> c = cf[q];
            const T f = col[q * W];
            d = fma(c.ma, d, f * c.rp);
            sr = fma(f, c.gr, sr);
            sl = fma(f, c.gl, sl);
            sx = fma(c.lam, d, sx);
            col[q * W] = d;
        }
    }
}

// Backward rows reading d~ from the slab (see bwd_rows).
template <typename T, int W, int NMAX, bool UNI = false>
__device__ __forceinline__ void bwd_rows_smem(const FusedBwd<T>* __restrict__ cb, const T* col,
                                              T D, T xl, T xn, T* xp, int64_t ldx, int len) {
#pragma unroll
    for (int q = NMAX - 1; q >= 0; --q) {
        if (NMAX == kSegLen || (UNI && q < kSegLen - 1) || q < len) {
            const FusedBwd<T> c = cb[q];
            const T cq = fma(xl, c.w, fma(c.mu, D, col[q * W]));
            xn = fma(c.al, xn, cq);
            __stcs(xp, xn);
            xp -= ldx;
        }
    }
}

// Backward rows of one segment from the exact carry xn, last row first;
// xp points at the segment's last row of X and walks up by ldx.
template <typename T, int NMAX, bool UNI = false>
__device__ __forceinline__ void bwd_rows(const FusedBwd<T>* __restrict__ cb,
                                         const T (&dr)[kSegMax], T D, T xl, T xn, T* xp,
                                         int64_t ldx, int len) {
#pragma unroll
    for (int q = NMAX - 1; q >= 0; --q) {
        if (NMAX == kSegLen || (UNI && q < kSegLen - 1) || q < len) {
            const FusedBwd<T> c = cb[q];
            const T cq = fma(xl, c.w, fma(c.mu, D, dr[q]));
            xn = fma(c.al, xn, cq);
            __stcs(xp, xn);
            xp -= ldx;
        }
    }
}

// Per-thread constants of the fused kernel.
struct FusedCtx {
    int tid, nc, lane, j, sg, t, a, b, len, c_lo, c_hi, row0, jb0, jb1;
};

// Persistent and software-pipelined. Each cluster walks the RHS tiles
// cluster_id, cluster_id + nclusters, ...; iteration k sweeps tile k+1
// forward (d~ in registers, the slab is handed back to the producer warp at
// once, which streams tile k+2 into it), then combines and back-substitutes
// tile k. A tile's DSMEM beta exchange therefore overlaps a back
// substitution and a forward sweep, and its HBM load overlaps a combination
// and a back substitution.
template <typename T, int W, bool LAG>
struct FusedTile {
    const FusedGeom& g;
    const FusedCtx& x;
    unsigned char* smem;
    const FusedLayout& L;
    const FusedFwd<T>* cf;
    const FusedBwd<T>* cb;
    const SegCoef* segc;
    const double* cm;
    uint64_t* bars;
    uint64_t* xbar;
    int crank, C;
    int64_t cluster_id, nclusters;
    T* X;
    const CUtensorMap* tmF;
    const CUtensorMap* tmF1;
    int nfull, rem;
    int64_t ntl_;

    // TMA of tile k's rows into the slab (one thread)
    __device__ __forceinline__ T* slab(int64_t k) const {
        return reinterpret_cast<T*>(smem + (LAG ? (k & 1) * L.slab_b : 0));
    }
    __device__ __forceinline__ uint64_t* slab_bars(int64_t k) const {
        return bars + (LAG ? (k & 1) * (nfull + (rem > 0)) : 0);
    }
    // mbarrier phase of tile k's slab barriers
    __device__ __forceinline__ uint32_t slab_phase(int64_t k) const {
        return uint32_t(LAG ? (k >> 1) : k) & 1u;
    }
    __device__ __forceinline__ void issue(int64_t k) const {
        T* sl = slab(k);
        uint64_t* bs = slab_bars(k);
        const int k0 = int((cluster_id + k * nclusters) * W);
        constexpr uint32_t box_bytes = uint32_t(W * kChunk * sizeof(T));
        for (int c = 0; c < nfull; ++c) {
            mbar_expect_tx(&bs[c], box_bytes);
            tma_load_2d(sl + size_t(c) * kChunk * W, tmF, k0, x.row0 + c * kChunk, &bs[c]);
        }
        if (rem) {  // tail rows through the one-row box
            mbar_expect_tx(&bs[nfull], uint32_t(rem * W * sizeof(T)));
            for (int r = 0; r < rem; ++r)
                tma_load_2d(sl + size_t(nfull * kChunk + r) * W, tmF1, k0,
                            x.row0 + nfull * kChunk + r, &bs[nfull]);
        }
        // tile k + 1 into L2 ahead of its load: doubles the bytes in flight
        // per CTA without shared memory (HBM latency ~4 us under load)
        if (g.prefetch && k + 1 < ntl_) {
            const int k1 = int((cluster_id + (k + 1) * nclusters) * W);
            for (int c = 0; c * kChunk < nfull * kChunk + rem; ++c)
                tma_prefetch_2d(tmF, k1, x.row0 + c * kChunk);
        }
    }

    __device__ __forceinline__ double* seg(int64_t k) const {
        return reinterpret_cast<double*>(smem + L.seg0 + (k & 1) * L.seg_b);
    }
    __device__ __forceinline__ double* allx(int64_t k) const {
        return reinterpret_cast<double*>(smem + L.all0 + (k & (LAG ? 3 : 1)) * L.all_b);
    }
    __device__ __forceinline__ uint64_t* xb(int64_t k) const { return &xbar[k & (LAG ? 3 : 1)]; }
    __device__ __forceinline__ uint32_t xphase(int64_t k) const {
        return uint32_t(k >> (LAG ? 2 : 1)) & 1u;
    }

    // forward sweep of tile k into dr; betas pushed after the scan
    __device__ __forceinline__ void forward(int64_t k, T (&dr)[kSegMax]) const {
        const int GSW = x.nc;
        if (x.tid == 0) mbar_expect_tx(xb(k), uint32_t(g.P * W * 2 * sizeof(double)));
        uint64_t* bs = slab_bars(k);
        for (int c = x.c_lo; c <= x.c_hi; ++c) mbar_wait(&bs[c], slab_phase(k));
        T* col = slab(k) + x.lane + (x.a - x.row0) * W;
        T d = T(0), sr = T(0), sl = T(0), sx = T(0);
        if constexpr (LAG) {  // d~ parked in place in the slab
            // segments of 31..33 rows (m % 32 == 0) share one instruction stream
            if (x.len >= kSegLen - 1)
                fwd_rows_smem<T, W, kSegMax, true>(cf, col, d, sr, sl, sx, x.len);
            else
                fwd_rows_smem<T, W, kSegMax>(cf, col, d, sr, sl, sx, x.len);
        } else {
            if (x.len >= kSegLen - 1)
                fwd_rows<T, W, kSegMax, true>(cf, col, dr, d, sr, sl, sx, x.len);
            else
                fwd_rows<T, W, kSegMax>(cf, col, dr, d, sr, sl, sx, x.len);
        }
        double* sk = seg(k);
        double* part = reinterpret_cast<double*>(smem + L.part);
        sk[x.tid] = double(d);         // d~ at the segment end
        sk[GSW + x.tid] = double(sx);  // Lam
        part[x.tid] = double(sr);
        part[GSW + x.tid] = double(sl);
    }

    // forward carries over the segments of a block; block betas
    __device__ __forceinline__ void fwd_scan(int64_t k, double& R, double& Lsum) const {
        R = 0.0;
        Lsum = 0.0;
        if (x.sg != 0) return;
        double* sk = seg(k);
        const double* part = reinterpret_cast<const double*>(smem + L.part);
        double D = 0.0;
        for (int q = 0; q < g.S; ++q) {
            const int id = (x.j * g.S + q) * W + x.lane;
            const double dend = sk[id];
            sk[id] = D;  // carry into segment q: D_{a-1}
            D = fma(segc[x.t * g.S + q].mu_end, D, dend);
            R += part[id];
            Lsum += part[x.nc + id];
        }
    }

    // st.async of this block's betas into every CTA of the cluster
    __device__ __forceinline__ void push(int64_t k, double R, double Lsum) const {
        if (x.sg != 0) return;
        const uint32_t src = smem_u32(allx(k)) + uint32_t((x.t * W + x.lane) * 16);
        const uint32_t bar = smem_u32(xb(k));
        for (int dst = 0; dst < C; ++dst) st_async_f64x2(mapa(src, dst), R, Lsum, mapa(bar, dst));
    }

    // boundary values of tile k this CTA needs: v = MR right + ML left, each
    // dot product split over 4 lanes and reduced with shuffles
    __device__ __forceinline__ void combine(int64_t k) const {
        mbar_wait(xb(k), xphase(k));
        const double* ax = allx(k);
        double* vals = reinterpret_cast<double*>(smem + L.vals);
        const int P = g.P, nout = (x.jb1 - x.jb0) * W;
        const int nwork = ((nout * 4 + 31) / 32) * 32;
        for (int idx = x.tid; idx < nwork; idx += x.nc) {
            const int o = idx >> 2, part = idx & 3;
            double s = 0.0;
            if (o < nout) {
                const int jb = o / W, ln = o % W;
                const double* Mr = cm + jb * 2 * P;
                for (int tt = part; tt < P; tt += 4) {
                    s = fma(Mr[tt], ax[(tt * W + ln) * 2], s);
                    s = fma(Mr[P + tt], ax[(tt * W + ln) * 2 + 1], s);
                }
            }
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            if (o < nout && part == 0) vals[x.jb0 * W + o] = s;
        }
    }

    // backward carries and back substitution of tile k (d~ from TMEM),
    // streamed to X
    __device__ __forceinline__ void backward(int64_t k, T (&dr)[kSegMax]) const {
        const int GSW = x.nc;
        double* sk = seg(k);
        const double* vals = reinterpret_cast<const double*>(smem + L.vals);
        const double xl = x.t > 0 ? vals[(x.t - 1) * W + x.lane] : 0.0;
        if (x.sg == 0) {
            double xb = x.t < g.p ? vals[x.t * W + x.lane] : 0.0;  // x at row e
            for (int q = g.S - 1; q >= 0; --q) {
                const int id = (x.j * g.S + q) * W + x.lane;
                const SegCoef sc = segc[x.t * g.S + q];
                const double xa = fma(xl, sc.k2, fma(sk[id], sc.k1, sk[GSW + id]));
                sk[2 * GSW + id] = xb;  // x at the row after the segment
                xb = fma(sc.nu, xb, xa);
            }
        }
        cta_sync(x.nc);
        const int64_t k0 = (cluster_id + k * nclusters) * W;
        const T D = T(sk[x.tid]);
        const T xlt = T(xl);
        const T xn = T(sk[2 * GSW + x.tid]);
        if (k0 + x.lane < g.N && x.len > 0) {
            T* xp = X + k0 + x.lane + int64_t(x.b - 1) * g.ldx;  // last row first
            if (x.len >= kSegLen - 1)
                bwd_rows<T, kSegMax, true>(cb, dr, D, xlt, xn, xp, g.ldx, x.len);
            else
                bwd_rows<T, kSegMax>(cb, dr, D, xlt, xn, xp, g.ldx, x.len);
        }
    }

    __device__ __forceinline__ void stamp(int64_t k, int slot) const {
        unsigned long long* tr = g_trace;
        if (tr && k == 2 && x.tid == 0) tr[blockIdx.x * 16 + slot] = clock64();
    }

    // LAG schedule, iteration k: forward sweep of tile k (d~ parked in its
    // slab) and push of its betas, then the combination and back
    // substitution of tile k-1, whose betas were pushed one iteration ago:
    // the cluster exchange no longer sits between a tile's two sweeps. Then
    // tile k's d~ moves to registers and its slab receives tile k+2.
    __device__ __forceinline__ void step_lag(int64_t k, int64_t ntl, T (&dr)[kSegMax]) const {
        stamp(k, 0);
        if (k < ntl) {
            forward(k, dr);
            stamp(k, 1);
            cta_sync(x.nc);
            double R, Lsum;
            fwd_scan(k, R, Lsum);
            push(k, R, Lsum);
        }
        stamp(k, 2);
        if (k >= 1) {
            combine(k - 1);
            stamp(k, 3);
            cta_sync(x.nc);
            stamp(k, 4);
            backward(k - 1, dr);
        }
        stamp(k, 5);
        if (k < ntl) {
            const T* col = slab(k) + x.lane + (x.a - x.row0) * W;
#pragma unroll
            for (int q = 0; q < kSegMax; ++q)
                if (q < x.len) dr[q] = col[q * W];
            cta_sync(x.nc);
            if (x.tid == 0 && k + 2 < ntl) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(k + 2);
            }
        }
        stamp(k, 6);
        unsigned long long* tr = g_trace;
        if (tr && x.tid == 0) {
            if (k == 0) tr[blockIdx.x * 16 + 10] = gtimer();
            tr[blockIdx.x * 16 + 11] = gtimer();
            tr[blockIdx.x * 16 + 12] = (unsigned long long)(k + 1);
        }
    }

    // iteration k: tile k end to end. The slab is handed back to the
    // producer right after the forward sweep (d~ stays in registers), so the
    // HBM load of tile k+1 overlaps the exchange, the combination and the
    // back substitution of tile k.
    __device__ __forceinline__ void step(int64_t k, int64_t ntl, T (&dr)[kSegMax]) const {
        stamp(k, 0);
        forward(k, dr);
        stamp(k, 1);
        cta_sync(x.nc);
        if (x.tid == 0 && k + 1 < ntl) {  // slab swept: stream the next tile into it
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(k + 1);
        }
        double R, Lsum;
        fwd_scan(k, R, Lsum);
        // pushing tile k only after combining tile k-1 keeps two exchange
        // buffers race-free (a peer's push of tile k+1 then needs this
        // CTA's betas of tile k)
        push(k, R, Lsum);
        stamp(k, 2);
        combine(k);
        stamp(k, 3);
        cta_sync(x.nc);
        stamp(k, 4);
        backward(k, dr);
        stamp(k, 5);
        stamp(k, 6);
        unsigned long long* tr = g_trace;
        if (tr && x.tid == 0) {
            if (k == 0) tr[blockIdx.x * 16 + 10] = gtimer();
            tr[blockIdx.x * 16 + 11] = gtimer();
            tr[blockIdx.x * 16 + 12] = (unsigned long long)(k + 1);
        }
    }
};

template <typename T, int W, bool LAG, bool GC>
__global__ void __launch_bounds__(kMaxThreads) fused_r_kernel(
    const __grid_constant__ CUtensorMap tmF, const __grid_constant__ CUtensorMap tmF1, T* X,
    FusedGeom g, const FusedFwd<T>* __restrict__ gff, const FusedBwd<T>* __restrict__ gfb,
    const SegCoef* __restrict__ gsegc, const double* __restrict__ gcmat) {
    extern __shared__ __align__(128) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int C = g.C, G = g.G, S = g.S, P = g.P, p = g.p, m = g.m;
    const int crank = int(cluster.block_rank());
    const int64_t cluster_id = blockIdx.x / C, nclusters = gridDim.x / C;
    const int64_t ntl = g.ntiles > cluster_id ? (g.ntiles - cluster_id + nclusters - 1) / nclusters : 0;
    // slab row 0 is global row c*G*m - 1 for every CTA (row -1 of CTA 0 is
    // out of bounds: TMA zero-fills it without touching memory)
    const int row0 = crank * G * m - 1;
    const int row1 = crank == C - 1 ? g.n : (crank + 1) * G * m - 1;
    const int crow0 = row0 < 0 ? 0 : row0;  // first coefficient row
    const FusedLayout L(g.rows_alloc, g.nchunks, G, S, P, W, int(sizeof(T)), LAG, GC);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* cbar = &bars[L.nslab * g.nchunks];      // plan tables
    uint64_t* xbar = &bars[L.nslab * g.nchunks + 1];  // [buffer]: betas of a tile from every peer
    const int nc = G * S * W;               // threads
    const int tid = threadIdx.x;
    const int nrows = row1 - row0;
    FusedCtx x;
    x.tid = tid;
    x.nc = nc;
    x.row0 = row0;
    x.jb0 = crank * G - 1 < 0 ? 0 : crank * G - 1;  // combination rows [jb0, jb1)
    x.jb1 = crank * G + G < p ? crank * G + G : p;
    // thread -> (block j, segment sg, rhs lane)
    x.lane = tid % W;
    const int h = tid / W;
    x.j = h / S;
    x.sg = h % S;
    x.t = crank * G + x.j;
    const int s = x.t == 0 ? 0 : x.t * m - 1;
    const int e = x.t == P - 1 ? g.n : (x.t + 1) * m - 1;
    x.a = s + x.sg * kSegLen;
    x.b = x.sg == S - 1 ? e : x.a + kSegLen;
    if (x.a > e) x.a = e;
    if (x.b > e) x.b = e;
    x.len = x.b - x.a;  // 0..kSegMax
    x.c_lo = x.len ? (x.a - row0) / kChunk : 0;
    x.c_hi = x.len ? (x.b - 1 - row0) / kChunk : -1;
    const FusedTile<T, W, LAG> ft{g, x, smem, L,
                             GC ? gff + x.a
                                : reinterpret_cast<const FusedFwd<T>*>(smem + L.ff) - crow0 + x.a,
                             GC ? gfb + x.a
                                : reinterpret_cast<const FusedBwd<T>*>(smem + L.fb) - crow0 + x.a,
                             reinterpret_cast<const SegCoef*>(smem + L.segc) - crank * G * S,
                             reinterpret_cast<const double*>(smem + L.cm),
                             bars, xbar, crank, C, cluster_id, nclusters, X,
                             &tmF, &tmF1, nrows / kChunk, nrows % kChunk, ntl};

    if (tid == 0) {
        for (int c = 0; c < L.nslab * (ft.nfull + (ft.rem > 0)); ++c) mbar_init(&bars[c], 1);
        mbar_init(cbar, 1);
        for (int i = 0; i < L.nall; ++i) mbar_init(&xbar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cluster.sync();  // peers may push into this CTA's exchange barriers from now on
    if (tid == 0) {
        // plan tables once (small, L2-resident), then the first tile
        const uint32_t crows = uint32_t(row1 - crow0);
        const uint32_t fwdb = GC ? 0u : crows * uint32_t(sizeof(FusedFwd<T>));
        const uint32_t bwdb = GC ? 0u : crows * uint32_t(sizeof(FusedBwd<T>));
        const uint32_t segb = uint32_t(G * S * sizeof(SegCoef));
        const uint32_t cmb = uint32_t(x.jb1 > x.jb0 ? (x.jb1 - x.jb0) * 2 * P * sizeof(double) : 0);
        mbar_expect_tx(cbar, fwdb + bwdb + segb + cmb);
        if (!GC) {
            bulk_load(smem + L.ff, gff + crow0, fwdb, cbar);
            bulk_load(smem + L.fb, gfb + crow0, bwdb, cbar);
        }
        bulk_load(smem + L.segc, gsegc + crank * G * S, segb, cbar);
        if (cmb) bulk_load(smem + L.cm, gcmat + size_t(x.jb0) * 2 * P, cmb, cbar);
        if (ntl > 0) ft.issue(0);
        if (LAG && ntl > 1) ft.issue(1);
    }
    mbar_wait(cbar, 0);
    T dr[kSegMax];
    if constexpr (LAG) {
        for (int64_t k = 0; k <= ntl; ++k) ft.step_lag(k, ntl, dr);
    } else {
        for (int64_t k = 0; k < ntl; ++k) ft.step(k, ntl, dr);
    }
}

// ---------------------------------------------------------------- host side
struct Choice {
    int W = 0, G = 0, C = 0, rows_alloc = 0, nchunks = 0;
    size_t smem = 0;
};

// Row width of an RHS tile: 128 B (choose() falls back to 256 B for tiny systems).
int tile_row_bytes() { return 128; }

// Smallest G (blocks per CTA) whose cluster C = P/G fits (<= 16 CTAs), then
// grow G while the CTA stays under the occupancy target.
Choice choose_w(const psw_plan* pl, int es, int row_bytes) {
    Choice ch;
    const int P = int(pl->P), m = int(pl->m), S = pl->nseg;
    const int W = row_bytes / es;
    if (S <= 0) return ch;
    static const int force_g = [] {
        const char* e = std::getenv("PSW_FUSED_G");  // tuning override
        return e ? std::atoi(e) : 0;
    }();
    for (int G = 1; G <= P; ++G) {
        if (P % G) continue;
        const int C = P / G;
        if (C > kMaxCluster) continue;
        if (force_g > 0 && G != force_g) continue;
        const int rows_alloc = G * m + 1;
        const int nchunks = (rows_alloc + kChunk - 1) / kChunk;
        const size_t smem =
            FusedLayout(rows_alloc, nchunks, G, S, P, W, es, false, false).total;
        if (smem > kSmemMax || G * S * W > kMaxThreads) break;
        if ((G * S * W) % 32) continue;  // consumer warps must be full
        if (ch.G == 0 || smem <= kSmemTarget) {
            ch.W = W;
            ch.G = G;
            ch.C = C;
            ch.rows_alloc = rows_alloc;
            ch.nchunks = nchunks;
            ch.smem = smem;
        }
        if (smem > kSmemTarget) break;
    }
    return ch;
}

Choice choose(const psw_plan* pl, int es) {
    if (!pl->uniform || pl->world != 1 || pl->n > (1 << 24) || !pl->d_ffwd) return Choice{};
    Choice ch = choose_w(pl, es, tile_row_bytes());
    if (ch.G == 0) ch = choose_w(pl, es, tile_row_bytes() == 128 ? 256 : 128);
    return ch;
}

bool encode_maps(CUtensorMap* tm, CUtensorMap* tm1, const void* F, int64_t N, int64_t n,
                 int64_t ldf, int es, int W) {
    auto encode = tensor_map_encoder();
    if (!encode) {
        set_error(PSW_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        return false;
    }
    const cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(n)};
    const cuuint64_t strides[1] = {cuuint64_t(ldf) * cuuint64_t(es)};
    const cuuint32_t box[2] = {cuuint32_t(W), cuuint32_t(kChunk)};
    const cuuint32_t box1[2] = {cuuint32_t(W), 1};
    const cuuint32_t estr[2] = {1, 1};
    const auto dt = es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r = encode(tm, dt, 2, const_cast<void*>(F), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
        r = encode(tm1, dt, 2, const_cast<void*>(F), dims, strides, box1, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error(PSW_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
        return false;
    }
    return true;
}

template <typename T, int W, bool LAG, bool GC>
int launch_w(const psw_plan* pl, const Choice& ch, const void* F, int64_t ldf, void* X,
             int64_t ldx, int64_t N, cudaStream_t s, void** ev, int nev) {
    CUtensorMap tm, tm1;
    if (!encode_maps(&tm, &tm1, F, N, pl->n, ldf, int(sizeof(T)), W)) return PSW_CUDA_ERROR;
    FusedGeom g;
    g.n = int(pl->n);
    g.P = int(pl->P);
    g.p = int(pl->p);
    g.m = int(pl->m);
    g.G = ch.G;
    g.C = ch.C;
    g.S = pl->nseg;
    g.rows_alloc = ch.rows_alloc;
    g.nchunks = ch.nchunks;
    g.prefetch = [] {  // L2 prefetch of the next tile (measured neutral on C1: off)
        const char* e = std::getenv("PSW_FUSED_PREFETCH");
        return e ? std::atoi(e) : 0;
    }();
    g.N = N;
    g.ldx = ldx;
    auto kern = fused_r_kernel<T, W, LAG, GC>;
    PSW_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ch.smem)));
    if (ch.C > 8) PSW_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int64_t tiles = (N + W - 1) / W;
    g.ntiles = tiles;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(unsigned(ch.G * g.S * W), 1, 1);
    cfg.dynamicSmemBytes = ch.smem;
    cfg.stream = s;
    PSW_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      cudaSharedmemCarveoutMaxShared));
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(ch.C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // pack a cluster's CTAs onto as few SMs as occupancy allows (the default
    // spread policy needs C distinct SMs of one GPC per cluster)
    attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[1].val.clusterSchedulingPolicyPreference =
        std::getenv("PSW_FUSED_SPREAD") ? cudaClusterSchedulingPolicySpread
                                        : cudaClusterSchedulingPolicyLoadBalancing;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    // persistent: as many clusters as can be co-resident (cached per config)
    static std::mutex mu;
    static std::vector<std::pair<std::array<int64_t, 6>, int>> cache;
    const std::array<int64_t, 6> key = {int64_t(sizeof(T)), W, ch.C, int64_t(ch.smem), pl->device,
                                        int64_t(LAG) + 4 * int64_t(GC)};
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
    int64_t nclusters = std::min<int64_t>(tiles, maxc);
    if (const char* e = std::getenv("PSW_FUSED_CLUSTERS"))  // tuning override
        nclusters = std::max<int64_t>(1, std::min<int64_t>(nclusters, std::atoll(e)));
    cfg.gridDim = dim3(unsigned(nclusters * ch.C), 1, 1);
    if (std::getenv("PSW_FUSED_VERBOSE"))
        std::fprintf(stderr, "fused: W=%d G=%d C=%d S=%d smem=%zu lag=%d gcoef=%d max_clusters=%d clusters=%lld\n",
                     W, ch.G, ch.C, g.S, ch.smem, int(LAG), int(GC), maxc, (long long)nclusters);
    mark(ev, nev, 0, s);
    PSW_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tm, tm1, static_cast<T*>(X), g,
                                    static_cast<const FusedFwd<T>*>(pl->d_ffwd),
                                    static_cast<const FusedBwd<T>*>(pl->d_fbwd), pl->d_seg,
                                    pl->d_cmat));
    mark(ev, nev, 1, s);
    note_launches(1);
    return PSW_OK;
}

template <typename T>
int launch_fused(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                 cudaStream_t s, void** ev, int nev) {
    const Choice ch = choose(pl, int(sizeof(T)));
    // the single-slab schedule with the coefficients in shared memory, 128-byte RHS
    // rows, or 256-byte rows where 128 bytes cannot fill a warp (choose(): tiny
    // systems of one segment per block). The LAG schedule and global-memory
    // coefficients (template parameters LAG, GC) were measured slower on C1 (124.6
    // and 184 us against 92.5 us before the segment fix) and are no longer built.
    return ch.W * int(sizeof(T)) == 256
               ? launch_w<T, 256 / sizeof(T), false, false>(pl, ch, F, ldf, X, ldx, N, s, ev, nev)
               : launch_w<T, 128 / sizeof(T), false, false>(pl, ch, F, ldf, X, ldx, N, s, ev, nev);
}

template <typename T>
int upload_fused(psw_plan* pl, const std::vector<FusedFwd<double>>& ffd,
                 const std::vector<FusedBwd<double>>& fbd, const std::vector<SegCoef>& seg) {
    const int64_t n = pl->n;
    std::vector<FusedFwd<T>> ff(n);
    std::vector<FusedBwd<T>> fb(n);
    for (int64_t q = 0; q < n; ++q) {
        const auto& a = ffd[q];
        const auto& b = fbd[q];
        ff[q] = {T(a.rp), T(a.ma), T(a.gr), T(a.gl), T(a.lam), T(0)};
        fb[q] = {T(b.mu), T(b.w), T(b.al), T(0)};
    }
    PSW_CUDA_TRY(cudaMalloc(&pl->d_ffwd, sizeof(FusedFwd<T>) * n));
    PSW_CUDA_TRY(cudaMalloc(&pl->d_fbwd, sizeof(FusedBwd<T>) * n));
    PSW_CUDA_TRY(cudaMalloc(&pl->d_seg, sizeof(SegCoef) * seg.size()));
    PSW_CUDA_TRY(cudaMemcpy(pl->d_ffwd, ff.data(), sizeof(FusedFwd<T>) * n, cudaMemcpyHostToDevice));
    PSW_CUDA_TRY(cudaMemcpy(pl->d_fbwd, fb.data(), sizeof(FusedBwd<T>) * n, cudaMemcpyHostToDevice));
    PSW_CUDA_TRY(cudaMemcpy(pl->d_seg, seg.data(), sizeof(SegCoef) * seg.size(), cudaMemcpyHostToDevice));
    pl->info.device_bytes += int64_t((sizeof(FusedFwd<T>) + sizeof(FusedBwd<T>)) * n +
                                     sizeof(SegCoef) * seg.size());
    return PSW_OK;
}

}  // namespace

int build_fused_tables(psw_plan* pl, const std::vector<double>& rp, const std::vector<double>& ma,
                       const std::vector<double>& gr, const std::vector<double>& gl,
                       const std::vector<double>& w, const std::vector<double>& al,
                       const std::vector<double>& cmat) {
    const int64_t n = pl->n, P = pl->P, m = pl->m;
    if (!cmat.empty()) {
        PSW_CUDA_TRY(cudaMalloc(&pl->d_cmat, sizeof(double) * cmat.size()));
        PSW_CUDA_TRY(cudaMemcpy(pl->d_cmat, cmat.data(), sizeof(double) * cmat.size(),
                                cudaMemcpyHostToDevice));
        pl->info.device_bytes += int64_t(sizeof(double) * cmat.size());
    }
    // Segmentation of every block into runs of at most kSegLen + 1 rows:
    // uniform partitions use S = ceil(m / kSegLen) segments for every block
    // (the FUSED kernel's thread map; block sizes m-1, m, m+1); others use
    // S_t = max(1, ceil((m_t - 1) / kSegLen)). The last segment of a block
    // absorbs the remainder (<= kSegLen + 1 rows).
    std::vector<int32_t> off(P + 1, 0);
    for (int64_t t = 0; t < P; ++t) {
        const int64_t mt = pl->blk[2 * t + 1] - pl->blk[2 * t];
        const int64_t St = pl->uniform ? (m + kSegLen - 1) / kSegLen
                                       : std::max<int64_t>(1, (mt - 1 + kSegLen - 1) / kSegLen);
        off[t + 1] = off[t] + int32_t(St);
    }
    pl->nseg = pl->uniform ? int((m + kSegLen - 1) / kSegLen) : 0;
    pl->seg_off = off;
    const int64_t NS = off[P];
    std::vector<FusedFwd<double>> ff(n);
    std::vector<FusedBwd<double>> fb(n);
    std::vector<SegCoef> seg(NS);
    std::vector<SegDesc> desc(NS);
    for (int64_t t = 0; t < P; ++t) {
        const int64_t s = pl->blk[2 * t], e = pl->blk[2 * t + 1];
        const int S = off[t + 1] - off[t];
        for (int sg = 0; sg < S; ++sg) {
            int64_t a = std::min(e, s + int64_t(sg) * kSegLen);
            int64_t b = sg == S - 1 ? e : std::min(e, a + kSegLen);
            double mu = 1.0, lam = 1.0, k1 = 0.0, k2 = 0.0;
            for (int64_t q = a; q < b; ++q) {
                mu *= ma[q];                        // prod_{u=a..q} ma_u
                ff[q] = {rp[q], ma[q], gr[q], gl[q], lam, 0.0};
                fb[q] = {mu, w[q], al[q], 0.0};
                k1 += lam * mu;
                k2 += lam * w[q];
                lam *= al[q];                       // prod_{u=a..q} al_u
            }
            seg[off[t] + sg] = {mu, k1, k2, lam};
            desc[off[t] + sg] = {int32_t(a), int32_t(b), int32_t(t), 0};
        }
    }
    PSW_CUDA_TRY(cudaMalloc(&pl->d_segdesc, sizeof(SegDesc) * NS));
    PSW_CUDA_TRY(cudaMemcpy(pl->d_segdesc, desc.data(), sizeof(SegDesc) * NS, cudaMemcpyHostToDevice));
    PSW_CUDA_TRY(cudaMalloc(&pl->d_segoff, sizeof(int32_t) * (P + 1)));
    PSW_CUDA_TRY(cudaMemcpy(pl->d_segoff, off.data(), sizeof(int32_t) * (P + 1), cudaMemcpyHostToDevice));
    pl->info.device_bytes += int64_t(sizeof(SegDesc) * NS + sizeof(int32_t) * (P + 1));
    const int rc = pl->dtype == PSW_F64 ? upload_fused<double>(pl, ff, fb, seg)
                                        : upload_fused<float>(pl, ff, fb, seg);
    if (rc != PSW_OK) return rc;
    if (int r = build_rs_tables(pl, desc, seg, ff, fb)) return r;
    return pl->world == 1 ? build_cluster_tables(pl, ff, fb) : PSW_OK;
}

int set_trace(void* buf) {
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    PSW_CUDA_TRY(cudaMemcpyToSymbol(g_trace, &p, sizeof(p)));
    return PSW_OK;
}

bool fused_supported(const psw_plan* pl, int layout, int64_t N, const void* F, int64_t ldf) {
    if (layout != PSW_LAYOUT_R || N < 1 || N > (int64_t{1} << 31)) return false;
    const int es = pl->dtype == PSW_F64 ? 8 : 4;
    // TMA: 16-byte aligned base and row pitch
    if ((reinterpret_cast<uintptr_t>(F) & 15) || ((size_t(ldf) * es) & 15)) return false;
    return choose(pl, es).G > 0;
}

int solve_fused(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx, int64_t N,
                int layout, cudaStream_t s, void** ev, int nev) {
    if (!fused_supported(pl, layout, N, F, ldf)) {
        set_error(PSW_NOT_SUPPORTED,
                  "fused path needs layout R, a uniform partition that fits a cluster, and "
                  "16-byte aligned F / row pitch");
        return PSW_NOT_SUPPORTED;
    }
    return pl->dtype == PSW_F64 ? launch_fused<double>(pl, F, ldf, X, ldx, N, s, ev, nev)
                                : launch_fused<float>(pl, F, ldf, X, ldx, N, s, ev, nev);
}

}  // namespace psw
