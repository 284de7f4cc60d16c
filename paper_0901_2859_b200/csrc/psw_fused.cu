// FUSED solve path: one kernel, F read once, X written once (the minimum
// traffic of SURVEY §8(d)); forward intermediates never leave the chip.
//
// Work decomposition (layout R, uniform partition n = P*m):
//   * an RHS tile = W right-hand sides (128 or 256 contiguous bytes per row);
//   * one thread-block CLUSTER of C CTAs owns the whole tile; CTA c owns G
//     consecutive blocks (P = C*G): rows [c*G*m - 1, (c+1)*G*m - 1), the
//     reference's half-open blocks (partition.hpp:26-29);
//   * TMA streams the CTA's rows (box W x 32 rows, one mbarrier per box) into
//     a shared-memory slab; the block's sweep coefficients arrive by one bulk
//     copy;
//   * every block is cut into S segments of kSegLen rows, one thread per
//     (block, segment, rhs), so a block's forward sweep, its two beta dot
//     products (betas.hpp:42-57) and the backward sweep run S-wide; segment
//     carries are exact affine scans (psw_internal.h, FusedFwd/FusedBwd);
//   * betas of all P blocks meet through distributed shared memory (DSMEM);
//     every CTA evaluates the dichotomy combination (boundary_solve.hpp:
//     96-121) level by level, the items of one level in parallel, with the
//     exact per-item arithmetic of the STAGED path;
//   * the backward sweep reads d~ from the slab and streams X with
//     evict-first stores.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>

#include "psw_device.cuh"
#include "psw_internal.h"

namespace cg = cooperative_groups;

namespace psw {
namespace {

constexpr int kChunk = 32;                 // rows per TMA box / mbarrier
constexpr int kMaxCluster = 16;
constexpr int kMaxThreads = 512;
constexpr size_t kSmemTarget = 72 * 1024;  // ~3 CTAs per SM
constexpr size_t kSmemMax = 200 * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(phase)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Optional per-CTA phase trace (psw_debug_trace): 16 slots per CTA,
// clock64() at phase boundaries, %globaltimer at start/end.
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PSW_TRACE(k)                                                         \
    do {                                                                     \
        if (trace && threadIdx.x == 0) trace[blockIdx.x * 16 + (k)] = clock64(); \
    } while (0)

struct FusedGeom {
    int n, P, p, m, G, C, S, rows_alloc, nchunks;
    int64_t N, ldx;
};

// Shared-memory carve-up (bytes), identical on host and device.
struct FusedLayout {
    size_t slab, ff, fb, seg, own, all, vals, segc, cm, bars, total;
    __host__ __device__ FusedLayout(int rows_alloc, int nchunks, int G, int S, int P, int W,
                                    int es) {
        auto up = [](size_t x) { return (x + 127) & ~size_t(127); };
        slab = 0;                                                   // rows x W values
        ff = up(size_t(rows_alloc) * W * es);                       // FusedFwd rows
        fb = up(ff + size_t(rows_alloc) * (es == 8 ? 48 : 32));     // FusedBwd rows
        seg = up(fb + size_t(rows_alloc) * (es == 8 ? 32 : 16));    // 4 x G*S*W doubles
        own = up(seg + size_t(4) * G * S * W * sizeof(double));     // 2 x G*W doubles
        all = up(own + size_t(2) * G * W * sizeof(double));         // 2 x P*W doubles
        vals = up(all + size_t(2) * P * W * sizeof(double));        // P x W doubles
        segc = up(vals + size_t(P) * W * sizeof(double));           // G*S SegCoef
        cm = up(segc + size_t(G) * S * sizeof(SegCoef));            // (G+1) x 2P doubles
        bars = up(cm + size_t(G + 1) * 2 * P * sizeof(double));
        total = bars + size_t(nchunks + 1) * sizeof(uint64_t);
    }
};

template <typename T, int W>
__global__ void __launch_bounds__(kMaxThreads) fused_r_kernel(
    const __grid_constant__ CUtensorMap tmF, const __grid_constant__ CUtensorMap tmF1, T* X,
    FusedGeom g, const FusedFwd<T>* __restrict__ gff, const FusedBwd<T>* __restrict__ gfb,
    const SegCoef* __restrict__ gsegc, const double* __restrict__ gcmat) {
    extern __shared__ __align__(128) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int C = g.C, G = g.G, S = g.S, P = g.P, p = g.p, m = g.m;
    const int crank = int(cluster.block_rank());
    const int64_t k0 = int64_t(blockIdx.x / C) * W;
    // slab row 0 is global row c*G*m - 1 for every CTA (row -1 of CTA 0 is
    // out of bounds: TMA zero-fills it without touching memory)
    const int row0 = crank * G * m - 1;
    const int row1 = crank == C - 1 ? g.n : (crank + 1) * G * m - 1;
    const int crow0 = row0 < 0 ? 0 : row0;  // first coefficient row

    const FusedLayout L(g.rows_alloc, g.nchunks, G, S, P, W, int(sizeof(T)));
    T* slab = reinterpret_cast<T*>(smem + L.slab);
    const FusedFwd<T>* ff = reinterpret_cast<const FusedFwd<T>*>(smem + L.ff) - crow0;
    const FusedBwd<T>* fb = reinterpret_cast<const FusedBwd<T>*>(smem + L.fb) - crow0;
    const int GSW = G * S * W;
    double* seg_d = reinterpret_cast<double*>(smem + L.seg);  // d~ end -> carry D_{a-1}
    double* seg_lam = seg_d + GSW;                             // Lam
    double* seg_br = seg_lam + GSW;                            // beta_R partial -> x carry
    double* seg_bl = seg_br + GSW;                             // beta_L partial
    double* own_r = reinterpret_cast<double*>(smem + L.own);
    double* own_l = own_r + G * W;
    double* all_r = reinterpret_cast<double*>(smem + L.all);
    double* all_l = all_r + P * W;
    double* vals = reinterpret_cast<double*>(smem + L.vals);
    const SegCoef* segc = reinterpret_cast<const SegCoef*>(smem + L.segc) - crank * G * S;
    // boundary rows [jb0, jb1) of the combination matrix this CTA needs
    const int jb0 = crank * G - 1 < 0 ? 0 : crank * G - 1;
    const int jb1 = crank * G + G < p ? crank * G + G : p;
    const double* cm = reinterpret_cast<const double*>(smem + L.cm);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* cbar = &bars[g.nchunks];

    const int tid = threadIdx.x;
    unsigned long long* const trace = g_trace;
    if (trace && tid == 0) trace[blockIdx.x * 16 + 14] = gtimer();
    PSW_TRACE(0);
    const int nrows = row1 - row0;
    const int nfull = nrows / kChunk, rem = nrows % kChunk;
    if (tid == 0) {
        for (int c = 0; c < nfull + (rem > 0); ++c) mbar_init(&bars[c], 1);
        mbar_init(cbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        // plan tables first (small, L2-resident), then the RHS rows
        const uint32_t crows = uint32_t(row1 - crow0);
        const uint32_t fwdb = crows * uint32_t(sizeof(FusedFwd<T>));
        const uint32_t bwdb = crows * uint32_t(sizeof(FusedBwd<T>));
        const uint32_t segb = uint32_t(G * S * sizeof(SegCoef));
        const uint32_t cmb = uint32_t(jb1 > jb0 ? (jb1 - jb0) * 2 * P * sizeof(double) : 0);
        mbar_expect_tx(cbar, fwdb + bwdb + segb + cmb);
        bulk_load(smem + L.ff, gff + crow0, fwdb, cbar);
        bulk_load(smem + L.fb, gfb + crow0, bwdb, cbar);
        bulk_load(smem + L.segc, gsegc + crank * G * S, segb, cbar);
        if (cmb) bulk_load(smem + L.cm, gcmat + size_t(jb0) * 2 * P, cmb, cbar);
        constexpr uint32_t box_bytes = uint32_t(W * kChunk * sizeof(T));
        for (int c = 0; c < nfull; ++c) {
            mbar_expect_tx(&bars[c], box_bytes);
            tma_load_2d(slab + size_t(c) * kChunk * W, &tmF, int(k0), row0 + c * kChunk, &bars[c]);
        }
        if (rem) {  // tail rows through the one-row box
            mbar_expect_tx(&bars[nfull], uint32_t(rem * W * sizeof(T)));
            for (int r = 0; r < rem; ++r)
                tma_load_2d(slab + size_t(nfull * kChunk + r) * W, &tmF1, int(k0),
                            row0 + nfull * kChunk + r, &bars[nfull]);
        }
    }

    // ---- thread -> (block j, segment sg, rhs lane)
    const int lane = tid % W, h = tid / W;
    const int j = h / S, sg = h % S;
    const int t = crank * G + j;
    const int s = t == 0 ? 0 : t * m - 1;
    const int e = t == P - 1 ? g.n : (t + 1) * m - 1;
    int a = s + sg * kSegLen;
    int b = sg == S - 1 ? e : a + kSegLen;
    if (a > e) a = e;
    if (b > e) b = e;

    // ---- forward sweep of the segment (from zero) + betas + Lam
    mbar_wait(cbar, 0);
    PSW_TRACE(1);
    double dd = 0.0, br = 0.0, bl = 0.0, lam = 0.0;
    if (a < b) {
        for (int c = (a - row0) / kChunk; c <= (b - 1 - row0) / kChunk; ++c) mbar_wait(&bars[c], 0);
        T d = T(0), sr = T(0), sl = T(0), sx = T(0);
        T* col = slab + lane;
#pragma unroll 4
        for (int q = a; q < b; ++q) {
            const FusedFwd<T> c = ff[q];
            const T f = col[(q - row0) * W];
            d = fma(c.ma, d, f * c.rp);
            sr = fma(f, c.gr, sr);
            sl = fma(f, c.gl, sl);
            sx = fma(c.lam, d, sx);
            col[(q - row0) * W] = d;
        }
        dd = double(d);
        br = double(sr);
        bl = double(sl);
        lam = double(sx);
    }
    PSW_TRACE(2);
    seg_d[tid] = dd;
    seg_lam[tid] = lam;
    seg_br[tid] = br;
    seg_bl[tid] = bl;
    __syncthreads();

    // ---- per (block, rhs): forward carries over the segments, block betas
    if (sg == 0) {
        double D = 0.0, R = 0.0, Lsum = 0.0;
        for (int k = 0; k < S; ++k) {
            const int id = (j * S + k) * W + lane;
            const double dend = seg_d[id];
            seg_d[id] = D;  // carry into segment k: D_{a-1}
            D = fma(segc[t * S + k].mu_end, D, dend);
            R += seg_br[id];
            Lsum += seg_bl[id];
        }
        own_r[j * W + lane] = R;
        own_l[j * W + lane] = Lsum;
    }
    PSW_TRACE(3);
    __syncthreads();
    PSW_TRACE(4);
    // ---- push this CTA's block betas into every CTA of the cluster (DSMEM)
    for (int idx = tid; idx < C * G * W; idx += blockDim.x) {
        const int dst = idx / (G * W), r = idx % (G * W);
        const int slot = (crank * G) * W + r;  // [block t][lane] in the tile
        double* rr = cluster.map_shared_rank(all_r, dst);
        double* rl = cluster.map_shared_rank(all_l, dst);
        rr[slot] = own_r[r];
        rl[slot] = own_l[r];
    }
    // one cluster barrier: every CTA holds every beta afterwards, and no CTA
    // touches another's shared memory again (CTAs may then exit freely)
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    PSW_TRACE(5);

    // ---- dichotomy combination as its tabulated linear map: the CTA's
    // boundary values v_j = sum_t MR[j][t] right_t + ML[j][t] left_t
    for (int idx = tid; idx < (jb1 - jb0) * W; idx += blockDim.x) {
        const int jb = idx / W, ln = idx % W;
        const double* Mr = cm + jb * 2 * P;
        const double* Ml = Mr + P;
        double sr = 0.0, sl = 0.0;
        for (int tt = 0; tt < P; ++tt) {
            sr = fma(Mr[tt], all_r[tt * W + ln], sr);
            sl = fma(Ml[tt], all_l[tt * W + ln], sl);
        }
        vals[(jb0 + jb) * W + ln] = sr + sl;
    }
    __syncthreads();

    PSW_TRACE(6);
    // ---- per (block, rhs): backward carries (x at each segment end)
    const double xl = t > 0 ? vals[(t - 1) * W + lane] : 0.0;
    if (sg == 0) {
        double xb = t < p ? vals[t * W + lane] : 0.0;  // x at row e
        for (int k = S - 1; k >= 0; --k) {
            const int id = (j * S + k) * W + lane;
            const SegCoef sc = segc[t * S + k];
            const double xa = fma(xl, sc.k2, fma(seg_d[id], sc.k1, seg_lam[id]));
            seg_br[id] = xb;  // x at the row after the segment
            xb = fma(sc.nu, xb, xa);
        }
    }
    __syncthreads();

    PSW_TRACE(7);
    // ---- backward sweep of the segment from its exact carry, streamed to X
    if (a < b) {
        const T D = T(seg_d[tid]);
        const T xlt = T(xl);
        T xn = T(seg_br[tid]);
        const T* col = slab + lane;
        const bool live = k0 + lane < g.N;
        T* xcol = X + k0 + lane;
#pragma unroll 4
        for (int q = b - 1; q >= a; --q) {
            const FusedBwd<T> c = fb[q];
            const T cq = fma(xlt, c.w, fma(c.mu, D, col[(q - row0) * W]));
            xn = fma(c.al, xn, cq);
            if (live) __stcs(xcol + int64_t(q) * g.ldx, xn);
        }
    }
    PSW_TRACE(8);
    if (trace && tid == 0) trace[blockIdx.x * 16 + 15] = gtimer();
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

struct Choice {
    int W = 0, G = 0, C = 0, rows_alloc = 0, nchunks = 0;
    size_t smem = 0;
};

// Row width of an RHS tile: 128 B (default) or 256 B (PSW_FUSED_ROW_BYTES).
int tile_row_bytes() {
    static int rb = [] {
        const char* e = std::getenv("PSW_FUSED_ROW_BYTES");
        return (e && std::atoi(e) == 256) ? 256 : 128;
    }();
    return rb;
}

// Smallest G (blocks per CTA) whose cluster C = P/G fits (<= 16 CTAs), then
// grow G while the CTA stays under the occupancy target.
Choice choose_w(const psw_plan* pl, int es, int row_bytes) {
    Choice ch;
    const int P = int(pl->P), m = int(pl->m), S = pl->nseg;
    const int W = row_bytes / es;
    if (S <= 0) return ch;
    for (int G = 1; G <= P; ++G) {
        if (P % G) continue;
        const int C = P / G;
        if (C > kMaxCluster) continue;
        const int rows_alloc = G * m + 1;
        const int nchunks = (rows_alloc + kChunk - 1) / kChunk;
        const size_t smem = FusedLayout(rows_alloc, nchunks, G, S, P, W, es).total;
        if (smem > kSmemMax || G * S * W > kMaxThreads) break;
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
    auto encode = encode_fn();
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

template <typename T, int W>
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
    g.N = N;
    g.ldx = ldx;
    auto kern = fused_r_kernel<T, W>;
    PSW_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ch.smem)));
    if (ch.C > 8) PSW_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int64_t tiles = (N + W - 1) / W;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(tiles * ch.C), 1, 1);
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
    if (ch.W * int(sizeof(T)) == 256)
        return launch_w<T, 256 / sizeof(T)>(pl, ch, F, ldf, X, ldx, N, s, ev, nev);
    return launch_w<T, 128 / sizeof(T)>(pl, ch, F, ldf, X, ldx, N, s, ev, nev);
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
    if (!pl->uniform || m < 1) return PSW_OK;
    const int S = int((m + kSegLen - 1) / kSegLen);
    pl->nseg = S;
    std::vector<FusedFwd<double>> ff(n);
    std::vector<FusedBwd<double>> fb(n);
    std::vector<SegCoef> seg(size_t(P) * S);
    for (int64_t t = 0; t < P; ++t) {
        const int64_t s = pl->blk[2 * t], e = pl->blk[2 * t + 1];
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
            seg[size_t(t) * S + sg] = {mu, k1, k2, lam};
        }
    }
    return pl->dtype == PSW_F64 ? upload_fused<double>(pl, ff, fb, seg)
                                : upload_fused<float>(pl, ff, fb, seg);
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
