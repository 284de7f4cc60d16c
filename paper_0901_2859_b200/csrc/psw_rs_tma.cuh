// RESWEEP K1/K3 on a TMA pipeline (layout R; included by psw_resweep.cu inside
// its anonymous namespace, after RsScratch / Work).
//
// The register-resident K1/K3 (rs_part_kernel / rs_solve_kernel) hold a
// segment's 33 rows in registers: 128 registers per thread, two CTAs per SM,
// and every CTA-wide barrier of the run fold leaves the SM with no loads in
// flight (ncu on C3: long-scoreboard + barrier stalls, 4.3 / 5.1 TB/s). Here
// the tiles live in shared memory instead:
//
//   one persistent CTA per SM = 8 consumer warps (warp = segment of the group,
//   lane = RHS) + 1 producer warp. The producer streams tiles
//   [group rows (<= 256)] x [W = 256 B of RHS] into a ring of S stages with
//   cp.async.bulk.tensor (32-row and 1-row boxes, one mbarrier per stage), and
//   per unit (group x a few RHS chunks) the group's descriptors and per-row
//   coefficients into one of two coefficient buffers (cp.async.bulk). K3's
//   tiles also carry the run carries and left boundary values of the chunk
//   (comb's output). Consumers never touch global memory on the way in; the
//   forward sweep writes d~ back into the stage, the back substitution reads
//   it and streams X out (st.global.cs, 256 B per warp and row).
//
// Work decomposition: unit u = (group u / nsets, RHS chunk set u % nsets); CTA
// b takes units b, b + grid, ... (K3: in reverse order, so its first re-reads
// of F are the rows K1 read last). A unit has >= S - 1 tiles, which is what
// lets two coefficient buffers serve S stages.

constexpr int kTmaWarps = kRsSeg;                 // consumer warps (segment each)
constexpr int kTmaThreads = (kTmaWarps + 1) * 32;  // + the producer warp
#ifndef PSW_F32_ROW_BYTES
#define PSW_F32_ROW_BYTES 256
#endif
// bytes of RHS per tile row: 32 fp64 RHS (one per lane); fp32 tiles take
// PSW_F32_ROW_BYTES (256: two RHS per lane, 128: one)
template <typename T>
__host__ __device__ constexpr int tma_rb() {
    return sizeof(T) == 8 ? 256 : PSW_F32_ROW_BYTES;
}
template <typename T>
__host__ __device__ constexpr int tma_w() {
    return tma_rb<T>() / int(sizeof(T));
}

struct TmaSched {
    int nchunks;  // ceil(N / W)
    int cs;       // chunks per unit (nominal; the last set of a group takes the rest)
    int nsets;    // units per group
    int nunits;
    int stages;
    int reverse;
    int mr;  // max runs per group (K3 aux slots per kind)
    int early;  // K3 store variant: release the previous stage after the forward sweep
    int xhint;  // K3 store variant: X stores with an evict-first L2 policy
};

struct TileIt {
    int u, g, c, c1, ord;
    bool first;
    // unit u = (group g, chunk set j); set j holds the chunks j, j + nsets,
    // ... so that the nsets CTAs working on a group at the same time touch
    // adjacent 256-byte pieces of every row
    __device__ __forceinline__ void unit(const TmaSched& s, int k) {
        const int v = blockIdx.x + k * int(gridDim.x);
        u = s.reverse ? s.nunits - 1 - v : v;
        g = u / s.nsets;
        c = u - g * s.nsets;
        c1 = s.nchunks;
        first = true;
    }
    __device__ __forceinline__ bool start(const TmaSched& s) {
        ord = 0;
        if (int(blockIdx.x) >= s.nunits) return false;
        unit(s, 0);
        return true;
    }
    __device__ __forceinline__ bool next(const TmaSched& s) {
        if ((c += s.nsets) < c1) {
            first = false;
            return true;
        }
        ++ord;
        if (int(blockIdx.x) + ord * int(gridDim.x) >= s.nunits) return false;
        unit(s, ord);
        return true;
    }
};

// group meta at the head of a coefficient buffer (all 16-byte multiples)
struct TmaMeta {
    RsGroup g;
    SegDesc desc[kRsSeg];
    SegCoef seg[kRsSeg];
    RsRun run[kRsSeg];
};
// bytes of group meta at the head of a coefficient buffer (K3 adds the
// closed-form carry weights of the group's slots)
constexpr int kMetaK1 = int(sizeof(TmaMeta));
constexpr int kMetaK3 = int(sizeof(TmaMeta) + kRsSeg * sizeof(CarryW));
static_assert(kMetaK1 % 16 == 0 && kMetaK3 % 16 == 0, "coefficient rows stay 16-byte aligned");

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumers_sync() {  // the 8 consumer warps only
    asm volatile("bar.sync 1, %0;" ::"n"(kTmaWarps * 32) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Producer: everything a tile needs, in the order the consumers take them.
// Coef = FusedFwd<T> (K1) or SolveCoef<T> (K3); AUX: K3's carries.
constexpr int kTmaMaxStages = 4;

// K3 carries of one tile: [D_in | x_B | x_l] x runs, W doubles each
template <typename T>
__device__ __forceinline__ void tma_aux(const RsGroup& G, int col, const TmaSched& sch,
                                        const RsScratch& sc, const double* __restrict__ V,
                                        int64_t ldv, unsigned char* stage, uint64_t* bar) {
    constexpr int W = tma_w<T>();
    double* aux = reinterpret_cast<double*>(stage + size_t(kTmaRows) * tma_rb<T>());
    for (int j = 0; j < G.r1 - G.r0; ++j) {
        const int64_t o = int64_t(G.r0 + j) * sc.ld + col;
        bulk_load(aux + (0 * sch.mr + j) * W, sc.dt + o, W * 8, bar);
        bulk_load(aux + (1 * sch.mr + j) * W, sc.br + o, W * 8, bar);
        const int t = G.t0 + j;
        if (t > 0) bulk_load(aux + (2 * sch.mr + j) * W, V + int64_t(t - 1) * ldv + col, W * 8, bar);
    }
}

template <typename T, typename Coef, bool AUX>
__device__ __forceinline__ void tma_produce(const CUtensorMap* m32, const CUtensorMap* m1,
                                            const TmaSched& sch, int32_t row0,
                                            const RsGroup* __restrict__ groups,
                                            const RsRun* __restrict__ runs,
                                            const SegDesc* __restrict__ desc,
                                            const SegCoef* __restrict__ segc,
                                            const Coef* __restrict__ coef,
                                            const CarryW* __restrict__ cw, const RsScratch& sc,
                                            const double* __restrict__ V, int64_t ldv,
                                            unsigned char* stage0, size_t stage_bytes,
                                            unsigned char* cbuf0, size_t cbuf_bytes,
                                            uint64_t* full, uint64_t* empty) {
    constexpr int W = tma_w<T>();
    constexpr int kMeta = AUX ? kMetaK3 : kMetaK1;
    const uint64_t pol = AUX && sch.reverse ? policy_evict_first() : policy_evict_normal();
    TileIt it;
    RsGroup G{};
    RsGroup pend_g[kTmaMaxStages];
    int pend_c[kTmaMaxStages];
    int i = 0;
    bool ok = it.start(sch);
    if (ok) G = groups[it.g];
    for (; ok; ++i) {
        const int st = i % sch.stages;
        if (i >= sch.stages) mbar_wait(&empty[st], uint32_t((i / sch.stages - 1) & 1));
        unsigned char* stage = stage0 + size_t(st) * stage_bytes;
        unsigned char* cb = cbuf0 + size_t(it.ord & 1) * cbuf_bytes;
        const int rows = G.rb - G.ra, ns = G.s1 - G.s0, nr = G.r1 - G.r0;
        const int nvl = nr - (G.t0 == 0 ? 1 : 0);  // K3: runs whose block has a left boundary value
        uint32_t bytes = uint32_t(rows) * tma_rb<T>();
        if (AUX) bytes += uint32_t(2 * nr + nvl) * W * 8;
        if (it.first)
            bytes += uint32_t(sizeof(RsGroup) + ns * (sizeof(SegDesc) + sizeof(SegCoef)) +
                              nr * sizeof(RsRun) + rows * sizeof(Coef) +
                              (AUX ? ns * sizeof(CarryW) : 0));
        mbar_expect_tx(&full[st], bytes);
        if (it.first) {  // the unit's group: meta + per-row coefficients
            TmaMeta* mt = reinterpret_cast<TmaMeta*>(cb);
            bulk_load(&mt->g, groups + it.g, sizeof(RsGroup), &full[st]);
            bulk_load(mt->desc, desc + G.s0, uint32_t(ns * sizeof(SegDesc)), &full[st]);
            bulk_load(mt->seg, segc + G.s0, uint32_t(ns * sizeof(SegCoef)), &full[st]);
            bulk_load(mt->run, runs + G.r0, uint32_t(nr * sizeof(RsRun)), &full[st]);
            if (AUX) bulk_load(cb + kMetaK1, cw + int64_t(it.g) * kRsSeg, uint32_t(ns * sizeof(CarryW)), &full[st]);
            bulk_load(cb + kMeta, coef + G.ra, uint32_t(rows * sizeof(Coef)), &full[st]);
        }
        const int col = it.c * W, r0 = G.ra - row0;
        const int n32 = rows >> 5;
        for (int j = 0; j < n32; ++j)
            tma_load_2d_hint(stage + size_t(j) * 32 * tma_rb<T>(), m32, col, r0 + 32 * j, &full[st], pol);
        for (int r = n32 * 32; r < rows; ++r)
            tma_load_2d_hint(stage + size_t(r) * tma_rb<T>(), m1, col, r0 + r, &full[st], pol);
        if (AUX) {
            // K3 is a programmatic dependent launch of the carry kernel: the
            // first S tiles' F rows go out before waiting for the carries
            if (i < kTmaMaxStages) {
                pend_g[i] = G;
                pend_c[i] = col;
            }
            const bool last = !TileIt(it).next(sch);
            if (i == sch.stages - 1 || (i < sch.stages && last)) {
                pdl_wait();
                for (int q = 0; q <= i; ++q)
                    tma_aux<T>(pend_g[q], pend_c[q], sch, sc, V, ldv,
                               stage0 + size_t(q) * stage_bytes, &full[q]);
            } else if (i >= sch.stages) {
                tma_aux<T>(G, col, sch, sc, V, ldv, stage, &full[st]);
            }
        }
        ok = it.next(sch);
        if (ok && it.first) G = groups[it.g];
    }
}

// ------------------------------------------------------------------ K1 (TMA)
template <typename T>
__global__ void __launch_bounds__(kTmaThreads, 1) rs_part_tma(
    const __grid_constant__ CUtensorMap m32, const __grid_constant__ CUtensorMap m1, int64_t N,
    int32_t row0, TmaSched sch, const RsGroup* __restrict__ groups, const RsRun* __restrict__ runs,
    const SegDesc* __restrict__ desc, const SegCoef* __restrict__ segc,
    const FusedFwd<T>* __restrict__ ff, RsScratch sc, uint32_t stage_bytes, uint32_t cbuf_bytes) {
    constexpr int W = tma_w<T>(), VPL = W / 32;
    extern __shared__ __align__(1024) unsigned char dyn[];
    unsigned char* stage0 = dyn;
    unsigned char* cbuf0 = dyn + size_t(sch.stages) * stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(cbuf0 + 2 * size_t(cbuf_bytes));
    uint64_t* empty = full + sch.stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    pdl_trigger();  // the fold kernel may be scheduled as K1's CTAs retire
    if (threadIdx.x == 0) {
        for (int s = 0; s < sch.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTmaWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kTmaWarps) {
        if (lane == 0)
            tma_produce<T, FusedFwd<T>, false>(&m32, &m1, sch, row0, groups, runs, desc, segc, ff,
                                               nullptr, sc, nullptr, 0, stage0, stage_bytes, cbuf0,
                                               cbuf_bytes, full, empty);
        return;
    }
    TileIt it;
    int i = 0;
    for (bool ok = it.start(sch); ok; ok = it.next(sch), ++i) {
        const int st = i % sch.stages;
        mbar_wait(&full[st], uint32_t((i / sch.stages) & 1));
        const T* tile = reinterpret_cast<const T*>(stage0 + size_t(st) * stage_bytes);
        const unsigned char* cb = cbuf0 + size_t(it.ord & 1) * cbuf_bytes;
        const TmaMeta* mt = reinterpret_cast<const TmaMeta*>(cb);
        const FusedFwd<T>* cf = reinterpret_cast<const FusedFwd<T>*>(cb + kMetaK1);
        const RsGroup G = mt->g;
        const bool sv = warp < G.s1 - G.s0;
        T d[VPL], lx[VPL];
        // segment beta partials in the solve precision (fp32: one FFMA per
        // product instead of two conversions and a DFMA; the 32-row partials
        // are summed in fp64 by the run fold), fp64 otherwise
        T br[VPL], bl[VPL];
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            d[v] = T(0);
            lx[v] = T(0);
            br[v] = T(0);
            bl[v] = T(0);
        }
        if (sv) {
            const SegDesc sd = mt->desc[warp];
            const int a = sd.a - G.ra, len = sd.b - sd.a;
            const FusedFwd<T>* c = cf + a;
            const T* f = tile + a * W + lane;
            auto sweep = [&](auto full_) {
                constexpr bool FULL = decltype(full_)::value;
#pragma unroll
                for (int r = 0; r < kSegMax; ++r) {
                    if (row_on<FULL>(r, len)) {
                        const FusedFwd<T> q = c[r];
#pragma unroll
                        for (int v = 0; v < VPL; ++v) {
                            const T fv = f[r * W + 32 * v];
                            d[v] = fma(q.ma, d[v], fv * q.rp);
                            br[v] = fma(fv, q.gr, br[v]);
                            bl[v] = fma(fv, q.gl, bl[v]);
                            lx[v] = fma(q.lam, d[v], lx[v]);
                        }
                    }
                }
            };
            if (len >= kSegLen - 1)
                sweep(std::true_type{});
            else
                sweep(std::false_type{});
        }
        // the segment's own (dead) first rows carry its exchange values:
        // doubles [0, W) d~ end, [W, 2W) Lam~, [2W, 3W) right, [3W, 4W) left
        if (sv) {
            __syncwarp();
            double* xw = reinterpret_cast<double*>(const_cast<T*>(tile) + (mt->desc[warp].a - G.ra) * W);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                xw[0 * W + lane + 32 * v] = double(d[v]);
                xw[1 * W + lane + 32 * v] = double(lx[v]);
                xw[2 * W + lane + 32 * v] = double(br[v]);
                xw[3 * W + lane + 32 * v] = double(bl[v]);
            }
        }
        consumers_sync();
        if (warp < G.r1 - G.r0) {  // one warp per run folds its segments (as rs_part_kernel)
            const RsRun rr = mt->run[warp];
            const int run = G.r0 + warp;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int64_t k = int64_t(it.c) * W + lane + 32 * v;
                double D = 0.0, lam = 0.0, nupre = 1.0, R = 0.0, L = 0.0;
                for (int s = rr.s0; s < rr.s1; ++s) {
                    const int j = s - G.s0;
                    const SegCoef q = mt->seg[j];
                    const double* xk = reinterpret_cast<const double*>(tile + (mt->desc[j].a - G.ra) * W);
                    const int l = lane + 32 * v;
                    lam = fma(nupre, fma(D, q.k1, xk[W + l]), lam);
                    D = fma(q.mu_end, D, xk[l]);
                    nupre *= q.nu;
                    R += xk[2 * W + l];
                    L += xk[3 * W + l];
                }
                if (k < N) {
                    const int64_t o = int64_t(run) * sc.ld + k;
                    sc.dt[o] = D;
                    sc.lam[o] = lam;
                    sc.br[o] = R;
                    sc.bl[o] = L;
                }
            }
        }
        // no second barrier: the exchange lives in this tile's stage, which
        // goes back only when every warp (the folding ones last) has arrived
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
}

// ------------------------------------------------------------------ K3 (TMA)
// Eight warps only (warp = segment, lane = RHS): with a ninth producer warp one
// SM sub-partition holds three warps and the register budget drops to 168,
// too few for d~ in registers. Thread 0 issues the loads instead, right
// after the tile's first barrier: by then every warp has taken its F rows
// and carries out of the stage (into registers) and released it. A unit's
// coefficient buffer is rewritten only for the unit after next, and units
// have >= S tiles, so it is free by then.
template <typename T>
struct K3Issuer {
    TileIt it;      // the next tile to issue
    RsGroup G;      // its unit's group
    bool ok;
    int n;          // tiles issued
};

template <typename T>
__device__ __forceinline__ void k3_issue(K3Issuer<T>& q, const TmaSched& sch,
                                         const CUtensorMap* m32, const CUtensorMap* m1,
                                         int32_t row0, const RsGroup* __restrict__ groups,
                                         const RsRun* __restrict__ runs,
                                         const SegDesc* __restrict__ desc,
                                         const SegCoef* __restrict__ segc,
                                         const SolveCoef<T>* __restrict__ coef,
                                         const CarryW* __restrict__ cw, const RsScratch& sc, const double* __restrict__ V,
                                         int64_t ldv, unsigned char* stage0, size_t stage_bytes,
                                         unsigned char* cbuf0, size_t cbuf_bytes, uint64_t* full,
                                         uint64_t pol) {
    constexpr int W = tma_w<T>();
    if (!q.ok) return;
    const int st = q.n % sch.stages;
    const RsGroup& G = q.G;
    unsigned char* stage = stage0 + size_t(st) * stage_bytes;
    const int rows = G.rb - G.ra, ns = G.s1 - G.s0, nr = G.r1 - G.r0;
    const int nvl = nr - (G.t0 == 0 ? 1 : 0);  // runs whose block has a left boundary value
    uint32_t bytes = uint32_t(rows) * tma_rb<T>() + uint32_t(2 * nr + nvl) * W * 8;
    if (q.it.first)
        bytes += uint32_t(sizeof(RsGroup) + ns * (sizeof(SegDesc) + sizeof(SegCoef) + sizeof(CarryW)) +
                          nr * sizeof(RsRun) + rows * sizeof(SolveCoef<T>));
    mbar_expect_tx(&full[st], bytes);
    if (q.it.first) {
        unsigned char* cb = cbuf0 + size_t(q.it.ord & 1) * cbuf_bytes;
        TmaMeta* mt = reinterpret_cast<TmaMeta*>(cb);
        bulk_load(&mt->g, groups + q.it.g, sizeof(RsGroup), &full[st]);
        bulk_load(mt->desc, desc + G.s0, uint32_t(ns * sizeof(SegDesc)), &full[st]);
        bulk_load(mt->seg, segc + G.s0, uint32_t(ns * sizeof(SegCoef)), &full[st]);
        bulk_load(mt->run, runs + G.r0, uint32_t(nr * sizeof(RsRun)), &full[st]);
        bulk_load(cb + kMetaK1, cw + int64_t(q.it.g) * kRsSeg, uint32_t(ns * sizeof(CarryW)), &full[st]);
        bulk_load(cb + kMetaK3, coef + G.ra, uint32_t(rows * sizeof(SolveCoef<T>)), &full[st]);
    }
    const int col = q.it.c * W, r0 = G.ra - row0, n32 = rows >> 5;
    for (int j = 0; j < n32; ++j)
        tma_load_2d_hint(stage + size_t(j) * 32 * tma_rb<T>(), m32, col, r0 + 32 * j, &full[st], pol);
    for (int r = n32 * 32; r < rows; ++r)
        tma_load_2d_hint(stage + size_t(r) * tma_rb<T>(), m1, col, r0 + r, &full[st], pol);
    double* aux = reinterpret_cast<double*>(stage + size_t(kTmaRows) * tma_rb<T>());
    for (int j = 0; j < nr; ++j) {  // [D_in | x_B | x_l] x runs, W doubles each
        const int64_t o = int64_t(G.r0 + j) * sc.ld + col;
        bulk_load(aux + (0 * sch.mr + j) * W, sc.dt + o, W * 8, &full[st]);
        bulk_load(aux + (1 * sch.mr + j) * W, sc.br + o, W * 8, &full[st]);
        const int t = G.t0 + j;
        if (t > 0) bulk_load(aux + (2 * sch.mr + j) * W, V + int64_t(t - 1) * ldv + col, W * 8, &full[st]);
    }
    ++q.n;
    q.ok = q.it.next(sch);
    if (q.ok && q.it.first) q.G = groups[q.it.g];  // used one issue later
}

template <typename T>
__global__ void __launch_bounds__(kTmaWarps * 32, 1) rs_solve_tma(
    const __grid_constant__ CUtensorMap m32, const __grid_constant__ CUtensorMap m1, T* X,
    int64_t ldx, int64_t N, int32_t row0, TmaSched sch, const RsGroup* __restrict__ groups,
    const RsRun* __restrict__ runs, const SegDesc* __restrict__ desc,
    const SegCoef* __restrict__ segc, const SolveCoef<T>* __restrict__ sco,
    const CarryW* __restrict__ cw, RsScratch sc, const double* __restrict__ V, int64_t ldv,
    uint32_t stage_bytes, uint32_t cbuf_bytes) {
    constexpr int W = tma_w<T>(), VPL = W / 32;
    extern __shared__ __align__(1024) unsigned char dyn[];
    unsigned char* stage0 = dyn;
    unsigned char* cbuf0 = dyn + size_t(sch.stages) * stage_bytes;
    double* xch = reinterpret_cast<double*>(cbuf0 + 2 * size_t(cbuf_bytes));  // [2][kRsSeg][W]
    uint64_t* full = reinterpret_cast<uint64_t*>(xch + 2 * kRsSeg * W);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    K3Issuer<T> iss;
    uint64_t pol = 0;
    // the issuing thread sits in the last warp: warp 0 folds the group's
    // first run between the two barriers, where the issue would delay it
    constexpr int kIssuer = (kTmaWarps - 1) * 32;
    if (threadIdx.x == kIssuer) {
        for (int s = 0; s < sch.stages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        pol = sch.reverse ? policy_evict_first() : policy_evict_normal();
        iss.n = 0;
        iss.ok = iss.it.start(sch);
        if (iss.ok) iss.G = groups[iss.it.g];
        for (int s = 0; s < sch.stages; ++s)
            k3_issue<T>(iss, sch, &m32, &m1, row0, groups, runs, desc, segc, sco, cw, sc, V, ldv,
                        stage0, stage_bytes, cbuf0, cbuf_bytes, full, pol);
    }
    __syncthreads();
    double(*s_d)[W] = reinterpret_cast<double(*)[W]>(xch);
    double(*s_l)[W] = s_d + kRsSeg;
    TileIt it;
    int i = 0;
    for (bool ok = it.start(sch); ok; ok = it.next(sch), ++i) {
        const int st = i % sch.stages;
        mbar_wait(&full[st], uint32_t((i / sch.stages) & 1));
        const T* tile = reinterpret_cast<const T*>(stage0 + size_t(st) * stage_bytes);
        const double* aux = reinterpret_cast<const double*>(stage0 + size_t(st) * stage_bytes +
                                                            size_t(kTmaRows) * tma_rb<T>());
        const unsigned char* cb = cbuf0 + size_t(it.ord & 1) * cbuf_bytes;
        const TmaMeta* mt = reinterpret_cast<const TmaMeta*>(cb);
        const SolveCoef<T>* cf = reinterpret_cast<const SolveCoef<T>*>(cb + kMetaK3);
        const CarryW* cws = reinterpret_cast<const CarryW*>(cb + kMetaK1);
        const RsGroup G = mt->g;
        const int ns = G.s1 - G.s0;
        const bool sv = warp < ns;
        SegDesc sd{0, 0, 0, 0};
        if (sv) sd = mt->desc[warp];
        const int a = sd.a - G.ra, len = sd.b - sd.a;
        const int jr = sv ? sd.t - G.t0 : 0;  // the segment's run within the group
        const bool hasl = sv && sd.t > 0;
        const SolveCoef<T>* c = cf + a;
        const T* f = tile + a * W + lane;
        // F rows and the run's carries out of the stage
        T v[kSegMax][VPL];
        double rD[VPL], rX[VPL], rL[VPL];
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
            const int l = lane + 32 * u;
            rD[u] = sv ? aux[(0 * sch.mr + jr) * W + l] : 0.0;
            rX[u] = sv ? aux[(1 * sch.mr + jr) * W + l] : 0.0;
            rL[u] = hasl ? aux[(2 * sch.mr + jr) * W + l] : 0.0;
        }
        const bool full_len = len >= kSegLen - 1;
        if (sv) {
            if (full_len) {
#pragma unroll
                for (int r = 0; r < kSegMax; ++r)
                    if (row_on<true>(r, len))
#pragma unroll
                        for (int u = 0; u < VPL; ++u) v[r][u] = f[r * W + 32 * u];
            } else {
#pragma unroll
                for (int r = 0; r < kSegMax; ++r)
                    if (row_on<false>(r, len))
#pragma unroll
                        for (int u = 0; u < VPL; ++u) v[r][u] = f[r * W + 32 * u];
            }
        }
        // forward from a zero carry, d~ in registers
        T d[VPL], lx[VPL];
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
            d[u] = T(0);
            lx[u] = T(0);
        }
        if (sv) {
            auto fwd = [&](auto full_) {
                constexpr bool FULL = decltype(full_)::value;
#pragma unroll
                for (int r = 0; r < kSegMax; ++r) {
                    if (row_on<FULL>(r, len)) {
                        const SolveCoef<T> q = c[r];
#pragma unroll
                        for (int u = 0; u < VPL; ++u) {
                            d[u] = fma(q.ma, d[u], v[r][u] * q.rp);
                            lx[u] = fma(q.lam, d[u], lx[u]);
                            v[r][u] = d[u];
                        }
                    }
                }
            };
            if (full_len)
                fwd(std::true_type{});
            else
                fwd(std::false_type{});
        }
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
            s_d[warp][lane + 32 * u] = double(d[u]);
            s_l[warp][lane + 32 * u] = double(lx[u]);
        }
        // stage reads done (generic proxy) before the next TMA write into it
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == kIssuer)  // stage st is free: the tile S ahead goes into it
            k3_issue<T>(iss, sch, &m32, &m1, row0, groups, runs, desc, segc, sco, cw, sc, V, ldv,
                        stage0, stage_bytes, cbuf0, cbuf_bytes, full, pol);
        // the segment's exact carries in closed form over its run (CarryW)
        T D[VPL], x[VPL], xl[VPL];
        if (sv) {
            const CarryW& q = cws[warp];
#pragma unroll
            for (int u = 0; u < VPL; ++u) {
                const int l = lane + 32 * u;
                double dc = q.P * rD[u];
                double xc = fma(q.Q, rX[u], fma(q.K2, rL[u], q.K1 * rD[u]));
#pragma unroll
                for (int i = 0; i < kRsSeg; ++i)
                    if (i < ns) {
                        const double dd = s_d[i][l];
                        dc = fma(q.A[i], dd, dc);
                        xc = fma(q.C[i], dd, fma(q.B[i], s_l[i][l], xc));
                    }
                D[u] = T(dc);
                x[u] = T(xc);
                xl[u] = T(rL[u]);
            }
        }
        __syncthreads();  // the exchange arrays are rewritten by the next tile
        if (sv) {
            bool kv[VPL];
#pragma unroll
            for (int u = 0; u < VPL; ++u) kv[u] = int64_t(it.c) * W + lane + 32 * u < N;
            T* xp = X + int64_t(sd.a - row0) * ldx + int64_t(it.c) * W + lane;
            auto bwd = [&](auto full_) {
                constexpr bool FULL = decltype(full_)::value;
#pragma unroll
                for (int r = kSegMax - 1; r >= 0; --r) {
                    if (row_on<FULL>(r, len)) {
                        const SolveCoef<T> q = c[r];
#pragma unroll
                        for (int u = 0; u < VPL; ++u) {
                            const T dq = fma(q.mu, D[u], v[r][u]);
                            x[u] = fma(q.al, x[u], fma(xl[u], q.w, dq));
                            if (kv[u]) __stcs(xp + int64_t(r) * ldx + 32 * u, x[u]);
                        }
                    }
                }
            };
            if (full_len)
                bwd(std::true_type{});
            else
                bwd(std::false_type{});
        }
    }
}

// ------------------------------------------------------------------ K3 (TMA in, TMA out)
// 8 consumer warps + a producer warp (168 registers: d~ stays in registers,
// the loops read shared memory through non-volatile asm loads the compiler
// may hoist over the x stores). X goes back through the stage: the back
// substitution writes x in place of F, one thread stores the tile with
// cp.async.bulk.tensor and releases the stage once the store has read it.
__device__ __forceinline__ double lds_f64(const double* p) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ float lds_f32(const float* p) {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
    return v;
}
template <typename T>
__device__ __forceinline__ T lds(const T* p) {
    if constexpr (sizeof(T) == 8)
        return lds_f64(reinterpret_cast<const double*>(p));
    else
        return lds_f32(reinterpret_cast<const float*>(p));
}
template <typename T>
__device__ __forceinline__ SolveCoef<T> lds_coef(const SolveCoef<T>* p) {
    SolveCoef<T> q;
    q.rp = lds(&p->rp);
    q.ma = lds(&p->ma);
    q.lam = lds(&p->lam);
    q.mu = lds(&p->mu);
    q.w = lds(&p->w);
    q.al = lds(&p->al);
    return q;
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, int c0, int c1,
                                                  const void* src, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(c0), "r"(c1), "r"(smem_u32(src)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <typename T>
__global__ void __launch_bounds__(kTmaThreads, 1) rs_solve_tma_st(
    const __grid_constant__ CUtensorMap m32, const __grid_constant__ CUtensorMap m1,
    const __grid_constant__ CUtensorMap x32, const __grid_constant__ CUtensorMap x1, int64_t N,
    int32_t row0, TmaSched sch, const RsGroup* __restrict__ groups, const RsRun* __restrict__ runs,
    const SegDesc* __restrict__ desc, const SegCoef* __restrict__ segc,
    const SolveCoef<T>* __restrict__ sco, const CarryW* __restrict__ cw, RsScratch sc,
    const double* __restrict__ V, int64_t ldv, uint32_t stage_bytes, uint32_t cbuf_bytes) {
    constexpr int W = tma_w<T>(), VPL = W / 32;
    extern __shared__ __align__(1024) unsigned char dyn[];
    unsigned char* stage0 = dyn;
    unsigned char* cbuf0 = dyn + size_t(sch.stages) * stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(cbuf0 + 2 * size_t(cbuf_bytes));
    uint64_t* empty = full + sch.stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < sch.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTmaWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kTmaWarps) {
        if (lane == 0)
            tma_produce<T, SolveCoef<T>, true>(&m32, &m1, sch, row0, groups, runs, desc, segc, sco,
                                               cw, sc, V, ldv, stage0, stage_bytes, cbuf0,
                                               cbuf_bytes, full, empty);
        return;
    }
    TileIt it;
    int i = 0, prev_st = -1;
    const bool early = sch.early != 0;
    for (bool ok = it.start(sch); ok; ok = it.next(sch), ++i) {
        const int st = i % sch.stages;
        mbar_wait(&full[st], uint32_t((i / sch.stages) & 1));
        T* tile = reinterpret_cast<T*>(stage0 + size_t(st) * stage_bytes);
        const double* aux = reinterpret_cast<const double*>(stage0 + size_t(st) * stage_bytes +
                                                            size_t(kTmaRows) * tma_rb<T>());
        const unsigned char* cb = cbuf0 + size_t(it.ord & 1) * cbuf_bytes;
        const TmaMeta* mt = reinterpret_cast<const TmaMeta*>(cb);
        const SolveCoef<T>* cf = reinterpret_cast<const SolveCoef<T>*>(cb + kMetaK3);
        const CarryW* cws = reinterpret_cast<const CarryW*>(cb + kMetaK1);
        const RsGroup G = mt->g;
        const int ns = G.s1 - G.s0;
        const bool sv = warp < ns;
        SegDesc sd{0, 0, 0, 0};
        if (sv) sd = mt->desc[warp];
        const int a = sd.a - G.ra, len = sd.b - sd.a;
        const int jr = sv ? sd.t - G.t0 : 0;
        const bool hasl = sv && sd.t > 0;
        const SolveCoef<T>* c = cf + a;
        T* f = tile + a * W + lane;
        const bool full_len = len >= kSegLen - 1;
        // forward from a zero carry, d~ in registers
        T v[kSegMax][VPL];
        T d[VPL], lx[VPL];
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
            d[u] = T(0);
            lx[u] = T(0);
        }
        if (sv) {
            auto fwd = [&](auto full_) {
                constexpr bool FULL = decltype(full_)::value;
#pragma unroll
                for (int r = 0; r < kSegMax; ++r) {
                    if (row_on<FULL>(r, len)) {
                        const T rp = lds(&c[r].rp), ma = lds(&c[r].ma), lam = lds(&c[r].lam);
#pragma unroll
                        for (int u = 0; u < VPL; ++u) {
                            d[u] = fma(ma, d[u], lds(f + r * W + 32 * u) * rp);
                            lx[u] = fma(lam, d[u], lx[u]);
                            v[r][u] = d[u];
                        }
                    }
                }
            };
            if (full_len)
                fwd(std::true_type{});
            else
                fwd(std::false_type{});
            // the segment's own (now dead) first rows carry its exchange
            // values: doubles [0, W) = d~ end, [W, 2W) = Lam~ (as doubles)
            __syncwarp();
            double* xw = reinterpret_cast<double*>(tile + a * W);
#pragma unroll
            for (int u = 0; u < VPL; ++u) {
                xw[lane + 32 * u] = double(d[u]);
                xw[W + lane + 32 * u] = double(lx[u]);
            }
        }
        // the previous tile's store has had a forward sweep's time to read
        // its stage: release this warp's share now rather than at the end
        if (lane == 0 && prev_st >= 0 && early) {
            bulk_wait_read<0>();
            mbar_arrive(&empty[prev_st]);
        }
        if (early) prev_st = -1;
        consumers_sync();
        T D[VPL], x[VPL], xl[VPL];
        if (sv) {
            // the segment's exact carries in closed form over its run (CarryW)
            const CarryW& q = cws[warp];
#pragma unroll
            for (int u = 0; u < VPL; ++u) {
                const int l = lane + 32 * u;
                const double rD = aux[(0 * sch.mr + jr) * W + l], rX = aux[(1 * sch.mr + jr) * W + l];
                const double rL = hasl ? aux[(2 * sch.mr + jr) * W + l] : 0.0;
                double dc = q.P * rD;
                double xc = fma(q.Q, rX, fma(q.K2, rL, q.K1 * rD));
#pragma unroll
                for (int k = 0; k < kRsSeg; ++k)
                    if (k < ns) {
                        const double* xk =
                            reinterpret_cast<const double*>(tile + (mt->desc[k].a - G.ra) * W);
                        const double dd = xk[l];
                        dc = fma(q.A[k], dd, dc);
                        xc = fma(q.C[k], dd, fma(q.B[k], xk[W + l], xc));
                    }
                D[u] = T(dc);
                x[u] = T(xc);
                xl[u] = T(rL);
            }
        }
        consumers_sync();  // every warp has its carries: the exchange rows may be overwritten
        if (sv) {
            auto bwd = [&](auto full_) {
                constexpr bool FULL = decltype(full_)::value;
#pragma unroll
                for (int r = kSegMax - 1; r >= 0; --r) {
                    if (row_on<FULL>(r, len)) {
                        const T mu = lds(&c[r].mu), w = lds(&c[r].w), al = lds(&c[r].al);
#pragma unroll
                        for (int u = 0; u < VPL; ++u) {
                            const T dq = fma(mu, D[u], v[r][u]);
                            x[u] = fma(al, x[u], fma(xl[u], w, dq));
                            f[r * W + 32 * u] = x[u];
                        }
                    }
                }
            };
            if (full_len)
                bwd(std::true_type{});
            else
                bwd(std::false_type{});
        }
        // each warp stores its own rows as soon as they are written
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            if (sv) {
                const int col = it.c * W, r0 = sd.a - row0, n32 = len >> 5;
                const T* src = tile + a * W;
                if (sch.xhint) {  // X is not read again here: first to go from L2
                    const uint64_t pol = policy_evict_first();
                    for (int j = 0; j < n32; ++j)
                        tma_store_2d_hint(&x32, col, r0 + 32 * j, src + size_t(j) * 32 * W, pol);
                    for (int r = n32 * 32; r < len; ++r)
                        tma_store_2d_hint(&x1, col, r0 + r, src + size_t(r) * W, pol);
                } else {
                    for (int j = 0; j < n32; ++j) tma_store_2d(&x32, col, r0 + 32 * j, src + size_t(j) * 32 * W);
                    for (int r = n32 * 32; r < len; ++r) tma_store_2d(&x1, col, r0 + r, src + size_t(r) * W);
                }
            }
            bulk_commit();
            // this warp's previous store has read its stage
            if (prev_st >= 0) {
                bulk_wait_read<1>();
                mbar_arrive(&empty[prev_st]);
            }
        }
        prev_st = st;
    }
    if (lane == 0) bulk_wait_all();
}

// ------------------------------------------------------------------ host side
template <typename T>
bool tma_encode(const void* F, int64_t ldf, int64_t N, int64_t rows, CUtensorMap* m32,
                CUtensorMap* m1) {
    const auto enc = tensor_map_encoder();
    constexpr int es = int(sizeof(T)), W = tma_w<T>();
    if (!enc || (reinterpret_cast<uintptr_t>(F) & 15) || (ldf * es) % 16 || N < W || rows < 1 ||
        ldf < N)
        return false;
    cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(ldf) * es};
    cuuint32_t box32[2] = {cuuint32_t(W), 32}, box1[2] = {cuuint32_t(W), 1}, one[2] = {1, 1};
    const CUtensorMapDataType dt =
        es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    for (int k = 0; k < 2; ++k)
        if (enc(k ? m1 : m32, dt, 2, const_cast<void*>(F), dims, strides, k ? box1 : box32, one,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    return true;
}

inline int tma_env(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

inline bool tma_enabled() { return tma_env("PSW_RS_TMA", 1) != 0; }

// shared memory of one launch; 0 when it does not fit one SM
inline size_t tma_smem(int stages, size_t stage_bytes, size_t cbuf_bytes, size_t xch_bytes) {
    return size_t(stages) * stage_bytes + 2 * cbuf_bytes + xch_bytes + 16 * size_t(stages) + 16;
}

template <typename T, typename Coef, bool AUX>
bool tma_plan(const psw_plan* pl, int64_t N, TmaSched& sch, size_t& stage_bytes,
              size_t& cbuf_bytes, size_t& smem, bool store = false) {
    constexpr int W = tma_w<T>();
    int dev = pl->device, nsm = 0, maxs = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    sch.mr = std::max(1, pl->rs_maxruns);
    sch.nchunks = int((N + W - 1) / W);
    stage_bytes = size_t(kTmaRows) * tma_rb<T>() + (AUX ? size_t(3) * sch.mr * W * 8 : 0);
    cbuf_bytes = size_t(AUX ? kMetaK3 : kMetaK1) + size_t(kTmaRows) * sizeof(Coef);
    const size_t xch = (store || !AUX) ? 0 : size_t(2) * kRsSeg * W * 8;
    sch.stages = std::min(tma_env("PSW_TMA_STAGES", 3), kTmaMaxStages);
    while (sch.stages > 2 && tma_smem(sch.stages, stage_bytes, cbuf_bytes, xch) > size_t(maxs))
        --sch.stages;
    smem = tma_smem(sch.stages, stage_bytes, cbuf_bytes, xch);
    if (smem > size_t(maxs) || nsm < 1) return false;
    // units of >= stages - 1 tiles (two coefficient buffers serve the ring)
    // K1: units of >= S - 1 tiles (its stages return after the unit's meta
    // reads); K3: >= S tiles (its stages return mid-tile)
    // Coefficient buffer k & 1 is rewritten for unit k + 2 once the stage of
    // the tile S back is released; unit k + 1 must be long enough for unit k
    // to be finished by then. K1 releases at its tile's end: units >= S - 1
    // tiles; K3 (registers) releases after the forward sweep: >= S tiles;
    // K3 (TMA store) releases one tile late, after the store read the
    // stage: >= S - 2 tiles, any unit for S <= 3 (and S >= 2, or the ring
    // would wait on itself).
    const int need = store ? std::max(1, sch.stages - 2) : (AUX ? sch.stages : sch.stages - 1);
    int cs = std::max(tma_env("PSW_TMA_CS", 4), need);
    if (sch.nchunks < need) sch.stages = AUX ? std::max(1, sch.nchunks) : 2;
    if (store && sch.stages < 2) return false;
    if (sch.nchunks <= cs) {
        cs = sch.nchunks;
        sch.nsets = 1;
    } else {
        sch.nsets = sch.nchunks / cs;  // sets of >= cs chunks
    }
    sch.cs = cs;
    sch.nunits = pl->rs_ngroups * sch.nsets;
    sch.reverse = AUX ? tma_env("PSW_TMA_REV", 1) : 0;
    sch.early = tma_env("PSW_K3_EARLY", 0);
    sch.xhint = tma_env("PSW_K3_XHINT", 0);  // measured: no difference  // measured: C3 K3 2.85 -> 3.02 ms with it
    (void)nsm;
    return true;
}

inline unsigned tma_grid(const psw_plan* pl, const TmaSched& sch) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pl->device);
    return unsigned(std::min(sch.nunits, std::max(nsm, 1)));
}

template <typename KernT>
cudaError_t tma_smem_attr(KernT kern, size_t smem) {
    // per kernel (several kernels share one signature)
    static std::mutex mu;
    static std::vector<std::pair<const void*, size_t>> set;
    std::lock_guard<std::mutex> lk(mu);
    const void* key = reinterpret_cast<const void*>(kern);
    for (auto& e : set)
        if (e.first == key) {
            if (smem <= e.second) return cudaSuccess;
            const cudaError_t r =
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            if (r == cudaSuccess) e.second = smem;
            return r;
        }
    const cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (r == cudaSuccess) set.push_back({key, smem});
    return r;
}

// K1 through the TMA pipeline; returns false (nothing launched) when the
// shape does not qualify
template <typename T>
bool launch_part_tma(const psw_plan* pl, const T* F, int64_t ldf, int64_t N, const RsScratch& sc,
                     cudaStream_t s, int& rc) {
    rc = PSW_OK;
    // each segment lends its first W / 8 rows (4 W doubles) to the exchange
    // each segment lends 4 W doubles of its first rows to the exchange
    if (!tma_enabled() || pl->rs_minseg < 32 * tma_w<T>() / tma_rb<T>()) return false;
    CUtensorMap m32, m1;
    if (!tma_encode<T>(F, ldf, N, pl->row1 - pl->row0, &m32, &m1)) return false;
    TmaSched sch;
    size_t sb, cb, smem;
    if (!tma_plan<T, FusedFwd<T>, false>(pl, N, sch, sb, cb, smem)) return false;
    auto kern = rs_part_tma<T>;
    if (cudaError_t e = tma_smem_attr(kern, smem)) {
        rc = cuda_fail(e, "rs_part_tma attribute");
        return true;
    }
    kern<<<tma_grid(pl, sch), kTmaThreads, smem, s>>>(
        m32, m1, N, int32_t(pl->row0), sch, pl->d_rs_group, pl->d_rs_run, pl->d_segdesc, pl->d_seg,
        static_cast<const FusedFwd<T>*>(pl->d_ffwd), sc, uint32_t(sb), uint32_t(cb));
    return true;
}

template <typename T>
bool launch_solve_tma(const psw_plan* pl, const T* F, int64_t ldf, T* X, int64_t ldx, int64_t N,
                      const RsScratch& sc, const double* V, int64_t ldv, cudaStream_t s, int& rc) {
    constexpr int W = tma_w<T>();
    rc = PSW_OK;
    if (!tma_enabled() || (ldv & 1) || ldv < (N + W - 1) / W * W) return false;
    CUtensorMap m32, m1;
    if (!tma_encode<T>(F, ldf, N, pl->row1 - pl->row0, &m32, &m1)) return false;
    // the store variant lends each segment's first rows to the exchange
    // (2 W doubles of its first rows)
    if (tma_env("PSW_K3_STORE", 1) && pl->rs_minseg >= 16 * W / tma_rb<T>()) {
        CUtensorMap x32, x1;
        if (tma_encode<T>(X, ldx, N, pl->row1 - pl->row0, &x32, &x1)) {
            TmaSched sch;
            size_t sb, cb, smem;
            if (!tma_plan<T, SolveCoef<T>, true>(pl, N, sch, sb, cb, smem, true)) return false;
            auto kern = rs_solve_tma_st<T>;
            if (cudaError_t e = tma_smem_attr(kern, smem)) {
                rc = cuda_fail(e, "rs_solve_tma_st attribute");
                return true;
            }
            if (cudaError_t e = launch_pdl(kern, dim3(tma_grid(pl, sch)), dim3(kTmaThreads), smem, s,
                                           m32, m1, x32, x1, N, int32_t(pl->row0), sch,
                                           pl->d_rs_group, pl->d_rs_run, pl->d_segdesc, pl->d_seg,
                                           static_cast<const SolveCoef<T>*>(pl->d_scoef),
                                           pl->d_rs_cw, sc, V, ldv, uint32_t(sb), uint32_t(cb)))
                rc = cuda_fail(e, "rs_solve_tma_st launch");
            return true;
        }
    }
    TmaSched sch;
    size_t sb, cb, smem;
    if (!tma_plan<T, SolveCoef<T>, true>(pl, N, sch, sb, cb, smem)) return false;
    auto kern = rs_solve_tma<T>;
    if (cudaError_t e = tma_smem_attr(kern, smem)) {
        rc = cuda_fail(e, "rs_solve_tma attribute");
        return true;
    }
    kern<<<tma_grid(pl, sch), kTmaWarps * 32, smem, s>>>(
        m32, m1, X, ldx, N, int32_t(pl->row0), sch, pl->d_rs_group, pl->d_rs_run, pl->d_segdesc,
        pl->d_seg, static_cast<const SolveCoef<T>*>(pl->d_scoef), pl->d_rs_cw, sc, V, ldv,
        uint32_t(sb), uint32_t(cb));
    return true;
}
