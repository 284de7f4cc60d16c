// CHUNKED solve path: segment-parallel sweeps over RHS chunks whose forward
// intermediates stay in L2, two streams deep.
//
// The RHS are cut into chunks of Nc right-hand sides such that a chunk's
// forward intermediates (parked in X, ~24 MB) stay in L2. Per chunk, three
// kernels:
//   fwd   one thread per (RHS, segment): the segment's rows swept forward from
//         a zero carry (local_solve.hpp:39-48 in the affine form of
//         psw_internal.h), d~ -> X, segment partials d~_end, Lam and the two
//         beta dot products (betas.hpp:42-57) -> scratch. 32+1 rows per thread,
//         all loads in flight at once; the segment's coefficients are staged
//         once per CTA in shared memory.
//   comb  one thread per RHS: block betas (sums of the segment partials) and
//         the exact level-order dichotomy (boundary_solve.hpp:96-121) in
//         shared memory -> boundary values;
//   bwd   one thread per (RHS, segment): the segment's exact carries folded
//         from the block's partials, then x_q = d~_q + mu_q D + x_l w_q +
//         al_q x_{q+1}, X streamed out.
// Consecutive chunks alternate between two streams forked from (and joined
// back to) the caller's stream, so one chunk's carries and back substitution
// overlap the next chunk's forward sweep. HBM sees F once and X once; the d~
// round trip is served by L2. Parallelism is RHS x segments (C1: 768 x 128
// threads per kernel) instead of the STAGED path's RHS x blocks.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "psw_device.cuh"
#include "psw_internal.h"

namespace psw {
namespace {

constexpr int kSegMax = kSegLen + 1;
constexpr int kThreads = 128;
constexpr int kMaxFold = 64;  // segments per block

template <typename T>
__device__ __forceinline__ void stage_rows(const T* src, int count, T* dst) {
    for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
}

// ---- forward sweep of one segment per thread (layout R) -------------------
template <typename T>
__global__ void __launch_bounds__(kThreads) seg_fwd_kernel(
    const T* F, int64_t ldf, T* X, int64_t ldx, int64_t k0, int64_t Nc, int64_t N,
    const SegDesc* __restrict__ desc, const FusedFwd<T>* __restrict__ ff, double* __restrict__ part) {
    __shared__ FusedFwd<T> cs[kSegMax];
    const int s = blockIdx.y;
    const SegDesc sd = desc[s];
    const int len = sd.b - sd.a;
    const int64_t kl = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t k = k0 + kl;
    const bool kv = kl < Nc && k < N;
    // the rows first: their round trip overlaps the coefficient staging
    const T* fp = F + int64_t(sd.a) * ldf + k;
    T v[kSegMax];
#pragma unroll
    for (int r = 0; r < kSegMax; ++r) v[r] = (kv && r < len) ? __ldcs(fp + r * ldf) : T(0);
    stage_rows(ff + sd.a, len, cs);
    if (!kv) return;
    T d = T(0);
    double sR = 0.0, sL = 0.0, sX = 0.0;
#pragma unroll
    for (int r = 0; r < kSegMax; ++r) {
        if (r < len) {
            const FusedFwd<T> c = cs[r];
            d = fma(c.ma, d, v[r] * c.rp);
            sR = fma(double(v[r]), double(c.gr), sR);
            sL = fma(double(v[r]), double(c.gl), sL);
            sX = fma(double(c.lam), double(d), sX);
            v[r] = d;
        }
    }
    T* xp = X + int64_t(sd.a) * ldx + k;
#pragma unroll
    for (int r = 0; r < kSegMax; ++r)
        if (r < len) xp[r * ldx] = v[r];
    double* ps = part + int64_t(s) * 4 * Nc + kl;
    ps[0] = double(d);
    ps[Nc] = sX;
    ps[2 * Nc] = sR;
    ps[3 * Nc] = sL;
}

// ---- block betas and combination, one thread per RHS ----------------------
// The block betas are the sums of the segment partials; they and the values
// live in shared memory (P <= kMaxBlocks), so the exact level-order
// dichotomy never waits on global memory.
constexpr int kCarryRhs = 32;       // RHS per CTA (one warp runs the combination)
constexpr int kCarryThreads = 512;  // (block, RHS) pairs summing partials
constexpr int kMaxBlocks = 96;

__global__ void __launch_bounds__(kCarryThreads) seg_combine_kernel(
    const double* __restrict__ part, double* __restrict__ V, int64_t k0, int64_t Nc, int64_t N,
    int P, int p, const int32_t* __restrict__ segoff, const CombineItem* __restrict__ items,
    const double* __restrict__ zr, const double* __restrict__ zl) {
    extern __shared__ double sh[];  // [2][P][32] betas + [p][32] values
    const int lane = threadIdx.x % kCarryRhs;
    const int64_t kl = int64_t(blockIdx.x) * kCarryRhs + lane;
    const bool kv = kl < Nc && k0 + kl < N;
    double* sl = sh;
    double* sr = sl + P * kCarryRhs;
    double* sv = sr + P * kCarryRhs;
    // block betas: one thread per (block, RHS), all partial loads in flight
    for (int i = threadIdx.x; i < P * kCarryRhs; i += blockDim.x) {
        const int t = i / kCarryRhs;
        double R = 0.0, L = 0.0;
        if (kv) {
            const double* pp = part + kl;
#pragma unroll 8
            for (int s = segoff[t]; s < segoff[t + 1]; ++s) {
                R += pp[(int64_t(s) * 4 + 2) * Nc];
                L += pp[(int64_t(s) * 4 + 3) * Nc];
            }
        }
        sl[i] = L;
        sr[i] = R;
    }
    __syncthreads();
    if (threadIdx.x >= kCarryRhs || !kv || p == 0) return;
    combine_rhs(items, p, sl + lane, sr + lane, kCarryRhs, zr, zl, sv + lane, kCarryRhs);
    for (int j = 0; j < p; ++j) V[int64_t(j) * Nc + kl] = sv[j * kCarryRhs + lane];
}

// ---- back substitution of one segment per thread (layout R) ----------------
// The segment's exact carries are folded here from the block's segment
// partials (<= 2 S_t loads per thread, all independent): D_{a-1} through the
// forward affine maps of the earlier segments, x_b through the backward maps
// of the later ones from x_r (psw_internal.h).
template <typename T>
__global__ void __launch_bounds__(kThreads) seg_bwd_kernel(
    T* X, int64_t ldx, int64_t k0, int64_t Nc, int64_t N, int p,
    const SegDesc* __restrict__ desc, const int32_t* __restrict__ segoff,
    const SegCoef* __restrict__ segc, const FusedBwd<T>* __restrict__ fb,
    const double* __restrict__ part, const double* __restrict__ V) {
    __shared__ FusedBwd<T> cs[kSegMax];
    __shared__ SegCoef sc[kMaxFold];
    const int s = blockIdx.y;
    const SegDesc sd = desc[s];
    const int len = sd.b - sd.a, t = sd.t;
    const int s0 = segoff[t], s1 = segoff[t + 1];
    const int64_t kl = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t k = k0 + kl;
    const bool kv = kl < Nc && k < N;
    T* xp = X + int64_t(sd.a) * ldx + k;
    T v[kSegMax];
#pragma unroll
    for (int r = 0; r < kSegMax; ++r) v[r] = (kv && r < len) ? __ldcg(xp + r * ldx) : T(0);
    for (int i = threadIdx.x; i < s1 - s0; i += blockDim.x) sc[i] = segc[s0 + i];
    stage_rows(fb + sd.a, len, cs);
    if (!kv) return;
    const double* pp = part + kl;
    // carries of the segments from s on (forward fold over the whole block)
    double Dm = 0.0, Ds = 0.0;
    double dfold[kMaxFold];
    for (int i = 0; i < s1 - s0; ++i) {
        dfold[i] = Dm;
        if (s0 + i == s) Ds = Dm;
        Dm = fma(sc[i].mu_end, Dm, pp[int64_t(s0 + i) * 4 * Nc]);
    }
    const double xl = t > 0 ? V[int64_t(t - 1) * Nc + kl] : 0.0;
    double x = t < p ? V[int64_t(t) * Nc + kl] : 0.0;
    for (int i = s1 - s0 - 1; i > s - s0; --i) {
        const double lam = pp[(int64_t(s0 + i) * 4 + 1) * Nc];
        x = fma(sc[i].nu, x, fma(xl, sc[i].k2, fma(dfold[i], sc[i].k1, lam)));
    }
    const T D = T(Ds), xlt = T(xl);
    T xn = T(x);
#pragma unroll
    for (int r = kSegMax - 1; r >= 0; --r) {
        if (r < len) {
            const FusedBwd<T> cc = cs[r];
            xn = fma(cc.al, xn, fma(xlt, cc.w, fma(cc.mu, D, v[r])));
            v[r] = xn;
        }
    }
#pragma unroll
    for (int r = 0; r < kSegMax; ++r)
        if (r < len) __stcs(xp + r * ldx, v[r]);
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// two internal streams per device, created once (non-blocking)
cudaStream_t side_stream(int dev, int which) {
    static std::mutex mu;
    static std::vector<cudaStream_t> streams;
    std::lock_guard<std::mutex> lk(mu);
    const size_t idx = size_t(dev) * 2 + which;
    if (streams.size() <= idx) streams.resize(idx + 1, nullptr);
    if (!streams[idx]) cudaStreamCreateWithFlags(&streams[idx], cudaStreamNonBlocking);
    return streams[idx];
}

int64_t chunk_rhs(const psw_plan* pl, int64_t N, int es) {
    const double mb = std::max(1, env_int("PSW_CHUNK_MB", 24));
    int64_t nc = int64_t(mb * 1048576.0 / (double(pl->n) * es)) / kThreads * kThreads;
    nc = std::max<int64_t>(kThreads, nc);
    return std::min<int64_t>(nc, (N + kThreads - 1) / kThreads * kThreads);
}

template <typename T>
int launch_chunked(const psw_plan* pl, const void* Fv, int64_t ldf, void* Xv, int64_t ldx,
                   int64_t N, cudaStream_t s, void** ev, int nev) {
    const T* F = static_cast<const T*>(Fv);
    T* X = static_cast<T*>(Xv);
    const int64_t NS = pl->seg_off.back();
    const int P = int(pl->P), p = int(pl->p);
    const int64_t Nc = chunk_rhs(pl, N, int(sizeof(T)));
    const int64_t nchunks = (N + Nc - 1) / Nc;
    const int nstreams = nchunks > 1 ? 2 : 1;
    // scratch per stream slot: segment partials, boundary values
    const size_t per = sizeof(double) * size_t(Nc) * (size_t(NS) * 4 + size_t(std::max(p, 1)));
    void* scratch = nullptr;
    PSW_CUDA_TRY(cudaMallocAsync(&scratch, per * nstreams, s));
    int dev = 0;
    PSW_CUDA_TRY(cudaGetDevice(&dev));
    cudaStream_t st[2] = {s, s};
    cudaEvent_t evs[3] = {nullptr, nullptr, nullptr};
    int rc = PSW_OK;
    mark(ev, nev, 0, s);
    if (nstreams == 2) {
        st[0] = side_stream(dev, 0);
        st[1] = side_stream(dev, 1);
        for (auto& e : evs) PSW_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        PSW_CUDA_TRY(cudaEventRecord(evs[0], s));  // fork after the caller's prior work
        PSW_CUDA_TRY(cudaStreamWaitEvent(st[0], evs[0], 0));
        PSW_CUDA_TRY(cudaStreamWaitEvent(st[1], evs[0], 0));
    }
    const auto* ff = static_cast<const FusedFwd<T>*>(pl->d_ffwd);
    const auto* fb = static_cast<const FusedBwd<T>*>(pl->d_fbwd);
    int64_t launches = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int slot = int(c % nstreams);
        cudaStream_t cs = st[slot];
        double* base = reinterpret_cast<double*>(static_cast<char*>(scratch) + per * slot);
        double* part = base;
        double* V = part + size_t(NS) * 4 * Nc;
        const int64_t k0 = c * Nc;
        const dim3 grid(unsigned((Nc + kThreads - 1) / kThreads), unsigned(NS));
        seg_fwd_kernel<T><<<grid, kThreads, 0, cs>>>(F, ldf, X, ldx, k0, Nc, N, pl->d_segdesc,
                                                     ff, part);
        seg_combine_kernel<<<unsigned((Nc + kCarryRhs - 1) / kCarryRhs),
                             unsigned(std::min(kCarryThreads, P * kCarryRhs)),
                             sizeof(double) * kCarryRhs * (3 * P), cs>>>(
            part, V, k0, Nc, N, P, p, pl->d_segoff, pl->d_items, pl->d_zr, pl->d_zl);
        seg_bwd_kernel<T><<<grid, kThreads, 0, cs>>>(X, ldx, k0, Nc, N, p, pl->d_segdesc,
                                                     pl->d_segoff, pl->d_seg, fb, part, V);
        launches += 3;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "chunked kernels");
    if (nstreams == 2) {  // join both side streams back into the caller's stream
        cudaEventRecord(evs[1], st[0]);
        cudaEventRecord(evs[2], st[1]);
        cudaStreamWaitEvent(s, evs[1], 0);
        cudaStreamWaitEvent(s, evs[2], 0);
        for (auto& x : evs) cudaEventDestroy(x);
    }
    mark(ev, nev, 1, s);
    cudaFreeAsync(scratch, s);
    if (rc == PSW_OK) note_launches(launches);
    return rc;
}

}  // namespace

bool chunked_supported(const psw_plan* pl, int layout, int64_t N) {
    if (pl->world != 1 || layout != PSW_LAYOUT_R || N < 1) return false;
    if (!pl->d_segdesc || pl->seg_off.empty() || pl->P > kMaxBlocks) return false;
    for (size_t t = 0; t + 1 < pl->seg_off.size(); ++t)
        if (pl->seg_off[t + 1] - pl->seg_off[t] > kMaxFold) return false;
    return pl->seg_off.back() < 65536;  // grid.y
}

int solve_chunked(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx,
                  int64_t N, int layout, cudaStream_t s, void** ev, int nev) {
    (void)layout;
    return pl->dtype == PSW_F64 ? launch_chunked<double>(pl, F, ldf, X, ldx, N, s, ev, nev)
                                : launch_chunked<float>(pl, F, ldf, X, ldx, N, s, ev, nev);
}

}  // namespace psw
