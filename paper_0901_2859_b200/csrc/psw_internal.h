// Internal declarations shared by the host setup (psw_plan.cpp) and the CUDA
// solve paths (psw_staged.cu, psw_fused.cu). Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "parsweep_b200.h"

namespace psw {

// ---- error plumbing (thread-local last error, psw_last_error_*) ----------
void set_error(int code, const std::string& msg, int64_t index = -1);
int clear_error();
int cuda_fail(cudaError_t e, const char* what);
void note_launches(int64_t k);   // accumulate per-call kernel launch count
void reset_launches();

#define PSW_CUDA_TRY(expr)                                   \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return ::psw::cuda_fail(_e, #expr); \
    } while (0)

// ---- per-row local sweep coefficients ------------------------------------
// Block t (0-based) owns rows [s_t, e_t) (0-based) = the reference half-open
// block [n_t, n_{t+1}) (partition.hpp:26-29). Its closed sweep block ends at
// h_t = e_t (t < p, the next boundary row) or n-1 (t = p)
// (local_solve.hpp:29-31). With the unit first row (t > 0) carrying the
// unknown boundary value x_l, the sweep of local_solve.hpp:39-48 /
// thomas.hpp:31-44 is affine in x_l:
//   forward   d_q = f_q * rp_q + ma_q * d_{q-1}          (d at the unit row = 0)
//   betas     bR += f_q * gR_q,  bL += f_q * gL_q         (betas.hpp:42-57)
//   backward  x_q = d_q + x_l * w_q + al_q * x_{q+1}       (x_{h_t} = x_r given)
// rp = 1/pivot, ma = -a_q/pivot, al = -c_q/pivot, w_q = ma_q w_{q-1}, w = 1 at
// the unit row; gR = row r_t of inv(A), gL = row r_{t-1} of inv(A) on block t.
template <typename T>
struct alignas(4 * sizeof(T)) FwdCoef {
    T rp, ma, gr, gl;
};
template <typename T>
struct alignas(16) BwdCoef {  // 16 B rows (TMA bulk-copy granule) for both dtypes
    T w, al;
};

// One dichotomy item in level order (boundary_solve.hpp:104-119): the
// boundary index i and its nearest already-known neighbours kl < i < kr
// (sentinels -1 and p).
struct CombineItem {
    int32_t i, kl, kr, pad;
};

// FUSED path: every block is cut into S segments of kSegLen rows that are
// swept by different threads. Within a segment [a, b) the forward recurrence
// is run from zero (d~) and the true value is d_q = d~_q + mu_q D_{a-1},
// mu_q = prod_{u=a..q} ma_u; the backward x_q = c_q + al_q x_{q+1},
// c_q = d_q + x_l w_q, is started from the exact carry x_b obtained by a scan
// over segment aggregates: x_a = sum_q lam_q c_q + nu x_b with
// lam_q = prod_{u=a..q-1} al_u, nu = prod_{u=a..b-1} al_u, and
// sum_q lam_q c_q = Lam + D_{a-1} K1 + x_l K2 (Lam = sum lam_q d~_q is
// accumulated by the forward sweep, K1 = sum lam mu, K2 = sum lam w).
#ifndef PSW_SEGLEN
#define PSW_SEGLEN 32
#endif
constexpr int kSegLen = PSW_SEGLEN;  // rows per segment (the last one of a block: + 1)
constexpr int kCoefPad = 64;  // zero rows appended to FwdCoef/BwdCoef tables
template <typename T>
struct alignas(16) FusedFwd {
    T rp, ma, gr, gl, lam, pad;
};
template <typename T>
struct alignas(16) FusedBwd {
    T mu, w, al, pad;
};
struct alignas(32) SegCoef {
    double mu_end, k1, k2, nu;
};
struct SegDesc {  // rows [a, b) of block t
    int32_t a, b, t, pad;
};

// RESWEEP (psw_resweep.cu): the segments of the plan's own blocks are taken
// kRsSeg at a time by one CTA ("group"); a run is the part of a group inside
// one block. Per run the K1 kernel leaves four aggregates per RHS, folded over
// the run's segments; the matrix-only aggregate of a run is a SegCoef
// (mu_end = prod mu_end, k1, k2, nu of the composed affine map).
#ifndef PSW_RSSEG
#define PSW_RSSEG 8
#endif
constexpr int kRsSeg = PSW_RSSEG;  // segments per group (one warp each)
struct RsGroup {
    int32_t s0, s1;  // segments [s0, s1)
    int32_t r0, r1;  // runs [r0, r1)
    int32_t ra, rb;  // rows [ra, rb) (global, 0-based)
    int32_t t0;      // global block of the first run (run j is block t0 + j)
    int32_t pad1;
};
struct RsRun {
    int32_t s0, s1;  // segments [s0, s1) of block t
    int32_t t, tl;   // global block, block index local to the plan's range
};
// RESWEEP K3 (TMA): the exact carries of segment slot w of a group in closed
// form over its run (the serial run fold unrolled): with dd_i / lam_i the
// zero-carry segment end values and Lam~ of the run's slots,
//   D_w = P D_in + sum_i A[i] dd_i
//   x_w = Q x_B + K2 x_l + K1 D_in + sum_j B[j] lam_j + sum_i C[i] dd_i
// (weights are zero outside w's run; psw_resweep.cu build_rs_tables)
struct CarryW {
    double P, Q, K1, K2;
    double A[8], B[8], C[8];
};
// per-row coefficients of the RESWEEP solve kernel (K3)
template <typename T>
struct alignas(16) SolveCoef {
    T rp, ma, lam, mu, w, al;
};

}  // namespace psw

// The plan: immutable after psw_plan_create.
struct psw_plan {
    int64_t n = 0, p = 0, P = 1;
    int dtype = PSW_F64;
    int device = 0;
    bool uniform = false;
    int64_t m = 0;  // rows per range when uniform (n / P)
    std::vector<int64_t> bnd;          // 1-based boundaries (reference Partition)
    std::vector<int32_t> blk;          // [2t] = s_t, [2t+1] = e_t (0-based, owned rows)
    std::vector<psw::CombineItem> items;
    psw_plan_info_t info{};

    // device-resident preliminary
    void* d_fwd = nullptr;   // FwdCoef<T>[n]
    void* d_bwd = nullptr;   // BwdCoef<T>[n]
    int32_t* d_blk = nullptr;
    double* d_zr = nullptr;  // p x p samples ZR[j][i] (preliminary.hpp:69)
    double* d_zl = nullptr;  // p x p samples ZL[j][i] (preliminary.hpp:71)
    psw::CombineItem* d_items = nullptr;
    std::vector<int32_t> lvl_off;      // item offsets of every dichotomy level (+ end)
    int32_t* d_lvl_off = nullptr;

    // FUSED path tables (uniform partitions only)
    int nseg = 0;                      // segments per block
    double* d_cmat = nullptr;          // [p][2P] combination matrix (see build_fused_tables)
    void* d_ffwd = nullptr;            // FusedFwd<T>[n]
    void* d_fbwd = nullptr;            // FusedBwd<T>[n]
    psw::SegCoef* d_seg = nullptr;     // per segment (block-major, see seg_off)
    psw::SegDesc* d_segdesc = nullptr; // per segment rows / block
    int32_t* d_segoff = nullptr;       // [P+1] first segment of every block
    // CLUSTER path: per-cluster-rank coefficient tables in the kernel's shared
    // memory layout, one per layout, built with the plan (psw_cluster.cu)
    void* d_ctab[2] = {nullptr, nullptr};
    int64_t ctab_stride[2] = {0, 0};
    std::vector<int32_t> seg_off;      // host copy

    // RESWEEP tables over the plan's own segments (psw_resweep.cu)
    int rs_ngroups = 0, rs_nruns = 0, rs_maxruns = 0;  // maxruns: most runs in one group
    int rs_minseg = 0;                                  // rows of the shortest own segment
    psw::RsGroup* d_rs_group = nullptr;
    psw::RsRun* d_rs_run = nullptr;
    psw::SegCoef* d_rs_runcoef = nullptr;  // composed affine map of every run
    int32_t* d_rs_runoff = nullptr;        // [Ploc + 1] first run of every own block
    void* d_scoef = nullptr;               // SolveCoef<T>[n]
    psw::CarryW* d_rs_cw = nullptr;        // [group][kRsSeg] closed-form carry weights

    // multi-GPU row shard (psw_shard_*); world == 1 for a full plan
    int rank = 0, world = 1;
    int64_t blk0 = 0, blk1 = 0;   // owned blocks [blk0, blk1)
    int64_t row0 = 0, row1 = 0;   // owned rows [row0, row1) (0-based, global)
};

namespace psw {
// Solve paths (psw_staged.cu / psw_fused.cu). All asynchronous on `s`.
int solve_staged(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                 int64_t N, int layout, cudaStream_t s, double* ext_bl, double* ext_br,
                 double* ext_v, void** events, int nevents);
bool fused_supported(const psw_plan* plan, int layout, int64_t N, const void* F, int64_t ldf);
// builds and uploads the FUSED tables from the per-row sweep coefficients
int build_fused_tables(psw_plan* pl, const std::vector<double>& rp, const std::vector<double>& ma,
                       const std::vector<double>& gr, const std::vector<double>& gl,
                       const std::vector<double>& w, const std::vector<double>& al,
                       const std::vector<double>& cmat);
// The dichotomy combination (boundary_solve.hpp:96-121) is linear in the
// betas: V = MR * right + ML * left. Returns [p][2P] rows (MR | ML), each
// column the reference combination of a unit beta vector (host, fp64,
// no FP contraction).
std::vector<double> combine_matrix(const psw_plan* pl, const std::vector<double>& zr,
                                   const std::vector<double>& zl);
bool cluster_supported(const psw_plan* plan, int layout, int64_t N, const void* F, int64_t ldf);
int solve_cluster(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                  int64_t N, int layout, cudaStream_t s, void** events, int nevents);
// CLUSTER coefficient tables of both layouts (psw_cluster.cu), built with the plan
int build_cluster_tables(psw_plan* pl, const std::vector<FusedFwd<double>>& ff,
                         const std::vector<FusedBwd<double>>& fb);

// RESWEEP (psw_resweep.cu): K1 part -> K2 combination -> K3 solve.
bool resweep_supported(const psw_plan* plan, int layout, int64_t N);
int solve_resweep(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                  int64_t N, int layout, cudaStream_t s, void** events, int nevents);
// RESWEEP tables (groups, runs, solve coefficients) over the plan's own blocks
int build_rs_tables(psw_plan* pl, const std::vector<SegDesc>& desc,
                    const std::vector<SegCoef>& seg, const std::vector<FusedFwd<double>>& ff,
                    const std::vector<FusedBwd<double>>& fb);
// row shards (psw_shard.cpp): forward = K1 + fold + the rank's share of the
// boundary values; backward = carries from the reduced values + K3
int64_t shard_workspace_bytes(const psw_plan* pl, int64_t N);
int shard_forward(const psw_plan* pl, const void* F, int64_t ldf, int64_t N, void* ws,
                  double* partials, int64_t ldv, cudaStream_t s);
int shard_backward(const psw_plan* pl, const void* F, int64_t ldf, void* X, int64_t ldx,
                   int64_t N, void* ws, const double* V, int64_t ldv, cudaStream_t s);
// AUTO path selection (psw_plan.cpp)
int auto_path(const psw_plan* pl, const void* F, int64_t ldf, const void* X, int64_t ldx,
              int64_t N, int layout);
// the STAGED dichotomy combination kernel (betas -> boundary values V, p x N)
int launch_combine(const psw_plan* plan, const double* bl, const double* br, int64_t N, double* V,
                   cudaStream_t s);
int solve_fused(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                int64_t N, int layout, cudaStream_t s, void** events, int nevents);
// records events[i] (if present) on s
inline void mark(void** events, int nevents, int i, cudaStream_t s) {
    if (events && i < nevents && events[i]) cudaEventRecord(static_cast<cudaEvent_t>(events[i]), s);
}
int set_trace(void* buf);  // psw_debug_trace (FUSED kernel phase stamps)
// Stream-ordered scratch from a library-owned memory pool per device that
// keeps its memory mapped between solves (the default pool trims at every
// synchronisation, and remapping ~0.1 GB of per-solve scratch costs more
// than a small kernel).
cudaError_t scratch_alloc(void** p, size_t bytes, int device, cudaStream_t s);
cudaError_t scratch_free(void* p, cudaStream_t s);
int fill_uniform(void* dst, int dtype, int64_t count, uint64_t seed, uint64_t offset, double lo,
                 double hi, cudaStream_t s);
int fill_normal(void* dst, int dtype, int64_t count, uint64_t seed, uint64_t offset,
                cudaStream_t s);
int l2_flush(void* scratch, int64_t bytes, cudaStream_t s);
}  // namespace psw
