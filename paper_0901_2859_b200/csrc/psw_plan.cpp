// Host side of the C ABI: validation, the fp64 preliminary phase, upload of
// the block-restricted data to HBM, and the public entry points.
//
// The preliminary mirrors compute_preliminary (dichotomy/preliminary.hpp:
// 171-199, DirectSymmetric route :139-143) operation for operation — this
// file is compiled with -ffp-contract=off so the inverse rows and Z samples
// are bitwise what the reference computes — but keeps only what the per-RHS
// kernels read: each inverse row restricted to its two adjacent blocks, the
// p x p Z-sample tables, and per-row sweep coefficients (psw_internal.h).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>

#include "psw_internal.h"

namespace {
thread_local int t_last_path = 0;  // psw_last_path
}  // namespace

namespace psw {

namespace {
thread_local std::string t_msg;
thread_local int64_t t_index = -1;
thread_local int64_t t_launches = 0;
constexpr double kPivotFloor = 1e-300;  // core/thomas.hpp:14
}  // namespace

void set_error(int code, const std::string& msg, int64_t index) {
    (void)code;
    t_msg = msg;
    t_index = index;
}
int clear_error() {
    t_msg.clear();
    t_index = -1;
    return PSW_OK;
}
int cuda_fail(cudaError_t e, const char* what) {
    set_error(PSW_CUDA_ERROR, std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                                  cudaGetErrorString(e) + ") in " + what);
    return e == cudaErrorMemoryAllocation ? PSW_OUT_OF_MEMORY : PSW_CUDA_ERROR;
}
void note_launches(int64_t k) { t_launches += k; }
void reset_launches() { t_launches = 0; }

namespace {

// core/thomas.hpp:22-45, same operation order (no contraction in this TU).
// Returns -1 on success or the failing (local) row.
int64_t thomas(int64_t n, const double* sub, const double* diag, const double* sup,
               const double* f, double* x, double* al, double* be) {
    double piv = diag[0];
    if (std::fabs(piv) < kPivotFloor) return 0;
    al[0] = (n > 1) ? -sup[0] / piv : 0.0;
    be[0] = f[0] / piv;
    for (int64_t i = 1; i < n; ++i) {
        piv = diag[i] + sub[i - 1] * al[i - 1];
        if (std::fabs(piv) < kPivotFloor) return i;
        al[i] = (i + 1 < n) ? -sup[i] / piv : 0.0;
        be[i] = (f[i] - sub[i - 1] * be[i - 1]) / piv;
    }
    x[n - 1] = be[n - 1];
    for (int64_t i = n - 1; i-- > 0;) x[i] = be[i] + al[i] * x[i + 1];
    return -1;
}

// ---- GRowProvider (dichotomy/preliminary.hpp:108-157) --------------------
// Inverse rows of A under a GRowStrategy; the constructor's Auto fallbacks
// (:111-132) and failure reports are the reference's, arithmetic included
// (core/symmetrize.hpp:21-37, core/inverse_rows.hpp:46-104; this file is
// compiled without FP contraction).
constexpr double kInverseScaleLimit = 1e280;  // core/inverse_rows.hpp:14

struct GRow {
    int strategy = PSW_GROW_DIRECT_SYMMETRIC;
    std::vector<double> scale, ssub, ssup;   // Symmetrize
    std::vector<double> y, z, y_rho, z_rho;  // ExplicitInverse
};

// core/inverse_rows.hpp:46-80: PSW_OK, PSW_ORACLE_FALLBACK_REQUIRED (msg) or
// a pivot breakdown (*bad)
int inverse_factors(int64_t n, const double* sub, const double* diag, const double* sup, GRow& g,
                    std::string& msg, int64_t& bad) {
    for (int64_t k = 0; k + 1 < n; ++k)
        if (sub[k] == 0.0 || sup[k] == 0.0) {
            msg = "zero off-diagonal entry: explicit inverse representation is undefined";
            return PSW_ORACLE_FALLBACK_REQUIRED;
        }
    std::vector<double> e(n, 0.0), al(n), be(n);
    g.y.assign(n, 0.0);
    g.z.assign(n, 0.0);
    e[n - 1] = 1.0;
    bad = thomas(n, sub, diag, sup, e.data(), g.y.data(), al.data(), be.data());
    if (bad >= 0) return PSW_PIVOT_BREAKDOWN;
    if (!(std::fabs(g.y[0]) >= 1.0 / kInverseScaleLimit)) {
        msg = "corner inverse entry underflows the usable scale";
        return PSW_ORACLE_FALLBACK_REQUIRED;
    }
    std::fill(e.begin(), e.end(), 0.0);
    e[0] = 1.0 / g.y[0];
    bad = thomas(n, sub, diag, sup, e.data(), g.z.data(), al.data(), be.data());
    if (bad >= 0) return PSW_PIVOT_BREAKDOWN;
    g.y_rho.resize(n);
    g.z_rho.resize(n);
    double rho = 1.0;
    for (int64_t j = 0; j < n; ++j) {
        if (j > 0) rho *= sup[j - 1] / sub[j - 1];
        if (!(std::fabs(rho) <= kInverseScaleLimit && std::fabs(rho) >= 1.0 / kInverseScaleLimit)) {
            msg = "cumulative off-diagonal ratio product left [1e-280, 1e280]";
            return PSW_ORACLE_FALLBACK_REQUIRED;
        }
        g.y_rho[j] = g.y[j] * rho;
        g.z_rho[j] = g.z[j] * rho;
        if (!std::isfinite(g.y_rho[j]) || !std::isfinite(g.z_rho[j])) {
            msg = "inverse factor overflow";
            return PSW_ORACLE_FALLBACK_REQUIRED;
        }
    }
    return PSW_OK;
}

// GRowProvider constructor: resolves the strategy; sets the error on failure
int grow_init(int64_t n, const double* sub, const double* diag, const double* sup, int requested,
              GRow& g) {
    int s = requested;
    if (s == PSW_GROW_AUTO) {
        bool sym = true;
        for (int64_t k = 0; k + 1 < n && sym; ++k) sym = sub[k] == sup[k];
        s = sym ? PSW_GROW_DIRECT_SYMMETRIC : PSW_GROW_SYMMETRIZE;
    }
    if (s == PSW_GROW_SYMMETRIZE) {  // core/symmetrize.hpp:21-37
        g.scale.assign(n, 1.0);
        g.ssub.assign(n > 1 ? n - 1 : 0, 0.0);
        g.ssup.assign(n > 1 ? n - 1 : 0, 0.0);
        int64_t fail = -1;
        for (int64_t k = 0; k + 1 < n; ++k) {
            const double product = sub[k] * sup[k];
            if (!(product > 0.0)) {
                fail = k;
                break;
            }
            g.scale[k + 1] = g.scale[k] * std::sqrt(sub[k] / sup[k]);
            const double off = std::copysign(std::sqrt(product), sup[k]);
            g.ssub[k] = off;
            g.ssup[k] = off;
        }
        if (fail < 0)
            for (double t : g.scale)
                if (!(std::isfinite(t) && t > 0.0)) {
                    fail = 0;
                    break;
                }
        if (fail >= 0) {
            if (requested != PSW_GROW_AUTO) {
                set_error(PSW_NOT_SYMMETRIZABLE,
                          "off-diagonal product sub[" + std::to_string(fail) + "]*super[" +
                              std::to_string(fail) +
                              "] is not positive; no diagonal similarity transform exists",
                          fail);
                return PSW_NOT_SYMMETRIZABLE;
            }
            s = PSW_GROW_EXPLICIT_INVERSE;
        }
    }
    if (s == PSW_GROW_EXPLICIT_INVERSE) {
        std::string msg;
        int64_t bad = -1;
        const int rc = inverse_factors(n, sub, diag, sup, g, msg, bad);
        if (rc == PSW_PIVOT_BREAKDOWN) {
            set_error(PSW_PIVOT_BREAKDOWN,
                      "pivot breakdown during forward elimination at row " + std::to_string(bad), bad);
            return rc;
        }
        if (rc == PSW_ORACLE_FALLBACK_REQUIRED) {
            if (requested != PSW_GROW_AUTO) {
                set_error(PSW_ORACLE_FALLBACK_REQUIRED, msg);
                return rc;
            }
            s = PSW_GROW_TRANSPOSE_SOLVE;
        }
    }
    g.strategy = s;
    return PSW_OK;
}

// GRowProvider::row (preliminary.hpp:136-156): row r0 (0-based) of inv(A)
// into x; returns the pivot-breakdown row or -1
int64_t grow_row(const GRow& g, int64_t n, const double* sub, const double* diag,
                 const double* sup, int64_t r0, double* x, double* e, double* al, double* be) {
    switch (g.strategy) {
        case PSW_GROW_DIRECT_SYMMETRIC:
            std::fill(e, e + n, 0.0);
            e[r0] = 1.0;
            return thomas(n, sub, diag, sup, e, x, al, be);
        case PSW_GROW_SYMMETRIZE: {
            std::fill(e, e + n, 0.0);
            e[r0] = 1.0;
            const int64_t bad = thomas(n, g.ssub.data(), diag, g.ssup.data(), e, x, al, be);
            if (bad >= 0) return bad;
            for (int64_t j = 0; j < n; ++j) x[j] *= g.scale[r0] / g.scale[j];
            return -1;
        }
        case PSW_GROW_EXPLICIT_INVERSE:
            for (int64_t j = 0; j < r0; ++j) x[j] = g.z[r0] * g.y_rho[j];
            for (int64_t j = r0; j < n; ++j) x[j] = g.y[r0] * g.z_rho[j];
            return -1;
        default:  // TransposeSolve: inverse_row_transpose (core/inverse_rows.hpp:99-104)
            std::fill(e, e + n, 0.0);
            e[r0] = 1.0;
            return thomas(n, sup, diag, sub, e, x, al, be);
    }
}

// Forward pivots only (for p == 0 the reference fails in the first solve's
// sweep of A itself, local_solve.hpp:49 -> thomas.hpp:32,38).
int64_t forward_breakdown(int64_t n, const double* sub, const double* diag, const double* sup) {
    double piv = diag[0];
    if (std::fabs(piv) < kPivotFloor) return 0;
    double al = (n > 1) ? -sup[0] / piv : 0.0;
    for (int64_t i = 1; i < n; ++i) {
        piv = diag[i] + sub[i - 1] * al;
        if (std::fabs(piv) < kPivotFloor) return i;
        al = (i + 1 < n) ? -sup[i] / piv : 0.0;
    }
    return -1;
}

// dichotomy/level_sets.hpp:18-37 -> level-ordered items with the nearest known
// neighbours that solve_boundaries finds by scanning (boundary_solve.hpp:106-113).
std::vector<psw::CombineItem> build_items(int64_t p, int64_t* terms_out,
                                          std::vector<int32_t>* lvl_off) {
    std::vector<psw::CombineItem> items;
    if (lvl_off) lvl_off->assign(1, 0);
    if (p == 0) {
        if (terms_out) *terms_out = 0;
        return items;
    }
    int64_t depth = 1;
    while ((int64_t{1} << depth) <= p) ++depth;
    std::vector<char> taken(p + 1, 0), known(p, 0);
    int64_t terms = 0;
    for (int64_t l = 1; l <= depth; ++l) {
        const int64_t stride = int64_t{1} << (depth - l);
        std::vector<int64_t> level;
        for (int64_t k = 1; k < (int64_t{1} << l); ++k) {
            const int64_t j = stride * k;
            if (j > p) break;
            if (taken[j]) continue;
            taken[j] = 1;
            level.push_back(j);
        }
        for (int64_t pos : level) {
            const int64_t i = pos - 1;
            int64_t kl = i - 1;
            while (kl >= 0 && !known[kl]) --kl;
            int64_t kr = i + 1;
            while (kr < p && !known[kr]) ++kr;
            items.push_back({int32_t(i), int32_t(kl), int32_t(kr), 0});
            // segment_particular counts (e - kl) + (kr - e) terms per call
            const int64_t per = kr - kl;
            terms += per * (1 + (kl >= 0) + (kr < p));
        }
        for (int64_t pos : level) known[pos - 1] = 1;
        if (lvl_off) lvl_off->push_back(int32_t(items.size()));
    }
    if (terms_out) *terms_out = terms;
    return items;
}

template <typename T>
int upload(psw_plan* pl, const std::vector<double>& rp, const std::vector<double>& ma,
           const std::vector<double>& gr, const std::vector<double>& gl,
           const std::vector<double>& w, const std::vector<double>& al,
           const std::vector<double>& zr, const std::vector<double>& zl) {
    const int64_t n = pl->n, p = pl->p;
    // kCoefPad zero rows past n: the PIPE path bulk-copies whole 32-row stages
    const int64_t na = n + kCoefPad;
    std::vector<FwdCoef<T>> fwd(na, FwdCoef<T>{});
    std::vector<BwdCoef<T>> bwd(na, BwdCoef<T>{});
    for (int64_t q = 0; q < n; ++q) {
        fwd[q] = {T(rp[q]), T(ma[q]), T(gr[q]), T(gl[q])};
        bwd[q] = {T(w[q]), T(al[q])};
    }
    PSW_CUDA_TRY(cudaMalloc(&pl->d_fwd, sizeof(FwdCoef<T>) * na));
    PSW_CUDA_TRY(cudaMalloc(&pl->d_bwd, sizeof(BwdCoef<T>) * na));
    PSW_CUDA_TRY(cudaMemcpy(pl->d_fwd, fwd.data(), sizeof(FwdCoef<T>) * na, cudaMemcpyHostToDevice));
    PSW_CUDA_TRY(cudaMemcpy(pl->d_bwd, bwd.data(), sizeof(BwdCoef<T>) * na, cudaMemcpyHostToDevice));
    PSW_CUDA_TRY(cudaMalloc(&pl->d_blk, sizeof(int32_t) * pl->blk.size()));
    PSW_CUDA_TRY(cudaMemcpy(pl->d_blk, pl->blk.data(), sizeof(int32_t) * pl->blk.size(),
                            cudaMemcpyHostToDevice));
    int64_t bytes = int64_t(sizeof(FwdCoef<T>) + sizeof(BwdCoef<T>)) * n +
                    int64_t(sizeof(int32_t) * pl->blk.size());
    if (p > 0) {
        // padded to a 16-byte multiple (bulk copies of the whole table)
        PSW_CUDA_TRY(cudaMalloc(&pl->d_zr, sizeof(double) * (p * p + 2)));
        PSW_CUDA_TRY(cudaMalloc(&pl->d_zl, sizeof(double) * (p * p + 2)));
        PSW_CUDA_TRY(cudaMemset(pl->d_zr, 0, sizeof(double) * (p * p + 2)));
        PSW_CUDA_TRY(cudaMemset(pl->d_zl, 0, sizeof(double) * (p * p + 2)));
        PSW_CUDA_TRY(cudaMemcpy(pl->d_zr, zr.data(), sizeof(double) * p * p, cudaMemcpyHostToDevice));
        PSW_CUDA_TRY(cudaMemcpy(pl->d_zl, zl.data(), sizeof(double) * p * p, cudaMemcpyHostToDevice));
        PSW_CUDA_TRY(cudaMalloc(&pl->d_items, sizeof(psw::CombineItem) * p));
        PSW_CUDA_TRY(cudaMemcpy(pl->d_items, pl->items.data(), sizeof(psw::CombineItem) * p,
                                cudaMemcpyHostToDevice));
        bytes += int64_t(2 * sizeof(double) * p * p + sizeof(psw::CombineItem) * p);
        PSW_CUDA_TRY(cudaMalloc(&pl->d_lvl_off, sizeof(int32_t) * pl->lvl_off.size()));
        PSW_CUDA_TRY(cudaMemcpy(pl->d_lvl_off, pl->lvl_off.data(),
                                sizeof(int32_t) * pl->lvl_off.size(), cudaMemcpyHostToDevice));
    }
    pl->info.device_bytes = bytes;
    return PSW_OK;
}

void free_plan(psw_plan* pl) {
    if (!pl) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(pl->device);
    void* ptrs[] = {pl->d_fwd, pl->d_bwd, pl->d_blk, pl->d_zr, pl->d_zl, pl->d_items,
                    pl->d_lvl_off, pl->d_ffwd, pl->d_fbwd, pl->d_seg, pl->d_cmat,
                    pl->d_segdesc, pl->d_segoff, pl->d_ctab[0], pl->d_ctab[1],
                    pl->d_rs_group, pl->d_rs_run, pl->d_rs_runcoef, pl->d_rs_runoff,
                    pl->d_scoef, pl->d_rs_cw};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    cudaSetDevice(prev);
    delete pl;
}

int validate_inputs(int64_t n, const double* sub, const double* diag, const double* sup,
                    int64_t p, const int64_t* bnd) {
    if (n < 2) {
        set_error(PSW_INVALID_ARGUMENT, "TridiagMatrix: order must be >= 2");
        return PSW_INVALID_ARGUMENT;
    }
    if (n > (int64_t{1} << 30)) {
        set_error(PSW_INVALID_ARGUMENT, "order exceeds 2^30 rows");
        return PSW_INVALID_ARGUMENT;
    }
    if (!sub || !diag || !sup || (p > 0 && !bnd) || p < 0) {
        set_error(PSW_INVALID_ARGUMENT, "null matrix or partition pointer");
        return PSW_INVALID_ARGUMENT;
    }
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(diag[i])) {
            set_error(PSW_INVALID_ARGUMENT, "TridiagMatrix: entries must be finite");
            return PSW_INVALID_ARGUMENT;
        }
    for (int64_t i = 0; i + 1 < n; ++i)
        if (!std::isfinite(sub[i]) || !std::isfinite(sup[i])) {
            set_error(PSW_INVALID_ARGUMENT, "TridiagMatrix: entries must be finite");
            return PSW_INVALID_ARGUMENT;
        }
    return psw_partition_validate(n, p, bnd);
}

}  // namespace

// Builds the plan for a (possibly sharded) solve. Rank/world select the
// owned block range for psw_shard_*; world == 1 is the full plan.
// `cmat_host` != nullptr: host-only run (no device needed) that stops after
// the preliminary and returns the combination matrix (psw_combine_matrix).
int build_plan(psw_plan** out, int64_t n, const double* sub, const double* diag,
               const double* sup, int64_t p, const int64_t* bnd, int dtype, int device,
               int rank, int world, std::vector<double>* cmat_host = nullptr, bool shard = false,
               int strategy = PSW_GROW_AUTO, int flags = 0);

int device_preliminary(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* bnd, const std::vector<int32_t>& blk,
                       std::vector<double>& gr, std::vector<double>& gl, std::vector<double>& zr,
                       std::vector<double>& zl, double& max_z, int64_t& bad_row, int* serial);

// Where the DirectSymmetric preliminary runs: on the GPU (psw_prelim.cu,
// bitwise the host setup) whenever a device is there and the 3p sweeps are
// long enough to pay for its allocation, copies and launches (about 2 ms;
// PSW_DEVICE_SETUP_MIN, default 3 p n >= 2^21 row steps: C2 8.5 -> 1.9 ms, C3
// 202 -> 12 ms, while a 4096-row system takes 0.4 ms on the host against 2 ms;
// tools/setup_bench.py); PSW_DEVICE_SETUP=0 keeps the host's worker
// threads, =1 forces the device. Without a device the host path runs, so that
// validation and PivotBreakdown are still reported before the missing device.
// test hook (psw_debug_preliminary): the raw tables of the preliminary
struct PrelimCapture {
    std::vector<double> gr, gl, zr, zl;
};
static thread_local PrelimCapture* t_capture = nullptr;

static bool want_device_setup(int64_t n, int64_t p, int device) {
    if (p <= 0 || n <= 0) return false;
    const char* e = std::getenv("PSW_DEVICE_SETUP");
    if (e && *e && std::atoi(e) == 0) return false;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return false;
    }
    if (e && *e) return true;
    const char* m = std::getenv("PSW_DEVICE_SETUP_MIN");
    const int64_t min_steps = m && *m ? std::atoll(m) : (int64_t{1} << 21);
    return 3 * p * n >= min_steps;
}

int build_plan(psw_plan** out, int64_t n, const double* sub, const double* diag,
               const double* sup, int64_t p, const int64_t* bnd, int dtype, int device,
               int rank, int world, std::vector<double>* cmat_host, bool shard, int strategy,
               int flags) {
    clear_error();
    if (!out) {
        set_error(PSW_INVALID_ARGUMENT, "null plan output");
        return PSW_INVALID_ARGUMENT;
    }
    *out = nullptr;
    if (dtype != PSW_F64 && dtype != PSW_F32) {
        set_error(PSW_INVALID_ARGUMENT, "dtype must be PSW_F64 or PSW_F32");
        return PSW_INVALID_ARGUMENT;
    }
    if (int rc = validate_inputs(n, sub, diag, sup, p, bnd)) return rc;
    if (world < 1 || rank < 0 || rank >= world || (p + 1) % world != 0) {
        set_error(PSW_INVALID_ARGUMENT,
                  "row sharding needs 0 <= rank < world and P = p+1 blocks divisible by world");
        return PSW_INVALID_ARGUMENT;
    }
    if (strategy < PSW_GROW_AUTO || strategy > PSW_GROW_TRANSPOSE_SOLVE) {
        set_error(PSW_INVALID_ARGUMENT, "unknown GRowStrategy");
        return PSW_INVALID_ARGUMENT;
    }
    const auto t0 = std::chrono::steady_clock::now();

    auto* pl = new (std::nothrow) psw_plan();
    if (!pl) {
        set_error(PSW_OUT_OF_MEMORY, "host allocation failed");
        return PSW_OUT_OF_MEMORY;
    }
    pl->n = n;
    pl->p = p;
    pl->P = p + 1;
    pl->dtype = dtype;
    pl->device = device;
    pl->rank = rank;
    pl->world = world;
    pl->bnd.assign(bnd, bnd + p);

    // block ranges (partition.hpp:26-29, 0-based owned rows)
    pl->blk.resize(2 * pl->P);
    for (int64_t t = 0; t <= p; ++t) {
        pl->blk[2 * t] = int32_t(t == 0 ? 0 : bnd[t - 1] - 1);
        pl->blk[2 * t + 1] = int32_t(t == p ? n : bnd[t] - 1);
    }
    // owned blocks and rows: rank r of `world` owns [r P/world, (r+1) P/world)
    {
        const int64_t Ploc = pl->P / world;
        pl->blk0 = int64_t(rank) * Ploc;
        pl->blk1 = pl->blk0 + Ploc;
        pl->row0 = pl->blk[2 * pl->blk0];
        pl->row1 = pl->blk[2 * (pl->blk1 - 1) + 1];
    }
    pl->uniform = (n % pl->P == 0);
    if (pl->uniform) {
        std::vector<int64_t> ref(p);
        if (p > 0 && psw_decompose(n, pl->P, ref.data()) != PSW_OK) pl->uniform = false;
        for (int64_t j = 0; pl->uniform && j < p; ++j) pl->uniform = ref[j] == bnd[j];
        clear_error();
    }
    pl->m = pl->uniform ? n / pl->P : 0;

    // ---- preliminary (preliminary.hpp:171-199) --------------------------
    std::vector<double> gr(n, 0.0), gl(n, 0.0), zr(p * p, 0.0), zl(p * p, 0.0);
    double max_z = 0.0;
    GRow grow;  // the GRowProvider is constructed before any boundary (:179-180)
    if (int rc = grow_init(n, sub, diag, sup, strategy, grow)) {
        delete pl;
        return rc;
    }
    pl->info.strategy_used = grow.strategy;
    if (p == 0) {
        int64_t bad = forward_breakdown(n, sub, diag, sup);
        if (bad >= 0) {
            set_error(PSW_PIVOT_BREAKDOWN,
                      "pivot breakdown during forward elimination at row " + std::to_string(bad),
                      bad);
            delete pl;
            return PSW_PIVOT_BREAKDOWN;
        }
    }
    bool host_sweeps = p > 0;
    if (p > 0 && !cmat_host && grow.strategy == PSW_GROW_DIRECT_SYMMETRIC &&
        want_device_setup(n, p, device)) {
        // the 3p sweeps on the GPU, bitwise the host restatement (psw_prelim.cu)
        int prev_dev = 0;
        cudaGetDevice(&prev_dev);
        cudaSetDevice(device);
        int64_t bad = -1;
        int serial = 0;
        const int rc = device_preliminary(n, sub, diag, sup, p, bnd, pl->blk, gr, gl, zr, zl, max_z,
                                          bad, &serial);
        cudaSetDevice(prev_dev);
        if (rc == PSW_PIVOT_BREAKDOWN) {
            set_error(PSW_PIVOT_BREAKDOWN,
                      "pivot breakdown during forward elimination at row " + std::to_string(bad),
                      bad);
            delete pl;
            return PSW_PIVOT_BREAKDOWN;
        }
        if (rc == PSW_OK) {
            pl->info.device_setup = serial ? 2 : 1;
            host_sweeps = false;
        } else if (rc != PSW_NOT_SUPPORTED) {  // NOT_SUPPORTED: a chain outgrew the device
            delete pl;                         // scratch window, the host does the sweeps
            return rc;
        } else {
            clear_error();
            gr.assign(n, 0.0);
            gl.assign(n, 0.0);
            zr.assign(p * p, 0.0);
            zl.assign(p * p, 0.0);
        }
    }
    if (host_sweeps) {
        // boundaries are independent items (preliminary.hpp:182-195); errors
        // are reported in the serial executor's order (boundary, then g,
        // z_left, z_right).
        struct Fail {
            int64_t j = -1, stage = 0, row = 0;
        };
        std::vector<Fail> fails(p);
        std::vector<std::vector<double>> zl_rows(p), zr_rows(p);  // sampled only
        std::atomic<int64_t> next{0};
        std::mutex mz_mu;
        auto worker = [&]() {
            std::vector<double> e(n), x(n), al(n), be(n), bd(n), bs(n), bu(n);
            double mz_local = 0.0;
            for (;;) {
                const int64_t j = next.fetch_add(1);
                if (j >= p) break;
                const int64_t r = bnd[j];
                Fail& f = fails[j];
                // g_j = row r of inv(A) by the resolved strategy (:136-156),
                // restricted to blocks j and j+1 (the only rows betas.hpp:46-55 reads)
                int64_t bad = grow_row(grow, n, sub, diag, sup, r - 1, x.data(), e.data(),
                                       al.data(), be.data());
                if (bad >= 0) { f = {j, 0, bad}; continue; }
                for (int32_t q = pl->blk[2 * j]; q < pl->blk[2 * j + 1]; ++q) gr[q] = x[q];
                for (int32_t q = pl->blk[2 * (j + 1)]; q < pl->blk[2 * (j + 1) + 1]; ++q) gl[q] = x[q];
                // z_left: b_left_matrix (:29-37), rhs e_last
                std::copy(diag, diag + r, bd.begin());
                bd[r - 1] = 1.0;
                std::copy(sub, sub + (r - 1), bs.begin());
                bs[r - 2] = 0.0;
                std::copy(sup, sup + (r - 1), bu.begin());
                std::fill(e.begin(), e.begin() + r, 0.0);
                e[r - 1] = 1.0;
                bad = thomas(r, bs.data(), bd.data(), bu.data(), e.data(), x.data(), al.data(), be.data());
                if (bad >= 0) { f = {j, 1, bad}; continue; }
                auto& zlr = zl_rows[j];
                zlr.resize(j + 1);
                for (int64_t i = 0; i <= j; ++i) zlr[i] = x[bnd[i] - 1];
                for (int64_t q = 0; q < r; ++q) mz_local = std::max(mz_local, std::fabs(x[q]));
                // z_right: b_right_matrix (:41-49), rhs e_first
                const int64_t m = n - r + 1;
                std::copy(diag + (r - 1), diag + n, bd.begin());
                bd[0] = 1.0;
                std::copy(sub + (r - 1), sub + (n - 1), bs.begin());
                std::copy(sup + (r - 1), sup + (n - 1), bu.begin());
                bu[0] = 0.0;
                std::fill(e.begin(), e.begin() + m, 0.0);
                e[0] = 1.0;
                bad = thomas(m, bs.data(), bd.data(), bu.data(), e.data(), x.data(), al.data(), be.data());
                if (bad >= 0) { f = {j, 2, bad}; continue; }
                auto& zrr = zr_rows[j];
                zrr.resize(p - j);
                for (int64_t i = j; i < p; ++i) zrr[i - j] = x[bnd[i] - r];
                for (int64_t q = 0; q < m; ++q) mz_local = std::max(mz_local, std::fabs(x[q]));
            }
            std::lock_guard<std::mutex> lk(mz_mu);
            max_z = std::max(max_z, mz_local);
        };
        int nth = int(std::min<int64_t>(p, std::max(1u, std::thread::hardware_concurrency())));
        nth = std::min(nth, 32);
        std::vector<std::thread> th;
        for (int w = 1; w < nth; ++w) th.emplace_back(worker);
        worker();
        for (auto& t : th) t.join();
        for (int64_t j = 0; j < p; ++j)
            if (fails[j].j >= 0) {
                const int64_t bad = fails[j].row;
                set_error(PSW_PIVOT_BREAKDOWN,
                          "pivot breakdown during forward elimination at row " + std::to_string(bad),
                          bad);
                delete pl;
                return PSW_PIVOT_BREAKDOWN;
            }
        // build_samples (preliminary.hpp:85-96)
        for (int64_t j = 0; j < p; ++j) {
            for (int64_t i = j; i < p; ++i) zr[j * p + i] = zr_rows[j][i - j];
            for (int64_t i = 0; i <= j; ++i) zl[j * p + i] = zl_rows[j][i];
        }
    }

    const auto t_prelim = std::chrono::steady_clock::now();
    if (t_capture) {
        t_capture->gr = gr;
        t_capture->gl = gl;
        t_capture->zr = zr;
        t_capture->zl = zl;
    }
    // ---- per-row sweep coefficients of every block (local_solve.hpp:25-50)
    std::vector<double> rp(n, 0.0), ma(n, 0.0), w(n, 0.0), alv(n, 0.0);
    for (int64_t t = 0; t <= p; ++t) {
        const int64_t s = pl->blk[2 * t], e = pl->blk[2 * t + 1];
        const int64_t h = (t == p) ? n - 1 : e;  // closed block end
        double alpha_prev;
        if (t > 0) {  // unit first row carrying x_{t-1}
            rp[s] = 0.0;
            ma[s] = 0.0;
            w[s] = 1.0;
            alv[s] = 0.0;
            alpha_prev = 0.0;
        } else {
            const double piv = diag[0];
            alpha_prev = (h > s) ? -sup[0] / piv : 0.0;
            rp[s] = 1.0 / piv;
            ma[s] = 0.0;
            w[s] = 0.0;
            alv[s] = alpha_prev;
        }
        const int64_t last = (t == p) ? n : e;  // owned rows beyond the first
        for (int64_t q = s + 1; q < last; ++q) {
            const double piv = diag[q] + sub[q - 1] * alpha_prev;
            const double a = (q < h) ? -sup[q] / piv : 0.0;
            rp[q] = 1.0 / piv;
            ma[q] = -sub[q - 1] / piv;
            w[q] = (t > 0) ? ma[q] * w[q - 1] : 0.0;
            alv[q] = a;
            alpha_prev = a;
        }
    }
    const auto t_coef = std::chrono::steady_clock::now();
    int64_t terms = 0;
    pl->items = build_items(p, &terms, &pl->lvl_off);
    if (cmat_host) {
        *cmat_host = combine_matrix(pl, zr, zl);
        delete pl;
        return PSW_OK;
    }

    // the device is only needed for the upload: host validation and the
    // preliminary (and its PivotBreakdown) come first, like the reference
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set_error(PSW_CUDA_ERROR, "no CUDA device available (the product has no CPU fallback)");
        delete pl;
        return PSW_CUDA_ERROR;
    }
    if (device < 0 || device >= ndev) {
        set_error(PSW_INVALID_ARGUMENT, "device ordinal out of range");
        delete pl;
        return PSW_INVALID_ARGUMENT;
    }
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    if (cudaSetDevice(device) != cudaSuccess) {
        set_error(PSW_CUDA_ERROR, "cudaSetDevice failed");
        delete pl;
        return PSW_CUDA_ERROR;
    }
    int rc = (dtype == PSW_F64) ? upload<double>(pl, rp, ma, gr, gl, w, alv, zr, zl)
                                : upload<float>(pl, rp, ma, gr, gl, w, alv, zr, zl);
    const auto t_upload = std::chrono::steady_clock::now();
    // PSW_PLAN_STAGED_ONLY: no segment tables (FUSED / CLUSTER / RESWEEP
    // unsupported, STAGED and the multi-matrix solve only) — a cheap plan for
    // the many one-RHS systems of the Fourier consumer
    if (rc == PSW_OK && !(flags & PSW_PLAN_STAGED_ONLY))
        rc = build_fused_tables(pl, rp, ma, gr, gl, w, alv,
                                pl->P <= 1024 || shard ? combine_matrix(pl, zr, zl)
                                                       : std::vector<double>());
    cudaSetDevice(prev_dev);
    if (rc != PSW_OK) {
        free_plan(pl);
        return rc;
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (const char* v = std::getenv("PSW_SETUP_VERBOSE"); v && std::atoi(v)) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr,
                     "psw setup n=%lld p=%lld: preliminary %.3f ms (%s), block coefficients %.3f ms, "
                     "upload %.3f ms, tables %.3f ms, total %.3f ms\n",
                     (long long)n, (long long)p, ms(t0, t_prelim),
                     pl->info.device_setup ? (pl->info.device_setup == 2 ? "device, serial chain" : "device")
                                           : "host",
                     ms(t_prelim, t_coef), ms(t_coef, t_upload), ms(t_upload, t1), ms(t0, t1));
    }
    auto& in = pl->info;
    in.n = n;
    in.p = p;
    in.dtype = dtype;
    in.device = device;
    in.uniform = pl->uniform ? 1 : 0;
    in.fused_ok = psw::fused_supported(pl, PSW_LAYOUT_R, 1 << 20, nullptr, 1 << 20) ? 1 : 0;
    in.combine_terms = terms;
    int64_t depth = 0;
    if (p > 0) {
        depth = 1;
        while ((int64_t{1} << depth) <= p) ++depth;
    }
    in.comm_rounds = p > 0 ? depth + 2 : 0;
    in.setup_seconds = std::chrono::duration<double>(t1 - t0).count();
    in.max_z_norm = max_z;
    *out = pl;
    return PSW_OK;
}

void destroy_plan(psw_plan* pl) { free_plan(pl); }

// boundary_solve.hpp:42-88 on the host, item by item (same arithmetic as
// the device combine_item; this TU has no FP contraction).
static void host_combine(const psw_plan* pl, const std::vector<double>& zr,
                         const std::vector<double>& zl, const double* left, const double* right,
                         double* V) {
    const int64_t p = pl->p;
    for (const auto& it : pl->items) {
        const int64_t i = it.i, kl = it.kl, kr = it.kr;
        double vi = 0.0, sl = 0.0, sr = 0.0;
        for (int64_t t = kl + 1; t <= kr; ++t) {
            vi += t <= i ? right[t] * zr[t * p + i] : left[t] * zl[(t - 1) * p + i];
            if (kl >= 0) sl += left[t] * zl[(t - 1) * p + kl];
            if (kr < p) sr += right[t] * zr[t * p + kr];
        }
        double v;
        if (kl >= 0 && kr < p) {
            const double b1 = V[kl] - sl, b2 = V[kr] - sr;
            const double m12 = zl[kr * p + kl], m21 = zr[kl * p + kr];
            const double det = 1.0 - m12 * m21;
            const double cl = (b1 - m12 * b2) / det, cr = (b2 - m21 * b1) / det;
            v = vi + cl * zr[kl * p + i] + cr * zl[kr * p + i];
        } else if (kr < p) {
            v = vi + (V[kr] - sr) * zl[kr * p + i];
        } else if (kl >= 0) {
            v = vi + (V[kl] - sl) * zr[kl * p + i];
        } else {
            v = vi;
        }
        V[i] = v;
    }
}

std::vector<double> combine_matrix(const psw_plan* pl, const std::vector<double>& zr,
                                   const std::vector<double>& zl) {
    const int64_t p = pl->p, P = pl->P;
    std::vector<double> M(size_t(p) * 2 * P, 0.0), unit(P, 0.0), zero(P, 0.0), col(p > 0 ? p : 1);
    for (int64_t t = 0; t < P; ++t) {
        unit[t] = 1.0;
        if (t < p) {  // right[t] (betas.hpp:46-49)
            host_combine(pl, zr, zl, zero.data(), unit.data(), col.data());
            for (int64_t j = 0; j < p; ++j) M[j * 2 * P + t] = col[j];
        }
        if (t > 0) {  // left[t] (betas.hpp:51-55)
            host_combine(pl, zr, zl, unit.data(), zero.data(), col.data());
            for (int64_t j = 0; j < p; ++j) M[j * 2 * P + P + t] = col[j];
        }
        unit[t] = 0.0;
    }
    return M;
}

}  // namespace psw

namespace psw {
// AUTO path choice (measured on B200): the on-chip paths first
// (CLUSTER for >= 128 RHS tiles of 128 B, FUSED), then the L2-chunked
// RESWEEP when a 32-RHS column of F is small next to L2 (its second read
// then hits L2), then RESWEEP, then STAGED.
cudaError_t scratch_alloc(void** p, size_t bytes, int device, cudaStream_t s) {
    static std::mutex mu;
    static std::vector<cudaMemPool_t> pools;
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (size_t(device) >= pools.size()) pools.resize(size_t(device) + 1, nullptr);
        if (!pools[size_t(device)]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = device;
            cudaMemPool_t np = nullptr;
            if (cudaError_t e = cudaMemPoolCreate(&np, &props)) return e;
            uint64_t keep = ~uint64_t(0);
            cudaMemPoolSetAttribute(np, cudaMemPoolAttrReleaseThreshold, &keep);
            pools[size_t(device)] = np;  // lives for the process
        }
        pool = pools[size_t(device)];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

cudaError_t scratch_free(void* p, cudaStream_t s) { return cudaFreeAsync(p, s); }

int auto_path(const psw_plan* pl, const void* F, int64_t ldf, const void* X, int64_t ldx,
              int64_t N, int layout) {
    const int64_t es = pl->dtype == PSW_F64 ? 8 : 4;
    if (N * es >= 128 * 128 && cluster_supported(pl, layout, N, F, ldf)) return PSW_PATH_CLUSTER;
    if (fused_supported(pl, layout, N, F, ldf)) return PSW_PATH_FUSED;
    // CHUNKED (RESWEEP over L2-sized RHS chunks) is explicit only: on the fp32
    // config its per-chunk launches cost more than the re-read they save
    // (27 vs 10.2 ms, round 2)
    // HOLD (one RHS tile of all rows held by the whole grid through one
    // persistent launch, fp32, F read once) is retired: 26.9 ms on the fp32
    // config against RESWEEP's 9.4 ms, and bound at about 8 ms by design (three
    // tiles fit the grid's shared memory against an exchange chain of three L2
    // hops)
    if (resweep_supported(pl, layout, N)) return PSW_PATH_RESWEEP;
    return PSW_PATH_STAGED;
}
}  // namespace psw

// ============================ C ABI ========================================
extern "C" {

const char* psw_last_error_message(void) { return psw::t_msg.c_str(); }
int64_t psw_last_error_index(void) { return psw::t_index; }
int psw_abi_version(void) { return PSW_ABI_VERSION; }
int64_t psw_last_launch_count(void) { return psw::t_launches; }

int psw_decompose(int64_t n, int64_t P, int64_t* out) {
    psw::clear_error();
    // runtime/decompose.hpp:33-47
    if (P <= 0 || n < 2 * P) {
        psw::set_error(PSW_TOO_MANY_PES, "cannot place " + std::to_string(n) + " rows on " +
                                             std::to_string(P) + " PEs with every range >= 2 rows");
        return PSW_TOO_MANY_PES;
    }
    if (!out && P > 1) {
        psw::set_error(PSW_INVALID_ARGUMENT, "null output");
        return PSW_INVALID_ARGUMENT;
    }
    const int64_t base = n / P, rem = n % P;
    int64_t last = 0;
    for (int64_t i = 0; i + 1 < P; ++i) {
        last += base + (i < rem ? 1 : 0);
        out[i] = last;  // induced_partition: right ends but the last (:23-29)
    }
    return PSW_OK;
}

int psw_partition_validate(int64_t n, int64_t p, const int64_t* b) {
    psw::clear_error();
    // dichotomy/partition.hpp:31-42
    if (n < 2) {
        psw::set_error(PSW_INVALID_ARGUMENT, "Partition: order must be >= 2");
        return PSW_INVALID_ARGUMENT;
    }
    int64_t prev = 0;
    for (int64_t j = 0; j < p; ++j) {
        if (b[j] < 2 || b[j] > n - 1) {
            psw::set_error(PSW_INVALID_ARGUMENT, "Partition: boundary " + std::to_string(b[j]) +
                                                     " is not interior to 1.." + std::to_string(n),
                           j);
            return PSW_INVALID_ARGUMENT;
        }
        if (b[j] <= prev) {
            psw::set_error(PSW_INVALID_ARGUMENT, "Partition: boundaries must be strictly increasing", j);
            return PSW_INVALID_ARGUMENT;
        }
        prev = b[j];
    }
    return PSW_OK;
}

int psw_plan_create(psw_plan** out, int64_t n, const double* sub, const double* diag,
                    const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                    int device) {
    return psw::build_plan(out, n, sub, diag, sup, p, boundaries, dtype, device, 0, 1);
}

int psw_plan_create_ex(psw_plan** out, int64_t n, const double* sub, const double* diag,
                       const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                       int device, int strategy) {
    return psw::build_plan(out, n, sub, diag, sup, p, boundaries, dtype, device, 0, 1, nullptr,
                           false, strategy);
}

int psw_plan_create_flags(psw_plan** out, int64_t n, const double* sub, const double* diag,
                          const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                          int device, int strategy, int flags) {
    return psw::build_plan(out, n, sub, diag, sup, p, boundaries, dtype, device, 0, 1, nullptr,
                           false, strategy, flags);
}

int psw_plan_destroy(psw_plan* plan) {
    psw::clear_error();
    psw::destroy_plan(plan);
    return PSW_OK;
}

int psw_plan_info(const psw_plan* plan, psw_plan_info_t* info) {
    psw::clear_error();
    if (!plan || !info) {
        psw::set_error(PSW_INVALID_ARGUMENT, "null plan or info");
        return PSW_INVALID_ARGUMENT;
    }
    *info = plan->info;
    return PSW_OK;
}

static int check_solve_args(const psw_plan* plan, const void* F, int64_t ldf, const void* X,
                            int64_t ldx, int64_t nrhs, int layout) {
    if (!plan) {
        psw::set_error(PSW_INVALID_ARGUMENT, "null plan");
        return PSW_INVALID_ARGUMENT;
    }
    if (nrhs < 0 || (nrhs > 0 && (!F || !X))) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid right-hand-side buffers");
        return PSW_INVALID_ARGUMENT;
    }
    if (layout != PSW_LAYOUT_R && layout != PSW_LAYOUT_S) {
        psw::set_error(PSW_INVALID_ARGUMENT, "layout must be PSW_LAYOUT_R or PSW_LAYOUT_S");
        return PSW_INVALID_ARGUMENT;
    }
    const int64_t need = layout == PSW_LAYOUT_R ? nrhs : plan->n;
    if (ldf < need || ldx < need) {
        psw::set_error(PSW_INVALID_ARGUMENT, "leading dimension too small for the layout");
        return PSW_INVALID_ARGUMENT;
    }
    if (plan->world != 1) {
        psw::set_error(PSW_INVALID_ARGUMENT, "sharded plan: use psw_shard_solve (or psw_shard_forward/backward)");
        return PSW_INVALID_ARGUMENT;
    }
    return PSW_OK;
}

int psw_last_path(void) { return t_last_path; }

int psw_solve_ex(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                 int64_t nrhs, int layout, void* stream, const psw_solve_opts* opts) {
    psw::clear_error();
    psw::reset_launches();
    if (int rc = check_solve_args(plan, F, ldf, X, ldx, nrhs, layout)) return rc;
    if (nrhs == 0) return PSW_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != plan->device) PSW_CUDA_TRY(cudaSetDevice(plan->device));
    auto s = static_cast<cudaStream_t>(stream);
    int path = opts ? opts->path : PSW_PATH_AUTO;
    const bool want_intermediates =
        opts && (opts->betas_left || opts->betas_right || opts->boundary_values);
    int rc;
    t_last_path = 0;
    void** ev = opts ? opts->events : nullptr;
    const int nev = opts ? opts->nevents : 0;
    if (path == PSW_PATH_AUTO && !want_intermediates)
        path = psw::auto_path(plan, F, ldf, X, ldx, nrhs, layout);
    t_last_path = path;
    auto unsupported = [&](const char* name) {
        psw::set_error(PSW_NOT_SUPPORTED, std::string(name) + " path does not support this plan/shape");
        return int(PSW_NOT_SUPPORTED);
    };
    if (path != PSW_PATH_STAGED && path != PSW_PATH_AUTO && want_intermediates) {
        rc = unsupported("only the staged");
    } else if (path == PSW_PATH_CHUNKED) {
        rc = unsupported("chunked (retired)");
    } else if (path == PSW_PATH_CLUSTER) {
        rc = psw::cluster_supported(plan, layout, nrhs, F, ldf)
                 ? psw::solve_cluster(plan, F, ldf, X, ldx, nrhs, layout, s, ev, nev)
                 : unsupported("cluster");
    } else if (path == PSW_PATH_RESWEEP) {
        rc = psw::resweep_supported(plan, layout, nrhs)
                 ? psw::solve_resweep(plan, F, ldf, X, ldx, nrhs, layout, s, ev, nev)
                 : unsupported("resweep");
    } else if (path == PSW_PATH_HOLD) {
        rc = unsupported("hold (retired)");
    } else if (path == PSW_PATH_FUSED) {
        rc = psw::fused_supported(plan, layout, nrhs, F, ldf)
                 ? psw::solve_fused(plan, F, ldf, X, ldx, nrhs, layout, s, ev, nev)
                 : unsupported("fused");
    } else if (path == PSW_PATH_STAGED || path == PSW_PATH_AUTO) {
        t_last_path = PSW_PATH_STAGED;
        rc = psw::solve_staged(plan, F, ldf, X, ldx, nrhs, layout, s,
                               opts ? opts->betas_left : nullptr,
                               opts ? opts->betas_right : nullptr,
                               opts ? opts->boundary_values : nullptr, ev, nev);
    } else {
        t_last_path = 0;
        psw::set_error(PSW_NOT_SUPPORTED, "unknown or retired solve path " + std::to_string(path));
        rc = PSW_NOT_SUPPORTED;
    }
    if (prev != plan->device) cudaSetDevice(prev);
    return rc;
}

int psw_solve(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
              int64_t nrhs, int layout, void* stream) {
    return psw_solve_ex(plan, F, ldf, X, ldx, nrhs, layout, stream, nullptr);
}

int psw_fill_uniform(void* dst, int dtype, int64_t count, uint64_t seed, uint64_t offset,
                     double lo, double hi, void* stream) {
    psw::clear_error();
    psw::reset_launches();
    return psw::fill_uniform(dst, dtype, count, seed, offset, lo, hi,
                             static_cast<cudaStream_t>(stream));
}

int psw_fill_normal(void* dst, int dtype, int64_t count, uint64_t seed, uint64_t offset,
                    void* stream) {
    psw::clear_error();
    psw::reset_launches();
    return psw::fill_normal(dst, dtype, count, seed, offset, static_cast<cudaStream_t>(stream));
}

int psw_l2_flush(void* scratch, int64_t bytes, void* stream) {
    psw::clear_error();
    return psw::l2_flush(scratch, bytes, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

extern "C" int psw_combine_matrix(int64_t n, const double* sub, const double* diag,
                                  const double* sup, int64_t p, const int64_t* boundaries,
                                  double* out) {
    std::vector<double> M;
    psw_plan* dummy = nullptr;
    const int rc = psw::build_plan(&dummy, n, sub, diag, sup, p, boundaries, PSW_F64, 0, 0, 1, &M);
    if (rc == PSW_OK && out) std::copy(M.begin(), M.end(), out);
    return rc;
}

// Test hook: the preliminary's tables as build_plan produced them (host
// sweeps or psw_prelim.cu, by PSW_DEVICE_SETUP), so that tests can compare
// bit patterns: gr/gl (n each: g_j on blocks j / j+1), zr/zl (p x p), max |z|
// and the plan's device_setup flag.
extern "C" int psw_debug_preliminary(int64_t n, const double* sub, const double* diag,
                                     const double* sup, int64_t p, const int64_t* boundaries,
                                     double* gr, double* gl, double* zr, double* zl,
                                     double* max_z, int32_t* device_setup) {
    psw::PrelimCapture cap;
    psw::t_capture = &cap;
    psw_plan* pl = nullptr;
    const int rc = psw::build_plan(&pl, n, sub, diag, sup, p, boundaries, PSW_F64, 0, 0, 1, nullptr,
                                   false, PSW_GROW_AUTO, PSW_PLAN_STAGED_ONLY);
    psw::t_capture = nullptr;
    if (rc != PSW_OK) return rc;
    std::copy(cap.gr.begin(), cap.gr.end(), gr);
    std::copy(cap.gl.begin(), cap.gl.end(), gl);
    std::copy(cap.zr.begin(), cap.zr.end(), zr);
    std::copy(cap.zl.begin(), cap.zl.end(), zl);
    if (max_z) *max_z = pl->info.max_z_norm;
    if (device_setup) *device_setup = pl->info.device_setup;
    psw::destroy_plan(pl);
    return PSW_OK;
}

extern "C" int psw_debug_trace(void* device_buffer) {
    psw::clear_error();
    return psw::set_trace(device_buffer);
}
