// TEST INFRASTRUCTURE ONLY — a C-ABI shim over the *unmodified* reference
// headers (/root/reference/proj/include). oracle/Makefile compiles this file
// against those headers in place (nothing is copied into the repo) and writes
// oracle/_ref/libpsw_ref.so. It serves two purposes:
//   1. pin the C restatement (psw_oracle.c) and the GPU product against the
//      reference's own outputs (tests/gen_golden.py, tests/test_oracle.py);
//   2. the CPU reference arm of bench.py (`--impl reference`, cpu_baseline).
// Signatures mirror psw_oracle.h with a `ref_` prefix.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "parsweep/core/errors.hpp"
#include "parsweep/core/thomas.hpp"
#include "parsweep/core/tridiag.hpp"
#include "parsweep/dichotomy/batch.hpp"
#include "parsweep/dichotomy/betas.hpp"
#include "parsweep/dichotomy/boundary_solve.hpp"
#include "parsweep/dichotomy/level_sets.hpp"
#include "parsweep/dichotomy/partition.hpp"
#include "parsweep/dichotomy/preliminary.hpp"
#include "parsweep/runtime/decompose.hpp"
#include "parsweep/runtime/run.hpp"
#include "parsweep/poisson/adi.hpp"
#include "parsweep/poisson/fourier.hpp"
#include "parsweep/poisson/model_problem.hpp"

namespace {

using parsweep::Partition;
using parsweep::TridiagMatrix;

thread_local std::string g_msg;

TridiagMatrix make_matrix(int64_t n, const double* sub, const double* diag, const double* sup) {
    TridiagMatrix A;
    A.sub.assign(sub, sub + (n - 1));
    A.diag.assign(diag, diag + n);
    A.super.assign(sup, sup + (n - 1));
    return A;
}

Partition make_partition(int64_t n, int64_t p, const int64_t* bnd) {
    Partition part;
    part.n = static_cast<std::size_t>(n);
    for (int64_t j = 0; j < p; ++j) part.boundaries.push_back(static_cast<std::size_t>(bnd[j]));
    return part;
}

// Error codes shared with psw_oracle.h / parsweep_b200.h.
template <class F>
int guarded(F&& body, int64_t* bad) {
    try {
        body();
        return 0;
    } catch (const parsweep::PivotBreakdown& e) {
        if (bad) *bad = static_cast<int64_t>(e.row);
        g_msg = e.what();
        return 2;
    } catch (const parsweep::TooManyPEs& e) {
        g_msg = e.what();
        return 3;
    } catch (const parsweep::NotSymmetrizable& e) {
        if (bad) *bad = static_cast<int64_t>(e.index);
        g_msg = e.what();
        return 8;
    } catch (const parsweep::OracleFallbackRequired& e) {
        g_msg = e.what();
        return 9;
    } catch (const parsweep::NonConvergence& e) {
        g_msg = e.what();
        return 11;
    } catch (const std::invalid_argument& e) {
        g_msg = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 10;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }

int ref_thomas(int64_t n, const double* sub, const double* diag, const double* sup,
               const double* f, double* x, int64_t* bad) {
    return guarded([&] {
        auto A = make_matrix(n, sub, diag, sup);
        auto r = parsweep::thomas_solve(A, std::span<const double>(f, static_cast<std::size_t>(n)));
        std::memcpy(x, r.data(), sizeof(double) * static_cast<std::size_t>(n));
    }, bad);
}

int ref_decompose(int64_t n, int64_t P, int64_t* boundaries) {
    return guarded([&] {
        auto part = parsweep::decompose(static_cast<std::size_t>(n), static_cast<std::size_t>(P))
                        .induced_partition();
        for (std::size_t j = 0; j < part.boundaries.size(); ++j)
            boundaries[j] = static_cast<int64_t>(part.boundaries[j]);
    }, nullptr);
}

int64_t ref_level_sets(int64_t p, int64_t* order, int64_t* level_off) {
    auto sets = parsweep::build_level_sets(static_cast<std::size_t>(p));
    int64_t w = 0;
    for (std::size_t l = 0; l < sets.levels.size(); ++l) {
        level_off[l] = w;
        for (auto pos : sets.levels[l]) order[w++] = static_cast<int64_t>(pos);
    }
    level_off[sets.levels.size()] = w;
    return static_cast<int64_t>(sets.levels.size());
}

int ref_preliminary_ex(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* bnd, int strategy, int* used, double* g,
                       double* zr_s, double* zl_s, double* max_z, int64_t* bad) {
    return guarded([&] {
        auto A = make_matrix(n, sub, diag, sup);
        auto part = make_partition(n, p, bnd);
        auto prelim = parsweep::compute_preliminary(A, part,
                                                    static_cast<parsweep::GRowStrategy>(strategy));
        if (used) *used = static_cast<int>(prelim.strategy_used);
        for (int64_t j = 0; j < p; ++j) {
            std::memcpy(g + j * n, prelim.at[j].g_row.data(), sizeof(double) * static_cast<std::size_t>(n));
            for (int64_t i = 0; i < p; ++i) {
                zr_s[j * p + i] = i >= j ? prelim.zr(j, i) : 0.0;
                zl_s[j * p + i] = i <= j ? prelim.zl(j, i) : 0.0;
            }
        }
        if (max_z) *max_z = prelim.max_z_norm();
    }, bad);
}

int ref_preliminary(int64_t n, const double* sub, const double* diag, const double* sup,
                    int64_t p, const int64_t* bnd, double* g, double* zr_s, double* zl_s,
                    double* max_z, int64_t* bad) {
    return ref_preliminary_ex(n, sub, diag, sup, p, bnd, 0, nullptr, g, zr_s, zl_s, max_z, bad);
}

// Solve through the reference's production entry point (batch.hpp:57-75),
// layout S (one contiguous system per RHS), with a GRowStrategy.
int ref_solve_batch_ex(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* bnd, int strategy, int64_t nrhs,
                       const double* F, int64_t ldf, double* X, int64_t ldx, int64_t* bad) {
    return guarded([&] {
        auto A = make_matrix(n, sub, diag, sup);
        auto part = make_partition(n, p, bnd);
        std::vector<std::vector<double>> series(static_cast<std::size_t>(nrhs));
        for (int64_t k = 0; k < nrhs; ++k) series[k].assign(F + k * ldf, F + k * ldf + n);
        auto sol = parsweep::solve_batch(A, part, series,
                                         static_cast<parsweep::GRowStrategy>(strategy));
        for (int64_t k = 0; k < nrhs; ++k)
            std::memcpy(X + k * ldx, sol[k].data(), sizeof(double) * static_cast<std::size_t>(n));
    }, bad);
}

int ref_solve_batch(int64_t n, const double* sub, const double* diag, const double* sup,
                    int64_t p, const int64_t* bnd, int64_t nrhs, const double* F, int64_t ldf,
                    double* X, int64_t ldx, int64_t* bad) {
    return ref_solve_batch_ex(n, sub, diag, sup, p, bnd, 0, nrhs, F, ldf, X, ldx, bad);
}

// Per-RHS intermediates of one solve: betas and boundary values.
int ref_betas_boundaries(int64_t n, const double* sub, const double* diag, const double* sup,
                         int64_t p, const int64_t* bnd, const double* f, double* left,
                         double* right, double* value, uint64_t* terms, int64_t* bad) {
    return guarded([&] {
        auto A = make_matrix(n, sub, diag, sup);
        auto part = make_partition(n, p, bnd);
        auto prelim = parsweep::compute_preliminary(A, part);
        auto b = parsweep::compute_betas(std::span<const double>(f, static_cast<std::size_t>(n)), part, prelim);
        parsweep::WorkCounters wc(1);
        auto v = parsweep::solve_boundaries(prelim, b, parsweep::serial_executor(), &wc);
        for (int64_t t = 0; t <= p; ++t) { left[t] = b.left[t]; right[t] = b.right[t]; }
        for (int64_t j = 0; j < p; ++j) value[j] = v[j];
        if (terms) *terms = wc.total_combine();
    }, bad);
}

// The as-shipped runtime (run.hpp:69-103). mode 0 = simulated, 1 = threaded.
// Writes RunStats JSON into json_out (cap bytes).
int ref_run_batch(int mode, int64_t workers, int64_t n, const double* sub, const double* diag,
                  const double* sup, int64_t p, const int64_t* bnd, int64_t nrhs, const double* F,
                  int64_t ldf, double* X, int64_t ldx, char* json_out, int64_t cap, int64_t* bad) {
    return guarded([&] {
        auto A = make_matrix(n, sub, diag, sup);
        auto part = make_partition(n, p, bnd);
        std::vector<std::vector<double>> series(static_cast<std::size_t>(nrhs));
        for (int64_t k = 0; k < nrhs; ++k) series[k].assign(F + k * ldf, F + k * ldf + n);
        auto m = mode == 0 ? parsweep::ExecMode::simulated()
                           : parsweep::ExecMode::threaded(static_cast<std::size_t>(workers));
        auto [sol, stats] = parsweep::run_batch(m, A, part, series);
        for (int64_t k = 0; k < nrhs; ++k)
            std::memcpy(X + k * ldx, sol[k].data(), sizeof(double) * static_cast<std::size_t>(n));
        auto js = stats.to_json();
        std::strncpy(json_out, js.c_str(), static_cast<std::size_t>(cap));
        if (cap > 0) json_out[cap - 1] = '\0';
    }, bad);
}

// CPU baseline driver: compute_preliminary once (timed as setup), then the
// reference per-RHS solve (batch.hpp:20-51) on `nthreads` std::threads over
// disjoint RHS slices with a shared const plan (labelled
// "harness RHS-parallel"). nthreads == 1 is the serial solve loop.
int ref_solve_rhs_parallel(int64_t n, const double* sub, const double* diag, const double* sup,
                           int64_t p, const int64_t* bnd, int64_t nrhs, const double* F,
                           int64_t ldf, double* X, int64_t ldx, int nthreads, double* setup_s,
                           double* solve_s, int64_t* bad) {
    return guarded([&] {
        auto A = make_matrix(n, sub, diag, sup);
        auto part = make_partition(n, p, bnd);
        part.validate();
        const auto t0 = std::chrono::steady_clock::now();
        const auto prelim = parsweep::compute_preliminary(A, part);
        const auto t1 = std::chrono::steady_clock::now();
        int w = nthreads < 1 ? 1 : nthreads;
        if (w > nrhs) w = static_cast<int>(nrhs > 0 ? nrhs : 1);
        const int64_t chunk = (nrhs + w - 1) / w;
        std::vector<std::exception_ptr> errs(static_cast<std::size_t>(w));
        auto body = [&](int wi) {
            try {
                std::vector<parsweep::LocalScratch> pool;
                for (int64_t k = wi * chunk; k < std::min<int64_t>(nrhs, (wi + 1) * chunk); ++k)
                    parsweep::solve_with_preliminary_into(
                        A, prelim, std::span<const double>(F + k * ldf, static_cast<std::size_t>(n)),
                        std::span<double>(X + k * ldx, static_cast<std::size_t>(n)),
                        parsweep::serial_executor(), nullptr, &pool);
            } catch (...) {
                errs[static_cast<std::size_t>(wi)] = std::current_exception();
            }
        };
        std::vector<std::thread> th;
        for (int wi = 1; wi < w; ++wi) th.emplace_back(body, wi);
        body(0);
        for (auto& t : th) t.join();
        const auto t2 = std::chrono::steady_clock::now();
        if (setup_s) *setup_s = std::chrono::duration<double>(t1 - t0).count();
        if (solve_s) *solve_s = std::chrono::duration<double>(t2 - t1).count();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    }, bad);
}

// CPU baseline with the preliminary built once: the
// reference's compute_preliminary on a WorkerPool of `workers` threads (its
// own parallel setup over boundaries, preliminary.hpp:182-195), then any
// number of solves on `nthreads` std::threads over disjoint RHS slices.
struct RefPlan {
    TridiagMatrix A;
    Partition part;
    parsweep::PreliminaryData prelim;
};

void* ref_plan_create(int64_t n, const double* sub, const double* diag, const double* sup,
                      int64_t p, const int64_t* bnd, int64_t workers, double* setup_s,
                      int64_t* bad) {
    RefPlan* out = nullptr;
    const int rc = guarded([&] {
        auto A = make_matrix(n, sub, diag, sup);
        auto part = make_partition(n, p, bnd);
        part.validate();
        parsweep::WorkerPool pool(static_cast<std::size_t>(workers < 1 ? 1 : workers));
        const auto t0 = std::chrono::steady_clock::now();
        auto prelim = parsweep::compute_preliminary(A, part, parsweep::GRowStrategy::Auto, pool);
        const auto t1 = std::chrono::steady_clock::now();
        if (setup_s) *setup_s = std::chrono::duration<double>(t1 - t0).count();
        out = new RefPlan{std::move(A), std::move(part), std::move(prelim)};
    }, bad);
    return rc == 0 ? out : nullptr;
}

int ref_plan_solve(void* h, int64_t nrhs, const double* F, int64_t ldf, double* X, int64_t ldx,
                   int nthreads, double* solve_s, int64_t* bad) {
    return guarded([&] {
        const RefPlan& rp = *static_cast<const RefPlan*>(h);
        const int64_t n = static_cast<int64_t>(rp.A.diag.size());
        int w = nthreads < 1 ? 1 : nthreads;
        if (w > nrhs) w = static_cast<int>(nrhs > 0 ? nrhs : 1);
        const int64_t chunk = (nrhs + w - 1) / w;
        std::vector<std::exception_ptr> errs(static_cast<std::size_t>(w));
        const auto t0 = std::chrono::steady_clock::now();
        auto body = [&](int wi) {
            try {
                std::vector<parsweep::LocalScratch> pool;
                for (int64_t k = wi * chunk; k < std::min<int64_t>(nrhs, (wi + 1) * chunk); ++k)
                    parsweep::solve_with_preliminary_into(
                        rp.A, rp.prelim,
                        std::span<const double>(F + k * ldf, static_cast<std::size_t>(n)),
                        std::span<double>(X + k * ldx, static_cast<std::size_t>(n)),
                        parsweep::serial_executor(), nullptr, &pool);
            } catch (...) {
                errs[static_cast<std::size_t>(wi)] = std::current_exception();
            }
        };
        std::vector<std::thread> th;
        for (int wi = 1; wi < w; ++wi) th.emplace_back(body, wi);
        body(0);
        for (auto& t : th) t.join();
        if (solve_s)
            *solve_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    }, bad);
}

void ref_plan_destroy(void* h) { delete static_cast<RefPlan*>(h); }

// ---- ADI consumer (poisson/adi.hpp), §8(f) rank 1 -----------------------
namespace {
parsweep::poisson::Grid2D make_grid(int64_t n1, int64_t n2, double h1, double h2, const double* v) {
    parsweep::poisson::Grid2D g(static_cast<std::size_t>(n1), static_cast<std::size_t>(n2), h1, h2);
    if (v) std::memcpy(g.values.data(), v, sizeof(double) * g.values.size());
    return g;
}
}  // namespace

int64_t ref_adi_iteration_bound(int64_t n, double eps) {
    return static_cast<int64_t>(parsweep::poisson::adi_iteration_bound(static_cast<std::size_t>(n), eps));
}

// AdiWorkspace(n1, n2, h1, h2, cycle, pes).parameters() -> taus[cycle]
int ref_adi_parameters(int64_t n1, int64_t n2, double h1, double h2, int64_t cycle, int64_t pes,
                       double* taus) {
    return guarded([&] {
        parsweep::poisson::AdiWorkspace ws(static_cast<std::size_t>(n1), static_cast<std::size_t>(n2),
                                           h1, h2, static_cast<std::size_t>(cycle),
                                           static_cast<std::size_t>(pes));
        for (std::size_t k = 0; k < ws.parameters().size(); ++k) taus[k] = ws.parameters()[k];
    }, nullptr);
}

// `steps` AdiIteration steps k = 0..steps-1 on u (in place)
int ref_adi_steps(int64_t n1, int64_t n2, double h1, double h2, int64_t cycle, int64_t pes,
                  const double* f, double* u, int64_t steps) {
    return guarded([&] {
        parsweep::poisson::AdiWorkspace ws(static_cast<std::size_t>(n1), static_cast<std::size_t>(n2),
                                           h1, h2, static_cast<std::size_t>(cycle),
                                           static_cast<std::size_t>(pes));
        auto fg = make_grid(n1, n2, h1, h2, f);
        auto ug = make_grid(n1, n2, h1, h2, u);
        parsweep::poisson::AdiIteration it(ws, fg);
        for (int64_t k = 0; k < steps; ++k) it.step(ug, static_cast<std::size_t>(k));
        std::memcpy(u, ug.values.data(), sizeof(double) * ug.values.size());
    }, nullptr);
}

// adi_solve(f, eps, u0, ws, serial, exact?) -> u, iterations
int ref_adi_solve(int64_t n1, int64_t n2, double h1, double h2, int64_t cycle, int64_t pes,
                  double eps, const double* f, const double* u0, const double* exact, double* u,
                  int64_t* iterations) {
    return guarded([&] {
        parsweep::poisson::AdiWorkspace ws(static_cast<std::size_t>(n1), static_cast<std::size_t>(n2),
                                           h1, h2, static_cast<std::size_t>(cycle),
                                           static_cast<std::size_t>(pes));
        auto fg = make_grid(n1, n2, h1, h2, f);
        auto ug = make_grid(n1, n2, h1, h2, u0);
        parsweep::poisson::Grid2D ex;
        if (exact) ex = make_grid(n1, n2, h1, h2, exact);
        auto r = parsweep::poisson::adi_solve(fg, eps, ug, ws, parsweep::serial_executor(),
                                              exact ? &ex : nullptr);
        std::memcpy(u, r.u.values.data(), sizeof(double) * r.u.values.size());
        *iterations = static_cast<int64_t>(r.iterations);
    }, nullptr);
}

// model_problem(n1, n2) -> f, exact
void ref_model_problem(int64_t n1, int64_t n2, double* f, double* exact) {
    auto [fg, eg] = parsweep::poisson::model_problem(static_cast<std::size_t>(n1),
                                                     static_cast<std::size_t>(n2));
    std::memcpy(f, fg.values.data(), sizeof(double) * fg.values.size());
    std::memcpy(exact, eg.values.data(), sizeof(double) * eg.values.size());
}

// ---- Fourier consumer (poisson/fourier.hpp), §8(f) rank 3 ---------------
// fourier_solve(f, FourierWorkspace(n1, n2, h1, h2, pes)) -> u; also the
// workspace's partition boundaries (p of them, *p_out)
int ref_fourier_solve(int64_t n1, int64_t n2, double h1, double h2, int64_t pes, const double* f,
                      double* u, int64_t* bnd_out, int64_t* p_out) {
    return guarded([&] {
        parsweep::poisson::FourierWorkspace ws(static_cast<std::size_t>(n1),
                                               static_cast<std::size_t>(n2), h1, h2,
                                               static_cast<std::size_t>(pes));
        auto fg = make_grid(n1, n2, h1, h2, f);
        auto ug = parsweep::poisson::fourier_solve(fg, ws);
        std::memcpy(u, ug.values.data(), sizeof(double) * ug.values.size());
        const auto& b = ws.partition().boundaries;
        *p_out = static_cast<int64_t>(b.size());
        for (std::size_t i = 0; i < b.size(); ++i) bnd_out[i] = static_cast<int64_t>(b[i]);
    }, nullptr);
}

int ref_hardware_concurrency(void) { return static_cast<int>(std::thread::hardware_concurrency()); }

}  // extern "C"
