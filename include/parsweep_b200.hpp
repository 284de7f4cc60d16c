// parsweep_b200.hpp — C++ drop-in over the C ABI (parsweep_b200.h).
//
// Mirrors the reference hot-path API of parsweep (proj/include/parsweep/):
//
//   reference                                         drop-in (namespace parsweep::gpu)
//   compute_preliminary(A, part)                      compute_preliminary(A, part) -> Plan
//     (dichotomy/preliminary.hpp:171-199)
//   solve_with_preliminary_into(A, prelim, f, out)    solve_with_preliminary_into(A, plan, f, out)
//     (dichotomy/batch.hpp:20-51)
//   solve_batch(A, part, series)                      solve_batch(A, part, series)
//     (dichotomy/batch.hpp:57-75)
//   decompose(n, p).induced_partition().boundaries    decompose_boundaries(n, p)
//     (runtime/decompose.hpp:23-47)
//   SolverError / PivotBreakdown / TooManyPEs /        same names, same fields
//   NotSymmetrizable / OracleFallbackRequired
//     (core/errors.hpp:9-62); invalid input -> std::invalid_argument
//
// The matrix and partition parameters are templates: any type with the
// reference's field names works, including parsweep::TridiagMatrix
// (.sub/.diag/.super std::vector<double>) and parsweep::Partition
// (.n, .boundaries std::vector<std::size_t>), so a reference user swaps the
// include and the namespace and keeps their data structures.
// Device-resident batches go through Plan::solve (cudaStream_t as void*).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "parsweep_b200.h"

namespace parsweep::gpu {

struct SolverError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct PivotBreakdown : SolverError {
    PivotBreakdown(std::size_t r, const std::string& msg) : SolverError(msg), row(r) {}
    std::size_t row;
};
struct TooManyPEs : SolverError {
    using SolverError::SolverError;
};
struct NotSymmetrizable : SolverError {  // core/errors.hpp:29-38
    NotSymmetrizable(std::size_t k, const std::string& msg) : SolverError(msg), index(k) {}
    std::size_t index;
};
struct OracleFallbackRequired : SolverError {  // core/errors.hpp:40-43
    using SolverError::SolverError;
};
struct NotSupported : SolverError {
    using SolverError::SolverError;
};
struct CudaError : SolverError {
    using SolverError::SolverError;
};

// Map a C-ABI status onto the reference's exception types.
inline void check(int rc) {
    if (rc == PSW_OK) return;
    const std::string msg = psw_last_error_message();
    switch (rc) {
        case PSW_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case PSW_PIVOT_BREAKDOWN:
            throw PivotBreakdown(static_cast<std::size_t>(psw_last_error_index()), msg);
        case PSW_TOO_MANY_PES: throw TooManyPEs(msg);
        case PSW_NOT_SUPPORTED: throw NotSupported(msg);
        case PSW_NOT_SYMMETRIZABLE:
            throw NotSymmetrizable(static_cast<std::size_t>(psw_last_error_index()), msg);
        case PSW_ORACLE_FALLBACK_REQUIRED: throw OracleFallbackRequired(msg);
        case PSW_OUT_OF_MEMORY: throw std::bad_alloc();
        default: throw CudaError(msg);
    }
}

inline std::vector<std::size_t> decompose_boundaries(std::size_t n, std::size_t P) {
    std::vector<int64_t> b(P > 1 ? P - 1 : 1);
    check(psw_decompose(static_cast<int64_t>(n), static_cast<int64_t>(P), b.data()));
    return {b.begin(), b.begin() + (P > 1 ? P - 1 : 0)};
}

// Device-resident preliminary data (the reference's PreliminaryData,
// dichotomy/preliminary.hpp:53-101, reduced to what the kernels read).
class Plan {
public:
    // strategy: psw_grow_strategy (the reference's GRowStrategy, preliminary.hpp:18-24)
    template <class Matrix, class PartitionT>
    Plan(const Matrix& A, const PartitionT& part, int dtype = PSW_F64, int device = 0,
         int strategy = PSW_GROW_AUTO) {
        const auto n = static_cast<int64_t>(A.diag.size());
        if (A.sub.size() + 1 != A.diag.size() || A.super.size() + 1 != A.diag.size())
            throw std::invalid_argument("TridiagMatrix: off-diagonal lengths must be n-1");
        std::vector<int64_t> b(part.boundaries.begin(), part.boundaries.end());
        if (static_cast<int64_t>(part.n) != n)
            throw std::invalid_argument("Partition order does not match the matrix");
        check(psw_plan_create_ex(&h_, n, A.sub.data(), A.diag.data(), A.super.data(),
                                 static_cast<int64_t>(b.size()), b.data(), dtype, device,
                                 strategy));
        n_ = n;
    }
    ~Plan() {
        if (h_) psw_plan_destroy(h_);
    }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
    Plan(Plan&& o) noexcept : h_(std::exchange(o.h_, nullptr)), n_(o.n_) {}
    Plan& operator=(Plan&& o) noexcept {
        std::swap(h_, o.h_);
        n_ = o.n_;
        return *this;
    }

    std::size_t n() const { return static_cast<std::size_t>(n_); }
    const psw_plan* handle() const { return h_; }
    psw_plan_info_t info() const {
        psw_plan_info_t i{};
        check(psw_plan_info(h_, &i));
        return i;
    }

    // Batched device solve (asynchronous on `stream`).
    void solve(const void* F, int64_t ldf, void* X, int64_t ldx, int64_t nrhs,
               int layout = PSW_LAYOUT_R, void* stream = nullptr) const {
        check(psw_solve(h_, F, ldf, X, ldx, nrhs, layout, stream));
    }

    // Host series in the reference's layout (one vector per system).
    std::vector<std::vector<double>> solve_series(
        const std::vector<std::vector<double>>& series) const {
        const std::size_t N = series.size();
        std::vector<double> F(N * n()), X(N * n());
        for (std::size_t k = 0; k < N; ++k) {
            if (series[k].size() != n()) throw std::invalid_argument("rhs length != n");
            std::copy(series[k].begin(), series[k].end(), F.begin() + k * n());
        }
        check(psw_solve_host(h_, F.data(), n_, X.data(), n_, static_cast<int64_t>(N),
                             PSW_LAYOUT_S));
        std::vector<std::vector<double>> out(N);
        for (std::size_t k = 0; k < N; ++k)
            out[k].assign(X.begin() + k * n(), X.begin() + (k + 1) * n());
        return out;
    }

private:
    psw_plan* h_ = nullptr;
    int64_t n_ = 0;
};

template <class Matrix, class PartitionT>
Plan compute_preliminary(const Matrix& A, const PartitionT& part, int strategy = PSW_GROW_AUTO) {
    return Plan(A, part, PSW_F64, 0, strategy);
}

// dichotomy/batch.hpp:20-51 for one host RHS (end to end through the GPU).
template <class Matrix>
void solve_with_preliminary_into(const Matrix&, const Plan& prelim, std::span<const double> f,
                                 std::span<double> out) {
    if (f.size() != prelim.n() || out.size() != prelim.n())
        throw std::invalid_argument("rhs/solution length != n");
    auto ld = static_cast<int64_t>(prelim.n());
    check(psw_solve_host(prelim.handle(), f.data(), ld, out.data(), ld, 1, PSW_LAYOUT_S));
}

// dichotomy/batch.hpp:57-75: validate, preliminary once, whole series.
template <class Matrix, class PartitionT>
std::vector<std::vector<double>> solve_batch(const Matrix& A, const PartitionT& part,
                                             const std::vector<std::vector<double>>& series) {
    std::vector<int64_t> b(part.boundaries.begin(), part.boundaries.end());
    check(psw_partition_validate(static_cast<int64_t>(part.n), static_cast<int64_t>(b.size()),
                                 b.data()));
    const Plan plan(A, part);
    return plan.solve_series(series);
}

}  // namespace parsweep::gpu
