// Drop-in check of include/parsweep_b200.hpp: reference-shaped types
// (field names of parsweep::TridiagMatrix / parsweep::Partition) solved
// through parsweep::gpu::solve_batch. Reads a case written by
// tests/test_cpp_dropin.py, writes the solutions back; the Python test
// compares them with the golden reference outputs.
//   drop_in <case.bin> <out.bin>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "parsweep_b200.hpp"

namespace user {  // what a reference user already has
struct TridiagMatrix {
    std::vector<double> sub, diag, super;
};
struct Partition {
    std::size_t n = 0;
    std::vector<std::size_t> boundaries;
};
}  // namespace user

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    FILE* in = std::fopen(argv[1], "rb");
    if (!in) return 2;
    int64_t hdr[3];  // n, p, N
    if (std::fread(hdr, sizeof(int64_t), 3, in) != 3) return 2;
    const int64_t n = hdr[0], p = hdr[1], N = hdr[2];
    user::TridiagMatrix A;
    A.sub.resize(n - 1);
    A.diag.resize(n);
    A.super.resize(n - 1);
    std::vector<int64_t> b(p);
    std::vector<std::vector<double>> F(N, std::vector<double>(n));
    bool ok = std::fread(A.sub.data(), 8, n - 1, in) == size_t(n - 1) &&
              std::fread(A.diag.data(), 8, n, in) == size_t(n) &&
              std::fread(A.super.data(), 8, n - 1, in) == size_t(n - 1) &&
              std::fread(b.data(), 8, p, in) == size_t(p);
    for (auto& f : F) ok = ok && std::fread(f.data(), 8, n, in) == size_t(n);
    std::fclose(in);
    if (!ok) return 2;
    user::Partition part{static_cast<std::size_t>(n), {b.begin(), b.end()}};
    try {
        auto X = parsweep::gpu::solve_batch(A, part, F);
        // the plan-level API too: one RHS end to end
        auto plan = parsweep::gpu::compute_preliminary(A, part);
        std::vector<double> x0(n);
        parsweep::gpu::solve_with_preliminary_into(A, plan, F[0], x0);
        for (int64_t i = 0; i < n; ++i)
            if (x0[i] != X[0][i]) {
                std::fprintf(stderr, "single-RHS path differs at %lld\n", (long long)i);
                return 3;
            }
        FILE* out = std::fopen(argv[2], "wb");
        for (auto& x : X) std::fwrite(x.data(), 8, n, out);
        std::fclose(out);
        // error mapping: too many PEs (decompose.hpp:34-35)
        try {
            parsweep::gpu::decompose_boundaries(7, 4);
            return 4;
        } catch (const parsweep::gpu::TooManyPEs&) {
        }
        // invalid partition -> std::invalid_argument (partition.hpp:31-42)
        try {
            user::Partition bad{static_cast<std::size_t>(n), {1}};
            parsweep::gpu::solve_batch(A, bad, F);
            return 5;
        } catch (const std::invalid_argument&) {
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    std::printf("drop-in ok\n");
    return 0;
}
