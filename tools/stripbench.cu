// Bandwidth of narrow column strips (W fp64 columns x all 4096 rows of the
// C1 layout, rows 32 KB apart) read by one CTA per strip: the access pattern
// of a solver that keeps a whole RHS strip on one SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/stripbench.cu -o tools/stripbench
#include <cstdio>
#include <cuda_runtime.h>

template <int W, bool COPY>
__global__ void __launch_bounds__(512) strip(const double* __restrict__ F, double* __restrict__ X, int n, int ld, double* out) {
    constexpr int SEGS = 512 / W;
    const int col = threadIdx.x % W, sg = threadIdx.x / W;
    const int L = n / SEGS;  // rows per thread
    const size_t k = size_t(blockIdx.x) * W + col;
    double s = 0;
    for (int r0 = 0; r0 < L; r0 += 32) {
        double v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = F[size_t(sg * L + r0 + r) * ld + k];
#pragma unroll
        for (int r = 0; r < 32; ++r) { s = fma(s, 0.5, v[r]); v[r] = s; }
        if (COPY) {
#pragma unroll
            for (int r = 0; r < 32; ++r) __stcs(X + size_t(sg * L + r0 + r) * ld + k, v[r]);
        }
    }
    if (s == 1.2345) out[0] = s;
}

int main() {
    const int rows = 4096, cols = 4096;
    const size_t bytes = size_t(rows) * cols * 8;
    double *F, *X, *out;
    cudaMalloc(&F, bytes);
    cudaMalloc(&X, bytes);
    cudaMalloc(&out, 8);
    cudaMemset(F, 0, bytes);
    char* flush;
    cudaMalloc(&flush, 512 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, double moved, auto launch) {
        float tot = 0;
        const int reps = 20;
        for (int it = 0; it < reps + 2; ++it) {
            cudaMemsetAsync(flush, it, 512 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 2) tot += ms;
        }
        printf("%-32s %8.2f us  %7.1f GB/s  %s\n", name, 1e3 * tot / reps, moved * reps / (tot * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("strip W=2 (16 B) read", bytes, [&] { strip<2, false><<<cols / 2, 512>>>(F, X, rows, cols, out); });
    run("strip W=4 (32 B) read", bytes, [&] { strip<4, false><<<cols / 4, 512>>>(F, X, rows, cols, out); });
    run("strip W=8 (64 B) read", bytes, [&] { strip<8, false><<<cols / 8, 512>>>(F, X, rows, cols, out); });
    run("strip W=16 (128 B) read", bytes, [&] { strip<16, false><<<cols / 16, 512>>>(F, X, rows, cols, out); });
    run("strip W=32 (256 B) read", bytes, [&] { strip<32, false><<<cols / 32, 512>>>(F, X, rows, cols, out); });
    run("strip W=4 (32 B) copy", 2 * bytes, [&] { strip<4, true><<<cols / 4, 512>>>(F, X, rows, cols, out); });
    run("strip W=8 (64 B) copy", 2 * bytes, [&] { strip<8, true><<<cols / 8, 512>>>(F, X, rows, cols, out); });
    run("strip W=16 (128 B) copy", 2 * bytes, [&] { strip<16, true><<<cols / 16, 512>>>(F, X, rows, cols, out); });
    run("strip W=32 (256 B) copy", 2 * bytes, [&] { strip<32, true><<<cols / 32, 512>>>(F, X, rows, cols, out); });
    return 0;
}
