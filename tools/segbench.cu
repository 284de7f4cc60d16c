// Read bandwidth of the RESWEEP K1 access pattern on the C1 layout (4096 rows
// x 4096 fp64 RHS, row pitch 32 KB): one thread per (RHS column group,
// 32-row segment), all rows of the segment loaded at once, vs a flat stream.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/segbench.cu -o tools/segbench
#include <cstdio>
#include <cuda_runtime.h>

__global__ void flat(const double4* __restrict__ a, size_t n4, double* out) {
    double s = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) {
        double4 v = a[i];
        s += v.x + v.y + v.z + v.w;
    }
    if (s == 1.2345) out[0] = s;
}

// VEC doubles per thread (1, 2, 4); grid (cols / (VEC*threads), rows / 32)
template <int VEC>
__global__ void seg(const double* __restrict__ F, int ld, double* out) {
    const int k = (blockIdx.x * blockDim.x + threadIdx.x) * VEC;
    const int a = blockIdx.y * 32;
    double s = 0;
    if constexpr (VEC == 1) {
        double v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = F[size_t(a + r) * ld + k];
#pragma unroll
        for (int r = 0; r < 32; ++r) s = fma(s, 0.5, v[r]);
    } else if constexpr (VEC == 2) {
        double2 v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = *reinterpret_cast<const double2*>(F + size_t(a + r) * ld + k);
#pragma unroll
        for (int r = 0; r < 32; ++r) s = fma(s, 0.5, v[r].x + v[r].y);
    } else {
        double4 v[16];
        double s2 = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = *reinterpret_cast<const double4*>(F + size_t(a + h * 16 + r) * ld + k);
#pragma unroll
            for (int r = 0; r < 16; ++r) s = fma(s, 0.5, v[r].x + v[r].y + v[r].z + v[r].w);
        }
        s += s2;
    }
    if (s == 1.2345) out[0] = s;
}

// copy pattern (read + write), VEC = 1
__global__ void segcopy(const double* __restrict__ F, double* __restrict__ X, int ld) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int a = blockIdx.y * 32;
    double v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = __ldcs(F + size_t(a + r) * ld + k);
    double d = 0;
#pragma unroll
    for (int r = 0; r < 32; ++r) { d = fma(d, 0.5, v[r]); v[r] = d; }
#pragma unroll
    for (int r = 31; r >= 0; --r) __stcs(X + size_t(a + r) * ld + k, v[r]);
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
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
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
        printf("%-40s %8.2f us  %7.1f GB/s  %s\n", name, 1e3 * tot / reps, moved * reps / (tot * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int g : {1, 2, 4, 8})
        run(g == 1 ? "flat read (grid = SMs*8 x 256)" : "flat read", bytes, [&] {
            flat<<<nsm * 8 * g, 256>>>(reinterpret_cast<const double4*>(F), bytes / 32, out);
        });
    for (int th : {64, 128, 256}) {
        char nm[64];
        snprintf(nm, sizeof nm, "seg VEC=1 threads=%d", th);
        run(nm, bytes, [&] { seg<1><<<dim3(cols / th, rows / 32), th>>>(F, cols, out); });
        snprintf(nm, sizeof nm, "seg VEC=2 threads=%d", th);
        run(nm, bytes, [&] { seg<2><<<dim3(cols / (2 * th), rows / 32), th>>>(F, cols, out); });
        snprintf(nm, sizeof nm, "seg VEC=4 threads=%d", th);
        run(nm, bytes, [&] { seg<4><<<dim3(cols / (4 * th), rows / 32), th>>>(F, cols, out); });
        snprintf(nm, sizeof nm, "segcopy VEC=1 threads=%d", th);
        run(nm, 2.0 * bytes, [&] { segcopy<<<dim3(cols / th, rows / 32), th>>>(F, X, cols); });
    }
    run("cudaMemcpy D2D", 2.0 * bytes, [&] { cudaMemcpyAsync(X, F, bytes, cudaMemcpyDeviceToDevice); });
    return 0;
}
