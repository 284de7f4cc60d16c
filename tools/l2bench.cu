// L2 vs HBM bandwidth probe (profiling aid): streams read-modify-write passes
// over buffers of growing size; buffers <= L2 stay resident across passes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bench l2bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rw(double* __restrict__ a, size_t n, int passes) {
    for (int p = 0; p < passes; ++p)
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
             i += size_t(gridDim.x) * blockDim.x)
            a[i] = a[i] * 1.0000001 + 1e-12;
}
__global__ void rd(const double* __restrict__ a, size_t n, int passes, double* out) {
    double s = 0;
    for (int p = 0; p < passes; ++p)
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
             i += size_t(gridDim.x) * blockDim.x)
            s += __ldcg(a + i);
    if (s == 12345.0) out[0] = s;
}
int main() {
    size_t maxb = size_t(1) << 30;
    double* a; cudaMalloc(&a, maxb); cudaMemset(a, 0, maxb);
    double* o; cudaMalloc(&o, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (size_t mb : {8, 16, 32, 48, 64, 96, 128, 256, 1024}) {
        size_t n = mb * (1 << 20) / 8;
        int passes = mb <= 128 ? 20 : 4;
        rw<<<148 * 8, 256>>>(a, n, 1);
        cudaEventRecord(e0); rw<<<148 * 8, 256>>>(a, n, passes); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double gbs_rw = 2.0 * n * 8 * passes / (ms * 1e-3) / 1e9;
        cudaEventRecord(e0); rd<<<148 * 8, 256>>>(a, n, passes, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double gbs_rd = 1.0 * n * 8 * passes / (ms * 1e-3) / 1e9;
        printf("%5zu MB: read+write %8.0f GB/s   read %8.0f GB/s\n", mb, gbs_rw, gbs_rd);
    }
    return 0;
}
