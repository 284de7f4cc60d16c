// Dependent-chain latency and throughput of FP64 / FP32 FMA on this GPU.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64lat.cu -o tools/fp64lat
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void chain(T* out, T a, T b, int iters, long long* cyc) {
    T x = out[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = fma(x, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// ILP chains per thread
template <typename T, int ILP>
__global__ void thr(T* out, T a, T b, int iters) {
    T x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = out[threadIdx.x] + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int j = 0; j < ILP; ++j) x[j] = fma(x[j], a, b);
    }
    T s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* d;
    float* f;
    long long* cyc;
    cudaMalloc(&d, 1 << 26);
    cudaMalloc(&f, 1 << 26);
    cudaMalloc(&cyc, 4096);
    cudaMemset(d, 0, 1 << 26);
    cudaMemset(f, 0, 1 << 26);
    long long h;
    const int iters = 1000;
    chain<double><<<1, 32>>>(d, 0.999, 0.001, iters, cyc);
    chain<double><<<1, 32>>>(d, 0.999, 0.001, iters, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", double(h) / (iters * 16));
    chain<float><<<1, 32>>>(f, 0.999f, 0.001f, iters, cyc);
    chain<float><<<1, 32>>>(f, 0.999f, 0.001f, iters, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("FFMA dependent latency: %.2f cycles\n", double(h) / (iters * 16));
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            const int it = 2000;
            cudaEventRecord(e0);
            for (int r = 0; r < 10; ++r) thr<double, 4><<<nsm, warps * 32>>>(d, 0.999, 0.001, it);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double fmas = 10.0 * nsm * warps * 32 * it * 8 * 4;
            if (rep) printf("DFMA throughput, %2d warps/SM, ILP 4: %.1f TFMA/s = %.1f FMA/clk/SM (at %d MHz nominal)\n",
                            warps, fmas / ms / 1e9, fmas / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
        }
    }
    return 0;
}
