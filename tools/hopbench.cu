// Latency of one inter-CTA exchange hop through L2 with flag-in-data words
// ({lo32, flag, hi32, flag} 16-byte stores, polled by the reader), as used by
// the HOLD path's exchange. Every CTA publishes 32 doubles, then polls the
// words of a CTA half the grid away; K dependent hops are timed.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/hopbench.cu -o tools/hopbench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ll_store(uint4* p, double v, uint32_t flag) {
    const uint64_t b = __double_as_longlong(v);
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(uint32_t(b)),
                 "r"(flag), "r"(uint32_t(b >> 32)), "r"(flag)
                 : "memory");
}
__device__ __forceinline__ double ll_load(const uint4* p, uint32_t flag) {
    uint32_t a, b, c, d;
    do {
        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                     : "l"(p)
                     : "memory");
    } while (b != flag || d != flag);
    return __longlong_as_double((uint64_t(c) << 32) | a);
}

// mode 0: each CTA reads one far CTA's 32 values; mode 1: every CTA reads
// `fan` CTAs' values (a gather of fan x 32 doubles, loads issued in batches of 16)
__global__ void hop_kernel(uint4* buf, int K, int fan, double* out, long long* cycles) {
    const int b = blockIdx.x, G = gridDim.x, lane = threadIdx.x;
    double v = b + lane * 1e-3;
    const long long t0 = clock64();
    for (int it = 0; it < K; ++it) {
        ll_store(buf + (size_t(it) * G + b) * 32 + lane, v, uint32_t(it + 1));
        double acc = 0.0;
        for (int f = 0; f < fan; ++f) {
            const int src = (b + G / 2 + f) % G;
            acc += ll_load(buf + (size_t(it) * G + src) * 32 + lane, uint32_t(it + 1));
        }
        v = acc * 0.5 + 1.0;
    }
    const long long t1 = clock64();
    if (lane == 0) {
        out[b] = v;
        cycles[b] = t1 - t0;
    }
}

int main(int argc, char** argv) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int K = 2000;
    uint4* buf;
    double* out;
    long long* cyc;
    cudaMalloc(&buf, size_t(K) * nsm * 32 * 16);
    cudaMalloc(&out, nsm * 8);
    cudaMalloc(&cyc, nsm * 8);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int fan : {1, 2, 4, 16, 64, 128}) {
        cudaMemset(buf, 0, size_t(K) * nsm * 32 * 16);
        void* args[] = {&buf, (void*)&K, &fan, &out, &cyc};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)hop_kernel, dim3(nsm), dim3(32), args, 0, 0);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("fan %3d: %s  %.3f us per hop (K = %d, %d CTAs)\n", fan, cudaGetErrorString(e),
               ms * 1e3 / K, K, nsm);
        fflush(stdout);
    }
    return 0;
}
