// Micro-benchmarks of fp64/fp32 dependent-chain latencies on the target GPU
// (profiling aid for the sweep kernels).  nvcc -arch=sm_100a -o ubench ubench.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int n) {
    double a = out[0], b = out[1], c = out[2];
    float fa = float(a), fb = float(b), fc = float(c);
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) a = a + c;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) fa = fmaf(fa, fb, fc);
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) a = a * b;
    long long t4 = clock64();
    out[3] = a + fa;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}
// throughput: many independent chains per thread, many warps
__global__ void thr(double* out, int n) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b = 1.0000001, c = 1e-9;
    for (int i = 0; i < n; ++i) { a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c); }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
int main() {
    double* d; long long* c; cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 64);
    double h[4] = {1.0, 1.0000001, 1e-9, 0}; cudaMemcpy(d, h, 32, cudaMemcpyHostToDevice);
    const int n = 4096;
    lat<<<1, 1>>>(d, c, n); lat<<<1, 1>>>(d, c, n);
    long long hc[4]; cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
    printf("latency cycles/op: DFMA %.1f DADD %.1f FFMA %.1f DMUL %.1f\n", hc[0] / double(n), hc[1] / double(n), hc[2] / double(n), hc[3] / double(n));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = 148 * 8, threads = 256, it = 20000;
    thr<<<blocks, threads>>>(d, it);
    cudaEventRecord(e0); thr<<<blocks, threads>>>(d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA throughput: %.2f TFLOP/s\n", 2.0 * 4 * double(it) * blocks * threads / (ms * 1e-3) / 1e12);
    return 0;
}
