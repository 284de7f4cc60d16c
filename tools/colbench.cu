// Read bandwidth of "column slice" access patterns on a row-major matrix
// (rows x cols doubles, 32 KB rows = the C1 layout R). Each CTA owns a
// slice of `wbytes` contiguous bytes per row and walks all rows in batches of
// `depth` rows per thread (loads in flight), like the solve kernels do.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/colbench.cu -o tools/colbench
#include <cstdio>
#include <cuda_runtime.h>

template <int DEPTH>
__global__ void slice_read(const double* __restrict__ A, int rows, int cols, int wdoubles,
                           int nslices, double* out) {
    // threads: wdoubles lanes x (blockDim / wdoubles) row groups
    const int lane = threadIdx.x % wdoubles, grp = threadIdx.x / wdoubles;
    const int ngrp = blockDim.x / wdoubles;
    double acc = 0.0;
    for (int sl = blockIdx.x; sl < nslices; sl += gridDim.x) {
        const double* base = A + size_t(sl) * wdoubles + lane;
        for (int r0 = grp * DEPTH; r0 < rows; r0 += ngrp * DEPTH) {
            double v[DEPTH];
#pragma unroll
            for (int u = 0; u < DEPTH; ++u) v[u] = __ldcs(base + size_t(r0 + u) * cols);
#pragma unroll
            for (int u = 0; u < DEPTH; ++u) acc += v[u];
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    const int rows = 4096, cols = 4096;
    double* A;
    double* out;
    cudaMalloc(&A, size_t(rows) * cols * 8);
    cudaMalloc(&out, 8);
    cudaMemset(A, 0, size_t(rows) * cols * 8);
    char* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int widths[] = {8, 16, 32, 64, 128, 256};
    for (int w : widths) {
        for (int threads : {256, 512, 1024}) {
            if (threads % w) continue;
            const int nslices = cols / w;
            for (int ctas_per_sm : {1, 2, 4}) {
                const int grid = nsm * ctas_per_sm;
                float best = 1e9f;
                for (int it = 0; it < 5; ++it) {
                    cudaMemsetAsync(flush, it, 256 << 20);
                    cudaEventRecord(e0);
                    slice_read<32><<<grid, threads>>>(A, rows, cols, w, nslices, out);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (it > 0 && ms < best) best = ms;
                }
                cudaError_t err = cudaGetLastError();
                printf("slice %5d B  threads %4d  ctas/SM %d  grid %4d : %7.1f GB/s %s\n", w * 8,
                       threads, ctas_per_sm, grid, double(rows) * cols * 8 / best / 1e6,
                       err == cudaSuccess ? "" : cudaGetErrorString(err));
            }
        }
    }
    return 0;
}
