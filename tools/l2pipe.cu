// Ceiling of a fused L2-chunk pipeline: one persistent
// cooperative kernel, phase c = { stream chunk c of F from HBM (the forward
// sweep's read), re-read chunk c - D (the back substitution's read, hoped to
// hit L2) and write chunk c - D of X }, one grid barrier per phase. Reports the
// algorithmic bandwidth (F read once + X written once) per chunk size and lag D,
// next to the same kernel with the re-read taken from a far-away address (a
// guaranteed miss: the 3s traffic pattern).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2pipe l2pipe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(1024, 2) pipe_kernel(const float4* __restrict__ F, float4* __restrict__ X,
                                               size_t chunk4, int nchunks, int D, size_t miss_off4,
                                               float* sink) {
    cg::grid_group grid = cg::this_grid();
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x, nt = size_t(gridDim.x) * blockDim.x;
    float acc = 0.f;
    for (int c = 0; c < nchunks + D; ++c) {
        if (c < nchunks) {
            const float4* f = F + size_t(c) * chunk4;
            size_t i = tid;
            for (; i + 3 * nt < chunk4; i += 4 * nt) {
                const float4 v0 = f[i], v1 = f[i + nt], v2 = f[i + 2 * nt], v3 = f[i + 3 * nt];
                acc += (v0.x + v1.y) + (v2.z + v3.w);
            }
            for (; i < chunk4; i += nt) acc += f[i].x;
        }
        if (c >= D) {
            const float4* f = F + size_t(c - D) * chunk4 + miss_off4;
            float4* x = X + size_t(c - D) * chunk4;
            size_t i = tid;
            for (; i + 3 * nt < chunk4; i += 4 * nt) {
                float4 v0 = f[i], v1 = f[i + nt], v2 = f[i + 2 * nt], v3 = f[i + 3 * nt];
                v0.x += 1.f;
                __stcs(x + i, v0);
                __stcs(x + i + nt, v1);
                __stcs(x + i + 2 * nt, v2);
                __stcs(x + i + 3 * nt, v3);
            }
            for (; i < chunk4; i += nt) __stcs(x + i, f[i]);
        }
        grid.sync();
    }
    if (acc == 123.456f) *sink = acc;
}

int main() {
    const size_t total = size_t(4) << 30;  // bytes of F used per run
    float4 *F, *X;
    float* sink;
    cudaMalloc(&F, 2 * total);
    cudaMalloc(&X, total);
    cudaMalloc(&sink, 4);
    cudaMemset(F, 0, 2 * total);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (size_t mb : {16, 32, 64}) {
        for (int D : {1, 2}) {
            for (int miss : {0, 1}) {
                size_t chunk4 = mb * (1 << 20) / 16;
                int nchunks = int(total / (mb << 20));
                size_t miss_off4 = miss ? total / 16 : 0;
                void* args[] = {&F, &X, &chunk4, &nchunks, &D, &miss_off4, &sink};
                float best = 1e9f;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(e0);
                    cudaLaunchCooperativeKernel((void*)pipe_kernel, dim3(2 * nsm), dim3(1024), args, 0, 0);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    best = ms < best ? ms : best;
                }
                cudaError_t err = cudaGetLastError();
                printf("chunk %3zu MB lag %d %s: %7.3f ms  %6.1f us/phase  algorithmic %6.0f GB/s%s\n", mb, D,
                       miss ? "re-read misses (3s)" : "re-read from L2   ", best, best * 1e3 / (nchunks + D),
                       2.0 * total / (best * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
            }
        }
    }
    return 0;
}
