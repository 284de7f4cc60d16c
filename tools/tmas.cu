// TMA probe: 16x16 fp64 box, rows contiguous (layout S), with/without swizzle and cluster
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_0901_2859_b200/csrc/psw_tma.cuh"
using namespace psw;
__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int r0, int dynoff) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    double* dst = reinterpret_cast<double*>(sm + dynoff);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_expect_tx(&bar, 2048);
        tma_load_2d(dst, &tm, r0, 0, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[blockIdx.x * 256 + i] = dst[i];
    if (threadIdx.x == 0 && blockIdx.x == 0) printf("smem base %% 1024 = %u\n", unsigned(__cvta_generic_to_shared(sm)) & 1023u);
}
int main(int argc, char** argv) {
    int swz = atoi(argv[1]), cl = atoi(argv[2]), r0 = atoi(argv[3]), dynoff = argc > 4 ? atoi(argv[4]) : 0;
    const int n = 4096, N = 32;
    double* F; cudaMalloc(&F, sizeof(double) * n * N);
    double* h = (double*)malloc(sizeof(double) * n * N);
    for (int i = 0; i < n * N; ++i) h[i] = i;
    cudaMemcpy(F, h, sizeof(double) * n * N, cudaMemcpyHostToDevice);
    double* out; cudaMalloc(&out, sizeof(double) * 256 * 16);
    CUtensorMap tm;
    cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(N)}; cuuint64_t str[1] = {cuuint64_t(n) * 8};
    cuuint32_t box[2] = {16, 16}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, F, dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", int(r));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 8192;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    if (cl > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, tm, out, r0, dynoff);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    printf("swz %d cluster %d r0 %d dynoff %d -> %s\n", swz, cl, r0, dynoff, cudaGetErrorString(e));
    if (e) return 1;
    cudaMemcpy(h, out, sizeof(double) * 256, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 20; ++i) printf("%g ", h[i]); printf("\n");
    return 0;
}
