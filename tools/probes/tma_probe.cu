// Minimal check of a rank-2 [1][n] uint8 TMA row load with arbitrary start.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_1608_00066_b200/csrc/ptx.cuh"
using namespace pbvd;
struct P { CUtensorMap tm; int x; uint8_t* out; };
__global__ void k(const __grid_constant__ P p, const CUtensorMap* gtm, int use_global) {
    __shared__ __align__(1024) uint8_t buf[256];
    __shared__ __align__(8) uint64_t bar;
    uint32_t mb = smem_u32(&bar);
    if (threadIdx.x == 0) { mbar_init(mb, 1); if (use_global & 2) fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(mb, 64);
        tma_load_row(smem_u32(buf), use_global ? (const void*)gtm : (const void*)&p.tm, p.x, mb);
    }
    mbar_wait(mb, 0);
    if (threadIdx.x < 64) p.out[threadIdx.x] = buf[threadIdx.x];
}
int main() {
    void* f = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    uint8_t *src, *out; cudaMalloc(&src, 1000); cudaMalloc(&out, 64);
    uint8_t h[1000]; for (int i = 0; i < 1000; ++i) h[i] = i & 255; cudaMemcpy(src, h, 1000, cudaMemcpyHostToDevice);
    P p; p.x = 37; p.out = out;
    cuuint64_t gdim[2] = {1000, 1}, gstr[1] = {1008}; cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r = enc(&p.tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, src, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    CUtensorMap* gtm; cudaMalloc(&gtm, sizeof(CUtensorMap)); cudaMemcpy(gtm, &p.tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    for (int g = 1; g >= 0; --g) {
        k<<<1, 64>>>(p, gtm, g | 0);
        cudaError_t e = cudaDeviceSynchronize();
        uint8_t o[64]; cudaMemcpy(o, out, 64, cudaMemcpyDeviceToHost);
        printf("global=%d err=%s first=%d last=%d\n", g, cudaGetErrorString(e), o[0], o[63]);
        if (e != cudaSuccess) break;
    }
    p.x = 970;
    k<<<1, 64>>>(p, gtm, 0); cudaError_t e = cudaDeviceSynchronize();
    uint8_t o[64]; cudaMemcpy(o, out, 64, cudaMemcpyDeviceToHost);
    printf("oob: err=%s o[29]=%d o[30]=%d o[31]=%d\n", cudaGetErrorString(e), o[29], o[30], o[31]);
}
