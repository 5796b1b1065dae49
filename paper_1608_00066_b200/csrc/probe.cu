// probe.cu -- measured ACS roofline of the chip (diagnostic entry point
// pbvd_probe_acs_peak, include/pbvd.h).
//
// The roofline the forward kernel is judged against is the issue rate of the
// MINIMAL instruction sequence that produces, per state and per block, a new
// path metric and its recorded survivor bit (Eq. 1; survivor bit,
// P:258), in the same 16x2 SIMD form the kernel uses:
//     m_other = O + BM_other                       (1 add, FMA or ALU pipe)
//     PM'     = min(E + BM_own, m_other)           (1 VIADDMNMX.S16x2)
//     t       = E - m_other + (BM_own + 0x7FFF)    (1 IADD3, sign = decision)
//     + 1/2 PRMT + 7/16 LOP3 to pack 32 decisions into a word
// i.e. 3.94 instructions per packed output (= 2 ACS).  This kernel runs that
// sequence from registers only (no memory traffic, no branch metrics, no
// exchange) on every SM and reports ACS/s -- an "ACS copy-bandwidth" in the
// sense of MEASURED_PEAKS.json's hbm_gbs.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/pbvd.h"
#include "ptx.cuh"

namespace pbvd {

constexpr int PROBE_S = 32;      // packed registers per thread (as the K=7, W=2 kernel)
constexpr int PROBE_NT = 128;

__global__ void __launch_bounds__(PROBE_NT) acs_probe_kernel(int iters, uint32_t seed,
                                                             uint32_t* sink) {
    uint32_t pm[PROBE_S];
#pragma unroll
    for (int k = 0; k < PROBE_S; ++k) pm[k] = seed * (k + 1) + threadIdx.x;
    uint32_t acc = 0;
    uint32_t b0 = (seed ^ 0x00110022u) + threadIdx.x * 0x00010001u;
    uint32_t b1 = (seed ^ 0x00330044u) + threadIdx.x * 0x00030002u;
    for (int it = 0; it < iters; ++it) {
        const uint32_t c0 = b0 + 0x7FFF7FFFu, c1 = b1 + 0x7FFF7FFFu;
        uint32_t t[PROBE_S];
#pragma unroll
        for (int k = 0; k < PROBE_S / 2; ++k) {
            const uint32_t E = pm[k], O = pm[k + PROBE_S / 2];
            const uint32_t m0 = add32(O, b1);
            const uint32_t nE = __viaddmin_s16x2(E, b0, m0);
            const uint32_t tE = sub_add(E, m0, c0);
            const uint32_t m1 = add32(O, b0);
            const uint32_t nO = __viaddmin_s16x2(E, b1, m1);
            const uint32_t tO = sub_add(E, m1, c1);
            pm[k] = nE;
            pm[k + PROBE_S / 2] = nO;
            t[k] = tE;
            t[k + PROBE_S / 2] = tO;
        }
#pragma unroll
        for (int kw = 0; kw < PROBE_S / 16; ++kw) {
            uint32_t wd = prmt(t[16 * kw], t[16 * kw + 8], 0xFBD9u);
#pragma unroll
            for (int m = 1; m < 8; ++m) {
                const uint32_t pmw = prmt(t[16 * kw + m], t[16 * kw + 8 + m], 0xFBD9u);
                const uint32_t M = 0x01010101u * ((1u << m) - 1u);
                wd = (wd & M) | (pmw & ~M);
            }
            acc ^= wd;
        }
        b0 += 0x00010003u;
        b1 += 0x00050001u;
    }
    uint32_t s = acc;
#pragma unroll
    for (int k = 0; k < PROBE_S; ++k) s += pm[k];
    if (s == 0x12345678u) sink[threadIdx.x] = s;   // practically never; defeats DCE
}

// The same sequence with the forward kernel's pipe balancing: the decision
// operand of every other output is formed by two IMADs (FMA pipe) instead of
// one IADD3 (ALU pipe).  4.44 instructions per packed output.
__global__ void __launch_bounds__(PROBE_NT) acs_probe_balanced_kernel(int iters, uint32_t seed,
                                                                      uint32_t one, uint32_t neg1,
                                                                      uint32_t* sink) {
    uint32_t pm[PROBE_S];
#pragma unroll
    for (int k = 0; k < PROBE_S; ++k) pm[k] = seed * (k + 1) + threadIdx.x;
    uint32_t acc = 0;
    uint32_t b0 = (seed ^ 0x00110022u) + threadIdx.x * 0x00010001u;
    uint32_t b1 = (seed ^ 0x00330044u) + threadIdx.x * 0x00030002u;
    for (int it = 0; it < iters; ++it) {
        const uint32_t c0 = b0 + 0x7FFF7FFFu, c1 = b1 + 0x7FFF7FFFu;
        uint32_t t[PROBE_S];
#pragma unroll
        for (int k = 0; k < PROBE_S / 2; ++k) {
            const uint32_t E = pm[k], O = pm[k + PROBE_S / 2];
            const uint32_t m0 = add32(O, b1);
            const uint32_t nE = __viaddmin_s16x2(E, b0, m0);
            const uint32_t tE = sub_add(E, m0, c0);
            const uint32_t m1 = add32(O, b0);
            const uint32_t nO = __viaddmin_s16x2(E, b1, m1);
            const uint32_t tO = imad(m1, neg1, imad(E, one, c1));
            pm[k] = nE;
            pm[k + PROBE_S / 2] = nO;
            t[k] = tE;
            t[k + PROBE_S / 2] = tO;
        }
#pragma unroll
        for (int kw = 0; kw < PROBE_S / 16; ++kw) {
            uint32_t wd = prmt(t[16 * kw], t[16 * kw + 8], 0xFBD9u);
#pragma unroll
            for (int m = 1; m < 8; ++m) {
                const uint32_t pmw = prmt(t[16 * kw + m], t[16 * kw + 8 + m], 0xFBD9u);
                const uint32_t M = 0x01010101u * ((1u << m) - 1u);
                wd = (wd & M) | (pmw & ~M);
            }
            acc ^= wd;
        }
        b0 += 0x00010003u;
        b1 += 0x00050001u;
    }
    uint32_t s = acc;
#pragma unroll
    for (int k = 0; k < PROBE_S; ++k) s += pm[k];
    if (s == 0x12345678u) sink[threadIdx.x] = s;
}

}  // namespace pbvd

extern "C" int pbvd_probe_acs_balanced(int device, double* acs_per_s, double* ms_out) {
    if (!acs_per_s) return PBVD_EINVAL;
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return PBVD_ECUDA;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pbvd::acs_probe_balanced_kernel,
                                                  pbvd::PROBE_NT, 0);
    if (occ < 1) occ = 1;
    const int grid = nsm * occ;
    const int iters = 4096;
    uint32_t* sink = nullptr;
    cudaEvent_t e0, e1;
    int rc = PBVD_OK;
    if (cudaMalloc(&sink, pbvd::PROBE_NT * 4) != cudaSuccess) rc = PBVD_ENOMEM;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4 && rc == PBVD_OK; ++rep) {
        cudaEventRecord(e0);
        pbvd::acs_probe_balanced_kernel<<<grid, pbvd::PROBE_NT>>>(iters, 0x9E3779B9u + rep, 1u,
                                                                 0xffffffffu, sink);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) rc = PBVD_ECUDA;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    if (rc == PBVD_OK) {
        const double acs = double(grid) * pbvd::PROBE_NT * iters * pbvd::PROBE_S * 2.0;
        *acs_per_s = acs / (double(best) * 1e-3);
        if (ms_out) *ms_out = best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (sink) cudaFree(sink);
    if (prev >= 0) cudaSetDevice(prev);
    return rc;
}

extern "C" int pbvd_probe_acs_peak(int device, double* acs_per_s, double* ms_out) {
    if (!acs_per_s) return PBVD_EINVAL;
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return PBVD_ECUDA;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pbvd::acs_probe_kernel, pbvd::PROBE_NT, 0);
    if (occ < 1) occ = 1;
    const int grid = nsm * occ;
    const int iters = 4096;
    uint32_t* sink = nullptr;
    cudaEvent_t e0, e1;
    int rc = PBVD_OK;
    if (cudaMalloc(&sink, pbvd::PROBE_NT * 4) != cudaSuccess) rc = PBVD_ENOMEM;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4 && rc == PBVD_OK; ++rep) {
        cudaEventRecord(e0);
        pbvd::acs_probe_kernel<<<grid, pbvd::PROBE_NT>>>(iters, 0x9E3779B9u + rep, sink);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) rc = PBVD_ECUDA;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;   // rep 0 is warm-up
    }
    if (rc == PBVD_OK) {
        // ACS per launch: threads * iters * PROBE_S packed outputs * 2 blocks
        const double acs = double(grid) * pbvd::PROBE_NT * iters * pbvd::PROBE_S * 2.0;
        *acs_per_s = acs / (double(best) * 1e-3);
        if (ms_out) *ms_out = best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (sink) cudaFree(sink);
    if (prev >= 0) cudaSetDevice(prev);
    return rc;
}
