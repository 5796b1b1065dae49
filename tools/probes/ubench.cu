// ubench.cu -- issue/pipe throughput of the integer instructions the PBVD
// forward kernel is made of, on this GPU (sm_100a).  For each op: every SM
// runs WARPS warps; each thread runs ITERS iterations over 16 independent
// register chains; result = warp-instructions per SM per clock.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CH 16
#define ITERS 2048

__device__ __forceinline__ uint32_t op_iadd3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("{.reg .u32 t; sub.u32 t, %1, %2; add.u32 %0, t, %3;}" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t op_imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t op_prmt(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("prmt.b32 %0, %1, %2, 0xFBD9;" : "=r"(d) : "r"(a), "r"(b)); return d + 0 * c; }
__device__ __forceinline__ uint32_t op_lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t op_viaddmin(uint32_t a, uint32_t b, uint32_t c) { return __viaddmin_s16x2(a, b, c); }
__device__ __forceinline__ uint32_t op_vmin(uint32_t a, uint32_t b, uint32_t c) { return __vmins2(a, b) ^ c; }
__device__ __forceinline__ uint32_t op_vibmin(uint32_t a, uint32_t b, uint32_t c) {
    bool p0, p1; uint32_t d = __vibmin_s16x2(a, b, &p0, &p1); return d + (p0 ? c : 0u); }
__device__ __forceinline__ uint32_t op_vadd2(uint32_t a, uint32_t b, uint32_t c) { return __vadd2(a, b) ^ c; }
__device__ __forceinline__ uint32_t op_shf(uint32_t a, uint32_t b, uint32_t c) { return __funnelshift_r(a, b, c); }
__device__ __forceinline__ uint32_t op_shfl(uint32_t a, uint32_t b, uint32_t c) { return __shfl_xor_sync(0xffffffffu, a, 1) + 0 * b * c; }
__device__ __forceinline__ uint32_t op_vote(uint32_t a, uint32_t b, uint32_t c) { return __ballot_sync(0xffffffffu, (a & 1) != 0) ^ b; }

#define KERNEL(NAME, OP)                                                                   \
    __global__ void k_##NAME(uint32_t* out, uint32_t seed, long long* cyc) {               \
        uint32_t r[CH];                                                                    \
        uint32_t b = seed ^ threadIdx.x, c = seed * 7u + threadIdx.x;                      \
        for (int i = 0; i < CH; ++i) r[i] = seed * (i + 3) + threadIdx.x;                  \
        __syncthreads();                                                                   \
        long long t0 = clock64();                                                          \
        for (int it = 0; it < ITERS; ++it) {                                               \
            _Pragma("unroll") for (int i = 0; i < CH; ++i) r[i] = OP(r[i], b, c);           \
        }                                                                                  \
        long long t1 = clock64();                                                          \
        uint32_t s = 0;                                                                    \
        for (int i = 0; i < CH; ++i) s += r[i];                                            \
        if (s == 0x9abcdef1u) out[threadIdx.x] = s;                                        \
        if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                                   \
    }

__device__ __forceinline__ uint32_t op_addc(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("mad.lo.u32 %0, %1, 1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t op_addimm(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("add.u32 %0, %1, 0x7fff7fff;" : "=r"(d) : "r"(a)); return d; }
__device__ __forceinline__ uint32_t op_vadd2r(uint32_t a, uint32_t b, uint32_t c) { return __vadd2(a, b); }
KERNEL(addc, op_addc)
KERNEL(addimm, op_addimm)
KERNEL(vadd2r, op_vadd2r)
KERNEL(iadd3, op_iadd3)
KERNEL(imad, op_imad)
KERNEL(prmt, op_prmt)
KERNEL(lop3, op_lop3)
KERNEL(viaddmin, op_viaddmin)
KERNEL(vmin, op_vmin)
KERNEL(vibmin, op_vibmin)
KERNEL(vadd2, op_vadd2)
KERNEL(shf, op_shf)
KERNEL(shfl, op_shfl)
KERNEL(vote, op_vote)

// mixes: alternate two ops on independent chains
#define MIX(NAME, OPA, OPB)                                                                \
    __global__ void k_##NAME(uint32_t* out, uint32_t seed, long long* cyc) {               \
        uint32_t r[CH];                                                                    \
        uint32_t b = seed ^ threadIdx.x, c = seed * 7u + threadIdx.x;                      \
        for (int i = 0; i < CH; ++i) r[i] = seed * (i + 3) + threadIdx.x;                  \
        __syncthreads();                                                                   \
        long long t0 = clock64();                                                          \
        for (int it = 0; it < ITERS; ++it) {                                               \
            _Pragma("unroll") for (int i = 0; i < CH; i += 2) {                            \
                r[i] = OPA(r[i], b, c);                                                    \
                r[i + 1] = OPB(r[i + 1], b, c);                                            \
            }                                                                              \
        }                                                                                  \
        long long t1 = clock64();                                                          \
        uint32_t s = 0;                                                                    \
        for (int i = 0; i < CH; ++i) s += r[i];                                            \
        if (s == 0x9abcdef1u) out[threadIdx.x] = s;                                        \
        if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                                   \
    }
MIX(mix_viaddmin_imad, op_viaddmin, op_imad)
MIX(mix_iadd3_imad, op_iadd3, op_imad)
MIX(mix_viaddmin_iadd3, op_viaddmin, op_iadd3)
MIX(mix_prmt_imad, op_prmt, op_imad)
MIX(mix_vote_viaddmin, op_vote, op_viaddmin)
MIX(mix_vibmin_imad, op_vibmin, op_imad)
MIX(mix_addc_addimm, op_addc, op_addimm)
MIX(mix_viaddmin_addimm, op_viaddmin, op_addimm)
MIX(mix_viaddmin_addc, op_viaddmin, op_addc)
MIX(mix_imad_addimm, op_imad, op_addimm)
MIX(mix_imad_addc, op_imad, op_addc)

typedef void (*kfn)(uint32_t*, uint32_t, long long*);

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    struct { const char* name; kfn f; int ops_per_chain_iter; } ks[] = {
        {"mad a*1+b", k_addc, 1}, {"add a+imm", k_addimm, 1}, {"__vadd2 reg", k_vadd2r, 1},
        {"IADD3 (sub+add)", k_iadd3, 1}, {"IMAD (mad.lo reg)", k_imad, 1}, {"PRMT", k_prmt, 1},
        {"LOP3", k_lop3, 1}, {"VIADDMNMX.S16x2", k_viaddmin, 1}, {"VIMNMX.S16x2 (+LOP3)", k_vmin, 2},
        {"VIMNMX.S16x2 w/ preds (+SEL/IADD)", k_vibmin, 2}, {"VIADD.16x2 (+LOP3)", k_vadd2, 2},
        {"SHF funnel", k_shf, 1}, {"SHFL.BFLY", k_shfl, 1}, {"VOTE.ballot (+LOP3)", k_vote, 2},
        {"mix VIADDMNMX|IMAD", k_mix_viaddmin_imad, 1}, {"mix IADD3|IMAD", k_mix_iadd3_imad, 1},
        {"mix VIADDMNMX|IADD3", k_mix_viaddmin_iadd3, 1}, {"mix PRMT|IMAD", k_mix_prmt_imad, 1},
        {"mix VOTE|VIADDMNMX", k_mix_vote_viaddmin, 1}, {"mix VIBMIN|IMAD", k_mix_vibmin_imad, 1},
        {"mix mad1|a+imm", k_mix_addc_addimm, 1}, {"mix VIADDMNMX|a+imm", k_mix_viaddmin_addimm, 1},
        {"mix VIADDMNMX|mad1", k_mix_viaddmin_addc, 1}, {"mix IMAD|a+imm", k_mix_imad_addimm, 1},
        {"mix IMAD|mad1", k_mix_imad_addc, 1},
    };
    uint32_t* out; long long* cyc;
    cudaMalloc(&out, 4096); cudaMalloc(&cyc, sizeof(long long) * nsm * 64);
    for (int warps : {4, 8, 16}) {
        printf("== %d warps per SM (1 CTA per SM)\n", warps);
        for (auto& k : ks) {
            k.f<<<nsm, 32 * warps>>>(out, 1, cyc);
            cudaDeviceSynchronize();
            k.f<<<nsm, 32 * warps>>>(out, 2, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[1024];
            cudaMemcpy(h, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
            double avg = 0; for (int i = 0; i < nsm; ++i) avg += double(h[i]); avg /= nsm;
            const double warp_instr = double(warps) * ITERS * CH;   // per SM (chains x iters)
            printf("  %-36s %6.3f warp-instr/clk/SM  (%s)\n", k.name, warp_instr / avg, cudaGetErrorString(e));
        }
    }
    return 0;
}
