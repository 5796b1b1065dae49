// variant.h -- registry of (code, lanes) kernel variants.  Each kern_*.cu
// translation unit instantiates the forward/traceback templates for one code
// and exports its variants; codes without a compiled variant are built at
// run time by jit.cu (NVRTC, same templates).  The host API (pbvd.cu) only
// sees this table: kernel entry points are plain handles launched with
// cudaLaunchKernelExC, so compiled and JIT variants are interchangeable.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "params.h"

namespace pbvd {

struct Variant {
    int K, R, W;
    uint32_t polys[4];
    int BPC, BPW, NT, T, ROW, NR_TB, TT, BOXB;
    int NT_TB;          // threads per traceback CTA
    size_t smem_fwd, smem_tb, smem_fused;
    int default_rank;   // lower = preferred default for the code
    bool jit;           // built at run time by NVRTC (jit.cu)
    // kernel entry points: a __global__ function address (compiled) or a
    // cudaKernel_t from cudaLibraryGetKernel (JIT), both accepted by
    // cudaFuncSetAttribute / cudaLaunchKernelExC
    const void* k_fwd;      // fwd_kernel<CF, false>(FwdParams)
    const void* k_fused;    // fwd_kernel<CF, true>(FwdParams)
    const void* k_mirror;   // fwd_kernel<CF, true, true, false>(FwdParams): fused + mirror copies
    const void* k_mirror_r; // fwd_kernel<CF, true, true, true>: mirror copies + recycled survivor regions
    const void* k_recycle;  // fwd_kernel<CF, true, false, true>(FwdParams): fused, recycled survivor regions
    // the same four forward kernels for punctured codes (PUNCT = true)
    const void* k_fwd_p;
    const void* k_fused_p;
    const void* k_mirror_p;
    const void* k_mirror_r_p;
    const void* k_recycle_p;
    const void* k_tb;       // tb_kernel<CF>(TbParams)
    mutable uint64_t prepared;   // per-device bit: dynamic smem attribute set
};

void add_variants_k3(std::vector<Variant>&);
void add_variants_k5(std::vector<Variant>&);
void add_variants_k7(std::vector<Variant>&);
void add_variants_k7r3(std::vector<Variant>&);
void add_variants_k9(std::vector<Variant>&);

const std::vector<Variant>& variants();

// Host-side constants of Cfg<Code<K, R, ...>, W> (they do not depend on the
// generator polynomials); false if (K, R, W) is not a supported shape.
bool variant_shape(int K, int R, int W, Variant* out);
// Default lane count of a K (the compiled variants' choice).
int default_lanes(int K);

// Run-time built variant for a code with no compiled kernel (NVRTC; cached
// in-process and on disk).  Returns nullptr and sets *err on failure.
const Variant* jit_variant(int K, int R, const uint32_t* polys, int W, std::string* err);

}  // namespace pbvd
