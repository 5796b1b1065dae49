// variant.h -- registry of compiled (code, lanes) kernel variants.  Each
// kern_*.cu translation unit instantiates the forward/traceback templates for
// one code and exports its variants; the host API (pbvd.cu) only sees this
// table, so kernels of different codes compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include "params.h"

namespace pbvd {

struct Variant {
    int K, R, W;
    uint32_t polys[4];
    int BPC, BPW, NT, T, ROW, NR_TB, TT, BOXB;
    bool direct;        // reads R = 2 soft bytes with 16-bit loads: needs an even llr address
    size_t smem_fwd, smem_tb, smem_fused;
    int default_rank;   // lower = preferred default for the code
    cudaError_t (*prepare)();
    void (*fwd)(int grid, cudaStream_t, const FwdParams&);
    void (*tb)(int grid, cudaStream_t, const TbParams&);
    void (*fused)(int grid, cudaStream_t, const FwdParams&);
};

void add_variants_k3(std::vector<Variant>&);
void add_variants_k5(std::vector<Variant>&);
void add_variants_k7(std::vector<Variant>&);
void add_variants_k7r3(std::vector<Variant>&);
void add_variants_k9(std::vector<Variant>&);

const std::vector<Variant>& variants();

}  // namespace pbvd
