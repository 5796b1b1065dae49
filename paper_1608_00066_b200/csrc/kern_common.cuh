// kern_common.cuh -- instantiation helpers for the kernel variants.
#pragma once
#include "fwd.cuh"
#include "tb.cuh"
#include "variant.h"

namespace pbvd {

template <class CF>
cudaError_t prepare_cf() {
    cudaError_t e = cudaFuncSetAttribute(fwd_kernel<CF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(CF::SMEM));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(tb_kernel<CF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(TbCfg<CF>::SMEM));
}
template <class CF>
void launch_fwd(int grid, cudaStream_t s, const FwdParams& p) {
    fwd_kernel<CF><<<grid, CF::NT, CF::SMEM, s>>>(p);
}
template <class CF>
void launch_tb(int grid, cudaStream_t s, const TbParams& p) {
    tb_kernel<CF><<<grid, TbCfg<CF>::NT, TbCfg<CF>::SMEM, s>>>(p);
}

template <class C, int W>
Variant make_variant(int rank) {
    using CF = Cfg<C, W>;
    static_assert(CF::SMEM <= 227 * 1024, "forward kernel shared memory");
    static_assert(TbCfg<CF>::SMEM <= 227 * 1024, "traceback kernel shared memory");
    Variant v{};
    v.K = C::K;
    v.R = C::R;
    v.W = W;
    for (int r = 0; r < 4; ++r) v.polys[r] = r < C::R ? C::g(r) : 0;
    v.BPC = CF::BPC;
    v.BOXB = CF::BOXB;
    v.BPW = CF::BPW;
    v.NT = CF::NT;
    v.T = CF::T;
    v.ROW = CF::ROW;
    v.NR_TB = TbCfg<CF>::NR;
    v.TT = TbCfg<CF>::TT;
    v.smem_fwd = CF::SMEM;
    v.smem_tb = TbCfg<CF>::SMEM;
    v.default_rank = rank;
    v.prepare = &prepare_cf<CF>;
    v.fwd = &launch_fwd<CF>;
    v.tb = &launch_tb<CF>;
    return v;
}

}  // namespace pbvd
