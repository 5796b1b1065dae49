// kern_common.cuh -- instantiation helpers for the kernel variants.
#pragma once
#include "fwd.cuh"
#include "tb.cuh"
#include "variant.h"

namespace pbvd {

template <class CF>
constexpr size_t fused_smem() {
    return CF::SMEM > TbwCfg<CF>::SMEM ? CF::SMEM : ((TbwCfg<CF>::SMEM + 127) / 128) * 128;
}
template <class CF>
cudaError_t prepare_cf() {
    cudaError_t e = cudaFuncSetAttribute(fwd_kernel<CF, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(CF::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fwd_kernel<CF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(fused_smem<CF>()));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(tb_kernel<CF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(TbCfg<CF>::SMEM));
}
template <class CF>
void launch_fwd(int grid, cudaStream_t s, const FwdParams& p) {
    fwd_kernel<CF, false><<<grid, CF::NT, CF::SMEM, s>>>(p);
}
// forward + in-warp traceback in one kernel (warp_traceback, tb.cuh)
template <class CF>
void launch_fused(int grid, cudaStream_t s, const FwdParams& p) {
    fwd_kernel<CF, true><<<grid, CF::NT, fused_smem<CF>(), s>>>(p);
}
// The traceback is launched with programmatic stream serialization (PDL):
// its CTAs may be scheduled as soon as every forward CTA has signalled
// griddepcontrol.launch_dependents, and it waits (griddepcontrol.wait) for
// the forward grid's memory before touching survivors.
template <class CF>
void launch_tb(int grid, cudaStream_t s, const TbParams& p) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(TbCfg<CF>::NT);
    cfg.dynamicSmemBytes = TbCfg<CF>::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, tb_kernel<CF>, p);
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
    v.direct = CF::DIRECT;
    v.BPW = CF::BPW;
    v.NT = CF::NT;
    v.T = CF::T;
    v.ROW = CF::ROW;
    v.NR_TB = TbCfg<CF>::NR;
    v.TT = TbCfg<CF>::TT;
    v.smem_fwd = CF::SMEM;
    v.smem_tb = TbCfg<CF>::SMEM;
    v.smem_fused = fused_smem<CF>();
    v.default_rank = rank;
    v.prepare = &prepare_cf<CF>;
    v.fwd = &launch_fwd<CF>;
    v.tb = &launch_tb<CF>;
    v.fused = &launch_fused<CF>;
    return v;
}

}  // namespace pbvd
