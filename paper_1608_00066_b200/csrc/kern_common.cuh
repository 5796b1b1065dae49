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

// The launch constants of a variant (host side; no kernel is instantiated).
template <class CF>
void fill_shape(Variant& v) {
    using C = typename CF::code;
    static_assert(CF::SMEM <= 227 * 1024, "forward kernel shared memory");
    static_assert(TbCfg<CF>::SMEM <= 227 * 1024, "traceback kernel shared memory");
    static_assert(fused_smem<CF>() <= 227 * 1024, "fused kernel shared memory");
    v.K = C::K;
    v.R = C::R;
    v.W = CF::W;
    for (int r = 0; r < 4; ++r) v.polys[r] = r < C::R ? C::g(r) : 0;
    v.BPC = CF::BPC;
    v.BOXB = CF::BOXB;
    v.BPW = CF::BPW;
    v.NT = CF::NT;
    v.T = CF::T;
    v.ROW = CF::ROW;
    v.NR_TB = TbCfg<CF>::NR;
    v.TT = TbCfg<CF>::TT;
    v.NT_TB = TbCfg<CF>::NT;
    v.smem_fwd = CF::SMEM;
    v.smem_tb = TbCfg<CF>::SMEM;
    v.smem_fused = fused_smem<CF>();
    v.default_rank = 0;
    v.jit = false;
    v.k_fwd = v.k_fused = v.k_mirror = v.k_recycle = v.k_tb = nullptr;
    v.k_fwd_p = v.k_fused_p = v.k_mirror_p = v.k_recycle_p = nullptr;
    v.k_mirror_r = v.k_mirror_r_p = nullptr;
    v.prepared = 0;
}

template <class C, int W>
Variant make_variant(int rank) {
    using CF = Cfg<C, W>;
    Variant v{};
    fill_shape<CF>(v);
    v.default_rank = rank;
    v.k_fwd = reinterpret_cast<const void*>(&fwd_kernel<CF, false>);
    v.k_fused = reinterpret_cast<const void*>(&fwd_kernel<CF, true>);
    v.k_mirror = reinterpret_cast<const void*>(&fwd_kernel<CF, true, true, false>);
    v.k_mirror_r = reinterpret_cast<const void*>(&fwd_kernel<CF, true, true, true>);
    v.k_recycle = reinterpret_cast<const void*>(&fwd_kernel<CF, true, false, true>);
    v.k_fwd_p = reinterpret_cast<const void*>(&fwd_kernel<CF, false, false, false, true>);
    v.k_fused_p = reinterpret_cast<const void*>(&fwd_kernel<CF, true, false, false, true>);
    v.k_mirror_p = reinterpret_cast<const void*>(&fwd_kernel<CF, true, true, false, true>);
    v.k_mirror_r_p = reinterpret_cast<const void*>(&fwd_kernel<CF, true, true, true, true>);
    v.k_recycle_p = reinterpret_cast<const void*>(&fwd_kernel<CF, true, false, true, true>);
    v.k_tb = reinterpret_cast<const void*>(&tb_kernel<CF>);
    return v;
}

}  // namespace pbvd
