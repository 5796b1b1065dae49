// tb.cuh -- traceback kernel of the PBVD on sm_100a (Alg. 1 K2).
//
// One thread per block walks the survivor path from the block's start state
// (min PM; state 0 for a terminated tail) at the last forward stage
// back through the L traceback stages, emitting the D decoded bits
// packed LSB-first.  This is the second kernel of
// "different parallelism": the forward kernel spends W lanes
// on a block pair, the traceback one thread per block.
//
// Survivors of a forward warp (64/W blocks) form one region
// [stage][lane][word]; the CTA streams the rows it walks, from the top down,
// in chunks of TT stages per region with cp.async.bulk (TMA engine) into a
// double-buffered shared-memory ring (mbarrier completion), so every
// dependent step of the walk is a shared-memory load instead of an HBM
// round trip.
//
// The walk tracks the PHYSICAL slot q of the current state (the forward
// kernel stores logical state u of stage s+1 at q = rotl_v(u, (s+1) mod v)):
// with p = s mod v, the decoded bit (state >> (v-1), Alg. 1) is
// bit p of q, and the predecessor 2*(state mod 2^{v-1}) + sp (line 225) is
// q with bit p replaced by the survivor bit sp -- no rotation per step.
#pragma once
#include <cstdint>
#include "params.h"
#include "ptx.cuh"

namespace pbvd {

template <class CF>
struct TbCfg {
    static constexpr int NT = 128;                          // blocks per CTA
    static constexpr int NR = NT / CF::BPW;                 // regions per CTA
    static constexpr int ROW = CF::ROW;                     // words per stage per region
    static constexpr int TT0 = 32768 / (NR * ROW * 4);
    static constexpr int TT = TT0 >= 64 ? 64 : (TT0 >= 32 ? 32 : (TT0 >= 16 ? 16 : 8));
    static constexpr size_t SMEM = size_t(2) * NR * TT * ROW * 4 + 64;
};

template <class CF>
__global__ void __launch_bounds__(128) tb_kernel(const __grid_constant__ TbParams p) {
    using TC = TbCfg<CF>;
    constexpr int V = CF::V, S = CF::S, W = CF::W, WPS = CF::WPS, BPW = CF::BPW;
    constexpr int NR = TC::NR, ROW = TC::ROW, TT = TC::TT;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* ring = reinterpret_cast<uint32_t*>(smem);               // [2][NR][TT][ROW]
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + size_t(2) * NR * TT * ROW * 4);

    const int tid = threadIdx.x;
    const bool edge = int(blockIdx.x) >= p.n_int_ctas;
    const int e = int(blockIdx.x) - p.n_int_ctas;

    int span, t0r, t1r, nreg;
    int64_t out_bit0;
    const uint32_t* rbase;        // region 0 of this CTA
    size_t rstride;               // words between regions
    bool active;
    int g, h, rloc;
    int32_t st;
    if (!edge) {
        span = p.span_int;
        t0r = p.t0r;
        t1r = p.t1r;
        const int64_t i = int64_t(blockIdx.x) * TC::NT + tid;
        active = i < p.n_int;
        const int64_t first_region = int64_t(blockIdx.x) * NR;
        const int64_t regions_total = (int64_t(p.n_int) + BPW - 1) / BPW;
        nreg = int(min(int64_t(NR), regions_total - first_region));
        rstride = size_t(span) * ROW;
        rbase = p.dec + size_t(first_region) * rstride;
        rloc = tid / BPW;
        g = (tid % BPW) >> 1;
        h = tid & 1;
        out_bit0 = p.out_bit0 + i * p.D;
        st = active ? p.start[i] : 0;
    } else {
        span = p.edges[e].span;
        t0r = p.edges[e].t0r;
        t1r = p.edges[e].t1r;
        active = (tid == 0);
        nreg = 1;
        rstride = size_t(p.span_edge_max) * ROW;
        rbase = p.dec_edge + size_t(e) * rstride;
        rloc = 0;
        g = 0;
        h = 0;
        out_bit0 = p.edges[e].out_bit0;
        st = p.start_edge[e];
    }

    const uint32_t mb0 = smem_u32(&mbar[0]), mb1 = smem_u32(&mbar[1]);
    if (tid == 0) {
        mbar_init(mb0, nreg);
        mbar_init(mb1, nreg);
    }
    __syncthreads();

    const int nrows = span - t0r;
    const int nchunks = (nrows + TT - 1) / TT;
    auto issue = [&](int j) {
        const int rhi = span - j * TT;
        const int rlo = max(t0r, rhi - TT);
        const uint32_t bytes = uint32_t(rhi - rlo) * ROW * 4u;
        const int buf = j & 1;
        if (tid < nreg) {
            const uint32_t mb = buf ? mb1 : mb0;
            mbar_arrive_expect_tx(mb, bytes);
            bulk_g2s(smem_u32(ring + (size_t(buf) * NR + tid) * TT * ROW),
                     rbase + size_t(tid) * rstride + size_t(rlo) * ROW, bytes, mb);
        }
    };

    // physical slot of the start state at stage `span` (phase span mod v)
    const int pe = span % V;
    uint32_t q = ((uint32_t(st) << pe) | (uint32_t(st) >> (V - pe))) & uint32_t(CF::N - 1);
    int ph = (span - 1) % V;                     // phase of row s = span-1
    uint32_t acc = 0;
    const int woff = g * W * WPS;
    uint32_t* out32 = reinterpret_cast<uint32_t*>(p.out);
    const bool words = (!edge) && p.word_out;

    issue(0);
    for (int j = 0; j < nchunks; ++j) {
        if (j + 1 < nchunks) issue(j + 1);
        mbar_wait((j & 1) ? mb1 : mb0, uint32_t(j >> 1) & 1u);
        const int rhi = span - j * TT;
        const int rlo = max(t0r, rhi - TT);
        if (active) {
            const uint32_t* buf = ring + (size_t(j & 1) * NR + rloc) * TT * ROW;
            for (int s = rhi - 1; s >= rlo; --s) {
                const uint32_t* row = buf + size_t(s - rlo) * ROW + woff;
                uint32_t wd, bitpos;
                if constexpr (S >= 16) {
                    wd = row[q >> 4];
                    bitpos = 16u * h + (q & 15u);
                } else {
                    constexpr int LS = ilog2(S), LH = ilog2(S / 2);
                    wd = row[q >> LS];
                    bitpos = 16u * h + 8u * ((q >> LH) & 1u) + (q & uint32_t(S / 2 - 1));
                }
                const uint32_t dec = (wd >> bitpos) & 1u;
                if (s < t1r) {
                    acc = (acc << 1) | ((q >> ph) & 1u);
                    const int eb = s - t0r;              // emitted bit index in the block
                    if (words) {
                        if ((eb & 31) == 0) out32[(out_bit0 + eb) >> 5] = acc;
                    } else if ((eb & 7) == 0) {
                        p.out[(out_bit0 + eb) >> 3] = uint8_t(acc & 0xffu);
                    }
                }
                q = (q & ~(1u << ph)) | (dec << ph);
                ph = (ph == 0) ? V - 1 : ph - 1;
            }
        }
        __syncthreads();
    }
}

}  // namespace pbvd
