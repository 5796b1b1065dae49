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
// in chunks of TT stages per region with cp.async.bulk (TMA engine) into an
// NBUF-deep shared-memory ring (one mbarrier per slot), so every dependent
// step of the walk is a shared-memory load instead of an HBM round trip.
//
// The walk tracks the PHYSICAL slot q of the current state (the forward
// kernel stores logical state u of stage s+1 at q = rotl_v(u, (s+1) mod v)):
// with p = s mod v, the decoded bit (state >> (v-1), Alg. 1) is
// bit p of q, and the predecessor 2*(state mod 2^{v-1}) + sp (line 225) is
// q with bit p replaced by the survivor bit sp -- no rotation per step.
// Both candidate survivor words of the predecessor are loaded one step ahead,
// so the dependent chain per step is a select and a shift, not a smem load.
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
    static constexpr int NBUF = 4;                          // ring depth (chunks)
    static constexpr int TT0 = 65536 / (NBUF * NR * ROW * 4);
    static constexpr int TT = TT0 >= 32 ? 32 : (TT0 >= 16 ? 16 : 8);
    static constexpr size_t RING = size_t(NBUF) * NR * TT * ROW * 4;
    static constexpr size_t SMEM = RING + 64;
};

template <class CF>
__device__ __forceinline__ uint32_t tb_word_index(uint32_t q, int woff) {
    if constexpr (CF::S >= 16) return uint32_t(woff) + (q >> 4);
    else return uint32_t(woff) + (q >> ilog2(CF::S));
}
template <class CF>
__device__ __forceinline__ uint32_t tb_bitpos(uint32_t q, uint32_t h) {
    if constexpr (CF::S >= 16) return 16u * h + (q & 15u);
    else {
        constexpr int LH = ilog2(CF::S / 2);
        return 16u * h + 8u * ((q >> LH) & 1u) + (q & uint32_t(CF::S / 2 - 1));
    }
}

template <class CF>
__global__ void __launch_bounds__(128) tb_kernel(const __grid_constant__ TbParams p) {
    using TC = TbCfg<CF>;
    constexpr int V = CF::V, W = CF::W, WPS = CF::WPS, BPW = CF::BPW;
    constexpr int NR = TC::NR, ROW = TC::ROW, TT = TC::TT, NBUF = TC::NBUF;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* ring = reinterpret_cast<uint32_t*>(smem);               // [NBUF][NR][TT][ROW]
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + TC::RING);

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

    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) mbar_init(smem_u32(&mbar[b]), nreg);
        fence_mbar_init();
    }
    __syncthreads();

    const int nrows = span - t0r;
    const int nchunks = (nrows + TT - 1) / TT;
    // chunk j holds rows [max(t0r, span-(j+1)TT), span-j*TT) at buffer offset
    // row - (span - (j+1)TT)
    auto issue = [&](int j) {
        const int rhi = span - j * TT;
        const int rlo = max(t0r, rhi - TT);
        const uint32_t bytes = uint32_t(rhi - rlo) * ROW * 4u;
        const int buf = j % NBUF;
        if (tid < nreg) {
            const uint32_t mb = smem_u32(&mbar[buf]);
            mbar_arrive_expect_tx(mb, bytes);
            bulk_g2s(smem_u32(ring + ((size_t(buf) * NR + tid) * TT + (rlo - (rhi - TT))) * ROW),
                     rbase + size_t(tid) * rstride + size_t(rlo) * ROW, bytes, mb);
        }
    };
    auto wait = [&](int j) {
        mbar_wait(smem_u32(&mbar[j % NBUF]), uint32_t(j / NBUF) & 1u);
    };
    // row pointer of stage s (for this thread's region and pair group)
    const int woff = g * W * WPS;
    auto rowp = [&](int s) -> const uint32_t* {
        const int j = (span - 1 - s) / TT;
        const int off = s - (span - (j + 1) * TT);
        return ring + ((size_t(j % NBUF) * NR + rloc) * TT + off) * ROW;
    };

    for (int j = 0; j < min(NBUF - 1, nchunks); ++j) issue(j);

    // physical slot of the start state at stage `span` (phase span mod v)
    const int pe = span % V;
    uint32_t q = ((uint32_t(st) << pe) | (uint32_t(st) >> (V - pe))) & uint32_t(CF::N - 1);
    int ph = (span - 1) % V;                     // phase of row s = span-1
    uint32_t acc = 0;
    uint32_t* out32 = reinterpret_cast<uint32_t*>(p.out);
    const bool words = (!edge) && p.word_out;
    uint32_t wcur = 0;

    // one step of Alg. 1 K2 at row s (phase ph): decoded bit, predecessor
    // slot, and the predecessor's survivor word from the preloaded candidates
    auto step = [&](const uint32_t* nrow, int s) {
        const uint32_t pb = 1u << ph;
        const uint32_t w0 = nrow[tb_word_index<CF>(q & ~pb, woff)];
        const uint32_t w1 = nrow[tb_word_index<CF>(q | pb, woff)];
        const uint32_t dec = (wcur >> tb_bitpos<CF>(q, uint32_t(h))) & 1u;
        acc = (acc << 1) | ((q >> ph) & 1u);
        const int eb = s - t0r;                      // emitted bit index (s < t1r)
        if (s < t1r) {
            if (words) {
                if ((eb & 31) == 0) out32[(out_bit0 + eb) >> 5] = acc;
            } else if ((eb & 7) == 0) {
                p.out[(out_bit0 + eb) >> 3] = uint8_t(acc & 0xffu);
            }
        }
        q = (q & ~pb) | (dec << ph);
        wcur = dec ? w1 : w0;
        ph = (ph == 0) ? V - 1 : ph - 1;
    };

    for (int j = 0; j < nchunks; ++j) {
        // chunk j and j+1 resident (the walk looks one row ahead)
        if (j + NBUF - 1 < nchunks) issue(j + NBUF - 1);
        wait(j);
        if (j + 1 < nchunks) wait(j + 1);
        const int rhi = span - j * TT;
        const int rlo = max(t0r, rhi - TT);
        if (active) {
            const uint32_t* row = rowp(rhi - 1);
            if (j == 0) wcur = row[tb_word_index<CF>(q, woff)];
            // the row below the chunk: next chunk's top row (any valid smem
            // address at the very bottom -- its words are never used)
            const uint32_t* below = (j + 1 < nchunks) ? rowp(rlo - 1) : row;
#pragma unroll 4
            for (int s = rhi - 1; s > rlo; --s) {
                row -= ROW;
                step(row, s);
            }
            step(below, rlo);
        }
        __syncthreads();          // slot j % NBUF free for chunk j + NBUF
    }
}

}  // namespace pbvd
