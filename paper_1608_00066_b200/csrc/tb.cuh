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
// with p = s mod v, the predecessor 2*(state mod 2^{v-1}) + sp (Alg. 1 line
// 225) is q with bit p replaced by the survivor bit sp -- no rotation.  The
// decoded bit of stage s (state >> (v-1), line 222) is bit p of q, which is
// exactly the survivor bit read at stage s+v: the output is the survivor-bit
// sequence delayed by v stages, so the walk shifts every survivor bit into a
// 32-bit accumulator and stores it as the output word once 32 bits are
// complete (the walk stops v stages above the decoding block's start).
// Chunks are aligned to multiples of v so full chunks run with compile-time
// phases; both candidate survivor words of the predecessor are loaded one step
// ahead, so the dependent chain per step is a select and a shift.
#pragma once
#include <cstdint>
#include <type_traits>
#include "params.h"
#include "ptx.cuh"

namespace pbvd {

template <class CF>
struct TbCfg {
    // blocks per CTA: 128, fewer for codes whose survivor rows are so wide
    // (K >= 11: 2 blocks per region, 512-byte rows) that a 3-deep ring of
    // v-row chunks for 128 blocks would not fit in 96 KB
    static constexpr bool fits(int nt) {
        return 3 * (nt / CF::BPW) * CF::V * CF::ROW * 4 <= 98304;
    }
    static constexpr int NT = fits(128) ? 128 : fits(64) ? 64 : fits(32) ? 32 : fits(16) ? 16 : 8;
    static_assert(NT >= CF::BPW, "traceback CTA holds whole regions");
    static constexpr int NR = NT / CF::BPW;                 // regions per CTA
    static constexpr int ROW = CF::ROW;                     // words per stage per region
    static constexpr int NBUF = 3;                          // ring depth (chunks)
    static constexpr int TT0 = 98304 / (NBUF * NR * ROW * 4);
    static constexpr int TTR = TT0 >= 32 ? 32 : (TT0 >= 16 ? 16 : 8);
    static constexpr int TT = (TTR / CF::V) * CF::V;        // chunk rows, a multiple of v
    static_assert(TT >= CF::V, "traceback chunk");
    static constexpr size_t RING = size_t(NBUF) * NR * TT * ROW * 4;
    static constexpr size_t SMEM = RING + 64;
    // bit of q above which the word index starts (q >> WSH selects the word)
    static constexpr int WSH = CF::S >= 16 ? 4 : ilog2(CF::S);
};

template <class CF>
__device__ __forceinline__ uint32_t tb_word_index(uint32_t q, int woff) {
    return uint32_t(woff) + (q >> TbCfg<CF>::WSH);
}
template <class CF>
__device__ __forceinline__ uint32_t tb_bitpos(uint32_t q, uint32_t hbit) {
    if constexpr (CF::S >= 16) return hbit + (q & 15u);
    else {
        constexpr int LH = ilog2(CF::S / 2);
        return hbit + 8u * ((q >> LH) & 1u) + (q & uint32_t(CF::S / 2 - 1));
    }
}

struct TbState {
    uint32_t q;        // physical slot of the current state
    uint32_t wcur;     // survivor word holding q's bit in the current row
    uint32_t acc;      // last 32 survivor bits, newest in bit 0 (per-step path)
    uint64_t acc64;    // last 64 survivor bits (cycle path)
    int cnt;           // steps until the next output word is complete
    int e;             // s - t0r - v of the current row
};

// One step at row s with compile-time phase PH: the survivor bit of q, the
// output accumulator, the predecessor slot and its survivor word (from the two
// candidates of row s-1 at nrow).
template <class CF, int PH>
__device__ __forceinline__ void tb_step(TbState& t, const uint32_t* nrow, int woff, uint32_t hbit) {
    constexpr uint32_t pb = 1u << PH;
    uint32_t w0, w1;
    if constexpr (PH >= TbCfg<CF>::WSH) {
        w0 = nrow[tb_word_index<CF>(t.q & ~pb, woff)];
        w1 = nrow[tb_word_index<CF>(t.q | pb, woff)];
    } else {
        w0 = w1 = nrow[tb_word_index<CF>(t.q, woff)];
    }
    const uint32_t dec = (t.wcur >> tb_bitpos<CF>(t.q, hbit)) & 1u;
    t.acc64 = (t.acc64 << 1) | dec;
    t.q = (t.q & ~pb) | (dec << PH);
    if constexpr (PH >= TbCfg<CF>::WSH) t.wcur = dec ? w1 : w0;
    else t.wcur = w0;
}

// the same with a runtime phase (partial chunks)
template <class CF>
__device__ __forceinline__ void tb_step_rt(TbState& t, int ph, const uint32_t* nrow, int woff,
                                           uint32_t hbit, uint32_t* out32, int64_t word0,
                                           int nwords) {
    const uint32_t pb = 1u << ph;
    const uint32_t w0 = nrow[tb_word_index<CF>(t.q & ~pb, woff)];
    const uint32_t w1 = nrow[tb_word_index<CF>(t.q | pb, woff)];
    const uint32_t dec = (t.wcur >> tb_bitpos<CF>(t.q, hbit)) & 1u;
    t.acc64 = (t.acc64 << 1) | dec;
    if ((t.e & 31) == 0 && t.e >= 0 && (t.e >> 5) < nwords)
        out32[word0 + (t.e >> 5)] = uint32_t(t.acc64);
    --t.e;
    t.q = (t.q & ~pb) | (dec << ph);
    t.wcur = dec ? w1 : w0;
}

// v steps, phases v-1 .. 0, from row `row` (phase v-1) downwards; the last
// step's predecessor row is `last_below`
template <class CF, int PH>
__device__ __forceinline__ void tb_steps(TbState& t, const uint32_t*& row,
                                         const uint32_t* last_below, int woff, uint32_t hbit) {
    const uint32_t* nrow = (PH == 0) ? last_below : row - CF::ROW;
    tb_step<CF, PH>(t, nrow, woff, hbit);
    row = nrow;
    if constexpr (PH > 0) tb_steps<CF, PH - 1>(t, row, last_below, woff, hbit);
}
// one cycle plus the output: at most one 32-bit word completes per cycle
// (v <= 8 < 32); it is the accumulator shifted back to the completing step
template <class CF>
__device__ __forceinline__ void tb_cycle(TbState& t, const uint32_t*& row,
                                         const uint32_t* last_below, int woff, uint32_t hbit,
                                         uint32_t* out32, int64_t word0, int nwords) {
    tb_steps<CF, CF::V - 1>(t, row, last_below, woff, hbit);
    const int eb = t.e, ea = t.e - CF::V;          // steps had e = eb .. ea+1
    const int w = eb >> 5;                         // floor (eb >= 0 checked below)
    if (eb >= 0 && (w << 5) > ea && w < nwords)
        out32[word0 + w] = uint32_t(t.acc64 >> ((w << 5) - ea - 1));
    t.e = ea;
}

// ---- compact walk (N <= 64, or one survivor word per pair) -----------------
// The survivor bits of ONE block at one stage form a small bit vector whose
// bit q is the survivor bit of physical slot q: for N = 64 the pair's four
// words (one 16-byte load shared by both lanes of the pair) halved by two
// PRMTs into a uint64; for one word per pair the word itself, indexed by
// tb_bitpos.  The load does not depend on the walk, so the dependent chain
// per step is only shift -> and -> bit insert.
template <class CF>
__host__ __device__ constexpr bool tb_compact() { return CF::N == 64 || CF::W * CF::WPS == 1; }
template <class CF>
using RowT = typename std::conditional<CF::N == 64, uint64_t, uint32_t>::type;

template <class CF>
__device__ __forceinline__ RowT<CF> row_bits(const uint32_t* row, int woff, uint32_t sel) {
    if constexpr (CF::N == 64) {
        const uint4 w = *reinterpret_cast<const uint4*>(row + woff);
        return (uint64_t(prmt(w.z, w.w, sel)) << 32) | prmt(w.x, w.y, sel);
    } else {
        return row[woff];
    }
}
template <class CF>
__device__ __forceinline__ uint32_t row_bit(RowT<CF> b, uint32_t q, uint32_t hbit) {
    if constexpr (CF::N == 64) return uint32_t(b >> q) & 1u;
    else return (b >> tb_bitpos<CF>(q, hbit)) & 1u;
}
// survivor bit of slot q moved to bit PH (other bits garbage): one variable
// shift (+ one constant shift), so the dependent chain per step is
// shift -> [shift] -> bit insert
template <class CF, int PH>
__device__ __forceinline__ uint32_t row_bit_at(RowT<CF> b, uint32_t q, uint32_t hbit) {
    uint32_t x;
    if constexpr (CF::N == 64) x = uint32_t(b >> q);
    else x = b >> tb_bitpos<CF>(q, hbit);
    if constexpr (PH == 0) {
        return x;
    } else {
        // funnel shift (ALU pipe, like the shift before and the insert after:
        // no cross-pipe latency on the walk's dependent chain)
        uint32_t y;
        asm("shf.l.wrap.b32 %0, %1, %1, %2;" : "=r"(y) : "r"(x), "n"(PH));
        return y;
    }
}
// the v steps of a cycle (phases v-1 .. 0): each replaces bit PH of q by the
// survivor bit it reads, so after the cycle q itself holds the cycle's v
// survivor bits in step order (bit 0 = newest) -- the output accumulator
// takes them in one shift-or per cycle (tbc_cycle), not one per step
template <class CF, int PH>
__device__ __forceinline__ void tbc_steps(TbState& t, const RowT<CF> (&b)[CF::V], uint32_t hbit) {
    const uint32_t xs = row_bit_at<CF, PH>(b[PH], t.q, hbit);
    t.q = bit_insert<1u << PH>(t.q, xs);
    if constexpr (PH > 0) tbc_steps<CF, PH - 1>(t, b, hbit);
}
template <class CF, int PH>
__device__ __forceinline__ void tbc_load(RowT<CF> (&b)[CF::V], const uint32_t* row, int woff,
                                         uint32_t sel) {
    b[PH] = row_bits<CF>(row, woff, sel);
    if constexpr (PH > 0) tbc_load<CF, PH - 1>(b, row - CF::ROW, woff, sel);
}
// v steps from row `row` (phase v-1) down, then the output word if complete
template <class CF>
__device__ __forceinline__ void tbc_cycle(TbState& t, const uint32_t* row, int woff, uint32_t sel,
                                          uint32_t hbit, uint32_t* out32, int64_t word0,
                                          int nwords) {
    RowT<CF> b[CF::V];
    tbc_load<CF, CF::V - 1>(b, row, woff, sel);
    tbc_steps<CF, CF::V - 1>(t, b, hbit);
    t.acc64 = (t.acc64 << CF::V) | t.q;
    const int eb = t.e, ea = t.e - CF::V;
    const int w = eb >> 5;
    if (eb >= 0 && (w << 5) > ea && w < nwords)
        out32[word0 + w] = uint32_t(t.acc64 >> ((w << 5) - ea - 1));
    t.e = ea;
}
template <class CF>
__device__ __forceinline__ void tbc_step_rt(TbState& t, int ph, const uint32_t* row, int woff,
                                            uint32_t sel, uint32_t hbit, uint32_t* out32,
                                            int64_t word0, int nwords) {
    const RowT<CF> b = row_bits<CF>(row, woff, sel);
    const uint32_t dec = row_bit<CF>(b, t.q, hbit);
    t.acc64 = (t.acc64 << 1) | dec;
    if ((t.e & 31) == 0 && t.e >= 0 && (t.e >> 5) < nwords)
        out32[word0 + (t.e >> 5)] = uint32_t(t.acc64);
    --t.e;
    t.q = (t.q & ~(1u << ph)) | (dec << ph);
}
// one chunk [lo, hi) of the compact walk; rows(r) = ring row of stage r
template <class CF, int TT, class RowFn>
__device__ __forceinline__ void tbc_chunk(TbState& t, int lo, int hi, int c, RowFn rows, int woff,
                                          uint32_t sel, uint32_t hbit, uint32_t* out32,
                                          int64_t word0, int nwords) {
    constexpr int V = CF::V;
    if (hi - lo == TT && lo == c * TT) {
        const uint32_t* row = rows(hi - 1);
        // unrolled: the next cycle's row loads overlap this cycle's chain
#pragma unroll
        for (int cy = 0; cy < TT / V; ++cy)
            tbc_cycle<CF>(t, row - cy * V * CF::ROW, woff, sel, hbit, out32, word0, nwords);
    } else {
        int ph = (hi - 1) % V;
        for (int s = hi - 1; s >= lo; --s) {
            tbc_step_rt<CF>(t, ph, rows(s), woff, sel, hbit, out32, word0, nwords);
            ph = (ph == 0) ? V - 1 : ph - 1;
        }
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
        st = 0;
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
        st = 0;
    }

    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) mbar_init(smem_u32(&mbar[b]), nreg);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();          // the forward grid's survivors and start states are complete
    if (!edge) {
        const int64_t i = int64_t(blockIdx.x) * TC::NT + tid;
        if (active) st = p.start[i];
    } else {
        st = p.start_edge[e];
    }

    // rows walked: [s_min, span); chunk c holds rows [c*TT, c*TT+TT) (clipped)
    const int s_min = min(span, t0r + V);
    const int c_top = (span - 1) / TT;
    const int c_bot = s_min / TT;
    const int nchunks = (s_min < span) ? c_top - c_bot + 1 : 0;
    auto chunk_rows = [&](int k, int& lo, int& hi) {        // k-th chunk walked
        const int c = c_top - k;
        lo = max(c * TT, s_min);
        hi = min(c * TT + TT, span);
    };
    auto slot_row = [&](int k, int r) -> const uint32_t* {  // row r of chunk k
        const int c = c_top - k;
        return ring + ((size_t(k % NBUF) * NR + rloc) * TT + (r - c * TT)) * ROW;
    };
    auto issue = [&](int k) {
        int lo, hi;
        chunk_rows(k, lo, hi);
        const uint32_t bytes = uint32_t(hi - lo) * ROW * 4u;
        if (tid < nreg) {
            const uint32_t mb = smem_u32(&mbar[k % NBUF]);
            const int c = c_top - k;
            mbar_arrive_expect_tx(mb, bytes);
            bulk_g2s(smem_u32(ring + ((size_t(k % NBUF) * NR + tid) * TT + (lo - c * TT)) * ROW),
                     rbase + size_t(tid) * rstride + size_t(lo) * ROW, bytes, mb);
        }
    };
    auto wait = [&](int k) { mbar_wait(smem_u32(&mbar[k % NBUF]), uint32_t(k / NBUF) & 1u); };

    for (int k = 0; k < min(NBUF - 1, nchunks); ++k) issue(k);

    // start state's physical slot at stage `span` (phase span mod v)
    const int pe = span % V;
    TbState t;
    t.q = ((uint32_t(st) << pe) | (uint32_t(st) >> (V - pe))) & uint32_t(CF::N - 1);
    // decoded bits of the top v stages come from the start state itself:
    // acc bit i = "survivor bit of stage span+i" := bit ((span+i) mod v) of q
    t.acc64 = 0;
    for (int i = V - 1; i >= 0; --i) t.acc64 = (t.acc64 << 1) | ((t.q >> ((span + i) % V)) & 1u);
    t.acc = 0;
    t.e = (span - 1) - t0r - V;
    t.cnt = 0;
    t.wcur = 0;
    const uint32_t hbit = 16u * uint32_t(h);
    const int woff = g * W * WPS;
    const int nbits = t1r - t0r;
    // words: blocks whose bits start on a 32-bit word and fill whole words
    // store aligned words; others (partial last block, unaligned output) bytes
    // (edge blocks too when their bits start on a word and fill whole words)
    const bool words = p.word_out && (!edge || (((out_bit0 | int64_t(t1r - t0r)) & 31) == 0));
    uint32_t* out32 = reinterpret_cast<uint32_t*>(p.out);
    const int64_t word0 = out_bit0 >> 5;
    const int nwords = (nbits + 31) >> 5;

    if (!words) {
        // edge blocks / unaligned output: plain per-step walk with byte stores
        // (every thread of the CTA takes part in the ring and its barriers)
        int ph = (span - 1) % V;
        uint32_t q = t.q;
        uint32_t bacc = 0;
        for (int k = 0; k < nchunks; ++k) {
            if (k + NBUF - 1 < nchunks) issue(k + NBUF - 1);
            wait(k);
            int lo, hi;
            chunk_rows(k, lo, hi);
            if (active) {
                for (int s = hi - 1; s >= lo; --s) {
                    const uint32_t* row = slot_row(k, s);
                    const uint32_t wd = row[tb_word_index<CF>(q, woff)];
                    const uint32_t dec = (wd >> tb_bitpos<CF>(q, hbit)) & 1u;
                    if (s < t1r) {
                        bacc = (bacc << 1) | ((q >> ph) & 1u);
                        const int eb = s - t0r;
                        if ((eb & 7) == 0) p.out[(out_bit0 + eb) >> 3] = uint8_t(bacc & 0xffu);
                    }
                    q = (q & ~(1u << ph)) | (dec << ph);
                    ph = (ph == 0) ? V - 1 : ph - 1;
                }
            }
            __syncthreads();
        }
        // rows below s_min: their (< v) decoded bits are still held in q
        if (active) {
            for (int s = s_min - 1; s >= t0r; --s) {
                if (s < t1r) {
                    bacc = (bacc << 1) | ((q >> ph) & 1u);
                    const int eb = s - t0r;
                    if ((eb & 7) == 0) p.out[(out_bit0 + eb) >> 3] = uint8_t(bacc & 0xffu);
                }
                ph = (ph == 0) ? V - 1 : ph - 1;
            }
        }
        return;
    }

    if constexpr (tb_compact<CF>()) {
        const uint32_t sel = h ? 0x7632u : 0x5410u;
        for (int k = 0; k < nchunks; ++k) {
            if (k + NBUF - 1 < nchunks) issue(k + NBUF - 1);
            wait(k);
            int lo, hi;
            chunk_rows(k, lo, hi);
            if (active)
                tbc_chunk<CF, TT>(t, lo, hi, c_top - k, [&](int r) { return slot_row(k, r); }, woff,
                                  sel, hbit, out32, word0, nwords);
            __syncthreads();      // slot k % NBUF free for chunk k + NBUF
        }
        return;
    }
    for (int k = 0; k < nchunks; ++k) {
        // chunk k and k+1 resident (the walk looks one row ahead)
        if (k + NBUF - 1 < nchunks) issue(k + NBUF - 1);
        wait(k);
        if (k + 1 < nchunks) wait(k + 1);
        int lo, hi;
        chunk_rows(k, lo, hi);
        if (active) {
            const uint32_t* row = slot_row(k, hi - 1);
            if (k == 0) t.wcur = row[tb_word_index<CF>(t.q, woff)];
            const uint32_t* below = (k + 1 < nchunks) ? slot_row(k + 1, lo - 1) : row;
            const int c = c_top - k;
            if (hi - lo == TT && lo == c * TT) {
                // full, v-aligned chunk: TT/v cycles with compile-time phases
#pragma unroll 1
                for (int cy = 0; cy < TT / V - 1; ++cy)
                    tb_cycle<CF>(t, row, row - V * ROW, woff, hbit, out32, word0, nwords);
                tb_cycle<CF>(t, row, below, woff, hbit, out32, word0, nwords);
            } else {
                int ph = (hi - 1) % V;
                for (int s = hi - 1; s >= lo; --s) {
                    const uint32_t* nrow = (s > lo) ? row - ROW : below;
                    tb_step_rt<CF>(t, ph, nrow, woff, hbit, out32, word0, nwords);
                    row = nrow;
                    ph = (ph == 0) ? V - 1 : ph - 1;
                }
            }
        }
        __syncthreads();          // slot k % NBUF free for chunk k + NBUF
    }
}

// ---------------------------------------------------------------------------
// Fused traceback (fwd_kernel<CF, true>): the forward warp walks its own
// blocks right after its forward pass -- one lane per block (NBL blocks per
// lane when a warp holds more than 32) -- streaming its survivor region from
// the top down through an NBUF-deep ring in the warp's (now free) shared
// memory with cp.async.bulk + mbarrier, exactly as tb_kernel does per CTA.
// The region was written by this warp moments earlier, so the rows come from
// L2; while one warp walks (latency bound), the other warps of its SM
// sub-partition keep the ALU pipes busy with their forward passes, and the
// second launch and its grid-wide dependency disappear.
#ifndef PBVD_FUSED_TT
#define PBVD_FUSED_TT 18
#endif
#ifndef PBVD_FUSED_NBUF
#define PBVD_FUSED_NBUF 3
#endif
template <class CF>
struct TbwCfg {
    static constexpr int NBUF = PBVD_FUSED_NBUF;             // ring depth (chunks)
    static constexpr int TT = CF::V * cmax(1, PBVD_FUSED_TT / CF::V);   // rows per chunk, multiple of v
    static constexpr int NBL = (CF::BPW + 31) / 32;         // blocks per lane
    static constexpr size_t RING = size_t(NBUF) * TT * CF::ROW * 4;
    static constexpr size_t SMEM = RING + 8 * NBUF;
    static constexpr int WSH = TbCfg<CF>::WSH;
};

template <class CF>
__device__ __forceinline__ void warp_traceback(uint8_t* wsm, const uint32_t* region, int span,
                                               int t0r, int t1r, int nblk,
                                               const uint32_t (&st)[TbwCfg<CF>::NBL],
                                               const int64_t (&obit)[TbwCfg<CF>::NBL], bool words,
                                               uint8_t* out, int lane,
                                               unsigned long long* dbg = nullptr) {
    using TC = TbwCfg<CF>;
    constexpr int V = CF::V, W = CF::W, WPS = CF::WPS, ROW = CF::ROW;
    constexpr int TT = TC::TT, NBUF = TC::NBUF, NBL = TC::NBL;
    uint32_t* ring = reinterpret_cast<uint32_t*>(wsm);                 // [NBUF][TT][ROW]
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wsm + TC::RING);

    __syncwarp();              // every lane is done with the forward's shared memory
    if (lane == 0) {
        for (int b = 0; b < NBUF; ++b) mbar_init(smem_u32(&mbar[b]), 1);
        fence_mbar_init();
        fence_proxy_async_all();   // survivor stores (generic) before the bulk reads
    }
    __syncwarp();

    const int s_min = min(span, t0r + V);
    const int c_top = (span - 1) / TT;
    const int c_bot = s_min / TT;
    const int nchunks = (s_min < span) ? c_top - c_bot + 1 : 0;
    auto chunk_rows = [&](int k, int& lo, int& hi) {
        const int c = c_top - k;
        lo = max(c * TT, s_min);
        hi = min(c * TT + TT, span);
    };
    auto slot_row = [&](int k, int r) -> const uint32_t* {
        const int c = c_top - k;
        return ring + (size_t(k % NBUF) * TT + (r - c * TT)) * ROW;
    };
    auto issue = [&](int k) {
        if (lane == 0) {
            int lo, hi;
            chunk_rows(k, lo, hi);
            const uint32_t bytes = uint32_t(hi - lo) * ROW * 4u;
            const uint32_t mb = smem_u32(&mbar[k % NBUF]);
            mbar_arrive_expect_tx(mb, bytes);
            bulk_g2s(smem_u32(slot_row(k, lo)), region + size_t(lo) * ROW, bytes, mb);
        }
    };
    auto wait = [&](int k) { mbar_wait(smem_u32(&mbar[k % NBUF]), uint32_t(k / NBUF) & 1u); };

    for (int k = 0; k < min(NBUF - 1, nchunks); ++k) issue(k);
    const int pe = span % V;
    const int nbits = t1r - t0r;
    const int nwords = (nbits + 31) >> 5;
    uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
    TbState t[NBL];
    bool act[NBL];
    int woff[NBL];
    uint32_t hbit[NBL];
#pragma unroll
    for (int m = 0; m < NBL; ++m) {
        const int i = lane + 32 * m;
        act[m] = i < nblk;
        woff[m] = (i >> 1) * W * WPS;
        hbit[m] = 16u * uint32_t(i & 1);
        t[m].q = ((st[m] << pe) | (st[m] >> (V - pe))) & uint32_t(CF::N - 1);
        t[m].acc64 = 0;
        for (int j = V - 1; j >= 0; --j)
            t[m].acc64 = (t[m].acc64 << 1) | ((t[m].q >> ((span + j) % V)) & 1u);
        t[m].acc = 0;
        t[m].e = (span - 1) - t0r - V;
        t[m].cnt = 0;
        t[m].wcur = 0;
    }

    if (!words) {
        // edge blocks / unaligned output: per-step walk with byte stores
        int ph0 = (span - 1) % V;
        uint32_t q[NBL], bacc[NBL];
#pragma unroll
        for (int m = 0; m < NBL; ++m) { q[m] = t[m].q; bacc[m] = 0; }
        for (int k = 0; k < nchunks; ++k) {
            if (k + NBUF - 1 < nchunks) issue(k + NBUF - 1);
            wait(k);
            int lo, hi;
            chunk_rows(k, lo, hi);
#pragma unroll
            for (int m = 0; m < NBL; ++m) {
                if (!act[m]) continue;
                int ph = ph0;
                for (int s = hi - 1; s >= lo; --s) {
                    const uint32_t* row = slot_row(k, s);
                    const uint32_t wd = row[tb_word_index<CF>(q[m], woff[m])];
                    const uint32_t dec = (wd >> tb_bitpos<CF>(q[m], hbit[m])) & 1u;
                    if (s < t1r) {
                        bacc[m] = (bacc[m] << 1) | ((q[m] >> ph) & 1u);
                        const int eb = s - t0r;
                        if ((eb & 7) == 0) out[(obit[m] + eb) >> 3] = uint8_t(bacc[m] & 0xffu);
                    }
                    q[m] = (q[m] & ~(1u << ph)) | (dec << ph);
                    ph = (ph == 0) ? V - 1 : ph - 1;
                }
            }
            ph0 = (ph0 - (hi - lo)) % V;
            if (ph0 < 0) ph0 += V;
            __syncwarp();
        }
#pragma unroll
        for (int m = 0; m < NBL; ++m) {
            if (!act[m]) continue;
            int ph = ph0;
            for (int s = s_min - 1; s >= t0r; --s) {
                if (s < t1r) {
                    bacc[m] = (bacc[m] << 1) | ((q[m] >> ph) & 1u);
                    const int eb = s - t0r;
                    if ((eb & 7) == 0) out[(obit[m] + eb) >> 3] = uint8_t(bacc[m] & 0xffu);
                }
                ph = (ph == 0) ? V - 1 : ph - 1;
            }
        }
        return;
    }

    if constexpr (tb_compact<CF>()) {
#ifdef PBVD_EXP_TIMING
        long long cw = 0, cc = 0;
#endif
        for (int k = 0; k < nchunks; ++k) {
#ifdef PBVD_EXP_TIMING
            const long long c0 = clock64();
#endif
            if (k + NBUF - 1 < nchunks) issue(k + NBUF - 1);
            wait(k);
#ifdef PBVD_EXP_TIMING
            const long long c1 = clock64();
            cw += c1 - c0;
#endif
            int lo, hi;
            chunk_rows(k, lo, hi);
#pragma unroll
            for (int m = 0; m < NBL; ++m) {
                if (!act[m]) continue;
                const uint32_t sel = hbit[m] ? 0x7632u : 0x5410u;
                tbc_chunk<CF, TT>(t[m], lo, hi, c_top - k, [&](int r) { return slot_row(k, r); },
                                  woff[m], sel, hbit[m], out32, obit[m] >> 5, nwords);
            }
#ifdef PBVD_EXP_TIMING
            cc += clock64() - c1;
            if (dbg && lane == 0 && k == nchunks - 1) { dbg[4] = cw; dbg[5] = cc; dbg[6] = nchunks; }
#endif
            __syncwarp();          // slot k % NBUF free for chunk k + NBUF
        }
        return;
    }
    for (int k = 0; k < nchunks; ++k) {
        if (k + NBUF - 1 < nchunks) issue(k + NBUF - 1);
        wait(k);
        if (k + 1 < nchunks) wait(k + 1);
        int lo, hi;
        chunk_rows(k, lo, hi);
        const int c = c_top - k;
#pragma unroll
        for (int m = 0; m < NBL; ++m) {
            if (!act[m]) continue;
            const int64_t word0 = obit[m] >> 5;
            const uint32_t* row = slot_row(k, hi - 1);
            if (k == 0) t[m].wcur = row[tb_word_index<CF>(t[m].q, woff[m])];
            const uint32_t* below = (k + 1 < nchunks) ? slot_row(k + 1, lo - 1) : row;
            if (hi - lo == TT && lo == c * TT) {
#pragma unroll 1
                for (int cy = 0; cy < TT / V - 1; ++cy)
                    tb_cycle<CF>(t[m], row, row - V * ROW, woff[m], hbit[m], out32, word0, nwords);
                tb_cycle<CF>(t[m], row, below, woff[m], hbit[m], out32, word0, nwords);
            } else {
                int ph = (hi - 1) % V;
                for (int s = hi - 1; s >= lo; --s) {
                    const uint32_t* nrow = (s > lo) ? row - ROW : below;
                    tb_step_rt<CF>(t[m], ph, nrow, woff[m], hbit[m], out32, word0, nwords);
                    row = nrow;
                    ph = (ph == 0) ? V - 1 : ph - 1;
                }
            }
        }
        __syncwarp();          // slot k % NBUF free for chunk k + NBUF
    }
}

}  // namespace pbvd
