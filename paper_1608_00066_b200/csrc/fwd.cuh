// fwd.cuh -- forward kernel of the PBVD on sm_100a: branch metrics + ACS +
// decision packing + survivor store + final argmin per block.
//
// Paper mapping (PAPER.md line numbers "P:n"):
//   ACS recursion, Eq. 1; encoder / trellis, Eq. 2 and the shift
//   S_2j,S_2j+1 -> S_j,S_{j+2^{v-1}}; butterfly outputs
//   alpha/beta/gamma/theta, Eqs. 3-6: only the 2^R distinct
//   codeword metrics of a stage are formed; survivor bit 0 =
//   upper branch; parallel-block geometry; traceback
//   start = min-PM state.
//
// B200 design (not the paper's GTX580/980 thread mapping):
//   * "block-SIMD": every 32-bit register holds the int16 path metrics of
//     ONE state for TWO blocks (lo half = even block, hi half = odd block);
//     all arithmetic is 16x2 SIMD, so BM and ACS cost is shared by a pair.
//   * W lanes of a warp hold the N states of a block pair, S = N/W states per
//     lane, all in registers.  The butterfly is done IN PLACE: at phase p
//     (stage mod v) the two inputs of a butterfly are the physical slots that
//     differ in physical bit p, and its x=0 / x=1 outputs overwrite them.
//     Logical state u lives in physical slot rotl_v(u, p) -- the index bits
//     rotate once per stage, so no data moves for register bits; when bit p
//     is a lane bit the partner values are fetched with one SHFL.BFLY per
//     register.
//   * path metrics use the non-negative biased branch metric
//     BM'(c) = BM(c) + 128R = sum_r (c_r ? lam_r + 128 : 128) in [0, 255R]
//     (a constant shift of the canonical metric, reading c-4: every decision
//     and tie is identical) and are re-normalised by the block minimum every
//     T stages, so all values stay in [0, 32767] (reading c-20) and plain
//     32-bit adds are exact 16x2 adds.
//   * ACS per output: 1 add (other candidate), 1 VIADDMNMX.S16x2 (the fused
//     add+min -- Blackwell DPX), 1 IADD3 (or 2 IMADs, FMA pipe) producing
//     m_own - m_other + 0x7FFF whose per-half sign bit is the decision
//     (m_other < m_own, tie -> upper).
//   * decisions: sign bits of 2 registers -> 4 bytes via PRMT sign-replicate,
//     8 such words merged by LOP3 into one 32-bit word (32 decisions); each
//     lane stores its WPS words of a stage straight to HBM (a warp writes
//     32*WPS contiguous words per stage, full 128-byte lines).
//   * every warp is an autonomous pipeline (no CTA barrier anywhere): it
//     copies its blocks' soft windows of the NEXT chunk with 16-byte cp.async
//     (LDGSTS) while it computes the current one, then (depunctured on the
//     fly for punctured codes) interleaves them into per-(pair, stage) words
//     of biased bytes u_r = lam_r + 128 for both blocks, read with one LDS per
//     stage one stage ahead of use and zero-extended to 16x2 by PRMT.  Shared
//     memory per warp is ~11 KB; the launch caps residency at 12 warps per SM.
#pragma once
#include <cstdint>
#include <type_traits>
#include <utility>
#include "params.h"
#include "ptx.cuh"
#include "tb.cuh"

// compile-time tunables (defaults are the measured best; DESIGN.md §7 lists
// the alternatives that were measured and removed)
#ifndef PBVD_MAXREG
#define PBVD_MAXREG 200
#endif
#ifndef PBVD_MAXREG_S64
#define PBVD_MAXREG_S64 200
#endif

namespace pbvd {

template <int K_, int R_, uint32_t G0, uint32_t G1, uint32_t G2 = 0, uint32_t G3 = 0>
struct Code {
    static constexpr int K = K_, R = R_, V = K_ - 1, N = 1 << (K_ - 1), NC = 1 << R_;
    __host__ __device__ static constexpr uint32_t g(int r) { return r == 0 ? G0 : r == 1 ? G1 : r == 2 ? G2 : G3; }
    // column i of the generator matrix, bit r = g^(r)_i
    __host__ __device__ static constexpr int col(int i) {
        int c = 0;
        for (int r = 0; r < R_; ++r) c |= int((g(r) >> i) & 1u) << r;
        return c;
    }
    static constexpr int gK = col(K_ - 1);   // beta  = alpha ^ gK       (Eq. 4)
    static constexpr int g0 = col(0);        // gamma = alpha ^ g0       (Eq. 5)
    static constexpr int ALL = (1 << R_) - 1;
    static constexpr bool symmetric = (gK == ALL) && (g0 == ALL);
};


template <class C, int W_>
struct Cfg {
    using code = C;
    static constexpr int V = C::V, N = C::N, R = C::R, NC = C::NC, W = W_;
    static constexpr int w = ilog2(W_);       // lane bits
    static constexpr int S = N / W_;          // states (registers) per lane
    static constexpr int LB = V - w;          // physical bits [0,LB) = register bits
    static constexpr int WPS = S >= 16 ? S / 16 : 1;   // decision words per lane per stage
    static constexpr int PPW = 32 / W_;       // block pairs per warp
    static constexpr int BPW = 2 * PPW;       // blocks per warp (= per survivor region)
    static constexpr int NWARP = 1;            // warps per CTA (each warp is autonomous)
    static constexpr int NT = NWARP * 32;
    // room for the unrolled stage state; 64 states per lane (K = 9 with 4
    // lanes, K = 7 with 1) hold twice the path metrics
    static constexpr int MAXREG = S >= 64 ? PBVD_MAXREG_S64 : PBVD_MAXREG;
    static constexpr int BPC = NWARP * BPW;   // blocks per CTA
    static constexpr int PPC = NWARP * PPW;   // pairs per CTA
    // int16 headroom of the biased metric BM'(c) = BM(c) + 128R in [0, 255R]
    // (reading c-4): PMs start a chunk at <= M0 = max(S_HEAD, v*128R) and grow
    // by <= 255R per stage, so after k <= T stages every PM, every E + BM and
    // every decision operand E + BM_own - m_other lies within +-(M0 + T*255R),
    // which must fit int16 (reading c-20).  T = stages per chunk = the
    // normalisation period: the largest multiple of v <= 32 that keeps it
    // (32 for every R <= 3 code; 24 for R = 4)
    static constexpr int M0 = cmax(S_HEAD, V * 128 * R);
    static constexpr int T = V * (cmin(32, (32767 - M0) / (255 * R)) / V);
    static_assert(T >= V, "normalisation period");
    static_assert(M0 + T * 255 * R <= 32767, "int16 headroom");
    // interior blocks start from all-zero metrics, so after a renormalisation
    // their metrics are within the state spread <= v*128R (no S_HEAD): when
    // v*128R + 2T*255R still fits int16 they renormalise every other chunk
    static constexpr int RN = (V * 128 * R + 2 * T * 255 * R <= 32767) ? 2 : 1;
    // raw window per block and chunk: the T*R soft bytes rounded out to
    // 16-byte vectors (+1 vector for the alignment superset)
    static constexpr int BOXB = ((T * R + 15) / 16) * 16 + 16;
    static constexpr int RAWB = ((BOXB / 16) & 1) ? BOXB : BOXB + 16;
    static constexpr int ROW = 32 * WPS;      // survivor words per stage per region
    // per (pair, stage): LW words of biased soft bytes [uA_2k, uB_2k, uA_2k+1, uB_2k+1]
    static constexpr int LW = (R + 1) / 2;
    // transform item = (pair, G stages): G*R bytes = whole words per block
    static constexpr int G = (R % 4 == 0) ? 1 : (R % 2 == 0) ? 2 : 4;
    static constexpr int NG = (T + G - 1) / G;                  // groups per chunk
    // operand row of a pair: T*LW words, padded by max(32/PPW, LW) words so
    // that the PPW rows start in distinct banks (conflict-free per-stage reads
    // across pairs) and, for LW = 2 (8-byte per-stage reads) or PPW <= 16,
    // stay 8-byte aligned
    static constexpr int LSTR = ((NG * G * LW + 31) / 32) * 32 + cmax(32 / PPW, LW);
    // per warp: raw windows [2][BPW][RAWB], operands [2][PPW][LSTR]
    static constexpr int NCYC = (T + V - 1) / V;          // cycles per chunk
    // window slot of block i in raw[.]: even blocks first, then odd
    // (h-major), so the PPW pairs' same-half windows are RAWB apart and a
    // warp's 32-bit transform reads hit 8 banks instead of 4 (a 16-byte
    // aligned window start can only reach banks = 0 mod 4)
    __host__ __device__ static constexpr int wslot(int i) {
        return (i & 1) * PPW + (i >> 1);
    }
    static constexpr size_t WRAW = size_t(2) * BPW * RAWB;         // double buffered
    static constexpr size_t WLAM = size_t(2) * PPW * LSTR * 4;   // double buffered
    static constexpr size_t WOFF = size_t(2) * BPW;                 // window byte offsets
    static constexpr size_t WPQ = ((WRAW + WLAM + WOFF + 7) / 8) * 8;   // offset of [BPW] int64 + [BPW] int
    static constexpr size_t WSMEM = ((WPQ + size_t(12) * BPW + 127) / 128) * 128;
    static constexpr size_t SMEM = NWARP * WSMEM;

    // alpha of the butterfly whose E slot has register index k, restricted
    // to the register bits (Eq. 3 on the physical->logical bit map of phase p)
    __host__ __device__ static constexpr int alpha_reg(int k, int p) {
        int a = 0;
        for (int b = 0; b < LB; ++b)
            if (b != p && ((k >> b) & 1)) a ^= C::col(((b - p) % V + V) % V);
        return a;
    }
    // R-bit mask of alpha bits a lane bit can flip at phase p
    __host__ __device__ static constexpr int lane_possible(int p) {
        int m = 0;
        for (int i = 0; i < w; ++i) {
            int b = LB + i;
            if (b != p) m |= C::col(((b - p) % V + V) % V);
        }
        return m;
    }
};

// lane part of alpha at phase p for lane-in-group lg
template <class CF, int P>
__device__ __forceinline__ int lane_alpha(int lg) {
    using C = typename CF::code;
    int a = 0;
#pragma unroll
    for (int i = 0; i < CF::w; ++i) {
        const int b = CF::LB + i;
        if (b != P && ((lg >> i) & 1)) a ^= C::col(((b - P) % CF::V + CF::V) % CF::V);
    }
    return a;
}

// biased soft bytes of one stage for a block pair (LW words, see Cfg::LW)
template <class CF>
struct XY {
    uint32_t v[CF::LW];
};

template <class CF>
__device__ __forceinline__ XY<CF> load_xy(const uint32_t* lamrow, int s) {
    XY<CF> r;
    if constexpr (CF::LW == 1) {
        r.v[0] = lamrow[s];
    } else {
        const uint2 a = *reinterpret_cast<const uint2*>(lamrow + 2 * s);
        r.v[0] = a.x; r.v[1] = a.y;
    }
    return r;
}

// Soft-value source of the ACS loop: the transformed per-pair words (lam row)
template <class CF>
struct SoftSrc {
    const uint32_t* lamrow = nullptr;
    __device__ __forceinline__ XY<CF> load(int s) const { return load_xy<CF>(lamrow, s); }
};

// The 2^R codeword metrics of one stage for a block pair, permuted by the
// lane's alpha offset: Pv[c] = BM'(c ^ flip) with the biased metric
//   BM'(c) = sum_r (c_r ? u_r : 128),  u_r = lam_r + 128 in [0, 255]
// = BM(c) + 128 R (a constant shift of the canonical metric, reading c-4).
// u_r is zero-extended to 16x2 straight from the stored bytes by PRMT; a lane
// whose alpha offset flips bit r takes (128, u_r) instead of (u_r, 128) by a
// per-lane PRMT selector (hoisted out of the loop by the compiler).
template <class CF, int POSS>
__device__ __forceinline__ void bm_vector(const XY<CF>& xy, int flip, uint32_t (&Pv)[CF::NC]) {
    constexpr int R = CF::R;
    constexpr uint32_t K128 = 0x00800080u;
    const uint32_t kb = 0x80u;                    // PRMT byte 4 = 0x80, byte 5 = 0
    uint32_t x[R], y[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t su = (r & 1) ? 0x5352u : 0x5150u;   // [u_A, 0, u_B, 0]
        if ((POSS >> r) & 1) {
            const bool f = (flip >> r) & 1;
            x[r] = prmt(xy.v[r >> 1], kb, f ? 0x5454u : su);
            y[r] = prmt(xy.v[r >> 1], kb, f ? su : 0x5454u);
        } else {
            x[r] = prmt(xy.v[r >> 1], kb, su);
            y[r] = K128;
        }
    }
#pragma unroll
    for (int c = 0; c < CF::NC; ++c) {
        uint32_t s = ((c & 1) ? x[0] : y[0]);
#pragma unroll
        for (int r = 1; r < R; ++r) s += ((c >> r) & 1) ? x[r] : y[r];
        Pv[c] = s;
    }
}

// Pack the S decision words (sign bits 15 / 31 of t[k]) into WPS words and
// store them to this lane's shared-memory row.  Bit layout of word kw:
// slot q_reg = 16*kw + (b & 15) of block half (b >> 4)   (S >= 16), or
// bit = 16*h + 8*(q_reg / (S/2)) + q_reg % (S/2)         (S < 16).
template <class CF>
__device__ __forceinline__ void pack_store(const uint32_t (&t)[CF::S], uint32_t inv,
                                           uint32_t* drow, bool st) {
    constexpr int S = CF::S, WPS = CF::WPS;
    constexpr uint32_t SEL = 0xFBD9u;   // [sgn a.b1, sgn b.b1, sgn a.b3, sgn b.b3]
    uint32_t words[WPS];
    if constexpr (S >= 16) {
#pragma unroll
        for (int kw = 0; kw < WPS; ++kw) {
            // P_m: bytes = sign of [t(m).A, t(8+m).A, t(m).B, t(8+m).B] (0x00/0xFF);
            // bit m of every byte from P_m by a chain of LOP3 merges
            uint32_t wd = prmt(t[16 * kw], t[16 * kw + 8], SEL);
#pragma unroll
            for (int m = 1; m < 8; ++m) {
                const uint32_t pm = prmt(t[16 * kw + m], t[16 * kw + 8 + m], SEL);
                const uint32_t M = 0x01010101u * ((1u << m) - 1u);
                wd = (wd & M) | (pm & ~M);
            }
            words[kw] = wd ^ inv;

        }
    } else {
        constexpr int H = S / 2;
        uint32_t wd = prmt(t[0], t[H], SEL);
#pragma unroll
        for (int m = 1; m < H; ++m) {
            const uint32_t pm = prmt(t[m], t[H + m], SEL);
            const uint32_t M = 0x01010101u * ((1u << m) - 1u);
            wd = (wd & M) | (pm & ~M);
        }
        words[0] = (wd ^ inv) & (0x01010101u * ((1u << H) - 1u));
    }
    if (!st) return;       // a row the traceback never reads (below its first row)
    // survivor stores with an L2 eviction-priority hint (the fused traceback
    // re-reads them from L2)
    const uint64_t pol = policy_evict_last_nv();
    if constexpr (WPS == 1) {
        st_global_hint(drow, words[0], pol);
    } else if constexpr (WPS == 2) {
        st_global_v2_hint(drow, words[0], words[1], pol);
    } else {
#pragma unroll
        for (int i = 0; i < WPS; i += 4)
            st_global_v4_hint(drow + i, words[i], words[i + 1], words[i + 2], words[i + 3], pol);
    }

}

// One trellis stage at compile-time phase P (Eq. 1 per output state).
// Pipe balancing: the decision operand t = E + BM_own + C - m_other is an
// IADD3 (ALU pipe) for outputs with FMA_OUT(k) false, and two IMADs (FMA
// pipe: E + (BM_own + C), then - m_other) otherwise, so the ALU pipe --
// which also carries VIADDMNMX, PRMT and LOP3 -- is not the only one busy.
template <class CF>
__host__ __device__ constexpr bool fma_out(int k) {
    return (k & 1) != 0;
}

template <class CF, int P>
__device__ __forceinline__ void acs_stage(uint32_t (&pm)[CF::S], const XY<CF>& xy, int flip,
                                          int lg, uint32_t* drow, bool st, uint32_t one,
                                          uint32_t neg1) {
    using C = typename CF::code;
    constexpr int S = CF::S, NC = CF::NC;
    constexpr int g0 = C::g0, gK = C::gK;
    uint32_t t[S];
    if constexpr (P < CF::LB) {
        // ---- butterfly partner in this lane (register bit P) --------------
        uint32_t Pv[NC], PC[NC];
        bm_vector<CF, CF::lane_possible(P)>(xy, flip, Pv);
#pragma unroll
        for (int c = 0; c < NC; ++c) PC[c] = add32(Pv[c], 0x7FFF7FFFu);
        constexpr int pb = 1 << P;
        if constexpr (NC <= 4) {
        // d-scheme: t = (E - O) + (PC_own - BM_other), the same 32-bit sum as
        // E - m_other + PC_own, with E - O shared by the butterfly's two
        // outputs and every add two-operand (either pipe): 3.5 instructions
        // per output like the IADD3/IMAD split, but free to balance the ALU and
        // FMA pipes (R = 2; for R = 3 the 8 extra per-stage constants cost
        // more than they save)
        uint32_t KC[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) KC[c] = PC[c] - Pv[c ^ g0];
#pragma unroll
        for (int k = 0; k < S; ++k) {
            if (k & pb) continue;
            const int a = CF::alpha_reg(k, P);
            const uint32_t E = pm[k], O = pm[k | pb];
            const uint32_t mO0 = add32(O, Pv[a ^ g0]);
            const uint32_t nE = __viaddmin_s16x2(E, Pv[a], mO0);
            const uint32_t mO1 = add32(O, Pv[a ^ gK ^ g0]);
            const uint32_t nO = __viaddmin_s16x2(E, Pv[a ^ gK], mO1);
            pm[k] = nE;
            pm[k | pb] = nO;
            const uint32_t d = imad(O, neg1, E);
            t[k] = add32(d, KC[a]);
            t[k | pb] = add32(d, KC[a ^ gK]);
        }
        pack_store<CF>(t, 0u, drow, st);
        return;
        }
#pragma unroll
        for (int k = 0; k < S; ++k) {
            if (k & pb) continue;
            const int a = CF::alpha_reg(k, P);
            const uint32_t E = pm[k], O = pm[k | pb];
            // x = 0: min(E + BM(alpha), O + BM(gamma))        (Eqs. 3, 5)
            const uint32_t mO0 = add32(O, Pv[a ^ g0]);
            const uint32_t nE = __viaddmin_s16x2(E, Pv[a], mO0);
            const uint32_t tE = sub_add(E, mO0, PC[a]);
            // x = 1: min(E + BM(beta), O + BM(theta))         (Eqs. 4, 6)
            const uint32_t mO1 = add32(O, Pv[a ^ gK ^ g0]);
            const uint32_t nO = __viaddmin_s16x2(E, Pv[a ^ gK], mO1);
            uint32_t tO;
            if constexpr (fma_out<CF>(1)) tO = imad(mO1, neg1, imad(E, one, PC[a ^ gK]));
            else tO = sub_add(E, mO1, PC[a ^ gK]);
            pm[k] = nE;
            pm[k | pb] = nO;
            t[k] = tE;
            t[k | pb] = tO;
        }
        pack_store<CF>(t, 0u, drow, st);
    } else {
        // ---- butterfly partner in lane lg ^ (1 << li) ----------------------
        constexpr int li = P - CF::LB;
        const uint32_t lb = uint32_t(lg >> li) & 1u;   // 0: E side (x=0), 1: O side (x=1)
        uint32_t recv[S];
#pragma unroll
        for (int k = 0; k < S; ++k) recv[k] = __shfl_xor_sync(0xffffffffu, pm[k], 1 << li);
        uint32_t Po[NC], Pr[NC], PCo[NC];
        const uint32_t Cc = 0x7FFF7FFFu + lb * 0x00010001u;   // inverted sense on O side
        if constexpr (C::symmetric) {
            // own: alpha (E side) / theta = alpha (O side); other: gamma = beta = ~alpha
            bm_vector<CF, CF::lane_possible(P)>(xy, flip, Po);
#pragma unroll
            for (int c = 0; c < NC; ++c) Pr[c] = Po[c ^ C::ALL];
        } else {
            const int fo = flip ^ (lb ? (gK ^ g0) : 0);
            const int fr = flip ^ (lb ? gK : g0);
            bm_vector<CF, CF::lane_possible(P) | (gK ^ g0)>(xy, fo, Po);
            bm_vector<CF, CF::lane_possible(P) | gK | g0>(xy, fr, Pr);
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) PCo[c] = add32(Po[c], Cc);
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const int a = CF::alpha_reg(k, P);
            const uint32_t own = pm[k];
            const uint32_t mR = add32(recv[k], Pr[a]);
            pm[k] = __viaddmin_s16x2(own, Po[a], mR);
            if (fma_out<CF>(k)) t[k] = imad(mR, neg1, imad(own, one, PCo[a]));
            else t[k] = sub_add(own, mR, PCo[a]);
        }
        pack_store<CF>(t, 0u - lb, drow, st);
    }
}

// v stages at phases P..v-1, the operands of stage P+1 loaded one stage ahead
// (one basic block: the scheduler overlaps stage P+1's loads and branch
// metrics with stage P's butterflies).
template <class CF, int P, bool FULL>
struct Cycle {
    static __device__ __forceinline__ void run(uint32_t (&pm)[CF::S], const SoftSrc<CF>& src,
                                               const int (&flip)[CF::V], int lg, uint32_t* drow,
                                               int s0, int nst, bool st, const XY<CF>& cur,
                                               uint32_t one, uint32_t neg1) {
        if constexpr (P < CF::V) {
            XY<CF> nxt = cur;
            if constexpr (P + 1 < CF::V) {
                if (FULL || s0 + P + 1 < nst) nxt = src.load(s0 + P + 1);
            }
            // drow: this cycle's first survivor row (stage s0), so each
            // stage's store address is a compile-time offset from it
            acs_stage<CF, P>(pm, cur, flip[P], lg, drow + P * CF::ROW, st, one, neg1);
            if constexpr (P + 1 < CF::V) {
                if (FULL || s0 + P + 1 < nst)
                    Cycle<CF, P + 1, FULL>::run(pm, src, flip, lg, drow, s0, nst, st, nxt, one,
                                                neg1);
            }
        }
    }
};

template <class CF, int... Ps>
__device__ __forceinline__ void init_flips(int (&flip)[CF::V], int lg,
                                           std::integer_sequence<int, Ps...>) {
    ((flip[Ps] = lane_alpha<CF, Ps>(lg)), ...);
}

__device__ __forceinline__ int64_t kept_before(const FwdParams& p, int64_t s, int R) {
    if (p.P == 1) return s * R;
    // floor division: the erasure pad of the first interior block may start
    // before stage 0 (those bytes are outside the window and zero-filled)
    int64_t q = s / p.P;
    int r = int(s - q * p.P);
    if (r < 0) { r += p.P; --q; }
    return q * p.kp + p.cum[r];
}

// MIRROR (fused only): after its walk each warp also copies its decoded bytes
// to the p.mirror destinations (the multi-GPU gather, pbvd_decode_blocks_mirrored);
// RECYCLE (fused only): interior jobs share p.n_regions survivor regions
// (streams larger than the workspace).  Separate instantiations, so the
// default kernel carries none of that code (measured: the recycling code
// alone costs the default kernel ~0.8 %, 8 more registers).
// PUNCT: punctured codes (P > 1): the soft windows are depunctured inside the
// transform slices; a separate instantiation so the dense kernels carry none
// of that code (a run-time split of the cycle loop cost them 0.4-0.8 %).
template <class CF, bool FUSED, bool MIRROR = false, bool RECYCLE = MIRROR, bool PUNCT = false>
__global__ void __launch_bounds__(CF::NT) __maxnreg__(CF::MAXREG) fwd_kernel(const __grid_constant__ FwdParams p) {
    constexpr int V = CF::V, N = CF::N, S = CF::S, W = CF::W, R = CF::R, T = CF::T;
    constexpr int BPW = CF::BPW, PPW = CF::PPW, ROW = CF::ROW, RAWB = CF::RAWB;
    constexpr int LW = CF::LW, G = CF::G, NG = CF::NG, LSTR = CF::LSTR;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* wbase = smem + size_t(warp) * CF::WSMEM;
    uint8_t* raw = wbase;                                                   // [2][BPW][RAWB]
    uint32_t* lam = reinterpret_cast<uint32_t*>(wbase + CF::WRAW);          // [2][PPW][LSTR]
    uint8_t* woffs = wbase + CF::WRAW + CF::WLAM;                           // [2][BPW]
    int64_t* pq_s = reinterpret_cast<int64_t*>(wbase + CF::WPQ);            // [BPW] (punctured codes)
    int* pr_s = reinterpret_cast<int*>(wbase + CF::WPQ + 8 * BPW);          // [BPW]

    // warp unit: interior warps first (BPW consecutive interior blocks), then
    // one unit per edge block (all lane groups replicate that block)
    if (PUNCT != (p.P != 1)) __trap();         // the host picks the instantiation by P
    const int64_t gw = int64_t(blockIdx.x) * CF::NWARP + warp;
    const bool edge = gw >= p.n_int_warps;
    const int e = int(gw - p.n_int_warps);
    if (edge && e >= p.n_edge) return;
#ifdef PBVD_EXP_TIMING
    auto gtime = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
    if (p.dbg && lane == 0) {
        unsigned smid; asm("mov.u32 %0, %%smid;" : "=r"(smid));
        p.dbg[32 * gw + 0] = gtime();
        p.dbg[32 * gw + 3] = smid;
        unsigned wid; asm("mov.u32 %0, %%warpid;" : "=r"(wid));
        p.dbg[32 * gw + 7] = wid;
    }
#endif
    const int span = edge ? p.edges[e].span : p.span_int;
    // first survivor row any traceback reads (tb.cuh: s_min = t0r + v)
    const int s_read = min(span, (edge ? p.edges[e].t0r : p.t0r) + V);
    const int nchunks = (span + T - 1) / T;
    const int64_t wb0 = gw * BPW;              // launch-relative first interior block

    auto block_lo = [&](int i) -> int64_t {
        if (edge) return p.edges[e].lo;
        int64_t bi = wb0 + i;
        if (bi >= p.n_int) bi = p.n_int - 1;
        return (p.b_int0 + bi) * p.D - p.L - p.pad;
    };
    const int nblk = edge ? 1 : BPW;
    const uintptr_t vlo = reinterpret_cast<uintptr_t>(p.llr);
    const uintptr_t vhi = vlo + uintptr_t(p.n_llr);
    // lane blocks i = lane + 32 m; punctured codes: each block's position in
    // the puncture period, split once per job (the only 64-bit division) and
    // kept in shared memory, so a chunk's kept index needs 32-bit arithmetic
    // only (the per-chunk 64-bit divisions cost C3 2 %)
    constexpr int NBL_L = (BPW + 31) / 32;
    if constexpr (PUNCT) {
#pragma unroll
        for (int m = 0; m < NBL_L; ++m) {
            const int i = lane + 32 * m;
            if (i < nblk) {
                const int64_t lo = block_lo(i);
                int64_t q = lo / p.P;
                int r = int(lo - q * p.P);
                if (r < 0) { r += p.P; --q; }   // floor (the first block's front pad may start before 0)
                pq_s[i] = q;
                pr_s[i] = r;
            }
        }
    }
    // kept index (relative to the launch window) of stage s0 >= 0 of lane block i
    // (only lane i's own entries are read: no barrier needed)
    auto kept_at = [&](int i, int s0) -> int64_t {
        if constexpr (!PUNCT) {
            return (block_lo(i) + s0) * R - p.kb_ws0;
        } else {
            const unsigned u = unsigned(pr_s[i] + s0);
            const unsigned q = u / unsigned(p.P);
            const unsigned r = u - q * unsigned(p.P);
            return (pq_s[i] + int64_t(q)) * p.kp + p.cum[r] - p.kb_ws0;
        }
    };

    // 16-byte cp.async of chunk c's soft windows: lane i copies block i's
    // window (rounded out to 16-byte vectors) to raw[c & 1][i]
    auto issue_raw = [&](int c) {
        const int s0 = c * T;
        const int nst = min(T, span - s0);
        uint8_t* rb = raw + size_t(c & 1) * BPW * RAWB;
#pragma unroll
        for (int m = 0; m < NBL_L; ++m) {
            const int i = lane + 32 * m;
            if (i >= nblk) break;
            const int64_t k0 = kept_at(i, s0);
            const uintptr_t ga = (vlo + uintptr_t(k0)) & ~uintptr_t(15);
            uint8_t* dst = rb + size_t(CF::wslot(i)) * RAWB;
            woffs[(c & 1) * BPW + i] = uint8_t((vlo + uintptr_t(k0)) & 15);
            if (ga >= vlo && ga + RAWB <= vhi) {
                // interior fast path: a fixed number of 16-byte vectors
#pragma unroll
                for (int j = 0; j < RAWB / 16; ++j)
                    cp_async16(smem_u32(dst + 16 * j), reinterpret_cast<const void*>(ga + 16 * j));
            } else {
                const int64_t k1 = kept_at(i, s0 + max(nst, 0));
                const uintptr_t gb = (vlo + uintptr_t(k1) + 15) & ~uintptr_t(15);
                for (uintptr_t x = ga; x < gb; x += 16, dst += 16) {
                    if (x >= vlo && x + 16 <= vhi) {
                        cp_async16(smem_u32(dst), reinterpret_cast<const void*>(x));
                    } else {
                        for (int j = 0; j < 16; ++j) {
                            const uintptr_t y = x + j;
                            dst[j] = (y >= vlo && y < vhi) ? *reinterpret_cast<const uint8_t*>(y) : 0;
                        }
                    }
                }
            }
        }
        cp_async_commit();
    };
    // Transform of chunk c, slice j of NCYC: the soft bytes of every (pair,
    // stage) are interleaved A/B, biased by +128 (u = lam ^ 0x80) and stored
    // as LW words to lam[c & 1][pair][stage].  One item = (pair, G stages) =
    // G*R/4 whole words per block, read as aligned words funnel-shifted to the
    // window offset.  Lane l always serves pair l % PPW (so its window bases
    // and offsets are per-slice constants); the W lanes of a pair split the
    // slice's GPS groups.
    constexpr int GPS = (NG + CF::NCYC - 1) / CF::NCYC;     // groups per pair per slice
    constexpr int TPER = (GPS + W - 1) / W;                 // items per lane per slice
    const int tp = lane % PPW, tsub = lane / PPW;
    // per-chunk part of the transform (window bases and shifts of this lane's
    // pair), computed once per chunk rather than once per slice
    struct TfmSetup {
        const uint8_t* base[2];
        uint32_t sh[2];
        uint32_t* lb;
    };
    // punctured codes (c-18): every dense word is depunctured on the fly from
    // the raw window -- a host table entry per (chunk start phase, dense word)
    // holds a PRMT selector over four consecutive kept bytes and the first
    // kept index (erasures select a byte of a zero operand) -- inside the
    // transform slices, so it overlaps the ACS cycles; sh[h] then packs the
    // table row (phase * NWD) << 8 and the window's byte offset
    constexpr int NWD = (T * R + 3) / 4;
    auto transform_setup = [&](int c) {
        TfmSetup ts;
        const uint8_t* rb = raw + size_t(c & 1) * BPW * RAWB;
        const uint8_t* wo = woffs + (c & 1) * BPW;
        ts.lb = lam + size_t(c & 1) * PPW * LSTR + size_t(tp) * LSTR;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = edge ? 0 : 2 * tp + h;
            const int o0 = int(wo[i]);
            if constexpr (!PUNCT) {
                ts.base[h] = rb + size_t(CF::wslot(i)) * RAWB + (o0 & ~3);
                ts.sh[h] = uint32_t(o0 & 3) * 8u;
            } else {
                const unsigned ph = unsigned(pr_s[i] + c * T) % unsigned(p.P);
                ts.base[h] = rb + size_t(CF::wslot(i)) * RAWB;
                ts.sh[h] = ((ph * unsigned(NWD)) << 8) | unsigned(o0);
            }
        }
        return ts;
    };
    // PUNCT (compile time): the cycle loop exists twice, dense and punctured,
    // selected once per chunk -- a run-time test inside the loop body split it
    // into basic blocks and cost the dense hot loop 62 instructions
    auto transform = [&](const TfmSetup& ts, int j, auto punct_tag) {
        constexpr bool PUNCT = decltype(punct_tag)::value;
        if (edge && tp != 0) return;              // an edge unit has one (replicated) pair
        constexpr int GW = G * R / 4;                     // words per block per item
        const uint8_t* const* base = ts.base;
        const uint32_t* sh = ts.sh;
        uint32_t* lb = ts.lb;
#pragma unroll
        for (int u = 0; u < TPER; ++u) {
            // straight-line: an item past the slice is computed on a clamped
            // group and not stored (no divergent branch inside the ACS loop)
            const int gl = tsub + W * u;                  // group within the slice
            const int g0 = j * GPS + gl;
            const bool valid = gl < GPS && g0 < NG;
            const int g = valid ? g0 : j * GPS;
            uint32_t v[2][GW];
            if constexpr (!PUNCT) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t* w = reinterpret_cast<const uint32_t*>(base[h] + 4 * GW * g);
                    uint32_t wl = w[0];
#pragma unroll
                    for (int k = 0; k < GW; ++k) {
                        const uint32_t wh = w[k + 1];
                        v[h][k] = __funnelshift_r(wl, wh, sh[h]) ^ 0x80808080u;   // u = lam + 128
                        wl = wh;
                    }
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t* win = reinterpret_cast<const uint32_t*>(base[h]);
                    const uint32_t* tab = p.dtab + (sh[h] >> 8);
                    const int woff = int(sh[h] & 0xffu);
#pragma unroll
                    for (int k = 0; k < GW; ++k) {
                        const uint32_t e = __ldg(tab + GW * g + k);
                        const int q = woff + int(e >> 16);
                        const uint32_t x = __funnelshift_r(win[q >> 2], win[(q >> 2) + 1], uint32_t(q & 3) * 8u);
                        v[h][k] = prmt(x, 0u, e & 0xffffu) ^ 0x80808080u;
                    }
                }
            }
            uint32_t ow[G * LW];
#pragma unroll
            for (int t = 0; t < G; ++t) {
#pragma unroll
                for (int q = 0; q < LW; ++q) {
                    const int ia = t * R + 2 * q;
                    const int ib = (2 * q + 1 < R) ? ia + 1 : ia;      // pad byte
                    if ((ia >> 2) == (ib >> 2)) {
                        const uint32_t sel = uint32_t(ia & 3) | (uint32_t(4 + (ia & 3)) << 4) |
                                             (uint32_t(ib & 3) << 8) | (uint32_t(4 + (ib & 3)) << 12);
                        ow[t * LW + q] = prmt(v[0][ia >> 2], v[1][ia >> 2], sel);
                    } else {
                        const uint32_t s2 = uint32_t(ia & 3) | (uint32_t(4 + (ib & 3)) << 4);
                        const uint32_t xa = prmt(v[0][ia >> 2], v[0][ib >> 2], s2);
                        const uint32_t xb = prmt(v[1][ia >> 2], v[1][ib >> 2], s2);
                        ow[t * LW + q] = prmt(xa, xb, 0x5140u);
                    }
                }
            }
            uint32_t* dst = lb + g * (G * LW);
            if (!valid) continue;
            if constexpr (G * LW == 2 && LSTR % 2 == 0) {
                *reinterpret_cast<uint2*>(dst) = make_uint2(ow[0], ow[1]);
            } else if constexpr (G * LW % 4 == 0 && LSTR % 4 == 0) {
#pragma unroll
                for (int k = 0; k < G * LW; k += 4)
                    *reinterpret_cast<uint4*>(dst + k) = make_uint4(ow[k], ow[k + 1], ow[k + 2], ow[k + 3]);
            } else {
#pragma unroll
                for (int k = 0; k < G * LW; ++k) dst[k] = ow[k];
            }
        }
    };

    const int lg = lane & (W - 1), grp = lane / W;
    const bool head = edge && (p.edges[e].flags & EDGE_HEAD);
    int flip[V];
    init_flips<CF>(flip, lg, std::make_integer_sequence<int, V>{});

    uint32_t pm[S];
#pragma unroll
    for (int k = 0; k < S; ++k)
        pm[k] = head ? ((lg == 0 && k == 0) ? 0u : uint32_t(S_HEAD) * 0x00010001u) : 0u;

    uint32_t* gdec = nullptr;
    // survivor region of an interior job; with recycling (fused streams
    // larger than the workspace) wait until the region's previous job has
    // finished its traceback -- it was launched n_regions jobs earlier, so
    // it is running or done and never waits on this one
    size_t region = size_t(gw);
    unsigned region_use = 0;
    if (FUSED && RECYCLE && !edge && p.n_regions > 0) {
        region = size_t(gw % p.n_regions);
        region_use = unsigned(gw / p.n_regions);
        if (region_use > 0) {
            // every lane polls (one transaction): a warp-uniform loop; a
            // region that never frees (impossible unless the grid's blocks
            // were dispatched out of order) traps after ~1 s instead of
            // hanging the device
            for (unsigned spin = 0;
                 !__all_sync(0xffffffffu, ld_acquire_u32(p.region_done + region) >= region_use); ++spin) {
                if (spin > (1u << 22)) __trap();
                __nanosleep(256);
            }
        }
    }
    if (!edge) {
        gdec = p.dec + region * size_t(p.span_int) * ROW;
    } else {
        gdec = p.dec_edge + size_t(e) * size_t(p.span_edge_max) * ROW;
    }

    {
        issue_raw(0);
        if (nchunks > 1) issue_raw(1);
        if (nchunks > 1) cp_async_wait<1>(); else cp_async_wait<0>();
        __syncwarp();
        {
            const TfmSetup ts0 = transform_setup(0);
#pragma unroll 1
            for (int j = 0; j < CF::NCYC; ++j) {
                transform(ts0, j, std::integral_constant<bool, PUNCT>{});
            }
        }
        __syncwarp();
        if (!edge && p.pad > 0) {
            // the front pad stages are erasures (lambda = 0, biased u = 128)
            const int n = p.pad * LW;
            for (int i = lane; i < PPW * n; i += 32) lam[(i / n) * LSTR + i % n] = 0x80808080u;
            __syncwarp();
        }
    }
#ifdef PBVD_EXP_TIMING
    if (p.dbg && lane == 0) p.dbg[32 * gw + 30] = gtime();   // prologue done
#endif
    for (int c = 0; c < nchunks; ++c) {
        const int nst = min(T, span - c * T);
        const bool next = c + 1 < nchunks;
        SoftSrc<CF> src;
        {
            // soft windows of chunk c+2 go in flight; those of chunk c+1 (issued a
            // chunk ago) must have landed before this chunk's transform slices
            if (c + 2 < nchunks) {
                issue_raw(c + 2);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncwarp();
            src.lamrow = lam + size_t(c & 1) * PPW * LSTR + size_t(edge ? 0 : grp) * LSTR;
        }
        // survivor rows of this chunk, this lane's WPS words (direct stores:
        // each warp writes 32 * WPS contiguous words per stage)
        uint32_t* drow = gdec + size_t(c) * T * ROW + size_t(lane) * CF::WPS;
        uint32_t* const drow0 = gdec + size_t(lane) * CF::WPS;     // rows [0, v): never read
        // cycles wholly below the traceback's first row (s_read >= v) write
        // their survivor rows over the region's rows [0, v) instead -- rows
        // no traceback reads, so those stores stay in L2 and never reach HBM
        // (one select per cycle; a predicate per store cost 0.5 %)
        const int st_lo = s_read - c * T;
        // whole v-stage cycles of the chunk run in the one hot loop (interior
        // spans are padded to a multiple of v); only an edge block's last
        // chunk can leave a remainder of < v stages
        const int ncyc = nst / V;
        {
            // each cycle's first-stage operands are loaded one cycle ahead
            // (within a cycle Cycle<> loads one stage ahead); the read past the
            // chunk's last stage stays inside the operand row's padding
            const TfmSetup tsn = transform_setup(c + 1);      // harmless past the last chunk
            {
                const std::integral_constant<bool, PUNCT> punct_tag{};
                XY<CF> first = src.load(0);
#pragma unroll 1
                for (int j = 0; j < ncyc; ++j) {
                    const int s0 = j * V;
                    const XY<CF> nfirst = src.load(s0 + V);
                    uint32_t* crow = (s0 + V > st_lo) ? drow + size_t(s0) * ROW : drow0;
                    Cycle<CF, 0, true>::run(pm, src, flip, lg, crow, s0, T, true, first, p.one,
                                            p.neg_one);
                    first = nfirst;
                    transform(tsn, j, punct_tag);
                }
            }
        }
        if (ncyc * V < nst)   // (the last chunk of an edge block)
            Cycle<CF, 0, false>::run(pm, src, flip, lg, drow + size_t(ncyc * V) * ROW, ncyc * V, nst, true,
                                     src.load(ncyc * V), p.one, p.neg_one);
        // renormalise: subtract the block minimum (per 16-bit half = per block);
        // interior warps every RN chunks (edge warps: head blocks hold S_HEAD)
        if (edge || CF::RN == 1 || (c % CF::RN) == CF::RN - 1) {
            uint32_t mn = pm[0];
#pragma unroll
            for (int k = 1; k < S; ++k) mn = __vmins2(mn, pm[k]);
#pragma unroll
            for (int o = 1; o < W; o <<= 1) mn = __vmins2(mn, __shfl_xor_sync(0xffffffffu, mn, o));
#pragma unroll
            for (int k = 0; k < S; ++k) pm[k] -= mn;
        }
        __syncwarp();      // every lane is done with lam[c & 1] before chunk c+2's transform
#ifdef PBVD_EXP_TIMING
        if (p.dbg && lane == 0 && c < 24) p.dbg[32 * gw + 8 + c] = gtime();
#endif
    }

    // ---- traceback start: min PM, lowest logical state on ties --------
    const int pend = span % V;
    // key = (PM << SB) | logical state: SB = max(8, v) bits of state (16 + 11 <= 32)
    constexpr int SB = V > 8 ? V : 8;
    constexpr uint32_t SMASK = (1u << SB) - 1u;
    uint32_t kA = 0xffffffffu, kB = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const uint32_t q = uint32_t(lg * S + k);
        const uint32_t u = ((q >> pend) | (q << (V - pend))) & uint32_t(N - 1);
        kA = min(kA, ((pm[k] & 0xffffu) << SB) | u);
        kB = min(kB, ((pm[k] >> 16) << SB) | u);
    }
#pragma unroll
    for (int o = 1; o < W; o <<= 1) {
        kA = min(kA, __shfl_xor_sync(0xffffffffu, kA, o));
        kB = min(kB, __shfl_xor_sync(0xffffffffu, kB, o));
    }
    // the paper's own rule (Alg. 1 K2 "state = 0"): no state
    // estimation, every block traces back from state S_0
    if (p.start_zero) kA = kB = 0u;
    if constexpr (FUSED) {
        // traceback of this warp's blocks, lane i = block i (+32, +64 ...)
        constexpr int NBL = TbwCfg<CF>::NBL;
        uint32_t stv[NBL];
        int64_t ob[NBL];
#pragma unroll
        for (int m = 0; m < NBL; ++m) {
            const int i = min(lane + 32 * m, BPW - 1);
            const int src = (i >> 1) * W;
            const uint32_t a = __shfl_sync(0xffffffffu, kA, src);
            const uint32_t b = __shfl_sync(0xffffffffu, kB, src);
            stv[m] = ((i & 1) ? b : a) & SMASK;
            ob[m] = p.out_bit0 + (wb0 + lane + 32 * m) * int64_t(p.D);
        }
        if (edge) {
            stv[0] = (p.edges[e].flags & EDGE_START0) ? 0u : (__shfl_sync(0xffffffffu, kA, 0) & SMASK);
            ob[0] = p.edges[e].out_bit0;
        }
        const int nblk_tb = edge ? 1 : int(min(int64_t(BPW), int64_t(p.n_int) - wb0));
#ifdef PBVD_EXP_TIMING
        if (p.dbg && lane == 0) p.dbg[32 * gw + 1] = gtime();
#endif
        warp_traceback<CF>(wbase, gdec, span, edge ? p.edges[e].t0r : p.t0r,
                           edge ? p.edges[e].t1r : p.t1r, nblk_tb, stv, ob,
                           p.word_out && (!edge || (((ob[0] | int64_t(p.edges[e].t1r -
                                                                        p.edges[e].t0r)) & 31) == 0)),
                           p.out, lane,
#ifdef PBVD_EXP_TIMING
                           p.dbg ? p.dbg + 32 * gw : nullptr);
#else
                           nullptr);
#endif
        if (RECYCLE && !edge && p.n_regions > 0) {
            // the region's rows have all been read (every bulk copy of the
            // walk was waited for): the next job in it may overwrite them
            __syncwarp();
            if (lane == 0) st_release_u32(p.region_done + region, region_use + 1u);
        }
        if constexpr (MIRROR) {
            // multi-GPU gather fused into this kernel: the warp's decoded
            // bytes (its blocks own whole, contiguous bytes) go to every
            // mirror destination (other ranks' buffers over NVLink)
            __syncwarp();          // the walk's stores of all lanes are visible
            int64_t bit0, nbits;
            if (!edge) {
                bit0 = p.out_bit0 + wb0 * int64_t(p.D);
                nbits = int64_t(nblk_tb) * p.D;
            } else {
                bit0 = p.edges[e].out_bit0;
                nbits = p.edges[e].t1r - p.edges[e].t0r;
            }
            mirror_copy(p.out + (bit0 >> 3), (nbits + 7) >> 3, p.mirror, p.n_mirror, lane, 32);
        }
#ifdef PBVD_EXP_TIMING
        __syncwarp();
        if (p.dbg && lane == 0) p.dbg[32 * gw + 2] = gtime();
#endif
        return;
    }
    if (lg == 0) {
        if (!edge) {
            const int64_t bi = wb0 + 2 * grp;
            if (bi < p.n_int) p.start[bi] = int32_t(kA & SMASK);
            if (bi + 1 < p.n_int) p.start[bi + 1] = int32_t(kB & SMASK);
        } else if (grp == 0) {
            p.start_edge[e] = (p.edges[e].flags & EDGE_START0) ? 0 : int32_t(kA & SMASK);
        }
    }
    pdl_launch_dependents();   // the traceback grid may start scheduling
}

}  // namespace pbvd
