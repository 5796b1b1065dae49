// params.h -- kernel parameter blocks shared by the host planner and the
// sm_100a kernels (plain structs, passed by value as kernel parameters).
#pragma once
#include <cstdint>

namespace pbvd {

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

constexpr int MAX_EDGE = 32;      // edge blocks per launch (more -> extra launches)
constexpr int MAX_MIRROR = 7;     // extra output destinations (peer GPUs' buffers)

// Multi-GPU gather fused into the decode (pbvd_decode_blocks_mirrored): the
// bytes [0, n) at src are copied to src + md[k] for k < nm -- the other
// ranks' gather buffers mapped into this process (CUDA IPC / peer access),
// by threads t = tid, tid + nthr, ... (32-bit words when aligned).
__device__ __forceinline__ void mirror_copy(const uint8_t* src, int64_t n, const int64_t* md,
                                            int nm, int tid, int nthr) {
    if (((reinterpret_cast<uintptr_t>(src) | uintptr_t(n)) & 3) == 0) {
        const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
        for (int64_t i = tid; i < n / 4; i += nthr) {
            const uint32_t v = s32[i];
            for (int k = 0; k < nm; ++k)
                *reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(src) + md[k] + 4 * i) = v;
        }
    } else {
        for (int64_t i = tid; i < n; i += nthr) {
            const uint8_t v = src[i];
            for (int k = 0; k < nm; ++k) const_cast<uint8_t*>(src)[md[k] + i] = v;
        }
    }
}
constexpr int S_HEAD = 8192;      // known-start sentinel, > v*128*R (reading c-12)

// One "edge" block: a block whose forward span is not the uniform
// [bD-L, bD+D+L) -- head blocks (span starts at stage 0, known start state),
// blocks clipped by the end of the stream, and the last block.
struct EdgeDesc {
    int64_t lo;        // absolute first stage of the forward span
    int64_t out_bit0;  // bit offset of the block's first decoded bit in d_bits
    int span;          // forward stages
    int t0r, t1r;      // decoding range relative to lo: [t0r, t1r)
    int flags;         // EDGE_HEAD | EDGE_START0
};
constexpr int EDGE_HEAD = 1;    // initial metrics: state 0 -> 0, others S_HEAD
constexpr int EDGE_START0 = 2;  // traceback starts in state 0 (terminated tail)

struct FwdParams {
    const int8_t* llr;     // this launch's soft values (first = kept index kb_ws0)
    int64_t n_llr;         // valid values from llr
    int64_t kb_ws0;        // absolute kept index of llr[0]
    int64_t b_int0;        // first interior block (absolute index)
    int n_int;             // interior blocks in this launch
    int n_int_warps;       // warp units for interior blocks; edge units follow
    int D, L;
    int span_int;          // D + 2L + pad (interior forward stages)
    int pad;               // interior spans start `pad` erasure stages early (a multiple of v)
    uint32_t one, neg_one; // 1 and 0xffffffff, opaque to the compiler (pipe balancing)
    int P;                 // puncture period (1 = none)
    int kp;                // kept values per period
    int cum[16];           // kept values in columns [0, p) of one period
    // depuncture table (P > 1): entry [ph0][w] for dense word w of a chunk
    // starting at phase ph0 -- bits 0-15 a PRMT selector over the 4 kept
    // bytes from bits 16-23 = first kept index of the word (nibble 4 = erasure)
    const uint32_t* dtab;
    uint32_t* dec;         // interior survivor regions
    int32_t* start;        // interior start states (logical state index)
    uint32_t* dec_edge;    // edge survivor regions
    int32_t* start_edge;   // edge start states
    int span_edge_max;     // stage capacity of one edge region
    int n_edge;
    // fused traceback (fwd_kernel<CF, true>): decoded bits go straight to out
    uint8_t* out;
    int64_t out_bit0;      // bit offset of the first interior block in out
    int t0r, t1r;          // interior decoding range relative to lo (L, L+D)
    int word_out;          // 1: interior blocks store aligned 32-bit words
    int start_zero;        // 1: every traceback starts in state 0 (PBVD_START_ZERO)
    int n_mirror;          // extra output destinations (fused mode, mirror_copy)
    int64_t mirror[MAX_MIRROR];   // byte offsets of the destinations from out
    // fused mode, streams larger than the survivor workspace: interior job
    // gw uses region gw % n_regions once the job before it there (gw -
    // n_regions) has finished its traceback (region_done[r] counts the jobs
    // done in region r this launch); 0: region = gw (one region per job)
    int n_regions;
    unsigned* region_done;
    unsigned long long* dbg;   // timing experiment only (PBVD_EXP_TIMING builds), else null
    EdgeDesc edges[MAX_EDGE];
};

struct TbParams {
    const uint32_t* dec;
    const int32_t* start;
    int n_int;
    int n_int_ctas;
    int span_int;
    int t0r, t1r;          // interior decoding range relative to lo (L, L+D)
    int D;
    int word_out;          // 1: interior blocks store aligned 32-bit words
    int64_t out_bit0;      // bit offset of the first interior block in d_bits
    uint8_t* out;
    const uint32_t* dec_edge;
    const int32_t* start_edge;
    int span_edge_max;
    int n_edge;
    EdgeDesc edges[MAX_EDGE];
};

}  // namespace pbvd
