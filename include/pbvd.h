/*
 * pbvd.h -- C ABI of the B200 (sm_100a) parallel block-based Viterbi decoder.
 *
 * The operation is the PBVD of Peng et al., arXiv 1608.00066 ("P:n" = line n
 * of PAPER.md):
 *   - a received stream of soft values is cut into blocks of D decoded stages;
 *     block b decodes [bD, bD+D) and runs its forward pass over the parallel
 *     block [bD-L, bD+D+L) (truncated block M = L, decoding block D,
 *     traceback block L);
 *   - the forward pass is the add-compare-select recursion of Eq. 1
 *     on the trellis of Eq. 2, with the branch metrics reduced to
 *     the 2^R distinct codeword metrics per stage (Eqs. 3-6);
 *   - one survivor bit per state per stage is kept ("bit 0 denotes the upper
 *     branch, bit 1 the lower");
 *   - the traceback (Alg. 1 K2) starts from the minimum path-metric
 *     state, walks back through the L traceback stages and emits the D
 *     decoded bits, packed 8 per byte.
 * Points the paper leaves open are fixed as in DESIGN.md §3 (readings c-1 ..
 * c-24): tie -> upper branch; head block = known start state 0; terminated
 * tail -> traceback from state 0; argmin ties -> lowest state index.
 *
 * Conventions
 *   polys     generator polynomials, bit K-1 = input tap g_{K-1}, bit 0 = g_0
 *             (e.g. CCSDS {0171, 0133}); output bit order follows the list.
 *   soft in   int8, one value per coded bit, [stage][r] order, punctured
 *             positions omitted; value > 0 favours coded bit 0 (BPSK 0 -> +1).
 *             Every int8 value (including -128) is accepted.
 *   bits out  packed LSB-first: info bit i -> byte i>>3, bit (i & 7); pad 0.
 *   TERMINATED the stream carries K-1 extra zero-tail stages after n_info;
 *             the last block traces back from state 0 and the tail is not
 *             emitted.
 *
 * Ownership / threading
 *   The caller owns every input and output buffer (device pointers unless a
 *   function says "host") and the CUDA stream.  The handle owns its code
 *   tables and a survivor workspace on its device (grown on demand, freed by
 *   pbvd_destroy).  Decode calls are asynchronous on `stream` (a cudaStream_t
 *   passed as void*, NULL = legacy default stream) unless stated otherwise.
 *   A handle must not be used from two host threads at once; use one handle
 *   per concurrent stream.
 *
 * Errors
 *   Every function returns PBVD_OK (0) or a negative pbvd_status; nothing is
 *   thrown or aborted across the ABI.  pbvd_last_error() gives a message for
 *   the last failure on a handle (including the CUDA error string).  There is
 *   no CPU fallback: a call that cannot run on the GPU fails.
 */
#ifndef PBVD_H
#define PBVD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pbvd_s *pbvd_t;

enum pbvd_status {
    PBVD_OK = 0,
    PBVD_EINVAL = -1,       /* bad argument (null pointer, range)              */
    PBVD_ENOMEM = -2,       /* device or host allocation failed                */
    PBVD_ECUDA = -3,        /* CUDA runtime / launch error                     */
    PBVD_EUNSUPPORTED = -4, /* no compiled kernel and the run-time (NVRTC) build
                               failed or the lane count is not a supported shape */
    PBVD_ESIZE = -5         /* buffer length inconsistent with n_info          */
};

#define PBVD_TERMINATED (1u << 0) /* stream ends with K-1 zero tail stages (c-13) */
#define PBVD_ALLOW_CATASTROPHIC (1u << 1) /* accept generators with no g_{K-1} or no g_0
                                            tap (SPEC S:53-55 warning-class override) */
#define PBVD_START_ZERO (1u << 2) /* the paper's own traceback start (§III.A: "a
                                    traceback procedure starts from a random state (state
                                    S_0, for example)"; Alg. 1 K2 initialises state = 0,
                                    P:215): EVERY block, interior, head and last, traces
                                    back from state 0 instead of the min-PM state of P:75
                                    (the alternative of reading c-10).  Costs BER at short
                                    L (Fig. 4; DESIGN.md §10 NEXT 3). */

/* Create a decoder on CUDA device `device`.
 *   K          constraint length, 3..12 (2^(K-1) states)
 *   R          generators per code (code rate 1/R before puncturing), 2..4
 *   polys      R generator polynomials (see Conventions); host pointer; each
 *              in [1, 2^K); some polynomial must have bit K-1 and some bit 0
 *              set unless flags has PBVD_ALLOW_CATASTROPHIC
 *   punct_period P >= 1; 1 = unpunctured
 *   punct      R*P keep flags, row r (generator r) then column p, i.e.
 *              punct[r*P + p]; host pointer, NULL iff P == 1.  Column p
 *              applies to stages s with s mod P == p (also the tail stages).
 *   D          decoded stages per block, D >= 8 and D % 8 == 0 (blocks own
 *              whole output bytes)
 *   L          truncation / traceback length (M = L), 1 <= L
 *   soft_bits  quantisation of the input, 1..8 (1 = hard +-1); advisory only
 *   flags      PBVD_TERMINATED | PBVD_ALLOW_CATASTROPHIC | PBVD_START_ZERO, or 0
 * Kernels: the codes listed by pbvd_supported() are compiled into the
 * library; any other (K, R, polys) is compiled at create time from the same
 * kernel templates with NVRTC (libnvrtc.so.12 loaded on demand; a few seconds
 * the first time, then cached in-process and on disk under $PBVD_JIT_CACHE,
 * default ~/.cache/pbvd_jit; PBVD_JIT_CACHE=off disables the disk cache).
 * Returns PBVD_EINVAL for bad arguments, PBVD_ECUDA for a bad device and
 * PBVD_EUNSUPPORTED if the run-time build fails; pbvd_last_error(NULL) then
 * gives the reason (thread-local). */
int pbvd_create(pbvd_t *out, int K, int R, const uint32_t *polys, int punct_period,
                const uint8_t *punct, int D, int L, int soft_bits, unsigned flags,
                int device);

/* Release the handle, its device tables and survivor workspace (and any host
 * pipeline streams).  h may be NULL.  The caller must have finished (or
 * synchronised) every decode issued on h and closed its pbvd_stream_t objects;
 * the caller's buffers are not touched.  No error is reported. */
void pbvd_destroy(pbvd_t h);

/* Number of int8 soft values of a stream with n_info info bits: R per stage
 * (one per coded bit, Eq. 2) over n_info stages plus the K-1 zero
 * tail stages if TERMINATED (reading c-13), minus the punctured positions
 * (reading c-18: column s mod P of the keep matrix).  PBVD_EINVAL for a NULL
 * handle or n_info < 1 (message in pbvd_last_error(h)). */
int64_t pbvd_llr_count(pbvd_t h, int64_t n_info);

/* Number of trellis stages (n_info, plus K-1 if TERMINATED) and of blocks
 * ceil(n_info/D) (the decoding blocks of P:93; the last one may hold
 * fewer than D bits, reading c-22).  PBVD_EINVAL as pbvd_llr_count. */
int64_t pbvd_stage_count(pbvd_t h, int64_t n_info);
int64_t pbvd_block_count(pbvd_t h, int64_t n_info);

/* Decode a whole stream: the PBVD of §III.A -- every
 * block's forward ACS over its parallel block [bD-L, bD+D+L) (Eq. 1, P:72-74;
 * branch metrics from the 2^R codeword metrics, Eqs. 3-6), survivor decisions
 * (P:258), traceback from the min-PM state (state 0 with
 * PBVD_START_ZERO) through the L traceback stages, D bits emitted per
 * block (Alg. 1 K2), packed LSB-first.
 *   d_llr  device, n_llr == pbvd_llr_count(n_info) int8 values, [stage][r]
 *   d_bits device, >= ceil(n_info/8) bytes, fully written (pad bits 0)
 *   stream cudaStream_t (NULL = legacy default stream)
 * Errors: PBVD_EINVAL (NULL pointer, n_info < 1), PBVD_ESIZE (n_llr differs
 * from pbvd_llr_count), PBVD_ENOMEM (workspace), PBVD_ECUDA (launch); the
 * message is in pbvd_last_error(h).  Asynchronous on `stream`. */
int pbvd_decode(pbvd_t h, const int8_t *d_llr, int64_t n_llr, uint8_t *d_bits, int64_t n_info,
                void *stream);

/* Decode blocks [block0, block0+nblocks) of a stream of n_info_total info bits
 * (the multi-GPU shard entry point).
 *   d_llr_window  device pointer to the first kept soft value of stage
 *                 window_stage0; the window holds window_n_llr values and must
 *                 cover every forward span of the range, i.e. stages
 *                 [max(0, block0*D - L), min(n_stages, (block0+nblocks)*D + L))
 *                 (all remaining stages if the range ends with the last block)
 *   d_bits        device, receives the bits of [block0*D, min((block0+nblocks)*D,
 *                 n_info)) packed LSB-first from byte 0 (ceil(bits/8) bytes)
 * Asynchronous on `stream`. */
int pbvd_decode_blocks(pbvd_t h, const int8_t *d_llr_window, int64_t window_stage0,
                       int64_t window_n_llr, int64_t n_info_total, int64_t block0,
                       int64_t nblocks, uint8_t *d_bits, void *stream);

/* pbvd_decode_blocks whose decoded bits are ALSO stored, by the traceback
 * itself, to n_mirrors (0..7) further destinations: d_mirrors[k] receives
 * the same bytes as d_bits.  The destinations may be other GPUs' memory
 * mapped into this process (CUDA IPC handles / peer access over NVLink), so a
 * multi-GPU run gathers its output inside the decode kernel -- the "final
 * gather" of P:112 fused with the traceback that produces the bits (each
 * warp copies its blocks' bytes to the mirrors right after its walk, while
 * other warps still compute) instead of a separate NCCL collective; in
 * two-kernel mode (pbvd_set_fused(h, 0)) the copies follow the traceback.  Each d_mirrors[k] must be congruent to
 * d_bits modulo 4 (PBVD_EINVAL otherwise).  Completion on a destination
 * device is the completion of this call's work on `stream` (synchronise or
 * barrier before reading there).  Asynchronous on `stream`. */
int pbvd_decode_blocks_mirrored(pbvd_t h, const int8_t *d_llr_window, int64_t window_stage0,
                                int64_t window_n_llr, int64_t n_info_total, int64_t block0,
                                int64_t nblocks, uint8_t *d_bits, uint8_t *const *d_mirrors,
                                int n_mirrors, void *stream);

/* End-to-end decode of blocks [block0, block0+nblocks) from HOST memory
 * (arguments as pbvd_decode_blocks, but h_llr_window / h_bits are host
 * pointers): the range is cut into segments that are copied to the device,
 * decoded and copied back on `n_streams` internal CUDA streams (1..8), so the
 * H2D / D2H transfers of one segment overlap the kernels of another -- the
 * multi-stream scheme of §IV.C.  For a whole stream pass
 * window_stage0 = 0, window_n_llr = pbvd_llr_count(n_info), block0 = 0,
 * nblocks = pbvd_block_count(n_info).  Host buffers should be pinned
 * (cudaHostAlloc / torch pin_memory) for overlap; pageable memory works but
 * serialises.  Synchronous: returns when h_bits is complete. */
int pbvd_decode_host(pbvd_t h, const int8_t *h_llr_window, int64_t window_stage0,
                     int64_t window_n_llr, int64_t n_info_total, int64_t block0,
                     int64_t nblocks, uint8_t *h_bits, int n_streams);

/* Continuous stream (halo carry across calls; the SDR use case of P:424).
 * A pbvd_stream_t belongs to one decoder handle and decodes ONE stream whose
 * soft values arrive in pieces of any length (a piece may end inside a
 * stage).  Each push appends d_llr (device, n_llr kept values in stream
 * order, as in pbvd_decode) and decodes every block whose forward span
 * [bD-L, bD+D+L) has fully arrived and which cannot be the last block,
 * writing their bits to d_bits (device, bits_cap bytes; whole blocks, so a
 * multiple of D bits) and the number of bits to *n_bits (0 if none is ready).
 * pbvd_stream_finish ends the stream: the remaining blocks (including the
 * last, traced back from state 0 if the handle is TERMINATED) are decoded to
 * d_bits and *n_bits = n_info - bits emitted before, where n_info = stages
 * received - (K-1 if TERMINATED).  The concatenation of all outputs equals
 * pbvd_decode of the concatenated soft values, bit for bit.  After finish the
 * object is empty and can take a new stream.  The soft values later blocks
 * still need (L stages of halo plus the unfinished block) are carried in
 * device buffers owned by the stream object, so the caller may reuse d_llr
 * once the push's work on `stream` is done.  All calls on one stream object
 * must use the same CUDA stream (or be ordered by the caller); the handle's
 * workspace is shared, so do not decode on the handle concurrently.
 * Errors: PBVD_EINVAL (null/negative), PBVD_ESIZE from a push whose ready
 * blocks do not fit bits_cap (nothing is consumed; retry with a larger
 * buffer -- (received stages / D + 1) * D bits always suffice) or from a
 * finish whose stream ends inside a stage or has no info bit (the object is
 * reset either way), PBVD_ENOMEM, PBVD_ECUDA. */
typedef struct pbvd_stream_s *pbvd_stream_t;
int pbvd_stream_open(pbvd_t h, pbvd_stream_t *out);
int pbvd_stream_push(pbvd_stream_t s, const int8_t *d_llr, int64_t n_llr, uint8_t *d_bits,
                     int64_t bits_cap, int64_t *n_bits, void *stream);
int pbvd_stream_finish(pbvd_stream_t s, uint8_t *d_bits, int64_t bits_cap, int64_t *n_bits,
                       void *stream);
void pbvd_stream_close(pbvd_stream_t s);

/* Tuning / introspection ------------------------------------------------- */

/* Lanes per block pair used by the forward kernel (1, 2, 4, 8; 0 = default
 * for the code).  Returns PBVD_EUNSUPPORTED if that variant is not compiled. */
int pbvd_set_lanes(pbvd_t h, int lanes);
int pbvd_get_lanes(pbvd_t h);

/* Kernel structure (default 1).  fused = 1: ONE kernel per launch group --
 * every forward warp traces back its own blocks right after its forward
 * pass (survivors re-read from L2 into the warp's shared memory).  fused = 0:
 * the paper's two kernels "with different parallelism" (Alg. 1 K1 + K2,
 * P:112): forward, then a traceback kernel with one thread per block.
 * Both produce identical bits.  Returns PBVD_EINVAL for a NULL handle. */
int pbvd_set_fused(pbvd_t h, int fused);
int pbvd_get_fused(pbvd_t h);

/* Upper bound on the survivor workspace in bytes (default 4 GiB: measured
 * best for C5 on B200 -- larger waves lose to address-translation misses);
 * decodes larger than one workspace run, in fused mode, as one launch whose
 * jobs recycle the workspace's survivor regions, and in two-kernel mode in
 * waves.  Returns PBVD_EINVAL below
 * 1 MiB. */
int pbvd_set_workspace_limit(pbvd_t h, size_t bytes);

/* When enabled, each decode records CUDA events around every kernel launch
 * on the caller's stream; pbvd_kernel_times() (after the stream is
 * synchronised) returns the summed forward and traceback kernel times (ms)
 * of the most recent decode call and the number of kernel launches. */
int pbvd_set_profiling(pbvd_t h, int enable);
int pbvd_kernel_times(pbvd_t h, float *fwd_ms, float *tb_ms, int *launches);

/* Survivor bytes written per decoded stage-block (N/8 * span) etc. */
typedef struct {
    int K, R, N, lanes, D, L, P;
    int64_t dec_bytes_per_block; /* survivor bytes of one interior block   */
    int64_t span;                /* forward stages of one interior block   */
    size_t workspace_bytes;      /* currently allocated                    */
    int jit;                     /* 1 if the kernels were built at run time */
    int host_lanes;              /* lanes of the variant pbvd_decode_host uses:
                                    the compiled one with the most lanes per
                                    pair (>= 16 states per lane; lowest
                                    per-warp latency -- that pipeline is
                                    PCIe-bound) unless pbvd_set_lanes fixed it */
} pbvd_info;
int pbvd_get_info(pbvd_t h, pbvd_info *info);

/* Diagnostic: the measured ACS roofline of device `device`.  Runs, from
 * registers only, the minimal 16x2 SIMD instruction sequence that produces a
 * path metric and a packed survivor bit per state and block (Eq. 1, P:72-74;
 * P:258) on every SM, and returns ACS per second (one ACS = one state of one
 * block at one stage) and the best kernel time in ms.  Synchronous. */
int pbvd_probe_acs_peak(int device, double *acs_per_s, double *ms);

/* The same probe with the forward kernel's pipe balancing (every other
 * decision operand formed by two IMADs on the FMA pipe): the measured ACS
 * rate of the balanced minimal sequence, a cross-check of the derived
 * roofline bench.py reports.  Same arguments/errors. */
int pbvd_probe_acs_balanced(int device, double *acs_per_s, double *ms);

/* Compiled (K, R, polys...) combinations, as text "K:R:o1,o2[,o3]:lanes;..."
 * (other codes are built at run time, see pbvd_create). */
const char *pbvd_supported(void);

const char *pbvd_strerror(int code);
/* Build (NVRTC) the kernels pbvd_create would JIT for (K, R, polys) with
 * `lanes` lanes per block pair (0 = default) and store them in the disk cache,
 * without touching a GPU -- e.g. to warm the cache ahead of time.  Returns
 * PBVD_OK, PBVD_EINVAL (arguments as pbvd_create) or PBVD_EUNSUPPORTED (no
 * such shape / compile failed; the reason is written to msg, msg_len bytes
 * incl. the terminating 0, if msg is not NULL).  Codes listed by
 * pbvd_supported() need no build. */
int pbvd_jit_prebuild(int K, int R, const uint32_t *polys, int lanes, char *msg, size_t msg_len);

/* Message of the last failure on h; for h == NULL, of the calling thread's
 * last failed pbvd_create. */
const char *pbvd_last_error(pbvd_t h);

/* Gather buffers shared across processes (the multi-GPU "decoded bits are
 * gathered" step, §III.A, fused into the decode by
 * pbvd_decode_blocks_mirrored): plumbing over CUDA IPC, so that every rank can
 * map every other rank's gather buffer and the traceback can store into it
 * over NVLink / NVSwitch.
 *   pbvd_ipc_export  d_ptr: any device pointer inside a cudaMalloc'ed
 *                    allocation of this process (e.g. a torch tensor's
 *                    data_ptr).  Writes the allocation's IPC handle
 *                    (PBVD_IPC_HANDLE_BYTES bytes, caller-owned) and d_ptr's
 *                    byte offset from the allocation base.
 *   pbvd_ipc_open    maps (handle, offset) of ANOTHER process into this one on
 *                    `device` (peer access enabled lazily) and returns the
 *                    pointer matching the exporter's d_ptr.  The mapping stays
 *                    valid until pbvd_ipc_close; the exporter must keep its
 *                    allocation alive until every importer has closed it.
 *   pbvd_ipc_close   unmaps a pointer from pbvd_ipc_open (same offset/device).
 * Errors: PBVD_EINVAL (null / not a device allocation), PBVD_ECUDA (the CUDA
 * IPC call failed -- e.g. no peer access between the devices); the message is
 * in pbvd_last_error(NULL).  Synchronous. */
#define PBVD_IPC_HANDLE_BYTES 64
int pbvd_ipc_export(const void *d_ptr, void *handle, int64_t *offset);
int pbvd_ipc_open(const void *handle, int64_t offset, int device, void **d_ptr);
int pbvd_ipc_close(void *d_ptr, int64_t offset, int device);

#ifdef __cplusplus
}
#endif
#endif /* PBVD_H */
