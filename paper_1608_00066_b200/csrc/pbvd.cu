// pbvd.cu -- C ABI (include/pbvd.h) of the B200 parallel block-based Viterbi
// decoder: validation, block planning (interior blocks with the
// uniform span [bD-L, bD+D+L) plus "edge" blocks at the stream ends), survivor
// workspace and waves, and the two kernel launches per wave (forward: fwd.cuh,
// traceback: tb.cuh).  Torch is not involved below this line.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pbvd.h"
#include "variant.h"

namespace pbvd {

const std::vector<Variant>& variants() {
    static const std::vector<Variant> v = [] {
        std::vector<Variant> r;
        add_variants_k3(r);
        add_variants_k5(r);
        add_variants_k7(r);
        add_variants_k7r3(r);
        add_variants_k9(r);
        return r;
    }();
    return v;
}

static std::mutex g_prep_mu;

}  // namespace pbvd

using namespace pbvd;

struct Workspace {
    void* p = nullptr;
    size_t bytes = 0;
};

// Resources of the host-buffer pipeline (pbvd_decode_host): per stream a
// survivor workspace and device staging buffers for the soft window / bits.
struct HostLane {
    cudaStream_t stream = nullptr;
    Workspace ws;
    int8_t* d_llr = nullptr;
    size_t llr_cap = 0;
    uint8_t* d_bits = nullptr;
    size_t bits_cap = 0;
    cudaEvent_t in_ready = nullptr;   // this lane's staging buffer holds its segment
    cudaEvent_t consumed = nullptr;   // its decode has read the staging buffer
};

struct pbvd_s {
    int device = 0;
    int K = 0, R = 0, V = 0, N = 0;
    uint32_t polys[4] = {0, 0, 0, 0};
    int P = 1, kp = 0;
    uint8_t punct[64] = {};
    int cum[16] = {};
    uint64_t keep = 0;
    uint32_t* dtab = nullptr;   // device depuncture table (P > 1), see FwdParams::dtab
    int D = 0, L = 0, soft_bits = 8;
    unsigned flags = 0;
    const Variant* var = nullptr;
    // variant of the host pipeline (pbvd_decode_host): PCIe-bound, so what
    // counts is the latency of the segment decoded after the last copy --
    // the compiled variant with the most lanes per pair (fewest states per
    // lane, >= 16) unless the caller fixed the lane count
    const Variant* host_var = nullptr;
    Workspace ws;
    size_t ws_limit = size_t(4) << 30;
    std::vector<HostLane> lanes;
    cudaStream_t h2d = nullptr;        // host pipeline: every H2D copy, in stream order
    bool prof = false;
    bool fused = true;     // forward + in-warp traceback in one kernel (pbvd_set_fused)
    int n_mirror = 0;      // extra output destinations of the current call (byte offsets)
    int64_t mirror[MAX_MIRROR] = {};
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, int>> ev_fwd, ev_tb;   // indices into ev_pool
    int launches = 0;
    std::string err;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int fail(pbvd_t h, int code, const std::string& msg) {
    if (h) h->err = msg;
    return code;
}

int cuda_fail(pbvd_t h, cudaError_t e, const char* where) {
    return fail(h, PBVD_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int64_t kept_before_h(const pbvd_s* h, int64_t s) {
    if (h->P == 1) return s * h->R;
    return (s / h->P) * h->kp + h->cum[s % h->P];
}

// Dynamic shared memory of a forward / fused launch: the variant's need, or
// more, so that at most FWD_WARPS_PER_SM one-warp CTAs are resident per SM
// (228 KB of shared memory per SM, 1 KB reserved per CTA).  Measured on B200
// (tools/r2f.sh): 3 warps per SM sub-partition beat 4 by 10 % at 2^26 bits
// (C2 119 vs 109 Gb/s, C3a 106 vs 97) -- more resident warps spread over
// more code (hot loop, traceback, prologue) and miss in the 32 KB
// instruction cache -- and 2 per sub-partition lose again (112).
// PBVD_FWD_WARPS_PER_SM overrides it (0 = no cap) for experiments.
constexpr int FWD_WARPS_PER_SM = 12;
size_t fwd_smem(size_t need) {
    static const int cap = [] {
        const char* e = std::getenv("PBVD_FWD_WARPS_PER_SM");
        return e ? std::atoi(e) : FWD_WARPS_PER_SM;
    }();
    if (cap <= 0) return need;
    const size_t per = ((size_t(228) * 1024 / size_t(cap) - 1024) / 128) * 128;
    return std::max(need, per);
}

int ensure_prepared(pbvd_t h, const Variant* v) {
    std::lock_guard<std::mutex> lk(g_prep_mu);
    const uint64_t bit = uint64_t(1) << (h->device & 63);
    if (!(v->prepared & bit)) {
        const std::pair<const void*, size_t> ks[11] = {{v->k_fwd, fwd_smem(v->smem_fwd)},
                                                       {v->k_mirror_r, fwd_smem(v->smem_fused)},
                                                       {v->k_mirror_r_p, fwd_smem(v->smem_fused)},
                                                       {v->k_fused, fwd_smem(v->smem_fused)},
                                                       {v->k_mirror, fwd_smem(v->smem_fused)},
                                                       {v->k_recycle, fwd_smem(v->smem_fused)},
                                                       {v->k_fwd_p, fwd_smem(v->smem_fwd)},
                                                       {v->k_fused_p, fwd_smem(v->smem_fused)},
                                                       {v->k_mirror_p, fwd_smem(v->smem_fused)},
                                                       {v->k_recycle_p, fwd_smem(v->smem_fused)},
                                                       {v->k_tb, v->smem_tb}};
        for (const auto& k : ks) {
            cudaError_t e = cudaFuncSetAttribute(k.first, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(k.second));
            if (e != cudaSuccess) return cuda_fail(h, e, "cudaFuncSetAttribute");
        }
        v->prepared |= bit;
    }
    return PBVD_OK;
}

// One launch of a variant's kernel (compiled function or JIT cudaKernel_t).
// The traceback grid uses programmatic stream serialization (PDL): its CTAs
// may be scheduled once every forward CTA has signalled
// griddepcontrol.launch_dependents, and they wait (griddepcontrol.wait) for
// the forward grid's memory before touching survivors.
template <class Params>
cudaError_t launch(const void* k, int grid, int nt, size_t smem, cudaStream_t s, const Params& p,
                   bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(nt));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    if (pdl) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    void* args[1] = {const_cast<Params*>(&p)};
    return cudaLaunchKernelExC(&cfg, k, args);
}

int ensure_buf(pbvd_t h, void** p, size_t* cap, size_t bytes) {
    if (*cap >= bytes) return PBVD_OK;
    if (*p) {
        cudaFree(*p);   // synchronises the device: no pending kernel uses it
        *p = nullptr;
        *cap = 0;
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(h, PBVD_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    *cap = bytes;
    return PBVD_OK;
}

int record(pbvd_t h, cudaStream_t s) {
    if (!h->prof) return -1;
    const int i = int(h->ev_fwd.size() + h->ev_tb.size()) * 2;
    while (int(h->ev_pool.size()) <= i + 1) {
        cudaEvent_t ev;
        if (cudaEventCreate(&ev) != cudaSuccess) return -1;
        h->ev_pool.push_back(ev);
    }
    (void)s;
    return i;
}

// Block plan of block b (readings c-12, c-13, c-14, c-22).
struct BlockGeo {
    int64_t t0, t1, lo, hi;
};
BlockGeo geo(const pbvd_s* h, int64_t n_info, int64_t n_stages, int64_t nb, int64_t b) {
    BlockGeo g;
    g.t0 = b * h->D;
    g.t1 = std::min<int64_t>(g.t0 + h->D, n_info);
    g.lo = std::max<int64_t>(0, g.t0 - h->L);
    g.hi = (b == nb - 1) ? n_stages : std::min<int64_t>(n_stages, g.t1 + h->L);
    return g;
}

int run_blocks(pbvd_t h, Workspace& W, const int8_t* llr, int64_t ws0, int64_t n_llr_win,
               int64_t n_info, int64_t B0, int64_t nblk, uint8_t* out, cudaStream_t stream) {
    const Variant* v = h->var;
    const int64_t n_stages = n_info + ((h->flags & PBVD_TERMINATED) ? h->V : 0);
    const int64_t nb = (n_info + h->D - 1) / h->D;
    const int64_t B1 = B0 + nblk;
    if (B0 < 0 || nblk < 1 || B1 > nb) return fail(h, PBVD_EINVAL, "block range outside the stream");
    if (ws0 < 0 || ws0 > n_stages) return fail(h, PBVD_EINVAL, "window_stage0 outside the stream");
    const int64_t kb_ws0 = kept_before_h(h, ws0);
    {   // the window must cover every forward span of the range
        const BlockGeo a = geo(h, n_info, n_stages, nb, B0);
        const BlockGeo z = geo(h, n_info, n_stages, nb, B1 - 1);
        if (a.lo < ws0 || kept_before_h(h, z.hi) - kb_ws0 > n_llr_win)
            return fail(h, PBVD_ESIZE, "soft-value window does not cover the blocks' spans");
    }
    int rc = ensure_prepared(h, v);
    if (rc) return rc;
    // interior blocks: lo = bD - L > 0 (a span starting at stage 0 is a head
    // block with the known start state, reading c-12), b < nb-1,
    // (b+1)D + L <= n_stages
    const int64_t D = h->D, L = h->L;
    const int64_t first_int = L / D + 1;
    const int64_t last_int = std::min<int64_t>(nb - 2, (n_stages - L - D) >= 0 ? (n_stages - L - D) / D : -1);
    const int64_t I0 = std::min(std::max(first_int, B0), B1);
    const int64_t I1 = std::max(I0, std::min(last_int + 1, B1));
    std::vector<EdgeDesc> edges;
    auto add_edge = [&](int64_t b) {
        const BlockGeo g = geo(h, n_info, n_stages, nb, b);
        EdgeDesc e{};
        e.lo = g.lo;
        e.out_bit0 = g.t0 - B0 * D;
        e.span = int(g.hi - g.lo);
        e.t0r = int(g.t0 - g.lo);
        e.t1r = int(g.t1 - g.lo);
        e.flags = (g.lo == 0 ? EDGE_HEAD : 0) |
                  ((b == nb - 1 && (h->flags & PBVD_TERMINATED)) ? EDGE_START0 : 0);
        edges.push_back(e);
    };
    for (int64_t b = B0; b < I0; ++b) add_edge(b);
    for (int64_t b = I1; b < B1; ++b) add_edge(b);
    int span_edge_max = 0;
    for (const auto& e : edges) span_edge_max = std::max(span_edge_max, e.span);

    // ---- workspace: one wave of interior survivors + edge survivors + starts
    // interior spans are padded at the FRONT with `pad` erasure stages so
    // their length is a multiple of v: every chunk then runs whole v-stage
    // cycles of the one hot loop (no separate partial-chunk code -- which
    // thrashed the instruction cache).  With all-equal initial metrics and
    // lambda = 0 every stage adds the same BM' to every state, so the
    // metrics at the true span start are still all equal (reading c-11):
    // the decisions read by the traceback are unchanged.
    const int pad = int((h->V - (D + 2 * L) % h->V) % h->V);
    const int span_int = int(D + 2 * L) + pad;
    const size_t region_bytes = size_t(span_int) * v->ROW * 4;      // BPW blocks
    const int64_t n_int = I1 - I0;
    const size_t edge_region_bytes = size_t(span_edge_max) * v->ROW * 4;
    // edge survivor regions: one per edge of a launch (launches beyond
    // MAX_EDGE edges reuse them in stream order)
    const size_t n_edge_slots = std::min<size_t>(MAX_EDGE, edges.size());
    const size_t edge_bytes = edge_region_bytes * n_edge_slots + 2 * MAX_EDGE * 4 + 256;
    const int64_t unit = std::max<int64_t>(v->BPW, 128);   // multiple of BPW and TB CTA (128)
    int64_t wave = n_int;
    if (n_int > 0) {
        const size_t budget = h->ws_limit > edge_bytes ? h->ws_limit - edge_bytes : 0;
        const int64_t per_unit = int64_t((unit / v->BPW) * region_bytes + unit * 4);
        int64_t units = std::max<int64_t>(1, int64_t(budget) / per_unit);
        wave = std::min<int64_t>(n_int, units * unit);
    }
    const int64_t wave_regions = (wave + v->BPW - 1) / v->BPW;
    const size_t int_bytes = size_t(wave_regions) * region_bytes;
    const size_t start_bytes = size_t(wave + 64) * 4;
    const size_t need = ((int_bytes + 255) & ~size_t(255)) + ((edge_bytes + 255) & ~size_t(255)) +
                        ((start_bytes + 255) & ~size_t(255));
    rc = ensure_buf(h, &W.p, &W.bytes, need);
    if (rc) return rc;
    uint8_t* wsb = static_cast<uint8_t*>(W.p);
    uint32_t* dec_int = reinterpret_cast<uint32_t*>(wsb);
    uint32_t* dec_edge = reinterpret_cast<uint32_t*>(wsb + ((int_bytes + 255) & ~size_t(255)));
    int32_t* start_edge = reinterpret_cast<int32_t*>(
        reinterpret_cast<uint8_t*>(dec_edge) + edge_region_bytes * n_edge_slots);
    int32_t* start_int = reinterpret_cast<int32_t*>(
        wsb + ((int_bytes + 255) & ~size_t(255)) + ((edge_bytes + 255) & ~size_t(255)));

    FwdParams fp{};
    fp.D = int(D);
    fp.L = int(L);
    fp.span_int = span_int;
    fp.one = 1u;
    fp.neg_one = 0xffffffffu;
    fp.P = h->P;
    fp.kp = h->kp;
    fp.dtab = h->dtab;
    for (int i = 0; i < 16; ++i) fp.cum[i] = h->cum[i];
    fp.dec = dec_int;
    fp.start = start_int;
    fp.dec_edge = dec_edge;
    fp.start_edge = start_edge;
    fp.span_edge_max = span_edge_max;
    fp.out = out;
    fp.n_mirror = h->fused ? h->n_mirror : 0;
    for (int k = 0; k < MAX_MIRROR; ++k) fp.mirror[k] = h->mirror[k];
    fp.t0r = int(L) + pad;
    fp.t1r = int(L + D) + pad;
    fp.pad = pad;
    fp.start_zero = (h->flags & PBVD_START_ZERO) ? 1 : 0;

    TbParams tp{};
    tp.dec = dec_int;
    tp.start = start_int;
    tp.span_int = span_int;
    tp.t0r = int(L) + pad;
    tp.t1r = int(L + D) + pad;
    tp.D = int(D);
    tp.out = out;
    tp.dec_edge = dec_edge;
    tp.start_edge = start_edge;
    tp.span_edge_max = span_edge_max;
    tp.word_out = ((D & 31) == 0) && ((reinterpret_cast<uintptr_t>(out) & 3) == 0) &&
                  (((I0 - B0) * D) % 32 == 0);

    // ---- launch groups: interior waves; head edges ride with the first wave,
    // tail edges with the last (at most MAX_EDGE per launch; the kernel
    // addresses the soft window with 64-bit offsets, so a wave may be any size)
    struct Group {
        int64_t i0, i1;                 // interior blocks [i0, i1)
        std::vector<EdgeDesc> edges;
        std::vector<int64_t> eblk;      // block index of each edge
    };
    std::vector<Group> groups;
    // fused mode: a stream larger than one wave runs as ONE launch whose jobs
    // recycle the wave's survivor regions (job gw -> region gw % regions,
    // after the region's previous job has traced back), so there is a single
    // grid tail instead of one per wave; two-kernel mode keeps waves (its
    // traceback grid needs every region of the wave at once)
    static const bool env_recycle = [] { const char* e = std::getenv("PBVD_RECYCLE"); return !e || std::atoi(e) != 0; }();
    const bool recycle = h->fused && env_recycle && n_int > wave;
    const int64_t launch_blocks = recycle ? n_int : wave;
    for (int64_t d0 = 0; d0 < n_int || (n_int == 0 && groups.empty()); d0 += launch_blocks) {
        groups.push_back({I0 + d0, I0 + std::min(n_int, d0 + launch_blocks), {}, {}});
        if (n_int == 0) break;
    }
    const int64_t n_head = I0 - B0;
    for (size_t k = 0; k < edges.size(); ++k) {
        Group& g = (int64_t(k) < n_head) ? groups.front() : groups.back();
        g.edges.push_back(edges[k]);
        g.eblk.push_back(int64_t(k) < n_head ? B0 + int64_t(k) : I1 + (int64_t(k) - n_head));
    }
    auto group_range = [&](const Group& g, int64_t& klo, int64_t& khi) {
        int64_t slo = INT64_MAX, shi = -1;
        if (g.i1 > g.i0) {
            slo = geo(h, n_info, n_stages, nb, g.i0).lo;
            shi = geo(h, n_info, n_stages, nb, g.i1 - 1).hi;
        }
        for (const auto& ed : g.edges) {
            slo = std::min(slo, ed.lo);
            shi = std::max(shi, ed.lo + ed.span);
        }
        klo = kept_before_h(h, slo);
        khi = kept_before_h(h, shi);
    };
    {   // too many edges for one launch: the rest get their own launches
        std::vector<Group> out;
        for (auto& g : groups) {
            Group core{g.i0, g.i1, {}, {}};
            std::vector<Group> extra;
            for (size_t k = 0; k < g.edges.size(); ++k) {
                Group* tgt = nullptr;
                if (core.edges.size() < size_t(MAX_EDGE)) tgt = &core;
                if (!tgt) {
                    if (extra.empty() || extra.back().edges.size() >= size_t(MAX_EDGE))
                        extra.push_back({0, 0, {}, {}});
                    tgt = &extra.back();
                }
                tgt->edges.push_back(g.edges[k]);
                tgt->eblk.push_back(g.eblk[k]);
            }
            if (core.i1 > core.i0 || !core.edges.empty()) out.push_back(core);
            for (auto& x : extra) out.push_back(x);
        }
        groups.swap(out);
    }

    for (const Group& g : groups) {
        const int64_t cnt = g.i1 - g.i0;
        const int ne = int(g.edges.size());
        int64_t klo, khi;
        group_range(g, klo, khi);
        fp.llr = llr + (klo - kb_ws0);
        fp.kb_ws0 = klo;
        fp.n_llr = khi - klo;
        fp.b_int0 = g.i0;
        fp.n_int = int(cnt);
        fp.n_int_warps = int((cnt + v->BPW - 1) / v->BPW);
        fp.n_edge = ne;
        tp.n_int = fp.n_int;
        tp.n_int_ctas = int((cnt + v->NT_TB - 1) / v->NT_TB);
        tp.out_bit0 = (g.i0 - B0) * D;
        fp.out_bit0 = tp.out_bit0;
        fp.word_out = tp.word_out;
        tp.n_edge = ne;
        for (int i = 0; i < ne; ++i) {
            fp.edges[i] = g.edges[size_t(i)];
            tp.edges[i] = g.edges[size_t(i)];
        }
        const int fgrid = int((fp.n_int_warps + ne + v->NT / 32 - 1) / (v->NT / 32));
        fp.n_regions = 0;
        fp.region_done = nullptr;
        if (recycle && fp.n_int_warps > wave_regions) {
            // the two-kernel start array is free in fused mode: region counters
            fp.n_regions = int(wave_regions);
            fp.region_done = reinterpret_cast<unsigned*>(start_int);
            cudaError_t me = cudaMemsetAsync(fp.region_done, 0, size_t(wave_regions) * 4, stream);
            if (me != cudaSuccess) return cuda_fail(h, me, "cudaMemsetAsync (region counters)");
        }
        const int ev = record(h, stream);
        if (ev >= 0) cudaEventRecord(h->ev_pool[ev], stream);
#ifdef PBVD_EXP_TIMING
        // timing experiment: per-warp (start, forward end, traceback end, smid)
        static unsigned long long* dbg = nullptr;
        const char* dump = std::getenv("PBVD_TIMING_DUMP");
        const size_t ndbg = size_t(fgrid) * 32;
        if (dump) {
            if (dbg) cudaFree(dbg);
            cudaMalloc(&dbg, ndbg * 8);
            cudaMemsetAsync(dbg, 0, ndbg * 8, stream);
            fp.dbg = dbg;
        }
#endif
        const bool punct = h->P > 1;     // the PUNCT instantiations (depuncture in the transform)
        const void* kf = fp.n_mirror > 0 ? (fp.n_regions > 0 ? (punct ? v->k_mirror_r_p : v->k_mirror_r)
                                                             : (punct ? v->k_mirror_p : v->k_mirror))
                         : fp.n_regions > 0 ? (punct ? v->k_recycle_p : v->k_recycle)
                                            : (punct ? v->k_fused_p : v->k_fused);
        cudaError_t le = h->fused ? launch(kf, fgrid, v->NT, fwd_smem(v->smem_fused), stream, fp, false)
                                  : launch(punct ? v->k_fwd_p : v->k_fwd, fgrid, v->NT,
                                           fwd_smem(v->smem_fwd), stream, fp, false);
        if (le != cudaSuccess) return cuda_fail(h, le, "forward kernel launch");
#ifdef PBVD_EXP_TIMING
        if (dump) {
            std::vector<unsigned long long> hb(ndbg);
            cudaMemcpyAsync(hb.data(), dbg, ndbg * 8, cudaMemcpyDeviceToHost, stream);
            cudaStreamSynchronize(stream);
            if (FILE* f = std::fopen(dump, "wb")) {
                std::fwrite(hb.data(), 8, ndbg, f);
                std::fclose(f);
            }
            fp.dbg = nullptr;
        }
#endif
        if (ev >= 0) {
            cudaEventRecord(h->ev_pool[ev + 1], stream);
            h->ev_fwd.push_back({ev, ev + 1});
        }
        h->launches += 1;
        if (!h->fused) {
            const int ev2 = record(h, stream);
            if (ev2 >= 0) cudaEventRecord(h->ev_pool[ev2], stream);
            le = launch(v->k_tb, tp.n_int_ctas + ne, v->NT_TB, v->smem_tb, stream, tp, true);
            if (le != cudaSuccess) return cuda_fail(h, le, "traceback kernel launch");
            if (ev2 >= 0) {
                cudaEventRecord(h->ev_pool[ev2 + 1], stream);
                h->ev_tb.push_back({ev2, ev2 + 1});
            }
            h->launches += 1;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(h, e, "kernel launch");
    }
    if (!h->fused && h->n_mirror > 0) {
        // two-kernel mode: the mirrors get the call's output by copies after
        // the traceback (fused mode copies inside the kernel, per warp)
        const int64_t nbytes = (std::min<int64_t>(B1 * D, n_info) - B0 * D + 7) / 8;
        for (int k = 0; k < h->n_mirror; ++k) {
            cudaError_t e = cudaMemcpyAsync(out + h->mirror[k], out, size_t(nbytes), cudaMemcpyDefault,
                                            stream);
            if (e != cudaSuccess) return cuda_fail(h, e, "mirror copy");
        }
    }
    return PBVD_OK;
}

// The variant that runs (K, R, polys) with `lanes` lanes per block pair (0 =
// the code's default): a compiled one if any, else a JIT build (jit.cu).
const Variant* select_variant(int K, int R, const uint32_t* polys, int lanes, std::string* why) {
    const Variant* best = nullptr;
    for (const auto& v : variants()) {
        if (v.K != K || v.R != R) continue;
        bool same = true;
        for (int r = 0; r < R; ++r) same &= (v.polys[r] == polys[r]);
        if (!same) continue;
        if (lanes == 0 ? (!best || v.default_rank < best->default_rank) : v.W == lanes) best = &v;
    }
    if (best) return best;
    return jit_variant(K, R, polys, lanes == 0 ? default_lanes(K) : lanes, why);
}

// The host pipeline's variant (see pbvd_s::host_var): among the COMPILED
// variants of the code (no extra JIT build), the one with the most lanes per
// pair that keeps >= 16 states per lane; else `dflt`.
const Variant* latency_variant(int K, int R, const uint32_t* polys, const Variant* dflt) {
    const Variant* best = dflt;
    for (const auto& v : variants()) {
        if (v.K != K || v.R != R || (1 << (K - 1)) / v.W < 16) continue;
        bool same = true;
        for (int r = 0; r < R; ++r) same &= (v.polys[r] == polys[r]);
        if (same && v.W > best->W) best = &v;
    }
    return best;
}

thread_local std::string g_create_err;   // pbvd_last_error(NULL)

int create_fail(int code, const std::string& msg) {
    g_create_err = msg;
    return code;
}

}  // namespace

extern "C" {

int pbvd_create(pbvd_t* out, int K, int R, const uint32_t* polys, int punct_period,
                const uint8_t* punct, int D, int L, int soft_bits, unsigned flags, int device) {
    g_create_err.clear();
    if (!out) return create_fail(PBVD_EINVAL, "null handle pointer");
    *out = nullptr;
    if (!polys || K < 3 || K > 12 || R < 2 || R > 4)
        return create_fail(PBVD_EINVAL, "need 3 <= K <= 12, 2 <= R <= 4 and a polynomial list");
    if (punct_period < 1 || punct_period > 16 || R * punct_period > 64)
        return create_fail(PBVD_EINVAL, "puncture period out of range");
    if ((punct_period > 1) != (punct != nullptr))
        return create_fail(PBVD_EINVAL, "puncture matrix must be given iff period > 1");
    if (D < 8 || (D % 8) != 0 || L < 1 || D > (1 << 24) || L > (1 << 20))
        return create_fail(PBVD_EINVAL, "need D >= 8, D % 8 == 0, L >= 1");
    if (soft_bits < 1 || soft_bits > 8) return create_fail(PBVD_EINVAL, "soft_bits outside 1..8");
    if (flags & ~(PBVD_TERMINATED | PBVD_ALLOW_CATASTROPHIC | PBVD_START_ZERO))
        return create_fail(PBVD_EINVAL, "unknown flag");
    uint32_t lead = 0, trail = 0;
    for (int r = 0; r < R; ++r) {
        if (polys[r] == 0 || polys[r] >= (1u << K))
            return create_fail(PBVD_EINVAL, "generator polynomial outside [1, 2^K)");
        lead |= (polys[r] >> (K - 1)) & 1u;
        trail |= polys[r] & 1u;
    }
    // leading / trailing coefficient rule of new_code: without
    // them the code's constraint length is not K; warning-class, overridable
    if (!(lead && trail) && !(flags & PBVD_ALLOW_CATASTROPHIC))
        return create_fail(PBVD_EINVAL, "no generator has the g_{K-1} (or g_0) tap; "
                                        "pass PBVD_ALLOW_CATASTROPHIC to decode it anyway");
    if (punct_period > 1) {
        int kept = 0;
        for (int i = 0; i < R * punct_period; ++i) kept += punct[i] ? 1 : 0;
        if (kept == 0) return create_fail(PBVD_EINVAL, "puncture matrix keeps no position");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return create_fail(PBVD_ECUDA, "no such CUDA device");
    }
    std::string why;
    const Variant* best = select_variant(K, R, polys, 0, &why);
    if (!best) return create_fail(PBVD_EUNSUPPORTED, why);
    const Variant* hbest = latency_variant(K, R, polys, best);
    pbvd_s* h = new (std::nothrow) pbvd_s();
    if (!h) return create_fail(PBVD_ENOMEM, "handle allocation");
    h->device = device;
    h->K = K;
    h->R = R;
    h->V = K - 1;
    h->N = 1 << (K - 1);
    for (int r = 0; r < R; ++r) h->polys[r] = polys[r];
    h->P = punct_period;
    h->D = D;
    h->L = L;
    h->soft_bits = soft_bits;
    h->flags = flags;
    h->var = best;
    h->host_var = hbest;
    if (punct_period > 1) {
        int kp = 0;
        for (int p = 0; p < punct_period; ++p) {
            h->cum[p] = kp;
            for (int r = 0; r < R; ++r) {
                const uint8_t k = punct[r * punct_period + p] ? 1 : 0;
                h->punct[r * punct_period + p] = k;
                if (k) h->keep |= uint64_t(1) << (r * punct_period + p);
                kp += k;
            }
        }
        if (kp == 0) {
            delete h;
            return create_fail(PBVD_EINVAL, "puncture matrix keeps no position");
        }
        h->kp = kp;
    } else {
        h->kp = R;
        h->keep = (uint64_t(1) << R) - 1;
    }
    if (punct_period > 1) {
        // depuncture table for the forward kernel (FwdParams::dtab): for a
        // chunk of T stages starting at phase ph0, dense word w (bytes 4w..4w+3
        // of the [stage][r] window) = PRMT(4 kept bytes from kept index base,
        // 0, sel); erasures select a byte of the zero operand (c-18)
        const int T = best->T, P = punct_period;
        const int nwd = (T * R + 3) / 4;
        std::vector<uint32_t> tab(size_t(P) * nwd);
        for (int ph0 = 0; ph0 < P; ++ph0) {
            std::vector<int> kidx(size_t(4) * nwd + 1), nextk(size_t(4) * nwd + 1);
            int ki = 0;
            for (int d = 0; d < 4 * nwd; ++d) {
                const int st = d / R, r = d % R, ph = (ph0 + st) % P;
                nextk[size_t(d)] = ki;
                kidx[size_t(d)] = h->punct[r * P + ph] ? ki++ : -1;
            }
            for (int w = 0; w < nwd; ++w) {
                int base = nextk[size_t(4 * w)];
                uint32_t sel = 0;
                for (int k = 0; k < 4; ++k) {
                    const int ix = kidx[size_t(4 * w + k)];
                    sel |= uint32_t(ix >= 0 ? ix - base : 4) << (4 * k);
                }
                tab[size_t(ph0) * nwd + w] = sel | (uint32_t(base) << 16);
            }
        }
        DeviceGuard g(device);
        if (cudaMalloc(&h->dtab, tab.size() * 4) != cudaSuccess ||
            cudaMemcpy(h->dtab, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            if (h->dtab) cudaFree(h->dtab);
            delete h;
            return create_fail(PBVD_ENOMEM, "depuncture table");
        }
    }
    *out = h;
    return PBVD_OK;
}

void pbvd_destroy(pbvd_t h) {
    if (!h) return;
    {
        DeviceGuard g(h->device);
        if (h->dtab) cudaFree(h->dtab);
        if (h->ws.p) cudaFree(h->ws.p);
        for (auto& ln : h->lanes) {
            if (ln.ws.p) cudaFree(ln.ws.p);
            if (ln.d_llr) cudaFree(ln.d_llr);
            if (ln.d_bits) cudaFree(ln.d_bits);
            if (ln.stream) cudaStreamDestroy(ln.stream);
            if (ln.in_ready) cudaEventDestroy(ln.in_ready);
            if (ln.consumed) cudaEventDestroy(ln.consumed);
        }
        for (auto ev : h->ev_pool) cudaEventDestroy(ev);
        if (h->h2d) cudaStreamDestroy(h->h2d);
    }
    delete h;
}

int64_t pbvd_stage_count(pbvd_t h, int64_t n_info) {
    if (!h) return PBVD_EINVAL;
    if (n_info < 1) return fail(h, PBVD_EINVAL, "n_info < 1");
    return n_info + ((h->flags & PBVD_TERMINATED) ? h->V : 0);
}

int64_t pbvd_block_count(pbvd_t h, int64_t n_info) {
    if (!h) return PBVD_EINVAL;
    if (n_info < 1) return fail(h, PBVD_EINVAL, "n_info < 1");
    return (n_info + h->D - 1) / h->D;
}

int64_t pbvd_llr_count(pbvd_t h, int64_t n_info) {
    if (!h) return PBVD_EINVAL;
    if (n_info < 1) return fail(h, PBVD_EINVAL, "n_info < 1");
    return kept_before_h(h, pbvd_stage_count(h, n_info));
}

int pbvd_decode_blocks(pbvd_t h, const int8_t* d_llr_window, int64_t window_stage0,
                       int64_t window_n_llr, int64_t n_info_total, int64_t block0,
                       int64_t nblocks, uint8_t* d_bits, void* stream) {
    if (!h) return PBVD_EINVAL;
    if (!d_llr_window || !d_bits || n_info_total < 1 || window_n_llr < 1)
        return fail(h, PBVD_EINVAL, "null pointer or empty stream");
    DeviceGuard g(h->device);
    h->ev_fwd.clear();
    h->ev_tb.clear();
    h->launches = 0;
    return run_blocks(h, h->ws, d_llr_window, window_stage0, window_n_llr, n_info_total, block0,
                      nblocks, d_bits, static_cast<cudaStream_t>(stream));
}

int pbvd_decode_blocks_mirrored(pbvd_t h, const int8_t* d_llr_window, int64_t window_stage0,
                                int64_t window_n_llr, int64_t n_info_total, int64_t block0,
                                int64_t nblocks, uint8_t* d_bits, uint8_t* const* d_mirrors,
                                int n_mirrors, void* stream) {
    if (!h) return PBVD_EINVAL;
    if (n_mirrors < 0 || n_mirrors > MAX_MIRROR || (n_mirrors > 0 && !d_mirrors) || !d_bits)
        return fail(h, PBVD_EINVAL, "0..7 mirror destinations");
    for (int k = 0; k < n_mirrors; ++k) {
        const int64_t d = reinterpret_cast<intptr_t>(d_mirrors[k]) - reinterpret_cast<intptr_t>(d_bits);
        if (!d_mirrors[k] || (d & 3)) return fail(h, PBVD_EINVAL, "mirror null or not congruent to d_bits mod 4");
        h->mirror[k] = d;
    }
    h->n_mirror = n_mirrors;
    const int rc = pbvd_decode_blocks(h, d_llr_window, window_stage0, window_n_llr, n_info_total,
                                      block0, nblocks, d_bits, stream);
    h->n_mirror = 0;
    return rc;
}

int pbvd_decode(pbvd_t h, const int8_t* d_llr, int64_t n_llr, uint8_t* d_bits, int64_t n_info,
                void* stream) {
    if (!h) return PBVD_EINVAL;
    if (!d_llr || !d_bits || n_info < 1) return fail(h, PBVD_EINVAL, "null pointer or empty stream");
    if (n_llr != pbvd_llr_count(h, n_info))
        return fail(h, PBVD_ESIZE, "n_llr != pbvd_llr_count(n_info)");
    return pbvd_decode_blocks(h, d_llr, 0, n_llr, n_info, 0, pbvd_block_count(h, n_info), d_bits,
                              stream);
}

int pbvd_decode_host(pbvd_t h, const int8_t* h_llr_window, int64_t window_stage0,
                     int64_t window_n_llr, int64_t n_info_total, int64_t block0, int64_t nblocks,
                     uint8_t* h_bits, int n_streams) {
    if (!h) return PBVD_EINVAL;
    if (!h_llr_window || !h_bits || n_info_total < 1 || window_n_llr < 1)
        return fail(h, PBVD_EINVAL, "null pointer or empty stream");
    const int64_t n_stages = n_info_total + ((h->flags & PBVD_TERMINATED) ? h->V : 0);
    const int64_t nb = (n_info_total + h->D - 1) / h->D;
    if (block0 < 0 || nblocks < 1 || block0 + nblocks > nb)
        return fail(h, PBVD_EINVAL, "block range outside the stream");
    if (n_streams < 1) n_streams = 1;
    if (n_streams > 8) n_streams = 8;
    DeviceGuard g(h->device);
    h->ev_fwd.clear();
    h->ev_tb.clear();
    h->launches = 0;
    const bool prof = h->prof;
    h->prof = false;                       // events are per caller stream only
    const Variant* var_saved = h->var;
    h->var = h->host_var;
    const int64_t kb0 = kept_before_h(h, window_stage0);
    // Pipeline (§IV.C, B200 form): every H2D copy goes through ONE
    // stream, in order, so each runs at the full link rate (copies on several
    // streams run concurrently on several copy engines and only share the
    // link); segment k's decode (and its D2H) runs on lane k % n_streams as
    // soon as its copy has landed, while later copies continue.  A lane's
    // staging buffer is refilled only after its previous decode has read it.
    // The stream is PCIe-bound, so what is left after the last H2D byte is
    // one segment's decode latency plus its D2H.
    // Segment plan: at least 4 and at most 4 per stream equal segments
    // (>= 16384 blocks each beyond 4: every H2D copy costs a few us of setup,
    // and a segment's decode must end before the next copy does), then a
    // small last one (4096 blocks: one warp per sub-partition, so its decode
    // -- all that is left after the last copy -- takes one lone warp's latency
    // and its D2H is short).  Measured (tools/e2e_sweep.py): C4 +8 %, C3a +4 %
    // e2e, C2 unchanged against 4 equal segments.  PBVD_HOST_NSEG /
    // PBVD_HOST_LAST override the plan.
    static const int64_t env_nseg = [] { const char* e = std::getenv("PBVD_HOST_NSEG"); return e ? std::atoll(e) : 0; }();
    static const int64_t env_last = [] { const char* e = std::getenv("PBVD_HOST_LAST"); return e ? std::atoll(e) : -1; }();
    int64_t last = env_last >= 0 ? env_last : (nblocks >= 4 * 4096 ? 4096 : 0);
    if (last >= nblocks) last = 0;
    const int64_t big_min = 16384;
    int64_t n_big = env_nseg > 0 ? env_nseg
                                 : std::max<int64_t>(4, std::min<int64_t>(4 * n_streams,
                                                                          (nblocks - last) / big_min));
    n_big = std::max<int64_t>(1, std::min(n_big, nblocks - last));
    const int64_t seg = (nblocks - last + n_big - 1) / n_big;
    std::vector<int64_t> seg_b0;
    for (int64_t b = block0; b < block0 + nblocks - last; b += seg) seg_b0.push_back(b);
    if (last > 0) seg_b0.push_back(block0 + nblocks - last);
    const int64_t nseg = int64_t(seg_b0.size());
    const int64_t seg_max = std::max(seg, last);
    if (!h->h2d && cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking) != cudaSuccess) {
        h->prof = prof;
        h->var = var_saved;
        return cuda_fail(h, cudaGetLastError(), "cudaStreamCreate");
    }
    while (int(h->lanes.size()) < n_streams) {
        HostLane ln;
        if (cudaStreamCreateWithFlags(&ln.stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ln.in_ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ln.consumed, cudaEventDisableTiming) != cudaSuccess) {
            h->prof = prof;
            h->var = var_saved;
            return cuda_fail(h, cudaGetLastError(), "cudaStreamCreate / cudaEventCreate");
        }
        h->lanes.push_back(ln);
    }
    int rc = PBVD_OK;
    const int64_t bit_base = block0 * h->D;
    // staging buffers sized for the largest segment, before any copy is queued
    for (int i = 0; i < n_streams && rc == PBVD_OK; ++i) {
        HostLane& ln = h->lanes[size_t(i)];
        const BlockGeo ga = geo(h, n_info_total, n_stages, nb, block0);
        const BlockGeo gz = geo(h, n_info_total, n_stages, nb, std::min(block0 + nblocks, block0 + seg_max) - 1);
        const int64_t span_max = (gz.hi - ga.lo) + 2 * (h->L + h->V) + h->D;
        rc = ensure_buf(h, reinterpret_cast<void**>(&ln.d_llr), &ln.llr_cap,
                        size_t(kept_before_h(h, span_max) + h->R * 16));
        if (!rc) rc = ensure_buf(h, reinterpret_cast<void**>(&ln.d_bits), &ln.bits_cap,
                                 size_t((seg_max * h->D + 7) / 8));
        if (!rc) {
            cudaEventRecord(ln.consumed, ln.stream);   // buffers free
        }
    }
    for (int64_t k = 0; k < nseg && rc == PBVD_OK; ++k) {
        HostLane& ln = h->lanes[size_t(k % n_streams)];
        const int64_t b0 = seg_b0[size_t(k)];
        const int64_t b1 = (k + 1 < nseg) ? seg_b0[size_t(k + 1)] : block0 + nblocks;
        const BlockGeo ga = geo(h, n_info_total, n_stages, nb, b0);
        const BlockGeo gz = geo(h, n_info_total, n_stages, nb, b1 - 1);
        const int64_t k0 = kept_before_h(h, ga.lo), k1 = kept_before_h(h, gz.hi);
        if (ga.lo < window_stage0 || k1 - kb0 > window_n_llr) {
            rc = fail(h, PBVD_ESIZE, "soft-value window does not cover the blocks' spans");
            break;
        }
        const size_t nllr = size_t(k1 - k0);
        const int64_t t0 = b0 * h->D, t1 = std::min<int64_t>(b1 * h->D, n_info_total);
        const size_t nbytes = size_t((t1 - t0 + 7) / 8);
        if (nllr > ln.llr_cap || nbytes > ln.bits_cap) {
            rc = fail(h, PBVD_ENOMEM, "host pipeline staging buffer too small");
            break;
        }
        // H2D on the copy stream once the lane's previous decode has read
        // the buffer
        cudaError_t e = cudaStreamWaitEvent(h->h2d, ln.consumed, 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(ln.d_llr, h_llr_window + (k0 - kb0), nllr, cudaMemcpyHostToDevice,
                                h->h2d);
        if (e == cudaSuccess) e = cudaEventRecord(ln.in_ready, h->h2d);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ln.stream, ln.in_ready, 0);
        if (e != cudaSuccess) {
            rc = cuda_fail(h, e, "cudaMemcpyAsync H2D");
            break;
        }
        rc = run_blocks(h, ln.ws, ln.d_llr, ga.lo, int64_t(nllr), n_info_total, b0, b1 - b0,
                        ln.d_bits, ln.stream);
        if (rc) break;
        e = cudaEventRecord(ln.consumed, ln.stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(h_bits + (t0 - bit_base) / 8, ln.d_bits, nbytes,
                                cudaMemcpyDeviceToHost, ln.stream);
        if (e != cudaSuccess) rc = cuda_fail(h, e, "cudaMemcpyAsync D2H");
    }
    {
        cudaError_t e = cudaStreamSynchronize(h->h2d);
        if (!rc && e != cudaSuccess) rc = cuda_fail(h, e, "host pipeline H2D");
    }
    for (int i = 0; i < n_streams; ++i) {
        cudaError_t e = cudaStreamSynchronize(h->lanes[size_t(i)].stream);
        if (!rc && e != cudaSuccess) rc = cuda_fail(h, e, "decode (host pipeline)");
    }
    h->prof = prof;
    h->var = var_saved;
    return rc;
}

// ---- continuous stream (the SDR use case) --------
// Soft values arrive in pieces of any length; every block whose forward span
// [bD-L, bD+D+L) has fully arrived (and which provably is not the last block)
// is decoded as soon as its data is there, with exactly the geometry the
// one-shot decode of the concatenated stream gives it, so the
// concatenated output equals pbvd_decode's.  The soft values a later block
// still needs (its L-stage halo) are carried over in a device window.

struct pbvd_stream_s {
    pbvd_t h = nullptr;
    int8_t* buf[2] = {nullptr, nullptr};
    size_t cap[2] = {0, 0};
    int cur = 0;
    int64_t win_stage0 = 0;   // buf[cur][0] = first kept value of this stage
    int64_t kwin0 = 0;        // = kept_before(win_stage0)
    int64_t received = 0;     // kept values pushed so far
    int64_t next_block = 0;   // first block not yet emitted
};

namespace {

// complete stages among the first k kept soft values
int64_t stages_complete(const pbvd_s* h, int64_t k) {
    if (h->P == 1) return k / h->R;
    const int64_t full = k / h->kp, rem = k % h->kp;
    int p = 0;
    while (p + 1 < h->P && h->cum[p + 1] <= rem) ++p;
    // column p is complete iff all its kept values arrived
    const int kept_p = (p + 1 < h->P ? h->cum[p + 1] : h->kp) - h->cum[p];
    const int64_t in_period = (rem - h->cum[p] >= kept_p) ? p + 1 : p;
    return full * h->P + in_period;
}

}  // namespace

int pbvd_stream_open(pbvd_t h, pbvd_stream_t* out) {
    if (!h || !out) return PBVD_EINVAL;
    *out = new (std::nothrow) pbvd_stream_s();
    if (!*out) return fail(h, PBVD_ENOMEM, "stream allocation");
    (*out)->h = h;
    return PBVD_OK;
}

void pbvd_stream_close(pbvd_stream_t s) {
    if (!s) return;
    {
        DeviceGuard g(s->h->device);
        for (auto* b : s->buf)
            if (b) cudaFree(b);
    }
    delete s;
}

int pbvd_stream_push(pbvd_stream_t s, const int8_t* d_llr, int64_t n_llr, uint8_t* d_bits,
                     int64_t bits_cap, int64_t* n_bits, void* stream) {
    if (!s || n_llr < 0 || (n_llr > 0 && !d_llr) || !n_bits) return PBVD_EINVAL;
    pbvd_t h = s->h;
    *n_bits = 0;
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t D = h->D, tailv = (h->flags & PBVD_TERMINATED) ? h->V : 0;
    // blocks b with (b+1)D + max(L, tail+1) <= received stages: the whole span
    // has arrived and b is not the last block (n_info > (b+1)D)
    const int64_t st_rx = stages_complete(h, s->received + n_llr);
    const int64_t margin = std::max<int64_t>(h->L, tailv + 1);
    const int64_t ready = std::max(s->next_block, st_rx >= margin ? (st_rx - margin) / D : 0);
    const int64_t nbits = (ready - s->next_block) * D;
    if (nbits > 0 && (!d_bits || bits_cap * 8 < nbits))
        return fail(h, PBVD_ESIZE, "stream output buffer too small (nothing consumed)");
    // carry: the soft values from the first stage a pending block reads
    const int64_t s0 = std::max<int64_t>(0, s->next_block * D - h->L);
    const int64_t k0 = kept_before_h(h, s0);
    const int64_t keep_n = s->received - k0;            // retained values
    const size_t need = size_t(keep_n + n_llr);
    if (need > 0) {
        const bool in_place = (k0 == s->kwin0) && s->cap[s->cur] >= need && s->buf[s->cur];
        if (!in_place) {
            const int nx = 1 - s->cur;
            if (s->cap[nx] < need) {
                int rc = ensure_buf(h, reinterpret_cast<void**>(&s->buf[nx]), &s->cap[nx],
                                    std::max(need, s->cap[nx] + s->cap[nx] / 2));
                if (rc) return rc;
            }
            if (keep_n > 0) {
                cudaError_t e = cudaMemcpyAsync(s->buf[nx], s->buf[s->cur] + (k0 - s->kwin0),
                                                size_t(keep_n), cudaMemcpyDeviceToDevice, st);
                if (e != cudaSuccess) return cuda_fail(h, e, "stream carry copy");
            }
            s->cur = nx;
            s->kwin0 = k0;
            s->win_stage0 = s0;
        }
        if (n_llr > 0) {
            cudaError_t e = cudaMemcpyAsync(s->buf[s->cur] + (s->received - s->kwin0), d_llr,
                                            size_t(n_llr), cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(h, e, "stream append copy");
        }
    }
    s->received += n_llr;
    if (nbits == 0) return PBVD_OK;
    // the geometry of these blocks is the same for any n_info > ready*D: use
    // the stages received so far
    h->ev_fwd.clear();
    h->ev_tb.clear();
    h->launches = 0;
    int rc = run_blocks(h, h->ws, s->buf[s->cur], s->win_stage0, s->received - s->kwin0,
                        st_rx - tailv, s->next_block, ready - s->next_block, d_bits, st);
    if (rc) return rc;
    s->next_block = ready;
    *n_bits = nbits;
    return PBVD_OK;
}

int pbvd_stream_finish(pbvd_stream_t s, uint8_t* d_bits, int64_t bits_cap, int64_t* n_bits,
                       void* stream) {
    if (!s || !n_bits) return PBVD_EINVAL;
    pbvd_t h = s->h;
    *n_bits = 0;
    DeviceGuard g(h->device);
    const int64_t tailv = (h->flags & PBVD_TERMINATED) ? h->V : 0;
    const int64_t n_stages = stages_complete(h, s->received);
    const int64_t n_info = n_stages - tailv;
    int rc = PBVD_OK;
    if (kept_before_h(h, n_stages) != s->received || n_info < 1) {
        rc = fail(h, PBVD_ESIZE, "stream ends inside a stage or holds no info bit");
    } else {
        const int64_t nb = (n_info + h->D - 1) / h->D;
        const int64_t nbits = n_info - s->next_block * h->D;
        if (nbits > 0) {
            if (!d_bits || bits_cap < (nbits + 7) / 8) {
                rc = fail(h, PBVD_ESIZE, "stream output buffer too small");
            } else {
                h->ev_fwd.clear();
                h->ev_tb.clear();
                h->launches = 0;
                rc = run_blocks(h, h->ws, s->buf[s->cur], s->win_stage0, s->received - s->kwin0,
                                n_info, s->next_block, nb - s->next_block, d_bits,
                                static_cast<cudaStream_t>(stream));
                if (!rc) *n_bits = nbits;
            }
        }
    }
    // the stream object is ready for the next stream (buffers kept)
    s->cur = 0;
    s->win_stage0 = s->kwin0 = s->received = s->next_block = 0;
    return rc;
}

int pbvd_set_lanes(pbvd_t h, int lanes) {
    if (!h) return PBVD_EINVAL;
    std::string why;
    const Variant* best = select_variant(h->K, h->R, h->polys, lanes, &why);
    if (!best) return fail(h, PBVD_EUNSUPPORTED, why);
    h->var = best;
    h->host_var = lanes == 0 ? latency_variant(h->K, h->R, h->polys, best) : best;
    return PBVD_OK;
}

int pbvd_get_lanes(pbvd_t h) { return h ? h->var->W : PBVD_EINVAL; }

int pbvd_set_fused(pbvd_t h, int fused) {
    if (!h) return PBVD_EINVAL;
    h->fused = fused != 0;
    return PBVD_OK;
}

int pbvd_get_fused(pbvd_t h) { return h ? int(h->fused) : PBVD_EINVAL; }

int pbvd_set_workspace_limit(pbvd_t h, size_t bytes) {
    if (!h) return PBVD_EINVAL;
    if (bytes < (size_t(1) << 20)) return fail(h, PBVD_EINVAL, "workspace limit below 1 MiB");
    h->ws_limit = bytes;
    return PBVD_OK;
}

int pbvd_set_profiling(pbvd_t h, int enable) {
    if (!h) return PBVD_EINVAL;
    h->prof = enable != 0;
    return PBVD_OK;
}

int pbvd_kernel_times(pbvd_t h, float* fwd_ms, float* tb_ms, int* launches) {
    if (!h) return PBVD_EINVAL;
    DeviceGuard g(h->device);
    float f = 0.f, t = 0.f;
    for (auto& pr : h->ev_fwd) {
        float ms = 0.f;
        cudaError_t e = cudaEventElapsedTime(&ms, h->ev_pool[pr.first], h->ev_pool[pr.second]);
        if (e != cudaSuccess) return cuda_fail(h, e, "cudaEventElapsedTime");
        f += ms;
    }
    for (auto& pr : h->ev_tb) {
        float ms = 0.f;
        cudaError_t e = cudaEventElapsedTime(&ms, h->ev_pool[pr.first], h->ev_pool[pr.second]);
        if (e != cudaSuccess) return cuda_fail(h, e, "cudaEventElapsedTime");
        t += ms;
    }
    if (fwd_ms) *fwd_ms = f;
    if (tb_ms) *tb_ms = t;
    if (launches) *launches = h->launches;
    return PBVD_OK;
}

int pbvd_get_info(pbvd_t h, pbvd_info* info) {
    if (!h || !info) return PBVD_EINVAL;
    info->K = h->K;
    info->R = h->R;
    info->N = h->N;
    info->lanes = h->var->W;
    info->D = h->D;
    info->L = h->L;
    info->P = h->P;
    info->span = h->D + 2 * h->L;
    info->dec_bytes_per_block = int64_t(h->D + 2 * h->L) * (h->N / 8 > 0 ? h->N / 8 : 1);
    info->jit = h->var->jit ? 1 : 0;
    info->host_lanes = h->host_var->W;
    info->workspace_bytes = h->ws.bytes;
    for (const auto& ln : h->lanes) info->workspace_bytes += ln.ws.bytes;
    return PBVD_OK;
}

const char* pbvd_supported(void) {
    static std::string s;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const auto& v : variants()) {
            char buf[96];
            std::snprintf(buf, sizeof buf, "%d:%d:", v.K, v.R);
            s += buf;
            for (int r = 0; r < v.R; ++r) {
                std::snprintf(buf, sizeof buf, "%s%o", r ? "," : "", v.polys[r]);
                s += buf;
            }
            std::snprintf(buf, sizeof buf, ":%d;", v.W);
            s += buf;
        }
    });
    return s.c_str();
}

const char* pbvd_strerror(int code) {
    switch (code) {
        case PBVD_OK: return "ok";
        case PBVD_EINVAL: return "invalid argument";
        case PBVD_ENOMEM: return "out of memory";
        case PBVD_ECUDA: return "CUDA error";
        case PBVD_EUNSUPPORTED: return "unsupported code shape or lane count (no compiled or JIT kernel)";
        case PBVD_ESIZE: return "buffer size inconsistent with n_info";
        default: return "unknown error";
    }
}

const char* pbvd_last_error(pbvd_t h) { return h ? h->err.c_str() : g_create_err.c_str(); }

// ---- gather buffers across processes (CUDA IPC; the fused gather of P:112)
namespace {
// cuMemGetAddressRange through the runtime's driver entry point (the library
// links cudart statically and not libcuda)
typedef int (*AddrRangeFn)(uintptr_t*, size_t*, uintptr_t);
AddrRangeFn addr_range_fn() {
    static AddrRangeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return AddrRangeFn(nullptr);
        return reinterpret_cast<AddrRangeFn>(f);
    }();
    return fn;
}
}  // namespace

int pbvd_ipc_export(const void* d_ptr, void* handle, int64_t* offset) {
    if (!d_ptr || !handle || !offset) return create_fail(PBVD_EINVAL, "null argument");
    AddrRangeFn fn = addr_range_fn();
    if (!fn) return create_fail(PBVD_ECUDA, "cuMemGetAddressRange unavailable");
    uintptr_t base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<uintptr_t>(d_ptr)) != 0)
        return create_fail(PBVD_EINVAL, "not a device allocation");
    cudaIpcMemHandle_t hd;
    cudaError_t e = cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return create_fail(PBVD_ECUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    }
    static_assert(sizeof(hd) == PBVD_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &hd, sizeof(hd));
    *offset = int64_t(reinterpret_cast<uintptr_t>(d_ptr) - base);
    return PBVD_OK;
}

int pbvd_ipc_open(const void* handle, int64_t offset, int device, void** d_ptr) {
    if (!handle || !d_ptr || offset < 0) return create_fail(PBVD_EINVAL, "null argument");
    DeviceGuard g(device);
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle, sizeof(hd));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return create_fail(PBVD_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    }
    *d_ptr = static_cast<uint8_t*>(base) + offset;
    return PBVD_OK;
}

int pbvd_ipc_close(void* d_ptr, int64_t offset, int device) {
    if (!d_ptr || offset < 0) return create_fail(PBVD_EINVAL, "null argument");
    DeviceGuard g(device);
    cudaError_t e = cudaIpcCloseMemHandle(static_cast<uint8_t*>(d_ptr) - offset);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return create_fail(PBVD_ECUDA, std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e));
    }
    return PBVD_OK;
}

}  // extern "C"
