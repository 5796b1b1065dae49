// jit.cu -- run-time kernels for codes with no compiled variant (SURVEY
// §8(f) NEXT 4: any generator polynomials, K 3..12, R 2..4).
//
// The forward / traceback kernels are templates on the code (the generator
// columns fix the butterfly groups of Eqs. 3-6, at compile time,
// so the branch metrics index registers statically).  For a code that is not
// instantiated in a kern_*.cu file, the SAME templates (fwd.cuh, tb.cuh) are
// compiled for sm_100a by NVRTC when the decoder is created, loaded with
// cudaLibraryLoadData and launched through the same Variant table as the
// compiled kernels.  Only the launch constants are needed on the host; they
// do not depend on the polynomials, so they come from the host instantiation
// of Cfg<> for the (K, R, W) shape (variant_shape below).
//
// NVRTC is loaded with dlopen on first use (no link-time dependency); the
// kernel sources are read from the package's csrc/ directory next to
// libpbvd.so (override: PBVD_JIT_SRC), with csrc/jit_std/ mapping the three
// standard headers the templates use onto libcu++.  Built cubins are cached
// in-process and on disk ($PBVD_JIT_CACHE, default ~/.cache/pbvd_jit; "off"
// disables), keyed by a hash of the generated source, the options and the
// kernel headers.
#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pbvd.h"
#include "kern_common.cuh"

namespace pbvd {

// ---- launch constants per (K, R, W) shape ----------------------------------

namespace {

template <int K, int R>
using DummyCode = Code<K, R, (1u << (K - 1)) | 1u, (1u << (K - 1)) | 1u,
                       (R > 2 ? ((1u << (K - 1)) | 1u) : 0u), (R > 3 ? ((1u << (K - 1)) | 1u) : 0u)>;

// supported lane counts: S = N / W states per lane, at most 64 registers;
// fewer than 16 states per lane (a survivor word shared by several lanes'
// sub-words) only with one lane per pair, W <= 32 (K = 12: one block pair
// per warp)
constexpr bool shape_ok(int K, int W) {
    return W >= 1 && W <= 32 && (1 << (K - 1)) / W >= 4 && (1 << (K - 1)) / W <= 64 &&
           ((1 << (K - 1)) / W >= 16 || W == 1);
}

template <int K, int R, int W>
bool shape_w(Variant* out) {
    if constexpr (shape_ok(K, W)) {
        fill_shape<Cfg<DummyCode<K, R>, W>>(*out);
        return true;
    } else {
        return false;
    }
}

template <int K, int R>
bool shape_kr(int W, Variant* out) {
    switch (W) {
        case 1: return shape_w<K, R, 1>(out);
        case 2: return shape_w<K, R, 2>(out);
        case 4: return shape_w<K, R, 4>(out);
        case 8: return shape_w<K, R, 8>(out);
        case 16: return shape_w<K, R, 16>(out);
        case 32: return shape_w<K, R, 32>(out);
        default: return false;
    }
}

template <int K>
bool shape_k(int R, int W, Variant* out) {
    switch (R) {
        case 2: return shape_kr<K, 2>(W, out);
        case 3: return shape_kr<K, 3>(W, out);
        case 4: return shape_kr<K, 4>(W, out);
        default: return false;
    }
}

}  // namespace

bool variant_shape(int K, int R, int W, Variant* out) {
    switch (K) {
        case 3: return shape_k<3>(R, W, out);
        case 4: return shape_k<4>(R, W, out);
        case 5: return shape_k<5>(R, W, out);
        case 6: return shape_k<6>(R, W, out);
        case 7: return shape_k<7>(R, W, out);
        case 8: return shape_k<8>(R, W, out);
        case 9: return shape_k<9>(R, W, out);
        case 10: return shape_k<10>(R, W, out);
        case 11: return shape_k<11>(R, W, out);
        case 12: return shape_k<12>(R, W, out);
        default: return false;
    }
}

// 64 states per lane from K = 9 up (K = 7: 32, the measured best)
int default_lanes(int K) { return K <= 6 ? 1 : K <= 8 ? 2 : (1 << (K - 1)) / 64; }

// ---- NVRTC (dlopen) ----------------------------------------------------------

namespace {

struct Nvrtc {
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
    decltype(&nvrtcAddNameExpression) add_name = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcGetLoweredName) lowered = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcGetErrorString) errstr = nullptr;
    bool ok = false;
    std::string why;
};

std::string cuda_home() {
    for (const char* e : {"CUDA_HOME", "CUDA_PATH"}) {
        const char* v = std::getenv(e);
        if (v && *v) return v;
    }
    return "/usr/local/cuda";
}

const Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* so = nullptr;
        const std::string cands[] = {"libnvrtc.so.12", "libnvrtc.so",
                                     cuda_home() + "/lib64/libnvrtc.so.12",
                                     cuda_home() + "/lib64/libnvrtc.so"};
        for (const auto& c : cands)
            if ((so = dlopen(c.c_str(), RTLD_NOW | RTLD_LOCAL))) break;
        if (!so) {
            n.why = "libnvrtc.so.12 not found (set CUDA_HOME)";
            return;
        }
#define PBVD_SYM(field, name)                                                   \
    n.field = reinterpret_cast<decltype(n.field)>(dlsym(so, name));             \
    if (!n.field) {                                                             \
        n.why = std::string("libnvrtc lacks ") + name;                          \
        return;                                                                 \
    }
        PBVD_SYM(create, "nvrtcCreateProgram")
        PBVD_SYM(destroy, "nvrtcDestroyProgram")
        PBVD_SYM(add_name, "nvrtcAddNameExpression")
        PBVD_SYM(compile, "nvrtcCompileProgram")
        PBVD_SYM(log_size, "nvrtcGetProgramLogSize")
        PBVD_SYM(log, "nvrtcGetProgramLog")
        PBVD_SYM(lowered, "nvrtcGetLoweredName")
        PBVD_SYM(cubin_size, "nvrtcGetCUBINSize")
        PBVD_SYM(cubin, "nvrtcGetCUBIN")
        PBVD_SYM(errstr, "nvrtcGetErrorString")
#undef PBVD_SYM
        n.ok = true;
    });
    return n;
}

std::string lib_dir() {
    Dl_info info{};
    if (dladdr(reinterpret_cast<void*>(&default_lanes), &info) && info.dli_fname) {
        std::string p = info.dli_fname;
        const size_t k = p.rfind('/');
        return k == std::string::npos ? std::string(".") : p.substr(0, k);
    }
    return ".";
}

std::string src_dir() {
    const char* v = std::getenv("PBVD_JIT_SRC");
    return (v && *v) ? std::string(v) : lib_dir() + "/csrc";
}

bool read_file(const std::string& path, std::string* out) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return false;
    std::ostringstream ss;
    ss << f.rdbuf();
    *out = ss.str();
    return true;
}

uint64_t fnv1a(uint64_t h, const std::string& s) {
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

std::string cache_dir() {
    const char* v = std::getenv("PBVD_JIT_CACHE");
    if (v && std::strcmp(v, "off") == 0) return "";
    if (v && *v) return v;
    const char* xdg = std::getenv("XDG_CACHE_HOME");
    if (xdg && *xdg) return std::string(xdg) + "/pbvd_jit";
    const char* home = std::getenv("HOME");
    return home && *home ? std::string(home) + "/.cache/pbvd_jit" : "";
}

void mkdirs(const std::string& d) {
    for (size_t k = 1; k <= d.size(); ++k)
        if (k == d.size() || d[k] == '/') mkdir(d.substr(0, k).c_str(), 0755);
}

// kernels per variant: fwd, fused, fused+mirror, traceback, fused+recycle,
// then the four forward kernels of punctured codes, then mirror+recycle
// (dense, punctured); the plain mirror kernels carry no recycling code
constexpr int NKERN = 11;

// cache file: "PBVDJIT3\n" + NKERN lowered names (one per line) + cubin bytes
constexpr char MAGIC[] = "PBVDJIT5\n";

bool cache_load(const std::string& path, std::string names[NKERN], std::string* cubin) {
    std::string all;
    if (!read_file(path, &all) || all.compare(0, sizeof MAGIC - 1, MAGIC) != 0) return false;
    size_t pos = sizeof MAGIC - 1;
    for (int i = 0; i < NKERN; ++i) {
        const size_t e = all.find('\n', pos);
        if (e == std::string::npos) return false;
        names[i] = all.substr(pos, e - pos);
        pos = e + 1;
    }
    *cubin = all.substr(pos);
    return !cubin->empty();
}

void cache_store(const std::string& dir, const std::string& path, const std::string names[NKERN],
                 const std::string& cubin) {
    mkdirs(dir);
    const std::string tmp = path + ".tmp" + std::to_string(getpid());
    {
        std::ofstream f(tmp, std::ios::binary);
        if (!f) return;
        f << MAGIC;
        for (int i = 0; i < NKERN; ++i) f << names[i] << '\n';
        f.write(cubin.data(), std::streamsize(cubin.size()));
        if (!f) return;
    }
    std::rename(tmp.c_str(), path.c_str());
}

struct JitEntry {
    Variant v;
    cudaLibrary_t lib = nullptr;
    std::string cubin;
};

std::mutex g_jit_mu;
std::vector<std::unique_ptr<JitEntry>> g_jit;

}  // namespace

// NVRTC build (or disk-cache hit) of the three kernels of (K, R, polys, W):
// cubin + lowered names.  Needs no GPU.
bool jit_compile(int K, int R, const uint32_t* polys, int W, std::string names[NKERN],
                 std::string* cubin, std::string* err) {
    auto fail = [&](const std::string& m) {
        if (err) *err = m;
        return false;
    };
    // generated translation unit: the kernel templates for this code
    char cfg[160];
    std::snprintf(cfg, sizeof cfg, "pbvd::Cfg<pbvd::Code<%d, %d, %uu, %uu, %uu, %uu>, %d>", K, R,
                  polys[0], polys[1], R > 2 ? polys[2] : 0u, R > 3 ? polys[3] : 0u, W);
    const std::string exprs[NKERN] = {std::string("pbvd::fwd_kernel<") + cfg + ", false>",
                                      std::string("pbvd::fwd_kernel<") + cfg + ", true>",
                                      std::string("pbvd::fwd_kernel<") + cfg + ", true, true, false>",
                                      std::string("pbvd::tb_kernel<") + cfg + ">",
                                      std::string("pbvd::fwd_kernel<") + cfg + ", true, false, true>",
                                      std::string("pbvd::fwd_kernel<") + cfg + ", false, false, false, true>",
                                      std::string("pbvd::fwd_kernel<") + cfg + ", true, false, false, true>",
                                      std::string("pbvd::fwd_kernel<") + cfg + ", true, true, false, true>",
                                      std::string("pbvd::fwd_kernel<") + cfg + ", true, false, true, true>",
                                      std::string("pbvd::fwd_kernel<") + cfg + ", true, true, true>",
                                      std::string("pbvd::fwd_kernel<") + cfg + ", true, true, true, true>"};
    const std::string source = "// pbvd JIT: " + std::string(cfg) +
                               "\n#include \"fwd.cuh\"\n#include \"tb.cuh\"\n";
    const std::string sdir = src_dir();
    const std::string cuinc = cuda_home() + "/include";
    const std::vector<std::string> opts = {"--gpu-architecture=sm_100a", "-std=c++17",
                                           "-default-device", "-lineinfo",
                                           "-I" + sdir + "/jit_std", "-I" + sdir, "-I" + cuinc};
    // cache key: source, options (not the include paths, which differ between
    // copies of the package), CUDA version and every header NVRTC reads here
    uint64_t key = fnv1a(1469598103934665603ull, source);
    for (const auto& o : opts)
        if (o.compare(0, 2, "-I") != 0) key = fnv1a(key, o);
    key = fnv1a(key, std::to_string(CUDART_VERSION));
    for (const char* hdr : {"fwd.cuh", "tb.cuh", "ptx.cuh", "params.h", "jit_std/cstdint",
                            "jit_std/type_traits", "jit_std/utility"}) {
        std::string body;
        if (!read_file(sdir + "/" + hdr, &body))
            return fail("JIT: kernel source " + sdir + "/" + hdr +
                        " not found (set PBVD_JIT_SRC to the package's csrc directory)");
        key = fnv1a(key, body);
    }
    char keyhex[17];
    std::snprintf(keyhex, sizeof keyhex, "%016llx", static_cast<unsigned long long>(key));
    const std::string cdir = cache_dir();
    const std::string cpath = cdir.empty() ? "" : cdir + "/pbvd_" + keyhex + ".cubin";
    if (!cpath.empty() && cache_load(cpath, names, cubin)) return true;

    const Nvrtc& n = nvrtc();
    if (!n.ok) return fail("JIT: " + n.why);
    nvrtcProgram prog = nullptr;
    nvrtcResult r = n.create(&prog, source.c_str(), "pbvd_jit.cu", 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) return fail(std::string("JIT: nvrtcCreateProgram: ") + n.errstr(r));
    for (const auto& e : exprs) n.add_name(prog, e.c_str());
    std::vector<const char*> copts;
    for (const auto& o : opts) copts.push_back(o.c_str());
    r = n.compile(prog, int(copts.size()), copts.data());
    if (r != NVRTC_SUCCESS) {
        size_t ls = 0;
        n.log_size(prog, &ls);
        std::string log(ls, '\0');
        if (ls) n.log(prog, &log[0]);
        n.destroy(&prog);
        if (log.size() > 4000) log = log.substr(0, 4000) + "...";
        return fail(std::string("JIT: NVRTC compile failed: ") + n.errstr(r) + "\n" + log);
    }
    for (int i = 0; i < NKERN; ++i) {
        const char* low = nullptr;
        if (n.lowered(prog, exprs[i].c_str(), &low) != NVRTC_SUCCESS || !low) {
            n.destroy(&prog);
            return fail("JIT: no lowered name for " + exprs[i]);
        }
        names[i] = low;
    }
    size_t cs = 0;
    n.cubin_size(prog, &cs);
    cubin->assign(cs, '\0');
    n.cubin(prog, &(*cubin)[0]);
    n.destroy(&prog);
    if (!cpath.empty()) cache_store(cdir, cpath, names, *cubin);
    return true;
}

const Variant* jit_variant(int K, int R, const uint32_t* polys, int W, std::string* err) {
    auto fail = [&](const std::string& m) -> const Variant* {
        if (err) *err = m;
        return nullptr;
    };
    Variant shape{};
    if (!variant_shape(K, R, W, &shape))
        return fail("no kernel shape for K=" + std::to_string(K) + " R=" + std::to_string(R) +
                    " lanes=" + std::to_string(W));
    std::lock_guard<std::mutex> lk(g_jit_mu);
    for (const auto& e : g_jit) {
        bool same = e->v.K == K && e->v.R == R && e->v.W == W;
        for (int r = 0; r < R && same; ++r) same = e->v.polys[r] == polys[r];
        if (same) return &e->v;
    }
    auto ent = std::make_unique<JitEntry>();
    std::string names[NKERN];
    if (!jit_compile(K, R, polys, W, names, &ent->cubin, err)) return nullptr;
    cudaError_t e = cudaLibraryLoadData(&ent->lib, ent->cubin.data(), nullptr, nullptr, 0, nullptr,
                                        nullptr, 0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(std::string("JIT: cudaLibraryLoadData: ") + cudaGetErrorString(e));
    }
    cudaKernel_t ks[NKERN] = {};
    for (int i = 0; i < NKERN; ++i) {
        e = cudaLibraryGetKernel(&ks[i], ent->lib, names[i].c_str());
        if (e != cudaSuccess) {
            cudaGetLastError();
            cudaLibraryUnload(ent->lib);
            return fail(std::string("JIT: cudaLibraryGetKernel: ") + cudaGetErrorString(e));
        }
    }
    ent->v = shape;
    for (int r = 0; r < 4; ++r) ent->v.polys[r] = r < R ? polys[r] : 0u;
    ent->v.jit = true;
    ent->v.k_fwd = reinterpret_cast<const void*>(ks[0]);
    ent->v.k_fused = reinterpret_cast<const void*>(ks[1]);
    ent->v.k_mirror = reinterpret_cast<const void*>(ks[2]);
    ent->v.k_tb = reinterpret_cast<const void*>(ks[3]);
    ent->v.k_recycle = reinterpret_cast<const void*>(ks[4]);
    ent->v.k_fwd_p = reinterpret_cast<const void*>(ks[5]);
    ent->v.k_fused_p = reinterpret_cast<const void*>(ks[6]);
    ent->v.k_mirror_p = reinterpret_cast<const void*>(ks[7]);
    ent->v.k_recycle_p = reinterpret_cast<const void*>(ks[8]);
    ent->v.k_mirror_r = reinterpret_cast<const void*>(ks[9]);
    ent->v.k_mirror_r_p = reinterpret_cast<const void*>(ks[10]);
    ent->v.prepared = 0;
    g_jit.push_back(std::move(ent));
    return &g_jit.back()->v;
}

}  // namespace pbvd

extern "C" int pbvd_jit_prebuild(int K, int R, const uint32_t* polys, int lanes, char* msg,
                                 size_t msg_len) {
    if (msg && msg_len) msg[0] = 0;
    if (!polys || K < 3 || K > 12 || R < 2 || R > 4) return PBVD_EINVAL;
    for (int r = 0; r < R; ++r)
        if (polys[r] == 0 || polys[r] >= (1u << K)) return PBVD_EINVAL;
    const int W = lanes == 0 ? pbvd::default_lanes(K) : lanes;
    pbvd::Variant shape{};
    std::string err;
    std::string names[pbvd::NKERN], cubin;
    int rc = PBVD_OK;
    if (!pbvd::variant_shape(K, R, W, &shape)) {
        err = "no kernel shape for that (K, R, lanes)";
        rc = PBVD_EUNSUPPORTED;
    } else if (!pbvd::jit_compile(K, R, polys, W, names, &cubin, &err)) {
        rc = PBVD_EUNSUPPORTED;
    }
    if (msg && msg_len) std::snprintf(msg, msg_len, "%s", err.c_str());
    return rc;
}
