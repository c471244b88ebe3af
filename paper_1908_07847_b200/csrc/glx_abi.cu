// glx_abi.cu -- the extern "C" boundary of libglycemlp_cuda.so (include/glycemlp_cuda.h).
//
// Host entry points mirror the reference's synchronous in-place contract of
// backend.run_train_segment (/root/reference/pkg/src/glycemlp/backend.py:208-234)
// and kernels.eval_counts (kernels.py:352-375); device entry points take
// caller-owned device buffers and a stream. Library-owned scratch (per-CTA
// gradient partials, kernel weight copies, descriptors) is cached per
// (device, stream) and only ever grows.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <chrono>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "glx_kernels.h"
#include "glycemlp_cuda.h"

using namespace glx;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define GLX_CK(expr)                                                                                       \
    do {                                                                                                   \
        cudaError_t e_ = (expr);                                                                           \
        if (e_ != cudaSuccess)                                                                             \
            return set_err(GLX_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                           __LINE__);                                                                      \
    } while (0)

#define GLX_LAUNCH(expr)          \
    do {                          \
        GLX_CK(expr);             \
        g_launches.fetch_add(1);  \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes < 256 ? 256 : bytes);
        if (e == cudaSuccess) cap = bytes < 256 ? 256 : bytes;
        return e;
    }
    template <typename T>
    T* as() const {
        return reinterpret_cast<T*>(p);
    }
};

// scratch tied to one (device, stream): stream order serialises its reuse
struct Workspace {
    DevBuf part, wk, desc, ctan, losspart, grad, wide, norm, tiles, gen, dbg;
};

std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, Workspace*> g_ws;

Workspace* workspace(cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto key = std::make_pair(dev, st);
    auto it = g_ws.find(key);
    if (it != g_ws.end()) return it->second;
    Workspace* w = new Workspace();
    g_ws[key] = w;
    return w;
}

// optional per-launch timing of the streaming epoch kernel (roofline evidence):
// an event pair recorded on the launching stream around every launch
struct Profiler {
    std::mutex mu;
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pairs;
    size_t used = 0;
} g_prof;

cudaError_t prof_begin(cudaStream_t st, cudaEvent_t* e1) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (!g_prof.on) {
        *e1 = nullptr;
        return cudaSuccess;
    }
    if (g_prof.used == g_prof.pairs.size()) {
        cudaEvent_t a, b;
        cudaError_t e = cudaEventCreate(&a);
        if (e != cudaSuccess) return e;
        e = cudaEventCreate(&b);
        if (e != cudaSuccess) return e;
        g_prof.pairs.emplace_back(a, b);
    }
    auto& pr = g_prof.pairs[g_prof.used++];
    *e1 = pr.second;
    return cudaEventRecord(pr.first, st);
}

int sm_count_current() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

// host-API state per device: own stream, staging buffers, optional input cache
struct HostState {
    std::mutex mu;
    cudaStream_t stream = nullptr;
    DevBuf w1, w2, x, t, lab, xp, stats, cnt, loss, flag, ex, exp_;
    DevBuf tlab, vx, vlab;  // checkpoint evaluation: train labels, test rows and labels
    const void* key_tlab = nullptr;
    const void* key_vx = nullptr;
    const void* key_vlab = nullptr;
    size_t bytes_vx = 0;
    const void* key_x = nullptr;
    size_t bytes_x = 0;
    const void* key_t = nullptr;
    size_t bytes_t = 0;
    const void* key_xp = nullptr;  // packed rows built from (key_x, key_t)
};
HostState g_host[64];

// ------------------------------------------------------------ online launch
struct NetReq {
    float* w_ih;
    float* w_ho;
    int H;
    int idx;
};

// hidden units per thread for the fp32 online kernel: for sweeps an MT-unit
// register tile (GLX_ONLINE_MT overrides) amortises the per-row reduction and
// barrier; a single network uses 2 units per thread when that makes it one warp
// (no cross-warp exchange: 292 vs 337 ns per row at 33-33-1), else 1
// (sweeps: 4 units per thread when networks of H >= 128 hold at least half of the
// hidden units -- config 3: 0.402 vs 0.417 ms/epoch -- else 2: small networks
// were 2x slower at 4)
int online_mt(size_t n_nets, bool ref64, int dp, int max_h, double big_frac) {
    if (ref64) return 1;
    const char* e = getenv("GLX_ONLINE_MT");
    int mt = e ? atoi(e) : (n_nets > 1 ? (big_frac >= 0.5 ? 4 : 2) : (max_h <= 64 ? 2 : 1));
    if (mt != 1 && mt != 2 && mt != 4) mt = 1;
    if (dp > 34) mt = 1;  // 64-wide rows: the MT tile would spill
    return mt;
}

// widths outside the register-tiled kernels (D > 63 or H > 512): one CTA per
// network, weights in global memory (glx_generic.cu)
int run_online_generic(const std::vector<NetReq>& nets, const float* X, const float* T, int64_t N, int D,
                       int64_t epochs, double lr, bool ref64, cudaStream_t st) {
    std::vector<GenNet> g(nets.size());
    int max_h = 0;
    for (size_t n = 0; n < nets.size(); n++) {
        g[n] = GenNet{nets[n].w_ih, nets[n].w_ho, nets[n].H, 0};
        max_h = std::max(max_h, nets[n].H);
    }
    if (online_generic_smem(D, max_h) > kGenMaxSmem)
        return set_err(GLX_ERR_INVALID, "online engine: input_dim %d with hidden_dim %d exceeds the shared-memory row "
                       "and activation buffers (%zu bytes > %zu)", D, max_h, online_generic_smem(D, max_h),
                       kGenMaxSmem);
    Workspace* ws = workspace(st);
    GLX_CK(ws->desc.ensure(g.size() * sizeof(GenNet)));
    GLX_CK(cudaMemcpyAsync(ws->desc.p, g.data(), g.size() * sizeof(GenNet), cudaMemcpyHostToDevice, st));
    GLX_LAUNCH(launch_online_generic(ws->desc.as<GenNet>(), (int)g.size(), max_h, X, T, N, D, epochs, lr, ref64, st));
    return GLX_OK;
}

int run_online(std::vector<NetReq> nets, const float* X, const float* T, int64_t N, int D, int64_t epochs, double lr,
               bool ref64, cudaStream_t st) {
    const int dp = online_dp_for(D);
    int max_h = 0;
    for (auto& n : nets) max_h = std::max(max_h, n.H);
    if (dp < 0 || max_h > 512) return run_online_generic(nets, X, T, N, D, epochs, lr, ref64, st);
    // exact path, one paper-size network: the f64-resident small kernel
    if (ref64 && nets.size() == 1 && nets[0].H <= 64 && dp <= 34 && online_ref64_small_smem(N, D) <= 160 * 1024 &&
        getenv("GLX_ONLINE_REF64_SMALL") == nullptr) {
        GLX_LAUNCH(launch_online_ref64_small(nets[0].w_ih, nets[0].w_ho, nets[0].H, X, T, N, D, epochs, lr, st));
        return GLX_OK;
    }
    // staged rows [N][dp], targets [N], lookahead dots [N] (glx_online.cu)
    const size_t xbytes = ((size_t)N * ((dp + 3) & ~3) * 4 + (size_t)N * 8 + 15) / 16 * 16;  // rows padded to 4
    const bool x_in_smem = xbytes <= 160 * 1024;
    double units = 0, big_units = 0;
    for (auto& n : nets) {
        units += n.H;
        if (n.H >= 128) big_units += n.H;
    }
    const int mt = online_mt(nets.size(), ref64, dp, max_h, units > 0 ? big_units / units : 0.0);
    const int cap = mt == 1 ? 16 : 8;  // warps per CTA (register budget of the MT-unit tile)
    // first-fit decreasing packing of networks into CTAs of <= cap warps / 15 networks
    std::stable_sort(nets.begin(), nets.end(), [](const NetReq& a, const NetReq& b) { return a.H > b.H; });
    struct Cta {
        int warps = 0;
        size_t scratch = 0;
        std::vector<int> members;
    };
    std::vector<Cta> ctas;
    std::vector<OnlineNetDesc> desc(nets.size());
    size_t open_from = 0;  // CTAs before this index are full
    for (size_t n = 0; n < nets.size(); n++) {
        const int nw = (nets[n].H + 32 * mt - 1) / (32 * mt);
        const size_t scr = (online_scratch_bytes(nets[n].H, ref64) + 15) / 16 * 16;
        size_t c = open_from;
        for (; c < ctas.size(); c++)
            if (ctas[c].warps + nw <= cap && ctas[c].members.size() < 15) break;
        if (c == ctas.size()) ctas.emplace_back();
        Cta& C = ctas[c];
        OnlineNetDesc& d = desc[n];
        d.w_ih = nets[n].w_ih;
        d.w_ho = nets[n].w_ho;
        d.H = nets[n].H;
        d.warp0 = C.warps;
        d.nwarps = nw;
        d.bar_id = 1 + (int)C.members.size();
        d.scratch_off = (int)((x_in_smem ? xbytes : 0) + C.scratch);
        d.pad = 0;
        C.warps += nw;
        C.scratch += scr;
        C.members.push_back((int)n);
        while (open_from < ctas.size() && ctas[open_from].warps >= cap) open_from++;
    }
    // descriptors grouped per CTA
    std::vector<OnlineNetDesc> ordered;
    std::vector<int2> cta_nets;
    int max_warps = 0;
    size_t max_scratch = 0;
    for (auto& C : ctas) {
        cta_nets.push_back(make_int2((int)ordered.size(), (int)C.members.size()));
        for (int m : C.members) ordered.push_back(desc[m]);
        max_warps = std::max(max_warps, C.warps);
        max_scratch = std::max(max_scratch, C.scratch);
    }
    Workspace* ws = workspace(st);
    GLX_CK(ws->desc.ensure(ordered.size() * sizeof(OnlineNetDesc)));
    GLX_CK(ws->ctan.ensure(cta_nets.size() * sizeof(int2)));
    GLX_CK(cudaMemcpyAsync(ws->desc.p, ordered.data(), ordered.size() * sizeof(OnlineNetDesc),
                           cudaMemcpyHostToDevice, st));
    GLX_CK(cudaMemcpyAsync(ws->ctan.p, cta_nets.data(), cta_nets.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    OnlineLaunch L;
    L.nets = ws->desc.as<OnlineNetDesc>();
    L.cta_nets = ws->ctan.as<int2>();
    L.n_ctas = (int)ctas.size();
    L.threads = max_warps * 32;
    L.smem_bytes = (x_in_smem ? xbytes : 0) + max_scratch;
    L.x_in_smem = x_in_smem;
    L.ref64 = ref64;
    L.mt = mt;
    L.one_warp = std::all_of(desc.begin(), desc.end(), [](const OnlineNetDesc& d) { return d.nwarps == 1; });
    L.X = X;
    L.T = T;
    L.N = N;
    L.D = D;
    L.epochs = epochs;
    L.lr = lr;
    GLX_LAUNCH(launch_online(L, st));
    // the copies above read pageable host memory that dies with this frame:
    // cudaMemcpyAsync from pageable memory has finished staging on return.
    return GLX_OK;
}

int check_dims(int64_t rows, int D, int H) {
    if (rows < 0) return set_err(GLX_ERR_SHAPE, "rows must be >= 0, got %lld", (long long)rows);
    if (D < 1) return set_err(GLX_ERR_SHAPE, "input_dim must be >= 1, got %d", D);
    if (H < 1) return set_err(GLX_ERR_SHAPE, "hidden_dim must be >= 1, got %d", H);
    return GLX_OK;
}

// epoch-kernel selection (kind 2: tcgen05 3xTF32 kernel, glx_batchtc.cu; 1: the
// three-role FP32 kernel, glx_batch3.cu; 0: the two-role kernel). Default: the
// first whose geometry fits. GLX_BATCH_KERNEL=3 starts at the three-role
// kernel, GLX_BATCH_KERNEL=2 forces the two-role kernel.
int batch_kernel_pref() {
    static int v = [] {
        const char* e = getenv("GLX_BATCH_KERNEL");
        return (e && e[0] == '2') ? 0 : (e && e[0] == '3') ? 1 : 2;
    }();
    return v;
}

// the tcgen05 kernel's per-tile time is set by its epilogue chain (32 units x 32 rows
// per warp), so narrow layers cost about as much as 128 units (0.115-0.12 ms per 1M
// rows for H <= 128, tools/batch_width_time.py); the FP32 kernels win below ~24 units
// (H = 16: 0.090 vs 0.116 ms). GLX_BATCH_KERNEL=tc forces the tcgen05 kernel for any H <= 256
constexpr int kTcMinH = 24;
// the rows-on-lanes kernel (H <= 64, from 2^17 rows) is flat at ~0.065 ms per 1M rows up
// to 32 units; the three-role FP32 kernel is level at H = 8 and slower above
constexpr int kRtMinH = 12;
bool force_tc() {
    const char* e = getenv("GLX_BATCH_KERNEL");
    return e && e[0] == 't' && e[1] == 'c';
}

bool force_rt() {
    const char* e = getenv("GLX_BATCH_KERNEL");
    return e && e[0] == 'r' && e[1] == 't';
}

bool train_geometry(int64_t N, int D, int H, BatchGeom* g, int* kind) {
    const int pref = batch_kernel_pref();
    // narrow layers with enough rows for the FAST precision: rows on the TMEM lanes
    // (glx_batchtc.cu batchrt_kernel); GLX_BATCH_KERNEL=tc keeps the unit-on-lanes kernel
    if (pref >= 2 && !force_tc() && (H >= kRtMinH || force_rt()) && batchrt_geometry(N, D, H, sm_count_current(), g)) {
        *kind = 3;
        return true;
    }
    if (pref >= 2 && (H >= kTcMinH || force_tc()) && batchtc_geometry(N, D, H, sm_count_current(), g)) {
        *kind = 2;
        return true;
    }
    // the three-role kernel wins where its forward/backward tiles are 4 units wide
    // (H % 4 == 0); narrower tiles stay on the two-role kernel (profiles/r01_summary.md)
    static const bool any_mt = getenv("GLX_BATCH3_ANY_MT") != nullptr;  // diagnostic: MT < 4 tiles too
    if (pref >= 1 && batch3_geometry(N, D, H, sm_count_current(), g) && (g->MT == 4 || any_mt)) {
        *kind = 1;
        return true;
    }
    *kind = 0;
    return batch_geometry(N, D, H, sm_count_current(), true, g);
}

// what the epoch kernel reads: the packed rows (kinds 0, 1) or, for the tcgen05
// kernel, their per-tile MMA operand layout, built here once per training call
// into the stream's workspace (one pass over the rows)
int epoch_input(Workspace* ws, const BatchGeom& g, int kind, const float* Xp, cudaStream_t st, const void** in) {
    if (kind != 2 && kind != 3) {
        *in = Xp;
        return GLX_OK;
    }
    GLX_CK(ws->tiles.ensure(kind == 3 ? batchrt_tile_bytes(g) : batchtc_tile_bytes(g)));
    if (kind == 3) GLX_LAUNCH(launch_batchrt_pack(g, Xp, ws->tiles.p, st));
    else GLX_LAUNCH(launch_batchtc_pack(g, Xp, ws->tiles.p, st));
    *in = ws->tiles.p;
    return GLX_OK;
}

cudaError_t launch_train_epoch(const BatchGeom& g, int kind, const void* in, const float* Wk, float* part,
                               cudaStream_t st, int* dbg = nullptr) {
    const float* Xp = (const float*)in;
    if (kind == 3) return launch_batchrt_epoch(g, in, Wk, part, st, dbg);
    if (kind == 2) return launch_batchtc_epoch(g, in, Wk, part, st, dbg);
    return kind == 1 ? launch_batch3_epoch(g, Xp, Wk, part, st) : launch_batch_epoch(g, Xp, Wk, part, true, st);
}

}  // namespace
namespace glx {
cudaError_t launch_batch_grad(const BatchGeom& g, const float* part, const float* Wk, double* grad, cudaStream_t st);
cudaError_t launch_batch_apply(int D, int H, float* W1, float* W2, const double* grad, double lr_over_n,
                               int* nonfinite, cudaStream_t st);
}  // namespace glx
namespace {

// any shape outside the batch kernels (kind 4, glx_generic.cu): this rank's f64
// gradient sum in the glx_batch_grad layout
int generic_grad(const float* w_ih, const float* w_ho, const float* Xp, int64_t N, int D, int H, double* grad,
                 cudaStream_t st) {
    Workspace* ws = workspace(st);
    GLX_CK(ws->gen.ensure(generic_work_bytes(N, D, H)));
    const int64_t nlaunch = 4 * ((N + (int64_t)generic_chunk_rows(N, H) - 1) / (int64_t)generic_chunk_rows(N, H));
    GLX_CK(generic_batch_grad(w_ih, w_ho, Xp, N, D, H, glx_packed_ld(D), ws->gen.p, grad, st));
    g_launches.fetch_add(nlaunch);
    return GLX_OK;
}

int generic_train(float* w_ih, float* w_ho, const float* Xp, int64_t N, int D, int H, int64_t epochs, double lr,
                  double* stats_hist, int32_t* nonfinite, cudaStream_t st) {
    Workspace* ws = workspace(st);
    const int64_t glen = (int64_t)H * (D + 1) + H + 1 + 5;
    GLX_CK(ws->grad.ensure((size_t)glen * sizeof(double)));
    double* grad = ws->grad.as<double>();
    for (int64_t e = 0; e < epochs; e++) {
        int rc = generic_grad(w_ih, w_ho, Xp, N, D, H, grad, st);
        if (rc) return rc;
        GLX_LAUNCH(launch_batch_apply(D, H, w_ih, w_ho, grad, lr / (double)N, nonfinite, st));
        if (stats_hist)  // loss, tp, tn, fp, fn at this epoch's starting weights
            GLX_CK(cudaMemcpyAsync(stats_hist + 5 * e, grad + glen - 5, 5 * sizeof(double), cudaMemcpyDeviceToDevice,
                                   st));
    }
    return GLX_OK;
}

// debug runs (GLX_FLAG_DEBUG, glx_set_debug): the tcgen05 epoch kernels stamp every
// tile hand-off between their roles and count the tiles each role handled
// (glx_batchtc.cu dbg_expect); after each epoch the host requires no stale stamp,
// one forward issue per row tile and one dh hand-off per row group of it
std::atomic<int> g_debug{0};

int pipeline_verify(const BatchGeom& g, int kind, const int* dbg, int64_t epoch, cudaStream_t st) {
    constexpr int kHdr = 16;  // glx_batchtc.cu kDbgHdr
    std::vector<int> h(kHdr + 2 * (size_t)g.ntiles);
    GLX_CK(cudaMemcpyAsync(h.data(), dbg, h.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaStreamSynchronize(st));
    if (h[0])
        return set_err(GLX_ERR_RACE, "epoch kernel pipeline check (kind %d), epoch %lld: %d stale hand-off(s); first: "
                       "check %d in CTA %d expected tile stamp %d, saw %d", kind, (long long)epoch, h[0], h[1], h[2],
                       h[3], h[4]);
    const int want_b = kind == 2 ? 2 : 4;  // row blocks (kind 2) / row quadrants (kind 3) per tile
    for (int64_t t = 0; t < g.ntiles; t++) {
        const int f = h[kHdr + t], b = h[kHdr + g.ntiles + t];
        if (f != 1 || b != want_b)
            return set_err(GLX_ERR_RACE, "epoch kernel pipeline check (kind %d), epoch %lld: row tile %lld had %d "
                           "forward issue(s) and %d dh hand-off(s), want 1 and %d", kind, (long long)epoch,
                           (long long)t, f, b, want_b);
    }
    return GLX_OK;
}

// GLX_DEBUG_INJECT_TILE=t (tests): the producer stamps row tile t wrongly, so a debug
// run must fail -- proof that the checker observes the hand-offs
int pipeline_inject(int* dbg, cudaStream_t st) {
    const char* e = getenv("GLX_DEBUG_INJECT_TILE");
    if (!e) return GLX_OK;
    static thread_local int v;
    v = atoi(e) + 1;
    GLX_CK(cudaMemcpyAsync(dbg + 6, &v, sizeof(int), cudaMemcpyHostToDevice, st));
    GLX_CK(cudaStreamSynchronize(st));
    return GLX_OK;
}

int batch_train_impl(float* w_ih, float* w_ho, const float* Xp, int64_t N, int D, int H, int64_t epochs, double lr,
                     double* stats_hist, int32_t* nonfinite, cudaStream_t st, bool debug = false) {
    BatchGeom g;
    int kind = 0;
    if (!train_geometry(N, D, H, &g, &kind)) return generic_train(w_ih, w_ho, Xp, N, D, H, epochs, lr, stats_hist,
                                                                  nonfinite, st);
    Workspace* ws = workspace(st);
    GLX_CK(ws->part.ensure((size_t)g.grid * g.PS * 4));
    GLX_CK(ws->wk.ensure((size_t)2 * g.WKS * 4));
    float* wk0 = ws->wk.as<float>();
    float* wk1 = wk0 + g.WKS;
    GLX_LAUNCH(launch_batch_prep(g, w_ih, w_ho, wk0, wk1, st));
    const void* in = nullptr;
    int rc = epoch_input(ws, g, kind, Xp, st, &in);
    if (rc) return rc;
    const double lr_over_n = lr / (double)N;
    const bool check = (debug || g_debug.load()) && (kind == 2 || kind == 3);
    int* dbg = nullptr;
    if (check) {
        GLX_CK(ws->dbg.ensure(pipeline_check_ints(g) * sizeof(int)));
        dbg = ws->dbg.as<int>();
    }
    for (int64_t e = 0; e < epochs; e++) {
        float* cur = (e & 1) ? wk1 : wk0;
        float* nxt = (e & 1) ? wk0 : wk1;
        if (check) {
            GLX_CK(cudaMemsetAsync(dbg, 0, pipeline_check_ints(g) * sizeof(int), st));
            int rc = pipeline_inject(dbg, st);
            if (rc) return rc;
        }
        cudaEvent_t pe = nullptr;
        GLX_CK(prof_begin(st, &pe));
        GLX_LAUNCH(launch_train_epoch(g, kind, in, cur, ws->part.as<float>(), st, dbg));
        if (pe) GLX_CK(cudaEventRecord(pe, st));
        if (check) {
            int rc = pipeline_verify(g, kind, dbg, e, st);
            if (rc) return rc;
        }
        GLX_LAUNCH(launch_batch_update(g, ws->part.as<float>(), w_ih, w_ho, cur, nxt, lr_over_n, true,
                                       stats_hist ? stats_hist + 5 * e : nullptr, nonfinite, st));
    }
    return GLX_OK;
}

}  // namespace

namespace glx {
size_t online_scratch_bytes(int H, bool ref64) {
    if (!ref64) return 2 * 16 * sizeof(float);
    const int nb = (H + 15) / 16;
    return (size_t)(nb * 17 + 2) * sizeof(double);
}
}  // namespace glx

namespace {
// ------------------------------------------------------------------------------
// Data plane of the data-parallel configurations (SURVEY.md 8(b) glx_dp_init,
// 8(e)): one NCCL communicator per rank, owned here. A DP epoch is
//   epoch kernel (this rank's rows) -> f64 gradient sum (batch_grad_kernel)
//   -> ncclAllReduce(sum, f64, P + 5 doubles) -> update + next weight copy
// and is captured once into CUDA graphs (one per parity of the double-buffered
// pre-scaled weight copy), replayed every epoch on a library-owned stream that
// is joined to the caller's stream by events.
struct DpComm {
    ncclComm_t comm = nullptr;
    int dev = 0, nranks = 1, rank = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    DevBuf grad, slot;
    // graph cache: the captured epoch is valid for these arguments
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    const void* key[7] = {};
    int64_t key_n = -1;
    int key_d = 0, key_h = 0;
    double key_lr = 0.0;
    int per_replay = 0;
    void drop_graphs() {
        for (auto& e : exec)
            if (e) {
                cudaGraphExecDestroy(e);
                e = nullptr;
            }
        key_n = -1;
    }
};

// NCCL is bound lazily at the first glx_dp_* call (no link-time dependency):
// the copy already loaded into the process when there is one (torch's bundled
// libnccl, so one NCCL serves the process), else $GLX_NCCL_LIB, else the
// image's libnccl.so.2. nccl.h supplies the types only.
struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* env = getenv("GLX_NCCL_LIB");
        if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return a;
        }
        a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
        a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
        a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
        a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.GetErrorString;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

#define GLX_NCCL_API()                                                             \
    do {                                                                           \
        if (!nccl().ok) return set_err(GLX_ERR_CUDA, "%s", nccl().why.c_str());    \
    } while (0)

bool dp_graphs_enabled() {  // GLX_DP_GRAPH=0: eager epochs (read per call, for A/B tests)
    const char* e = getenv("GLX_DP_GRAPH");
    return !(e && e[0] == '0');
}

#define GLX_NCCL(expr)                                                                                          \
    do {                                                                                                        \
        ncclResult_t r_ = (expr);                                                                               \
        if (r_ != ncclSuccess)                                                                                  \
            return set_err(GLX_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, nccl().GetErrorString(r_), __FILE__,  \
                           __LINE__);                                                                           \
    } while (0)

// one epoch on dp->st: kernels of this rank's rows, the all-reduce, the update
// (profile: per-launch events around the epoch kernel, eager epochs only)
int dp_epoch_enqueue(DpComm* dp, const BatchGeom& g, int kind, bool have_rows, const void* in, float* part,
                     float* wk_cur, float* wk_nxt, float* w_ih, float* w_ho, double lr_over_n, int32_t* nonfinite,
                     bool profile) {
    cudaStream_t st = dp->st;
    const int64_t glen = (int64_t)g.P1 + g.H + 1 + 5;
    double* grad = dp->grad.as<double>();
    if (have_rows) {
        cudaEvent_t pe = nullptr;
        if (profile) GLX_CK(prof_begin(st, &pe));
        GLX_CK(launch_train_epoch(g, kind, in, wk_cur, part, st));
        if (pe) GLX_CK(cudaEventRecord(pe, st));
        GLX_CK(launch_batch_grad(g, part, wk_cur, grad, st));
    } else {
        GLX_CK(cudaMemsetAsync(grad, 0, glen * sizeof(double), st));
    }
    GLX_NCCL(nccl().AllReduce(grad, grad, (size_t)glen, ncclDouble, ncclSum, dp->comm, st));
    GLX_CK(launch_batch_dp_update(g, w_ih, w_ho, wk_nxt, grad, lr_over_n, dp->slot.as<double>(), nonfinite, st));
    return GLX_OK;
}

// shapes outside the batch kernels: eager epochs of the any-shape gradient, the
// all-reduce and the plain update
int dp_train_generic(DpComm* dp, float* w_ih, float* w_ho, const float* Xp, int64_t N, int64_t N_total, int D, int H,
                     int64_t epochs, double lr, double* stats_hist, int32_t* nonfinite, cudaStream_t caller) {
    GLX_CK(cudaSetDevice(dp->dev));
    const int64_t glen = (int64_t)H * (D + 1) + H + 1 + 5;
    GLX_CK(dp->grad.ensure((size_t)glen * sizeof(double)));
    double* grad = dp->grad.as<double>();
    GLX_CK(cudaEventRecord(dp->ev_in, caller));
    GLX_CK(cudaStreamWaitEvent(dp->st, dp->ev_in, 0));
    for (int64_t e = 0; e < epochs; e++) {
        if (N > 0) {
            int rc = generic_grad(w_ih, w_ho, Xp, N, D, H, grad, dp->st);
            if (rc) return rc;
        } else {
            GLX_CK(cudaMemsetAsync(grad, 0, glen * sizeof(double), dp->st));
        }
        GLX_NCCL(nccl().AllReduce(grad, grad, (size_t)glen, ncclDouble, ncclSum, dp->comm, dp->st));
        GLX_LAUNCH(launch_batch_apply(D, H, w_ih, w_ho, grad, lr / (double)N_total, nonfinite, dp->st));
        if (stats_hist)
            GLX_CK(cudaMemcpyAsync(stats_hist + 5 * e, grad + glen - 5, 5 * sizeof(double), cudaMemcpyDeviceToDevice,
                                   dp->st));
    }
    GLX_CK(cudaEventRecord(dp->ev_out, dp->st));
    GLX_CK(cudaStreamWaitEvent(caller, dp->ev_out, 0));
    return GLX_OK;
}

int dp_train_batch(DpComm* dp, float* w_ih, float* w_ho, const float* Xp, int64_t N, int64_t N_total, int D, int H,
                   int64_t epochs, double lr, double* stats_hist, int32_t* nonfinite, cudaStream_t caller) {
    BatchGeom g;
    int kind = 0;
    if (!train_geometry(std::max<int64_t>(N, 1), D, H, &g, &kind))
        return dp_train_generic(dp, w_ih, w_ho, Xp, N, N_total, D, H, epochs, lr, stats_hist, nonfinite, caller);
    GLX_CK(cudaSetDevice(dp->dev));
    Workspace* ws = workspace(dp->st);
    GLX_CK(ws->part.ensure((size_t)g.grid * g.PS * 4));
    GLX_CK(ws->wk.ensure((size_t)2 * g.WKS * 4));
    GLX_CK(dp->grad.ensure(((size_t)g.P1 + H + 1 + 5) * sizeof(double)));
    GLX_CK(dp->slot.ensure(5 * sizeof(double)));
    float* wk0 = ws->wk.as<float>();
    float* wk1 = wk0 + g.WKS;
    float* part = ws->part.as<float>();
    const double lr_over_n = lr / (double)N_total;
    const bool rows = N > 0;
    GLX_CK(cudaEventRecord(dp->ev_in, caller));
    GLX_CK(cudaStreamWaitEvent(dp->st, dp->ev_in, 0));
    GLX_LAUNCH(launch_batch_prep(g, w_ih, w_ho, wk0, wk1, dp->st));
    const void* in = Xp;
    if (rows) {
        int rc = epoch_input(ws, g, kind, Xp, dp->st, &in);
        if (rc) return rc;
    }
    const int per_epoch = rows ? 3 : 1;
    if (dp_graphs_enabled()) {
        const void* key[7] = {w_ih, w_ho, in, nonfinite, ws->wk.p, ws->part.p, dp->grad.p};
        const bool hit = dp->exec[0] && dp->key_n == N && dp->key_d == D && dp->key_h == H &&
                         dp->key_lr == lr_over_n && std::equal(key, key + 7, dp->key);
        if (!hit) {
            dp->drop_graphs();
            for (int par = 0; par < 2; par++) {
                cudaGraph_t graph = nullptr;
                GLX_CK(cudaStreamBeginCapture(dp->st, cudaStreamCaptureModeThreadLocal));
                int rc = dp_epoch_enqueue(dp, g, kind, rows, in, part, par ? wk1 : wk0, par ? wk0 : wk1, w_ih, w_ho,
                                          lr_over_n, nonfinite, false);
                cudaError_t ec = cudaStreamEndCapture(dp->st, &graph);
                if (rc) {
                    if (graph) cudaGraphDestroy(graph);
                    return rc;
                }
                GLX_CK(ec);
                cudaError_t ei = cudaGraphInstantiate(&dp->exec[par], graph, 0);
                cudaGraphDestroy(graph);
                GLX_CK(ei);
            }
            std::copy(key, key + 7, dp->key);
            dp->key_n = N;
            dp->key_d = D;
            dp->key_h = H;
            dp->key_lr = lr_over_n;
        }
        for (int64_t e = 0; e < epochs; e++) {
            GLX_CK(cudaGraphLaunch(dp->exec[e & 1], dp->st));
            g_launches.fetch_add(per_epoch);
            if (stats_hist)
                GLX_CK(cudaMemcpyAsync(stats_hist + 5 * e, dp->slot.p, 5 * sizeof(double), cudaMemcpyDeviceToDevice,
                                       dp->st));
        }
    } else {
        for (int64_t e = 0; e < epochs; e++) {
            int rc = dp_epoch_enqueue(dp, g, kind, rows, in, part, (e & 1) ? wk1 : wk0, (e & 1) ? wk0 : wk1, w_ih,
                                      w_ho, lr_over_n, nonfinite, true);
            if (rc) return rc;
            g_launches.fetch_add(per_epoch);
            if (stats_hist)
                GLX_CK(cudaMemcpyAsync(stats_hist + 5 * e, dp->slot.p, 5 * sizeof(double), cudaMemcpyDeviceToDevice,
                                       dp->st));
        }
    }
    GLX_CK(cudaEventRecord(dp->ev_out, dp->st));
    GLX_CK(cudaStreamWaitEvent(caller, dp->ev_out, 0));
    return GLX_OK;
}
}  // namespace

extern "C" {

const char* glx_last_error(void) { return g_err.c_str(); }
int glx_version(void) { return 100; }
uint64_t glx_launch_count(void) { return g_launches.load(); }

int glx_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int glx_sm_count(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
    return n;
}

void glx_cache_clear(void) {
    for (auto& h : g_host) {
        std::lock_guard<std::mutex> lk(h.mu);
        h.key_x = h.key_t = h.key_xp = nullptr;
        h.key_tlab = h.key_vx = h.key_vlab = nullptr;
        h.bytes_x = h.bytes_t = h.bytes_vx = 0;
    }
}

// --------------------------------------------------------------- device API

int glx_train_online(float* w_ih, float* w_ho, const float* X, const float* T, int64_t N, int32_t D, int32_t H,
                     int64_t epochs, double lr, int32_t numerics, void* stream) {
    int rc = check_dims(N, D, H);
    if (rc) return rc;
    if (epochs < 0) return set_err(GLX_ERR_INVALID, "epochs must be >= 0");
    if (N == 0 || epochs == 0) return GLX_OK;
    std::vector<NetReq> nets{{w_ih, w_ho, H, 0}};
    return run_online(nets, X, T, N, D, epochs, lr, numerics == GLX_REF64, (cudaStream_t)stream);
}

int glx_train_sweep(int64_t n_nets, const int32_t* H_per_net, const int64_t* w_off, float* w_pool, const float* X,
                    const float* T, int64_t N, int32_t D, int64_t epochs, double lr, int32_t numerics, void* stream) {
    if (n_nets < 0) return set_err(GLX_ERR_INVALID, "n_nets must be >= 0");
    if (n_nets == 0 || N == 0 || epochs == 0) return GLX_OK;
    std::vector<NetReq> nets;
    nets.reserve((size_t)n_nets);
    for (int64_t n = 0; n < n_nets; n++) {
        const int H = H_per_net[n];
        int rc = check_dims(N, D, H);
        if (rc) return rc;
        float* wi = w_pool + w_off[n];
        nets.push_back({wi, wi + (int64_t)H * (D + 1), H, (int)n});
    }
    return run_online(nets, X, T, N, D, epochs, lr, numerics == GLX_REF64, (cudaStream_t)stream);
}

int32_t glx_packed_ld(int32_t D) {
    int dp = pick_dp(D);  // the batch kernels' weight-row stride: a row holds at least that many floats
    if (dp < 0) dp = D + 1;
    return ((std::max(D + 2, dp)) + 3) / 4 * 4;
}

int glx_pack_rows(const float* X, const float* T, const uint8_t* labels, int64_t N, int32_t D, float* Xp,
                  void* stream) {
    if (N < 0 || D < 1) return set_err(GLX_ERR_SHAPE, "bad pack shape");
    if (N == 0) return GLX_OK;
    GLX_LAUNCH(launch_pack_rows(X, T, labels, N, D, glx_packed_ld(D), Xp, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_pack_rows_minmax(const float* X, const float* T, const uint8_t* labels, int64_t N, int32_t D,
                         const float* col_min, const float* col_max, float* Xp, void* stream) {
    if (N < 0 || D < 1) return set_err(GLX_ERR_SHAPE, "bad pack shape");
    if (!col_min || !col_max) return set_err(GLX_ERR_INVALID, "col_min and col_max are required");
    if (N == 0) return GLX_OK;
    GLX_LAUNCH(launch_pack_rows(X, T, labels, N, D, glx_packed_ld(D), Xp, (cudaStream_t)stream, col_min, col_max));
    return GLX_OK;
}

int glx_pcg64_uniform_f32(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t first_output,
                          int64_t n_floats, float* out, void* stream) {
    if (first_output < 0 || n_floats < 0) return set_err(GLX_ERR_INVALID, "bad pcg64 range");
    const uint64_t st4[4] = {state_hi, state_lo, inc_hi, inc_lo};
    GLX_LAUNCH(launch_pcg64_f32(st4, first_output, n_floats, out, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_pcg64_coin(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t first_output,
                   int64_t n, uint8_t* labels, void* stream) {
    if (first_output < 0 || n < 0) return set_err(GLX_ERR_INVALID, "bad pcg64 range");
    const uint64_t st4[4] = {state_hi, state_lo, inc_hi, inc_lo};
    GLX_LAUNCH(launch_pcg64_coin(st4, first_output, n, labels, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_planted_score(const float* X, int64_t N, int32_t D, const int32_t* pick, const double* coef, int32_t k,
                      double* score, void* stream) {
    if (N < 0 || D < 1 || k < 1 || k > D) return set_err(GLX_ERR_SHAPE, "bad planted-score shape");
    if (N == 0) return GLX_OK;
    GLX_LAUNCH(launch_planted_score(X, N, D, pick, coef, k, score, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_label_ge(const double* score, int64_t N, const double* threshold, uint8_t* labels, void* stream) {
    if (N < 0) return set_err(GLX_ERR_SHAPE, "bad label shape");
    if (N == 0) return GLX_OK;
    GLX_LAUNCH(launch_label_ge(score, N, threshold, labels, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_minmax_fit(const float* X, int64_t N, int32_t D, float* col_min, float* col_max, void* stream) {
    if (N < 1 || D < 1) return set_err(GLX_ERR_SHAPE, "normalize_fit needs at least one row and column");
    cudaStream_t st = (cudaStream_t)stream;
    Workspace* ws = workspace(st);
    GLX_CK(ws->norm.ensure((size_t)2 * D * sizeof(int)));
    GLX_CK(launch_minmax_fit(X, N, D, ws->norm.as<int>(), col_min, col_max, st));
    g_launches.fetch_add(3);
    return GLX_OK;
}

int glx_minmax_apply(const float* X, int64_t N, int32_t D, const float* col_min, const float* col_max, float* Y,
                     void* stream) {
    if (N < 0 || D < 1) return set_err(GLX_ERR_SHAPE, "bad normalize shape");
    if (N == 0) return GLX_OK;
    GLX_LAUNCH(launch_minmax_apply(X, N, D, col_min, col_max, Y, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_train_batch(float* w_ih, float* w_ho, const float* Xp, int64_t N, int32_t D, int32_t H, int64_t epochs,
                    double lr, double* stats_hist, int32_t* nonfinite, void* stream) {
    int rc = check_dims(N, D, H);
    if (rc) return rc;
    if (N == 0 || epochs <= 0) return GLX_OK;
    return batch_train_impl(w_ih, w_ho, Xp, N, D, H, epochs, lr, stats_hist, nonfinite, (cudaStream_t)stream);
}

int64_t glx_batch_grad_len(int32_t D, int32_t H) { return (int64_t)H * (D + 1) + H + 1 + 5; }

int glx_batch_kernel_kind(int64_t N, int32_t D, int32_t H) {
    BatchGeom g;
    int kind = -1;
    if (N < 1 || D < 1 || H < 1) return -1;
    if (!train_geometry(N, D, H, &g, &kind)) return 4;  // the any-shape engine (glx_generic.cu)
    return kind;
}

int glx_batch_grad(const float* w_ih, const float* w_ho, const float* Xp, int64_t N, int32_t D, int32_t H,
                   double* grad, void* stream) {
    int rc = check_dims(N, D, H);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (N == 0) {
        GLX_CK(cudaMemsetAsync(grad, 0, sizeof(double) * glx_batch_grad_len(D, H), st));
        return GLX_OK;
    }
    BatchGeom g;
    int kind = 0;
    if (!train_geometry(N, D, H, &g, &kind)) return generic_grad(w_ih, w_ho, Xp, N, D, H, grad, st);
    Workspace* ws = workspace(st);
    GLX_CK(ws->part.ensure((size_t)g.grid * g.PS * 4));
    GLX_CK(ws->wk.ensure((size_t)2 * g.WKS * 4));
    float* wk0 = ws->wk.as<float>();
    GLX_LAUNCH(launch_batch_prep(g, w_ih, w_ho, wk0, wk0 + g.WKS, st));
    const void* in = nullptr;
    rc = epoch_input(ws, g, kind, Xp, st, &in);
    if (rc) return rc;
    const bool check = g_debug.load() && (kind == 2 || kind == 3);
    int* dbg = nullptr;
    if (check) {
        GLX_CK(ws->dbg.ensure(pipeline_check_ints(g) * sizeof(int)));
        dbg = ws->dbg.as<int>();
        GLX_CK(cudaMemsetAsync(dbg, 0, pipeline_check_ints(g) * sizeof(int), st));
    }
    cudaEvent_t pe = nullptr;
    GLX_CK(prof_begin(st, &pe));
    GLX_LAUNCH(launch_train_epoch(g, kind, in, wk0, ws->part.as<float>(), st, dbg));
    if (pe) GLX_CK(cudaEventRecord(pe, st));
    if (check) {
        rc = pipeline_verify(g, kind, dbg, 0, st);
        if (rc) return rc;
    }
    GLX_LAUNCH(launch_batch_grad(g, ws->part.as<float>(), wk0, grad, st));
    return GLX_OK;
}

int glx_batch_apply(float* w_ih, float* w_ho, const double* grad, int32_t D, int32_t H, double lr_over_n,
                    int32_t* nonfinite, void* stream) {
    if (D < 1 || H < 1) return set_err(GLX_ERR_SHAPE, "bad shape");
    GLX_LAUNCH(launch_batch_apply(D, H, w_ih, w_ho, grad, lr_over_n, nonfinite, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_eval(const float* w_ih, const float* w_ho, const float* X, const uint8_t* labels, int64_t N, int32_t D,
             int32_t H, int32_t K, uint64_t* counts4, double* loss, void* stream) {
    int rc = check_dims(N, D, H);
    if (rc) return rc;
    if (K < 1 || K > 16) return set_err(GLX_ERR_INVALID, "output_dim must be in [1, 16], got %d", K);
    cudaStream_t st = (cudaStream_t)stream;
    if (N == 0) {
        GLX_CK(cudaMemsetAsync(loss, 0, sizeof(double), st));
        return GLX_OK;
    }
    const int nparts = eval_nparts(N, H, K);
    Workspace* ws = workspace(st);
    GLX_CK(ws->losspart.ensure((size_t)nparts * sizeof(double)));
    GLX_LAUNCH(launch_eval_ref64(w_ih, w_ho, X, labels, N, D, H, K, reinterpret_cast<unsigned long long*>(counts4),
                                 ws->losspart.as<double>(), nparts, st));
    GLX_LAUNCH(launch_eval_finish(ws->losspart.as<double>(), nparts, loss, st));
    return GLX_OK;
}

int glx_forward(const float* w_ih, const float* w_ho, const float* X, int64_t N, int32_t D, int32_t H, int32_t K,
                float* hidden, float* out, void* stream) {
    int rc = check_dims(N, D, H);
    if (rc) return rc;
    if (K < 1 || K > 16) return set_err(GLX_ERR_INVALID, "output_dim must be in [1, 16], got %d", K);
    if (!hidden || !out) return set_err(GLX_ERR_INVALID, "hidden and out are required");
    if (N == 0) return GLX_OK;
    GLX_CK(launch_forward(w_ih, w_ho, X, N, D, H, K, hidden, out, (cudaStream_t)stream));
    g_launches.fetch_add(2);
    return GLX_OK;
}

int glx_layer_forward(const float* W, const float* X, int64_t N, int32_t m, int32_t n, float* out, void* stream) {
    if (N < 0 || m < 1 || n < 1) return set_err(GLX_ERR_SHAPE, "bad layer shape (N=%lld m=%d n=%d)", (long long)N, m, n);
    if (N == 0) return GLX_OK;
    GLX_LAUNCH(launch_layer_forward(W, X, N, m, n, out, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_layer_backward(const float* x, const float* acts, const double* err, int32_t n, int32_t m, double* deltas,
                       double* grads, void* stream) {
    if (m < 0 || n < 1) return set_err(GLX_ERR_SHAPE, "bad layer shape (m=%d n=%d)", m, n);
    GLX_LAUNCH(launch_layer_backward(x, acts, err, n, m, deltas, grads, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_layer_forward_checked(const float* W, const float* X, int64_t N, int32_t m, int32_t n, float* out,
                              int32_t* write_counts, void* stream) {
    if (N < 0 || m < 1 || n < 1) return set_err(GLX_ERR_SHAPE, "bad layer shape (N=%lld m=%d n=%d)", (long long)N, m, n);
    if (!write_counts) return set_err(GLX_ERR_INVALID, "write_counts is required");
    if (N == 0) return GLX_OK;
    GLX_LAUNCH(launch_layer_forward(W, X, N, m, n, out, (cudaStream_t)stream, write_counts));
    return GLX_OK;
}

int glx_layer_backward_checked(const float* x, const float* acts, const double* err, int32_t n, int32_t m,
                               double* deltas, double* grads, int32_t* write_counts, void* stream) {
    if (m < 0 || n < 1) return set_err(GLX_ERR_SHAPE, "bad layer shape (m=%d n=%d)", m, n);
    if (!write_counts) return set_err(GLX_ERR_INVALID, "write_counts is required");
    GLX_LAUNCH(launch_layer_backward(x, acts, err, n, m, deltas, grads, (cudaStream_t)stream, write_counts));
    return GLX_OK;
}

int glx_forward_pair_debug(const float* w_ih, const float* w_ho, const float* x, int32_t D, int32_t H, int32_t K,
                           float* hidden, float* out, int32_t* stamps, int32_t* status, int32_t workers,
                           void* stream) {
    int rc = check_dims(1, D, H);
    if (rc) return rc;
    if (K < 1 || K > 16) return set_err(GLX_ERR_INVALID, "output_dim must be in [1, 16], got %d", K);
    if (workers < 1 || workers > 32) return set_err(GLX_ERR_INVALID, "workers must be in [1, 32], got %d", workers);
    GLX_LAUNCH(launch_forward_pair_debug(w_ih, w_ho, x, D, H, K, hidden, out, stamps, status, workers,
                                         (cudaStream_t)stream));
    return GLX_OK;
}

int glx_backprop_error(const float* W, const double* deltas, int32_t n, int32_t m, double* err_prev, void* stream) {
    if (m < 1 || n < 1) return set_err(GLX_ERR_SHAPE, "bad layer shape (m=%d n=%d)", m, n);
    GLX_LAUNCH(launch_backprop_error(W, deltas, n, m, err_prev, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_instance_gradients(const float* w_ho, const float* x, const float* hidden, const float* out, double target,
                           int32_t D, int32_t H, double* g_ih, double* g_ho, void* stream) {
    int rc = check_dims(1, D, H);
    if (rc) return rc;
    GLX_LAUNCH(launch_instance_gradients(w_ho, x, hidden, out, target, D, H, g_ih, g_ho, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_eval_packed(const float* w_ih, const float* w_ho, const float* Xp, int64_t N, int32_t D, int32_t H,
                    double* stats, void* stream) {
    int rc = check_dims(N, D, H);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (N == 0) {
        GLX_CK(cudaMemsetAsync(stats, 0, 5 * sizeof(double), st));
        return GLX_OK;
    }
    BatchGeom g;
    if (!batch_geometry(N, D, H, sm_count_current(), false, &g))
        return set_err(GLX_ERR_INVALID, "eval kernel: unsupported shape D=%d H=%d", D, H);
    Workspace* ws = workspace(st);
    GLX_CK(ws->part.ensure((size_t)g.grid * g.PS * 4));
    GLX_CK(ws->wk.ensure((size_t)2 * g.WKS * 4));
    float* wk0 = ws->wk.as<float>();
    GLX_LAUNCH(launch_batch_prep(g, w_ih, w_ho, wk0, wk0 + g.WKS, st));
    GLX_LAUNCH(launch_batch_epoch(g, Xp, wk0, ws->part.as<float>(), false, st));
    GLX_LAUNCH(launch_batch_update(g, ws->part.as<float>(), nullptr, nullptr, wk0, nullptr, 0.0, false, stats,
                                   nullptr, st));
    return GLX_OK;
}

// ----------------------------------------------------------------- host API

static HostState* host_state(int32_t device, int* rc) {
    if (device < 0 || device >= 64) {
        *rc = set_err(GLX_ERR_INVALID, "device %d out of range", device);
        return nullptr;
    }
    HostState* h = &g_host[device];
    return h;
}

#define HOST_PROLOGUE(device)                                                              \
    int rc_ = GLX_OK;                                                                      \
    HostState* hs = host_state(device, &rc_);                                              \
    if (!hs) return rc_;                                                                   \
    std::lock_guard<std::mutex> lk_(hs->mu);                                               \
    GLX_CK(cudaSetDevice(device));                                                         \
    if (!hs->stream) GLX_CK(cudaStreamCreateWithFlags(&hs->stream, cudaStreamNonBlocking)); \
    cudaStream_t st = hs->stream;

// upload feats/targets unless the cache says they are already resident
static int stage_inputs(HostState* hs, const float* feats, size_t xbytes, const float* targets, size_t tbytes,
                        bool cache, cudaStream_t st) {
    const bool hit = cache && hs->key_x == feats && hs->bytes_x == xbytes && hs->key_t == targets &&
                     hs->bytes_t == tbytes && hs->x.p && hs->t.p;
    if (hit) return GLX_OK;
    hs->key_x = hs->key_t = hs->key_xp = nullptr;
    GLX_CK(hs->x.ensure(xbytes));
    GLX_CK(hs->t.ensure(tbytes));
    if (xbytes) GLX_CK(cudaMemcpyAsync(hs->x.p, feats, xbytes, cudaMemcpyHostToDevice, st));
    if (tbytes) GLX_CK(cudaMemcpyAsync(hs->t.p, targets, tbytes, cudaMemcpyHostToDevice, st));
    if (cache) {
        hs->key_x = feats;
        hs->bytes_x = xbytes;
        hs->key_t = targets;
        hs->bytes_t = tbytes;
    }
    return GLX_OK;
}

// online segment on the host state's device buffers (weights uploaded, not downloaded)
static int online_segment_dev(HostState* hs, const float* w_ih, const float* w_ho, const float* feats,
                              const float* targets, int64_t rows, int32_t input_dim, int32_t hidden_dim,
                              int64_t epochs, double lr, int32_t numerics, int32_t flags, cudaStream_t st) {
    const size_t n1 = (size_t)hidden_dim * (input_dim + 1), n2 = (size_t)hidden_dim + 1;
    GLX_CK(hs->w1.ensure(n1 * 4));
    GLX_CK(hs->w2.ensure(n2 * 4));
    int rc = stage_inputs(hs, feats, (size_t)rows * input_dim * 4, targets, (size_t)rows * 4,
                          (flags & GLX_FLAG_CACHE_INPUTS) != 0, st);
    if (rc) return rc;
    GLX_CK(cudaMemcpyAsync(hs->w1.p, w_ih, n1 * 4, cudaMemcpyHostToDevice, st));
    GLX_CK(cudaMemcpyAsync(hs->w2.p, w_ho, n2 * 4, cudaMemcpyHostToDevice, st));
    if (epochs == 0) return GLX_OK;
    std::vector<NetReq> nets{{hs->w1.as<float>(), hs->w2.as<float>(), hidden_dim, 0}};
    return run_online(nets, hs->x.as<float>(), hs->t.as<float>(), rows, input_dim, epochs, lr, numerics == GLX_REF64,
                      st);
}

int glx_run_train_segment(float* w_ih, float* w_ho, const float* feats, const float* targets, int64_t rows,
                          int32_t input_dim, int32_t hidden_dim, int64_t epochs, double lr, int32_t numerics,
                          int32_t device, int32_t flags) {
    int rc = check_dims(rows, input_dim, hidden_dim);
    if (rc) return rc;
    if (epochs < 0) return set_err(GLX_ERR_INVALID, "epochs must be >= 0, got %lld", (long long)epochs);
    if (rows == 0 || epochs == 0) return GLX_OK;
    HOST_PROLOGUE(device);
    const size_t n1 = (size_t)hidden_dim * (input_dim + 1), n2 = (size_t)hidden_dim + 1;
    rc = online_segment_dev(hs, w_ih, w_ho, feats, targets, rows, input_dim, hidden_dim, epochs, lr, numerics, flags,
                            st);
    if (rc) return rc;
    GLX_CK(cudaMemcpyAsync(w_ih, hs->w1.p, n1 * 4, cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaMemcpyAsync(w_ho, hs->w2.p, n2 * 4, cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaStreamSynchronize(st));
    return GLX_OK;
}

// full-batch segment on the host state's device buffers (weights uploaded, not downloaded)
static int batch_segment_dev(HostState* hs, const float* w_ih, const float* w_ho, const float* feats,
                             const float* targets, int64_t rows, int32_t input_dim, int32_t hidden_dim,
                             int64_t epochs, double lr, bool want_stats, int32_t flags, cudaStream_t st) {
    const int ld = glx_packed_ld(input_dim);
    const size_t n1 = (size_t)hidden_dim * (input_dim + 1), n2 = (size_t)hidden_dim + 1;
    GLX_CK(hs->w1.ensure(n1 * 4));
    GLX_CK(hs->w2.ensure(n2 * 4));
    int rc = GLX_OK;
    const bool cache = (flags & GLX_FLAG_CACHE_INPUTS) != 0;
    const bool packed_hit = cache && hs->key_xp == feats && hs->key_x == feats && hs->key_t == targets &&
                            hs->bytes_x == (size_t)rows * input_dim * 4;
    if (!packed_hit) {
        rc = stage_inputs(hs, feats, (size_t)rows * input_dim * 4, targets, (size_t)rows * 4, cache, st);
        if (rc) return rc;
        GLX_CK(hs->xp.ensure((size_t)rows * ld * 4));
        GLX_LAUNCH(launch_pack_rows(hs->x.as<float>(), hs->t.as<float>(), nullptr, rows, input_dim, ld,
                                    hs->xp.as<float>(), st));
        if (cache) hs->key_xp = feats;
    }
    GLX_CK(hs->stats.ensure((size_t)5 * std::max<int64_t>(epochs, 1) * sizeof(double)));
    GLX_CK(hs->flag.ensure(sizeof(int)));
    GLX_CK(cudaMemsetAsync(hs->flag.p, 0, sizeof(int), st));
    GLX_CK(cudaMemcpyAsync(hs->w1.p, w_ih, n1 * 4, cudaMemcpyHostToDevice, st));
    GLX_CK(cudaMemcpyAsync(hs->w2.p, w_ho, n2 * 4, cudaMemcpyHostToDevice, st));
    if (epochs == 0) return GLX_OK;
    return batch_train_impl(hs->w1.as<float>(), hs->w2.as<float>(), hs->xp.as<float>(), rows, input_dim, hidden_dim,
                            epochs, lr, want_stats ? hs->stats.as<double>() : nullptr, hs->flag.as<int>(), st,
                            (flags & GLX_FLAG_DEBUG) != 0);
}

int glx_run_train_segment_batch(float* w_ih, float* w_ho, const float* feats, const float* targets, int64_t rows,
                                int32_t input_dim, int32_t hidden_dim, int64_t epochs, double lr,
                                double* stats_hist, int32_t device, int32_t flags) {
    int rc = check_dims(rows, input_dim, hidden_dim);
    if (rc) return rc;
    if (epochs < 0) return set_err(GLX_ERR_INVALID, "epochs must be >= 0, got %lld", (long long)epochs);
    if (rows == 0 || epochs == 0) return GLX_OK;
    HOST_PROLOGUE(device);
    const size_t n1 = (size_t)hidden_dim * (input_dim + 1), n2 = (size_t)hidden_dim + 1;
    rc = batch_segment_dev(hs, w_ih, w_ho, feats, targets, rows, input_dim, hidden_dim, epochs, lr,
                           stats_hist != nullptr, flags, st);
    if (rc) return rc;
    GLX_CK(cudaMemcpyAsync(w_ih, hs->w1.p, n1 * 4, cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaMemcpyAsync(w_ho, hs->w2.p, n2 * 4, cudaMemcpyDeviceToHost, st));
    if (stats_hist)
        GLX_CK(cudaMemcpyAsync(stats_hist, hs->stats.p, (size_t)5 * epochs * sizeof(double), cudaMemcpyDeviceToHost,
                               st));
    GLX_CK(cudaStreamSynchronize(st));
    return GLX_OK;
}

int glx_eval_counts(const float* w_ih, const float* w_ho, const float* feats, const uint8_t* labels, int64_t rows,
                    int32_t input_dim, int32_t hidden_dim, int32_t output_dim, int32_t numerics, int64_t* counts4,
                    double* loss_sum, int32_t device, int32_t flags) {
    int rc = check_dims(rows, input_dim, hidden_dim);
    if (rc) return rc;
    if (output_dim < 1 || output_dim > 16)
        return set_err(GLX_ERR_INVALID, "output_dim must be in [1, 16], got %d", output_dim);
    for (int q = 0; q < 4; q++) counts4[q] = 0;
    if (loss_sum) *loss_sum = 0.0;
    if (rows == 0) return GLX_OK;
    HOST_PROLOGUE(device);
    const size_t n1 = (size_t)hidden_dim * (input_dim + 1), n2 = (size_t)output_dim * (hidden_dim + 1);
    GLX_CK(hs->w1.ensure(n1 * 4));
    GLX_CK(hs->w2.ensure(n2 * 4));
    GLX_CK(hs->cnt.ensure(4 * sizeof(uint64_t)));
    GLX_CK(hs->loss.ensure(8 * sizeof(double)));
    GLX_CK(cudaMemcpyAsync(hs->w1.p, w_ih, n1 * 4, cudaMemcpyHostToDevice, st));
    GLX_CK(cudaMemcpyAsync(hs->w2.p, w_ho, n2 * 4, cudaMemcpyHostToDevice, st));
    // evaluation inputs use their own buffers (train and test splits alternate;
    // the training-input cache stays intact)
    (void)flags;
    const size_t xbytes = (size_t)rows * input_dim * 4;
    GLX_CK(hs->lab.ensure((size_t)rows));
    GLX_CK(cudaMemcpyAsync(hs->lab.p, labels, (size_t)rows, cudaMemcpyHostToDevice, st));
    DevBuf* xb = &hs->ex;
    GLX_CK(xb->ensure(xbytes));
    GLX_CK(cudaMemcpyAsync(xb->p, feats, xbytes, cudaMemcpyHostToDevice, st));
    uint64_t hc[4] = {0, 0, 0, 0};
    double hl[5] = {0, 0, 0, 0, 0};
    BatchGeom eg;
    const bool fused_eval = batch_geometry(rows, input_dim, hidden_dim, sm_count_current(), false, &eg);
    if (numerics == GLX_REF64 || output_dim > 1 || !fused_eval) {  // exact kernel (any shape)
        GLX_CK(cudaMemsetAsync(hs->cnt.p, 0, 4 * sizeof(uint64_t), st));
        rc = glx_eval(hs->w1.as<float>(), hs->w2.as<float>(), xb->as<float>(), hs->lab.as<uint8_t>(), rows, input_dim,
                      hidden_dim, output_dim, hs->cnt.as<uint64_t>(), hs->loss.as<double>(), st);
        if (rc) return rc;
        GLX_CK(cudaMemcpyAsync(hc, hs->cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
        GLX_CK(cudaMemcpyAsync(hl, hs->loss.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        GLX_CK(cudaStreamSynchronize(st));
        for (int q = 0; q < 4; q++) counts4[q] = (int64_t)hc[q];
        if (loss_sum) *loss_sum = hl[0];
        return GLX_OK;
    }
    // fast FP32 path: pack rows (labels as targets) then the fused streaming forward
    const int ld = glx_packed_ld(input_dim);
    GLX_CK(hs->exp_.ensure((size_t)rows * ld * 4));
    GLX_LAUNCH(launch_pack_rows(xb->as<float>(), nullptr, hs->lab.as<uint8_t>(), rows, input_dim, ld,
                                hs->exp_.as<float>(), st));
    rc = glx_eval_packed(hs->w1.as<float>(), hs->w2.as<float>(), hs->exp_.as<float>(), rows, input_dim, hidden_dim,
                         hs->loss.as<double>(), st);
    if (rc) return rc;
    GLX_CK(cudaMemcpyAsync(hl, hs->loss.p, 5 * sizeof(double), cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaStreamSynchronize(st));
    if (loss_sum) *loss_sum = hl[0];
    for (int q = 0; q < 4; q++) counts4[q] = (int64_t)llround(hl[1 + q]);
    return GLX_OK;
}

// upload a host buffer into `buf` unless (key, bytes) says it is resident
static int stage_buf(DevBuf& buf, const void*& key, size_t* key_bytes, const void* src, size_t bytes, bool cache,
                     cudaStream_t st) {
    if (cache && key == src && buf.p && (!key_bytes || *key_bytes == bytes)) return GLX_OK;
    key = nullptr;
    GLX_CK(buf.ensure(bytes));
    if (bytes) GLX_CK(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, st));
    if (cache) {
        key = src;
        if (key_bytes) *key_bytes = bytes;
    }
    return GLX_OK;
}

int glx_run_train_segment_eval(float* w_ih, float* w_ho, const float* feats, const float* targets,
                               const uint8_t* labels, int64_t rows, const float* test_feats,
                               const uint8_t* test_labels, int64_t test_rows, int32_t input_dim, int32_t hidden_dim,
                               int64_t epochs, double lr, int32_t numerics, int32_t mode, int32_t device,
                               int32_t flags, int64_t* counts8, double* loss2, int32_t* finite, double* train_seconds) {
    int rc = check_dims(rows, input_dim, hidden_dim);
    if (rc) return rc;
    if (test_rows < 0) return set_err(GLX_ERR_SHAPE, "test_rows must be >= 0");
    if (epochs < 0) return set_err(GLX_ERR_INVALID, "epochs must be >= 0, got %lld", (long long)epochs);
    if (mode != 0 && mode != 1) return set_err(GLX_ERR_INVALID, "mode must be 0 (online) or 1 (batch)");
    if (rows == 0) return set_err(GLX_ERR_SHAPE, "training rows must not be empty");
    auto t0 = std::chrono::steady_clock::now();
    HOST_PROLOGUE(device);
    const size_t n1 = (size_t)hidden_dim * (input_dim + 1), n2 = (size_t)hidden_dim + 1;
    rc = mode == 0 ? online_segment_dev(hs, w_ih, w_ho, feats, targets, rows, input_dim, hidden_dim, epochs, lr,
                                        numerics, flags, st)
                   : batch_segment_dev(hs, w_ih, w_ho, feats, targets, rows, input_dim, hidden_dim, epochs, lr, false,
                                       flags, st);
    if (rc) return rc;
    // checkpoint evaluation on the device, same stream: exact (ref64) counts for the
    // train rows (already resident) and the test rows; the eval's own device time is
    // excluded from train_seconds
    const bool cache = (flags & GLX_FLAG_CACHE_INPUTS) != 0;
    cudaEvent_t e0, e1;
    GLX_CK(cudaEventCreate(&e0));
    GLX_CK(cudaEventCreate(&e1));
    GLX_CK(cudaEventRecord(e0, st));
    rc = stage_buf(hs->tlab, hs->key_tlab, nullptr, labels, (size_t)rows, cache, st);
    if (!rc && test_rows) rc = stage_buf(hs->vx, hs->key_vx, &hs->bytes_vx, test_feats,
                                         (size_t)test_rows * input_dim * 4, cache, st);
    if (!rc && test_rows) rc = stage_buf(hs->vlab, hs->key_vlab, nullptr, test_labels, (size_t)test_rows, cache, st);
    if (rc) return rc;
    GLX_CK(hs->cnt.ensure(8 * sizeof(uint64_t)));
    GLX_CK(hs->loss.ensure(8 * sizeof(double)));
    GLX_CK(hs->flag.ensure(sizeof(int)));
    GLX_CK(cudaMemsetAsync(hs->cnt.p, 0, 8 * sizeof(uint64_t), st));
    GLX_CK(cudaMemsetAsync(hs->loss.p, 0, 2 * sizeof(double), st));
    GLX_CK(cudaMemsetAsync(hs->flag.p, 0, sizeof(int), st));
    GLX_LAUNCH(launch_nonfinite(hs->w1.as<float>(), (int64_t)n1, hs->w2.as<float>(), (int64_t)n2, hs->flag.as<int>(),
                                st));
    uint64_t* cnt = hs->cnt.as<uint64_t>();
    double* loss = hs->loss.as<double>();
    rc = glx_eval(hs->w1.as<float>(), hs->w2.as<float>(), hs->x.as<float>(), hs->tlab.as<uint8_t>(), rows, input_dim,
                  hidden_dim, 1, cnt, loss, st);
    if (!rc && test_rows)
        rc = glx_eval(hs->w1.as<float>(), hs->w2.as<float>(), hs->vx.as<float>(), hs->vlab.as<uint8_t>(), test_rows,
                      input_dim, hidden_dim, 1, cnt + 4, loss + 1, st);
    if (rc) return rc;
    GLX_CK(cudaEventRecord(e1, st));
    uint64_t hc[8];
    double hl[2];
    int hf = 0;
    GLX_CK(cudaMemcpyAsync(w_ih, hs->w1.p, n1 * 4, cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaMemcpyAsync(w_ho, hs->w2.p, n2 * 4, cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaMemcpyAsync(hc, hs->cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaMemcpyAsync(hl, hs->loss.p, sizeof(hl), cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaMemcpyAsync(&hf, hs->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaStreamSynchronize(st));
    float eval_ms = 0.f;
    GLX_CK(cudaEventElapsedTime(&eval_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (int q = 0; q < 8; q++) counts8[q] = (int64_t)hc[q];
    if (loss2) {
        loss2[0] = hl[0];
        loss2[1] = test_rows ? hl[1] : 0.0;
    }
    if (finite) *finite = hf ? 0 : 1;
    if (train_seconds) {
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *train_seconds = std::max(0.0, wall - eval_ms * 1e-3);
    }
    return GLX_OK;
}

int glx_tc_gemm_bf16(const void* A, const void* B, int32_t M, int32_t N, int32_t K, int32_t epilogue, float* d_f32,
                     void* d_bf16, const float* bias, int32_t ldd, void* stream) {
    if (M < 1 || N < 1 || K < 1 || K % 64 || N % 32)
        return set_err(GLX_ERR_SHAPE, "tc gemm needs K %% 64 == 0 and N %% 32 == 0 (M=%d N=%d K=%d)", M, N, K);
    GLX_LAUNCH(launch_tc_gemm(A, B, M, N, K, epilogue, d_f32, d_bf16, bias, ldd, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_wide_make_shard(int64_t row0, int64_t N, uint64_t seed, void* Xb, void* XT, uint8_t* labels, void* stream) {
    if (N < 64 || N % 64) return set_err(GLX_ERR_SHAPE, "wide data needs N %% 64 == 0 (got %lld)", (long long)N);
    if (row0 < 0) return set_err(GLX_ERR_INVALID, "row0 must be >= 0");
    GLX_LAUNCH(launch_wide_gen(Xb, XT, labels, N, seed, row0, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_wide_make_data(int64_t N, uint64_t seed, void* Xb, void* XT, uint8_t* labels, void* stream) {
    return glx_wide_make_shard(0, N, seed, Xb, XT, labels, stream);
}

int64_t glx_wide_grad_len(void) { return kWideP + 3; }

int glx_wide_grad(const float* w_ih, const float* w_ho, const void* Xb, const void* XT, const uint8_t* labels,
                  int64_t N, double* grad, void* stream) {
    if (N < 64 || N % 64) return set_err(GLX_ERR_SHAPE, "wide gradient needs N %% 64 == 0 (got %lld)", (long long)N);
    if (!grad) return set_err(GLX_ERR_INVALID, "grad must be a device buffer of glx_wide_grad_len() doubles");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t C = std::min<int64_t>(N, (int64_t)1 << 20);
    const int splits = 8;
    Workspace* ws = workspace(st);
    GLX_CK(ws->wide.ensure(wide_work_bytes(C, splits)));
    GLX_CK(wide_grad(w_ih, w_ho, Xb, XT, labels, N, ws->wide.as<unsigned char>(), C, splits, grad, st,
                     [](bool) {}));
    g_launches.fetch_add(3 + wide_launches_per_chunk() * (uint64_t)((N + C - 1) / C));
    return GLX_OK;
}

// ---------------------------------------------------------- wide, tf32 path
int glx_wide_make_shard_tf32(int64_t row0, int64_t N, uint64_t seed, float* X, float* XT, uint8_t* labels,
                             void* stream) {
    if (N < 32 || N % 32) return set_err(GLX_ERR_SHAPE, "wide tf32 data needs N %% 32 == 0 (got %lld)", (long long)N);
    if (row0 < 0) return set_err(GLX_ERR_INVALID, "row0 must be >= 0");
    GLX_LAUNCH(launch_wide_gen_tf32(X, XT, labels, N, seed, row0, (cudaStream_t)stream));
    return GLX_OK;
}

static int64_t wide32_chunk(int64_t N) { return std::min<int64_t>(N, (int64_t)1 << 19); }  // rows per chunk

int glx_wide_grad_tf32(const float* w_ih, const float* w_ho, const float* X, const float* XT, const uint8_t* labels,
                       int64_t N, double* grad, void* stream) {
    if (N < 32 || N % 32) return set_err(GLX_ERR_SHAPE, "wide tf32 gradient needs N %% 32 == 0 (got %lld)", (long long)N);
    if (!grad) return set_err(GLX_ERR_INVALID, "grad must be a device buffer of glx_wide_grad_len() doubles");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t C = wide32_chunk(N);
    const int splits = 8;
    Workspace* ws = workspace(st);
    GLX_CK(ws->wide.ensure(wide32_work_bytes(C, splits)));
    GLX_CK(wide_grad_tf32(w_ih, w_ho, X, XT, labels, N, ws->wide.as<unsigned char>(), C, splits, grad, st,
                          [](bool) {}));
    g_launches.fetch_add(3 + wide32_launches_per_chunk() * (uint64_t)((N + C - 1) / C));
    return GLX_OK;
}

int glx_wide_train_tf32(float* w_ih, float* w_ho, const float* X, const float* XT, const uint8_t* labels, int64_t N,
                        int64_t epochs, double lr, double* stats_hist, int32_t* nonfinite, void* stream) {
    if (N < 32 || N % 32) return set_err(GLX_ERR_SHAPE, "wide tf32 training needs N %% 32 == 0 (got %lld)", (long long)N);
    if (epochs < 0) return set_err(GLX_ERR_INVALID, "epochs must be >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t C = wide32_chunk(N);
    const int splits = 8;
    Workspace* ws = workspace(st);
    GLX_CK(ws->wide.ensure(wide32_work_bytes(C, splits)));
    for (int64_t e = 0; e < epochs; e++) {
        double* stats = stats_hist ? stats_hist + 3 * e : nullptr;
        cudaEvent_t pe = nullptr;
        cudaError_t perr = cudaSuccess;
        auto prof = [&](bool begin) {
            if (begin) {
                cudaError_t r = prof_begin(st, &pe);
                if (r != cudaSuccess) perr = r;
            } else if (pe) {
                cudaError_t r = cudaEventRecord(pe, st);
                if (r != cudaSuccess) perr = r;
                pe = nullptr;
            }
        };
        GLX_CK(wide_epoch_tf32(w_ih, w_ho, X, XT, labels, N, lr, ws->wide.as<unsigned char>(), C, splits, stats,
                               nonfinite, st, prof));
        GLX_CK(perr);
        g_launches.fetch_add(4 + wide32_launches_per_chunk() * (uint64_t)((N + C - 1) / C));
    }
    return GLX_OK;
}

int glx_wide_apply(float* w_ih, float* w_ho, const double* grad, double lr_over_n, int32_t* nonfinite, void* stream) {
    if (!grad) return set_err(GLX_ERR_INVALID, "grad must not be NULL");
    GLX_CK(wide_apply(w_ih, w_ho, grad, lr_over_n, nonfinite, (cudaStream_t)stream));
    g_launches.fetch_add(1);
    return GLX_OK;
}

int glx_wide_train(float* w_ih, float* w_ho, const void* Xb, const void* XT, const uint8_t* labels, int64_t N,
                   int64_t epochs, double lr, double* stats_hist, int32_t* nonfinite, void* stream) {
    if (N < 64 || N % 64) return set_err(GLX_ERR_SHAPE, "wide training needs N %% 64 == 0 (got %lld)", (long long)N);
    if (epochs < 0) return set_err(GLX_ERR_INVALID, "epochs must be >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t C = std::min<int64_t>(N, (int64_t)1 << 20);  // rows per chunk (multiple of 64)
    const int splits = 8;
    Workspace* ws = workspace(st);
    GLX_CK(ws->wide.ensure(wide_work_bytes(C, splits)));
    for (int64_t e = 0; e < epochs; e++) {
        double* stats = stats_hist ? stats_hist + 3 * e : nullptr;
        if (stats) GLX_CK(cudaMemsetAsync(stats, 0, 3 * sizeof(double), st));
        cudaEvent_t pe = nullptr;
        cudaError_t perr = cudaSuccess;
        auto prof = [&](bool begin) {
            if (begin) {
                cudaError_t r = prof_begin(st, &pe);
                if (r != cudaSuccess) perr = r;
            } else if (pe) {
                cudaError_t r = cudaEventRecord(pe, st);
                if (r != cudaSuccess) perr = r;
                pe = nullptr;
            }
        };
        GLX_CK(wide_epoch(w_ih, w_ho, Xb, XT, labels, N, lr, ws->wide.as<unsigned char>(), C, splits, stats,
                          nonfinite, st, prof));
        GLX_CK(perr);
        g_launches.fetch_add(4 + wide_launches_per_chunk() * (uint64_t)((N + C - 1) / C));
    }
    return GLX_OK;
}

// ------------------------------------------------------------ data parallel
int glx_dp_unique_id(uint8_t* id128) {
    if (!id128) return set_err(GLX_ERR_INVALID, "id buffer is NULL");
    GLX_NCCL_API();
    ncclUniqueId id;
    GLX_NCCL(nccl().GetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(id128, &id, sizeof(id));
    return GLX_OK;
}

int glx_dp_init(int32_t device, int32_t nranks, int32_t rank, const uint8_t* id128, void** comm_out) {
    if (!id128 || !comm_out) return set_err(GLX_ERR_INVALID, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return set_err(GLX_ERR_INVALID, "rank %d of %d out of range", rank, nranks);
    GLX_NCCL_API();
    GLX_CK(cudaSetDevice(device));
    DpComm* dp = new DpComm();
    dp->dev = device;
    dp->nranks = nranks;
    dp->rank = rank;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclResult_t r = nccl().CommInitRank(&dp->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete dp;
        return set_err(GLX_ERR_CUDA, "ncclCommInitRank failed: %s", nccl().GetErrorString(r));
    }
    GLX_CK(cudaStreamCreateWithFlags(&dp->st, cudaStreamNonBlocking));
    GLX_CK(cudaEventCreateWithFlags(&dp->ev_in, cudaEventDisableTiming));
    GLX_CK(cudaEventCreateWithFlags(&dp->ev_out, cudaEventDisableTiming));
    *comm_out = dp;
    return GLX_OK;
}

int glx_dp_finalize(void* comm) {
    DpComm* dp = (DpComm*)comm;
    if (!dp) return GLX_OK;
    cudaSetDevice(dp->dev);
    cudaStreamSynchronize(dp->st);
    dp->drop_graphs();
    ncclResult_t r = nccl().CommDestroy(dp->comm);
    cudaEventDestroy(dp->ev_in);
    cudaEventDestroy(dp->ev_out);
    cudaStreamDestroy(dp->st);
    if (dp->grad.p) cudaFree(dp->grad.p);
    if (dp->slot.p) cudaFree(dp->slot.p);
    delete dp;
    if (r != ncclSuccess) return set_err(GLX_ERR_CUDA, "ncclCommDestroy failed: %s", nccl().GetErrorString(r));
    return GLX_OK;
}

int glx_dp_allreduce_f64(void* comm, double* buf, int64_t n, int32_t op, void* stream) {
    DpComm* dp = (DpComm*)comm;
    if (!dp) return set_err(GLX_ERR_INVALID, "communicator is NULL");
    if (n < 0 || (op != 0 && op != 1)) return set_err(GLX_ERR_INVALID, "bad count or op");
    GLX_CK(cudaSetDevice(dp->dev));
    GLX_NCCL(nccl().AllReduce(buf, buf, (size_t)n, ncclDouble, op ? ncclMax : ncclSum, dp->comm, (cudaStream_t)stream));
    return GLX_OK;
}

int glx_dp_train_batch(void* comm, float* w_ih, float* w_ho, const float* Xp, int64_t N, int64_t N_total, int32_t D,
                       int32_t H, int64_t epochs, double lr, double* stats_hist, int32_t* nonfinite, void* stream) {
    DpComm* dp = (DpComm*)comm;
    if (!dp) return set_err(GLX_ERR_INVALID, "communicator is NULL");
    int rc = check_dims(N, D, H);
    if (rc) return rc;
    if (N_total < N || N_total < 1) return set_err(GLX_ERR_SHAPE, "total rows %lld < local rows %lld",
                                                   (long long)N_total, (long long)N);
    if (epochs <= 0) return GLX_OK;
    return dp_train_batch(dp, w_ih, w_ho, Xp, N, N_total, D, H, epochs, lr, stats_hist, nonfinite,
                          (cudaStream_t)stream);
}

int glx_dp_run_train_segment_batch(void* comm, float* w_ih, float* w_ho, const float* feats, const float* targets,
                                   int64_t rows, int64_t rows_total, int32_t input_dim, int32_t hidden_dim,
                                   int64_t epochs, double lr, double* stats_hist, int32_t flags) {
    DpComm* dp = (DpComm*)comm;
    if (!dp) return set_err(GLX_ERR_INVALID, "communicator is NULL");
    int rc = check_dims(rows, input_dim, hidden_dim);
    if (rc) return rc;
    if (epochs < 0) return set_err(GLX_ERR_INVALID, "epochs must be >= 0, got %lld", (long long)epochs);
    if (rows_total < rows || rows_total < 1)
        return set_err(GLX_ERR_SHAPE, "total rows %lld < local rows %lld", (long long)rows_total, (long long)rows);
    if (epochs == 0) return GLX_OK;
    HOST_PROLOGUE(dp->dev);
    const size_t n1 = (size_t)hidden_dim * (input_dim + 1), n2 = (size_t)hidden_dim + 1;
    rc = batch_segment_dev(hs, w_ih, w_ho, feats, targets, rows, input_dim, hidden_dim, 0, lr, false, flags, st);
    if (rc) return rc;
    GLX_CK(hs->stats.ensure((size_t)5 * epochs * sizeof(double)));
    rc = dp_train_batch(dp, hs->w1.as<float>(), hs->w2.as<float>(), hs->xp.as<float>(), rows, rows_total, input_dim,
                        hidden_dim, epochs, lr, stats_hist ? hs->stats.as<double>() : nullptr, hs->flag.as<int>(), st);
    if (rc) return rc;
    GLX_CK(cudaMemcpyAsync(w_ih, hs->w1.p, n1 * 4, cudaMemcpyDeviceToHost, st));
    GLX_CK(cudaMemcpyAsync(w_ho, hs->w2.p, n2 * 4, cudaMemcpyDeviceToHost, st));
    if (stats_hist)
        GLX_CK(cudaMemcpyAsync(stats_hist, hs->stats.p, (size_t)5 * epochs * sizeof(double), cudaMemcpyDeviceToHost,
                               st));
    GLX_CK(cudaStreamSynchronize(st));
    return GLX_OK;
}

void glx_set_debug(int32_t on) { g_debug.store(on ? 1 : 0); }

void glx_profile_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = on != 0;
    g_prof.used = 0;
}

int glx_profile_read(double* total_ms, int64_t* launches) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    double tot = 0.0;
    for (size_t i = 0; i < g_prof.used; i++) {
        GLX_CK(cudaEventSynchronize(g_prof.pairs[i].second));
        float ms = 0.f;
        GLX_CK(cudaEventElapsedTime(&ms, g_prof.pairs[i].first, g_prof.pairs[i].second));
        tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = (int64_t)g_prof.used;
    g_prof.used = 0;
    return GLX_OK;
}

int glx_fp32_peak(int32_t device, int32_t iters, double* tflops, double* ms) {
    GLX_CK(cudaSetDevice(device));
    const int sms = glx_sm_count(device);
    const int blocks = sms * 8;
    float* out = nullptr;
    GLX_CK(cudaMalloc(&out, (size_t)blocks * 256 * 4));
    cudaEvent_t e0, e1;
    GLX_CK(cudaEventCreate(&e0));
    GLX_CK(cudaEventCreate(&e1));
    GLX_LAUNCH(launch_fp32_peak(out, 16, blocks, nullptr));  // warm-up
    GLX_CK(cudaEventRecord(e0, nullptr));
    GLX_LAUNCH(launch_fp32_peak(out, iters, blocks, nullptr));
    GLX_CK(cudaEventRecord(e1, nullptr));
    GLX_CK(cudaEventSynchronize(e1));
    float t = 0.f;
    GLX_CK(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = (double)blocks * 256 * (double)iters * 16 * 8 * 4;
    if (ms) *ms = t;
    if (tflops) *tflops = flops / ((double)t * 1e-3) / 1e12;
    return GLX_OK;
}

}  // extern "C"
