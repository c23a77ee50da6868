// api.cu -- the C ABI (include/gcm.h): argument validation, the per-(device,
// stream) workspace cache, algorithm dispatch and the failure report.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "internal.h"
#include "tma.cuh"

namespace gcm {

// Every ABI entry point that enqueues work first consumes a stale sticky-free error a
// previous failed call may have left (cudaGetLastError), so a later launch check never
// reports an old failure after new work was already enqueued (gcm.h: an error return
// means nothing was enqueued by THIS call's failing step).
void clear_stale_error() { (void)cudaGetLastError(); }

gcm_status_t check_cuda(cudaError_t e) {
    if (e == cudaSuccess) return GCM_OK;
    if (std::getenv("GCM_DEBUG")) std::fprintf(stderr, "gcm: CUDA error %d: %s\n", (int)e, cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) return GCM_ENOMEM;
    return GCM_ECUDA;
}

bool g_profile_on = false;
static std::atomic<long long> g_launches{0};
void count_launch(int n) {
    if (g_profile_on) g_launches += n;
}

namespace {

struct ProfRec {
    std::string name;
    cudaEvent_t b, e;
};
std::mutex g_prof_mutex;
std::vector<ProfRec> g_prof_open, g_prof_done;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t prof_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t ev = g_event_pool.back();
        g_event_pool.pop_back();
        return ev;
    }
    cudaEvent_t ev = nullptr;
    cudaEventCreate(&ev);
    return ev;
}

}  // namespace

void prof_record(const char *name, cudaStream_t stream, bool begin) {
    std::lock_guard<std::mutex> lock(g_prof_mutex);
    cudaEvent_t ev = prof_event();
    cudaEventRecord(ev, stream);
    if (begin) {
        g_prof_open.push_back({name, ev, nullptr});
    } else {
        for (size_t i = g_prof_open.size(); i-- > 0;) {
            if (g_prof_open[i].name == name) {
                g_prof_open[i].e = ev;
                g_prof_done.push_back(g_prof_open[i]);
                g_prof_open.erase(g_prof_open.begin() + i);
                return;
            }
        }
        g_event_pool.push_back(ev);
    }
}

namespace {

std::mutex g_ws_mutex;
std::map<std::pair<int, cudaStream_t>, Workspace> g_ws;

// gcm_modify_host's per-device staging: its own non-blocking stream and one device
// buffer (L + V + info), grown on demand and freed by gcm_release_workspace.
struct HostStage {
    cudaStream_t stream = nullptr;
    void *buf = nullptr;
    size_t cap = 0;
};
std::mutex g_host_mutex;
std::map<int, HostStage> g_host;

__global__ void info_finalize_kernel(const unsigned long long *key, gcm_info_t *info, int64_t count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const unsigned long long kv = key[i];
    gcm_info_t r;
    if (kv == kInfoNone) {
        r.code = 0;
        r.col = 0;
        r.row = 0;
    } else {
        r.code = (kv & 1ull) ? 1 : 2;
        r.col = (int32_t)(kv >> 41);
        r.row = (int64_t)((kv >> 1) & ((1ull << 40) - 1));
    }
    info[i] = r;
}

gcm_status_t validate(const double *L, int64_t n, int64_t ldl, const double *V, int64_t k, int sigma) {
    if (n < 0 || k < 0 || ldl < std::max<int64_t>(1, n)) return GCM_EINVAL;
    if (sigma != 1 && sigma != -1) return GCM_EINVAL;
    if (n > 0 && k > 0 && (L == nullptr || V == nullptr)) return GCM_EINVAL;
    if (n >= (1ll << 40) || k >= (1ll << 22)) return GCM_EINVAL;
    return GCM_OK;
}

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool encode_tmap_f64(CUtensorMap *m, const void *base, int rank, int64_t rows, int64_t cols, int64_t ldl,
                     int64_t batch, int64_t strideL, unsigned box_rows, unsigned box_cols, CUtensorMapSwizzle swz,
                     CUtensorMapDataType dtype, int esize) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p) {
            clear_stale_error();
            return false;
        }
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    if (rank != 2 && rank != 3) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)rows, (cuuint64_t)cols, (cuuint64_t)batch};
    const cuuint64_t strides[2] = {(cuuint64_t)ldl * esize, (cuuint64_t)strideL * esize};
    const cuuint32_t box[3] = {box_rows, box_cols, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, dtype, (cuuint32_t)rank, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

gcm_algo_t pick_algo(int64_t n, int64_t k, gcm_algo_t algo) {
    if (algo != GCM_ALGO_AUTO) return algo;
    const char *env = std::getenv("GCM_ALGO");
    if (env && std::strcmp(env, "sweep") == 0) return GCM_ALGO_SWEEP;
    if (env && std::strcmp(env, "blocked") == 0) return GCM_ALGO_BLOCKED;
    if (env && std::strcmp(env, "panel") == 0) return GCM_ALGO_PANEL;
    // the chain-shortened path wins once there is more
    // than a handful of row blocks; tiny factors keep the two-kernel sweep; large factors
    // take the column-block (panel) algorithm, whose solve chain and residual updates run on
    // the FP64 tensor cores and whose sweeps and Apply overlap the chain on parallel streams
    // (profiles/r02cq_crossover.txt: level with BLOCKED at n ~ 4700 for k <= 16, ~ 6000 for
    // k = 32; n = 5000, k = 16: 0.329 vs 0.342 ms; n = 10000, k = 32: 1.08 vs 1.48 ms).
    if (n >= 6500 || (n >= 4700 && k <= 16)) return GCM_ALGO_PANEL;
    return n >= 256 ? GCM_ALGO_BLOCKED : GCM_ALGO_SWEEP;
}

gcm_status_t get_workspace(cudaStream_t stream, size_t bytes, size_t nkeys, Workspace **out) {
    int dev = 0;
    gcm_status_t st = check_cuda(cudaGetDevice(&dev));
    if (st != GCM_OK) return st;
    const size_t key_bytes = ((nkeys * sizeof(unsigned long long) + 255) / 256) * 256;
    const size_t need = key_bytes + ((bytes + 255) / 256) * 256;
    std::lock_guard<std::mutex> lock(g_ws_mutex);
    Workspace &ws = g_ws[{dev, stream}];
    if (ws.bytes < need) {
        if (ws.key) {
            // the old buffer may still be in use by work queued on this stream
            st = check_cuda(cudaStreamSynchronize(stream));
            if (st != GCM_OK) return st;
            cudaFree(ws.key);
            ws = Workspace{};
        }
        const size_t alloc = need + need / 4;
        void *p = nullptr;
        st = check_cuda(cudaMalloc(&p, alloc));
        if (st != GCM_OK) {
            clear_stale_error();
            return st;
        }
        // device flags compare against a per-call epoch: start from all-zero
        st = check_cuda(cudaMemsetAsync(p, 0, alloc, stream));
        if (st != GCM_OK) return st;
        ws.key = static_cast<unsigned long long *>(p);
        ws.bytes = alloc;
        ws.epoch = 0;
    }
    ws.panels = reinterpret_cast<double *>(reinterpret_cast<char *>(ws.key) + key_bytes);
    ws.extra = ws.panels;
    *out = &ws;
    return GCM_OK;
}

gcm_status_t finalize_info(const unsigned long long *key, gcm_info_t *d_info, int64_t count, cudaStream_t stream) {
    if (!d_info || count <= 0) return GCM_OK;
    const int threads = 128;
    const unsigned grid = (unsigned)((count + threads - 1) / threads);
    info_finalize_kernel<<<grid, threads, 0, stream>>>(key, d_info, count);
    count_launch();
    return check_cuda(cudaGetLastError());
}

size_t single_workspace_bytes(int64_t n, int64_t k, gcm_algo_t algo) {
    const int64_t nblk = (n + kD - 1) / kD;
    size_t bytes = (size_t)nblk * panel_doubles((int)std::min<int64_t>(k, kKMax)) * sizeof(double);
    if (algo == GCM_ALGO_BLOCKED) bytes = std::max(bytes, blocked_workspace_bytes(n, k));
    return bytes;
}

gcm_status_t run_single(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma, gcm_algo_t algo,
                        unsigned long long *key, Workspace *ws, cudaStream_t stream) {
    gcm_status_t st = check_cuda(cudaMemsetAsync(key, 0xff, sizeof(unsigned long long), stream));
    if (st != GCM_OK) return st;
    if (algo == GCM_ALGO_BLOCKED) return modify_blocked(L, n, ldl, V, k, sigma, key, ws, stream);
    return modify_sweep(L, n, ldl, V, k, sigma, key, ws->panels, stream);
}

static gcm_status_t modify_impl(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                                gcm_info_t *d_info, gcm_algo_t algo, cudaStream_t stream) {
    gcm_status_t st = validate(L, n, ldl, V, k, sigma);
    if (st != GCM_OK) return st;
    clear_stale_error();
    if (n == 0 || k == 0) {
        if (d_info) return check_cuda(cudaMemsetAsync(d_info, 0, sizeof(gcm_info_t), stream));
        return GCM_OK;
    }
    algo = pick_algo(n, k, algo);
    if (algo == GCM_ALGO_PANEL) return modify_panel(L, n, ldl, V, k, sigma, d_info, stream);
    Workspace *ws = nullptr;
    st = get_workspace(stream, single_workspace_bytes(n, k, algo), 1, &ws);
    if (st != GCM_OK) return st;
    st = run_single(L, n, ldl, V, k, sigma, algo, ws->key, ws, stream);
    if (st != GCM_OK) return st;
    return finalize_info(ws->key, d_info, 1, stream);
}

}  // namespace gcm

using namespace gcm;

extern "C" {

gcm_status_t gcm_modify(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma, gcm_stream_t stream) {
    return modify_impl(L, n, ldl, V, k, sigma, nullptr, GCM_ALGO_AUTO, (cudaStream_t)stream);
}

gcm_status_t gcm_modify_info(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma, gcm_info_t *d_info,
                             gcm_stream_t stream) {
    return modify_impl(L, n, ldl, V, k, sigma, d_info, GCM_ALGO_AUTO, (cudaStream_t)stream);
}

gcm_status_t gcm_modify_ex(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma, gcm_info_t *d_info,
                           gcm_algo_t algo, gcm_stream_t stream) {
    if (algo != GCM_ALGO_AUTO && algo != GCM_ALGO_SWEEP && algo != GCM_ALGO_BLOCKED && algo != GCM_ALGO_PANEL)
        return GCM_EINVAL;
    return modify_impl(L, n, ldl, V, k, sigma, d_info, algo, (cudaStream_t)stream);
}

// Single precision (PAPER.md 111: the paper's experiments ran fp32 and fp64): the panel-order
// sweep (GCM_ALGO_SWEEP, the paper's own kernel structure) instantiated for float.
gcm_status_t gcm_modify_f32(float *L, int64_t n, int64_t ldl, float *V, int64_t k, int sigma, gcm_info_t *d_info,
                            gcm_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (n < 0 || k < 0 || ldl < std::max<int64_t>(1, n) || (sigma != 1 && sigma != -1)) return GCM_EINVAL;
    if (n > 0 && k > 0 && (L == nullptr || V == nullptr)) return GCM_EINVAL;
    if (n >= (1ll << 40) || k >= (1ll << 22)) return GCM_EINVAL;
    clear_stale_error();
    if (n == 0 || k == 0) return d_info ? check_cuda(cudaMemsetAsync(d_info, 0, sizeof(gcm_info_t), stream)) : GCM_OK;
    const int64_t nblk = (n + kD - 1) / kD;
    Workspace *ws = nullptr;
    gcm_status_t st = get_workspace(
        stream, (size_t)nblk * panel_doubles((int)std::min<int64_t>(k, kKMax)) * sizeof(float), 1, &ws);
    if (st != GCM_OK) return st;
    st = check_cuda(cudaMemsetAsync(ws->key, 0xff, sizeof(unsigned long long), stream));
    if (st == GCM_OK)
        st = modify_sweep_f32(L, n, ldl, V, k, sigma, ws->key, reinterpret_cast<float *>(ws->panels), stream);
    if (st != GCM_OK) return st;
    return finalize_info(ws->key, d_info, 1, stream);
}

static constexpr int64_t kHostCB = 256;

int64_t gcm_modify_host_bytes(int64_t n, int64_t k) {
    if (n < 0 || k < 0) return -1;
    int64_t b = n * k;
    for (int64_t j0 = 0; j0 < n; j0 += kHostCB) {
        const int64_t j1 = std::min<int64_t>(n, j0 + kHostCB);
        b += j1 * (j1 - j0);
    }
    return b * (int64_t)sizeof(double);
}

gcm_status_t gcm_modify_host(double *L_host, int64_t n, int64_t ldl, double *V_host, int64_t k, int sigma,
                             gcm_info_t *h_info) {
    gcm_status_t st = validate(L_host, n, ldl, V_host, k, sigma);
    if (st != GCM_OK) return st;
    if (n == 0 || k == 0) {
        if (h_info) std::memset(h_info, 0, sizeof(*h_info));
        return GCM_OK;
    }
    clear_stale_error();
    std::lock_guard<std::mutex> lock(g_host_mutex);
    int dev = 0;
    st = check_cuda(cudaGetDevice(&dev));
    if (st != GCM_OK) return st;
    HostStage &slot = g_host[dev];
    if (!slot.stream) {
        st = check_cuda(cudaStreamCreateWithFlags(&slot.stream, cudaStreamNonBlocking));
        if (st != GCM_OK) return st;
    }
    const size_t lbytes = (size_t)n * ldl * sizeof(double), vbytes = (size_t)n * k * sizeof(double);
    const size_t need = lbytes + vbytes + 256 + sizeof(gcm_info_t);
    if (slot.cap < need) {
        // the previous call synchronised its stream: the old buffer is idle; drop it first
        // (its memory may be needed), and leave the slot empty if the new allocation fails
        if (slot.buf) cudaFree(slot.buf);
        slot.buf = nullptr;
        slot.cap = 0;
        void *p = nullptr;
        st = check_cuda(cudaMalloc(&p, need));
        if (st != GCM_OK) {
            clear_stale_error();
            return st;
        }
        slot.buf = p;
        slot.cap = need;
    }
    cudaStream_t s = slot.stream;
    char *base = static_cast<char *>(slot.buf);
    double *dL = reinterpret_cast<double *>(base);
    double *dV = reinterpret_cast<double *>(base + lbytes);
    gcm_info_t *dinfo = reinterpret_cast<gcm_info_t *>(base + ((lbytes + vbytes + 255) / 256) * 256);
    // Only the upper triangle is referenced (gcm.h): move it as column blocks of
    // kHostCB columns, block [j0, j1) carrying rows 0..j1-1 (one 2-D copy each).
    auto copy_tri = [&](double *dst, const double *src, cudaMemcpyKind kind) {
        gcm_status_t r = GCM_OK;
        for (int64_t j0 = 0; j0 < n && r == GCM_OK; j0 += kHostCB) {
            const int64_t j1 = std::min<int64_t>(n, j0 + kHostCB);
            r = check_cuda(cudaMemcpy2DAsync(dst + j0 * ldl, ldl * sizeof(double), src + j0 * ldl,
                                             ldl * sizeof(double), j1 * sizeof(double), j1 - j0, kind, s));
        }
        return r;
    };
    st = copy_tri(dL, L_host, cudaMemcpyHostToDevice);
    if (st == GCM_OK) st = check_cuda(cudaMemcpyAsync(dV, V_host, vbytes, cudaMemcpyHostToDevice, s));
    if (st == GCM_OK) st = modify_impl(dL, n, ldl, dV, k, sigma, dinfo, GCM_ALGO_AUTO, s);
    if (st == GCM_OK) st = copy_tri(L_host, dL, cudaMemcpyDeviceToHost);
    if (st == GCM_OK) st = check_cuda(cudaMemcpyAsync(V_host, dV, vbytes, cudaMemcpyDeviceToHost, s));
    if (st == GCM_OK && h_info)
        st = check_cuda(cudaMemcpyAsync(h_info, dinfo, sizeof(gcm_info_t), cudaMemcpyDeviceToHost, s));
    const gcm_status_t sync = check_cuda(cudaStreamSynchronize(s));
    return st != GCM_OK ? st : sync;
}

gcm_status_t gcm_modify_batched(double *L, int64_t n, int64_t ldl, int64_t strideL, double *V, int64_t strideV,
                                int64_t k, int sigma, int64_t batch, gcm_info_t *d_info, gcm_stream_t stream) {
    if (batch < 0) return GCM_EINVAL;
    gcm_status_t st = validate(L, n, ldl, V, k, sigma);
    if (st != GCM_OK) return st;
    if (batch > 1 && (strideL < ldl * n || strideV < n * k)) return GCM_EINVAL;
    if (batch == 0) return GCM_OK;
    clear_stale_error();
    if (n == 0 || k == 0) {
        if (d_info) return check_cuda(cudaMemsetAsync(d_info, 0, sizeof(gcm_info_t) * batch, (cudaStream_t)stream));
        return GCM_OK;
    }
    return modify_batched(L, n, ldl, strideL, V, strideV, k, sigma, batch, d_info, (cudaStream_t)stream);
}

gcm_status_t gcm_profile_enable(int on) {
    g_profile_on = on != 0;
    return GCM_OK;
}

int gcm_profile_read(char *names, int64_t *counts, double *ms, int max_entries) {
    std::lock_guard<std::mutex> lock(g_prof_mutex);
    std::vector<std::string> order;
    std::map<std::string, std::pair<int64_t, double>> agg;
    int err = 0;
    for (auto &r : g_prof_done) {
        float t = 0.f;
        if (cudaEventSynchronize(r.e) != cudaSuccess || cudaEventElapsedTime(&t, r.b, r.e) != cudaSuccess) err = 1;
        if (!agg.count(r.name)) order.push_back(r.name);
        agg[r.name].first += 1;
        agg[r.name].second += t;
        g_event_pool.push_back(r.b);
        g_event_pool.push_back(r.e);
    }
    g_prof_done.clear();
    if (err) return -1;
    int n = 0;
    for (auto &nm : order) {
        if (n >= max_entries) break;
        std::strncpy(names + 32 * n, nm.c_str(), 31);
        names[32 * n + 31] = 0;
        counts[n] = agg[nm].first;
        ms[n] = agg[nm].second;
        ++n;
    }
    return n;
}

int64_t gcm_profile_launches(void) { return (int64_t)g_launches.exchange(0); }

const char *gcm_status_string(gcm_status_t s) {
    switch (s) {
        case GCM_OK: return "GCM_OK";
        case GCM_EINVAL: return "GCM_EINVAL: invalid argument";
        case GCM_ECUDA: return "GCM_ECUDA: CUDA launch or runtime error";
        case GCM_ENOMEM: return "GCM_ENOMEM: device allocation failed";
        case GCM_ENCCL: return "GCM_ENCCL: NCCL error";
        case GCM_ENOTSUP: return "GCM_ENOTSUP: not supported in this build";
    }
    return "unknown gcm status";
}

gcm_status_t gcm_release_workspace(void) {
    int cur = 0;
    cudaGetDevice(&cur);
    {
        std::lock_guard<std::mutex> lock(g_ws_mutex);
        for (auto &kv : g_ws) {
            if (kv.second.key) {
                cudaSetDevice(kv.first.first);
                cudaStreamSynchronize(kv.first.second);
                cudaFree(kv.second.key);
            }
        }
        g_ws.clear();
    }
    {
        std::lock_guard<std::mutex> lock(g_host_mutex);
        for (auto &kv : g_host) {  // the staging stream is kept; its buffer (n*ldl doubles) is not
            if (kv.second.buf) {
                cudaSetDevice(kv.first);
                cudaStreamSynchronize(kv.second.stream);
                cudaFree(kv.second.buf);
                kv.second.buf = nullptr;
                kv.second.cap = 0;
            }
        }
    }
    cudaSetDevice(cur);
    clear_stale_error();
    return GCM_OK;
}

const char *gcm_version(void) { return "gcm 0.1 sm_100a"; }

}  // extern "C"
