// api.cu -- the C ABI of libcleora (include/cleora.h): handle life cycle, argument checks,
// device memory ownership, stream ordering, timing, and the multi-GPU exchange.
//
// Every step of the hot path runs in this library's kernels (build.cu, init.cu,
// spmm_norm.cu); the Python binding only marshals arguments.  There is no CPU fallback.
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/cleora.h"
#include "common.cuh"

namespace cleora {

// NVTX range around every C-ABI call (header-only NVTX 3: free unless a profiler is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

static std::atomic<int64_t> g_launches{0};
void count_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void trace(const char* what, cudaStream_t s, bool sync) {
    static const bool on = getenv("CLEORA_TRACE") != nullptr;
    if (!on) return;
    static thread_local std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    if (sync) cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[cleora trace] %-28s %8.3f ms%s\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(), sync ? " (synced)" : "");
    last = now;
}

// ---------------------------------------------------------------- small readbacks
namespace {
struct SmallSegs {
    const uint8_t* src[kMaxSmallReads];
    int off[kMaxSmallReads], len[kMaxSmallReads];
    int n;
};
__global__ void k_read_small(const SmallSegs sg, uint8_t* __restrict__ dst) {
    for (int q = 0; q < sg.n; q++)
        for (int i = threadIdx.x; i < sg.len[q]; i += blockDim.x) dst[sg.off[q] + i] = sg.src[q][i];
    __threadfence_system();
}
struct Mapped {
    std::mutex mu;
    uint8_t* h = nullptr;
    uint8_t* d = nullptr;
};
Mapped g_mapped[kMaxDevices];
}  // namespace

Status read_small(void* h_dst, const void* d_src, size_t bytes, cudaStream_t s) {
    const SmallRead r{h_dst, d_src, bytes};
    return read_small_n(&r, 1, s);
}

// Several small device ranges in one kernel and one stream synchronisation (each host round trip
// leaves the GPU idle until the next launch: the build merges its readbacks with this).
Status read_small_n(const SmallRead* r, int n, cudaStream_t s) {
    if (n < 1 || n > kMaxSmallReads) return Status::make(4, "read_small: 1..kMaxSmallReads ranges");
    SmallSegs sg{};
    size_t bytes = 0;
    for (int q = 0; q < n; q++) {
        sg.src[q] = reinterpret_cast<const uint8_t*>(r[q].d_src);
        sg.off[q] = (int)bytes;
        sg.len[q] = (int)r[q].bytes;
        bytes += (r[q].bytes + 7) / 8 * 8;
        if (bytes > 4096) return Status::make(4, "read_small: more than 4096 bytes");
    }
    sg.n = n;
    if (bytes == 0) return Status::ok();
    int dev = 0;
    CL_CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= kMaxDevices) return Status::make(4, "read_small: device ordinal beyond kMaxDevices");
    Mapped& m = g_mapped[dev];
    std::lock_guard<std::mutex> lk(m.mu);
    if (!m.h) {
        CL_CUDA_TRY(cudaHostAlloc((void**)&m.h, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
        CL_CUDA_TRY(cudaHostGetDevicePointer((void**)&m.d, m.h, 0));
    }
    k_read_small<<<1, 256, 0, s>>>(sg, m.d);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    CL_CUDA_TRY(cudaStreamSynchronize(s));
    for (int q = 0; q < n; q++) memcpy(r[q].h_dst, m.h + sg.off[q], r[q].bytes);
    return Status::ok();
}

// ---------------------------------------------------------------- device memory
// Small buffers come from the device's default stream-ordered pool.  Large ones (>= 1 MiB: the T
// replicas, CSR arrays, sort buffers) come from a process-wide cache of cudaMalloc segments, handed
// out whole and reused by exact (2 MiB-rounded) size: a graph built, embedded and destroyed over and
// over (the bench step; a service embedding many graphs of one shape) reuses the same physical
// blocks.  Measured on B200 before any cache: pool growth in the middle of a run stalled single steps
// by 40-140 ms (scripts/step_jitter.py).
// Stream order: a freed segment carries the events recorded on the streams that freed it; whoever
// reuses it waits on them first.  Segments go back to the driver on cleora_release_cached_memory(),
// beyond the cap (CLEORA_CACHE_MAX_FRAC of HBM, 0.8), or when a cudaMalloc fails (then largest
// first, and the allocation is retried; cleora_oom_fallbacks counts these).
static std::mutex g_pool_mu;
static bool g_pool_cfg[64];

namespace {
constexpr size_t kCacheMin = (size_t)1 << 20;
constexpr size_t kCacheGrain = (size_t)2 << 20;
struct Segment {                    // a cudaMalloc block, handed out or cached
    size_t bytes;
    int dev;
    bool free;
    std::vector<cudaEvent_t> ready; // cached: the next user waits on these
};
std::mutex g_cache_mu;
std::map<char*, Segment> g_segs;    // every segment, by address
size_t g_free_bytes = 0;            // bytes in cached (free) segments
std::vector<cudaEvent_t> g_ev_pool;
std::atomic<int64_t> g_oom_fallbacks{0};

size_t round_block(size_t b) { return (b + kCacheGrain - 1) / kCacheGrain * kCacheGrain; }

cudaEvent_t ev_get() {              // caller holds g_cache_mu
    if (!g_ev_pool.empty()) {
        cudaEvent_t e = g_ev_pool.back();
        g_ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return e;
}

// Take cached segments out of the cache: all of `dev` (-1: every device), or only the largest one.
// The caller frees them with cudaFree after waiting for their events.
struct Dropped {
    char* p;
    int dev;
    std::vector<cudaEvent_t> ready;
};
std::vector<Dropped> take_free(int dev, bool largest_only) {
    std::vector<Dropped> out;
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto best = g_segs.end();
    for (auto it = g_segs.begin(); it != g_segs.end();) {
        Segment& r = it->second;
        if (r.free && (dev < 0 || r.dev == dev)) {
            if (largest_only) {
                if (best == g_segs.end() || r.bytes > best->second.bytes) best = it;
            } else {
                out.push_back({it->first, r.dev, std::move(r.ready)});
                g_free_bytes -= r.bytes;
                it = g_segs.erase(it);
                continue;
            }
        }
        ++it;
    }
    if (largest_only && best != g_segs.end()) {
        out.push_back({best->first, best->second.dev, std::move(best->second.ready)});
        g_free_bytes -= best->second.bytes;
        g_segs.erase(best);
    }
    return out;
}

void free_dropped(std::vector<Dropped>& v) {
    int cur = -1;
    cudaGetDevice(&cur);
    for (auto& d : v) {
        cudaSetDevice(d.dev);
        for (auto e : d.ready) {
            cudaEventSynchronize(e);
            cudaEventDestroy(e);
        }
        cudaFree(d.p);
    }
    if (cur >= 0) cudaSetDevice(cur);
    v.clear();
}

void release_cached(int dev /* -1: all */) {
    auto v = take_free(dev, false);
    free_dropped(v);
}

bool release_largest(int dev) {
    auto v = take_free(dev, true);
    if (v.empty()) return false;
    free_dropped(v);
    return true;
}

// A cached segment of `dev` of exactly `rb` bytes (2 MiB-rounded); the stream waits for its events.
// Caller holds g_cache_mu.  Exact sizes, no splitting: two alternatives were measured on c5's e2e
// pipeline, where one step's working set nearly fills the 180 GB, and dropped -- splitting segments
// (best fit, merging freed neighbours) let pieces of long-lived buffers pin large segments, and lending
// transient buffers segments up to twice their size wasted the rest; either way a 22.7 GB sort buffer
// later found no room and nothing to give back, a hard out-of-memory error where exact whole segments
// only cost cudaFree/cudaMalloc round trips (profiles/r02_bench_c5_oom.txt).
void* take_cached(int dev, size_t rb, cudaStream_t s) {
    for (auto& kv : g_segs) {
        Segment& r = kv.second;
        if (!r.free || r.dev != dev || r.bytes != rb) continue;
        for (auto e : r.ready) {
            cudaStreamWaitEvent(s, e, 0);
            g_ev_pool.push_back(e);
        }
        r.ready.clear();
        r.free = false;
        g_free_bytes -= r.bytes;
        return kv.first;
    }
    return nullptr;
}
}  // namespace

Status dalloc(void** p, size_t bytes, cudaStream_t s, const char* what, int flags) {
    // kAllocTransient is a hint only (both kinds are served alike); kAllocBase: a whole cudaMalloc
    // segment whatever the size (T buffers: CUDA IPC cannot export pool memory)
    const bool block = flags & kAllocBase;
    *p = nullptr;
    int dev = 0;
    CL_CUDA_TRY(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (dev < 64 && !g_pool_cfg[dev]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            g_pool_cfg[dev] = true;
        }
    }
    if (bytes == 0) bytes = 16;
    static const bool no_cache = getenv("CLEORA_NO_CACHE") != nullptr;
    const bool big = block || (bytes >= kCacheMin && !no_cache);
    const size_t rb = round_block(bytes);
    if (big) {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        if (void* q = take_cached(dev, rb, s)) {
            *p = q;
            return Status::ok();
        }
    }
    for (;;) {
        cudaError_t e;
        if (big) {
            // cached segments are plain device allocations (not pool memory): they outlive streams
            e = cudaMalloc(p, rb);
        } else {
            e = cudaMallocAsync(p, bytes, s);
        }
        if (e == cudaSuccess) break;
        cudaGetLastError();
        *p = nullptr;
        // out of memory: give cached segments back to the driver, largest first, until it fits
        if (e == cudaErrorMemoryAllocation && !(flags & kAllocNoEvict) && release_largest(dev)) {
            g_oom_fallbacks.fetch_add(1);
            static const bool tr = getenv("CLEORA_TRACE") != nullptr;
            if (tr) fprintf(stderr, "[cleora trace] out of memory for %s (%zu bytes): released a cached segment\n", what, bytes);
            continue;
        }
        char buf[256];
        snprintf(buf, sizeof buf, "cudaMalloc(%zu bytes) for %s: %s", bytes, what, cudaGetErrorString(e));
        return Status::make(4, buf);
    }
    if (big) {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        g_segs.emplace((char*)*p, Segment{rb, dev, false, {}});
    }
    return Status::ok();
}

static size_t cache_cap_bytes(int dev) {
    static size_t cap[64];
    if (dev < 0 || dev >= 64) return 0;
    if (!cap[dev]) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        const char* e = getenv("CLEORA_CACHE_MAX_FRAC");
        const double f = e ? atof(e) : 0.8;
        cap[dev] = (size_t)(f * (double)tot) + 1;
    }
    return cap[dev];
}

void dfree(void* p, cudaStream_t s) {
    if (!p) return;
    bool cached = false;
    int dev = -1;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto it = g_segs.find((char*)p);
        if (it != g_segs.end() && !it->second.free) {
            Segment& r = it->second;
            dev = r.dev;
            if (cudaEvent_t e = ev_get()) {
                cudaEventRecord(e, s);        // the segment is free once s reaches this point
                r.ready.push_back(e);
            }
            r.free = true;
            g_free_bytes += r.bytes;
            cached = true;
        }
    }
    if (!cached) {
        cudaFreeAsync(p, s);
        return;
    }
    // bound what stays cached: segments beyond the cap go back to the driver, largest first
    while (g_free_bytes > cache_cap_bytes(dev) && release_largest(dev)) {
    }
}

// ---------------------------------------------------------------- NCCL, resolved at run time
// The library does not link NCCL: when world > 1 it binds to the libnccl.so.2 already loaded
// into the process (torch's) or loads it, so the process never holds two NCCL copies.
struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { n.why = std::string("dlopen libnccl.so.2: ") + dlerror(); return; }
#define BIND(f, name)                                                   \
    n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, name));              \
    if (!n.f) { n.why = std::string("dlsym ") + name; return; }
        BIND(GetUniqueId, "ncclGetUniqueId");
        BIND(CommInitRank, "ncclCommInitRank");
        BIND(Broadcast, "ncclBroadcast");
        BIND(AllGather, "ncclAllGather");
        BIND(AllReduce, "ncclAllReduce");
        BIND(GroupStart, "ncclGroupStart");
        BIND(GroupEnd, "ncclGroupEnd");
        BIND(CommDestroy, "ncclCommDestroy");
        BIND(GetErrorString, "ncclGetErrorString");
#undef BIND
        n.ok = true;
    });
    return n;
}

#define CL_NCCL_TRY(expr)                                                                         \
    do {                                                                                          \
        ncclResult_t _r = (expr);                                                                 \
        if (_r != ncclSuccess)                                                                    \
            return Status::make(4, std::string(#expr) + ": " + nccl().GetErrorString(_r));       \
    } while (0)

static int heavy_thresh_default(int dflt) {
    const char* e = getenv("CLEORA_HEAVY_THRESH");
    int v = e ? atoi(e) : dflt;
    if (v < 8) v = 8;
    if (v > 4096) v = 4096;
    return v;
}

}  // namespace cleora

using namespace cleora;

struct cleora_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int32_t n = 0;
    // nnz: stored entries of the whole M (all shards); zero_rows, max_degree: of the whole M, -1 until
    // read back (one GPU: lazily by cleora_info; row-sharded: combined over the ranks at the build)
    int64_t nnz = 0, n_edges_in = 0, zero_rows = -1, max_degree = -1;
    int directed = 0;
    // CSR of M: one GPU -> csr[0] = all rows; world > 1 -> csr[0] = this rank's rows only (row-sharded
    // build: row_ptr has N + 1 entries, shard-local offsets, 0 before the shard and nnz after it);
    // loopback -> csr[p] = emulated rank p's shard
    std::vector<Csr> csr;
    int32_t* indeg = nullptr;       // row-sharded builds: the whole graph's in-degree (shard_plan)
    // deferred exchange: per emulated rank (loopback) or for this rank, mask[r] bit q = peer q gathers r
    std::vector<uint8_t*> pmask;
    bool sharded = false;
    // environment switches, read by cleora_init
    int env_cold_first = -1, env_csr_prefetch = 1;
    bool env_write_zero = false, env_no_hot = false, env_defer = true;
    int gmode = 0;                  // gather engine for the current dp (gather_mode)
    bool halves = false;            // dp = 1024 steps run as two half-row passes (cleora_init decides)
    // lazy normalisation between the half-row steps of one iterate call: fp64 first-half sums of squares
    // [0..N), then the scaled weights of the largest shard (fp32); the row scales live behind each T
    // buffer's rows (spmm_tma.cu, reading R21)
    double* lazy_buf = nullptr;
    bool env_lazy = true, env_t0_all = false;
    bool env_drop_ungathered = true;    // lazy steps skip the stores of never-gathered rows (CLEORA_KEEP_UNGATHERED=1: not)
    // T_0 written only for the rows a step can gather (in-degree > 0, g->indeg): the other rows are
    // never read before the first step overwrites them, unless T_0 itself is read -- complete_t0 fills
    // them in then (fetch, trim, merge, reconstruct, set_rows)
    mutable bool t0_partial = false;
    uint64_t t0_seed = 0;
    int heavy_thresh = 64;
    Schedule sched;
    int32_t d = 0, dp = 0;
    float* T[2] = {nullptr, nullptr};
    float* partials = nullptr;
    int32_t tag_dp = 0;             // row stride the hot-row tags in col (bit 31) were chosen for
    Csr& own() { return csr[csr.size() > 1 ? rank : 0]; }
    const Csr& own() const { return csr[csr.size() > 1 ? rank : 0]; }
    Csr& of(int p) { return csr[csr.size() > 1 ? p : 0]; }
    // cleora_fetch_async: D2H on a copy stream, concurrent with later work on `stream`
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_copied = nullptr;
    mutable bool copy_pending = false;
    // cleora_fetch_nonzero: this shard's rows with entries (or every row: nz_all), selected once per
    // handle, and the device staging buffer of the packed copy (both freed by free_T after the copy)
    int32_t* nz_ids = nullptr;
    int64_t nz_n = -1;
    bool nz_all = false;
    float* stage = nullptr;
    size_t stage_bytes = 0;
    bool rows_set = false;          // cleora_set_rows since the last step: a row without entries may be != 0
    bool trimmed = false;           // cleora_trim: only T[cur] (and occ, d_scal) left
    int32_t* occ = nullptr;         // chunked builds: endpoint occurrences per node (reading R14)
    int32_t n_graphs = 0;           // batched handles (cleora_build_batch): graphs in the batch
    int64_t* d_base = nullptr;      //   [n_graphs + 1] first row of every graph (device)
    int32_t n_chunks = 0, chunk = 0;
    uint64_t chunk_seed = 0;
    int64_t n_hot = 0;
    int64_t n_ref = -1;             // rows with in-degree > 0 (known once hot_tag ran)
    int cur = 0;
    int64_t iters = 0;
    int rank = 0, world = 1;
    std::vector<int64_t> cuts;
    int64_t r0 = 0, r1 = 0;
    ncclComm_t comm = nullptr;
    // host-side collectives (world > 1 without NCCL): the caller's all-gather (cleora_opts)
    cleora_allgather_fn host_ag = nullptr;
    void* host_ctx = nullptr;
    // exchange of the row shards after every step (world > 1), see exchange_mode below
    int xmode = 0;
    bool zclean[2] = {false, false};   // rows without entries are already 0 in T[b]
    // X_PEER: the other ranks' T[0], T[1], opened through CUDA IPC (rank order, self skipped)
    float* peer_T[2][kMaxPeers] = {};
    int* d_flag = nullptr;             // 1 int: operand of the per-step NCCL barrier
    // X_LOOPBACK: all `world` replicas live in this process; rep[p] = rank p's T pair
    // (rep[rank] aliases T), sched_p[p] = rank p's schedule
    std::vector<std::array<float*, 2>> rep;
    std::vector<Schedule> sched_p;
    int64_t max_items = 0;          // partial-vector slots the schedule(s) may use (upper bound)
    int sched_thresh = -1;          // heavy_thresh the current schedule(s) were built with
    int chunk_rows = kChunkRows;    // light-chunk row cap for the current gather engine
    int sched_rows = -1;            // chunk_rows the current schedule(s) were built with
    size_t partials_floats = 0;     // capacity of `partials`
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_spmm, ev_x;
    std::vector<cudaEvent_t> ev_pool;
    int64_t n_spmm = 0, n_x = 0;
    double ms_spmm = 0, ms_min = 1e300, ms_max = 0, ms_x = 0;
    int64_t bytes = 0;
};

namespace {

int fail(const Status& s) {
    set_error(s.msg);
    return s.code;
}
int usage(const char* m) {
    set_error(m);
    return CLEORA_EUSAGE;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int now = -1;
        if (prev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != prev) cudaSetDevice(prev);
    }
};

cudaEvent_t get_event(cleora_graph* g) {
    if (!g->ev_pool.empty()) {
        cudaEvent_t e = g->ev_pool.back();
        g->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

Status collect_timing(cleora_graph* g) {
    if (g->ev_spmm.empty() && g->ev_x.empty()) return Status::ok();
    CL_CUDA_TRY(cudaStreamSynchronize(g->stream));
    for (auto& p : g->ev_spmm) {
        float ms = 0;
        CL_CUDA_TRY(cudaEventElapsedTime(&ms, p.first, p.second));
        g->n_spmm++;
        g->ms_spmm += ms;
        g->ms_min = std::min(g->ms_min, (double)ms);
        g->ms_max = std::max(g->ms_max, (double)ms);
        g->ev_pool.push_back(p.first);
        g->ev_pool.push_back(p.second);
    }
    for (auto& p : g->ev_x) {
        float ms = 0;
        CL_CUDA_TRY(cudaEventElapsedTime(&ms, p.first, p.second));
        g->n_x++;
        g->ms_x += ms;
        g->ev_pool.push_back(p.first);
        g->ev_pool.push_back(p.second);
    }
    g->ev_spmm.clear();
    g->ev_x.clear();
    return Status::ok();
}

// Exchange modes (world > 1).  X_PEER is the product path: the SpMM epilogue stores every
// finished row into all replicas over NVLink (peer pointers from CUDA IPC), then one 4-byte NCCL
// all-reduce per step orders the steps across ranks.  X_NCCL: the SpMM writes only the local
// replica and an all-gather-v (grouped in-place ncclBroadcast) follows -- the fallback when the
// GPUs cannot map each other's memory, or on request (CLEORA_F_EXCHANGE_NCCL).  X_LOOPBACK:
// `world` ranks emulated in one process on one GPU (tests): the same fused kernel writes its
// rows into the other ranks' replicas, which are local buffers; ranks run one after another.
enum { X_NONE = 0, X_NCCL = 1, X_PEER = 2, X_LOOPBACK = 3 };

// CUDA IPC mappings of peer T buffers, cached process-wide by (device, handle bytes).  A peer's T
// blocks come from its block cache, so the next handle of the same shape usually exports the very same
// blocks: cleora_init then finds them mapped already instead of opening (and later closing) them
// again -- round 1 opened and closed every peer buffer in every cleora_init, i.e. in every timed
// multi-GPU bench step.  A mapping stays valid while the exporting process keeps the block (the
// block cache only hands it back to the driver on cleora_release_cached_memory or out of memory);
// cleora_release_cached_memory also closes every mapping here.  Bounded: beyond kIpcCacheMax
// entries the oldest not-in-use mapping is closed.
namespace {
struct IpcEntry {
    int dev;
    cudaIpcMemHandle_t h;
    void* p;
    int users;
    uint64_t stamp;
};
std::mutex g_ipc_mu;
std::vector<IpcEntry> g_ipc;
uint64_t g_ipc_clock = 0;
constexpr size_t kIpcCacheMax = 64;
std::atomic<int64_t> g_ipc_opens{0};

Status ipc_open(int dev, const cudaIpcMemHandle_t& h, void** out) {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    for (auto& e : g_ipc)
        if (e.dev == dev && !memcmp(&e.h, &h, sizeof h)) {
            e.users++;
            e.stamp = ++g_ipc_clock;
            *out = e.p;
            return Status::ok();
        }
    void* p = nullptr;
    cudaError_t r = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (r != cudaSuccess) {
        cudaGetLastError();
        return Status::make(4, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(r));
    }
    g_ipc_opens.fetch_add(1);
    if (g_ipc.size() >= kIpcCacheMax) {          // close the oldest idle mapping
        size_t at = g_ipc.size();
        for (size_t i = 0; i < g_ipc.size(); i++)
            if (g_ipc[i].users == 0 && (at == g_ipc.size() || g_ipc[i].stamp < g_ipc[at].stamp)) at = i;
        if (at < g_ipc.size()) {
            cudaIpcCloseMemHandle(g_ipc[at].p);
            g_ipc.erase(g_ipc.begin() + at);
        }
    }
    g_ipc.push_back({dev, h, p, 1, ++g_ipc_clock});
    *out = p;
    return Status::ok();
}

void ipc_release(void* p) {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    for (auto& e : g_ipc)
        if (e.p == p && e.users > 0) {
            e.users--;
            return;
        }
}

void ipc_close_all() {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    for (size_t i = 0; i < g_ipc.size();) {
        if (g_ipc[i].users == 0) {
            cudaIpcCloseMemHandle(g_ipc[i].p);
            g_ipc.erase(g_ipc.begin() + i);
        } else {
            i++;
        }
    }
}
}  // namespace

void close_peers(cleora_graph* g) {
    for (int b = 0; b < 2; b++)
        for (int i = 0; i < kMaxPeers; i++)
            if (g->peer_T[b][i]) {
                ipc_release(g->peer_T[b][i]);      // the mapping stays cached (see ipc_open)
                g->peer_T[b][i] = nullptr;
            }
}

void free_csr(cleora_graph* g) {
    for (auto& c : g->csr) {
        dfree(c.row_ptr, g->stream);
        dfree(c.col, g->stream);
        dfree(c.val, g->stream);
        dfree(c.deg, g->stream);
        dfree(c.d_scal, g->stream);
        c = Csr();
    }
}

void free_schedules(cleora_graph* g) {
    auto drop = [g](Schedule& sc) {
        dfree(sc.items, g->stream);
        dfree(sc.counters, g->stream);
        dfree(sc.work, g->stream);
        dfree(sc.light_start, g->stream);
        dfree(sc.counts, g->stream);
        sc = Schedule();
    };
    if (g->sched_p.empty()) {
        drop(g->sched);
    } else {
        for (auto& sc : g->sched_p) drop(sc);   // g->sched aliases sched_p[rank]
        g->sched = Schedule();
    }
    g->max_items = 0;
    g->sched_thresh = -1;
    g->sched_rows = -1;
}

// The schedule (heavy-row CTA items, light chunks) for this handle's rows -- for every emulated
// rank in loopback -- with the current heavy_thresh.
Status make_schedules(cleora_graph* g) {
    free_schedules(g);
    if (!g->sched_p.empty()) {
        for (int p = 0; p < g->world; p++) {
            CL_TRY(build_schedule(g->of(p).row_ptr, g->n, g->cuts[p], g->cuts[p + 1], g->of(p).nnz,
                                  g->of(p).max_degree, g->heavy_thresh, g->chunk_rows, g->stream, &g->sched_p[p]));
            g->max_items = std::max(g->max_items, g->sched_p[p].n_slots_max);
        }
        g->sched = g->sched_p[g->rank];
    } else {
        CL_TRY(build_schedule(g->own().row_ptr, g->n, g->r0, g->r1, g->own().nnz, g->own().max_degree, g->heavy_thresh,
                              g->chunk_rows, g->stream, &g->sched));
        g->max_items = g->sched.n_slots_max;
    }
    g->sched_thresh = g->heavy_thresh;
    g->sched_rows = g->chunk_rows;
    return Status::ok();
}

// An asynchronous fetch may still be reading T: stream-order the next use of T after it.
void order_after_side(const cleora_graph* g) {
    if (g->copy_pending) {
        cudaStreamWaitEvent(g->stream, g->ev_copied, 0);
        g->copy_pending = false;
    }
}

// T_0 is read before any step (fetch, trim, merge, reconstruct, set_rows): write the rows init left
// out (in-degree 0), in every local replica
Status complete_t0(const cleora_graph* gc) {
    cleora_graph* g = const_cast<cleora_graph*>(gc);
    if (!g->t0_partial) return Status::ok();
    if (g->iters == 0 && g->cur == 0 && g->T[0] && g->indeg) {
        CL_TRY(launch_hash_init(g->T[0], g->n, g->d, g->dp, g->t0_seed, g->stream, g->d_base, g->n_graphs, g->indeg, 2));
        if (g->xmode == X_LOOPBACK)
            for (int p = 0; p < g->world; p++)
                if (p != g->rank && g->rep[p][0])
                    CL_TRY(launch_hash_init(g->rep[p][0], g->n, g->d, g->dp, g->t0_seed, g->stream, g->d_base,
                                            g->n_graphs, g->indeg, 2));
    }
    g->t0_partial = false;
    return Status::ok();
}

void free_T(cleora_graph* g) {
    if (g->copy_stream) cudaStreamSynchronize(g->copy_stream);    // the blocks go back to the cache
    g->copy_pending = false;
    dfree(g->nz_ids, g->stream);
    g->nz_ids = nullptr;
    g->nz_n = -1;
    dfree(g->stage, g->stream);
    g->stage = nullptr;
    g->stage_bytes = 0;
    close_peers(g);
    for (size_t p = 0; p < g->rep.size(); p++)
        if ((int)p != g->rank)
            for (int i = 0; i < 2; i++) dfree(g->rep[p][i], g->stream);
    if (!g->rep.empty()) g->rep.assign(g->rep.size(), {nullptr, nullptr});
    for (int i = 0; i < 2; i++) {
        dfree(g->T[i], g->stream);
        g->T[i] = nullptr;
    }
    dfree(g->partials, g->stream);
    g->partials = nullptr;
    g->partials_floats = 0;
    dfree(g->lazy_buf, g->stream);
    g->lazy_buf = nullptr;
    g->zclean[0] = g->zclean[1] = false;
}

// Stream-ordered barrier over all ranks (a 1-int all-reduce): work enqueued after it on any rank
// runs after every rank's work enqueued before it -- including the SpMM's peer stores.
// NCCL communicators are process-wide and cached by (unique id, world, rank, device): a job builds
// many handles from one unique id (every bench step, every graph a service embeds), and NCCL serves
// one ncclCommInitRank per unique id -- a second init from the same id would wait for a bootstrap
// root that is gone -- besides costing far more than a step.  Handles share the communicator in
// stream order (every rank issues its handles' collectives in the same order); it lives until the
// process ends.
struct CommEntry {
    std::string key;
    ncclComm_t comm;
};
static std::mutex g_comm_mu;
static std::vector<CommEntry> g_comms;

Status comm_get(const uint8_t* id128, int world, int rank, int dev, ncclComm_t* out) {
    std::string key(reinterpret_cast<const char*>(id128), NCCL_UNIQUE_ID_BYTES);
    key += ":" + std::to_string(world) + ":" + std::to_string(rank) + ":" + std::to_string(dev);
    std::lock_guard<std::mutex> lk(g_comm_mu);
    for (auto& e : g_comms)
        if (e.key == key) {
            *out = e.comm;
            return Status::ok();
        }
    Nccl& nc = nccl();
    ncclUniqueId id;
    memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c = nullptr;
    CL_NCCL_TRY(nc.CommInitRank(&c, world, id, rank));
    g_comms.push_back({key, c});
    *out = c;
    return Status::ok();
}

// ---- collectives of a multi-rank handle: NCCL (g->comm) or the caller's host all-gather (g->host_ag)

// all-gather of `bytes` host bytes per rank (blocking): all[p * bytes ...] = rank p's `mine`
Status comm_allgather(cleora_graph* g, const void* mine, void* all, size_t bytes) {
    if (g->host_ag) {
        if (g->host_ag(g->host_ctx, mine, all, (int64_t)bytes) != 0)
            return Status::make(4, "host all-gather (cleora_opts.host_allgather) failed");
        return Status::ok();
    }
    Nccl& N = nccl();
    const int W = g->world;
    void* d = nullptr;
    CL_TRY(dalloc(&d, bytes * W + 16, g->stream, "all-gather buffer", kAllocTransient));
    Status st = Status::ok();
    do {
        if (cudaMemcpyAsync((char*)d + bytes * g->rank, mine, bytes, cudaMemcpyHostToDevice, g->stream) != cudaSuccess) {
            st = Status::make(4, "all-gather staging copy");
            break;
        }
        ncclResult_t r = N.AllGather((char*)d + bytes * g->rank, d, bytes, ncclChar, g->comm, g->stream);
        if (r != ncclSuccess) { st = Status::make(4, std::string("ncclAllGather: ") + N.GetErrorString(r)); break; }
        if (cudaMemcpyAsync(all, d, bytes * W, cudaMemcpyDeviceToHost, g->stream) != cudaSuccess ||
            cudaStreamSynchronize(g->stream) != cudaSuccess) {
            st = Status::make(4, "all-gather read-back");
            break;
        }
    } while (0);
    dfree(d, g->stream);
    return st;
}

// Failure agreement: every rank reports whether its part of a collective call succeeded,
// so that one rank's failure (out of memory, say) makes every rank return an error instead of
// leaving the others blocked in the next collective.  Returns the local status, or EINTERNAL naming
// the first failed rank when only another rank failed.
Status comm_agree(cleora_graph* g, const Status& local) {
    if (g->world <= 1 || g->xmode == X_LOOPBACK) return local;
    const int mine = local.good() ? 0 : (local.code ? local.code : 4);
    std::vector<int> all(g->world, 0);
    CL_TRY(comm_allgather(g, &mine, all.data(), sizeof(int)));
    if (!local.good()) return local;
    for (int p = 0; p < g->world; p++)
        if (all[p]) return Status::make(4, "rank " + std::to_string(p) + " of " + std::to_string(g->world) + " failed");
    return Status::ok();
}

// Stream-ordered barrier over all ranks: work enqueued after it on any rank runs after every rank's
// work enqueued before it (the SpMM's peer stores included).  NCCL: a 1-int all-reduce on the stream.
// Host all-gather: the stream is synchronised first, then a 1-byte all-gather.
Status rank_barrier(cleora_graph* g) {
    if (g->host_ag) {
        CL_CUDA_TRY(cudaStreamSynchronize(g->stream));
        char b = 0;
        std::vector<char> all(g->world);
        return comm_allgather(g, &b, all.data(), 1);
    }
    Nccl& N = nccl();
    CL_NCCL_TRY(N.AllReduce(g->d_flag, g->d_flag, 1, ncclInt32, ncclMax, g->comm, g->stream));
    return Status::ok();
}

// X_PEER set-up (collective, inside cleora_init): all-gather the IPC handles of every rank's
// T[0], T[1] and map the others' (ipc_open: cached across handles).  Any rank that cannot map them
// makes all ranks fall back to X_NCCL (the decision is all-gathered, so every rank takes the same
// path); with host collectives there is no fallback and the call fails on every rank.
Status open_peers(cleora_graph* g) {
    const int W = g->world;
    if (W - 1 > kMaxPeers) {
        if (g->host_ag) return Status::make(4, "cleora_init: host collectives need peer mappings (world <= 8)");
        g->xmode = X_NCCL;
        return Status::ok();
    }
    cudaIpcMemHandle_t mine[2];
    int ok = 1;
    for (int b = 0; b < 2; b++)
        if (cudaIpcGetMemHandle(&mine[b], g->T[b]) != cudaSuccess) {
            cudaGetLastError();
            ok = 0;
        }
    const size_t hb = sizeof(mine);
    std::vector<char> all(hb * W);
    CL_TRY(comm_allgather(g, mine, all.data(), hb));
    std::string why;
    int i = 0;
    for (int p = 0; p < W && ok; p++) {
        if (p == g->rank) continue;
        for (int b = 0; b < 2 && ok; b++) {
            cudaIpcMemHandle_t h;
            memcpy(&h, all.data() + hb * p + sizeof(cudaIpcMemHandle_t) * b, sizeof h);
            void* ptr = nullptr;
            Status so = ipc_open(g->device, h, &ptr);
            if (!so.good()) {
                ok = 0;
                why = so.msg;
            } else {
                g->peer_T[b][i] = (float*)ptr;
            }
        }
        i++;
    }
    // all ranks agree: peer stores only if every rank mapped every peer
    std::vector<int> oks(W, 0);
    CL_TRY(comm_allgather(g, &ok, oks.data(), sizeof(int)));
    bool all_ok = true;
    for (int p = 0; p < W; p++) all_ok = all_ok && oks[p];
    if (!all_ok) {
        close_peers(g);
        if (g->host_ag) return Status::make(4, "cleora_init: peer mapping failed on a rank" + (why.empty() ? "" : ": " + why));
        g->xmode = X_NCCL;
    }
    return Status::ok();
}

// The per-peer masks of the deferred exchange (see cleora_init).  Loopback: every emulated rank's
// shard is local, so all the need arrays are; otherwise this rank's is all-gathered with the others'.
Status build_peer_masks(cleora_graph* g) {
    const int W = g->world;
    const size_t N = (size_t)g->n;
    uint8_t* all = nullptr;
    CL_TRY(dalloc((void**)&all, N * W, g->stream, "need flags", kAllocTransient));
    Status st = Status::ok();
    if (g->xmode == X_LOOPBACK) {
        for (int p = 0; p < W && st.good(); p++) st = need_flags(g->of(p).col, g->of(p).nnz, g->n, g->stream, all + N * p);
    } else {
        st = need_flags(g->own().col, g->own().nnz, g->n, g->stream, all + N * g->rank);
        if (st.good() && g->host_ag) {
            std::vector<uint8_t> h(N * W);
            cudaError_t e = cudaMemcpyAsync(h.data() + N * g->rank, all + N * g->rank, N, cudaMemcpyDeviceToHost, g->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
            if (e != cudaSuccess) st = Status::make(4, std::string("need flags: ") + cudaGetErrorString(e));
            if (st.good()) {
                std::vector<uint8_t> mine(h.begin() + N * g->rank, h.begin() + N * (g->rank + 1));
                st = comm_allgather(g, mine.data(), h.data(), N);
            }
            if (st.good() && cudaMemcpyAsync(all, h.data(), N * W, cudaMemcpyHostToDevice, g->stream) != cudaSuccess)
                st = Status::make(4, "need flags upload");
            if (st.good() && cudaStreamSynchronize(g->stream) != cudaSuccess) st = Status::make(4, "need flags upload");
        } else if (st.good()) {
            Nccl& Nc = nccl();
            ncclResult_t r = Nc.AllGather(all + N * g->rank, all, N, ncclUint8, g->comm, g->stream);
            if (r != ncclSuccess) st = Status::make(4, std::string("ncclAllGather: ") + Nc.GetErrorString(r));
        }
    }
    const int nm = g->xmode == X_LOOPBACK ? W : 1;
    for (int i = 0; i < nm && st.good(); i++) {
        uint8_t* m = nullptr;
        st = dalloc((void**)&m, N, g->stream, "peer masks");
        if (st.good()) {
            g->pmask.push_back(m);
            st = peer_masks(all, g->n, W, g->xmode == X_LOOPBACK ? i : g->rank, g->stream, m);
        }
    }
    dfree(all, g->stream);
    return st;
}

Status exchange(cleora_graph* g, float* buf) {
    // all-gather(-v) of the row shards into every replica: one in-place broadcast per rank
    Nccl& N = nccl();
    CL_NCCL_TRY(N.GroupStart());
    for (int p = 0; p < g->world; p++) {
        const int64_t b = g->cuts[p], e = g->cuts[p + 1];
        if (e <= b) continue;
        float* ptr = buf + b * (int64_t)g->dp;
        CL_NCCL_TRY(N.Broadcast(ptr, ptr, (size_t)(e - b) * g->dp, ncclFloat32, p, g->comm, g->stream));
    }
    CL_NCCL_TRY(N.GroupEnd());
    return Status::ok();
}

struct BatchSpec {
    const int64_t* edge_ptr;    // host [n_graphs + 1]
    const int32_t* node_count;  // host [n_graphs]
    int32_t n_graphs;
};

// The build proper (inputs staged on the device, CSR, shard cuts); collective work only through
// shard-independent steps, so a failure here is agreed on by do_build before it returns.
Status build_body(const int32_t* src, const int32_t* dst, const float* w, int64_t E, int32_t N, int directed,
                  const cleora_opts* o, cleora_graph* g, const BatchSpec* batch) {
    // a1: device copies of the COO when the caller passed host memory
    const int32_t* dsrc = src;
    const int32_t* ddst = dst;
    const float* dw = w;
    void *bs = nullptr, *bd = nullptr, *bw = nullptr;
    void *gs = nullptr, *gd = nullptr;
    struct Staged {           // freed on every return path
        cleora_graph* g;
        void** p[5];
        ~Staged() { for (auto q : p) { dfree(*q, g->stream); *q = nullptr; } }
    } staged{g, {&bs, &bd, &bw, &gs, &gd}};
    const bool on_dev = o && o->input_on_device;
    if (!on_dev) {
        CL_TRY(dalloc(&bs, E * sizeof(int32_t), g->stream, "input src", kAllocTransient));
        CL_TRY(dalloc(&bd, E * sizeof(int32_t), g->stream, "input dst", kAllocTransient));
        CL_CUDA_TRY(cudaMemcpyAsync(bs, src, E * sizeof(int32_t), cudaMemcpyHostToDevice, g->stream));
        CL_CUDA_TRY(cudaMemcpyAsync(bd, dst, E * sizeof(int32_t), cudaMemcpyHostToDevice, g->stream));
        if (w) {
            CL_TRY(dalloc(&bw, E * sizeof(float), g->stream, "input weight", kAllocTransient));
            CL_CUDA_TRY(cudaMemcpyAsync(bw, w, E * sizeof(float), cudaMemcpyHostToDevice, g->stream));
        }
        dsrc = (const int32_t*)bs;
        ddst = (const int32_t*)bd;
        dw = (const float*)bw;
    }
    trace("build: inputs staged", g->stream, true);
    // batched handle: local ids -> rows of the block-diagonal M
    if (batch) {
        std::vector<int64_t> base(batch->n_graphs + 1, 0);
        for (int i = 0; i < batch->n_graphs; i++) base[i + 1] = base[i] + batch->node_count[i];
        g->n_graphs = batch->n_graphs;
        void* d_ep = nullptr;
        Status st0 = dalloc((void**)&g->d_base, base.size() * sizeof(int64_t), g->stream, "batch bases");
        if (st0.good()) st0 = dalloc(&d_ep, base.size() * sizeof(int64_t), g->stream, "batch edge offsets", kAllocTransient);
        if (st0.good()) st0 = dalloc(&gs, E * sizeof(int32_t), g->stream, "batch src", kAllocTransient);
        if (st0.good()) st0 = dalloc(&gd, E * sizeof(int32_t), g->stream, "batch dst", kAllocTransient);
        if (st0.good()) {
            cudaMemcpyAsync(g->d_base, base.data(), base.size() * sizeof(int64_t), cudaMemcpyHostToDevice, g->stream);
            cudaMemcpyAsync(d_ep, batch->edge_ptr, base.size() * sizeof(int64_t), cudaMemcpyHostToDevice, g->stream);
            st0 = batch_global_ids(dsrc, ddst, E, (const int64_t*)d_ep, g->d_base, batch->n_graphs, g->stream,
                                   (int32_t*)gs, (int32_t*)gd);
        }
        dfree(d_ep, g->stream);
        CL_TRY(st0);
        dsrc = (const int32_t*)gs;
        ddst = (const int32_t*)gd;
    }
    BuildExtra bx;
    if (o && o->n_chunks >= 1) {
        g->n_chunks = o->n_chunks;
        g->chunk = o->chunk;
        g->chunk_seed = o->chunk_seed;
        CL_TRY(dalloc((void**)&g->occ, (size_t)N * sizeof(int32_t), g->stream, "chunk occurrences"));
        bx.n_chunks = o->n_chunks;
        bx.chunk = o->chunk;
        bx.chunk_key = sm64(o->chunk_seed + 0x9E3779B97F4A7C15ull);
        bx.occ = g->occ;
    }
    g->cuts.assign(g->world + 1, 0);
    if (g->world == 1) {
        BuildOut b;
        CL_TRY(build_csr(dsrc, ddst, dw, E, N, directed, g->stream, &b, &bx));
        trace("build: csr", g->stream, true);
        g->csr.assign(1, Csr());
        g->csr[0] = Csr{b.row_ptr, b.col, b.val, b.deg, b.d_scal, b.nnz, b.zero_rows, b.max_degree};
        g->nnz = b.nnz;
        g->zero_rows = b.zero_rows;
        g->max_degree = b.max_degree;
        g->cuts[1] = N;
    } else {
        // row-sharded: cuts from every row's entry count, then only this rank's rows
        // (every emulated rank's, in loopback)
        std::vector<int64_t> ent(g->world + 1, 0);
        g->sharded = true;
        CL_TRY(shard_plan(dsrc, ddst, dw, E, N, directed, &bx, g->world, g->stream, g->cuts.data(), ent.data(),
                          &g->indeg));
        const bool lb = g->xmode == X_LOOPBACK;
        g->csr.assign(lb ? g->world : 1, Csr());
        for (int p = lb ? 0 : g->rank; p < (lb ? g->world : g->rank + 1); p++) {
            BuildExtra bp = bx;
            bp.row_lo = (int32_t)g->cuts[p];
            bp.row_hi = (int32_t)g->cuts[p + 1];
            bp.shard_entries = ent[p + 1] - ent[p];
            BuildOut b;
            CL_TRY(build_csr(dsrc, ddst, dw, E, N, directed, g->stream, &b, &bp));
            g->of(p) = Csr{b.row_ptr, b.col, b.val, b.deg, b.d_scal, b.nnz, b.zero_rows, b.max_degree};
        }
        trace("build: shard csr", g->stream, true);
    }
    g->r0 = g->cuts[g->rank];
    g->r1 = g->cuts[g->rank + 1];
    g->bytes = (int64_t)(N + 1) * 8 + g->own().nnz * 8 + (int64_t)N * 8;
    return Status::ok();
}

Status do_build(const int32_t* src, const int32_t* dst, const float* w, int64_t E, int32_t N, int directed,
                const cleora_opts* o, cleora_graph* g, const BatchSpec* batch = nullptr) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return Status::make(4, "cleora_build: no CUDA device visible (libcleora has no CPU fallback)");
    }
    int dev = (o && o->device >= 0) ? o->device : -1;
    if (dev < 0) CL_CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= ndev) return Status::make(2, "cleora_build: device ordinal out of range");
    CL_CUDA_TRY(cudaSetDevice(dev));
    int major = 0;
    CL_CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) return Status::make(4, "cleora_build: libcleora is compiled for sm_100a (B200) only");
    g->device = dev;
    if (o && o->stream) {
        g->stream = (cudaStream_t)o->stream;
    } else {
        CL_CUDA_TRY(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
        g->own_stream = true;
    }
    g->timing = o && (o->flags & CLEORA_F_TIMING);
    g->n = N;
    g->n_edges_in = E;
    g->directed = directed;
    g->heavy_thresh = heavy_thresh_default(64);   // set per kernel by cleora_init
    g->rank = (o && o->world > 1) ? o->rank : 0;
    g->world = (o && o->world > 1) ? o->world : 1;
    const bool loopback = g->world > 1 && o && (o->flags & CLEORA_F_LOOPBACK);
    if (loopback) {
        g->sched_p.resize(g->world);        // every rank's schedule lives here (built by init)
        g->rep.assign(g->world, {nullptr, nullptr});
        g->xmode = X_LOOPBACK;
    }
    // collectives first (NCCL communicator: itself collective), then the build, whose outcome every
    // rank agrees on before returning
    if (g->world > 1 && !loopback) {
        g->xmode = (o->flags & CLEORA_F_EXCHANGE_NCCL) ? X_NCCL : X_PEER;
        CL_TRY(dalloc((void**)&g->d_flag, 16, g->stream, "barrier flag"));
        CL_CUDA_TRY(cudaMemsetAsync(g->d_flag, 0, 16, g->stream));
        if (o->nccl_id) {
            Nccl& nc = nccl();
            if (!nc.ok) return Status::make(4, "cleora_build: NCCL unavailable: " + nc.why);
            CL_TRY(comm_get(o->nccl_id, g->world, g->rank, dev, &g->comm));
        } else {
            g->host_ag = o->host_allgather;
            g->host_ctx = o->host_ctx;
            if (g->xmode == X_NCCL) return Status::make(2, "cleora_build: CLEORA_F_EXCHANGE_NCCL needs nccl_id");
        }
    }
    Status st = build_body(src, dst, w, E, N, directed, o, g, batch);
    if (g->world > 1 && st.good()) {
        // the whole M's facts: entries, rows without entries, longest row -- summed / maxed over the shards
        std::vector<unsigned long long> f(3 * g->csr.size());
        for (size_t p = 0; p < g->csr.size(); p++) {
            f[3 * p] = (unsigned long long)g->csr[p].zero_rows;
            f[3 * p + 1] = (unsigned long long)g->csr[p].max_degree;
            f[3 * p + 2] = (unsigned long long)g->csr[p].nnz;
        }
        if (st.good() && !loopback) {
            std::vector<unsigned long long> all(3 * g->world);
            Status sa = comm_agree(g, st);
            if (sa.good()) sa = comm_allgather(g, f.data(), all.data(), 3 * sizeof(unsigned long long));
            if (!sa.good()) return sa;
            f.swap(all);
        }
        if (st.good()) {
            unsigned long long z = 0, mx = 0, nz = 0;
            for (size_t q = 0; q < f.size() / 3; q++) {
                z += f[3 * q];
                mx = std::max(mx, f[3 * q + 1]);
                nz += f[3 * q + 2];
            }
            g->zero_rows = (int64_t)z;
            g->max_degree = (int64_t)mx;
            g->nnz = (int64_t)nz;
            return Status::ok();
        }
    }
    if (g->world > 1 && !loopback) return comm_agree(g, st);
    // no final synchronisation: the CSR's last kernels run on while the caller goes on to
    // cleora_init (stream order keeps everything that reads them behind them)
    return st;
}

}  // namespace

namespace {

constexpr size_t kStageBytes = 256ull << 20;    // packed rows per device-to-host slice

Status ensure_copy_stream(cleora_graph* g) {
    if (g->copy_stream) return Status::ok();
    CL_CUDA_TRY(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
    CL_CUDA_TRY(cudaEventCreateWithFlags(&g->ev_ready, cudaEventDisableTiming));
    CL_CUDA_TRY(cudaEventCreateWithFlags(&g->ev_copied, cudaEventDisableTiming));
    return Status::ok();
}

Status fetch_nonzero(cleora_graph* g, float* out_rows, int32_t* out_ids, int64_t capacity, int64_t* n_rows,
                     int32_t out_on_device, bool wait) {
    // every row while T may hold non-zero rows without entries: T_0 (no step yet) or rows the caller set
    const bool all = g->iters == 0 || g->rows_set;
    const int64_t n = all ? g->r1 - g->r0 : (g->r1 - g->r0) - g->own().zero_rows;
    *n_rows = n;
    if (!out_rows && !out_ids) return Status::ok();
    if (capacity < n) return Status::make(2, "cleora_fetch_nonzero: capacity below the row count (query it first)");
    if (n == 0) return Status::ok();
    CL_TRY(complete_t0(g));
    CL_TRY(ensure_copy_stream(g));
    if (!g->nz_ids || g->nz_all != all) {
        if (!all && g->trimmed)
            return Status::make(2, "cleora_fetch_nonzero: the handle was trimmed before its rows were selected "
                                   "(call cleora_fetch_nonzero_async before cleora_trim)");
        if (g->nz_ids) {            // the copy stream may still read the previous selection
            CL_CUDA_TRY(cudaStreamSynchronize(g->copy_stream));
            dfree(g->nz_ids, g->stream);
            g->nz_ids = nullptr;
        }
        CL_TRY(dalloc((void**)&g->nz_ids, (size_t)n * sizeof(int32_t), g->stream, "nonzero row ids"));
        CL_TRY(select_rows_with_entries(all ? nullptr : g->own().row_ptr, g->r0, g->r1, all, g->nz_ids, g->stream));
        g->nz_n = n;
        g->nz_all = all;
    }
    const size_t row_bytes = (size_t)g->d * sizeof(float);
    // nothing enqueued from here on may overwrite what an earlier copy of this handle still reads
    order_after_side(g);
    const float* T = g->T[g->cur];
    if (out_rows && out_on_device) {
        // device outputs: packed in stream order, nothing for the copy engine
        CL_TRY(pack_rows(T, g->dp, g->d, g->nz_ids, n, out_rows, g->stream));
        if (out_ids)
            CL_CUDA_TRY(cudaMemcpyAsync(out_ids, g->nz_ids, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                        g->stream));
        if (wait) CL_CUDA_TRY(cudaStreamSynchronize(g->stream));
        return Status::ok();
    }
    // Host outputs.  The rows are packed on the handle's stream right behind the steps, into one staging
    // buffer for the whole result when it can be had, and leave in one DMA on the copy stream.  (Packing
    // slice by slice on the copy stream instead made every slice's pack wait for SMs behind the next
    // graph's persistent SpMM launch: c4's pipelined e2e 240 ms where the DMA alone needs ~172.)  If the
    // whole result does not fit beside the handle, 256 MB slices are packed and copied one after another
    // on the copy stream.
    const size_t full = (size_t)n * row_bytes;
    bool whole = false;
    if (out_rows) {
        // CLEORA_FETCH_SLICES=1 (read per call): always the sliced path (tests, A/B)
        const char* fs = getenv("CLEORA_FETCH_SLICES");
        const bool force_slices = fs && fs[0] == '1';
        if (!force_slices) {
            if (g->stage && g->stage_bytes < full) {
                dfree(g->stage, g->stream);      // ordered after the earlier copy by order_after_side
                g->stage = nullptr;
                g->stage_bytes = 0;
            }
            // only from the cache or free memory: evicting cached blocks for it would make the next
            // graph's build allocate them again (c5's pipeline, where HBM is full); else slices
            if (!g->stage &&
                dalloc((void**)&g->stage, full, g->stream, "fetch staging (whole result)", kAllocNoEvict).good())
                g->stage_bytes = full;
            whole = g->stage != nullptr;
        }
        if (!g->stage) {
            g->stage_bytes = (size_t)std::min<int64_t>(n, std::max<int64_t>(1, (int64_t)(kStageBytes / row_bytes))) *
                             row_bytes;
            CL_TRY(dalloc((void**)&g->stage, g->stage_bytes, g->stream, "fetch staging"));
        }
        if (whole) CL_TRY(pack_rows(T, g->dp, g->d, g->nz_ids, n, g->stage, g->stream));
    }
    // the copy starts when the work enqueued so far on the handle's stream is done
    CL_CUDA_TRY(cudaEventRecord(g->ev_ready, g->stream));
    CL_CUDA_TRY(cudaStreamWaitEvent(g->copy_stream, g->ev_ready, 0));
    if (out_rows && whole) {
        CL_CUDA_TRY(cudaMemcpyAsync(out_rows, g->stage, full, cudaMemcpyDeviceToHost, g->copy_stream));
    } else if (out_rows) {
        // slice k: pack on the SMs, then one linear DMA; the next slice's pack queues behind this copy
        // on the same stream, so one staging buffer suffices
        const int64_t per = (int64_t)(std::min(g->stage_bytes, kStageBytes) / row_bytes);
        for (int64_t k0 = 0; k0 < n; k0 += per) {
            const int64_t cnt = std::min<int64_t>(per, n - k0);
            CL_TRY(pack_rows(T, g->dp, g->d, g->nz_ids + k0, cnt, g->stage, g->copy_stream));
            CL_CUDA_TRY(cudaMemcpyAsync(out_rows + k0 * (int64_t)g->d, g->stage, (size_t)cnt * row_bytes,
                                        cudaMemcpyDeviceToHost, g->copy_stream));
        }
    }
    if (out_ids)
        CL_CUDA_TRY(cudaMemcpyAsync(out_ids, g->nz_ids, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                    g->copy_stream));
    CL_CUDA_TRY(cudaEventRecord(g->ev_copied, g->copy_stream));
    g->copy_pending = true;
    if (wait) CL_CUDA_TRY(cudaStreamSynchronize(g->copy_stream));
    return Status::ok();
}

}  // namespace

extern "C" {

const char* cleora_last_error(void) { return g_err.c_str(); }

int64_t cleora_kernel_launches(void) { return g_launches.load(); }

int cleora_release_cached_memory(void) {
    ipc_close_all();
    release_cached(-1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_release_cached_memory: ") + cudaGetErrorString(e)));
    return CLEORA_OK;
}

int cleora_build(const int32_t* src, const int32_t* dst, const float* weight, int64_t n_edges, int32_t n_nodes,
                 int32_t directed, const cleora_opts* opts, cleora_graph** out) {
    NvtxRange _nvtx("cleora_build");
    if (!out) return usage("cleora_build: out is NULL");
    *out = nullptr;
    if (!src || !dst) return usage("cleora_build: src/dst is NULL");
    if (n_nodes <= 0) return usage("cleora_build: n_nodes must be > 0");
    if (n_edges <= 0) return usage("cleora_build: n_edges must be > 0 (non-empty edge list)");
    if (opts && opts->world > 1) {
        if (opts->world - 1 > kMaxPeers && (opts->flags & CLEORA_F_LOOPBACK))
            return usage("cleora_build: loopback emulation supports at most 8 ranks");
        if (!opts->nccl_id && !opts->host_allgather && !(opts->flags & CLEORA_F_LOOPBACK))
            return usage("cleora_build: world > 1 needs nccl_id or host_allgather");
        if (opts->rank < 0 || opts->rank >= opts->world) return usage("cleora_build: rank outside [0, world)");
        if (opts->world > 255) return usage("cleora_build: world > 255 (shard cuts and counts are read back in one 4 KB read)");
    }
    if (opts && opts->n_chunks != 0) {
        if (opts->n_chunks < 0 || opts->chunk < 0 || opts->chunk >= opts->n_chunks)
            return usage("cleora_build: chunk must be in [0, n_chunks)");
    }
    DeviceGuard guard(opts ? opts->device : -1);
    cleora_graph* g = new cleora_graph();
    Status s = do_build(src, dst, weight, n_edges, n_nodes, directed ? 1 : 0, opts, g);
    if (!s.good()) {
        cleora_destroy(g);
        return fail(s);
    }
    *out = g;
    return CLEORA_OK;
}

int cleora_expand(const int64_t* he_ptr, const int32_t* he_nodes, const float* he_weight, int64_t n_hyperedges,
                  int32_t n_nodes, int32_t mode, int32_t device, int32_t on_device, void* stream, int32_t* out_src,
                  int32_t* out_dst, float* out_weight, int64_t capacity, int64_t* n_out) {
    NvtxRange _nvtx("cleora_expand");
    if (!he_ptr || !he_nodes || !n_out) return usage("cleora_expand: NULL argument");
    if (n_hyperedges < 1 || n_nodes < 1) return usage("cleora_expand: n_hyperedges and n_nodes must be >= 1");
    if (mode != CLEORA_EXPAND_CLIQUE && mode != CLEORA_EXPAND_STAR) return usage("cleora_expand: unknown mode");
    if (mode == CLEORA_EXPAND_STAR && (int64_t)n_nodes + n_hyperedges > INT32_MAX)
        return usage("cleora_expand: n_nodes + n_hyperedges exceeds the int32 id range");
    if ((out_dst == nullptr) != (out_src == nullptr)) return usage("cleora_expand: out_src and out_dst go together");
    *n_out = 0;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(Status::make(4, "cleora_expand: no CUDA device visible (libcleora has no CPU fallback)"));
    }
    DeviceGuard guard(device);
    cudaStream_t s = stream ? (cudaStream_t)stream : cudaStreamPerThread;
    int64_t n_members = 0;
    const int64_t* dptr = he_ptr;
    const int32_t* dnodes = he_nodes;
    const float* dw = he_weight;
    void *bp = nullptr, *bn = nullptr, *bw = nullptr;
    void *os = nullptr, *od = nullptr, *ow = nullptr;
    Status st = Status::ok();
    if (on_device) {
        cudaError_t e = cudaMemcpyAsync(&n_members, he_ptr + n_hyperedges, sizeof n_members, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_expand: ") + cudaGetErrorString(e)));
        if (n_members < 0) return usage("cleora_expand: he_ptr must start at 0 and be non-decreasing");
    } else {
        n_members = he_ptr[n_hyperedges];
        if (he_ptr[0] != 0) return usage("cleora_expand: he_ptr[0] must be 0");
        for (int64_t i = 0; i < n_hyperedges; i++)
            if (he_ptr[i + 1] < he_ptr[i]) return usage("cleora_expand: he_ptr must be non-decreasing");
        st = dalloc(&bp, (n_hyperedges + 1) * sizeof(int64_t), s, "expand he_ptr", kAllocTransient);
        if (st.good()) st = dalloc(&bn, (n_members > 0 ? n_members : 1) * sizeof(int32_t), s, "expand members", kAllocTransient);
        if (st.good() && he_weight) st = dalloc(&bw, n_hyperedges * sizeof(float), s, "expand weights", kAllocTransient);
        if (st.good()) {
            cudaMemcpyAsync(bp, he_ptr, (n_hyperedges + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
            if (n_members > 0) cudaMemcpyAsync(bn, he_nodes, n_members * sizeof(int32_t), cudaMemcpyHostToDevice, s);
            if (he_weight) cudaMemcpyAsync(bw, he_weight, n_hyperedges * sizeof(float), cudaMemcpyHostToDevice, s);
            dptr = (const int64_t*)bp;
            dnodes = (const int32_t*)bn;
            dw = (const float*)bw;
        }
    }
    if (st.good() && !on_device && out_src) {
        // count first, then stage the outputs on the device
        st = expand_hypergraph(dptr, dnodes, dw, n_hyperedges, n_members, n_nodes, mode, s, nullptr, nullptr, nullptr, 0,
                               n_out);
        if (st.good() && *n_out > capacity) st = Status::make(2, "cleora_expand: capacity smaller than the edge count");
        if (st.good() && *n_out > 0) {
            st = dalloc(&os, *n_out * sizeof(int32_t), s, "expand out src", kAllocTransient);
            if (st.good()) st = dalloc(&od, *n_out * sizeof(int32_t), s, "expand out dst", kAllocTransient);
            if (st.good() && out_weight) st = dalloc(&ow, *n_out * sizeof(float), s, "expand out weight", kAllocTransient);
        }
    }
    if (st.good()) {
        int32_t* ts = on_device ? out_src : (int32_t*)os;
        int32_t* td = on_device ? out_dst : (int32_t*)od;
        float* tw = on_device ? out_weight : (float*)ow;
        if (out_src && (on_device || *n_out > 0))
            st = expand_hypergraph(dptr, dnodes, dw, n_hyperedges, n_members, n_nodes, mode, s, ts, td, tw, capacity, n_out);
        else if (!out_src)
            st = expand_hypergraph(dptr, dnodes, dw, n_hyperedges, n_members, n_nodes, mode, s, nullptr, nullptr, nullptr,
                                   0, n_out);
    }
    if (st.good() && !on_device && out_src && *n_out > 0) {
        cudaMemcpyAsync(out_src, os, *n_out * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(out_dst, od, *n_out * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        if (out_weight) cudaMemcpyAsync(out_weight, ow, *n_out * sizeof(float), cudaMemcpyDeviceToHost, s);
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = Status::make(4, std::string("cleora_expand: ") + cudaGetErrorString(e));
    }
    cudaStreamSynchronize(s);
    dfree(os, s);
    dfree(od, s);
    dfree(ow, s);
    dfree(bp, s);
    dfree(bn, s);
    dfree(bw, s);
    if (!st.good()) return fail(st);
    return CLEORA_OK;
}

int cleora_build_batch(const int32_t* src, const int32_t* dst, const float* weight, const int64_t* edge_ptr,
                       const int32_t* node_count, int32_t n_graphs, int32_t directed, const cleora_opts* opts,
                       cleora_graph** out) {
    NvtxRange _nvtx("cleora_build_batch");
    if (!out) return usage("cleora_build_batch: out is NULL");
    *out = nullptr;
    if (!src || !dst || !edge_ptr || !node_count) return usage("cleora_build_batch: NULL argument");
    if (n_graphs < 1) return usage("cleora_build_batch: n_graphs must be >= 1");
    if (edge_ptr[0] != 0) return usage("cleora_build_batch: edge_ptr[0] must be 0");
    int64_t ntot = 0;
    for (int i = 0; i < n_graphs; i++) {
        if (node_count[i] < 1) return usage("cleora_build_batch: every node_count must be >= 1");
        if (edge_ptr[i + 1] < edge_ptr[i]) return usage("cleora_build_batch: edge_ptr must be non-decreasing");
        ntot += node_count[i];
    }
    if (ntot > INT32_MAX) return usage("cleora_build_batch: the batch has more than 2^31-1 nodes");
    const int64_t E = edge_ptr[n_graphs];
    if (E <= 0) return usage("cleora_build_batch: the batch has no edges");
    if (opts && (opts->world > 1 || opts->n_chunks != 0))
        return usage("cleora_build_batch: batches are single-GPU and unchunked");
    DeviceGuard guard(opts ? opts->device : -1);
    cleora_graph* g = new cleora_graph();
    BatchSpec b{edge_ptr, node_count, n_graphs};
    Status s = do_build(src, dst, weight, E, (int32_t)ntot, directed ? 1 : 0, opts, g, &b);
    if (!s.good()) {
        cleora_destroy(g);
        return fail(s);
    }
    *out = g;
    return CLEORA_OK;
}

int cleora_init(cleora_graph* g, int32_t d, uint64_t seed) {
    NvtxRange _nvtx("cleora_init");
    if (!g) return usage("cleora_init: graph is NULL");
    if (g->trimmed) return usage("cleora_init: the handle was trimmed (cleora_trim)");
    if (d < 1 || d > CLEORA_MAX_D) return usage("cleora_init: d must be in [1, CLEORA_MAX_D]");
    DeviceGuard guard(g->device);
    order_after_side(g);
    const int32_t dp = (d + 3) / 4 * 4;
    // environment switches (measurement and diagnosis): read once here, not per launch
    g->env_cold_first = getenv("CLEORA_COLD_FIRST") ? atoi(getenv("CLEORA_COLD_FIRST")) : -1;
    g->env_write_zero = getenv("CLEORA_WRITE_ZERO_ROWS") != nullptr;
    g->env_csr_prefetch = getenv("CLEORA_CSR_PREFETCH") ? atoi(getenv("CLEORA_CSR_PREFETCH")) : 1;
    g->env_no_hot = getenv("CLEORA_NO_HOT") != nullptr;
    g->env_defer = getenv("CLEORA_NO_DEFER") == nullptr;
    g->env_lazy = !(getenv("CLEORA_LAZY") && atoi(getenv("CLEORA_LAZY")) == 0);
    g->env_t0_all = getenv("CLEORA_T0_ALL") && atoi(getenv("CLEORA_T0_ALL")) != 0;
    g->env_drop_ungathered = !(getenv("CLEORA_KEEP_UNGATHERED") && atoi(getenv("CLEORA_KEEP_UNGATHERED")) != 0);
    if (dp != g->dp || !g->T[0]) {
        free_T(g);
        // N x dp rows, then N fp32 row scales (lazy steps, reading R21: a peer's scales ride in the same
        // allocation, so the IPC mapping of its T covers them); the scales start at 0
        const size_t tb = ((size_t)g->n * dp + (size_t)g->n) * sizeof(float);
        Status sa = Status::ok();
        // peers map T through CUDA IPC, which exports whole allocations: T at a segment's base
        const int tflags = g->xmode == X_PEER ? kAllocBase : 0;
        for (int i = 0; i < 2 && sa.good(); i++) sa = dalloc((void**)&g->T[i], tb, g->stream, "embedding T", tflags);
        // test hook: this rank's T allocation fails (CLEORA_TEST_FAIL_T_RANK=r), to exercise the agreement
        if (const char* fr = getenv("CLEORA_TEST_FAIL_T_RANK"))
            if (g->world > 1 && atoi(fr) == g->rank && sa.good())
                sa = Status::make(4, "cleora_init: injected allocation failure (CLEORA_TEST_FAIL_T_RANK)");
        if (sa.good() && g->xmode == X_LOOPBACK) {
            g->rep[g->rank] = {g->T[0], g->T[1]};
            for (int p = 0; p < g->world && sa.good(); p++) {
                if (p == g->rank) continue;
                for (int i = 0; i < 2 && sa.good(); i++)
                    sa = dalloc((void**)&g->rep[p][i], tb, g->stream, "loopback replica");
            }
        }
        for (int i = 0; i < 2 && sa.good(); i++)
            if (cudaMemsetAsync(g->T[i] + (size_t)g->n * dp, 0, (size_t)g->n * sizeof(float), g->stream) != cudaSuccess)
                sa = Status::make(4, "cleora_init: memset of the row scales failed");
        if (sa.good() && g->xmode == X_LOOPBACK)
            for (int p = 0; p < g->world && sa.good(); p++)
                for (int i = 0; i < 2 && sa.good(); i++)
                    if (p != g->rank &&
                        cudaMemsetAsync(g->rep[p][i] + (size_t)g->n * dp, 0, (size_t)g->n * sizeof(float), g->stream) != cudaSuccess)
                        sa = Status::make(4, "cleora_init: memset of the row scales failed");
        // every rank must have its replicas before any maps them (failure agreement)
        if (g->xmode == X_PEER || g->xmode == X_NCCL) sa = comm_agree(g, sa);
        if (sa.good() && g->xmode == X_PEER) sa = open_peers(g);   // collective; may switch every rank to X_NCCL
        if (!sa.good()) {
            free_T(g);
            return fail(sa);
        }
    }
    g->d = d;
    g->dp = dp;
    g->cur = 0;
    g->iters = 0;
    g->zclean[0] = g->zclean[1] = false;
    // a9: T_0 -- on graphs whose T exceeds the L2 hot-row budget (where the write is milliseconds), only
    // the rows a step can gather (in-degree > 0; the in-degree is the hot-row tags' input anyway);
    // the rest is filled in only if T_0 itself is read (complete_t0).  c4: 2.3M of 4.85M rows.
    {
        const char* hb = getenv("CLEORA_HOT_MB");
        const int64_t budget = (int64_t)(hb ? atof(hb) : 72.0) * 1024 * 1024;
        const int32_t* sel = nullptr;
        if (!g->env_t0_all && g->nnz > 0 && (int64_t)g->n * dp * 4 > budget) {
            if (!g->indeg && !g->sharded) {
                Status s = in_degree(g->csr[0].col, g->csr[0].nnz, g->n, g->directed ? nullptr : g->csr[0].row_ptr,
                                     g->stream, &g->indeg);
                if (!s.good()) return fail(s);
            }
            sel = g->indeg;
        }
        Status s = launch_hash_init(g->T[0], g->n, d, dp, seed, g->stream, g->d_base, g->n_graphs, sel, sel ? 1 : 0);
        if (!s.good()) return fail(s);
        if (g->xmode == X_LOOPBACK)   // every emulated rank initialises its own replica
            for (int p = 0; p < g->world; p++)
                if (p != g->rank) {
                    s = launch_hash_init(g->rep[p][0], g->n, d, dp, seed, g->stream, g->d_base, g->n_graphs, sel,
                                         sel ? 1 : 0);
                    if (!s.good()) return fail(s);
                }
        g->t0_partial = sel != nullptr;
        g->t0_seed = seed;
    }
    // heavy rows: > 64 entries with TMA bulk gathers, > 256 with cp.async / LDG gathers (measured:
    // c2 12.68 vs 12.80 ms per step with 64 / 256; c5 427 -> 375 ms, c4@256 8.10 -> 7.27 ms with 256);
    // every sequential fp32 run stays <= 256 terms (256-entry blocks keep the error ~3e-7)
    g->gmode = gather_mode(dp);
    // Half-row passes (spmm_tma.cu; bitwise the whole-row result for the same schedule): with 2 KB
    // instead of 4 KB gathers twice as many rows fit the L2, which pays where the gather stream dwarfs
    // T -- c4: nnz = 13.9 N, 28.2 -> 25.7 ms per step (min; profiles/r02_halves_ab.txt) -- and costs
    // where it does not (c2: nnz = 5 N, 2.65 -> 3.14 ms; c3: 2.8 N).  The passes gather 2 KB pieces
    // with cp.async (TMA bulk copies of 2 KB are issue-bound: 36 ms), heavy rows above 256 entries,
    // light chunks of 12 rows -- the d = 512 settings.  CLEORA_HALVES=0/1 forces them off/on.
    {
        const char* e = getenv("CLEORA_HALVES");
        const bool able = dp == 1024 && g->gmode != kGatherLdg;
        g->halves = able && (e ? atoi(e) != 0 : g->nnz >= 8 * (int64_t)g->n);
        if (g->halves && !getenv("CLEORA_GATHER") && !getenv("CLEORA_FORCE_TMA")) g->gmode = kGatherAsync;
    }
    g->heavy_thresh = heavy_thresh_default(g->gmode == kGatherBulk ? 64 : 256);
    // light-chunk row cap per gather engine and row size (measured, scripts/r01/chunk_sweep*.sh, min
    // launch ms): TMA bulk (d = 1024) 6 rows, c3 2.04 -> 1.42 vs 31; cp.async at d = 512 12 rows, c3
    // 0.86 -> 0.75; cp.async at d = 256 31 rows (c3 0.518 vs 0.581 at 8); LDG at d <= 128 16 rows,
    // f4 1.39 -> 1.25, c3@128 0.508 -> 0.490, c4@128 4.296 -> 4.306; half-row passes: 12 (their
    // 2 KB pieces behave like d = 512 rows)
    {
        const int mode = g->gmode;
        g->chunk_rows = mode == kGatherBulk ? (g->halves ? 12 : 6)
                                            : mode == kGatherAsync ? (dp > 256 ? 12 : kChunkRows)
                                                                   : (dp <= 128 ? 16 : kChunkRows);
    }
    if (g->sched_thresh != g->heavy_thresh || g->sched_rows != g->chunk_rows) {
        Status s = make_schedules(g);
        if (!s.good()) return fail(s);
    }
    if (g->max_items > 0 && g->partials_floats < (size_t)g->max_items * dp) {
        dfree(g->partials, g->stream);
        g->partials = nullptr;
        g->partials_floats = 0;
        Status s = dalloc((void**)&g->partials, (size_t)g->max_items * dp * sizeof(float), g->stream,
                          "heavy-row partials");
        if (!s.good()) return fail(s);
        g->partials_floats = (size_t)g->max_items * dp;
    }
    if (g->tag_dp != dp * (g->halves ? -1 : 1) && !g->env_no_hot && g->nnz > 0) {
        // L2 residency hints: tag (bit 31 of col, in place) the columns whose rows are re-read
        // most (highest in-degree) so that their gathers use an evict_last policy, within a
        // budget of the 126 MB L2.  Row-sharded: every shard's columns, from the whole graph's
        // in-degree (shard_plan), so the tags do not depend on the number of ranks.
        const char* e = getenv("CLEORA_HOT_MB");
        const int64_t budget = (int64_t)(e ? atof(e) : 72.0) * 1024 * 1024;
        Status s = Status::ok();
        // T within the budget: everything fits in L2 anyway, nothing to pin (and no host round trip)
        if ((int64_t)g->n * dp * 4 <= budget) g->n_hot = 0;
        for (size_t p = 0; p < g->csr.size() && s.good() && (int64_t)g->n * dp * 4 > budget; p++)
            s = hot_tag(g->csr[p].col, g->csr[p].nnz, g->n, (int64_t)dp * 4 / (g->halves ? 2 : 1), budget, g->stream,
                        &g->n_hot, &g->n_ref,
                        g->directed || g->sharded ? nullptr : g->csr[p].row_ptr, g->indeg);
        if (!s.good()) {
            free_T(g);
            return fail(s);
        }
        g->tag_dp = dp * (g->halves ? -1 : 1);      // the tags depend on the gathered row size
    }
    if (g->sharded && (g->xmode == X_PEER || g->xmode == X_LOOPBACK) && g->pmask.empty() && g->env_defer) {
        // deferred exchange (reading R20): which peers gather which rows.  Every rank flags the columns
        // its shard gathers; the flags are all-gathered; rank p's mask of row r has bit q set when its
        // q-th peer's shard gathers r.  (Collective in X_PEER: every rank takes this branch together.)
        Status s = build_peer_masks(g);
        if (s.good() && g->xmode == X_PEER) s = comm_agree(g, s);
        if (!s.good()) {
            for (auto m : g->pmask) dfree(m, g->stream);
            g->pmask.clear();
            return fail(s);
        }
    }
    if (g->xmode == X_PEER) {
        // no rank may store into another's replicas before that rank is done with its
        // previous steps and has re-initialised
        Status s = rank_barrier(g);
        if (!s.good()) return fail(s);
    }
    return CLEORA_OK;
}

int cleora_iterate(cleora_graph* g, int32_t k) {
    NvtxRange _nvtx("cleora_iterate");
    if (!g) return usage("cleora_iterate: graph is NULL");
    if (g->trimmed) return usage("cleora_iterate: the handle was trimmed (cleora_trim)");
    if (k < 0) return usage("cleora_iterate: k must be >= 0");
    if (!g->T[0]) return usage("cleora_iterate: call cleora_init first");
    DeviceGuard guard(g->device);
    order_after_side(g);
    const int nsh = g->xmode == X_LOOPBACK ? g->world : 1;
    // Lazy normalisation (reading R21): with half-row passes, every step of this call but the
    // last leaves its rows unnormalised with their scales aside, and the next step folds the scales
    // into its weights -- the last step writes normalised rows, so what T holds between calls is
    // unchanged.  Saves the first half's read-back and rewrite (c4: 9.4 GB of 188 GB per step).
    // One GPU, loopback and peer stores alike (the peers receive the unnormalised halves and the scales
    // like any row, so P does not change a bit); not with the NCCL all-gather fallback.
    const bool lazy = g->halves && g->env_lazy && k >= 2 &&
                      (g->world == 1 || g->xmode == X_LOOPBACK || g->xmode == X_PEER);
    if (lazy && !g->lazy_buf) {
        int64_t nnz_max = 0;
        for (const Csr& c : g->csr) nnz_max = std::max(nnz_max, c.nnz);
        const size_t bytes = (size_t)(g->n + 1) / 2 * 2 * sizeof(double) + (size_t)nnz_max * sizeof(float);
        Status s = dalloc((void**)&g->lazy_buf, bytes, g->stream, "lazy sums and weights");
        if (!s.good()) return fail(s);
    }
    for (int32_t i = 0; i < k; i++) {
        const int in = g->cur, out = 1 - g->cur;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (g->timing) {
            e0 = get_event(g);
            e1 = get_event(g);
            cudaEventRecord(e0, g->stream);
        }
        for (int sh = 0; sh < nsh; sh++) {
            // rank p's launch; outside loopback p is this rank and there is one launch
            const int p = g->xmode == X_LOOPBACK ? sh : g->rank;
            const Schedule& sc = g->xmode == X_LOOPBACK ? g->sched_p[p] : g->sched;
            SpmmArgs a;
            const Csr& c = g->of(p);
            a.row_ptr = c.row_ptr;
            a.col = c.col;
            a.val = c.val;
            a.gather_mode = g->gmode;
            a.T_in = g->xmode == X_LOOPBACK ? g->rep[p][in] : g->T[in];
            a.T_out = g->xmode == X_LOOPBACK ? g->rep[p][out] : g->T[out];
            a.dp = g->dp;
            a.r0 = g->cuts[p];
            a.r1 = g->cuts[p + 1];
            a.heavy_thresh = g->heavy_thresh;
            a.items = sc.items;
            a.counts = sc.counts;
            a.n_items_max = sc.n_items_max;
            a.partials = g->partials;
            a.counters = sc.counters;
            // with hot rows pinned (power-law graphs) the other gathers are evicted first; without
            // (e.g. lattices, whose re-reads are local) they keep the normal policy (measured: c2, c4, c3)
            a.cold_first = g->env_cold_first >= 0 ? g->env_cold_first : (g->n_hot > 0 ? 1 : 0);
            a.work = sc.work;
            a.light_start = sc.light_start;
            a.n_peers = 0;
            for (int q = 0; q < kMaxPeers; q++) a.peer_out[q] = nullptr;
            if (g->xmode == X_LOOPBACK) {
                for (int q = 0; q < g->world; q++)
                    if (q != p) a.peer_out[a.n_peers++] = g->rep[q][out];
            } else if (g->xmode == X_PEER) {
                for (int q = 0; q < g->world - 1; q++) a.peer_out[a.n_peers++] = g->peer_T[out][q];
            }
            a.skip_zero_rows = (g->zclean[out] && !g->env_write_zero) ? 1 : 0;
            a.csr_prefetch = g->env_csr_prefetch;
            // deferred exchange: before the last step of this call only gathered rows go to the peers;
            // the last step sends every row, so a fetch on any rank sees the whole T
            a.peer_mask = (a.n_peers > 0 && !g->pmask.empty() && i + 1 < k) ? g->pmask[g->pmask.size() > 1 ? p : 0]
                                                                              : nullptr;
            a.pass = 0;
            a.scale_off = (int64_t)g->n * g->dp;
            a.ss_half = lazy && i + 1 < k ? g->lazy_buf : nullptr;
            a.lazy_out = 0;
            a.drop_rows = (a.ss_half && g->env_drop_ungathered) ? g->indeg : nullptr;
            Status s = Status::ok();
            if (lazy && i > 0) {
                // T_in holds the previous step's rows unnormalised: fold their scales into the weights
                float* lv = reinterpret_cast<float*>(g->lazy_buf + (g->n + 1) / 2 * 2);   // 16-byte aligned
                s = launch_lazy_vals(c.val, c.col, a.T_in + a.scale_off, c.nnz, lv, g->stream);
                a.val = lv;
            }
            if (g->halves && s.good()) {
                a.pass = 1;
                s = launch_spmm_norm(a, g->stream);
                a.pass = 2;
                a.lazy_out = lazy && i + 1 < k ? 1 : 0;
            }
            if (s.good()) s = launch_spmm_norm(a, g->stream);
            if (!s.good()) return fail(s);
        }
        if (g->timing) {
            cudaEventRecord(e1, g->stream);
            g->ev_spmm.emplace_back(e0, e1);
        }
        if (g->xmode == X_NCCL || g->xmode == X_PEER) {
            if (g->timing) {
                e0 = get_event(g);
                e1 = get_event(g);
                cudaEventRecord(e0, g->stream);
            }
            // X_NCCL: all-gather-v of the shards; X_PEER: the rows are already in every
            // replica, only the step order across ranks is enforced
            Status s = g->xmode == X_NCCL ? exchange(g, g->T[out]) : rank_barrier(g);
            if (!s.good()) return fail(s);
            if (g->timing) {
                cudaEventRecord(e1, g->stream);
                g->ev_x.emplace_back(e0, e1);
            }
        }
        g->zclean[out] = true;     // every row of T[out] was written (or was already 0)
        g->cur = out;
        g->iters++;
        g->rows_set = false;
    }
    return CLEORA_OK;
}

int cleora_fetch(const cleora_graph* g, int64_t row_begin, int64_t row_end, float* out, int32_t out_on_device) {
    NvtxRange _nvtx("cleora_fetch");
    if (!g || !out) return usage("cleora_fetch: NULL argument");
    if (!g->T[0]) return usage("cleora_fetch: call cleora_init first");
    if (row_begin < 0 || row_end > g->n || row_begin > row_end) return usage("cleora_fetch: rows outside [0, N]");
    if (row_end == row_begin) return CLEORA_OK;
    DeviceGuard guard(g->device);
    {
        Status st0 = complete_t0(g);
        if (!st0.good()) return fail(st0);
    }
    order_after_side(g);
    const float* src = g->T[g->cur] + row_begin * (int64_t)g->dp;
    const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    cudaError_t e;
    if (g->d == g->dp)   // dense rows: one linear copy (full PCIe rate into pinned memory)
        e = cudaMemcpyAsync(out, src, (size_t)(row_end - row_begin) * g->d * sizeof(float), kind, g->stream);
    else
        e = cudaMemcpy2DAsync(out, (size_t)g->d * sizeof(float), src, (size_t)g->dp * sizeof(float),
                              (size_t)g->d * sizeof(float), (size_t)(row_end - row_begin), kind, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_fetch: ") + cudaGetErrorString(e)));
    return CLEORA_OK;
}

int cleora_fetch_async(cleora_graph* g, int64_t row_begin, int64_t row_end, float* out, int32_t out_on_device) {
    NvtxRange _nvtx("cleora_fetch_async");
    if (!g || !out) return usage("cleora_fetch_async: NULL argument");
    if (!g->T[0]) return usage("cleora_fetch_async: call cleora_init first");
    if (row_begin < 0 || row_end > g->n || row_begin > row_end) return usage("cleora_fetch_async: rows outside [0, N]");
    if (row_end == row_begin) return CLEORA_OK;
    DeviceGuard guard(g->device);
    {
        Status st0 = complete_t0(g);
        if (!st0.good()) return fail(st0);
    }
    cudaError_t e = cudaSuccess;
    if (!g->copy_stream) {
        e = cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_ready, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_copied, cudaEventDisableTiming);
        if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_fetch_async: ") + cudaGetErrorString(e)));
    }
    // the copy starts when the work enqueued so far on the handle's stream is done
    order_after_side(g);
    e = cudaEventRecord(g->ev_ready, g->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(g->copy_stream, g->ev_ready, 0);
    const float* src = g->T[g->cur] + row_begin * (int64_t)g->dp;
    const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (e == cudaSuccess) {
        if (g->d == g->dp)
            e = cudaMemcpyAsync(out, src, (size_t)(row_end - row_begin) * g->d * sizeof(float), kind, g->copy_stream);
        else
            e = cudaMemcpy2DAsync(out, (size_t)g->d * sizeof(float), src, (size_t)g->dp * sizeof(float),
                                  (size_t)g->d * sizeof(float), (size_t)(row_end - row_begin), kind, g->copy_stream);
    }
    if (e == cudaSuccess) e = cudaEventRecord(g->ev_copied, g->copy_stream);
    if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_fetch_async: ") + cudaGetErrorString(e)));
    g->copy_pending = true;
    return CLEORA_OK;
}

int cleora_fetch_nonzero_async(cleora_graph* g, float* out_rows, int32_t* out_ids, int64_t capacity, int64_t* n_rows,
                               int32_t out_on_device) {
    NvtxRange _nvtx("cleora_fetch_nonzero_async");
    if (!g || !n_rows) return usage("cleora_fetch_nonzero_async: NULL argument");
    if (!g->T[0]) return usage("cleora_fetch_nonzero_async: call cleora_init first");
    DeviceGuard guard(g->device);
    Status st = fetch_nonzero(g, out_rows, out_ids, capacity, n_rows, out_on_device, false);
    return st.good() ? CLEORA_OK : fail(st);
}

int cleora_fetch_nonzero(cleora_graph* g, float* out_rows, int32_t* out_ids, int64_t capacity, int64_t* n_rows,
                         int32_t out_on_device) {
    NvtxRange _nvtx("cleora_fetch_nonzero");
    if (!g || !n_rows) return usage("cleora_fetch_nonzero: NULL argument");
    if (!g->T[0]) return usage("cleora_fetch_nonzero: call cleora_init first");
    DeviceGuard guard(g->device);
    Status st = fetch_nonzero(g, out_rows, out_ids, capacity, n_rows, out_on_device, true);
    return st.good() ? CLEORA_OK : fail(st);
}

int cleora_merge_chunks(cleora_graph* const* chunks, int32_t n_chunks, float* out, int32_t out_on_device) {
    NvtxRange _nvtx("cleora_merge_chunks");
    if (!chunks || !out) return usage("cleora_merge_chunks: NULL argument");
    if (n_chunks < 1) return usage("cleora_merge_chunks: n_chunks must be >= 1");
    const cleora_graph* g0 = chunks[0];
    if (!g0) return usage("cleora_merge_chunks: NULL handle");
    for (int q = 0; q < n_chunks; q++) {
        const cleora_graph* g = chunks[q];
        if (!g) return usage("cleora_merge_chunks: NULL handle");
        if (g->device != g0->device || g->n != g0->n || g->d != g0->d || g->dp != g0->dp)
            return usage("cleora_merge_chunks: chunks differ in device, n_nodes or d");
        if (!g->occ) return usage("cleora_merge_chunks: a handle was built without n_chunks (no occurrence counts)");
        if (!g->T[0]) return usage("cleora_merge_chunks: a chunk is not initialised");
    }
    DeviceGuard guard(g0->device);
    cudaStream_t s = g0->stream;
    for (int q = 0; q < n_chunks; q++) {
        Status st0 = complete_t0(chunks[q]);
        if (!st0.good()) return fail(st0);
    }
    for (int q = 0; q < n_chunks; q++) order_after_side(chunks[q]);
    for (int q = 1; q < n_chunks; q++)
        if (chunks[q]->stream != s) {
            cudaError_t e = cudaStreamSynchronize(chunks[q]->stream);
            if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_merge_chunks: ") + cudaGetErrorString(e)));
        }
    std::vector<const void*> h_ptr(2 * (size_t)n_chunks);
    for (int q = 0; q < n_chunks; q++) {
        h_ptr[q] = chunks[q]->T[chunks[q]->cur];
        h_ptr[n_chunks + q] = chunks[q]->occ;
    }
    void* d_ptr = nullptr;
    float* stage = nullptr;
    const bool direct = out_on_device && g0->d == g0->dp;
    Status st = dalloc(&d_ptr, h_ptr.size() * sizeof(void*), s, "merge pointer table", kAllocTransient);
    if (st.good() && !direct) st = dalloc((void**)&stage, (size_t)g0->n * g0->dp * sizeof(float), s, "merge staging", kAllocTransient);
    cudaError_t e = cudaSuccess;
    if (st.good()) {
        e = cudaMemcpyAsync(d_ptr, h_ptr.data(), h_ptr.size() * sizeof(void*), cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) st = Status::make(4, std::string("cleora_merge_chunks: ") + cudaGetErrorString(e));
    }
    if (st.good())
        st = launch_merge(reinterpret_cast<const float* const*>(d_ptr),
                          reinterpret_cast<const int32_t* const*>(reinterpret_cast<const void* const*>(d_ptr) + n_chunks),
                          n_chunks, g0->n, g0->dp, direct ? out : stage, s);
    if (st.good() && !direct) {
        e = cudaMemcpy2DAsync(out, (size_t)g0->d * sizeof(float), stage, (size_t)g0->dp * sizeof(float),
                              (size_t)g0->d * sizeof(float), (size_t)g0->n,
                              out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) st = Status::make(4, std::string("cleora_merge_chunks: ") + cudaGetErrorString(e));
    }
    e = cudaStreamSynchronize(s);
    if (st.good() && e != cudaSuccess) st = Status::make(4, std::string("cleora_merge_chunks: ") + cudaGetErrorString(e));
    dfree(stage, s);
    dfree(d_ptr, s);
    if (!st.good()) return fail(st);
    return CLEORA_OK;
}

int cleora_reconstruct(const cleora_graph* g, const int32_t* new_idx, const int32_t* known_idx, const float* weight,
                       int64_t n_edges, int32_t n_new, int32_t inputs_on_device, float* out, int32_t out_on_device) {
    NvtxRange _nvtx("cleora_reconstruct");
    if (!g || !new_idx || !known_idx || !out) return usage("cleora_reconstruct: NULL argument");
    if (g->trimmed) return usage("cleora_reconstruct: the handle was trimmed (cleora_trim)");
    if (!g->T[0]) return usage("cleora_reconstruct: call cleora_init first");
    if (n_new < 1) return usage("cleora_reconstruct: n_new must be >= 1");
    if (n_edges < 1) return usage("cleora_reconstruct: n_edges must be >= 1");
    DeviceGuard guard(g->device);
    {
        Status st0 = complete_t0(g);
        if (!st0.good()) return fail(st0);
    }
    order_after_side(g);
    cudaStream_t s = g->stream;
    const int32_t N2 = std::max(n_new, g->n);   // row space of the new nodes' transition rows
    void *bs = nullptr, *bd = nullptr, *bw = nullptr;
    const int32_t* dsrc = new_idx;
    const int32_t* ddst = known_idx;
    const float* dw = weight;
    Status st = Status::ok();
    if (!inputs_on_device) {
        st = dalloc(&bs, n_edges * sizeof(int32_t), s, "reconstruct new_idx", kAllocTransient);
        if (st.good()) st = dalloc(&bd, n_edges * sizeof(int32_t), s, "reconstruct known_idx", kAllocTransient);
        if (st.good() && weight) st = dalloc(&bw, n_edges * sizeof(float), s, "reconstruct weight", kAllocTransient);
        if (st.good()) {
            cudaMemcpyAsync(bs, new_idx, n_edges * sizeof(int32_t), cudaMemcpyHostToDevice, s);
            cudaMemcpyAsync(bd, known_idx, n_edges * sizeof(int32_t), cudaMemcpyHostToDevice, s);
            if (weight) cudaMemcpyAsync(bw, weight, n_edges * sizeof(float), cudaMemcpyHostToDevice, s);
            dsrc = (const int32_t*)bs;
            ddst = (const int32_t*)bd;
            dw = (const float*)bw;
        }
    }
    BuildOut b;
    Schedule sc;
    float* Tnew = nullptr;
    float* parts = nullptr;
    if (st.good()) {
        BuildExtra bx;
        bx.dst_limit = g->n;                     // columns index this graph's rows
        // new_idx must lie in [0, n_new): validated as a row id below N2, then checked here
        st = build_csr(dsrc, ddst, dw, n_edges, N2, 1, s, &b, &bx);
    }
    if (st.good() && n_new < N2) {
        // rows in [n_new, N2) must be empty: a new_idx >= n_new is out of range
        int64_t tail[2] = {0, 0};
        st = read_small(&tail[0], b.row_ptr + n_new, sizeof(int64_t), s);
        if (st.good()) st = read_small(&tail[1], b.row_ptr + N2, sizeof(int64_t), s);
        if (st.good() && tail[1] != tail[0]) st = Status::make(3, "cleora_reconstruct: new_idx outside [0, n_new)");
    }
    if (st.good()) st = build_schedule(b.row_ptr, N2, 0, n_new, b.nnz, b.max_degree, g->heavy_thresh, g->chunk_rows, s, &sc);
    if (st.good()) st = dalloc((void**)&Tnew, (size_t)n_new * g->dp * sizeof(float), s, "reconstructed rows");
    if (st.good() && sc.n_slots_max > 0)
        st = dalloc((void**)&parts, (size_t)sc.n_slots_max * g->dp * sizeof(float), s, "reconstruct partials", kAllocTransient);
    if (st.good()) {
        SpmmArgs a;
        a.row_ptr = b.row_ptr;
        a.col = b.col;
        a.val = b.val;
        a.T_in = g->T[g->cur];
        a.T_out = Tnew;
        a.dp = g->dp;
        a.r0 = 0;
        a.r1 = n_new;
        a.heavy_thresh = g->heavy_thresh;
        a.items = sc.items;
        a.counts = sc.counts;
        a.n_items_max = sc.n_items_max;
        a.partials = parts;
        a.counters = sc.counters;
        a.work = sc.work;
        a.light_start = sc.light_start;
        a.cold_first = 0;
        a.n_peers = 0;
        for (int q = 0; q < kMaxPeers; q++) a.peer_out[q] = nullptr;
        a.skip_zero_rows = 0;
        a.csr_prefetch = 0;
        a.lazy_out = 0;
        a.scale_off = 0;
        a.ss_half = nullptr;
        a.drop_rows = nullptr;
        a.peer_mask = nullptr;
        a.gather_mode = g->gmode;
        a.pass = 0;
        st = launch_spmm_norm(a, s);
    }
    if (st.good()) {
        cudaError_t e = cudaMemcpy2DAsync(out, (size_t)g->d * sizeof(float), Tnew, (size_t)g->dp * sizeof(float),
                                          (size_t)g->d * sizeof(float), (size_t)n_new,
                                          out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = Status::make(4, std::string("cleora_reconstruct: ") + cudaGetErrorString(e));
    }
    cudaStreamSynchronize(s);
    dfree(parts, s);
    dfree(Tnew, s);
    dfree(sc.items, s);
    dfree(sc.counters, s);
    dfree(sc.work, s);
    dfree(sc.light_start, s);
    dfree(sc.counts, s);
    dfree(b.row_ptr, s);
    dfree(b.col, s);
    dfree(b.val, s);
    dfree(b.deg, s);
    dfree(b.d_scal, s);
    dfree(bs, s);
    dfree(bd, s);
    dfree(bw, s);
    if (!st.good()) return fail(st);
    return CLEORA_OK;
}

int cleora_fetch_replica(const cleora_graph* g, int32_t rank, int64_t row_begin, int64_t row_end, float* host_out) {
    NvtxRange _nvtx("cleora_fetch_replica");
    if (!g || !host_out) return usage("cleora_fetch_replica: NULL argument");
    if (g->trimmed && rank != g->rank) return usage("cleora_fetch_replica: the handle was trimmed (cleora_trim)");
    if (!g->T[0]) return usage("cleora_fetch_replica: call cleora_init first");
    if (g->xmode != X_LOOPBACK) {
        if (rank != g->rank) return usage("cleora_fetch_replica: only this rank's replica is local");
        return cleora_fetch(g, row_begin, row_end, host_out, 0);
    }
    if (rank < 0 || rank >= g->world) return usage("cleora_fetch_replica: rank outside [0, world)");
    if (row_begin < 0 || row_end > g->n || row_begin > row_end) return usage("cleora_fetch_replica: rows outside [0, N]");
    if (row_end == row_begin) return CLEORA_OK;
    DeviceGuard guard(g->device);
    {
        Status st0 = complete_t0(g);
        if (!st0.good()) return fail(st0);
    }
    order_after_side(g);
    const float* src = g->rep[rank][g->cur] + row_begin * (int64_t)g->dp;
    cudaError_t e = cudaMemcpy2DAsync(host_out, (size_t)g->d * sizeof(float), src, (size_t)g->dp * sizeof(float),
                                      (size_t)g->d * sizeof(float), (size_t)(row_end - row_begin),
                                      cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_fetch_replica: ") + cudaGetErrorString(e)));
    return CLEORA_OK;
}

int cleora_set_rows(cleora_graph* g, int64_t row_begin, int64_t row_end, const float* host_in) {
    NvtxRange _nvtx("cleora_set_rows");
    if (!g || !host_in) return usage("cleora_set_rows: NULL argument");
    if (g->trimmed) return usage("cleora_set_rows: the handle was trimmed (cleora_trim)");
    if (!g->T[0]) return usage("cleora_set_rows: call cleora_init first");
    if (row_begin < 0 || row_end > g->n || row_begin > row_end) return usage("cleora_set_rows: rows outside [0, N]");
    if (row_end == row_begin) return CLEORA_OK;
    DeviceGuard guard(g->device);
    {
        Status st0 = complete_t0(g);
        if (!st0.good()) return fail(st0);
    }
    order_after_side(g);
    // loopback: every emulated rank sets the same rows in its own replica
    const int nrep = g->xmode == X_LOOPBACK ? g->world : 1;
    cudaError_t e = cudaSuccess;
    for (int p = 0; p < nrep && e == cudaSuccess; p++) {
        float* base = g->xmode == X_LOOPBACK ? g->rep[p][g->cur] : g->T[g->cur];
        e = cudaMemcpy2DAsync(base + row_begin * (int64_t)g->dp, (size_t)g->dp * sizeof(float), host_in,
                              (size_t)g->d * sizeof(float), (size_t)g->d * sizeof(float),
                              (size_t)(row_end - row_begin), cudaMemcpyHostToDevice, g->stream);
    }
    g->zclean[g->cur] = false;
    g->rows_set = true;
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_set_rows: ") + cudaGetErrorString(e)));
    return CLEORA_OK;
}

int cleora_fetch_csr(const cleora_graph* g, int64_t* row_ptr, int32_t* col, float* val, double* deg) {
    NvtxRange _nvtx("cleora_fetch_csr");
    if (!g) return usage("cleora_fetch_csr: graph is NULL");
    if (g->trimmed) return usage("cleora_fetch_csr: the handle was trimmed (cleora_trim)");
    DeviceGuard guard(g->device);
    const Csr& c = g->own();
    cudaError_t e = cudaSuccess;
    if (row_ptr && e == cudaSuccess)
        e = cudaMemcpyAsync(row_ptr, c.row_ptr, ((size_t)g->n + 1) * 8, cudaMemcpyDeviceToHost, g->stream);
    if (col && e == cudaSuccess && c.nnz > 0)
        e = cudaMemcpyAsync(col, c.col, (size_t)c.nnz * 4, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (col && e == cudaSuccess)
        for (int64_t k = 0; k < c.nnz; k++) col[k] &= kColMask;     // drop the hot-row tags
    if (val && e == cudaSuccess && c.nnz > 0)
        e = cudaMemcpyAsync(val, c.val, (size_t)c.nnz * 4, cudaMemcpyDeviceToHost, g->stream);
    if (deg && e == cudaSuccess) e = cudaMemcpyAsync(deg, c.deg, (size_t)g->n * 8, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_fetch_csr: ") + cudaGetErrorString(e)));
    return CLEORA_OK;
}

int cleora_info(cleora_graph* g, cleora_info_t* o) {
    if (!g || !o) return usage("cleora_info: NULL argument");
    memset(o, 0, sizeof *o);
    o->n_nodes = g->n;
    o->nnz = g->nnz;
    o->n_edges_in = g->n_edges_in;
    o->d = g->d;
    o->d_stride = g->dp;
    o->iterations = g->iters;
    o->zero_rows = g->zero_rows;
    o->max_degree = g->max_degree;
    if (g->sched.counts && g->sched.n_items < 0) {      // schedule counts: on the device until asked for
        DeviceGuard g0(g->device);
        int64_t c[4] = {0, 0, 0, 0};
        Status s = read_small(c, g->sched.counts, sizeof c, g->stream);
        if (!s.good()) return fail(s);
        g->sched.n_light = c[0];
        g->sched.n_items = c[1];
        g->sched.n_heavy_rows = c[2];
    }
    o->heavy_rows = std::max<int64_t>(0, g->sched.n_heavy_rows);
    o->heavy_items = std::max<int64_t>(0, g->sched.n_items);
    o->shard_begin = g->r0;
    o->shard_end = g->r1;
    o->rank = g->rank;
    o->world = g->world;
    o->hot_rows = g->n_hot;
    o->n_graphs = g->n_graphs;
    o->shard_nnz = g->csr.empty() ? 0 : g->own().nnz;
    o->launches_per_step = g->T[0] ? (g->halves ? 2 : 1) : 0;
    o->referenced_rows = g->n_ref;
    o->exchange = g->xmode;
    o->device_bytes = g->bytes + ((g->T[0] ? 1 : 0) + (g->T[1] ? 1 : 0)) * (int64_t)g->n * g->dp * 4 +
                      (int64_t)g->partials_floats * 4 +
                      g->sched.n_items_max * (int64_t)sizeof(HeavyItem) + g->sched.n_slots_max * 4 +
                      (g->sched.light_start ? (g->r1 - g->r0 + 1) * 8 : 0);
    DeviceGuard guard(g->device);
    cudaError_t e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_info: ") + cudaGetErrorString(e)));
    return CLEORA_OK;
}

int cleora_stats(cleora_graph* g, cleora_stats_t* o, int32_t reset) {
    if (!g || !o) return usage("cleora_stats: NULL argument");
    DeviceGuard guard(g->device);
    Status s = collect_timing(g);
    if (!s.good()) return fail(s);
    o->spmm_launches = g->n_spmm;
    o->spmm_ms_total = g->ms_spmm;
    o->spmm_ms_min = g->n_spmm ? g->ms_min : 0.0;
    o->spmm_ms_max = g->ms_max;
    o->exchange_launches = g->n_x;
    o->exchange_ms_total = g->ms_x;
    if (reset) {
        g->n_spmm = g->n_x = 0;
        g->ms_spmm = g->ms_x = g->ms_max = 0;
        g->ms_min = 1e300;
    }
    return CLEORA_OK;
}

int cleora_trim(cleora_graph* g) {
    NvtxRange _nvtx("cleora_trim");
    if (!g) return usage("cleora_trim: graph is NULL");
    if (!g->T[0]) return usage("cleora_trim: call cleora_init first");
    if (g->trimmed) return CLEORA_OK;
    DeviceGuard guard(g->device);
    {
        Status st0 = complete_t0(g);
        if (!st0.good()) return fail(st0);
    }
    // no order_after_side here: an asynchronous fetch of T[cur] keeps running on the copy stream and
    // reads nothing freed below (T[cur] stays); copy_pending stays set, so later fetches, merges and
    // destroy still order after it.  (Waiting here made the handle's stream -- often shared with the
    // next graph's build -- queue behind the D2H copy: ADVICE r1.)
    close_peers(g);
    for (size_t p = 0; p < g->rep.size(); p++)
        if ((int)p != g->rank)
            for (int i = 0; i < 2; i++) {
                dfree(g->rep[p][i], g->stream);
                g->rep[p][i] = nullptr;
            }
    const int other = 1 - g->cur;
    dfree(g->T[other], g->stream);
    g->T[other] = nullptr;
    if (g->cur == 1) {          // the kept buffer becomes T[0] ("initialised" checks look at T[0])
        g->T[0] = g->T[1];
        g->T[1] = nullptr;
        g->cur = 0;
    }
    if (!g->rep.empty()) g->rep[g->rank] = {g->T[0], nullptr};
    dfree(g->lazy_buf, g->stream);
    g->lazy_buf = nullptr;
    dfree(g->partials, g->stream);
    g->partials = nullptr;
    g->partials_floats = 0;
    free_schedules(g);
    // keep the build scalars (cleora_info reads zero_rows / max_degree lazily from csr[0].d_scal)
    for (auto& c : g->csr) {
        dfree(c.row_ptr, g->stream);
        dfree(c.col, g->stream);
        dfree(c.val, g->stream);
        dfree(c.deg, g->stream);
        c.row_ptr = nullptr;
        c.col = nullptr;
        c.val = nullptr;
        c.deg = nullptr;
    }
    dfree(g->indeg, g->stream);
    g->indeg = nullptr;
    for (auto m : g->pmask) dfree(m, g->stream);
    g->pmask.clear();
    g->bytes = 0;
    g->trimmed = true;
    return CLEORA_OK;
}

int cleora_sync(const cleora_graph* g) {
    if (!g) return usage("cleora_sync: graph is NULL");
    DeviceGuard guard(g->device);
    cudaError_t e = cudaStreamSynchronize(g->stream);
    if (e == cudaSuccess && g->copy_stream) e = cudaStreamSynchronize(g->copy_stream);
    if (e != cudaSuccess) return fail(Status::make(4, std::string("cleora_sync: ") + cudaGetErrorString(e)));
    return CLEORA_OK;
}

void cleora_destroy(cleora_graph* g) {
    if (!g) return;
    DeviceGuard guard(g->device);
    if (g->stream) {
        cudaStreamSynchronize(g->stream);
        free_T(g);
        free_csr(g);
        dfree(g->indeg, g->stream);
        for (auto m : g->pmask) dfree(m, g->stream);
        g->pmask.clear();
        free_schedules(g);
        dfree(g->d_flag, g->stream);
        dfree(g->occ, g->stream);
        dfree(g->d_base, g->stream);
        cudaStreamSynchronize(g->stream);
    }
    for (auto& p : g->ev_spmm) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    for (auto& p : g->ev_x) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    for (auto e : g->ev_pool) cudaEventDestroy(e);
    if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
    if (g->ev_ready) cudaEventDestroy(g->ev_ready);
    if (g->ev_copied) cudaEventDestroy(g->ev_copied);
    // g->comm belongs to the process-wide cache (comm_get)
    if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
    delete g;
}

int cleora_probe_gather(int32_t device, int32_t row_bytes, int64_t table_bytes, int64_t n_gathers, double* gbs) {
    NvtxRange _nvtx("cleora_probe_gather");
    if (!gbs) return usage("cleora_probe_gather: gbs is NULL");
    if (table_bytes < row_bytes || n_gathers < 1 || n_gathers > INT32_MAX)
        return usage("cleora_probe_gather: table_bytes >= row_bytes and 1 <= n_gathers < 2^31 required");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(Status::make(4, "cleora_probe_gather: no CUDA device visible"));
    }
    DeviceGuard guard(device);
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
        return fail(Status::make(4, "cleora_probe_gather: stream"));
    Status st = probe_gather(row_bytes, table_bytes, n_gathers, s, gbs);
    cudaStreamDestroy(s);
    if (!st.good()) return fail(st);
    return CLEORA_OK;
}

int64_t cleora_ipc_opens(void) { return g_ipc_opens.load(); }

int64_t cleora_oom_fallbacks(void) { return g_oom_fallbacks.load(); }

int cleora_nccl_id_size(void) { return NCCL_UNIQUE_ID_BYTES; }

int cleora_nccl_get_unique_id(uint8_t* out128) {
    if (!out128) return usage("cleora_nccl_get_unique_id: NULL");
    Nccl& n = nccl();
    if (!n.ok) return fail(Status::make(4, "NCCL unavailable: " + n.why));
    ncclUniqueId id;
    ncclResult_t r = n.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(Status::make(4, std::string("ncclGetUniqueId: ") + n.GetErrorString(r)));
    memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
    return CLEORA_OK;
}

int cleora_plan_shards(const int64_t* row_ptr, int64_t n, int32_t world, int64_t* cuts) {
    if (!row_ptr || !cuts) return usage("cleora_plan_shards: NULL argument");
    if (n < 0 || world < 1) return usage("cleora_plan_shards: n >= 0 and world >= 1 required");
    const int64_t nnz = row_ptr[n];
    cuts[0] = 0;
    for (int p = 1; p < world; p++) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if ((__int128)row_ptr[mid] * world >= (__int128)p * nnz) hi = mid; else lo = mid + 1;
        }
        cuts[p] = lo;
    }
    cuts[world] = n;
    return CLEORA_OK;
}

}  // extern "C"
