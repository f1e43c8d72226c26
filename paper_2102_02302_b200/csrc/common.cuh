// common.cuh -- shared declarations of libcleora (the B200 product path).
// Nothing here is shared with oracle/ (task rule 3: the two share no code).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace cleora {

// ---------------------------------------------------------------- error plumbing
void set_error(const std::string& msg);     // thread-local message for cleora_last_error()

struct Status {
    int code = 0;
    std::string msg;
    static Status ok() { return Status(); }
    static Status make(int c, const std::string& m) { Status s; s.code = c; s.msg = m; return s; }
    bool good() const { return code == 0; }
};

#define CL_CUDA_TRY(expr)                                                                  \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return ::cleora::Status::make(4, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define CL_TRY(expr)                                                                       \
    do {                                                                                   \
        ::cleora::Status _s = (expr);                                                      \
        if (!_s.good()) return _s;                                                         \
    } while (0)

// Read `bytes` (<= 4096) of device memory into host memory, in stream order, then wait for the
// stream.  A kernel stores them into mapped pinned memory, so the read never queues behind a large
// device-to-host DMA on the copy engine (cleora_fetch_async of another handle).
Status read_small(void* h_dst, const void* d_src, size_t bytes, cudaStream_t s);
constexpr int kMaxSmallReads = 4;
struct SmallRead {
    void* h_dst;
    const void* d_src;
    size_t bytes;
};
Status read_small_n(const SmallRead* r, int n, cudaStream_t s);

// Host-side phase trace (stderr) when CLEORA_TRACE is set; `sync` waits for the stream first.
void trace(const char* what, cudaStream_t s, bool sync);

// Process-wide launch counter (cleora_kernel_launches).
void count_launches(int64_t n);

// ---------------------------------------------------------------- device buffers
// Stream-ordered allocation from the device's default pool (release threshold raised so
// repeated build/destroy cycles do not return memory to the driver).
// flags: kAllocBase -- at the base of a cudaMalloc segment (CUDA IPC exports whole allocations);
// kAllocTransient -- freed before the API call returns (a hint: the cache serves both alike, api.cu;
// small builds carve such buffers out of one arena, build.cu)
// kAllocNoEvict -- on out-of-memory fail at once instead of releasing cached segments
enum { kAllocBase = 1, kAllocTransient = 2, kAllocNoEvict = 4 };
Status dalloc(void** p, size_t bytes, cudaStream_t s, const char* what, int flags = 0);
void dfree(void* p, cudaStream_t s);

// fetch.cu: the rows of [r0, r1) with entries in M (all = every row), ascending, into ids[0 .. n);
// and the packing of T rows ids[0 .. n) into dense rows of d floats (cleora_fetch_nonzero)
Status select_rows_with_entries(const int64_t* row_ptr, int64_t r0, int64_t r1, bool all, int32_t* ids,
                                cudaStream_t s);
Status pack_rows(const float* T, int32_t dp, int32_t d, const int32_t* ids, int64_t n, float* out, cudaStream_t s);

// SplitMix64 output function (the mixer of the T_0 hash, reading R1, and of the chunk
// assignment, reading R13).
__host__ __device__ __forceinline__ uint64_t sm64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------- schedule
// A CTA work item of the heavy path: entries [k0, k1) of row `row`, which is part `part`
// of `nparts` of that row.  Rows of several parts: the item's partial vector lives at partials +
// slot * dp (the row's parts have consecutive slots), the row's completion counter at
// counters[slot - part]; single-part rows need neither (slot = -1).
struct HeavyItem {
    int64_t k0, k1;
    int32_t row, part, nparts, slot;
};
static_assert(sizeof(HeavyItem) == 32, "HeavyItem layout");

constexpr int kWarpsPerCta = 8;     // 256 threads
constexpr int kMaxPeers = 7;        // other replicas a launch writes into (8 GPUs per box)
constexpr int kMaxDevices = 64;     // per-device launch configuration tables
constexpr int kMaxV = 8;            // float4 per lane per column slice (slice = 1024 floats)

struct SpmmArgs {
    const int64_t* row_ptr;
    const int32_t* col;     // column ids; bit 31 = "hot" tag (hot_tag below), masked on use
    const float* val;
    const float* T_in;
    float* T_out;
    int32_t dp;             // row stride in floats (multiple of 4)
    int64_t r0, r1;         // rows this launch computes on the light path (shard)
    int32_t heavy_thresh;   // rows with more entries than this are on the heavy path
    const HeavyItem* items;
    const int64_t* counts;  // schedule counts on the device (Schedule::counts): [0] light chunks, [1] items
    int64_t n_items_max;    // host upper bound of counts[1] (0: no heavy rows possible)
    float* partials;        // partial-vector slots * dp floats
    unsigned* counters;     // completion counters of multi-part rows, 0 between launches
    unsigned* work;         // 3 work tickets of the persistent kernel, 0 between launches
    const int64_t* light_start;   // light chunks (Schedule::light_start)
    int32_t cold_first;     // TMA path: gathers of non-hot rows with evict_first (else evict_normal)
    // Fused exchange (multi-GPU): every finished row is also stored into the T_out replicas of
    // the other ranks -- NVLink peer pointers opened through CUDA IPC, or, in loopback
    // emulation, the other local replicas -- so the all-gather overlaps the SpMM row by row.
    int32_t n_peers;
    float* peer_out[kMaxPeers];
    // non-NULL: a non-empty row r goes to peer q only when bit q of peer_mask[r] is set (a row of that
    // peer's shard gathers r); the rest of the exchange is deferred to the last step of an iterate
    // call, which sends every row to every peer
    const uint8_t* peer_mask;
    // Rows without entries are already 0 in T_out (written by an earlier iteration): skip them.
    int32_t skip_zero_rows;
    int32_t csr_prefetch;   // register kernel: L1-prefetch each light chunk's CSR words
    int32_t gather_mode;    // kGather* for this dp (gather_mode(dp), read once by cleora_init)
    // Half-row passes (dp = 1024 only; spmm_tma.cu): 0 = whole rows; 1 = columns [0, 512), written
    // unnormalised into T_out and nowhere else; 2 = columns [512, 1024), then the whole row is finished
    // from T_out's first half -- bitwise the whole-row result (see spmm_tma.cu)
    int32_t pass;
    // Lazy normalisation between the half-row steps of one iterate call (spmm_tma.cu, reading R21).
    // ss_half non-NULL (a lazy step): pass 1 stores each light row's fp64 sum of squares over the first
    // half and sends that half, unnormalised, to the peers too; lazy_out (its pass 2): y is written
    // unnormalised and 1 / ||y|| goes to the row scales, which sit scale_off floats behind the rows of
    // T_out and of every peer replica.  The next step gathers those rows with weights that carry the
    // scales (launch_lazy_vals), so its kernels need nothing else.
    int32_t lazy_out;
    int64_t scale_off;
    double* ss_half;
    // A lazy step only (non-NULL only with ss_half): a row with entries whose drop_rows (in-degree) is 0
    // is never gathered, so no later step of the call reads it and the call's last step computes it
    // anew -- its rows, row scale and first-half sum are not stored (c4: 450k rows, 1.85 GB per step)
    const int32_t* drop_rows;
};

// A lazy step's row scale: into T_out's scales and every peer replica's (the row's peer mask, as its rows)
__device__ __forceinline__ void put_scale(const SpmmArgs& a, int64_t row, float v, bool empty = false) {
    a.T_out[a.scale_off + row] = v;
    if (a.n_peers > 0) {
        const unsigned m = (empty || !a.peer_mask) ? 0xffu : a.peer_mask[row];
        for (int p = 0; p < a.n_peers; p++)
            if ((m >> p) & 1u) a.peer_out[p][a.scale_off + row] = v;
    }
}

// Store float4 f of row `row` of the iteration's output into T_out and every peer replica.  `empty`:
// the row has no entries (its zeros always reach the peers, which then skip it like this rank does).
__device__ __forceinline__ void put_out4(const SpmmArgs& a, int64_t row, int f, const float4& v, bool empty = false) {
    const int64_t off = row * (int64_t)a.dp;
    __stcs(reinterpret_cast<float4*>(a.T_out + off) + f, v);
    if (a.n_peers > 0) {
        const unsigned m = (empty || !a.peer_mask) ? 0xffu : a.peer_mask[row];
        for (int p = 0; p < a.n_peers; p++)
            if ((m >> p) & 1u) __stcs(reinterpret_cast<float4*>(a.peer_out[p] + off) + f, v);
    }
}

// A CSR of M (or of one row shard of it) on the device
struct Csr {
    int64_t* row_ptr = nullptr;
    int32_t* col = nullptr;
    float* val = nullptr;
    double* deg = nullptr;
    unsigned long long* d_scal = nullptr;   // build scalars ([2] zero rows of its rows, [3] max degree)
    int64_t nnz = 0;
    int64_t zero_rows = 0, max_degree = 0;  // of its rows (read back with the build's verdict)
};

// build.cu
struct BuildOut {
    int64_t nnz = 0;
    int64_t* row_ptr = nullptr;
    int32_t* col = nullptr;
    float* val = nullptr;
    double* deg = nullptr;
    // device scalars of the build ([2] rows without entries, [3] largest row, [4] nnz); the caller
    // frees the buffer.  Their host copies come back with the build's one readback, after its last kernel.
    unsigned long long* d_scal = nullptr;
    int64_t zero_rows = 0, max_degree = 0;
};
// Optional parts of a build: keep only the edges of chunk `chunk` of `n_chunks` (Algorithm 1
// line 1, reading R13), count every node's endpoint occurrences among the kept edges (reading
// R14; `occ` int32[N], zeroed here), and require dst < dst_limit (inductive CSRs, whose columns
// index another graph's rows).
struct BuildExtra {
    int32_t n_chunks = 0, chunk = 0;
    uint64_t chunk_key = 0;     // sm64(chunk_seed + 0x9E3779B97F4A7C15)
    int32_t* occ = nullptr;
    int32_t dst_limit = -1;     // -1: N
    // row-sharded build: only rows [row_lo, row_hi) (row_hi = -1: all), whose entries (after mirroring,
    // before merging) number shard_entries; the edges were validated and occ counted by shard_plan
    int32_t row_lo = 0, row_hi = -1;
    int64_t shard_entries = 0;
};
Status build_csr(const int32_t* d_src, const int32_t* d_dst, const float* d_w, int64_t E, int32_t N,
                 int directed, cudaStream_t s, BuildOut* out, const BuildExtra* extra = nullptr);

// Light-row work units: chunks [light_start[c], light_start[c+1]) of at most kChunkRows
// consecutive rows whose entries start within one window of `chunk_entries` entries, so a
// ticket's work is bounded in rows (row pointers fit one register per lane) and in entries
// (no long tail behind a chunk of medium-degree rows).
constexpr int kChunkRows = 31;
// Built without a host round trip: the counts stay on the device (read by the SpMM kernels; read back
// only by cleora_info), the arrays are sized by host upper bounds.
struct Schedule {
    int64_t n_items_max = 0, n_slots_max = 0;   // host upper bounds: items, partial-vector slots
    int64_t n_heavy_rows = -1, n_items = -1, n_light = -1;   // host copies of counts, -1: not read yet
    HeavyItem* items = nullptr;
    unsigned* counters = nullptr;   // [n_slots_max]
    unsigned* work = nullptr;   // [4] persistent-kernel tickets
    int64_t* light_start = nullptr;   // [n_light + 1] (allocated for r1 - r0 + 1)
    int64_t* counts = nullptr;  // device: [0] light chunks, [1] items, [2] heavy rows, [3] partial slots
};
// nnz: entries of rows [r0, r1), max_degree: their longest row (upper bounds are enough)
Status build_schedule(const int64_t* d_row_ptr, int32_t N, int64_t r0, int64_t r1, int64_t nnz, int64_t max_degree,
                      int heavy_thresh, int chunk_rows, cudaStream_t s, Schedule* out);
// Row-sharded builds (world > 1): validate every edge, count every row's entries (mirrored, before
// merging), cut the rows into `world` shards balanced on those counts (cut p = first row whose entry
// prefix reaches p * total / world; h_cuts[world + 1]), h_ent[p] = entries before cut p, and the
// whole graph's in-degree (int32[N], device, caller frees) for the hot-row tags and the exchange's
// referenced-row flags.  extra: chunk filter and occ (counted here).  EDATA on a bad edge.
Status shard_plan(const int32_t* d_src, const int32_t* d_dst, const float* d_w, int64_t E, int32_t N, int directed,
                  const BuildExtra* extra, int world, cudaStream_t s, int64_t* h_cuts, int64_t* h_ent,
                  int32_t** d_indeg);
// need[v] = 1 if a row of this CSR (shard) gathers v, else 0 (N bytes)
Status need_flags(const int32_t* d_col, int64_t nnz, int32_t N, cudaStream_t s, uint8_t* d_need);
// mask[r] bit q = peer q needs row r, from the ranks' need arrays (need_all[p * N + r]); the peers of
// `rank` are the other ranks in rank order (the order of SpmmArgs::peer_out)
Status peer_masks(const uint8_t* d_need_all, int32_t N, int world, int rank, cudaStream_t s, uint8_t* d_mask);

// Hot-row tagging for L2 residency hints, in place: col[k] = (col[k] & 0x7fffffff) |
// (indeg(col[k]) >= 2^b) << 31, b the smallest power of two such that the hot rows' bytes fit
// `budget_bytes` (node ids are < 2^31, so bit 31 is free).  Returns the number of hot rows in
// *n_hot (0 => no row is tagged).  Every reader of col masks bit 31.
constexpr int32_t kColMask = 0x7fffffff;
Status hot_tag(int32_t* d_col, int64_t nnz, int32_t N, int64_t row_bytes, int64_t budget_bytes,
               cudaStream_t s, int64_t* n_hot, int64_t* n_ref /* rows with in-degree > 0, or NULL */,
               const int64_t* d_row_ptr_sym /* undirected graphs: in-degree = row length, else NULL */,
               const int32_t* d_indeg = nullptr /* precomputed in-degree (row-sharded builds), else NULL */);

// chunks.cu: out = sum_q w_qv Tq[q] (Algorithm 1 lines 10-12); d_Tq / d_occ are device arrays
// of Q device pointers; out and every Tq[q] are N x dp
Status launch_merge(const float* const* d_Tq, const int32_t* const* d_occ, int Q, int64_t N, int dp, float* d_out,
                    cudaStream_t s);

// expand.cu: hypergraph -> edge list (mode 0 clique, 1 star); all pointers device; d_os == NULL
// counts only (*n_out); EUSAGE when capacity < *n_out
Status expand_hypergraph(const int64_t* d_ptr, const int32_t* d_nodes, const float* d_w, int64_t n_he, int64_t n_members,
                         int32_t n_nodes, int mode, cudaStream_t s, int32_t* d_os, int32_t* d_od, float* d_ow,
                         int64_t capacity, int64_t* n_out);

// init.cu
// sel (NULL: every row): an in-degree array; sel_mode 1 writes only the rows with in-degree > 0 (the
// rows a step can gather), 2 only the others (completing T_0 when it is read before any step)
Status launch_hash_init(float* T, int64_t N, int32_t d, int32_t dp, uint64_t seed, cudaStream_t s,
                        const int64_t* d_base = nullptr, int32_t n_graphs = 0, const int32_t* sel = nullptr,
                        int sel_mode = 0);
// In-degree of every column of a CSR (undirected: the row lengths), device int32[N], long-lived
Status in_degree(const int32_t* d_col, int64_t nnz, int32_t N, const int64_t* d_row_ptr_sym, cudaStream_t s,
                 int32_t** out);

// build.cu, batched handles: global ids = local ids + base[graph of the edge]; edge_ptr and
// base are [n_graphs + 1] device arrays.  Returns EDATA (with the first bad edge) for a local id
// outside its graph.
Status batch_global_ids(const int32_t* d_src, const int32_t* d_dst, int64_t E, const int64_t* d_edge_ptr,
                        const int64_t* d_base, int32_t n_graphs, cudaStream_t s, int32_t* d_gsrc, int32_t* d_gdst);

// spmm_norm.cu (register gathers; any d) and spmm_tma.cu (TMA bulk gathers; dp <= 1024)
Status launch_spmm_norm(const SpmmArgs& a, cudaStream_t s);
enum { kGatherLdg = 0, kGatherBulk = 1, kGatherAsync = 2 };
int gather_mode(int dp);          // which gather engine serves rows of dp floats
// probe.cu: random-row gather rate (GB/s) from an L2-resident table of table_bytes (diagnostic)
Status probe_gather(int row_bytes, int64_t table_bytes, int64_t n_gathers, cudaStream_t s, double* gbs);
bool tma_path_supported(int dp);  // gather_mode(dp) uses the shared-memory ring kernel
Status launch_spmm_tma(const SpmmArgs& a, cudaStream_t s);
// Lazy normalisation (reading R21): val_out[e] = fp32_rn(val[e] * scale[col[e]]) for the step that
// gathers unnormalised rows -- the scales are folded into the weights before the SpMM, so its gather
// stream carries no scale lookups (spmm_tma.cu)
Status launch_lazy_vals(const float* val, const int32_t* col, const float* scale, int64_t nnz, float* val_out,
                        cudaStream_t s);

}  // namespace cleora
