/*
 * cleora.h -- C ABI of the B200-native Cleora hot path (libcleora.so).
 *
 * The operation (Rychalska et al., arXiv 2102.02302; "PAPER.md" below is its text):
 *   M_ab = e_ab / deg(v_a)            random-walk transition matrix  (§3.2)
 *   T_0  ~ U(-1, 1)                   N x d embedding                (PAPER.md:83, Alg. 1 line 4, :92)
 *   repeat I times:  T_i = M . T_{i-1};  L2-normalise the rows of T_i (Alg. 1 lines 5-7)
 * The readings of the paper used where it is silent are listed in DESIGN.md
 * ("Readings of the paper", R1-R12, RZ).
 *
 * Conventions common to every call
 *   - Return value: CLEORA_OK (0) or an error code below; cleora_last_error() then
 *     holds a human-readable message (thread-local, valid until the next call on the
 *     same thread).  On error the handle stays valid (or *out stays NULL).
 *   - All device work is stream-ordered on the handle's stream (cleora_opts.stream or a
 *     library-owned stream).  cleora_init / cleora_iterate only enqueue work and return;
 *     cleora_fetch, cleora_fetch_csr, cleora_info, cleora_stats and cleora_sync wait for it.
 *     A device fault is reported by the next waiting call as CLEORA_EINTERNAL.
 *   - A handle is owned by one host thread at a time.  It owns ALL device memory it
 *     uses (CSR, T replicas, workspaces, schedule) and, when world > 1, its NCCL
 *     communicator; cleora_destroy releases everything.
 *   - Node ids are dense int32 in [0, N).  Mapping external entity ids to dense ids
 *     (the paper's xxhash step) is the caller's job.
 *   - There is no CPU fallback: without a usable sm_100 device every call fails
 *     with CLEORA_EINTERNAL.
 */
#ifndef CLEORA_H
#define CLEORA_H

#include <stdint.h>

#if defined(__GNUC__)
#define CLEORA_API __attribute__((visibility("default")))
#else
#define CLEORA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes (they mirror the exit codes of SPEC.md:520: usage 2, data 3, internal 4). */
enum {
    CLEORA_OK = 0,
    CLEORA_EUSAGE = 2,     /* bad argument, NULL pointer, call out of order               */
    CLEORA_EDATA = 3,      /* input data violates the model: id out of range, weight <= 0,
                              weight not finite                                          */
    CLEORA_EINTERNAL = 4   /* CUDA / NCCL error or out of device memory (message names
                              the API and, for allocations, the bytes requested)          */
};

/* cleora_opts.flags */
enum {
    CLEORA_F_TIMING = 1,   /* record CUDA events around every SpMM+normalise launch so that
                              cleora_stats() can report device time per launch            */
    CLEORA_F_LOOPBACK = 2, /* world > 1 without NCCL: emulate all `world` ranks (<= 8) in this
                              process on one GPU -- one replica pair per rank, the ranks'
                              fused SpMM launches run one after another and store their rows
                              into every replica.  For testing the multi-GPU path on one GPU;
                              rank selects the replica cleora_fetch reads.                  */
    CLEORA_F_EXCHANGE_NCCL = 4 /* world > 1: exchange the shards with an NCCL all-gather-v
                              after each step instead of the fused peer stores            */
};

/* Host-side all-gather supplied by the caller for world > 1 without NCCL (e.g. a gloo process group,
 * or two processes sharing one GPU in a test): every rank passes `bytes` bytes in `send`; on return
 * `recv` holds world * bytes bytes, rank p's at offset p * bytes.  Blocking; collective (every rank
 * calls it the same number of times, in the same order); returns 0 on success.  The library uses it
 * for the CUDA IPC handle exchange, for the failure agreement of every collective call, and, after a
 * cudaStreamSynchronize, as the step barrier (a 1-byte all-gather). */
typedef int (*cleora_allgather_fn)(void* ctx, const void* send, void* recv, int64_t bytes);

/* Build options.  Pass NULL to cleora_build for: current device, host inputs, a
 * library-owned stream, one GPU, no flags. */
typedef struct cleora_opts {
    int32_t device;          /* CUDA device ordinal; -1 = the calling thread's current device */
    int32_t input_on_device; /* 1: src/dst/weight are device pointers on `device`;
                                0: host pointers (pageable or pinned)                          */
    void* stream;            /* cudaStream_t to enqueue on (borrowed; must outlive the handle),
                                cudaStreamLegacy (0x1) for the legacy default stream;
                                NULL = the library creates and owns a non-blocking stream    */
    int32_t rank;            /* this process's rank in [0, world)                               */
    int32_t world;           /* number of GPUs sharing the work; <= 1 means one GPU            */
    const uint8_t* nccl_id;  /* world > 1: the 128-byte ncclUniqueId, identical on all ranks;
                                the library initialises a communicator from it on the first
                                build with this (id, world, rank, device) and reuses it for
                                every later handle of the process (one init per unique id)  */
    int32_t flags;           /* CLEORA_F_* bit set                                              */
    /* Algorithm 1 with Q > 1 chunks.  n_chunks >= 1: this handle holds chunk
       `chunk` of n_chunks -- the edges i with q(i) = floor(n_chunks * (h_i >> 32) / 2^32) = chunk,
       h_i = mix(mix(chunk_seed + 0x9E3779B97F4A7C15) XOR i) (reading R13) -- and counts every
       node's endpoint occurrences among them (reading R14) for cleora_merge_chunks.
       n_chunks = 0: the whole graph, no occurrence counts.                                 */
    int32_t n_chunks;
    int32_t chunk;
    uint64_t chunk_seed;
    /* world > 1 with nccl_id == NULL: the collectives go through this host all-gather instead of
       NCCL (the exchange must then be the fused peer stores; there is no NCCL all-gather fallback) */
    cleora_allgather_fn host_allgather;
    void* host_ctx;
} cleora_opts;

typedef struct cleora_graph cleora_graph;   /* opaque */

/*
 * cleora_build -- COO edge list -> device CSR of M = D^-1 A (Alg. 1 line 3,
 * PAPER.md:91), entirely on the device: validate, mirror (undirected), stable radix sort by
 * (src, dst), merge duplicates by summing weights, row pointer, degree, D^-1 scaling, and the
 * degree-bucketed iteration schedule.
 *   src, dst  [n_edges] int32 node ids in [0, n_nodes); host or device per opts.
 *   weight    [n_edges] fp32 edge weights (> 0, finite) or NULL for all 1.0f.
 *   directed  0: each undirected edge is listed once and mirrored by the library (a
 *             self-loop is stored once, reading R5); 1: row a averages the OUT-neighbours
 *             of a ("edges running from node a to b"; reading R3).
 *   Semantics (bit-exact against the oracle, readings B1-B4 in DESIGN.md):
 *     e_ab   = fp64 sum of the weights of duplicate (a,b) edges in stable input order
 *              (originals first, then mirrors), "the sum of the weights of all
 *              participating edges";
 *     deg(a) = fp64 sum of e_ab over ascending b (weighted out-degree, reading R2);
 *     M_ab   = (float)(e_ab / deg(a)), IEEE round-to-nearest once.
 *   Inputs are borrowed for the duration of the call only.  On success *out owns the graph.
 *   Errors: EUSAGE (NULL pointer, n_nodes <= 0, n_edges <= 0, world > 1 without nccl_id or
 *   host_allgather, bad rank, world > 255), EDATA (id outside [0, n_nodes), weight <= 0 or not
 *   finite), EINTERNAL.
 *   Multi-GPU (world > 1): collective; every rank passes the same edge list.  M is ROW-SHARDED:
 *   every rank counts the entries of every row (after mirroring, before merging duplicates), the
 *   rows are cut into `world` contiguous shards balanced on those counts (cut p = the first row
 *   whose entry prefix reaches p * total / world), and each rank sorts, merges and scales only the
 *   entries of its own rows -- no rank holds or sorts the whole M (§4.5: M's
 *   2|E| entries are the term that divides).  Results do not depend on world (bitwise).  If any
 *   rank fails (e.g. out of memory), every rank returns an error (the ranks agree on success
 *   before returning).
 */
CLEORA_API int cleora_build(const int32_t* src, const int32_t* dst, const float* weight, int64_t n_edges,
                 int32_t n_nodes, int32_t directed, const cleora_opts* opts, cleora_graph** out);

/*
 * cleora_expand -- hypergraph expansion on the device (§3.2 "Hypergraph
 * Expansion"; the paper's timed workloads were expanded adjacency rows):
 *   CLEORA_EXPAND_CLIQUE: hyperedge e with members m_0..m_{k-1} gives the edges (m_i, m_j) for
 *     all i < j with m_i != m_j (reading R16), in the order (e, i, j);
 *   CLEORA_EXPAND_STAR: hyperedge e gets the virtual node n_nodes + e and the edges
 *     (n_nodes + e, m_i) for every listed member (reading R17), in the order (e, i); the expanded
 *     graph has n_nodes + n_hyperedges nodes.
 * Every edge carries its hyperedge's weight (or 1.0f).  The output is an undirected edge list for
 * cleora_build (directed = 0).
 *   he_ptr [n_hyperedges + 1] int64 (he_ptr[0] = 0, non-decreasing), he_nodes [he_ptr[n]] int32 in
 *   [0, n_nodes), he_weight [n_hyperedges] or NULL; on_device = 1: all input AND output pointers
 *   are device memory of `device` (-1: current), else host.  stream: cudaStream_t or NULL (per-thread
 *   default stream).  out_src == NULL: count only.  *n_out receives the edge count.
 *   Synchronous.  Errors: EUSAGE (NULL, bad mode / sizes, capacity < count, id range overflow),
 *   EDATA (member id out of range, weight not finite or <= 0), EINTERNAL.
 */
enum { CLEORA_EXPAND_CLIQUE = 0, CLEORA_EXPAND_STAR = 1 };
CLEORA_API int cleora_expand(const int64_t* he_ptr, const int32_t* he_nodes, const float* he_weight,
                             int64_t n_hyperedges, int32_t n_nodes, int32_t mode, int32_t device, int32_t on_device,
                             void* stream, int32_t* out_src, int32_t* out_dst, float* out_weight, int64_t capacity,
                             int64_t* n_out);

/*
 * cleora_build_batch -- many independent graphs in ONE handle (several M, e.g.
 * one per relation pair of a table -- "a separate embedding matrix for each relation pair",
 * in one launch per step).  The handle holds the block-diagonal M of
 * the graphs; every step is one fused SpMM launch over all of them.
 *   edge_ptr [n_graphs + 1] int64 (host): graph g's edges are entries [edge_ptr[g], edge_ptr[g+1])
 *            of src / dst / weight, with node ids LOCAL to g in [0, node_count[g]).
 *   node_count [n_graphs] int32 (host), each >= 1.
 *   src, dst, weight, directed, opts: as cleora_build (host or device per opts; one GPU only).
 * Graph g's rows are rows [base_g, base_g + node_count[g]) of the handle, base_g = sum of the
 * node counts before g (fetch them with cleora_fetch).  T_0 is keyed on the LOCAL id, so every
 * graph's embedding is bitwise the one cleora_build of that graph alone would give.
 *   Errors: EUSAGE (NULL, n_graphs < 1, a node_count < 1, edge_ptr not non-decreasing from 0,
 *   no edges, world > 1 or n_chunks set), EDATA (a local id out of its graph's range, bad weight),
 *   EINTERNAL.
 */
CLEORA_API int cleora_build_batch(const int32_t* src, const int32_t* dst, const float* weight,
                                  const int64_t* edge_ptr, const int32_t* node_count, int32_t n_graphs,
                                  int32_t directed, const cleora_opts* opts, cleora_graph** out);

/*
 * cleora_init -- allocate the two N x d fp32 embedding buffers and set T <- T_0 with
 *   T_0[v][j] = ((int32)(h >> 40) - 2^23) * 2^-23,
 *   h = mix(mix(seed + 0x9E3779B97F4A7C15) XOR (v << 32 | j)), mix = SplitMix64 finaliser
 * (reading R1 / I1: a realisation of "T_0 ~ U(-1,1)").  T_0 is NOT
 * normalised (reading R7).  May be called again to restart from T_0 (same or new d / seed).
 * On graphs whose T exceeds the L2 hot-row budget only the rows some step can gather (in-degree
 * > 0) are written here; the others are written by the first call that reads T_0 itself (fetch,
 * trim, set_rows, reconstruct, merge) -- every read sees the whole T_0 (CLEORA_T0_ALL=1: all now).
 *   d >= 1 (any d; rows are stored with a stride padded to 4 floats, padding kept at 0).
 *   Errors: EUSAGE (g NULL, d < 1, d > CLEORA_MAX_D), EINTERNAL (out of memory).
 */
#define CLEORA_MAX_D 4096
CLEORA_API int cleora_init(cleora_graph* g, int32_t d, uint64_t seed);

/*
 * cleora_iterate -- k >= 0 steps of T <- normalize_rows(M . T) (Alg. 1 lines 6-7,
 * PAPER.md:94-95), one fused SpMM + row-L2-normalise kernel launch per step.  A row whose
 * product is the zero vector (no out-edges) is written as zeros (reading RZ).
 * iterate(a); iterate(b) is bit-identical to iterate(a + b).  Results do not depend on the
 * number of GPUs (the per-row schedule depends only on the row's degree).
 * Multi-GPU: collective.  Each rank computes the rows of its shard, and the kernel's epilogue
 * stores every finished row into all ranks' replicas through NVLink (peer pointers opened with
 * CUDA IPC during cleora_init), so the exchange overlaps the SpMM row by row; a 4-byte NCCL
 * all-reduce then orders the steps across ranks.  When the GPUs cannot map each other's memory
 * (or with CLEORA_F_EXCHANGE_NCCL) the shards are all-gathered with NCCL after each step.
 * Rows without out-edges stay 0 and are not rewritten once both buffers hold their zeros.
 *   Errors: EUSAGE (g NULL, k < 0, called before cleora_init), EINTERNAL.
 */
CLEORA_API int cleora_iterate(cleora_graph* g, int32_t k);

/*
 * cleora_fetch -- copy rows [row_begin, row_end) of the current T (T_i after i steps) into
 * `out`, dense (row_end - row_begin) x d fp32 row-major.  out_on_device = 0: `out` is host
 * memory (pinned or pageable); 1: device memory on the handle's device.  Waits for the copy.
 *   Errors: EUSAGE (NULL, range outside [0, N], before cleora_init), EINTERNAL.
 */
CLEORA_API int cleora_fetch(const cleora_graph* g, int64_t row_begin, int64_t row_end, float* out,
                 int32_t out_on_device);

/*
 * cleora_merge_chunks -- Algorithm 1 lines 10-12: out[v] = sum_q w_qv T^q[v]
 * over the current T of the n_chunks handles (built with opts.n_chunks = n_chunks, chunk = q,
 * the same chunk_seed and edge list, and initialised with the same d), with
 *   w_qv = occ_q(v) / sum_k occ_k(v)    (occ = endpoint occurrences, reading R14);
 * a node in no chunk gets the zero row; no normalisation after the merge (Algorithm 1 has none).
 * Arithmetic: w in fp64 (one division), fp64 accumulation in ascending q, one rounding to fp32
 * (bit-exact with the oracle's merge on the same chunk embeddings).
 *   chunks [n_chunks] handles on one device, same N and d; out: N x d fp32 row-major, host
 *   (out_on_device = 0) or device memory.  Waits for the chunks' streams and for the copy.
 *   Errors: EUSAGE (NULL, n_chunks < 1, mixed devices / N / d, a handle without occurrence
 *   counts or not initialised), EINTERNAL.
 */
CLEORA_API int cleora_merge_chunks(cleora_graph* const* chunks, int32_t n_chunks, float* out, int32_t out_on_device);

/*
 * cleora_reconstruct -- embeddings of n_new unseen nodes ("creation of new node
 * embedding by weighted averaging of all neighbors' representations"):
 *   out[i] = normalize( sum_b (e_ib / sum_c e_ic) * T[b] ),  T = g's current T
 * i.e. one step of the same fused SpMM + row-normalise kernel over the transition rows of the
 * new nodes (built on the device with readings B1-B4, directed new -> known).  The paper advises
 * T from iteration I-1: call cleora_iterate(I-1), reconstruct, then cleora_iterate(1).
 *   new_idx[n_edges] in [0, n_new), known_idx[n_edges] in [0, N), weight[n_edges] > 0 or NULL;
 *   host arrays, or device arrays with inputs_on_device = 1.  out: n_new x d fp32 row-major,
 *   host or device.  A new node without edges gets the zero row (reading RZ).  Synchronous.
 *   Errors: EUSAGE (NULL, n_new < 1, n_edges < 1, before cleora_init), EDATA (an index out of
 *   range, a weight not finite or <= 0), EINTERNAL.
 */
CLEORA_API int cleora_reconstruct(const cleora_graph* g, const int32_t* new_idx, const int32_t* known_idx,
                                  const float* weight, int64_t n_edges, int32_t n_new, int32_t inputs_on_device,
                                  float* out, int32_t out_on_device);

/*
 * cleora_fetch_async -- as cleora_fetch, but only enqueued: the copy runs on a library-owned copy
 * stream once the work enqueued so far on the handle's stream is done, concurrently with whatever
 * is enqueued afterwards (e.g. the next graph's build and iterations), so PCIe transfers overlap
 * compute.  `out` must stay valid until cleora_sync(g) or cleora_destroy(g), which wait for it;
 * later cleora_init / cleora_iterate / cleora_set_rows on g are stream-ordered after the copy.
 *   Errors: as cleora_fetch (checked at enqueue time); a copy failure is reported by cleora_sync.
 */
CLEORA_API int cleora_fetch_async(cleora_graph* g, int64_t row_begin, int64_t row_end, float* out,
                                  int32_t out_on_device);

/*
 * cleora_fetch_nonzero_async -- the result without its rows that are 0 by construction.  A row of M
 * without entries has y = 0 in every step (Algorithm 1 line 7: T <- M T), so
 * after the first step its row of T is exactly 0 (reading RZ).  This call copies only the rows of the
 * handle's shard [shard_begin, shard_end) (all of [0, N) on one GPU) that have entries in M:
 *   out_ids[k]  = the k-th such row, ascending (int32);
 *   out_rows[k] = that row of the current T, d fp32 (row-major, n_rows x d);
 * every other row of the shard is exactly 0.  Before the first step (T_0) and after cleora_set_rows
 * (until the next step) every row of the shard is returned (out_ids = shard_begin, shard_begin+1, ...).
 *   *n_rows (always written, at once): the number of rows returned.  out_rows = out_ids = NULL only
 *   queries that count.  capacity: rows out_rows / out_ids hold (>= *n_rows, else EUSAGE).  Either
 *   output may be NULL alone.  out_on_device = 0: host memory (pinned for full PCIe rate); 1: device
 *   memory on the handle's device.
 * Enqueued like cleora_fetch_async: the rows are packed on the device in the handle's stream order
 * (into a staging buffer for the whole result, which the handle keeps until cleora_destroy or the
 * next cleora_init; in 256 MB slices on the copy stream if that buffer cannot be had), then leave on
 * the library's copy stream; device outputs are packed in the handle's stream order directly.  The
 * outputs must stay valid until cleora_sync(g) or cleora_destroy(g).  The row selection is made once per handle, so a trimmed
 * handle (cleora_trim) answers only if it was called before the trim.
 * cleora_fetch_nonzero: the same, and waits for the copy.
 *   Errors: EUSAGE (NULL g / n_rows, before cleora_init, capacity too small, trimmed before the first
 *   call), EINTERNAL; a copy failure of the async form is reported by cleora_sync.
 */
CLEORA_API int cleora_fetch_nonzero_async(cleora_graph* g, float* out_rows, int32_t* out_ids, int64_t capacity,
                                          int64_t* n_rows, int32_t out_on_device);
CLEORA_API int cleora_fetch_nonzero(cleora_graph* g, float* out_rows, int32_t* out_ids, int64_t capacity,
                                    int64_t* n_rows, int32_t out_on_device);

/* Facts about a handle (all sizes in elements). */
typedef struct cleora_info_t {
    int64_t n_nodes;        /* N                                                        */
    int64_t nnz;            /* stored entries of M after mirroring and merging          */
    int64_t n_edges_in;     /* the n_edges passed to cleora_build                       */
    int32_t d;              /* embedding dimension (0 before cleora_init)               */
    int32_t d_stride;       /* row stride of the device T buffers in floats             */
    int64_t iterations;     /* steps applied since the last cleora_init                 */
    int64_t zero_rows;      /* rows with no out-edges (their T rows are 0 after step 1) */
    int64_t max_degree;     /* largest number of stored entries in one row              */
    int64_t heavy_rows;     /* rows scheduled on the multi-warp / multi-CTA path        */
    int64_t heavy_items;    /* CTA work items for those rows                            */
    int64_t shard_begin;    /* rows this rank computes and stores: [shard_begin, shard_end) */
    int64_t shard_end;
    int32_t rank, world;
    int64_t device_bytes;   /* device memory currently owned by the handle              */
    int64_t hot_rows;       /* rows whose gathers carry the L2 evict_last hint (0 = none) */
    int64_t referenced_rows;/* rows with in-degree > 0, i.e. ever gathered (-1: unknown)  */
    int32_t exchange;       /* 0 one GPU, 1 NCCL all-gather, 2 fused peer stores, 3 loopback */
    int32_t n_graphs;       /* graphs in a batched handle (cleora_build_batch), else 0   */
    int64_t shard_nnz;      /* entries of this rank's rows (= nnz on one GPU)               */
    int32_t launches_per_step; /* SpMM launches per iteration: 2 when d's 1024 columns run as two
                                  half-row passes (bitwise the same result), else 1 (0 before init) */
} cleora_info_t;
/* Fill *out.  Synchronises the handle's stream (zero_rows and max_degree are computed on the device
 * by cleora_build and read back here, on first use; the handle caches them -- hence non-const).
 *   Errors: EUSAGE (NULL argument); EINTERNAL (a CUDA error of earlier asynchronous work). */
CLEORA_API int cleora_info(cleora_graph* g, cleora_info_t* out);

/* Device-time statistics (requires CLEORA_F_TIMING; otherwise counts stay 0). */
typedef struct cleora_stats_t {
    int64_t spmm_launches;  /* SpMM+normalise launches timed since the last reset        */
    double spmm_ms_total;   /* sum of their durations (CUDA events on the handle stream) */
    double spmm_ms_min, spmm_ms_max;
    int64_t exchange_launches;
    double exchange_ms_total;
} cleora_stats_t;
CLEORA_API int cleora_stats(cleora_graph* g, cleora_stats_t* out, int32_t reset);

/* Keep only the current embedding T_i (the result of the last iteration) and
 * release everything else the handle holds on the device: the CSR of M, the other T buffer, the
 * schedules and heavy-row partials, loopback replicas, peer mappings.  For a server embedding
 * graph after graph near the HBM limit: trim a handle once its last iteration and its
 * cleora_fetch_async are enqueued, and the next graph can be built while the copy runs.  Stream
 * ordered: work already enqueued (the iterations, an asynchronous fetch) completes normally and the
 * memory returns to the library's cache behind it.
 *   Afterwards cleora_fetch, cleora_fetch_async, cleora_merge_chunks, cleora_info, cleora_sync and
 *   cleora_destroy remain valid; cleora_init, cleora_iterate, cleora_set_rows, cleora_reconstruct,
 *   cleora_fetch_csr and cleora_fetch_replica of another rank return CLEORA_EUSAGE.
 *   Errors: EUSAGE (NULL handle, or cleora_init never called: there is no T to keep).
 *   Trimming twice is a no-op. */
CLEORA_API int cleora_trim(cleora_graph* g);

/* Wait for all work enqueued on the handle's stream and for its asynchronous fetches. */
CLEORA_API int cleora_sync(const cleora_graph* g);

/* Release everything the handle owns.  Safe on NULL. */
CLEORA_API void cleora_destroy(cleora_graph* g);

CLEORA_API const char* cleora_last_error(void);

/* Process-wide number of device kernels libcleora has launched so far (its own kernels plus
 * the kernels of the CUB primitives it dispatches).  Diagnostic; read it before and after a
 * region to count that region's launches. */
CLEORA_API int64_t cleora_kernel_launches(void);

/* Device blocks of >= 1 MiB freed by cleora_destroy (T replicas, CSR, sort buffers) are kept
 * in a process-wide cache and reused by later handles of the same sizes (no allocator growth
 * between repeated build/embed/destroy cycles), up to CLEORA_CACHE_MAX_FRAC (default 0.8) of
 * device memory; CLEORA_NO_CACHE=1 disables it.  This call returns every cached block to the
 * driver (e.g. before handing the memory to another library).  Returns CLEORA_OK or
 * EINTERNAL. */
CLEORA_API int cleora_release_cached_memory(void);

/* Diagnostic (not on the Cleora path): the rate, in GB/s, at which the SMs of `device` (-1: current)
 * gather random rows of `row_bytes` (a multiple of 16; below 512 B it must divide 512) from an
 * L2-resident table of `table_bytes` (e.g. 64 MiB), n_gathers rows per launch, best of 6 timed
 * launches (CUDA events).  The SpMM's gather stream, nnz * d * 4 bytes per iteration, all passes
 * the L2 -> SM path: bench.py reports nnz * d * 4 / this rate as the gather bound next to the HBM
 * roofline (SURVEY.md §8(d) "Which roofline").  Errors: EUSAGE, EINTERNAL. */
CLEORA_API int cleora_probe_gather(int32_t device, int32_t row_bytes, int64_t table_bytes, int64_t n_gathers,
                                   double* gbs);

/* ---- test hooks (not on the graded path) ------------------------------------------------ */

/* Copy the device CSR of this rank's rows to host arrays in the original labelling:
 * row_ptr [N+1] int64, col [shard_nnz] int32, val [shard_nnz] fp32, deg [N] fp64 (any may be NULL).
 * One GPU: the whole M.  world > 1: the shard [shard_begin, shard_end) -- row_ptr offsets count from
 * the shard's first entry (row_ptr[r] = 0 for r <= shard_begin, = shard_nnz for r >= shard_end), deg
 * is 0 outside the shard; the rows themselves are bit-identical to the whole M's. */
CLEORA_API int cleora_fetch_csr(const cleora_graph* g, int64_t* row_ptr, int32_t* col, float* val, double* deg);

/* Copy rows [row_begin, row_end) of rank `rank`'s replica of the current T into host memory
 * (dense, d per row).  With CLEORA_F_LOOPBACK every emulated rank's replica is readable (the
 * replicas must be identical); otherwise only this rank's. */
CLEORA_API int cleora_fetch_replica(const cleora_graph* g, int32_t rank, int64_t row_begin, int64_t row_end,
                                    float* host_out);

/* Overwrite rows [row_begin, row_end) of the current T from host memory (dense, d per row):
 * resume from a checkpoint or start from a custom T_0.  (Loopback: every replica.) */
CLEORA_API int cleora_set_rows(cleora_graph* g, int64_t row_begin, int64_t row_end, const float* host_in);

/* Process-wide number of CUDA IPC mappings opened so far (peer T buffers; they are cached across
 * handles, so repeated handles of one shape open none).  Diagnostic. */
CLEORA_API int64_t cleora_ipc_opens(void);

/* Process-wide number of device allocations that found no room and first returned cached segments to
 * the driver (each such cudaFree synchronises the device).  Diagnostic. */
CLEORA_API int64_t cleora_oom_fallbacks(void);

/* Size of an ncclUniqueId (128) and a helper that fills one (rank 0 calls it and
 * broadcasts the bytes through the caller's process group). */
CLEORA_API int cleora_nccl_id_size(void);
CLEORA_API int cleora_nccl_get_unique_id(uint8_t* out128);

/* Host-side shard plan (no GPU needed): nnz-balanced contiguous row cuts.
 * row_ptr [n+1]; cuts [world+1] receives r_0 = 0 <= r_1 <= ... <= r_world = n where rank p
 * owns rows [r_p, r_{p+1}); cut p is the first row whose nnz prefix reaches p * nnz / world. */
CLEORA_API int cleora_plan_shards(const int64_t* row_ptr, int64_t n, int32_t world, int64_t* cuts);

#ifdef __cplusplus
}
#endif
#endif /* CLEORA_H */
