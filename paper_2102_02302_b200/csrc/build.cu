// build.cu -- on-device construction of M = D^-1 A in CSR and of the iteration schedule.
//
// PAPER.md:79-81 (§3.2 "Embedding"): M_ab = e_ab / deg(v_a), e_ab = number of a->b edges, or
// the sum of their weights.  Algorithm 1 line 3 builds M per chunk; here Q = 1.
// Bit-exact contract with the oracle (readings B1-B4):
//   B1 entries = originals in input order, then mirrors (undirected, u != v) in input order;
//      STABLE sort by (src, dst)                      -> cub radix sort (stable) on src*N+dst, the
//                                                        weights as payload
//   B2 e_ab   = fp64 sum in that stable order        -> one thread per run, sequential
//   B3 deg(a) = fp64 sum of e_ab over ascending b     -> one warp per row, sequential fold
//   B4 val    = fp32_rn(e_ab / deg(a))                -> IEEE double divide, one rounding
// This translation unit must not be compiled with --use_fast_math.
#include <algorithm>
#include <mutex>

#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"

namespace cleora {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n, int per_thread = 1) {
    int64_t b = (n + (int64_t)kThreads * per_thread - 1) / ((int64_t)kThreads * per_thread);
    if (b < 1) b = 1;
    if (b > (1 << 30)) b = 1 << 30;
    return (int)b;
}

// n_drop counts entries that sort to the end as `sentinel` and are not part of M: mirrors of
// self-loops (reading R5) and, when chunking, every entry of an edge outside the chunk.
__global__ void k_validate_expand(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                  const float* __restrict__ w, int64_t E, int32_t N, int32_t dst_limit, int directed,
                                  uint64_t sentinel, uint64_t* __restrict__ keys, uint32_t* __restrict__ pos,
                                  unsigned long long* __restrict__ err_first, int* __restrict__ err_kind,
                                  unsigned long long* __restrict__ n_drop, int32_t n_chunks, int32_t chunk,
                                  uint64_t chunk_key, int32_t* __restrict__ occ) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += stride) {
        int32_t u = src[i], v = dst[i];
        bool bad_id = u < 0 || u >= N || v < 0 || v >= dst_limit;
        bool bad_w = false;
        if (w) {
            float x = w[i];
            bad_w = !(isfinite(x) && x > 0.0f);
        }
        if (bad_id || bad_w) {
            atomicMin(err_first, (unsigned long long)i);
            atomicOr(err_kind, bad_id ? 1 : 2);
            u = 0; v = 0;
        }
        // chunk q(i) = floor(Q * (h_i >> 32) / 2^32), h_i = mix(key ^ i)  (reading R13)
        const bool keep = n_chunks <= 1 ||
                          (int32_t)(((sm64(chunk_key ^ (uint64_t)i) >> 32) * (uint64_t)n_chunks) >> 32) == chunk;
        if (keep && occ) {
            atomicAdd(occ + u, 1);               // endpoint occurrences (reading R14)
            atomicAdd(occ + v, 1);
        }
        keys[i] = keep ? (uint64_t)(uint32_t)u * (uint64_t)N + (uint64_t)(uint32_t)v : sentinel;
        if (pos) pos[i] = __float_as_uint(w ? w[i] : 1.0f);   // sort payload: the weight itself
        unsigned long long drop = keep ? 0 : 1;
        if (!directed) {
            if (!keep || u == v) {
                keys[E + i] = sentinel;          // the mirror of a self-loop is dropped (reading R5)
                drop++;
            } else {
                keys[E + i] = (uint64_t)(uint32_t)v * (uint64_t)N + (uint64_t)(uint32_t)u;
            }
            if (pos) pos[E + i] = __float_as_uint(w ? w[i] : 1.0f);
        }
        if (drop) atomicAdd(n_drop, drop);
    }
}

// over all n_ent sorted keys: the dropped entries (sentinel keys, sorted last) start no run
__global__ void k_head_flags(const uint64_t* __restrict__ keys, int64_t n, uint64_t sentinel,
                             uint8_t* __restrict__ flags) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        flags[i] = (keys[i] != sentinel && (i == 0 || keys[i] != keys[i - 1])) ? 1 : 0;
}

// B2: one thread per (a,b) run: sequential fp64 sum in stable order.
// keys are (src - row_lo) * N + dst (row_lo = the first row of the shard, 0 for a whole graph)
// nnz (runs) and the dropped-entry count are read on the device: the build reads nothing back before
// its last kernel (grids are sized for every entry)
__global__ void k_merge_runs(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ pos,
                             const int64_t* __restrict__ run_start, const unsigned long long* __restrict__ d_nnz,
                             const unsigned long long* __restrict__ d_ndrop, int64_t n_ent,
                             const float* __restrict__ w, int64_t E, int32_t N, int32_t row_lo,
                             int32_t* __restrict__ rows, int32_t* __restrict__ col, double* __restrict__ e_ab) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nnz = (int64_t)*d_nnz, n_valid = n_ent - (int64_t)*d_ndrop;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nnz; u += stride) {
        int64_t s = run_start[u], e = (u + 1 < nnz) ? run_start[u + 1] : n_valid;
        uint64_t k = keys[s];
        rows[u] = (int32_t)(k / (uint64_t)N) + row_lo;
        col[u] = (int32_t)(k % (uint64_t)N);
        double acc = 0.0;
        if (w) {
            // the payload sorted with the keys is the weight (bits); the sort is stable, so a run's
            // weights come in input order (originals, then mirrors: reading B2) and are read in sequence
            for (int64_t i = s; i < e; i++) acc = acc + (double)__uint_as_float(pos[i]);
        } else {
            for (int64_t i = s; i < e; i++) acc = acc + 1.0;
        }
        e_ab[u] = acc;
    }
}

// row_ptr from the row of each (sorted) unique entry; deterministic, no atomics.
__global__ void k_row_ptr(const int32_t* __restrict__ rows, const unsigned long long* __restrict__ d_nnz, int32_t N,
                          int64_t* __restrict__ row_ptr) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nnz = (int64_t)*d_nnz;
    if (nnz == 0)                                  // no entries at all (an empty chunk or shard)
        for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= N; r += stride) row_ptr[r] = 0;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nnz; u += stride) {
        int32_t r = rows[u];
        int32_t prev = (u == 0) ? -1 : rows[u - 1];
        for (int32_t rr = prev + 1; rr <= r; rr++) row_ptr[rr] = u;
        if (u == nnz - 1)
            for (int64_t rr = (int64_t)r + 1; rr <= N; rr++) row_ptr[rr] = nnz;
    }
}

// B3: deg(a) = sum over ascending b of e_ab, the sequential left-to-right fp64 sum.
// A warp takes 32 consecutive rows.  Rows with <= 32 entries: one lane each, literally the
// sequential sum.  Longer rows: the whole warp, one row after another (ballot).  Fast path
// there: when every e_ab of the row is an integer multiple of 2^q (q = the smallest "last set
// bit" exponent over the row's values, e_ab_exp_q below) and the total is below 2^(53+q), every
// partial sum in ANY order is a multiple of 2^q below 2^(53+q) -- exactly representable -- so every
// order, the sequential one included, returns the exact total: the parallel sum IS the sequential
// result.  (q >= 0 -- integers -- covers unit-weight graphs; c4's lognormal fp32 weights give
// q ~ -30 against totals ~2^17, so its weighted hub rows take it too: the 92k-entry row's
// sequential fold was 1.2 ms of every c4 build.)  Otherwise the lanes load 32 consecutive e_ab
// (coalesced) and one lane folds them in ascending order -- the sequential sum again.
__device__ __forceinline__ int e_ab_exp_q(double x) {     // x = m * 2^q with m odd (x > 0, normal)
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const unsigned long long mant = b & ((1ull << 52) - 1);
    const int e = (int)((b >> 52) & 0x7ff);
    return e - 1075 + (mant ? __ffsll((long long)mant) - 1 : 52);
}
__device__ double degree_long_row(const double* __restrict__ e_ab, int64_t k0, int64_t k1, int lane,
                                  double* __restrict__ stage) {
    // 8 independent partial sums per lane keep 8 loads in flight on hub rows
    double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int q = 1 << 20;
    int64_t k = k0 + lane;
    for (; k + 7 * 32 < k1; k += 8 * 32) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; u++) x[u] = e_ab[k + 32 * u];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            q = min(q, e_ab_exp_q(x[u]));
            p[u] += x[u];
        }
    }
    for (; k < k1; k += 32) {
        const double x = e_ab[k];
        q = min(q, e_ab_exp_q(x));
        p[0] += x;
    }
    double s = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        q = min(q, __shfl_xor_sync(0xffffffffu, q, o));
    }
    // exact-order-independence test on the computed total, with a margin that covers its own rounding
    // when the condition fails (relative error < n * 2^-53 < 2^-20): s is then exact whenever it passes
    const bool exact = q > -1000 && q < 960 && s <= ldexp(1.0 - 0x1p-20, 53 + q);
    if (!exact) {
        // general case: the sequential fold, by lane 0, from 32 values the warp stages in shared
        // memory (coalesced load of the next 32 issued before the fold, so the chain of dependent
        // fp64 adds is the only serial part; round 1 shuffled every value to every lane: ~25
        // cycles per entry, 2.8 ms per c4 build on its weighted hub rows)
        // Blocks of 8 x 32 values: the next block's loads are issued before this block is folded, so a
        // hub row (c4: 92k entries) waits for memory once per 256 entries, not once per 32 (1.9 ms ->
        // the fold's own dependent-add chain)
        s = 0.0;
        double nxt[8];
#pragma unroll
        for (int u = 0; u < 8; u++) nxt[u] = k0 + 32 * u + lane < k1 ? e_ab[k0 + 32 * u + lane] : 0.0;
        for (int64_t kb = k0; kb < k1; kb += 256) {
            double cur[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                cur[u] = nxt[u];
                const int64_t q = kb + 256 + 32 * u + lane;
                nxt[u] = q < k1 ? e_ab[q] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int64_t cb = kb + 32 * u;
                if (cb >= k1) break;                  // warp-uniform
                const int n = (int)min((int64_t)32, k1 - cb);
                stage[lane] = cur[u];
                __syncwarp();
                if (lane == 0) {
                    // all 32 values into registers first, then the dependent chain of adds alone
                    // (4 at a time, the shared-memory latency sat inside the chain: c4's 92k-entry hub
                    // row folded at ~23 cycles per entry)
                    double v[32];
#pragma unroll
                    for (int q = 0; q < 32; q++) v[q] = stage[q];
#pragma unroll
                    for (int q = 0; q < 32; q++)
                        if (q < n) s = s + v[q];
                }
                __syncwarp();
            }
        }
        s = __shfl_sync(0xffffffffu, s, 0);
    }
    return s;
}

// Rows longer than this are folded by k_degree_long, one warp per row: the warp that owns a group of
// 32 rows would otherwise fold its long rows one after another -- on R-MAT the hubs share low ids
// (c4: one warp folded several hub rows of up to 92k weighted entries in sequence, 1.9 ms per build)
constexpr int64_t kDegLong = 1024;

// zero rows are counted inside [row_lo, row_hi) only (a shard's rows; the whole graph otherwise)
__global__ void k_degree(const int64_t* __restrict__ row_ptr, const double* __restrict__ e_ab, int32_t N,
                         int32_t row_lo, int32_t row_hi, double* __restrict__ deg,
                         unsigned long long* __restrict__ zero_rows, unsigned long long* __restrict__ max_deg,
                         int32_t* __restrict__ long_rows, unsigned long long* __restrict__ n_long) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    __shared__ double stage[kThreads / 32][32];
    // zero-row count and max degree: per-lane registers, one atomic per block at the end (per-row
    // atomics on two addresses serialise in L2)
    unsigned long long my_zero = 0, my_max = 0;
    for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < N; base += nwarps * 32) {
        const int64_t a = base + lane;
        int64_t k0 = 0, k1 = 0;
        if (a < N) {
            k0 = row_ptr[a];
            k1 = row_ptr[a + 1];
            if (k1 == k0 && a >= row_lo && a < row_hi) my_zero++;
            else my_max = max(my_max, (unsigned long long)(k1 - k0));
        }
        const bool lng = a < N && k1 - k0 > 32;
        if (a < N && !lng) {
            double s = 0.0;
            int64_t k = k0;
            for (; k + 4 <= k1; k += 4) {            // 4 loads in flight, the same left-to-right sum
                const double x0 = e_ab[k], x1 = e_ab[k + 1], x2 = e_ab[k + 2], x3 = e_ab[k + 3];
                s = s + x0;
                s = s + x1;
                s = s + x2;
                s = s + x3;
            }
            for (; k < k1; k++) s = s + e_ab[k];
            deg[a] = s;
        }
        const bool defer = lng && k1 - k0 > kDegLong;
        if (defer) long_rows[atomicAdd(n_long, 1ull)] = (int32_t)a;
        unsigned m = __ballot_sync(0xffffffffu, lng && !defer);
        while (m) {
            const int l = __ffs(m) - 1;
            m &= m - 1;
            const double s = degree_long_row(e_ab, __shfl_sync(0xffffffffu, k0, l), __shfl_sync(0xffffffffu, k1, l), lane,
                                             stage[threadIdx.x >> 5]);
            if (lane == 0) deg[base + l] = s;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        my_zero += __shfl_xor_sync(0xffffffffu, my_zero, o);
        my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
    }
    __shared__ unsigned long long s_zero[32], s_max[32];
    const int warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_zero[warp] = my_zero;
        s_max[warp] = my_max;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long z = 0, mx = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            z += s_zero[w];
            mx = max(mx, s_max[w]);
        }
        if (z) atomicAdd(zero_rows, z);
        if (mx) atomicMax(max_deg, mx);
    }
}

// the rows k_degree deferred, one warp each (any order: each row's fold is its own)
__global__ void k_degree_long(const int64_t* __restrict__ row_ptr, const double* __restrict__ e_ab,
                              const int32_t* __restrict__ long_rows, const unsigned long long* __restrict__ n_long,
                              double* __restrict__ deg) {
    const int lane = threadIdx.x & 31;
    __shared__ double stage[kThreads / 32][32];
    const int64_t n = (int64_t)*n_long;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
        const int32_t a = long_rows[i];
        const double v = degree_long_row(e_ab, row_ptr[a], row_ptr[a + 1], lane, stage[threadIdx.x >> 5]);
        if (lane == 0) deg[a] = v;
    }
}

// B4: val = fp32_rn(e_ab / deg(a)).
__global__ void k_values(const int32_t* __restrict__ rows, const double* __restrict__ e_ab,
                         const double* __restrict__ deg, const unsigned long long* __restrict__ d_nnz,
                         float* __restrict__ val) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nnz = (int64_t)*d_nnz;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride)
        val[k] = __double2float_rn(e_ab[k] / deg[rows[k]]);
}

struct IsHeavy {
    const int64_t* rp;
    int64_t thresh;
    __host__ __device__ bool operator()(int64_t r) const { return rp[r + 1] - rp[r] > thresh; }
};

// r starts a light chunk: the first row, every `rows`-th row (<= kChunkRows), or the first row whose entries
// begin in a new window of `win` entries (counted from the shard's first entry)
struct IsChunkStart {
    const int64_t* rp;
    int64_t r0, win, rows;
    __host__ __device__ bool operator()(int64_t r) const {
        if (r == r0 || (r - r0) % rows == 0) return true;
        return (rp[r] - rp[r0]) / win != (rp[r - 1] - rp[r0]) / win;
    }
};

__global__ void k_put_end(int64_t* __restrict__ starts, const int64_t* __restrict__ n, int64_t end) {
    starts[*n] = end;
}

// chunks of one row each: starts[i] = r0 + i for i <= nr, and their count
__global__ void k_iota_starts(int64_t* __restrict__ starts, int64_t r0, int64_t nr, int64_t* __restrict__ n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nr; i += stride) starts[i] = r0 + i;
    if (blockIdx.x == 0 && threadIdx.x == 0) *n = nr;
}

// h < *nh (heavy rows found): items of the row, and its partial-vector slots (multi-part rows only);
// h in [*nh, nh_max]: 0, so the scans' last entries are the totals
__global__ void k_items_per_row(const int64_t* __restrict__ rp, const int64_t* __restrict__ hrows,
                                const int64_t* __restrict__ nh, int64_t nh_max, int64_t per_item,
                                int64_t* __restrict__ nit, int64_t* __restrict__ nsl) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n = *nh;
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h <= nh_max; h += stride) {
        int64_t c = 0;
        if (h < n) {
            const int64_t r = hrows[h];
            c = (rp[r + 1] - rp[r] + per_item - 1) / per_item;
        }
        nit[h] = c;
        nsl[h] = c > 1 ? c : 0;
    }
}

__global__ void k_fill_items(const int64_t* __restrict__ rp, const int64_t* __restrict__ hrows,
                             const int64_t* __restrict__ nh, int64_t nh_max, const int64_t* __restrict__ first,
                             const int64_t* __restrict__ sfirst, int64_t per_item, HeavyItem* __restrict__ items,
                             int64_t* __restrict__ counts) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n = *nh;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        counts[1] = first[nh_max];                // totals (inputs past *nh are 0)
        counts[3] = sfirst[nh_max];
    }
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < n; h += stride) {
        const int64_t r = hrows[h];
        const int64_t k0 = rp[r], k1 = rp[r + 1];
        const int64_t np = (k1 - k0 + per_item - 1) / per_item;
        for (int64_t p = 0; p < np; p++) {
            HeavyItem it;
            it.k0 = k0 + p * per_item;
            it.k1 = min(k1, it.k0 + per_item);
            it.row = (int32_t)r;
            it.part = (int32_t)p;
            it.nparts = (int32_t)np;
            it.slot = np > 1 ? (int32_t)(sfirst[h] + p) : -1;
            items[first[h] + p] = it;
        }
    }
}

// ---- row-sharded builds (world > 1): every rank reads the whole COO, counts the
// entries of every row (after mirroring, before merging), cuts the rows into nnz-balanced shards,
// and keeps only the entries of its own rows -- M is never materialised whole on any rank.

// cnt[a] += entries of row a; indeg[b] += entries of column b (directed only: for undirected
// graphs the pattern is symmetric and indeg = cnt); occ as k_validate_expand; validation as
// k_validate_expand (first bad edge, kind)
__global__ void k_count_rows(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                             const float* __restrict__ w, int64_t E, int32_t N, int directed,
                             unsigned long long* __restrict__ cnt, int32_t* __restrict__ indeg,
                             unsigned long long* __restrict__ err_first, int* __restrict__ err_kind, int32_t n_chunks,
                             int32_t chunk, uint64_t chunk_key, int32_t* __restrict__ occ) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += stride) {
        const int32_t u = src[i], v = dst[i];
        const bool bad_id = u < 0 || u >= N || v < 0 || v >= N;
        bool bad_w = false;
        if (w) {
            const float x = w[i];
            bad_w = !(isfinite(x) && x > 0.0f);
        }
        if (bad_id || bad_w) {
            atomicMin(err_first, (unsigned long long)i);
            atomicOr(err_kind, bad_id ? 1 : 2);
            continue;
        }
        const bool keep = n_chunks <= 1 ||
                          (int32_t)(((sm64(chunk_key ^ (uint64_t)i) >> 32) * (uint64_t)n_chunks) >> 32) == chunk;
        if (!keep) continue;
        if (occ) {
            atomicAdd(occ + u, 1);
            atomicAdd(occ + v, 1);
        }
        atomicAdd(cnt + u, 1ull);
        if (directed) {
            atomicAdd(indeg + v, 1);
        } else if (u != v) {
            atomicAdd(cnt + v, 1ull);
        }
    }
}

__global__ void k_cnt_to_indeg(const unsigned long long* __restrict__ cnt, int32_t N, int32_t* __restrict__ indeg) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < N; v += stride) indeg[v] = (int32_t)cnt[v];
}

// cuts[p] = first row whose entry prefix reaches p * total / world; ent[p] = prefix[cuts[p]]
__global__ void k_cuts_ent(const int64_t* __restrict__ prefix, int32_t N, int world, int64_t* __restrict__ cuts,
                           int64_t* __restrict__ ent) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > world) return;
    const int64_t tot = prefix[N];
    int64_t c;
    if (p == 0) {
        c = 0;
    } else if (p == world) {
        c = N;
    } else {
        int64_t lo = 0, hi = N;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((__int128)prefix[mid] * world >= (__int128)p * tot) hi = mid; else lo = mid + 1;
        }
        c = lo;
    }
    cuts[p] = c;
    ent[p] = prefix[c];
}

// entry i of the mirrored list (i < E: edge i as given; i >= E: the mirror of edge i - E) is in the
// shard: valid (checked by k_count_rows), in the chunk, not the dropped mirror of a self-loop, and
// its source row in [lo, hi).  cub::DeviceSelect keeps the selected indices in input order, so the
// shard's entries keep their relative order of the whole list (readings B1, B2: the same sums).
struct InShard {
    const int32_t* src;
    const int32_t* dst;
    int64_t E;
    int32_t lo, hi;
    int directed;
    int32_t n_chunks, chunk;
    uint64_t chunk_key;
    __device__ bool operator()(uint32_t i) const {
        const bool mirror = (int64_t)i >= E;
        const int64_t e = mirror ? (int64_t)i - E : (int64_t)i;
        const int32_t u = src[e], v = dst[e];
        if (mirror && (directed || u == v)) return false;
        const int32_t r = mirror ? v : u;
        if (r < lo || r >= hi) return false;
        return n_chunks <= 1 ||
               (int32_t)(((sm64(chunk_key ^ (uint64_t)e) >> 32) * (uint64_t)n_chunks) >> 32) == chunk;
    }
};

// keys of the selected entries, and (weighted) their weights in place of their positions: the sort
// payload is the weight itself (see k_merge_runs)
__global__ void k_shard_keys(uint32_t* __restrict__ pos, int64_t n, const int32_t* __restrict__ src,
                             const int32_t* __restrict__ dst, const float* __restrict__ w, int64_t E, int32_t N,
                             int32_t lo, uint64_t* __restrict__ keys) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        const int64_t i = pos[k];
        const bool mirror = i >= E;
        const int64_t e = mirror ? i - E : i;
        const int32_t u = mirror ? dst[e] : src[e], v = mirror ? src[e] : dst[e];
        keys[k] = (uint64_t)(uint32_t)(u - lo) * (uint64_t)N + (uint64_t)(uint32_t)v;
        if (w) pos[k] = __float_as_uint(w[e]);
    }
}

// Small builds carve their transient buffers out of one block (an arena), so that a graph of 10^5
// entries costs one allocation instead of ~12 cudaMallocAsync / cudaFreeAsync pairs -- on such graphs
// the host's enqueue rate, not the GPU, sets the build time (c1: profiles/r02_c1_trace.json).
struct Arena {
    char* base = nullptr;
    size_t cap = 0, used = 0;
};
thread_local Arena tl_arena;

template <class T>
struct DevBuf {
    T* p = nullptr;
    cudaStream_t s = nullptr;
    bool in_arena = false;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    ~DevBuf() { drop(); }
    // transient unless the buffer outlives the call (released into a CSR or a schedule)
    Status alloc(size_t n, cudaStream_t st, const char* what, bool long_lived = false) {
        s = st;
        const size_t bytes = n * sizeof(T) + 16;
        Arena& a = tl_arena;
        if (!long_lived && a.base) {
            const size_t off = (a.used + 255) & ~(size_t)255;
            if (off + bytes <= a.cap) {
                p = reinterpret_cast<T*>(a.base + off);
                a.used = off + bytes;
                in_arena = true;
                return Status::ok();
            }
        }
        return dalloc((void**)&p, bytes, st, what, long_lived ? 0 : kAllocTransient);
    }
    T* release() { T* q = p; p = nullptr; return q; }      // long-lived buffers only
    void drop() {                                           // free now (a no-op inside the arena)
        if (p && !in_arena) dfree(p, s);
        p = nullptr;
    }
};

// Installs an arena of `bytes` for the current thread (if bytes > 0 and it can be had) until the
// guard goes out of scope; nested guards leave an installed arena alone.
struct ArenaGuard {
    bool mine = false;
    cudaStream_t s;
    ArenaGuard(size_t bytes, cudaStream_t st) : s(st) {
        static const bool off = getenv("CLEORA_NO_ARENA") != nullptr;   // A/B switch
        if (off || bytes == 0 || tl_arena.base) return;
        void* p = nullptr;
        if (!dalloc(&p, bytes, st, "build arena", kAllocTransient).good()) return;
        tl_arena = Arena{(char*)p, bytes, 0};
        mine = true;
    }
    ~ArenaGuard() {
        if (!mine) return;
        dfree(tl_arena.base, s);
        tl_arena = Arena{};
    }
};

// ---- one-kernel build of small graphs (DESIGN §7 "Build kernels").  On a graph of 10^5 entries
// the general build is ~20 dependent launches of a few microseconds each (c1: 0.136 ms of a 0.25 ms
// step).  This path does the same B1-B4 in ONE cooperative kernel with five grid-wide barriers:
//   P0 validate, count every row's entries (after mirroring, before merging)
//   P1 exclusive scan of the counts -> bucket starts and cursors (two phases around a barrier)
//   P2 scatter every entry into its row's bucket as (dst << 32 | list position) + weight
//   P3 a warp per row: sort the bucket by that key (rank sort in shared memory; rows <= kSmallCap)
//      = the stable (src, dst) order of B1; merge runs of equal dst summing their weights in list
//      order in fp64 (B2); count the merged entries
//   P4 scan the merged counts -> row_ptr; per row: deg = the sequential fp64 fold over ascending
//      dst (B3), val = fp32_rn(e_ab / deg) (B4), written at row_ptr
// Same bits as the general path (tested: test_small_build_bitwise).  A row longer than kSmallCap
// entries makes the kernel stop after P1 and report it; the caller then runs the general path.
constexpr int kSmallCap = 256;
constexpr int kSmallThreads = 256;
constexpr int kSmallWarps = kSmallThreads / 32;

struct SmallArgs {
    const int32_t* src;
    const int32_t* dst;
    const float* w;
    int64_t E;
    int32_t N;
    int directed;
    int32_t* start;      // [N + 1] entry counts, then bucket starts (zeroed by the caller)
    int32_t* flags;      // [4] (zeroed): [0] error kind, [1] longest row (entries), [2] 1 = too long
    int32_t* cur;        // [N] bucket cursors
    int32_t* ucnt;       // [N] merged entries per row
    int64_t* bsum;       // [2 * gridDim.x] block totals: entries, merged entries
    uint64_t* bkey;      // [n_all] bucketed entries: dst << 32 | position in the mirrored list
    float* bw;           // [n_all] their weights (weighted graphs)
    int32_t* mcol;       // [n_all] merged entries at bucket positions: column, e_ab
    double* me;
    int64_t* row_ptr;    // outputs (the CSR of build_csr)
    int32_t* col;
    float* val;
    double* deg;
    unsigned long long* scal;   // (zeroed) [0] first bad edge [2] zero rows [3] longest row [4] nnz
};

union SmallScanTmp {
    typename cub::BlockScan<int64_t, kSmallThreads>::TempStorage scan;
    typename cub::BlockReduce<int64_t, kSmallThreads>::TempStorage red;
};

__device__ __forceinline__ bool small_edge(const SmallArgs& a, int64_t i, int32_t& u, int32_t& v) {
    u = a.src[i];
    v = a.dst[i];
    bool bad_w = false;
    if (a.w) {
        const float x = a.w[i];
        bad_w = !(isfinite(x) && x > 0.0f);
    }
    const bool bad_id = u < 0 || u >= a.N || v < 0 || v >= a.N;
    return !(bad_id || bad_w);
}

// sum of bsum[q * G + 0 .. q * G + b), b = this block (all threads get it)
__device__ int64_t small_block_offset(const int64_t* bsum, SmallScanTmp& tmp, int64_t* bcast) {
    int64_t x = 0;
    for (int q = threadIdx.x; q < (int)blockIdx.x; q += blockDim.x) x += bsum[q];
    x = cub::BlockReduce<int64_t, kSmallThreads>(tmp.red).Sum(x);
    if (threadIdx.x == 0) *bcast = x;
    __syncthreads();
    x = *bcast;
    __syncthreads();
    return x;
}

// rows [r0, r1) of this block, a contiguous sub-range per thread: out[r] = offset + exclusive prefix
// of in[] (and out2[r], if given); returns the block's total
template <class T>
__device__ int64_t small_block_scan(const int32_t* in, int64_t r0, int64_t r1, int64_t offset, T* out, int32_t* out2,
                                    SmallScanTmp& tmp) {
    const int64_t n = r1 - r0, per = (n + blockDim.x - 1) / blockDim.x;
    const int64_t a0 = r0 + min(n, per * threadIdx.x), a1 = r0 + min(n, per * (threadIdx.x + 1));
    int64_t x = 0;
    for (int64_t r = a0; r < a1; r++) x += in[r];
    int64_t ex = 0, tot = 0;
    cub::BlockScan<int64_t, kSmallThreads>(tmp.scan).ExclusiveSum(x, ex, tot);
    __syncthreads();
    int64_t run = offset + ex;
    for (int64_t r = a0; r < a1; r++) {
        const int32_t c = in[r];
        out[r] = (T)run;
        if (out2) out2[r] = (int32_t)run;
        run += c;
    }
    return tot;
}

__global__ void __launch_bounds__(kSmallThreads) k_build_small(const SmallArgs a) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    extern __shared__ unsigned char small_smem[];
    __shared__ SmallScanTmp tmp;
    __shared__ int64_t bcast;
    __shared__ int64_t s_tot[kSmallWarps];
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t N = a.N;
    const int64_t G = gridDim.x;
    // this block's rows in P1, P3, P4
    const int64_t R = (N + G - 1) / G;
    const int64_t r0 = min((int64_t)N, (int64_t)blockIdx.x * R), r1 = min((int64_t)N, r0 + R);

    // P0: validate and count
    for (int64_t i = tid; i < a.E; i += nth) {
        int32_t u, v;
        if (!small_edge(a, i, u, v)) {
            atomicMax(a.scal + 0, ~(unsigned long long)i);     // the first bad edge is the largest ~i
            atomicOr(a.flags + 0, (u < 0 || u >= N || v < 0 || v >= N) ? 1 : 2);
            continue;
        }
        atomicAdd(a.start + u, 1);
        if (!a.directed && u != v) atomicAdd(a.start + v, 1);   // the mirror of a self-loop is dropped (R5)
    }
    grid.sync();

    // P1a: block totals and the longest row
    {
        int64_t x = 0;
        int32_t mx = 0;
        for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
            const int32_t c = a.start[r];
            x += c;
            mx = max(mx, c);
        }
        x = cub::BlockReduce<int64_t, kSmallThreads>(tmp.red).Sum(x);
        if (threadIdx.x == 0) a.bsum[blockIdx.x] = x;
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && mx > 0) atomicMax(a.flags + 1, mx);
    }
    grid.sync();
    if (__ldcg(a.flags + 1) > kSmallCap) {                    // the general path builds this graph
        if (tid == 0) a.flags[2] = 1;
        return;
    }
    // P1b: bucket starts and cursors (start[N] = all entries)
    {
        const int64_t off = small_block_offset(a.bsum, tmp, &bcast);
        const int64_t tot = small_block_scan<int32_t>(a.start, r0, r1, off, a.start, a.cur, tmp);
        if (r1 == N && r1 > r0 && threadIdx.x == 0) a.start[N] = (int32_t)(off + tot);
        if (N == 0 && tid == 0) a.start[0] = 0;
    }
    grid.sync();

    // P2: scatter (position in the mirrored list: i for an edge as given, E + i for its mirror)
    for (int64_t i = tid; i < a.E; i += nth) {
        int32_t u, v;
        if (!small_edge(a, i, u, v)) continue;
        const float x = a.w ? a.w[i] : 1.0f;
        int32_t q = atomicAdd(a.cur + u, 1);
        a.bkey[q] = ((uint64_t)(uint32_t)v << 32) | (uint64_t)i;
        if (a.w) a.bw[q] = x;
        if (!a.directed && u != v) {
            q = atomicAdd(a.cur + v, 1);
            a.bkey[q] = ((uint64_t)(uint32_t)u << 32) | (uint64_t)(a.E + i);
            if (a.w) a.bw[q] = x;
        }
    }
    grid.sync();

    // P3: a warp per row of this block: sort, merge runs, count
    {
        uint64_t* kin = reinterpret_cast<uint64_t*>(small_smem) + (size_t)warp * 2 * kSmallCap;
        uint64_t* kout = kin + kSmallCap;
        float* win = reinterpret_cast<float*>(reinterpret_cast<uint64_t*>(small_smem) + (size_t)kSmallWarps * 2 * kSmallCap) +
                     (size_t)warp * 2 * kSmallCap;
        float* wout = win + kSmallCap;
        int64_t wtot = 0;
        for (int64_t r = r0 + warp; r < r1; r += kSmallWarps) {
            const int32_t b = a.start[r], n = a.start[r + 1] - b;
            for (int j = lane; j < n; j += 32) {
                kin[j] = a.bkey[b + j];
                if (a.w) win[j] = a.bw[b + j];
            }
            __syncwarp();
            for (int j = lane; j < n; j += 32) {       // keys are distinct (positions): rank = slot
                const uint64_t k = kin[j];
                int rk = 0;
                for (int t = 0; t < n; t++) rk += kin[t] < k;
                kout[rk] = k;
                if (a.w) wout[rk] = win[j];
            }
            __syncwarp();
            int32_t u = 0;                             // merged entries so far
            for (int c = 0; c < n; c += 32) {
                const int j = c + lane;
                const uint32_t cj = j < n ? (uint32_t)(kout[j] >> 32) : 0u;
                const bool head = j < n && (j == 0 || (uint32_t)(kout[j - 1] >> 32) != cj);
                const unsigned m = __ballot_sync(0xffffffffu, head);
                if (head) {
                    double acc = 0.0;                  // B2: list order within the run
                    for (int t = j; t < n && (uint32_t)(kout[t] >> 32) == cj; t++)
                        acc = acc + (a.w ? (double)wout[t] : 1.0);
                    const int32_t ui = u + __popc(m & ((1u << lane) - 1u));
                    a.mcol[b + ui] = (int32_t)cj;
                    a.me[b + ui] = acc;
                }
                u += __popc(m);
            }
            if (lane == 0) a.ucnt[r] = u;
            wtot += u;
            __syncwarp();
        }
        if (lane == 0) s_tot[warp] = wtot;
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t x = 0;
            for (int q = 0; q < kSmallWarps; q++) x += s_tot[q];
            a.bsum[G + blockIdx.x] = x;
        }
    }
    grid.sync();

    // P4: row_ptr, then degree and values of this block's rows
    {
        const int64_t off = small_block_offset(a.bsum + G, tmp, &bcast);
        const int64_t tot = small_block_scan<int64_t>(a.ucnt, r0, r1, off, a.row_ptr, nullptr, tmp);
        if (r1 == N && r1 > r0 && threadIdx.x == 0) {
            a.row_ptr[N] = off + tot;
            a.scal[4] = (unsigned long long)(off + tot);
        }
        if (N == 0 && tid == 0) a.row_ptr[0] = 0;
        if (tid == 0)                                  // the verdict: first bad edge, as build_csr's scal[0]
            a.scal[0] = __ldcg(a.flags + 0) ? ~__ldcg(a.scal + 0) : ~0ull;
        __syncthreads();                               // this block's row_ptr
        unsigned long long zeros = 0, mx = 0;
        for (int64_t r = r0 + warp; r < r1; r += kSmallWarps) {
            const int32_t b = a.start[r], u = a.ucnt[r];
            const int64_t rp = a.row_ptr[r];
            double s = 0.0;                            // B3: sequential over ascending dst
            for (int c = 0; c < u; c += 32) {
                const int n = min(32, u - c);
                const double x = lane < n ? a.me[b + c + lane] : 0.0;
                for (int t = 0; t < n; t++) s = s + __shfl_sync(0xffffffffu, x, t);
            }
            for (int j = lane; j < u; j += 32) {
                a.col[rp + j] = a.mcol[b + j];
                a.val[rp + j] = __double2float_rn(a.me[b + j] / s);   // B4
            }
            if (lane == 0) {
                a.deg[r] = s;
                if (u == 0) zeros++;
                else mx = max(mx, (unsigned long long)u);
            }
        }
        if (lane == 0) {
            if (zeros) atomicAdd(a.scal + 2, zeros);
            if (mx) atomicMax(a.scal + 3, mx);
        }
    }
}

// The one-kernel build (above) of a graph of <= kSmallMaxEntries mirrored entries.  *done = false:
// a row is longer than kSmallCap, nothing was built (the general path follows).
constexpr int64_t kSmallMaxEntries = (int64_t)1 << 21;
constexpr int32_t kSmallMaxRows = 1 << 24;

Status build_small(const int32_t* d_src, const int32_t* d_dst, const float* d_w, int64_t E, int32_t N, int directed,
                   cudaStream_t s, BuildOut* out, bool* done) {
    *done = false;
    const int64_t n_all = directed ? E : 2 * E;
    constexpr size_t smem = (size_t)kSmallWarps * 2 * kSmallCap * (sizeof(uint64_t) + sizeof(float));
    static int occ[kMaxDevices], nsm[kMaxDevices];
    static std::mutex mu;
    int dev = 0;
    CL_CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= kMaxDevices) return Status::make(4, "build: device ordinal beyond kMaxDevices");
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!occ[dev]) {
            CL_CUDA_TRY(cudaFuncSetAttribute(k_build_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CL_CUDA_TRY(cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev));
            int b = 0;
            CL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_build_small, kSmallThreads, smem));
            occ[dev] = b < 1 ? -1 : b;
        }
    }
    if (occ[dev] < 1) return Status::ok();             // cannot be co-resident: general path
    // every block resident (cooperative launch); no more blocks than a thread per edge or row needs
    // (P3/P4 walk a warp's rows one after another: ~2 rows per warp keeps that chain short)
    const int64_t want = std::max<int64_t>((E + kSmallThreads - 1) / kSmallThreads, ((int64_t)N + 2 * kSmallWarps - 1) / (2 * kSmallWarps));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm[dev] * occ[dev], want));

    ArenaGuard arena((size_t)n_all * 32 + (size_t)N * 16 + ((size_t)1 << 20), s);
    DevBuf<int32_t> zeroed, cur, ucnt, mcol;
    DevBuf<int64_t> bsum;
    DevBuf<uint64_t> bkey;
    DevBuf<float> bw;
    DevBuf<double> me;
    DevBuf<unsigned long long> scal;
    DevBuf<int64_t> row_ptr;
    DevBuf<int32_t> col;
    DevBuf<float> val;
    DevBuf<double> deg;
    CL_TRY(zeroed.alloc((size_t)N + 1 + 4, s, "small build counts"));
    CL_TRY(cur.alloc(N, s, "small build cursors"));
    CL_TRY(ucnt.alloc(N, s, "small build merged counts"));
    CL_TRY(bsum.alloc(2 * (size_t)grid, s, "small build block sums"));
    CL_TRY(bkey.alloc(n_all, s, "small build buckets"));
    if (d_w) CL_TRY(bw.alloc(n_all, s, "small build bucket weights"));
    CL_TRY(mcol.alloc(n_all, s, "small build merged cols"));
    CL_TRY(me.alloc(n_all, s, "small build e_ab"));
    CL_TRY(scal.alloc(8, s, "scalars", true));
    CL_TRY(row_ptr.alloc((size_t)N + 1, s, "CSR row_ptr", true));
    CL_TRY(col.alloc(n_all, s, "CSR col", true));
    CL_TRY(val.alloc(n_all, s, "CSR val", true));
    CL_TRY(deg.alloc(N, s, "degree", true));
    CL_CUDA_TRY(cudaMemsetAsync(zeroed.p, 0, ((size_t)N + 1 + 4) * sizeof(int32_t), s));
    CL_CUDA_TRY(cudaMemsetAsync(scal.p, 0, 8 * sizeof(unsigned long long), s));
    SmallArgs a;
    a.src = d_src;
    a.dst = d_dst;
    a.w = d_w;
    a.E = E;
    a.N = N;
    a.directed = directed;
    a.start = zeroed.p;
    a.flags = zeroed.p + N + 1;
    a.cur = cur.p;
    a.ucnt = ucnt.p;
    a.bsum = bsum.p;
    a.bkey = bkey.p;
    a.bw = bw.p;
    a.mcol = mcol.p;
    a.me = me.p;
    a.row_ptr = row_ptr.p;
    a.col = col.p;
    a.val = val.p;
    a.deg = deg.p;
    a.scal = scal.p;
    void* args[] = {&a};
    CL_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_build_small, dim3(grid), dim3(kSmallThreads), args, smem, s));
    count_launches(1);
    unsigned long long h_scal[5] = {0, 0, 0, 0, 0};
    int32_t h_flags[4] = {0, 0, 0, 0};
    {
        const SmallRead rd[2] = {{h_scal, scal.p, 5 * sizeof(unsigned long long)}, {h_flags, a.flags, 4 * sizeof(int32_t)}};
        CL_TRY(read_small_n(rd, 2, s));
    }
    trace("csr: one-kernel build", s, false);
    if (h_flags[0]) {
        char buf[256];
        snprintf(buf, sizeof buf, "cleora_build: edge %llu: %s", (unsigned long long)h_scal[0],
                 (h_flags[0] & 1) ? "node id outside [0, n_nodes)" : "weight not finite or <= 0");
        return Status::make(3, buf);
    }
    if (h_flags[2]) return Status::ok();               // a row longer than kSmallCap: general path
    out->nnz = (int64_t)h_scal[4];
    out->zero_rows = (int64_t)h_scal[2];
    out->max_degree = (int64_t)h_scal[3];
    out->d_scal = scal.release();
    out->row_ptr = row_ptr.release();
    out->col = col.release();
    out->val = val.release();
    out->deg = deg.release();
    *done = true;
    return Status::ok();
}

}  // namespace

Status build_csr(const int32_t* d_src, const int32_t* d_dst, const float* d_w, int64_t E, int32_t N,
                 int directed, cudaStream_t s, BuildOut* out, const BuildExtra* extra) {
    const BuildExtra none;
    const BuildExtra& x = extra ? *extra : none;
    // shard mode (x.row_hi >= 0): only the entries of rows [row_lo, row_hi), x.shard_entries of them,
    // selected from the mirrored list in order; the edges were validated (and occ counted) by
    // shard_plan, so nothing is dropped here
    const bool shard = x.row_hi >= 0;
    const int32_t lo = shard ? x.row_lo : 0, hi = shard ? x.row_hi : N;
    const int64_t n_all = directed ? E : 2 * E;         // entries of the mirrored list
    // small whole graphs: one kernel (CLEORA_SMALL_BUILD=0: always the general path, for A/B and tests)
    const char* sme = getenv("CLEORA_SMALL_MAX_ENTRIES");            // A/B of the size limit
    const int64_t small_max = sme ? atoll(sme) : kSmallMaxEntries;
    if (!shard && x.n_chunks <= 1 && !x.occ && x.dst_limit < 0 && n_all <= small_max && N <= kSmallMaxRows) {
        const char* e = getenv("CLEORA_SMALL_BUILD");
        if (!e || atoi(e) != 0) {
            bool done = false;
            CL_TRY(build_small(d_src, d_dst, d_w, E, N, directed, s, out, &done));
            if (done) return Status::ok();
        }
    }
    const int64_t n_ent = shard ? x.shard_entries : n_all;
    if (n_all >= (int64_t)UINT32_MAX) return Status::make(2, "cleora_build: too many edges (entry positions are 32-bit)");
    const uint64_t NN = (uint64_t)(hi - lo) * (uint64_t)N;
    const uint64_t sentinel = NN;                        // sorts after every valid key
    const int end_bit = 64 - __builtin_clzll(sentinel | 1ull);

    // small builds: one block for every transient buffer (sort keys x2, payloads x2, flags, run starts,
    // rows, e_ab, CUB temporaries: < 64 bytes per entry)
    ArenaGuard arena(n_ent <= (1 << 20) ? (size_t)n_ent * 64 + ((size_t)4 << 20) : 0, s);
    DevBuf<uint64_t> keys, keys2;
    DevBuf<uint32_t> pos, pos2;                          // sort payload: the entries' weights (fp32 bits)
    DevBuf<unsigned long long> scal;                     // [0] err_first [1] n_self [2] zero_rows [3] max_deg [4] nnz
    DevBuf<int> err_kind;
    // unit weights: e_ab is the run length, the same in any order, so the sort needs no payload -- a
    // third less traffic.  Weighted: the payload is the weight, so the merge reads each run's weights in
    // sequence (round 1 sorted positions and gathered w[pos] at random: c4 1.45 ms per build)
    const bool keys_only = d_w == nullptr;
    CL_TRY(keys.alloc(n_ent, s, "sort keys"));
    CL_TRY(keys2.alloc(n_ent, s, "sort keys (alt)"));
    if (!keys_only || shard) CL_TRY(pos.alloc(n_ent, s, "sort payload"));
    if (!keys_only) CL_TRY(pos2.alloc(n_ent, s, "sort payload (alt)"));
    CL_TRY(scal.alloc(8, s, "scalars", true));
    CL_TRY(err_kind.alloc(1, s, "scalars"));
    CL_CUDA_TRY(cudaMemsetAsync(scal.p, 0, 8 * sizeof(unsigned long long), s));
    CL_CUDA_TRY(cudaMemsetAsync(scal.p, 0xFF, sizeof(unsigned long long), s));   // err_first = max
    CL_CUDA_TRY(cudaMemsetAsync(err_kind.p, 0, sizeof(int), s));

    if (shard) {
        // positions of the shard's entries in list order, then their keys
        thrust::counting_iterator<uint32_t> it(0);
        InShard pred{d_src, d_dst, E, lo, hi, directed, x.n_chunks, x.chunk, x.chunk_key};
        size_t tmp_bytes = 0;
        CL_CUDA_TRY(cub::DeviceSelect::If(nullptr, tmp_bytes, it, pos.p, scal.p + 5, n_all, pred, s));
        {
            DevBuf<uint8_t> tmp;
            CL_TRY(tmp.alloc(tmp_bytes, s, "shard select temp"));
            CL_CUDA_TRY(cub::DeviceSelect::If(tmp.p, tmp_bytes, it, pos.p, scal.p + 5, n_all, pred, s));
        }
        k_shard_keys<<<grid_for(n_ent, 4), kThreads, 0, s>>>(pos.p, n_ent, d_src, d_dst, d_w, E, N, lo, keys.p);
        CL_CUDA_TRY(cudaGetLastError());
        count_launches(3);
        trace("csr: shard select+keys", s, false);
    } else {
        if (x.occ) CL_CUDA_TRY(cudaMemsetAsync(x.occ, 0, (size_t)N * sizeof(int32_t), s));
        k_validate_expand<<<grid_for(E, 4), kThreads, 0, s>>>(d_src, d_dst, d_w, E, N, x.dst_limit < 0 ? N : x.dst_limit,
                                                              directed, sentinel, keys.p, pos.p, scal.p + 0, err_kind.p,
                                                              scal.p + 1, x.n_chunks, x.chunk, x.chunk_key, x.occ);
        CL_CUDA_TRY(cudaGetLastError());
        count_launches(1);
        trace("csr: validate+expand", s, false);
    }

    // B1: stable radix sort by (src, dst) over the bits the keys use
    {
        cub::DoubleBuffer<uint64_t> kb(keys.p, keys2.p);
        cub::DoubleBuffer<uint32_t> vb(pos.p, pos2.p);
        size_t tmp_bytes = 0;
        if (keys_only)
            CL_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, kb, n_ent, 0, end_bit, s));
        else
            CL_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, n_ent, 0, end_bit, s));
        DevBuf<uint8_t> tmp;
        CL_TRY(tmp.alloc(tmp_bytes, s, "radix sort temp"));
        if (keys_only)
            CL_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, kb, n_ent, 0, end_bit, s));
        else
            CL_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kb, vb, n_ent, 0, end_bit, s));
        count_launches(2 + (end_bit + 7) / 8);            // histogram, exclusive sum, one onesweep pass per 8 bits
        if (kb.Current() != keys.p) std::swap(keys.p, keys2.p);
        if (!keys_only && vb.Current() != pos.p) std::swap(pos.p, pos2.p);
    }
    keys2.drop();
    if (keys_only) pos.drop();             // shard mode: positions only made the keys
    trace("csr: radix sort", s, true);

    // B2: run starts of equal keys, merged weights.  Over all n_ent keys (the dropped entries carry
    // the sentinel and start no run), so the validation verdict and the run count come back to the
    // host together below -- on invalid input this work is simply discarded
    DevBuf<uint8_t> flags;
    DevBuf<int64_t> run_start;
    CL_TRY(flags.alloc(n_ent, s, "head flags"));
    CL_TRY(run_start.alloc(n_ent, s, "run starts"));
    k_head_flags<<<grid_for(n_ent, 4), kThreads, 0, s>>>(keys.p, n_ent, sentinel, flags.p);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    {
        thrust::counting_iterator<int64_t> it(0);
        size_t tmp_bytes = 0;
        CL_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, flags.p, run_start.p, scal.p + 4, n_ent, s));
        DevBuf<uint8_t> tmp;
        CL_TRY(tmp.alloc(tmp_bytes, s, "select temp"));
        CL_CUDA_TRY(cub::DeviceSelect::Flagged(tmp.p, tmp_bytes, it, flags.p, run_start.p, scal.p + 4, n_ent, s));
        count_launches(2);
    }
    flags.drop();
    trace("csr: run select", s, false);

    // the merged entries are at most the sorted ones: everything below is sized for n_ent and reads the
    // real count (scal[4]) on the device, so the build's only host round trip comes after its last kernel
    DevBuf<int32_t> rows, col;
    DevBuf<double> e_ab, deg;
    DevBuf<int64_t> row_ptr;
    DevBuf<float> val;
    CL_TRY(rows.alloc(n_ent, s, "entry rows"));
    CL_TRY(col.alloc(n_ent, s, "CSR col", true));
    CL_TRY(e_ab.alloc(n_ent, s, "e_ab"));
    k_merge_runs<<<grid_for(n_ent, 4), kThreads, 0, s>>>(keys.p, pos.p, run_start.p, scal.p + 4, scal.p + 1, n_ent, d_w,
                                                         E, N, lo, rows.p, col.p, e_ab.p);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    trace("csr: merge runs", s, true);
    run_start.drop();
    keys.drop();
    pos.drop();
    pos2.drop();

    CL_TRY(row_ptr.alloc((size_t)N + 1, s, "CSR row_ptr", true));
    CL_CUDA_TRY(cudaMemsetAsync(row_ptr.p, 0, sizeof(int64_t), s));
    k_row_ptr<<<grid_for(n_ent, 4), kThreads, 0, s>>>(rows.p, scal.p + 4, N, row_ptr.p);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);

    trace("csr: row_ptr", s, true);
    CL_TRY(deg.alloc(N, s, "degree", true));
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int blocks = std::min(grid_for(N, 1), sms * 16);   // 32 rows per warp step, grid-stride
        // rows of > kDegLong entries: at most n_ent / (kDegLong + 1) of them
        const int64_t nl_max = std::max<int64_t>(1, n_ent / (kDegLong + 1));
        DevBuf<int32_t> long_rows;
        CL_TRY(long_rows.alloc(nl_max, s, "long rows"));
        k_degree<<<blocks, kThreads, 0, s>>>(row_ptr.p, e_ab.p, N, lo, hi, deg.p, scal.p + 2, scal.p + 3, long_rows.p,
                                             scal.p + 6);
        CL_CUDA_TRY(cudaGetLastError());
        if (n_ent > kDegLong) {
            const int lb = (int)std::min<int64_t>(sms * 8, (nl_max + kThreads / 32 - 1) / (kThreads / 32));
            k_degree_long<<<lb, kThreads, 0, s>>>(row_ptr.p, e_ab.p, long_rows.p, scal.p + 6, deg.p);
            CL_CUDA_TRY(cudaGetLastError());
            count_launches(1);
        }
    }
    count_launches(1);
    trace("csr: degree", s, true);
    CL_TRY(val.alloc(n_ent, s, "CSR val", true));
    k_values<<<grid_for(n_ent, 4), kThreads, 0, s>>>(rows.p, e_ab.p, deg.p, scal.p + 4, val.p);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    // one host round trip: validation verdict (first bad edge, kind) and the graph's facts (entries,
    // rows without entries, longest row).  On invalid input the work above ran on placeholder ids
    // (0) and is simply discarded.
    unsigned long long h_scal[5] = {0, 0, 0, 0, 0};
    int h_kind = 0;
    {
        const SmallRead rd[2] = {{h_scal, scal.p, 5 * sizeof(unsigned long long)}, {&h_kind, err_kind.p, sizeof(int)}};
        CL_TRY(read_small_n(rd, 2, s));
    }
    if (h_kind) {
        char buf[256];
        snprintf(buf, sizeof buf, "cleora_build: edge %llu: %s", (unsigned long long)h_scal[0],
                 (h_kind & 1) ? (x.dst_limit >= 0 ? "node id outside its range" : "node id outside [0, n_nodes)")
                              : "weight not finite or <= 0");
        return Status::make(3, buf);
    }
    out->nnz = (int64_t)h_scal[4];
    out->zero_rows = (int64_t)h_scal[2];
    out->max_degree = (int64_t)h_scal[3];
    out->d_scal = scal.release();
    out->row_ptr = row_ptr.release();
    out->col = col.release();
    out->val = val.release();
    out->deg = deg.release();
    return Status::ok();
}

Status build_schedule(const int64_t* d_row_ptr, int32_t N, int64_t r0, int64_t r1, int64_t nnz, int64_t max_degree,
                      int heavy_thresh, int chunk_rows, cudaStream_t s, Schedule* out) {
    (void)N;
    const int64_t nr = r1 - r0;
    *out = Schedule();
    {
        DevBuf<unsigned> work;
        DevBuf<int64_t> counts;
        CL_TRY(work.alloc(4, s, "work tickets", true));
        CL_TRY(counts.alloc(4, s, "schedule counts", true));
        CL_CUDA_TRY(cudaMemsetAsync(work.p, 0, 4 * sizeof(unsigned), s));
        CL_CUDA_TRY(cudaMemsetAsync(counts.p, 0, 4 * sizeof(int64_t), s));
        out->work = work.release();
        out->counts = counts.release();
    }
    if (nr <= 0) {
        out->n_heavy_rows = out->n_items = out->n_light = 0;
        return Status::ok();
    }
    {
        // light chunks (see Schedule); window from CLEORA_CHUNK_ENTRIES, default 1024 entries
        const char* e = getenv("CLEORA_CHUNK_ENTRIES");
        int64_t win = e ? atoll(e) : 1024;
        if (win < 1) win = 1;
        DevBuf<int64_t> starts;
        CL_TRY(starts.alloc(nr + 1, s, "light chunk starts", true));
        thrust::counting_iterator<int64_t> it(r0);
        // small graphs: fewer rows per chunk, so that every warp of the persistent grid gets work
        // (c1, 10k rows: 31-row chunks left most of the 2,368 warps idle and one warp walked 31
        // short rows one after another); ~4 chunks per warp of a 148-SM grid at 16 warps per SM
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // at most `chunk_rows` (the caller's, per gather engine: fewer rows per chunk keep the rows
        // in flight across the grid close to row order, so rows that share neighbours fetch them
        // close together in time -- cf. DESIGN §7)
        int64_t cap = chunk_rows;
        if (const char* cr = getenv("CLEORA_CHUNK_ROWS")) cap = atoll(cr);   // measurement override
        if (cap < 1 || cap > kChunkRows) cap = kChunkRows;
        int64_t rows = nr / ((int64_t)sms * 16 * 4);
        if (rows < 1) rows = 1;
        if (rows > cap) rows = cap;
        if (rows == 1) {
            // one row per chunk (small graphs): every row starts a chunk -- one kernel, no selection
            k_iota_starts<<<grid_for(nr + 1, 4), kThreads, 0, s>>>(starts.p, r0, nr, out->counts + 0);
            CL_CUDA_TRY(cudaGetLastError());
            count_launches(1);
        } else {
            IsChunkStart pred{d_row_ptr, r0, win, rows};
            size_t tmp_bytes = 0;
            CL_CUDA_TRY(cub::DeviceSelect::If(nullptr, tmp_bytes, it, starts.p, out->counts + 0, nr, pred, s));
            DevBuf<uint8_t> tmp;
            CL_TRY(tmp.alloc(tmp_bytes, s, "select temp"));
            CL_CUDA_TRY(cub::DeviceSelect::If(tmp.p, tmp_bytes, it, starts.p, out->counts + 0, nr, pred, s));
            k_put_end<<<1, 1, 0, s>>>(starts.p, out->counts + 0, r1);       // starts[n_light] = r1
            CL_CUDA_TRY(cudaGetLastError());
            count_launches(3);
        }
        out->light_start = starts.release();
    }
    // heavy rows: at most nnz / (heavy_thresh + 1) of them
    const int64_t nh_max = max_degree <= heavy_thresh ? 0 : std::min(nr, nnz / ((int64_t)heavy_thresh + 1));
    if (nh_max == 0) {
        out->n_heavy_rows = out->n_items = 0;
        return Status::ok();
    }
    const int64_t per_item = (int64_t)heavy_thresh * kWarpsPerCta;
    DevBuf<int64_t> hrows;
    CL_TRY(hrows.alloc(nr, s, "heavy rows"));
    {
        thrust::counting_iterator<int64_t> it(r0);
        IsHeavy pred{d_row_ptr, heavy_thresh};
        size_t tmp_bytes = 0;
        CL_CUDA_TRY(cub::DeviceSelect::If(nullptr, tmp_bytes, it, hrows.p, out->counts + 2, nr, pred, s));
        DevBuf<uint8_t> tmp;
        CL_TRY(tmp.alloc(tmp_bytes, s, "select temp"));
        CL_CUDA_TRY(cub::DeviceSelect::If(tmp.p, tmp_bytes, it, hrows.p, out->counts + 2, nr, pred, s));
        count_launches(2);
    }
    DevBuf<int64_t> nit, nsl, first, sfirst;
    CL_TRY(nit.alloc(nh_max + 1, s, "items per heavy row"));
    CL_TRY(nsl.alloc(nh_max + 1, s, "slots per heavy row"));
    CL_TRY(first.alloc(nh_max + 1, s, "first item"));
    CL_TRY(sfirst.alloc(nh_max + 1, s, "first slot"));
    k_items_per_row<<<grid_for(nh_max + 1), kThreads, 0, s>>>(d_row_ptr, hrows.p, out->counts + 2, nh_max, per_item,
                                                              nit.p, nsl.p);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    {
        size_t tb1 = 0, tb2 = 0;
        CL_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb1, nit.p, first.p, nh_max + 1, s));
        CL_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb2, nsl.p, sfirst.p, nh_max + 1, s));
        DevBuf<uint8_t> tmp;
        CL_TRY(tmp.alloc(std::max(tb1, tb2), s, "scan temp"));
        CL_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb1, nit.p, first.p, nh_max + 1, s));
        CL_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, nsl.p, sfirst.p, nh_max + 1, s));
        count_launches(4);
    }
    // upper bounds: every item but a row's last holds per_item entries; a row of several parts has
    // more than per_item entries, so its parts are fewer than 2 * entries / per_item
    out->n_items_max = nh_max + nnz / per_item + 1;
    out->n_slots_max = 2 * (nnz / per_item) + 1;
    DevBuf<HeavyItem> items;
    DevBuf<unsigned> counters;
    CL_TRY(items.alloc(out->n_items_max, s, "heavy items", true));
    CL_TRY(counters.alloc(out->n_slots_max, s, "heavy counters", true));
    CL_CUDA_TRY(cudaMemsetAsync(counters.p, 0, out->n_slots_max * sizeof(unsigned), s));
    k_fill_items<<<grid_for(nh_max), kThreads, 0, s>>>(d_row_ptr, hrows.p, out->counts + 2, nh_max, first.p, sfirst.p,
                                                       per_item, items.p, out->counts);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    out->items = items.release();
    out->counters = counters.release();
    return Status::ok();
}

namespace {
// undirected graphs: M's pattern is symmetric, so a node's in-degree is its row length
__global__ void k_row_lengths(const int64_t* __restrict__ rp, int32_t N, int32_t* __restrict__ len) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < N; v += stride)
        len[v] = (int32_t)(rp[v + 1] - rp[v]);
}
__global__ void k_indegree(const int32_t* __restrict__ col, int64_t nnz, int32_t* __restrict__ indeg) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride)
        atomicAdd(indeg + (col[k] & kColMask), 1);
}
// c[0] += #rows with indeg >= t, c[1] += #rows with indeg >= t + 1, c[2] += #rows with indeg > 0
// t = max(2, *kth) (the K-th largest in-degree, read on the device), or INT32_MAX without one
__global__ void k_count_ge(const int32_t* __restrict__ indeg, int32_t N, const int32_t* __restrict__ kth,
                           unsigned long long* __restrict__ c) {
    const int32_t t = kth ? max(*kth, 2) : INT32_MAX;
    unsigned long long a = 0, b = 0, z = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < N; v += stride) {
        const int32_t x = indeg[v];
        a += x >= t;
        b += x > t;
        z += x > 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        z += __shfl_xor_sync(0xffffffffu, z, o);
    }
    if ((threadIdx.x & 31) == 0 && (a | b | z)) {
        atomicAdd(c, a);
        atomicAdd(c + 1, b);
        atomicAdd(c + 2, z);
    }
}
__global__ void k_tag(int32_t* __restrict__ col, int64_t nnz, const int32_t* __restrict__ indeg, int32_t t) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
        const int32_t c = col[k] & kColMask;
        col[k] = indeg[c] >= t ? (int32_t)((uint32_t)c | 0x80000000u) : c;
    }
}
}  // namespace

Status in_degree(const int32_t* d_col, int64_t nnz, int32_t N, const int64_t* d_row_ptr_sym, cudaStream_t s,
                 int32_t** out) {
    DevBuf<int32_t> indeg;
    CL_TRY(indeg.alloc(N, s, "in-degree", true));
    if (d_row_ptr_sym) {
        k_row_lengths<<<grid_for(N, 4), kThreads, 0, s>>>(d_row_ptr_sym, N, indeg.p);
    } else {
        CL_CUDA_TRY(cudaMemsetAsync(indeg.p, 0, (size_t)N * 4, s));
        if (nnz > 0) k_indegree<<<grid_for(nnz, 4), kThreads, 0, s>>>(d_col, nnz, indeg.p);
    }
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    *out = indeg.release();
    return Status::ok();
}

Status hot_tag(int32_t* d_col, int64_t nnz, int32_t N, int64_t row_bytes, int64_t budget_bytes, cudaStream_t s,
               int64_t* n_hot, int64_t* n_ref, const int64_t* d_row_ptr_sym, const int32_t* d_indeg_in) {
    // hot rows = the K = budget / row_bytes rows of largest in-degree (exact threshold: the K-th
    // largest in-degree, from a radix sort of the in-degrees; ties at the threshold are kept
    // unless they overshoot the budget by more than a quarter)
    DevBuf<int32_t> indeg_own, sorted;
    DevBuf<unsigned long long> cnt;
    const int32_t* indeg = d_indeg_in;         // row-sharded builds: the whole graph's, from shard_plan
    if (!indeg) CL_TRY(indeg_own.alloc(N, s, "in-degree"));
    CL_TRY(sorted.alloc(N, s, "sorted in-degree"));
    CL_TRY(cnt.alloc(3, s, "hot count"));
    if (!indeg) {
        if (d_row_ptr_sym) {                   // no atomics (c5: 36 ms of contended hub counters)
            k_row_lengths<<<grid_for(N, 4), kThreads, 0, s>>>(d_row_ptr_sym, N, indeg_own.p);
        } else {
            CL_CUDA_TRY(cudaMemsetAsync(indeg_own.p, 0, (size_t)N * 4, s));
            k_indegree<<<grid_for(nnz, 4), kThreads, 0, s>>>(d_col, nnz, indeg_own.p);
        }
        CL_CUDA_TRY(cudaGetLastError());
        count_launches(1);
        indeg = indeg_own.p;
    }
    {
        size_t tmp_bytes = 0;
        CL_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, indeg, sorted.p, (int64_t)N, 0, 32, s));
        DevBuf<uint8_t> tmp;
        CL_TRY(tmp.alloc(tmp_bytes, s, "in-degree sort temp"));
        CL_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, indeg, sorted.p, (int64_t)N, 0, 32, s));
        count_launches(2 + 4);
    }
    int64_t K = budget_bytes / (row_bytes > 0 ? row_bytes : 1);
    if (K > N) K = N;
    // threshold t = the K-th largest in-degree, at least 2 (a row read once or never gains nothing
    // from pinning); counted on the device, then read back with the counts in one round trip
    const int32_t* kth = K > 0 ? sorted.p + (N - K) : nullptr;
    CL_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, 3 * sizeof(unsigned long long), s));
    k_count_ge<<<grid_for(N, 8), kThreads, 0, s>>>(indeg, N, kth, cnt.p);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    unsigned long long c[3];
    int32_t t = INT32_MAX;
    if (kth) {
        const SmallRead rd[2] = {{c, cnt.p, sizeof c}, {&t, kth, sizeof t}};
        CL_TRY(read_small_n(rd, 2, s));
        if (t < 2) t = 2;
    } else {
        CL_TRY(read_small(c, cnt.p, sizeof c, s));
    }
    int64_t nh = (int64_t)c[0];           // rows with in-degree >= t
    if (t != INT32_MAX && nh > K + K / 4) {
        t += 1;
        nh = (int64_t)c[1];               // rows with in-degree >= t + 1
    }
    // pin only when the hot rows are re-read far more often than the average gathered row
    // (power-law graphs); on near-regular graphs (lattices: in-degree <= 6) pinning evicts the
    // rows whose re-reads are local in time, and everything keeps the normal policy (measured:
    // c3: threshold 1.4x the mean, 2.09 ms unpinned vs 2.43 ms pinned; c2: 4.7x, 2.70 ms pinned vs
    // 2.95 ms unpinned)
    const double avg_in = c[2] ? (double)nnz / (double)c[2] : 0.0;
    if (t != INT32_MAX && (double)t < 3.0 * avg_in) t = INT32_MAX;
    if (t == INT32_MAX) nh = 0;
    *n_hot = nh;
    if (n_ref) *n_ref = (int64_t)c[2];
    if (nnz > 0) {
        k_tag<<<grid_for(nnz, 4), kThreads, 0, s>>>(d_col, nnz, indeg, t);
        count_launches(1);
    }
    CL_CUDA_TRY(cudaGetLastError());
    return Status::ok();
}

namespace {
__global__ void k_batch_ids(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t E,
                            const int64_t* __restrict__ edge_ptr, const int64_t* __restrict__ base, int32_t n_graphs,
                            int32_t* __restrict__ gsrc, int32_t* __restrict__ gdst,
                            unsigned long long* __restrict__ err_first) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += stride) {
        int lo = 0, hi = n_graphs - 1;                // graph of edge i: last g with edge_ptr[g] <= i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (edge_ptr[mid] <= i) lo = mid; else hi = mid - 1;
        }
        const int64_t b = base[lo], cnt = base[lo + 1] - b;
        const int32_t u = src[i], v = dst[i];
        if (u < 0 || u >= cnt || v < 0 || v >= cnt) {
            atomicMin(err_first, (unsigned long long)i);
            gsrc[i] = (int32_t)b;
            gdst[i] = (int32_t)b;
        } else {
            gsrc[i] = (int32_t)(b + u);
            gdst[i] = (int32_t)(b + v);
        }
    }
}
}  // namespace

Status batch_global_ids(const int32_t* d_src, const int32_t* d_dst, int64_t E, const int64_t* d_edge_ptr,
                        const int64_t* d_base, int32_t n_graphs, cudaStream_t s, int32_t* d_gsrc, int32_t* d_gdst) {
    DevBuf<unsigned long long> err;
    CL_TRY(err.alloc(1, s, "batch error"));
    CL_CUDA_TRY(cudaMemsetAsync(err.p, 0xFF, sizeof(unsigned long long), s));
    k_batch_ids<<<grid_for(E, 4), kThreads, 0, s>>>(d_src, d_dst, E, d_edge_ptr, d_base, n_graphs, d_gsrc, d_gdst, err.p);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    unsigned long long h = 0;
    CL_TRY(read_small(&h, err.p, sizeof h, s));
    if (h != ~0ull) {
        char buf[160];
        snprintf(buf, sizeof buf, "cleora_build_batch: edge %llu: node id outside [0, node_count) of its graph", h);
        return Status::make(3, buf);
    }
    return Status::ok();
}

Status shard_plan(const int32_t* d_src, const int32_t* d_dst, const float* d_w, int64_t E, int32_t N, int directed,
                  const BuildExtra* extra, int world, cudaStream_t s, int64_t* h_cuts, int64_t* h_ent,
                  int32_t** d_indeg) {
    const BuildExtra none;
    const BuildExtra& x = extra ? *extra : none;
    if ((int64_t)(directed ? E : 2 * E) >= (int64_t)UINT32_MAX)
        return Status::make(2, "cleora_build: too many edges (entry positions are 32-bit)");
    if (world + 1 > 4096 / 16) return Status::make(2, "cleora_build: world > 255 for a row-sharded build");
    DevBuf<unsigned long long> cnt, scal;
    DevBuf<int64_t> prefix, cuts, ent;
    DevBuf<int32_t> indeg;
    DevBuf<int> kind;
    CL_TRY(cnt.alloc((size_t)N + 1, s, "row entry counts"));
    CL_TRY(indeg.alloc(N, s, "in-degree", true));
    CL_TRY(scal.alloc(1, s, "scalars"));
    CL_TRY(kind.alloc(1, s, "scalars"));
    CL_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, ((size_t)N + 1) * sizeof(unsigned long long), s));
    if (directed) CL_CUDA_TRY(cudaMemsetAsync(indeg.p, 0, (size_t)N * sizeof(int32_t), s));
    CL_CUDA_TRY(cudaMemsetAsync(scal.p, 0xFF, sizeof(unsigned long long), s));
    CL_CUDA_TRY(cudaMemsetAsync(kind.p, 0, sizeof(int), s));
    if (x.occ) CL_CUDA_TRY(cudaMemsetAsync(x.occ, 0, (size_t)N * sizeof(int32_t), s));
    k_count_rows<<<grid_for(E, 4), kThreads, 0, s>>>(d_src, d_dst, d_w, E, N, directed, cnt.p, indeg.p, scal.p, kind.p,
                                                     x.n_chunks, x.chunk, x.chunk_key, x.occ);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    if (!directed) {
        k_cnt_to_indeg<<<grid_for(N, 4), kThreads, 0, s>>>(cnt.p, N, indeg.p);
        CL_CUDA_TRY(cudaGetLastError());
        count_launches(1);
    }
    CL_TRY(prefix.alloc((size_t)N + 1, s, "row entry prefix"));
    {
        size_t tmp_bytes = 0;
        const int64_t* in = reinterpret_cast<const int64_t*>(cnt.p);   // counts < 2^63: same bits
        CL_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, in, prefix.p, (int64_t)N + 1, s));
        DevBuf<uint8_t> tmp;
        CL_TRY(tmp.alloc(tmp_bytes, s, "scan temp"));
        CL_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, in, prefix.p, (int64_t)N + 1, s));
        count_launches(2);
    }
    CL_TRY(cuts.alloc(world + 1, s, "shard cuts"));
    CL_TRY(ent.alloc(world + 1, s, "shard entries"));
    k_cuts_ent<<<(world + 128) / 128, 128, 0, s>>>(prefix.p, N, world, cuts.p, ent.p);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    unsigned long long bad = 0;
    int h_kind = 0;
    {
        const SmallRead rd[4] = {{&bad, scal.p, sizeof bad}, {&h_kind, kind.p, sizeof h_kind},
                                 {h_cuts, cuts.p, (world + 1) * sizeof(int64_t)},
                                 {h_ent, ent.p, (world + 1) * sizeof(int64_t)}};
        CL_TRY(read_small_n(rd, 4, s));
    }
    if (h_kind) {
        char buf[256];
        snprintf(buf, sizeof buf, "cleora_build: edge %llu: %s", bad,
                 (h_kind & 1) ? "node id outside [0, n_nodes)" : "weight not finite or <= 0");
        return Status::make(3, buf);
    }
    *d_indeg = indeg.release();
    return Status::ok();
}

namespace {
__global__ void k_need_flags(const int32_t* __restrict__ col, int64_t nnz, uint8_t* __restrict__ need) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) need[col[k] & kColMask] = 1;
}
// mask[r] bit q = peer q (the ranks other than `rank`, in rank order) gathers row r
__global__ void k_peer_masks(const uint8_t* __restrict__ need, int32_t N, int world, int rank, uint8_t* __restrict__ mask) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride) {
        unsigned m = 0;
        for (int q = 0, p = 0; p < world; p++) {
            if (p == rank) continue;
            m |= (unsigned)(need[(int64_t)p * N + r] != 0) << q;
            q++;
        }
        mask[r] = (uint8_t)m;
    }
}
}  // namespace

Status need_flags(const int32_t* d_col, int64_t nnz, int32_t N, cudaStream_t s, uint8_t* d_need) {
    CL_CUDA_TRY(cudaMemsetAsync(d_need, 0, (size_t)N, s));
    if (nnz > 0) {
        k_need_flags<<<grid_for(nnz, 4), kThreads, 0, s>>>(d_col, nnz, d_need);
        CL_CUDA_TRY(cudaGetLastError());
        count_launches(1);
    }
    return Status::ok();
}

Status peer_masks(const uint8_t* d_need_all, int32_t N, int world, int rank, cudaStream_t s, uint8_t* d_mask) {
    k_peer_masks<<<grid_for(N, 4), kThreads, 0, s>>>(d_need_all, N, world, rank, d_mask);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    return Status::ok();
}

}  // namespace cleora
