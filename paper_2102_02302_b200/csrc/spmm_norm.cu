// spmm_norm.cu -- one Cleora iteration: T_out = normalize_rows(M . T_in), fused.
//
// Algorithm 1 lines 6-7: "T_i = M . T_{i-1}; L2 normalize rows of T_i".
// M is the CSR of D^-1 A (build.cu).  A row of the product is a weighted average of gathered
// neighbour rows of T_in ("iterated L2-normalized weighted averaging of
// neighboring nodes' representations"), so the kernel is a sparse gather-reduce, bound by
// memory traffic, not by arithmetic: no tensor cores.
//
// Schedule (chosen per row from its degree only, so the result is independent of the number
// of GPUs and bitwise reproducible run to run -- no floating-point atomics anywhere):
//   light rows (cnt <= heavy_thresh): one warp per row, 8 rows per CTA, in row-id order.
//     Lane l owns float4 columns l, l+32, ..., gathers every neighbour row with 16-byte
//     read-only loads (a warp instruction covers 512 contiguous bytes), FMAs into fp32
//     registers in ascending-k order, then reduces sum(y^2) in fp64 with warp shuffles and
//     writes y / ||y|| with 16-byte streaming stores.
//   heavy rows (cnt > heavy_thresh): CTA work items of <= 8*heavy_thresh entries; the 8 warps
//     split an item evenly, combine their partial vectors through shared memory in warp order,
//     and either normalise directly (one item) or publish the item's partial vector; the last
//     CTA to finish a row (atomic ticket) sums the partials in part order in fp64 and
//     normalises.  This is the merge-path split for power-law hubs; it also bounds every
//     sequential fp32 summation to <= heavy_thresh terms (the precision requirement of
//     SURVEY.md §0.4 / DESIGN.md §Precision).
//   Rows whose product is the zero vector (no out-edges) are written as zeros (reading RZ).
#include <mutex>

#include "common.cuh"
#include "spmm_common.cuh"

#ifndef CLEORA_V1_U
#define CLEORA_V1_U 4          // rows of <= 512 B: neighbours per load batch (8 spilled at 64 regs)
#endif
#ifndef CLEORA_V1_PAIR
#define CLEORA_V1_PAIR 16      // rows of <= 512 B: two rows of <= this many entries per warp
#endif
#ifndef CLEORA_PAIR_PU
#define CLEORA_PAIR_PU 2       // paired rows: neighbours per half-warp per step (A/B: r01 1-4 -> 3; r02 with the compiled-in stride 2-4 -> 2)
#endif
#ifndef CLEORA_V1_DPC
#define CLEORA_V1_DPC 1        // rows of exactly 512 B (dp = 128): a kernel with the stride compiled in
#endif
#ifndef CLEORA_V1_BLOCKS
#define CLEORA_V1_BLOCKS 4     // rows of <= 512 B: resident CTAs per SM
#endif

namespace cleora {

namespace {

// L2 cache policies (createpolicy): hot rows (col bit 31, see hot_tag) stay resident
// (evict_last), other gathers go first (evict_first) when hot rows exist, CSR words are streamed.
struct Pol {
    uint64_t hot, cold, csr;
};

template <bool H>
__device__ __forceinline__ Pol make_pol(const SpmmArgs& a) {
    Pol p{0, 0, 0};
    if (!H) return p;                              // no hot rows: loads without cache hints
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p.hot));
    if (a.cold_first)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p.cold));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p.cold));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p.csr));
    return p;
}

__device__ __forceinline__ float4 ldg4_pol(const float4* p, uint64_t pol) {
    float4 x;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                 : "l"(p), "l"(pol));
    return x;
}

__device__ __forceinline__ int32_t ldcsr_i32(const int32_t* p, uint64_t pol) {
    int32_t x;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(x) : "l"(p), "l"(pol));
    return x;
}

__device__ __forceinline__ float ldcsr_f32(const float* p, uint64_t pol) {
    float x;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(x) : "l"(p), "l"(pol));
    return x;
}

// H = false (no hot rows, so every gather would carry evict_normal): plain loads -- no 64-bit
// policy registers live across the row loop (at V = 1 the 64-register budget of 4 CTAs per SM
// spilled the row-loop state: ncu on the f4 batch counted ~54 local loads/stores per row)
template <bool H, int V>
__device__ __forceinline__ float4 gather4(const float4* p, int32_t ct, const Pol& pol) {
    if (H) return ldg4_pol(p, ct < 0 ? pol.hot : pol.cold);
    return __ldg(p);
}
template <bool H>
__device__ __forceinline__ int32_t csr_i32(const int32_t* p, const Pol& pol) {
    if (H) return ldcsr_i32(p, pol.csr);
    int32_t x;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(x) : "l"(p));
    return x;
}
template <bool H>
__device__ __forceinline__ float csr_f32(const float* p, const Pol& pol) {
    if (H) return ldcsr_f32(p, pol.csr);
    float x;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(x) : "l"(p));
    return x;
}

// acc[v] += sum_{k in [k0,k1)} val[k] * T_in[col[k]][cbase + 4*(lane + 32 v) .. +3], ascending k.
template <int V, bool H, int DPC = 0>
__device__ __forceinline__ void accumulate_warp(const SpmmArgs& a, const Pol& pol, int64_t k0, int64_t k1, int cbase,
                                                int lane, float4 (&acc)[V]) {
    // neighbours per batch: U*V 16-byte loads in flight
    constexpr int U = V == 1 ? CLEORA_V1_U : ((16 / V > 8) ? 8 : 16 / V);
    const int dp = DPC > 0 ? DPC : a.dp;
    bool ok[V];
#pragma unroll
    for (int v = 0; v < V; v++) ok[v] = cbase + 4 * (lane + 32 * v) < dp;
    const float* tb = a.T_in + cbase + 4 * lane;
    for (int64_t kb = k0; kb < k1; kb += 32) {
        const int n = (int)min((int64_t)32, k1 - kb);
        int32_t mc = 0;
        float mw = 0.0f;
        if (lane < n) {
            if (a.csr_prefetch) {                           // prefetched into L1 by the chunk
                mc = __ldg(a.col + kb + lane);              // bit 31: hot row
                mw = __ldg(a.val + kb + lane);
            } else {
                mc = csr_i32<H>(a.col + kb + lane, pol);
                mw = csr_f32<H>(a.val + kb + lane, pol);
            }
        }
        int j = 0;
        for (; j + U <= n; j += U) {
            float4 x[U][V];
            float w[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int ct = __shfl_sync(kFull, mc, j + u);
                w[u] = __shfl_sync(kFull, mw, j + u);
                const float4* p = reinterpret_cast<const float4*>(tb + (int64_t)(ct & kColMask) * dp);
#pragma unroll
                for (int v = 0; v < V; v++)
                    x[u][v] = ok[v] ? gather4<H, V>(p + 32 * v, ct, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int v = 0; v < V; v++) fma4(acc[v], w[u], x[u][v]);
        }
        for (; j < n; j++) {
            const int ct = __shfl_sync(kFull, mc, j);
            const float w = __shfl_sync(kFull, mw, j);
            const float4* p = reinterpret_cast<const float4*>(tb + (int64_t)(ct & kColMask) * dp);
#pragma unroll
            for (int v = 0; v < V; v++)
                if (ok[v]) fma4(acc[v], w, gather4<H, V>(p + 32 * v, ct, pol));
        }
    }
}

template <int V, bool H, int DPC = 0>
__device__ void light_row(const SpmmArgs& a, const Pol& pol, int64_t row, int64_t k0, int64_t k1, int lane) {
    constexpr int SW = 128 * V;                   // floats per column slice
    const int dp = DPC > 0 ? DPC : a.dp;
    const int ns = (dp + SW - 1) / SW;
    if (k1 == k0 && a.skip_zero_rows) return;     // already 0 in T_out (reading RZ)
    float4* out = reinterpret_cast<float4*>(a.T_out + row * (int64_t)dp);
    double ss = 0.0;
    float4 acc[V];
    for (int sl = 0; sl < ns; sl++) {
        const int cbase = sl * SW;
#pragma unroll
        for (int v = 0; v < V; v++) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        accumulate_warp<V, H, DPC>(a, pol, k0, k1, cbase, lane, acc);
#pragma unroll
        for (int v = 0; v < V; v++) {
            const int f = cbase / 4 + lane + 32 * v;
            if (4 * f < dp) {
                ss += sq4(acc[v]);
                if (ns > 1) out[f] = acc[v];      // unnormalised; rescaled below
            }
        }
    }
    ss = warp_sum(ss);
    const double inv = inv_norm(ss);
    if (ns == 1) {
#pragma unroll
        for (int v = 0; v < V; v++) {
            const int f = lane + 32 * v;
            if (4 * f < dp) put_out4(a, row, f, scale4(acc[v], inv), k1 == k0);
        }
    } else {
        for (int f = lane; 4 * f < dp; f += 32) put_out4(a, row, f, scale4(out[f], inv), k1 == k0);
    }
}

// Rows of <= 512 B (dp <= 128): two rows per warp, one per half-warp.  Lane hl of half h owns the
// float4 columns hl and hl + 16 of row `row`; each loop step gathers PU neighbours of BOTH rows, so the
// shuffles, address math and loop control of one step serve two rows (ncu on the f4 batch: ~52
// instructions per entry with one row per warp, bound by issue).  Bitwise the same result as
// light_row<1>: every element is the same ascending-k fp32 FMA chain, and Σy² is the same fp64
// tree -- lane hl adds its two columns (= the xor-16 step of the 32-lane butterfly), then the
// xor 8/4/2/1 steps stay inside the half.  `live` = false: this half has no row (odd tail, heavy
// row); it still executes every shuffle.
// DPC: the row stride as a compile-time constant (128: f4 batches, c1), 0 = a.dp at run time
template <bool H, int DPC>
__device__ void light_row_pair(const SpmmArgs& a, const Pol& pol, int64_t row, int64_t k0, int64_t k1, bool live,
                               int lane) {
    constexpr int PU = CLEORA_PAIR_PU;             // neighbours per half per step
    const int hl = lane & 15, base = lane & 16;
    const int dp = DPC > 0 ? DPC : a.dp;
    const bool ok0 = 4 * hl < dp, ok1 = 4 * (hl + 16) < dp;
    const int64_t n_row = live ? k1 - k0 : 0;
    const int64_t n_max = max(n_row, __shfl_xor_sync(kFull, n_row, 16));
    if (n_max == 0 && a.skip_zero_rows) return;    // both rows already 0 in T_out (reading RZ)
    float4 acc0 = make_float4(0.f, 0.f, 0.f, 0.f), acc1 = acc0;
    const float* tb = a.T_in + 4 * hl;
    for (int64_t kb = 0; kb < n_max; kb += 16) {
        const int n = (int)max((int64_t)0, min((int64_t)16, n_row - kb));   // this half's entries here
        const int nb = (int)min((int64_t)16, n_max - kb);                   // warp-uniform
        int32_t mc = 0;
        float mw = 0.0f;
        if (hl < n) {
            if (a.csr_prefetch) {
                mc = __ldg(a.col + k0 + kb + hl);
                mw = __ldg(a.val + k0 + kb + hl);
            } else {
                mc = csr_i32<H>(a.col + k0 + kb + hl, pol);
                mw = csr_f32<H>(a.val + k0 + kb + hl, pol);
            }
        }
        for (int j = 0; j < nb; j += PU) {
            float4 x[PU][2];
            float w[PU];
#pragma unroll
            for (int u = 0; u < PU; u++) {
                const bool act = j + u < n;
                const int src = base + (j + u < 16 ? j + u : 0);
                const int ct = __shfl_sync(kFull, mc, src);
                w[u] = __shfl_sync(kFull, mw, src);
                const float4* p = reinterpret_cast<const float4*>(tb + (int64_t)(ct & kColMask) * dp);
                x[u][0] = act && ok0 ? gather4<H, 1>(p, ct, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
                x[u][1] = act && ok1 ? gather4<H, 1>(p + 16, ct, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < PU; u++)
                if (j + u < n) {
                    fma4(acc0, w[u], x[u][0]);
                    fma4(acc1, w[u], x[u][1]);
                }
        }
    }
    double ss = 0.0;
    if (ok0) ss += sq4(acc0);
    if (ok1) ss += sq4(acc1);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
    if (!live || (n_row == 0 && a.skip_zero_rows)) return;
    const double inv = inv_norm(ss);
    if (ok0) put_out4(a, row, hl, scale4(acc0, inv), n_row == 0);
    if (ok1) put_out4(a, row, hl + 16, scale4(acc1, inv), n_row == 0);
}

template <int V, bool H>
__device__ void heavy_item(const SpmmArgs& a, const Pol& pol, int64_t idx, float4* red, double* scratch, int* flag) {
    constexpr int SW = 128 * V;
    constexpr int Q = 32 * V;                     // float4 per slice
    const HeavyItem it = a.items[idx];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
    const int dp = a.dp, nq = dp / 4;
    const int ns = (dp + SW - 1) / SW;
    const int64_t len = it.k1 - it.k0;
    const int64_t sub = (len + kWarpsPerCta - 1) / kWarpsPerCta;
    const int64_t wk0 = min(it.k0 + warp * sub, it.k1), wk1 = min(wk0 + sub, it.k1);
    const bool single = it.nparts == 1;
    float4* dst = reinterpret_cast<float4*>(single ? a.T_out + (int64_t)it.row * dp : a.partials + (int64_t)it.slot * dp);

    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    double ss = 0.0;
    for (int sl = 0; sl < ns; sl++) {
        float4 acc[V];
#pragma unroll
        for (int v = 0; v < V; v++) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        accumulate_warp<V, H>(a, pol, wk0, wk1, sl * SW, lane, acc);
#pragma unroll
        for (int v = 0; v < V; v++) red[warp * Q + lane + 32 * v] = acc[v];
        __syncthreads();
        if (t < Q) {
            const int f = sl * Q + t;
            float4 s = red[t];
#pragma unroll
            for (int w = 1; w < kWarpsPerCta; w++) {   // warp order: deterministic
                const float4 r = red[w * Q + t];
                s.x += r.x; s.y += r.y; s.z += r.z; s.w += r.w;
            }
            y = s;
            if (f < nq) {
                ss += sq4(y);
                if (!(single && ns == 1)) dst[f] = y;
            }
        }
        __syncthreads();
    }
    if (single) {
        const double tot = block_sum(ss, scratch);
        const double inv = inv_norm(tot);
        if (ns == 1) {
            if (t < Q && t < nq) put_out4(a, it.row, t, scale4(y, inv));
        } else {
            __syncthreads();   // dst (= this row of T_out) holds the unnormalised slices
            for (int f = t; f < nq; f += blockDim.x) put_out4(a, it.row, f, scale4(dst[f], inv));
        }
        return;
    }
    // publish this part; the last CTA of the row finishes it
    __threadfence();
    __syncthreads();
    if (t == 0) {
        const unsigned prev = atomicAdd(a.counters + (it.slot - it.part), 1u);
        *flag = (prev == (unsigned)it.nparts - 1) ? 1 : 0;
    }
    __syncthreads();
    if (!*flag) return;
    __threadfence();
    const int64_t first = it.slot - it.part;
    const float4* parts = reinterpret_cast<const float4*>(a.partials + first * (int64_t)dp);
    const int64_t pstride = dp / 4;
    double zx = 0, zy = 0, zz = 0, zw = 0;
    double ss2 = 0.0;
    for (int f = t; f < nq; f += blockDim.x) {
        zx = zy = zz = zw = 0.0;
        for (int q = 0; q < it.nparts; q++) {     // part order: deterministic
            const float4 p = __ldcg(parts + q * pstride + f);
            zx += p.x; zy += p.y; zz += p.z; zw += p.w;
        }
        ss2 += zx * zx + zy * zy + zz * zz + zw * zw;
    }
    const double tot = block_sum(ss2, scratch);
    const double inv = inv_norm(tot);
    if (nq <= (int)blockDim.x) {
        if (t < nq)
            put_out4(a, it.row, t,
                     make_float4((float)(zx * inv), (float)(zy * inv), (float)(zz * inv), (float)(zw * inv)));
    } else {
        for (int f = t; f < nq; f += blockDim.x) {
            zx = zy = zz = zw = 0.0;
            for (int q = 0; q < it.nparts; q++) {
                const float4 p = __ldcg(parts + q * pstride + f);
                zx += p.x; zy += p.y; zz += p.z; zw += p.w;
            }
            put_out4(a, it.row, f,
                     make_float4((float)(zx * inv), (float)(zy * inv), (float)(zz * inv), (float)(zw * inv)));
        }
    }
    if (t == 0) a.counters[first] = 0u;           // ready for the next launch
}

// Persistent kernel: one wave of CTAs (SM count x resident CTAs per SM).  Work is handed out
// dynamically through global tickets so that no warp waits for another: CTAs first take heavy
// items one at a time (a.work[0]); then every warp takes light chunks (<= 31 consecutive rows)
// (a.work[1]).  The last warp to finish resets the tickets (a.work[2] counts finished warps), so
// the counters are 0 again at the next launch.  Which warp computes a row never changes its
// arithmetic, so results stay bitwise deterministic.

// rows of <= 512 bytes (V = 1) are latency-bound with one row at a time per warp: 4 CTAs (32 warps)
// per SM at <= 64 registers; wider rows need the registers for their accumulators (2 CTAs)
template <int V>
constexpr int kNormMinBlocks = V == 1 ? CLEORA_V1_BLOCKS : 2;   // V = 2 at 3 CTAs spills: c5 357 -> 478 ms

template <int V, bool H, int DPC>
__global__ void __launch_bounds__(kWarpsPerCta * 32, kNormMinBlocks<V>) k_spmm_norm(const SpmmArgs a) {
    extern __shared__ float4 red[];
    __shared__ double scratch[kWarpsPerCta];
    __shared__ int flag;
    __shared__ unsigned s_item;
    const int lane = threadIdx.x & 31;
    const Pol pol = make_pol<H>(a);               // once per thread, not per row
    const int64_t n_items = a.n_items_max > 0 ? a.counts[1] : 0;   // schedule counts live on the device
    if (n_items > 0) {
        for (;;) {
            if (threadIdx.x == 0) s_item = atomicAdd(a.work + 0, 1u);
            __syncthreads();
            const int64_t it = s_item;
            __syncthreads();
            if (it >= n_items) break;
            heavy_item<V, H>(a, pol, it, red, scratch, &flag);
        }
    }
    const int64_t nchunks = a.counts[0];
    // few chunks (small graphs: c1 has ~10k one-row chunks for 4,736 warps): static round robin --
    // warp w takes chunks w, w + W, ...; a grid-wide ticket would serialise ~15k atomics on one L2
    // address, the longest part of such a launch.  Otherwise the ticket balances uneven rows.
    const int64_t nw = (int64_t)gridDim.x * kWarpsPerCta;
    const bool stat = nchunks <= 4 * nw;
    int64_t sc = (int64_t)blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
    for (;;) {
        unsigned c = 0;
        if (stat) {
            if (sc >= nchunks) break;
            c = (unsigned)sc;
            sc += nw;
        } else {
            if (lane == 0) c = atomicAdd(a.work + 1, 1u);
            c = __shfl_sync(kFull, c, 0);
            if ((int64_t)c >= nchunks) break;
        }
        const int64_t rb = a.light_start[c];
        const int64_t re = a.light_start[c + 1];
        const int64_t rpl = (lane <= re - rb) ? a.row_ptr[rb + lane] : 0;
        if (a.csr_prefetch) {
            // bring the chunk's CSR words into L1 up front, so each row's col/val load is an L1 hit
            // instead of one more dependent memory round trip per (short) row
            const int64_t eb = __shfl_sync(kFull, rpl, 0), ee = __shfl_sync(kFull, rpl, (int)(re - rb));
            if (ee - eb <= 4096)
                for (int64_t off = (eb & ~31ll) + 32 * lane; off < ee; off += 32 * 32) {
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(a.col + off));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(a.val + off));
                }
        }
        if constexpr (V == 1 && CLEORA_V1_PAIR > 0) {
            // two consecutive short rows (<= CLEORA_V1_PAIR entries each) share the warp, one per
            // half; a longer row runs alone (pairing it with a short one would idle half the warp)
            for (int64_t r = rb; r < re;) {
                const int i = (int)(r - rb);
                const int64_t e0 = __shfl_sync(kFull, rpl, i), e1 = __shfl_sync(kFull, rpl, i + 1);
                const bool two = r + 1 < re;
                const int64_t e2 = __shfl_sync(kFull, rpl, two ? i + 2 : i + 1);
                const int64_t lim = min((int64_t)CLEORA_V1_PAIR, (int64_t)a.heavy_thresh);
                if (two && e1 - e0 <= lim && e2 - e1 <= lim) {
                    const bool hi = lane >= 16;
                    light_row_pair<H, DPC>(a, pol, r + (hi ? 1 : 0), hi ? e1 : e0, hi ? e2 : e1, true, lane);
                    r += 2;
                } else {
                    if (e1 - e0 <= a.heavy_thresh) light_row<V, H, DPC>(a, pol, r, e0, e1, lane);
                    r += 1;
                }
            }
        } else {
            for (int64_t r = rb; r < re; r++) {
                const int64_t k0 = __shfl_sync(kFull, rpl, (int)(r - rb));
                const int64_t k1 = __shfl_sync(kFull, rpl, (int)(r - rb + 1));
                if (k1 - k0 > a.heavy_thresh) continue;
                light_row<V, H>(a, pol, r, k0, k1, lane);
            }
        }
    }
    // peer stores (multi-GPU) are system-scope visible before this launch counts as done; the
    // rank barrier that follows on the stream then publishes them to the other ranks
    if (a.n_peers > 0) __threadfence_system();
    if (stat && n_items == 0) return;             // no ticket was taken: nothing to reset
    if (lane == 0) {
        __threadfence();
        const unsigned done = atomicAdd(a.work + 2, 1u);
        if (done == gridDim.x * kWarpsPerCta - 1) {
            a.work[0] = 0u;
            a.work[1] = 0u;
            a.work[2] = 0u;
        }
    }
}

template <int V, bool H, int DPC = 0>
Status launch_vh(const SpmmArgs& a, cudaStream_t s) {
    const size_t smem = (size_t)kWarpsPerCta * 32 * V * sizeof(float4);
    // per device: the smem attribute and the occupancy are per device
    static int bps[kMaxDevices], nsm[kMaxDevices];
    static std::mutex mu;
    int dev = 0;
    CL_CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= kMaxDevices) return Status::make(4, "k_spmm_norm: device ordinal beyond kMaxDevices");
    int blocks_per_sm = 0, sms = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!bps[dev]) {
            CL_CUDA_TRY(cudaFuncSetAttribute(k_spmm_norm<V, H, DPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CL_CUDA_TRY(cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev));
            int b = 0;
            CL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_spmm_norm<V, H, DPC>, kWarpsPerCta * 32, smem));
            bps[dev] = b < 1 ? 1 : b;
        }
        blocks_per_sm = bps[dev];
        sms = nsm[dev];
    }
    if (a.r1 <= a.r0 && a.n_items_max == 0) return Status::ok();
    const int grid = sms * blocks_per_sm;                // one persistent wave
    k_spmm_norm<V, H, DPC><<<grid, kWarpsPerCta * 32, smem, s>>>(a);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    return Status::ok();
}

// cache hints only when there are hot rows (a.cold_first: hot_tag pinned some rows)
template <int V>
Status launch_v(const SpmmArgs& a, cudaStream_t s) {
    if (CLEORA_V1_DPC && V == 1 && a.dp == 128)   // full 512 B rows: no per-column bounds, shifts for addresses
        return a.cold_first ? launch_vh<V, true, 128>(a, s) : launch_vh<V, false, 128>(a, s);
    if (CLEORA_V1_DPC && V == 1 && a.dp == 64)
        return a.cold_first ? launch_vh<V, true, 64>(a, s) : launch_vh<V, false, 64>(a, s);
    return a.cold_first ? launch_vh<V, true>(a, s) : launch_vh<V, false>(a, s);
}

}  // namespace

Status launch_spmm_norm(const SpmmArgs& a, cudaStream_t s) {
    if (a.gather_mode != kGatherLdg || a.pass > 0) return launch_spmm_tma(a, s);
    if (a.dp <= 128) return launch_v<1>(a, s);
    if (a.dp <= 256) return launch_v<2>(a, s);
    if (a.dp <= 512) return launch_v<4>(a, s);
    return launch_v<8>(a, s);
}

}  // namespace cleora
