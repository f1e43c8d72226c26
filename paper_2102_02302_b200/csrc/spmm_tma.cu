// spmm_tma.cu -- one Cleora iteration T_out = normalize_rows(M . T_in), gathering neighbour rows
// through a shared-memory ring.
//
// Algorithm 1 lines 6-7.  Same schedule and arithmetic as spmm_norm.cu (the path
// for rows <= 512 B and > 4 KB), but the neighbour rows are not loaded through registers: each warp
// owns a ring of S shared-memory slots, one row of T_in (dp*4 bytes) per slot, filled S entries
// ahead of the consumer either by 1-D TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx,
// issued by lane 0; 4 KB rows) or by per-lane 16-byte cp.async (0.5-4 KB rows, where the bulk-copy
// engine's issue rate binds; see gather_mode).  Bytes in flight are therefore bounded by shared
// memory (~190 KB per SM) instead of the register file, which is what a latency-bound gather
// needs; registers only hold the fp32 accumulator (dp/32 floats per lane).
//
// Light rows (<= heavy_thresh entries): a warp takes a ticket for a light chunk (<= 31 consecutive
// rows, entry-bounded, see Schedule) and streams their entries flat through its ring -- the
// pipeline keeps running across row boundaries, where the finished row is reduced (fp64 sum of
// squares, warp shuffles), scaled and written with 16-byte streaming stores (and, multi-GPU, into
// every peer replica).  Heavy rows: CTA work items; each warp streams a contiguous sub-range, the 8
// partial vectors are combined through shared memory in warp order, and multi-item rows finish in
// the last CTA (atomic ticket) with an fp64 sum in part order.  Each row accumulates its entries
// in ascending order from 0, exactly as spmm_norm.cu does, so every engine produces bitwise
// identical results (tested).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "spmm_common.cuh"

namespace cleora {

namespace {

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}


__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            saddr(dst)),
        "l"(src), "r"(bytes), "r"(saddr(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// streamed-once CSR words: no L1 allocation, first out of L2
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p, uint64_t pol) {
    int32_t x;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(x) : "l"(p), "l"(pol));
    return x;
}
__device__ __forceinline__ float ld_stream_f32(const float* p, uint64_t pol) {
    float x;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(x) : "l"(p), "l"(pol));
    return x;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(saddr(bar)),
        "r"(parity)
        : "memory");
}


struct Ring {
    float4* buf;       // S slots of slot_f4 float4
    uint64_t* bar;     // S mbarriers (arrival count 1: lane 0's arrive.expect_tx)
    int S;
    int slot_f4;
    uint32_t bytes;    // dp * 4
    int cs;            // next slot to consume
    uint32_t ph;       // parity bit of each slot
    uint64_t pol_hot;  // L2 policy for gathers of hot rows (evict_last)
    uint64_t pol_cold; // ... of all other rows (evict_normal; evict_first with a.cold_first)
    uint64_t pol_csr;  // streamed-once CSR words (evict_first)
};

// c: column index, bit 31 set when the row is "hot" (high in-degree, see hot_tag in build.cu):
// hot rows are gathered with an evict_last L2 policy so the most re-read rows stay resident.
//
// Two ways to fill a slot.  SA == 0: lane 0 issues one 1-D bulk copy (TMA, cp.async.bulk) that
// completes on the slot's mbarrier.  SA > 0 (rows below 2 KB, where the bulk-copy engine's issue
// rate binds): every lane copies its own float4 columns with 16-byte cp.async (LDGSTS) and
// commits one cp.async group per slot; a lane only ever reads the columns it copied, so
// `cp.async.wait_group SA-1` (all but the SA-1 most recent groups complete) is the whole
// handshake.  Exactly one group is committed per issue -- an empty one past the end of the
// stream -- so that positional wait always names the slot being consumed.
template <int V, bool FULL, int SA, bool HALF>
__device__ __forceinline__ void ring_issue(const SpmmArgs& a, Ring& r, int slot, int32_t c, int lane) {
    // a.dp is the row stride; half-row passes gather 128 * V floats starting at column 512 * (pass == 2)
    const int64_t col0 = (HALF && a.pass == 2) ? 128 * V : 0;
    if (SA > 0) {
        const int dp = FULL ? 128 * V : a.dp;     // gathered width
        const float4* src = reinterpret_cast<const float4*>(a.T_in + (int64_t)(c & 0x7fffffff) * a.dp + col0) + lane;
        float4* dst = r.buf + (size_t)slot * r.slot_f4 + lane;
        const uint64_t pol = c < 0 ? r.pol_hot : r.pol_cold;
#pragma unroll
        for (int v = 0; v < V; v++)
            if (FULL || 4 * (lane + 32 * v) < dp)
                asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(saddr(dst + 32 * v)),
                             "l"(src + 32 * v), "l"(pol)
                             : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        return;
    }
    if (lane == 0) {
        mbar_expect_tx(r.bar + slot, r.bytes);
        bulk_g2s_hint(r.buf + (size_t)slot * r.slot_f4, a.T_in + (int64_t)(c & 0x7fffffff) * a.dp + col0, r.bytes,
                      r.bar + slot, c < 0 ? r.pol_hot : r.pol_cold);
    }
}

template <int SA>
__device__ __forceinline__ void ring_skip() {       // keep one group per issue (see ring_issue)
    if (SA > 0) asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int SA>
__device__ __forceinline__ void ring_wait(Ring& r, int sl) {
    if (SA > 0) {
        asm volatile("cp.async.wait_group %0;" ::"n"(SA > 0 ? SA - 1 : 0) : "memory");
    } else {
        mbar_wait(r.bar + sl, (r.ph >> sl) & 1u);
        r.ph ^= 1u << sl;
    }
}

// `empty`: the row has no entries (its output is the zero vector, reading RZ); with
// a.skip_zero_rows the zeros are already in T_out and nothing is written.
//
// Half-row passes (a.pass, V = 4 of the whole row's 8 float4 per lane): pass 1 stores the first half
// of y unnormalised into T_out (empty rows: nothing); pass 2 reads that half back, continues the
// lane's sum of squares over v = 0..3 (first half) then 4..7 (its own) -- the whole-row kernel's
// order --, so the row scale, and every output bit, are the whole-row kernel's.
template <int V, bool FULL, bool HALF>
__device__ __forceinline__ void finalize_row_t(const SpmmArgs& a, int64_t row, float4 (&acc)[V], int lane,
                                               bool empty) {
    const int dp = FULL ? 128 * V : a.dp;
    if (empty && a.skip_zero_rows) return;           // acc is still all zeros
    // a lazy step's never-gathered row (a.drop_rows): nothing to store, the call's last step computes it
    const bool drop = HALF && !empty && a.drop_rows && __ldg(a.drop_rows + row) == 0;
    if (HALF && a.pass == 1) {
        if (!empty && !drop) {
            if (a.ss_half) {                         // lazy step: this half's sum of squares for pass 2, and
                double ss = 0.0;                     // the half itself, unnormalised, to the peers as well
#pragma unroll
                for (int v = 0; v < V; v++) ss += sq4(acc[v]);
                ss = warp_sum(ss);
                if (lane == 0) a.ss_half[row] = ss;
#pragma unroll
                for (int v = 0; v < V; v++) put_out4(a, row, lane + 32 * v, acc[v]);
            } else {
                float4* out = reinterpret_cast<float4*>(a.T_out + row * (int64_t)a.dp);
#pragma unroll
                for (int v = 0; v < V; v++) __stcg(out + lane + 32 * v, acc[v]);
            }
        }
#pragma unroll
        for (int v = 0; v < V; v++) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    if (HALF && a.pass == 2 && a.lazy_out) {
        // lazy step: both halves stay unnormalised in T_out (the first from pass 1), the row scale goes
        // to the row scales -- no read-back and rewrite of the first half (c4: 2 x 4.7 GB per step)
        if (drop) {                                  // warp-uniform (one row per warp)
#pragma unroll
            for (int v = 0; v < V; v++) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            return;
        }
        double ss = 0.0;
#pragma unroll
        for (int v = 0; v < V; v++) ss += sq4(acc[v]);
        ss = warp_sum(ss);
        if (!empty) ss += __ldcg(a.ss_half + row);
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int v = 0; v < V; v++) {
            if (empty) put_out4(a, row, lane + 32 * v, z, true);
            put_out4(a, row, 32 * V + lane + 32 * v, acc[v], empty);
            acc[v] = z;
        }
        if (lane == 0) put_scale(a, row, (float)inv_norm(ss), empty);
        return;
    }
    if (HALF && a.pass == 2) {
        float4 h[V];
        const float4* out = reinterpret_cast<const float4*>(a.T_out + row * (int64_t)a.dp);
#pragma unroll
        for (int v = 0; v < V; v++) h[v] = empty ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldcg(out + lane + 32 * v);
        double ss = 0.0;
#pragma unroll
        for (int v = 0; v < V; v++) ss += sq4(h[v]);
#pragma unroll
        for (int v = 0; v < V; v++) ss += sq4(acc[v]);
        ss = warp_sum(ss);
        const double inv = inv_norm(ss);
#pragma unroll
        for (int v = 0; v < V; v++) {
            put_out4(a, row, lane + 32 * v, scale4(h[v], inv), empty);
            put_out4(a, row, 32 * V + lane + 32 * v, scale4(acc[v], inv), empty);   // float4 index in the row
            acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        return;
    }
    double ss = 0.0;
#pragma unroll
    for (int v = 0; v < V; v++)
        if (FULL || 4 * (lane + 32 * v) < dp) ss += sq4(acc[v]);
    ss = warp_sum(ss);
    const double inv = inv_norm(ss);
#pragma unroll
    for (int v = 0; v < V; v++) {
        const int f = lane + 32 * v;
        if (FULL || 4 * f < dp) put_out4(a, row, f, scale4(acc[v], inv), empty);
        acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// Stream CSR entries [E0, E1) through the warp's ring into acc.  ROWS: the entries belong to
// rows [ra, rz) whose bounds are in rpl (lane i holds row_ptr[rb + i]); rows are finalised at
// their boundaries (zero rows included).  On return every issued copy has been consumed.
template <int V, bool FULL, bool ROWS, int SA, bool HALF>
__device__ void stream_entries(const SpmmArgs& a, Ring& r, int64_t E0, int64_t E1, float4 (&acc)[V], int64_t rb,
                               int64_t rpl, int64_t ra, int64_t rz, int lane) {
    const int dp = FULL ? 128 * V : a.dp;
    int64_t row = ra;
    int64_t kend = ROWS ? __shfl_sync(kFull, rpl, (int)(ra - rb + 1)) : E1;
    const int32_t* colp = a.col;   // bit 31 = hot tag (ring_issue picks the L2 policy from it)
    int32_t mc0 = 0, mc1 = 0;
    float mw0 = 0.f, mw1 = 0.f;
    if (E0 + lane < E1) {
        mc0 = ld_stream_i32(colp + E0 + lane, r.pol_csr);
        mw0 = ld_stream_f32(a.val + E0 + lane, r.pol_csr);
    }
    if (E0 + 32 + lane < E1) {
        mc1 = ld_stream_i32(colp + E0 + 32 + lane, r.pol_csr);
        mw1 = ld_stream_f32(a.val + E0 + 32 + lane, r.pol_csr);
    }
    // prologue: the first min(S, n) entries (cp.async mode: S groups, empty ones past the end)
    {
        const int pro = (int)min((int64_t)r.S, E1 - E0);
        int sl = r.cs;
        for (int i = 0; i < pro; i++) {
            const int32_t c = __shfl_sync(kFull, mc0, i);
            ring_issue<V, FULL, SA, HALF>(a, r, sl, c, lane);
            sl = (sl + 1 == r.S) ? 0 : sl + 1;
        }
        for (int i = pro; i < (SA > 0 ? SA : 0); i++) ring_skip<SA>();
    }
    for (int64_t kb = E0; kb < E1; kb += 32) {
        const int n = (int)min((int64_t)32, E1 - kb);
        for (int j = 0; j < n; j++) {
            const int64_t e = kb + j;
            if (ROWS) {
                while (e >= kend) {                       // row boundary (warp-uniform)
                    const int64_t kbeg = __shfl_sync(kFull, rpl, (int)(row - rb));
                    finalize_row_t<V, FULL, HALF>(a, row, acc, lane, kbeg == kend);
                    row++;
                    kend = __shfl_sync(kFull, rpl, (int)(row - rb + 1));
                }
            }
            const float w = __shfl_sync(kFull, mw0, j);
            const int sl = r.cs;
            ring_wait<SA>(r, sl);
            const float4* src = r.buf + (size_t)sl * r.slot_f4 + lane;
#pragma unroll
            for (int v = 0; v < V; v++)
                if (FULL || 4 * (lane + 32 * v) < dp) fma4(acc[v], w, src[32 * v]);
            __syncwarp();
            // refill the slot just consumed with entry e + S (S <= 32, so it is in block 0 or 1)
            const int jp = j + r.S;
            const int32_t cp = (jp < 32) ? __shfl_sync(kFull, mc0, jp) : __shfl_sync(kFull, mc1, jp - 32);
            if (e + r.S < E1)
                ring_issue<V, FULL, SA, HALF>(a, r, sl, cp, lane);
            else
                ring_skip<SA>();
            r.cs = (sl + 1 == r.S) ? 0 : sl + 1;
        }
        mc0 = mc1;
        mw0 = mw1;
        mc1 = 0;
        mw1 = 0.f;
        if (kb + 64 + lane < E1) {
            mc1 = ld_stream_i32(colp + kb + 64 + lane, r.pol_csr);
            mw1 = ld_stream_f32(a.val + kb + 64 + lane, r.pol_csr);
        }
    }
    if (ROWS) {
        while (row < rz) {                                // last row and trailing zero rows
            const int64_t kbeg = __shfl_sync(kFull, rpl, (int)(row - rb));
            const int64_t kfin = __shfl_sync(kFull, rpl, (int)(row - rb + 1));
            finalize_row_t<V, FULL, HALF>(a, row, acc, lane, kbeg == kfin);
            row++;
        }
    }
}

template <int V, bool FULL, int SA, bool HALF>
__device__ void heavy_item_t(const SpmmArgs& a, int64_t idx, Ring& r, float4* smem, int ring_f4, double* scratch,
                             int* flag) {
    const HeavyItem it = a.items[idx];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
    const int dp = FULL ? 128 * V : a.dp;
    const int nq = dp / 4;
    const int64_t len = it.k1 - it.k0;
    const int64_t sub = (len + kWarpsPerCta - 1) / kWarpsPerCta;
    const int64_t wk0 = min(it.k0 + warp * sub, it.k1), wk1 = min(wk0 + sub, it.k1);
    float4 acc[V];
#pragma unroll
    for (int v = 0; v < V; v++) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    stream_entries<V, FULL, false, SA, HALF>(a, r, wk0, wk1, acc, 0, 0, 0, 0, lane);
    // this warp's partial vector -> slot 0 of its ring (drained), combined in warp order
    float4* red = r.buf;
#pragma unroll
    for (int v = 0; v < V; v++)
        if (FULL || 4 * (lane + 32 * v) < dp) red[lane + 32 * v] = acc[v];
    __syncthreads();
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    double ss = 0.0;
    if (HALF) {
        // half-row passes: thread t stands for float4 t of the WHOLE row, as in the whole-row kernel
        // (blockDim = 256 = a.dp / 4).  Pass 1 combines the first half (t < 128); pass 2 the second
        // half (t >= 128) and takes the first from T_out (single-part rows) or the partials (below).
        const int half = 128 * V / 4;                 // float4 per half row
        const bool mine = a.pass == 1 ? t < half : t >= half;
        const int tc = a.pass == 1 ? t : t - half;
        if (mine) {
            y = smem[tc];
#pragma unroll
            for (int w = 1; w < kWarpsPerCta; w++) {
                const float4 q = smem[(size_t)w * ring_f4 + tc];
                y.x += q.x; y.y += q.y; y.z += q.z; y.w += q.w;
            }
        }
        // a lazy step's never-gathered row (a.drop_rows): stores skipped, block-uniform
        const bool drop = a.drop_rows && __ldg(a.drop_rows + it.row) == 0;
        if (it.nparts == 1) {
            float4* outr = reinterpret_cast<float4*>(a.T_out + (int64_t)it.row * a.dp);
            if (a.pass == 1) {
                if (mine && !drop) {
                    if (a.ss_half) put_out4(a, it.row, t, y);   // lazy step: the peers get the half too
                    else __stcg(outr + t, y);
                }
            } else {
                if (!mine) y = __ldcg(outr + t);
                const double tot = block_sum(sq4(y), scratch);
                const double inv = inv_norm(tot);
                if (a.lazy_out) {                     // lazy step: unnormalised, the scale aside
                    if (mine && !drop) put_out4(a, it.row, t, y);
                    if (t == 0 && !drop) put_scale(a, it.row, (float)inv);
                } else {
                    put_out4(a, it.row, t, scale4(y, inv));
                }
            }
        } else {
            float4* part = reinterpret_cast<float4*>(a.partials + (int64_t)it.slot * a.dp);
            if (mine) part[t] = y;
            if (a.pass == 2) {
                __threadfence();
                __syncthreads();
                if (t == 0) {
                    const unsigned prev = atomicAdd(a.counters + (it.slot - it.part), 1u);
                    *flag = (prev == (unsigned)it.nparts - 1) ? 1 : 0;
                }
                __syncthreads();
                if (*flag) {                          // the whole-row kernel's finish, over the whole row
                    __threadfence();
                    const int nqf = a.dp / 4;
                    const float4* parts = reinterpret_cast<const float4*>(a.partials + (int64_t)(it.slot - it.part) * a.dp);
                    double zx = 0, zy = 0, zz = 0, zw = 0;
                    if (t < nqf) {
                        for (int q = 0; q < it.nparts; q++) {
                            const float4 p = __ldcg(parts + (int64_t)q * nqf + t);
                            zx += p.x; zy += p.y; zz += p.z; zw += p.w;
                        }
                    }
                    const double tot = block_sum(zx * zx + zy * zy + zz * zz + zw * zw, scratch);
                    const double inv = inv_norm(tot);
                    if (a.lazy_out) {                 // lazy step: unnormalised, the scale aside
                        if (t < nqf && !drop)
                            put_out4(a, it.row, t, make_float4((float)zx, (float)zy, (float)zz, (float)zw));
                        if (t == 0 && !drop) put_scale(a, it.row, (float)inv);
                    } else if (t < nqf) {
                        put_out4(a, it.row, t,
                                 make_float4((float)(zx * inv), (float)(zy * inv), (float)(zz * inv), (float)(zw * inv)));
                    }
                    if (t == 0) a.counters[it.slot - it.part] = 0u;
                }
            }
        }
        __syncthreads();
        fence_proxy_async_smem();
        return;
    }
    if (t < nq) {
        y = smem[t];
#pragma unroll
        for (int w = 1; w < kWarpsPerCta; w++) {
            const float4 q = smem[(size_t)w * ring_f4 + t];
            y.x += q.x; y.y += q.y; y.z += q.z; y.w += q.w;
        }
        ss = sq4(y);
    }
    if (it.nparts == 1) {
        const double tot = block_sum(ss, scratch);
        const double inv = inv_norm(tot);
        if (t < nq) put_out4(a, it.row, t, scale4(y, inv));
    } else {
        float4* part = reinterpret_cast<float4*>(a.partials + (int64_t)it.slot * dp);
        if (t < nq) part[t] = y;
        __threadfence();
        __syncthreads();
        if (t == 0) {
            const unsigned prev = atomicAdd(a.counters + (it.slot - it.part), 1u);
            *flag = (prev == (unsigned)it.nparts - 1) ? 1 : 0;
        }
        __syncthreads();
        if (*flag) {
            __threadfence();
            const float4* parts = reinterpret_cast<const float4*>(a.partials + (int64_t)(it.slot - it.part) * dp);
            double zx = 0, zy = 0, zz = 0, zw = 0;
            if (t < nq) {
                for (int q = 0; q < it.nparts; q++) {     // part order: deterministic
                    const float4 p = __ldcg(parts + (int64_t)q * nq + t);
                    zx += p.x; zy += p.y; zz += p.z; zw += p.w;
                }
            }
            const double tot = block_sum(zx * zx + zy * zy + zz * zz + zw * zw, scratch);
            const double inv = inv_norm(tot);
            if (t < nq)
                put_out4(a, it.row, t,
                         make_float4((float)(zx * inv), (float)(zy * inv), (float)(zz * inv), (float)(zw * inv)));
            if (t == 0) a.counters[it.slot - it.part] = 0u;
        }
    }
    __syncthreads();              // red (ring slot 0) is refilled by TMA next: order the generic
    fence_proxy_async_smem();     // accesses before the async-proxy writes
}

template <int V, bool FULL, int SA, bool HALF>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 2) k_spmm_tma(const SpmmArgs a, int S) {
    extern __shared__ __align__(128) float4 smem[];
    __shared__ double scratch[kWarpsPerCta];
    __shared__ int flag;
    __shared__ unsigned s_item;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int dp = FULL ? 128 * V : a.dp;
    const int slot_f4 = dp / 4;
    const int ring_f4 = S * slot_f4;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kWarpsPerCta * ring_f4);
    Ring r;
    r.buf = smem + (size_t)warp * ring_f4;
    r.bar = bars + warp * S;
    r.S = S;
    r.slot_f4 = slot_f4;
    r.bytes = (uint32_t)dp * 4u;
    r.cs = 0;
    r.ph = 0u;
    r.pol_hot = policy_evict_last();
    r.pol_cold = a.cold_first ? policy_evict_first() : policy_evict_normal();
    r.pol_csr = policy_evict_first();
    if (SA == 0) {
        if (lane == 0)
            for (int i = 0; i < S; i++) mbar_init(r.bar + i, 1);
        mbar_fence_init();
    }
    __syncthreads();

    const int64_t n_items = a.n_items_max > 0 ? a.counts[1] : 0;   // schedule counts live on the device
    if (n_items > 0) {
        for (;;) {
            if (threadIdx.x == 0) s_item = atomicAdd(a.work + 0, 1u);
            __syncthreads();
            const int64_t it = s_item;
            __syncthreads();
            if (it >= n_items) break;
            heavy_item_t<V, FULL, SA, HALF>(a, it, r, smem, ring_f4, scratch, &flag);
        }
    }
    const int64_t nchunks = a.counts[0];
    float4 acc[V];
#pragma unroll
    for (int v = 0; v < V; v++) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    // few chunks: static round robin, no ticket (as k_spmm_norm)
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
        int64_t row = rb;
        while (row < re) {   // segments of consecutive light rows; heavy rows are skipped
            int64_t k0 = __shfl_sync(kFull, rpl, (int)(row - rb));
            int64_t k1 = __shfl_sync(kFull, rpl, (int)(row - rb + 1));
            if (k1 - k0 > a.heavy_thresh) {
                row++;
                continue;
            }
            const int64_t E0 = k0;
            int64_t z = row + 1;
            while (z < re) {
                k0 = k1;
                k1 = __shfl_sync(kFull, rpl, (int)(z - rb + 1));
                if (k1 - k0 > a.heavy_thresh) break;
                z++;
            }
            const int64_t E1 = __shfl_sync(kFull, rpl, (int)(z - rb));
            stream_entries<V, FULL, true, SA, HALF>(a, r, E0, E1, acc, rb, rpl, row, z, lane);
            row = z;
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

struct TmaCfg {
    int blocks_per_sm = 0, sms = 0, S = 0;
    size_t smem = 0;
    int dp = -1;
};

// Launch configuration per device (the smem attribute is per device) and row stride.
template <int V, bool FULL, int SA, bool HALF = false>
Status launch_tma_v(const SpmmArgs& a, cudaStream_t s) {
    static TmaCfg cfg[kMaxDevices];
    static std::mutex mu;
    int dev = 0;
    CL_CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= kMaxDevices) return Status::make(4, "k_spmm_tma: device ordinal beyond kMaxDevices");
    TmaCfg c;
    {
        std::lock_guard<std::mutex> lk(mu);
        TmaCfg& cc = cfg[dev];
        const int width = FULL ? 128 * V : a.dp;      // floats gathered per row (half a row in a half pass)
        if (cc.dp != width) {
            const int slot = width * 4;
            // per-CTA ring budget ~96 KB so that two CTAs (16 warps) share an SM
            int S = SA > 0 ? SA : (96 * 1024) / (kWarpsPerCta * slot);
            if (S > 16 && SA == 0) S = 16;
            if (S < 2) S = 2;
            cc.S = S;
            cc.smem = (size_t)kWarpsPerCta * S * slot + (SA > 0 ? 0 : (size_t)kWarpsPerCta * S * sizeof(uint64_t));
            CL_CUDA_TRY(cudaFuncSetAttribute(k_spmm_tma<V, FULL, SA, HALF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)cc.smem));
            CL_CUDA_TRY(cudaDeviceGetAttribute(&cc.sms, cudaDevAttrMultiProcessorCount, dev));
            CL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cc.blocks_per_sm, k_spmm_tma<V, FULL, SA, HALF>,
                                                                      kWarpsPerCta * 32, cc.smem));
            if (cc.blocks_per_sm < 1) cc.blocks_per_sm = 1;
            cc.dp = width;
        }
        c = cc;
    }
    if (a.r1 <= a.r0 && a.n_items_max == 0) return Status::ok();
    k_spmm_tma<V, FULL, SA, HALF><<<c.sms * c.blocks_per_sm, kWarpsPerCta * 32, c.smem, s>>>(a, c.S);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    return Status::ok();
}

// cp.async ring depth by row width (~96 KB of ring per CTA; <= 32 for the CSR register windows)
template <int V>
constexpr int kAsyncSlots = V == 1 ? 24 : (V == 2 ? 12 : (V == 4 ? 6 : 3));

template <int V, bool FULL, bool HALF = false>
Status launch_mode(const SpmmArgs& a, cudaStream_t s, int mode) {
    if (mode == kGatherAsync) return launch_tma_v<V, FULL, kAsyncSlots<V>, HALF>(a, s);
    return launch_tma_v<V, FULL, 0, HALF>(a, s);
}

// val_out[e] = fp32_rn(val[e] * scale[col[e]]): one rounding of the exact product (a float times a
// float is exact in fp64) -- the weight of an entry whose column row is stored unnormalised
// Four entries per thread with 16-byte loads and stores (the four scale lookups in flight together;
// one entry per thread left the pass latency-bound at ~2.9 TB/s) when col / val / val_out are 16-byte
// aligned (vec); the last nnz % 4 entries -- or all of them otherwise -- go one by one.
__global__ void k_lazy_vals(const float* __restrict__ val, const int32_t* __restrict__ col,
                            const float* __restrict__ scale, int64_t nnz, float* __restrict__ val_out, int vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = vec ? nnz / 4 : 0;
    const int4* c4 = reinterpret_cast<const int4*>(col);
    const float4* v4 = reinterpret_cast<const float4*>(val);
    float4* o4 = reinterpret_cast<float4*>(val_out);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const int4 c = __ldcs(c4 + i);
        const float4 v = __ldcs(v4 + i);
        const float s0 = __ldg(scale + (c.x & 0x7fffffff)), s1 = __ldg(scale + (c.y & 0x7fffffff));
        const float s2 = __ldg(scale + (c.z & 0x7fffffff)), s3 = __ldg(scale + (c.w & 0x7fffffff));
        __stcs(o4 + i, make_float4((float)((double)v.x * (double)s0), (float)((double)v.y * (double)s1),
                                   (float)((double)v.z * (double)s2), (float)((double)v.w * (double)s3)));
    }
    for (int64_t e = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += stride)
        val_out[e] = (float)((double)val[e] * (double)__ldg(scale + (col[e] & 0x7fffffff)));
}

}  // namespace

Status launch_lazy_vals(const float* val, const int32_t* col, const float* scale, int64_t nnz, float* val_out,
                        cudaStream_t s) {
    if (nnz <= 0) return Status::ok();
    int dev = 0, sms = 148;
    CL_CUDA_TRY(cudaGetDevice(&dev));
    CL_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t want = (nnz / 4 + 255) / 256 + 1;
    const int grid = (int)std::min<int64_t>(want, (int64_t)sms * 16);
    const int vec = ((reinterpret_cast<uintptr_t>(val) | reinterpret_cast<uintptr_t>(col) |
                      reinterpret_cast<uintptr_t>(val_out)) & 15) == 0;
    k_lazy_vals<<<grid, 256, 0, s>>>(val, col, scale, nnz, val_out, vec);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    return Status::ok();
}

// Gather engine by row size (measured on B200, ms per SpMM launch):
//  - 4 KB rows (dp = 1024): TMA bulk copies, one per neighbour row issued by one lane (c2 2.54 min,
//    cp.async the same, LDG 3.48 mean);
//  - 0.5-4 KB (128 < dp < 1024): the bulk-copy engine's issue rate binds (~6.7e9 copies/s: c5 made
//    2.84e9 copies in 0.43 s with DRAM 58% busy), per-lane 16-byte cp.async into the same ring
//    does not (c5 332 vs bulk 432 vs LDG 357; c4 at d = 256: 7.27 vs 9.45 vs 8.16; at d = 512:
//    12.8 vs 18.9 vs 16.3);
//  - <= 512 B (dp <= 128): the register kernel at 32 warps per SM (c4 at d = 128: LDG 5.10 vs
//    cp.async 6.55 vs bulk 8.93);
//  - > 4 KB: the register kernel (column slices).
// CLEORA_GATHER=bulk|async|ldg overrides (CLEORA_NO_TMA = ldg, CLEORA_FORCE_TMA = bulk).
int gather_mode(int dp) {
    const char* e = getenv("CLEORA_GATHER");
    if (dp > 1024 || getenv("CLEORA_NO_TMA") || (e && !strcmp(e, "ldg"))) return kGatherLdg;
    if (getenv("CLEORA_FORCE_TMA") || (e && !strcmp(e, "bulk"))) return kGatherBulk;
    if (e && !strcmp(e, "async")) return kGatherAsync;
    if (dp == 1024) return kGatherBulk;
    return dp > 128 ? kGatherAsync : kGatherLdg;
}

bool tma_path_supported(int dp) { return gather_mode(dp) != kGatherLdg; }

Status launch_spmm_tma(const SpmmArgs& a, cudaStream_t s) {
    const int mode = a.gather_mode;
    if (a.pass > 0) {                                 // half-row passes of dp = 1024 rows: 2 KB gathers
        if (a.dp != 1024) return Status::make(4, "half-row passes need dp = 1024");
        return launch_mode<4, true, true>(a, s, mode);
    }
    if (a.dp == 1024) return launch_mode<8, true>(a, s, mode);
    if (a.dp == 512) return launch_mode<4, true>(a, s, mode);
    if (a.dp == 256) return launch_mode<2, true>(a, s, mode);
    if (a.dp == 128) return launch_mode<1, true>(a, s, mode);
    if (a.dp < 128) return launch_mode<1, false>(a, s, mode);
    if (a.dp < 256) return launch_mode<2, false>(a, s, mode);
    if (a.dp < 512) return launch_mode<4, false>(a, s, mode);
    return launch_mode<8, false>(a, s, mode);
}

}  // namespace cleora
