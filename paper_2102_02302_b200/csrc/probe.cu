// probe.cu -- the second roofline of the gather path, measured live: the rate at which SMs can
// gather random rows of a given size from an L2-resident table (cleora_probe_gather).
//
// The SpMM's operand stream is nnz * d * 4 bytes of neighbour-row gathers (SURVEY.md §8(d),
// "Which roofline"), avg-degree times the size of T; every gathered byte passes the L2 -> SM path,
// whether it hits in L2 or is filled from HBM.  bench.py divides that stream by this rate
// ("roofline.gather_bound").  Diagnostic only: no part of the Cleora path calls it.
//
// Rows of R bytes are loaded with 16-byte ld.global.cg (L2 only), lanes split across rows when
// R < 512 B so every lane issues a load, U = 8 independent rows in flight per lane group; row
// indices come from a precomputed random table read coalesced (no per-load hashing on the issue
// path -- the round-1 microbenchmark, scripts/l2bw.cu, was ALU-bound on its per-lane hash at
// 256 B rows).
#include <algorithm>

#include "common.cuh"

namespace cleora {

namespace {

__global__ void k_probe_index(int32_t* __restrict__ idx, int64_t n, int64_t rows, uint64_t key) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        idx[i] = (int32_t)(sm64(key ^ (uint64_t)i) % (uint64_t)rows);
}

__global__ void k_probe_fill(float4* __restrict__ t, int64_t n4) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
        t[i] = make_float4(1.f, 2.f, 3.f, (float)(i & 1023));
}

// lanes per row L = min(32, row_f4); a warp step covers 32 / L rows x U in flight
template <int U>
__global__ void __launch_bounds__(256) k_probe_gather(const float4* __restrict__ table, const int32_t* __restrict__ idx,
                                                      int64_t n_idx, int row_f4, unsigned* __restrict__ sink) {
    const int lane = threadIdx.x & 31;
    const int L = row_f4 < 32 ? row_f4 : 32;
    const int per = 32 / L;                        // rows per warp per slot
    const int grp = lane / L, sub = lane % L;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t step = (int64_t)per * U;
    unsigned acc = 0;
    for (int64_t base = warp * step; base < n_idx; base += nwarps * step) {
        int32_t r[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = base + (int64_t)u * per + grp;
            r[u] = i < n_idx ? __ldg(idx + i) : -1;
        }
        for (int f = sub; f < row_f4; f += L) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; u++)
                v[u] = r[u] >= 0 ? __ldcg(table + (int64_t)r[u] * row_f4 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < U; u++)
                acc ^= __float_as_uint(v[u].x) ^ __float_as_uint(v[u].y) ^ __float_as_uint(v[u].z) ^
                       __float_as_uint(v[u].w);
        }
    }
    if (acc == 0x9e3779b9u) *sink = acc;           // never true in practice; keeps the loads live
}

}  // namespace

Status probe_gather(int row_bytes, int64_t table_bytes, int64_t n_gathers, cudaStream_t s, double* gbs) {
    if (row_bytes < 16 || row_bytes % 16) return Status::make(2, "cleora_probe_gather: row_bytes must be a multiple of 16");
    const int row_f4 = row_bytes / 16;
    if (row_f4 < 32 && (32 % row_f4)) return Status::make(2, "cleora_probe_gather: rows below 512 B must divide 512 B");
    const int64_t rows = std::max<int64_t>(1, table_bytes / row_bytes);
    int dev = 0, sms = 148;
    CL_CUDA_TRY(cudaGetDevice(&dev));
    CL_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    float4* table = nullptr;
    int32_t* idx = nullptr;
    unsigned* sink = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    Status st = dalloc((void**)&table, (size_t)rows * row_bytes, s, "probe table", kAllocTransient);
    if (st.good()) st = dalloc((void**)&idx, (size_t)n_gathers * 4, s, "probe indices", kAllocTransient);
    if (st.good()) st = dalloc((void**)&sink, 16, s, "probe sink");
    double best = 0.0;
    if (st.good()) {
        k_probe_fill<<<sms * 4, 256, 0, s>>>(table, rows * row_f4);
        k_probe_index<<<sms * 4, 256, 0, s>>>(idx, n_gathers, rows, 0x5eedull);
        count_launches(2);
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int t = 0; t < 8 && st.good(); t++) {
            cudaEventRecord(e0, s);
            k_probe_gather<8><<<sms * 8, 256, 0, s>>>(table, idx, n_gathers, row_f4, sink);
            cudaEventRecord(e1, s);
            count_launches(1);
            cudaError_t e = cudaEventSynchronize(e1);
            if (e != cudaSuccess) { st = Status::make(4, std::string("probe: ") + cudaGetErrorString(e)); break; }
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            const double r = (double)n_gathers * row_bytes / (ms * 1e-3) / 1e9;
            if (t >= 2) best = std::max(best, r);      // 2 warm-up launches
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    cudaStreamSynchronize(s);
    dfree(table, s);
    dfree(idx, s);
    dfree(sink, s);
    CL_TRY(st);
    *gbs = best;
    return Status::ok();
}

}  // namespace cleora
