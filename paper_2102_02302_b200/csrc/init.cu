// init.cu -- T_0 from a hash of (node id, dimension): "T_0 ~ U(-1,1)" (
// Algorithm 1 line 4), realised as reading R1:
//   h   = mix(mix(seed + 0x9E3779B97F4A7C15) ^ (v << 32 | j)),   mix = SplitMix64 finaliser
//   T_0 = ((int32)(h >> 40) - 2^23) * 2^-23  in [-1, 1 - 2^-23]   (exact in fp32)
// Padding columns j in [d, dp) are written as 0.  One thread per float4, 16-byte stores.
#include "common.cuh"

namespace cleora {

namespace {

constexpr uint64_t kC1 = 0xBF58476D1CE4E5B9ull, kC2 = 0x94D049BB133111EBull;

// The same value as ((int32)(sm64(base ^ j) >> 40) - 2^23) * 2^-23 for 0 <= j < 2^30, with the per-row work hoisted
// (the kernel is integer-ALU bound, not HBM bound, when written naively):
//   z1 = base ^ j ^ (base >> 30)            (j < 2^30 contributes nothing to z1 >> 30)
//   z2 = z1 * C1  = lo*C1lo + ((lo*C1hi + hi*C1lo) << 32), hi*C1lo a per-row constant
//   z3 = z2 ^ (z2 >> 27)
//   h >> 40 = (z3 * C2) >> 40               (the final xor-shift by 31 does not reach bit 40)
// so only the high word of z3*C2 is formed.  Bit-exact with the oracle (tested).
struct RowHash {
    uint32_t b1_lo, b1_hi, k1;   // b1 = base ^ (base >> 30); k1 = lo32(b1_hi * C1lo)
};

__device__ __forceinline__ RowHash row_hash(uint64_t base) {
    const uint64_t b1 = base ^ (base >> 30);
    RowHash r;
    r.b1_lo = (uint32_t)b1;
    r.b1_hi = (uint32_t)(b1 >> 32);
    r.k1 = r.b1_hi * (uint32_t)kC1;
    return r;
}

__device__ __forceinline__ float hash_elem(const RowHash& r, uint32_t j) {
    const uint32_t lo = r.b1_lo ^ j;
    const uint64_t t = (uint64_t)lo * (uint32_t)kC1;                       // lo * C1lo
    const uint32_t z2_lo = (uint32_t)t;
    const uint32_t z2_hi = (uint32_t)(t >> 32) + lo * (uint32_t)(kC1 >> 32) + r.k1;
    const uint32_t z3_lo = z2_lo ^ __funnelshift_r(z2_lo, z2_hi, 27);      // low word of z2 >> 27
    const uint32_t z3_hi = z2_hi ^ (z2_hi >> 27);
    const uint32_t z4_hi = __umulhi(z3_lo, (uint32_t)kC2) + z3_lo * (uint32_t)(kC2 >> 32) +
                           z3_hi * (uint32_t)kC2;
    return (float)((int32_t)(z4_hi >> 8) - 8388608) * (1.0f / 8388608.0f);
}

// One warp per row (grid-stride over rows): lane l writes float4 columns l, l+32, ... -- no
// 64-bit division per element, 512 contiguous bytes per warp store instruction.
// lid (batched handles, NULL otherwise): every row's id local to its graph; the hash keys on it, so
// each graph of a batch gets its own T_0.
// sel (NULL: every row): the in-degree; sel_mode 1 writes the rows with in-degree > 0, 2 the others
__global__ void k_hash_init(float4* __restrict__ T, int64_t N, int32_t d, int32_t dp, uint64_t s,
                            const int32_t* __restrict__ lid, const int32_t* __restrict__ sel, int sel_mode) {
    const int lane = threadIdx.x & 31;
    const int q = dp / 4;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < N; v += wstride) {
        if (sel && ((sel[v] != 0) != (sel_mode == 1))) continue;     // warp-uniform
        const int64_t id = lid ? (int64_t)lid[v] : v;
        const RowHash rh = row_hash(s ^ ((uint64_t)id << 32));
        float4* row = T + v * q;
#pragma unroll 2
        for (int f = lane; f < q; f += 32) {
            const uint32_t j0 = 4u * f;                  // < d: dp is d rounded up to 4
            float4 o = make_float4(hash_elem(rh, j0), hash_elem(rh, j0 + 1), hash_elem(rh, j0 + 2),
                                   hash_elem(rh, j0 + 3));
            if (j0 + 4 > (uint32_t)d) {                  // the padded tail of a row (d % 4 != 0)
                o.y = j0 + 1 < (uint32_t)d ? o.y : 0.0f;
                o.z = j0 + 2 < (uint32_t)d ? o.z : 0.0f;
                o.w = 0.0f;
            }
            __stcs(row + f, o);
        }
    }
}

// Local row ids of a batch: one warp per graph writes base[g+1] - base[g] consecutive ids (a binary
// search over the graph bases per row in k_hash_init made it latency-bound: f4, 2,000 graphs, 0.64 ms
// for 1.1 GB of T_0)
__global__ void k_local_ids(const int64_t* __restrict__ base, int32_t n_graphs, int32_t* __restrict__ lid) {
    const int lane = threadIdx.x & 31;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < n_graphs; g += wstride) {
        const int64_t b = base[g], e = base[g + 1];
        for (int64_t r = b + lane; r < e; r += 32) lid[r] = (int32_t)(r - b);
    }
}

}  // namespace

Status launch_hash_init(float* T, int64_t N, int32_t d, int32_t dp, uint64_t seed, cudaStream_t s,
                        const int64_t* d_base, int32_t n_graphs, const int32_t* sel, int sel_mode) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t key = sm64(seed + 0x9E3779B97F4A7C15ull);
    int64_t blocks = (N * 32 + 255) / 256;              // one warp per row ...
    const int64_t cap = (int64_t)sms * 8 * 4;            // ... grid-stride, a multiple of the SM count
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    int32_t* lid = nullptr;
    if (d_base) {
        CL_TRY(dalloc((void**)&lid, (size_t)N * sizeof(int32_t), s, "batch local ids", kAllocTransient));
        int64_t gb = ((int64_t)n_graphs * 32 + 255) / 256;
        if (gb > (int64_t)sms * 8) gb = (int64_t)sms * 8;
        k_local_ids<<<(unsigned)(gb < 1 ? 1 : gb), 256, 0, s>>>(d_base, n_graphs, lid);
        count_launches(1);
    }
    k_hash_init<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<float4*>(T), N, d, dp, key, lid, sel, sel_mode);
    const cudaError_t e = cudaGetLastError();
    count_launches(1);
    if (lid) dfree(lid, s);
    CL_CUDA_TRY(e);
    return Status::ok();
}

}  // namespace cleora
