// init.cu -- T_0 from a hash of (node id, dimension): "T_0 ~ U(-1,1)" (
// Algorithm 1 line 4), realised as reading R1:
//   h   = mix(mix(seed + 0x9E3779B97F4A7C15) ^ (v << 32 | j)),   mix = SplitMix64 finaliser
//   T_0 = ((int32)(h >> 40) - 2^23) * 2^-23  in [-1, 1 - 2^-23]   (exact in fp32)
// Padding columns j in [d, dp) are written as 0.  One thread per float4, 16-byte stores.
#include "common.cuh"

namespace cleora {

namespace {

__host__ __device__ __forceinline__ uint64_t sm64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float h2f(uint64_t h) {
    // (h >> 40) has 24 bits; subtracting 2^23 and scaling by 2^-23 is exact in fp32
    return (float)((int32_t)(h >> 40) - 8388608) * (1.0f / 8388608.0f);
}

// One warp per row (grid-stride over rows): lane l writes float4 columns l, l+32, ... -- no
// 64-bit division per element, 512 contiguous bytes per warp store instruction.
__global__ void k_hash_init(float4* __restrict__ T, int64_t N, int32_t d, int32_t dp, uint64_t s) {
    const int lane = threadIdx.x & 31;
    const int q = dp / 4;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < N; v += wstride) {
        const uint64_t base = s ^ ((uint64_t)v << 32);
        float4* row = T + v * q;
        for (int f = lane; f < q; f += 32) {
            const int j0 = 4 * f;
            float4 o;
            o.x = (j0 + 0 < d) ? h2f(sm64(base ^ (uint64_t)(j0 + 0))) : 0.0f;
            o.y = (j0 + 1 < d) ? h2f(sm64(base ^ (uint64_t)(j0 + 1))) : 0.0f;
            o.z = (j0 + 2 < d) ? h2f(sm64(base ^ (uint64_t)(j0 + 2))) : 0.0f;
            o.w = (j0 + 3 < d) ? h2f(sm64(base ^ (uint64_t)(j0 + 3))) : 0.0f;
            row[f] = o;
        }
    }
}

}  // namespace

Status launch_hash_init(float* T, int64_t N, int32_t d, int32_t dp, uint64_t seed, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t key = sm64(seed + 0x9E3779B97F4A7C15ull);
    int64_t blocks = (N * 32 + 255) / 256;              // one warp per row ...
    const int64_t cap = (int64_t)sms * 8 * 4;            // ... grid-stride, a multiple of the SM count
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k_hash_init<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<float4*>(T), N, d, dp, key);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    return Status::ok();
}

}  // namespace cleora
