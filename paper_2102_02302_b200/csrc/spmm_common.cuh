// spmm_common.cuh -- device helpers shared by the SpMM + normalise kernels (product code).
#pragma once

#include "common.cuh"

namespace cleora {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float4 ldg4(const float4* p) { return __ldg(p); }

__device__ __forceinline__ void fma4(float4& acc, float w, const float4& x) {
    acc.x = fmaf(w, x.x, acc.x);
    acc.y = fmaf(w, x.y, acc.y);
    acc.z = fmaf(w, x.z, acc.z);
    acc.w = fmaf(w, x.w, acc.w);
}

__device__ __forceinline__ double sq4(const float4& y) {
    return (double)y.x * y.x + (double)y.y * y.y + (double)y.z * y.z + (double)y.w * y.w;
}

// 1 / ||y|| from the fp64 sum of squares (0 for the zero vector: reading RZ).  rsqrt in fp64
// (within an ulp or two of 2^-53 relative, far below the fp32 output's 2^-24) instead of a
// correctly rounded 1.0 / sqrt(): the IEEE division and square root were 6.6% of the register
// kernel's instructions on short rows (ncu, f4 batch)
__device__ __forceinline__ double inv_norm(double ss) { return ss > 0.0 ? rsqrt(ss) : 0.0; }

__device__ __forceinline__ float4 scale4(const float4& y, double inv) {
    return make_float4((float)((double)y.x * inv), (float)((double)y.y * inv), (float)((double)y.z * inv),
                       (float)((double)y.w * inv));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarpsPerCta; w++) s += scratch[w];   // fixed order: deterministic
    return s;
}

}  // namespace
}  // namespace cleora
