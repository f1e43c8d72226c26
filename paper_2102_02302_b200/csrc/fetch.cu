// fetch.cu -- cleora_fetch_nonzero: the rows of T that a step can make non-zero, packed for the copy.
//
// After one step, a row of M without entries is exactly 0 in T (y = 0 and its normalisation leaves 0,
// reading RZ; Algorithm 1 line 7), so the rows with entries plus their ids are the
// whole result.  On the bench graph (c4) 52.6% of the rows have no entries: the device-to-host copy of
// the result, which bounds the end-to-end step, halves.  The ids are selected once per handle (they
// depend on M only); the rows are packed into a device staging buffer in the handle's stream order and
// copied out as one linear DMA (api.cu fetch_nonzero; 256 MB slices when the whole buffer cannot be had).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"

namespace cleora {

namespace {

constexpr int kThreads = 256;

struct HasEntries {
    const int64_t* row_ptr;
    __device__ bool operator()(int64_t r) const { return row_ptr[r + 1] > row_ptr[r]; }
};

__global__ void k_iota_rows(int64_t r0, int64_t n, int32_t* __restrict__ ids) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) ids[i] = (int32_t)(r0 + i);
}

// one warp per row: row ids[k] of T (stride dp floats) -> out row k (stride d floats)
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_pack_rows(const float* __restrict__ T, int32_t dp, int32_t d,
                                                        const int32_t* __restrict__ ids, int64_t n,
                                                        float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n; k += nwarps) {
        const float* src = T + (int64_t)__ldg(ids + k) * dp;
        float* dst = out + k * (int64_t)d;
        if (VEC) {
            const float4* s4 = reinterpret_cast<const float4*>(src);
            float4* d4 = reinterpret_cast<float4*>(dst);
            for (int c = lane; c < (d >> 2); c += 32) __stcs(d4 + c, __ldcs(s4 + c));
        } else {
            for (int c = lane; c < d; c += 32) dst[c] = src[c];
        }
    }
}

int grid_rows(int64_t n) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + kThreads / 32 - 1) / (kThreads / 32), (int64_t)sms * 8));
}

}  // namespace

// ids[0 .. n) = the rows r in [r0, r1) with row_ptr[r+1] > row_ptr[r], ascending (all = every row).
// `n` is the count the caller knows from the build (the rows of the range minus its rows without
// entries); the selection writes its own count into device scratch that nobody reads.
Status select_rows_with_entries(const int64_t* row_ptr, int64_t r0, int64_t r1, bool all, int32_t* ids,
                                cudaStream_t s) {
    const int64_t n = r1 - r0;
    if (n <= 0) return Status::ok();
    if (all) {
        k_iota_rows<<<grid_rows((n + 31) / 32), kThreads, 0, s>>>(r0, n, ids);
        CL_CUDA_TRY(cudaGetLastError());
        count_launches(1);
        return Status::ok();
    }
    thrust::counting_iterator<int64_t> first(r0);
    HasEntries pred{row_ptr};
    int64_t* d_count = nullptr;
    size_t temp = 0;
    CL_CUDA_TRY(cub::DeviceSelect::If(nullptr, temp, first, ids, d_count, n, pred, s));
    void* buf = nullptr;
    CL_TRY(dalloc(&buf, temp + 256, s, "nonzero-row selection", kAllocTransient));
    d_count = reinterpret_cast<int64_t*>(buf);
    cudaError_t e = cub::DeviceSelect::If(reinterpret_cast<char*>(buf) + 256, temp, first, ids, d_count, n, pred, s);
    dfree(buf, s);
    CL_CUDA_TRY(e);
    count_launches(2);
    return Status::ok();
}

// out row k (d floats, dense) = T row ids[k] (stride dp floats), k in [0, n)
Status pack_rows(const float* T, int32_t dp, int32_t d, const int32_t* ids, int64_t n, float* out, cudaStream_t s) {
    if (n <= 0) return Status::ok();
    const bool vec = (d & 3) == 0 && (dp & 3) == 0 && ((uintptr_t)out & 15) == 0 && ((uintptr_t)T & 15) == 0;
    if (vec)
        k_pack_rows<true><<<grid_rows(n), kThreads, 0, s>>>(T, dp, d, ids, n, out);
    else
        k_pack_rows<false><<<grid_rows(n), kThreads, 0, s>>>(T, dp, d, ids, n, out);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    return Status::ok();
}

}  // namespace cleora
