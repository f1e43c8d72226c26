// l2bw.cu -- the second roofline of the gather path: L2->SM read bandwidth on this B200.
//
// Measures, with CUDA events (best of 10 after 3 warm-ups), the read bandwidth of
//   (1) streaming float4 loads over a buffer of S bytes (S <= 96 MB: L2-resident; 4 GB: HBM),
//   (2) random whole-row gathers (row = R bytes, 16-B vector loads, one warp per row) from a
//       table of S bytes -- the access pattern of the SpMM's neighbour-row gathers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw scripts/l2bw.cu
// Prints one JSON object per line.
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s: %s\"}\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_stream(const float4* __restrict__ p, int64_t n4, int reps, float* out) {
    float acc = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; r++)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            float4 v = __ldcg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 123.456f) *out = acc;
}

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// each warp gathers `per_warp` random rows of row_f4 float4 (16-B loads, 4 rows in flight)
__global__ void k_gather(const float4* __restrict__ p, int64_t rows, int row_f4, int per_warp, float* out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float acc = 0.f;
    for (int i = 0; i < per_warp; i += 4) {
        int64_t r[4];
#pragma unroll
        for (int u = 0; u < 4; u++) r[u] = (int64_t)(mix(w * 1000003ull + i + u) % (uint64_t)rows);
#pragma unroll
        for (int u = 0; u < 4; u++)
            for (int f = lane; f < row_f4; f += 32) {
                float4 v = __ldcg(p + r[u] * row_f4 + f);
                acc += v.x + v.y + v.z + v.w;
            }
    }
    if (acc == 123.456f) *out = acc;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t big = (size_t)4 << 30;
    float4* buf;
    float* out;
    CK(cudaMalloc(&buf, big));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(buf, 0, big));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t sizes[] = {(size_t)16 << 20, (size_t)32 << 20, (size_t)64 << 20, (size_t)96 << 20, big};
    for (size_t S : sizes) {
        const int64_t n4 = S / 16;
        const int reps = S <= ((size_t)96 << 20) ? 20 : 2;
        float best = 1e30f;
        for (int t = 0; t < 13; t++) {
            cudaEventRecord(e0);
            k_stream<<<sms * 4, 512>>>(buf, n4, reps, out);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (t >= 3 && ms < best) best = ms;
        }
        printf("{\"test\": \"stream_read\", \"bytes\": %zu, \"GBps\": %.1f}\n", S, (double)S * reps / (best * 1e-3) / 1e9);
    }
    const int row_bytes[] = {256, 1024, 4096};
    for (size_t S : sizes) {
        for (int rb : row_bytes) {
            const int row_f4 = rb / 16;
            const int64_t rows = S / rb;
            const int per_warp = 64;
            const int blocks = sms * 8;
            float best = 1e30f;
            for (int t = 0; t < 13; t++) {
                cudaEventRecord(e0);
                k_gather<<<blocks, 256>>>(buf, rows, row_f4, per_warp, out);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (t >= 3 && ms < best) best = ms;
            }
            const double bytes = (double)blocks * 8 * per_warp * rb;
            printf("{\"test\": \"gather_rows\", \"table_bytes\": %zu, \"row_bytes\": %d, \"GBps\": %.1f}\n", S, rb,
                   bytes / (best * 1e-3) / 1e9);
        }
    }
    CK(cudaGetLastError());
    return 0;
}
