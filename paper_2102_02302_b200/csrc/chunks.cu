// chunks.cu -- Algorithm 1 with Q > 1 chunks: the merge
//     T_v = sum_q w_qv T^q_v,   w_qv = occ_q(v) / sum_k occ_k(v)
// with occ_q(v) = v's endpoint occurrences among chunk q's edges (reading R14, counted by the
// chunk's build).  A node in no chunk gets the zero row; nothing is renormalised (Algorithm 1
// has no normalisation after the merge).  The arithmetic is pinned to the oracle's, bit for bit:
// one IEEE fp64 division per weight, fp64 multiply-then-add (explicit _rn intrinsics, so no FMA
// contraction) in ascending q, one rounding to fp32.
//
// HBM-bound: reads Q x N x dp x 4 bytes of chunk embeddings, writes N x dp x 4.  One warp per
// row, lane = float4 column, 16-byte loads and streaming stores.
#include "common.cuh"

namespace cleora {

namespace {

__global__ void k_merge(const float* const* __restrict__ Tq, const int32_t* const* __restrict__ occ, int Q, int64_t N,
                        int dp, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int nq = dp / 4;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < N; v += wstride) {
        int64_t tot = 0;
        for (int q = 0; q < Q; q++) tot += occ[q][v];
        float4* o = reinterpret_cast<float4*>(out + v * (int64_t)dp);
        for (int f = lane; f < nq; f += 32) {
            double ax = 0.0, ay = 0.0, az = 0.0, aw = 0.0;
            if (tot > 0) {
                for (int q = 0; q < Q; q++) {
                    const double w = __ddiv_rn((double)occ[q][v], (double)tot);
                    const float4 x = __ldcs(reinterpret_cast<const float4*>(Tq[q] + v * (int64_t)dp) + f);
                    ax = __dadd_rn(ax, __dmul_rn(w, (double)x.x));
                    ay = __dadd_rn(ay, __dmul_rn(w, (double)x.y));
                    az = __dadd_rn(az, __dmul_rn(w, (double)x.z));
                    aw = __dadd_rn(aw, __dmul_rn(w, (double)x.w));
                }
            }
            __stcs(o + f, make_float4(__double2float_rn(ax), __double2float_rn(ay), __double2float_rn(az),
                                      __double2float_rn(aw)));
        }
    }
}

}  // namespace

Status launch_merge(const float* const* d_Tq, const int32_t* const* d_occ, int Q, int64_t N, int dp, float* d_out,
                    cudaStream_t s) {
    int dev = 0, sms = 148;
    CL_CUDA_TRY(cudaGetDevice(&dev));
    CL_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int64_t blocks = (N * 32 + 255) / 256;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    if (blocks < 1) blocks = 1;
    k_merge<<<(unsigned)blocks, 256, 0, s>>>(d_Tq, d_occ, Q, N, dp, d_out);
    CL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    return Status::ok();
}

}  // namespace cleora
