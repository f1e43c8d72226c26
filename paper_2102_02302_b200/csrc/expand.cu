// expand.cu -- hypergraph expansion on the device (§3.2 "Hypergraph Expansion";
// SURVEY §8(f) f3): the step before the hot path in the paper's own pipeline, whose timed
// workloads were adjacency rows treated as hyperedges, clique-expanded (Facebook, RoadNet) or
// star-expanded (YouTube, LiveJournal).
//
// Clique (reading R16): hyperedge e with members m_0..m_{k-1} (listed order) emits the undirected
// edges (m_i, m_j) for every i < j with m_i != m_j (equal members make no self-loop), in the order
// (e, i, j), each with the hyperedge's weight.  Star (reading R17): hyperedge e gets the virtual
// node n_nodes + e and emits (n_nodes + e, m_i) for every listed member, in the order (e, i).
//
// Both are integer work: one warp per hyperedge; a clique counts and then writes its pairs with
// warp ballots over j for every i (O(k^2 / 32) per hyperedge), output offsets from a CUB scan.
#include <cub/cub.cuh>

#include "common.cuh"

namespace cleora {

namespace {

constexpr int kThreads = 256;

// bad[0]: first member id out of range; bad[1]: first bad weight; bad[2]: first hyperedge e whose
// offsets are not ptr[0] = 0, ptr[e] <= ptr[e+1] (a malformed ptr would make the expansion kernels
// write outside the output, so it is rejected before they run, as on the host path)
__global__ void k_expand_check(const int64_t* __restrict__ ptr, const int32_t* __restrict__ nodes, int64_t n,
                               int32_t n_nodes, const float* __restrict__ w, int64_t n_he,
                               unsigned long long* __restrict__ bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        if (nodes[i] < 0 || nodes[i] >= n_nodes) atomicMin(bad, (unsigned long long)i);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_he; e += stride) {
        if (w && !(isfinite(w[e]) && w[e] > 0.0f)) atomicMin(bad + 1, (unsigned long long)e);
        if ((e == 0 && ptr[0] != 0) || ptr[e + 1] < ptr[e]) atomicMin(bad + 2, (unsigned long long)e);
    }
}

// count (out == nullptr) or write the clique pairs of each hyperedge
__global__ void k_clique(const int64_t* __restrict__ ptr, const int32_t* __restrict__ nodes, int64_t n_he,
                         const float* __restrict__ hw, const int64_t* __restrict__ offset, int64_t* __restrict__ count,
                         int32_t* __restrict__ os, int32_t* __restrict__ od, float* __restrict__ ow) {
    const int lane = threadIdx.x & 31;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n_he; e += wstride) {
        const int64_t b = ptr[e], k = ptr[e + 1] - b;
        int64_t pos = offset ? offset[e] : 0;
        const float wt = hw ? hw[e] : 1.0f;
        for (int64_t i = 0; i < k; i++) {
            const int32_t mi = nodes[b + i];
            for (int64_t j0 = i + 1; j0 < k; j0 += 32) {
                const int64_t j = j0 + lane;
                const int32_t mj = j < k ? nodes[b + j] : mi;
                const bool emit = j < k && mj != mi;
                const unsigned m = __ballot_sync(0xffffffffu, emit);
                if (offset && emit) {
                    const int64_t at = pos + __popc(m & ((1u << lane) - 1u));
                    os[at] = mi;
                    od[at] = mj;
                    if (ow) ow[at] = wt;
                }
                pos += __popc(m);
            }
        }
        if (!offset && lane == 0) count[e] = pos;
    }
}

__global__ void k_star(const int64_t* __restrict__ ptr, const int32_t* __restrict__ nodes, int64_t n_he,
                       int32_t n_nodes, const float* __restrict__ hw, int32_t* __restrict__ os, int32_t* __restrict__ od,
                       float* __restrict__ ow) {
    const int lane = threadIdx.x & 31;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n_he; e += wstride) {
        const int64_t b = ptr[e], k = ptr[e + 1] - b;
        const float wt = hw ? hw[e] : 1.0f;
        for (int64_t i = lane; i < k; i += 32) {
            os[b + i] = (int32_t)(n_nodes + e);
            od[b + i] = nodes[b + i];
            if (ow) ow[b + i] = wt;
        }
    }
}

int warp_grid(int64_t items) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t b = (items * 32 + kThreads - 1) / kThreads;
    if (b > (int64_t)sms * 32) b = (int64_t)sms * 32;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

Status expand_hypergraph(const int64_t* d_ptr, const int32_t* d_nodes, const float* d_w, int64_t n_he, int64_t n_members,
                         int32_t n_nodes, int mode, cudaStream_t s, int32_t* d_os, int32_t* d_od, float* d_ow,
                         int64_t capacity, int64_t* n_out) {
    // validation
    {
        unsigned long long* bad = nullptr;
        CL_TRY(dalloc((void**)&bad, 3 * sizeof(unsigned long long), s, "expand check"));
        cudaMemsetAsync(bad, 0xFF, 3 * sizeof(unsigned long long), s);
        const int64_t n = n_members > n_he ? n_members : n_he;
        k_expand_check<<<warp_grid((n + 31) / 32), kThreads, 0, s>>>(d_ptr, d_nodes, n_members, n_nodes, d_w, n_he, bad);
        count_launches(1);
        unsigned long long h[3];
        Status rs = read_small(h, bad, sizeof h, s);
        dfree(bad, s);
        CL_TRY(rs);
        char buf[160];
        if (h[2] != ~0ull) {
            snprintf(buf, sizeof buf, "cleora_expand: he_ptr must start at 0 and be non-decreasing (hyperedge %llu)", h[2]);
            return Status::make(2, buf);
        }
        if (h[0] != ~0ull) {
            snprintf(buf, sizeof buf, "cleora_expand: member %llu: node id outside [0, n_nodes)", h[0]);
            return Status::make(3, buf);
        }
        if (h[1] != ~0ull) {
            snprintf(buf, sizeof buf, "cleora_expand: hyperedge %llu: weight not finite or <= 0", h[1]);
            return Status::make(3, buf);
        }
    }
    if (mode == 1) {                                       // star: k edges per hyperedge, offsets = ptr
        *n_out = n_members;
        if (!d_os) return Status::ok();
        if (capacity < n_members) return Status::make(2, "cleora_expand: capacity smaller than the edge count");
        k_star<<<warp_grid(n_he), kThreads, 0, s>>>(d_ptr, d_nodes, n_he, n_nodes, d_w, d_os, d_od, d_ow);
        CL_CUDA_TRY(cudaGetLastError());
        count_launches(1);
        CL_CUDA_TRY(cudaStreamSynchronize(s));
        return Status::ok();
    }
    // clique: count, exclusive scan, write
    int64_t *cnt = nullptr, *off = nullptr, *tot = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    Status st = dalloc((void**)&cnt, (n_he + 1) * sizeof(int64_t), s, "clique counts", kAllocTransient);
    if (st.good()) st = dalloc((void**)&off, (n_he + 1) * sizeof(int64_t), s, "clique offsets", kAllocTransient);
    if (st.good()) st = dalloc((void**)&tot, 2 * sizeof(int64_t), s, "clique total");
    int64_t total = 0;
    if (st.good()) {
        k_clique<<<warp_grid(n_he), kThreads, 0, s>>>(d_ptr, d_nodes, n_he, d_w, nullptr, cnt, nullptr, nullptr, nullptr);
        count_launches(1);
        cudaMemsetAsync(cnt + n_he, 0, sizeof(int64_t), s);
        cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, n_he + 1, s);
        st = dalloc(&tmp, tmp_bytes, s, "clique scan temp", kAllocTransient);
    }
    if (st.good()) {
        cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, n_he + 1, s);
        count_launches(2);
        st = read_small(&total, off + n_he, sizeof total, s);
    }
    if (st.good()) {
        *n_out = total;
        if (d_os) {
            if (capacity < total) {
                st = Status::make(2, "cleora_expand: capacity smaller than the edge count");
            } else {
                k_clique<<<warp_grid(n_he), kThreads, 0, s>>>(d_ptr, d_nodes, n_he, d_w, off, nullptr, d_os, d_od, d_ow);
                count_launches(1);
                cudaError_t e = cudaGetLastError();
                if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                if (e != cudaSuccess) st = Status::make(4, std::string("cleora_expand: ") + cudaGetErrorString(e));
            }
        }
    }
    cudaStreamSynchronize(s);
    dfree(tmp, s);
    dfree(tot, s);
    dfree(off, s);
    dfree(cnt, s);
    return st;
}

}  // namespace cleora
