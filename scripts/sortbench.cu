// Microbenchmark: ways to sort (src, dst) entry keys for the CSR build.  (a) CUB SortKeys on 64-bit
// keys src*N+dst over ceil(log2 N^2) bits (the build's current choice); (b) two stable 32-bit
// SortPairs passes (by dst carrying src, then by src carrying dst); (c) CUB SortKeys on 64-bit keys
// with a 32-bit-per-half decomposition is not available, so (c) = (a) with all 64 bits for scale.
// Usage: sortbench [n_entries] [N]
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1); } } while (0)

int main(int argc, char** argv) {
    const long n = argc > 1 ? atol(argv[1]) : 17215056;
    const long N = argc > 2 ? atol(argv[2]) : 2151882;
    std::mt19937_64 rng(1);
    std::vector<unsigned long long> hk(n);
    std::vector<unsigned> hs(n), hd(n);
    for (long i = 0; i < n; i++) { hs[i] = rng() % N; hd[i] = rng() % N; hk[i] = (unsigned long long)hs[i] * N + hd[i]; }
    unsigned long long *k0, *k1; unsigned *s0, *s1, *d0, *d1;
    CK(cudaMalloc(&k0, n * 8)); CK(cudaMalloc(&k1, n * 8));
    CK(cudaMalloc(&s0, n * 4)); CK(cudaMalloc(&s1, n * 4)); CK(cudaMalloc(&d0, n * 4)); CK(cudaMalloc(&d1, n * 4));
    int end_bit = 64 - __builtin_clzll((unsigned long long)N * N | 1);
    int nbits = 32 - __builtin_clz((unsigned)N | 1);
    size_t t1 = 0, t2 = 0;
    cub::DoubleBuffer<unsigned long long> kb(k0, k1);
    cub::DeviceRadixSort::SortKeys(nullptr, t1, kb, (int)n, 0, end_bit);
    cub::DoubleBuffer<unsigned> ks(d0, d1), vs(s0, s1);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, ks, vs, (int)n, 0, nbits);
    void* tmp; CK(cudaMalloc(&tmp, t1 > t2 ? t1 : t2));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; rep++) {
        CK(cudaMemcpy(k0, hk.data(), n * 8, cudaMemcpyHostToDevice));
        kb = cub::DoubleBuffer<unsigned long long>(k0, k1);
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortKeys(tmp, t1, kb, (int)n, 0, end_bit);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms1; cudaEventElapsedTime(&ms1, a, b);
        CK(cudaMemcpy(d0, hd.data(), n * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(s0, hs.data(), n * 4, cudaMemcpyHostToDevice));
        ks = cub::DoubleBuffer<unsigned>(d0, d1); vs = cub::DoubleBuffer<unsigned>(s0, s1);
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(tmp, t2, ks, vs, (int)n, 0, nbits);   // by dst
        cub::DoubleBuffer<unsigned> ks2(vs.Current(), vs.Alternate()), vs2(ks.Current(), ks.Alternate());
        cub::DeviceRadixSort::SortPairs(tmp, t2, ks2, vs2, (int)n, 0, nbits); // stable by src
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms2; cudaEventElapsedTime(&ms2, a, b);
        printf("{\"n\": %ld, \"N\": %ld, \"keys64_bits\": %d, \"keys64_ms\": %.4f, \"pairs32x2_bits\": %d, \"pairs32x2_ms\": %.4f}\n",
               n, N, end_bit, ms1, nbits, ms2);
    }
    return 0;
}
