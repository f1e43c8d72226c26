// Microbenchmark (round 2): sorting a CSR build's entries as (row, col) 64-bit keys with CUB's radix
// sort (the build's choice) vs scattering them into row buckets first and sorting each row's columns
// with cub::DeviceSegmentedSort (a candidate for unit-weight graphs, where equal keys need no stable
// order).  Row lengths follow a power law (P(len >= x) ~ x^-1.1, like c2/c4/c5), columns uniform.
// Usage: segsort_bench n_items n_rows
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); exit(1); } } while (0)

int main(int argc, char** argv) {
    const long n_target = argc > 1 ? atol(argv[1]) : 69000000;
    const long N = argc > 2 ? atol(argv[2]) : 4850000;
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::vector<long> off(N + 1, 0);
    const double mean = (double)n_target / N;
    for (long r = 0; r < N; r++) {              // Pareto(alpha = 1.1) lengths scaled to the mean, capped
        double x = std::pow(1.0 - U(rng), -1.0 / 1.1) - 1.0;
        long len = (long)(x * mean * 0.1 + 0.5);
        if (len > 2000000) len = 2000000;
        off[r + 1] = off[r] + len;
    }
    const long n = off[N];
    if (n >= (1L << 31)) { printf("{\"error\": \"n too large for int offsets\"}\n"); return 0; }
    std::vector<int> hcol(n);
    std::vector<unsigned long long> hkey(n);
    for (long r = 0; r < N; r++)
        for (long k = off[r]; k < off[r + 1]; k++) {
            hcol[k] = (int)(rng() % N);
            hkey[k] = (unsigned long long)r * N + hcol[k];
        }
    // shuffle keys so the radix sort starts from an unsorted list (the build's input order)
    for (long k = n - 1; k > 0; k--) { long j = rng() % (k + 1); std::swap(hkey[k], hkey[j]); }
    int *c0, *c1; int* doff; unsigned long long *k0, *k1;
    CK(cudaMalloc(&c0, n * 4)); CK(cudaMalloc(&c1, n * 4)); CK(cudaMalloc(&doff, (N + 1) * 4));
    CK(cudaMalloc(&k0, n * 8)); CK(cudaMalloc(&k1, n * 8));
    std::vector<int> hoff(N + 1);
    for (long r = 0; r <= N; r++) hoff[r] = (int)off[r];
    CK(cudaMemcpy(doff, hoff.data(), (N + 1) * 4, cudaMemcpyHostToDevice));
    const int end_bit = 64 - __builtin_clzll((unsigned long long)N * N | 1);
    size_t t1 = 0, t2 = 0;
    cub::DoubleBuffer<unsigned long long> kb(k0, k1);
    CK(cub::DeviceRadixSort::SortKeys(nullptr, t1, kb, (int)n, 0, end_bit));
    CK(cub::DeviceSegmentedSort::SortKeys(nullptr, t2, c0, c1, (int)n, (int)N, doff, doff + 1));
    void* tmp; CK(cudaMalloc(&tmp, t1 > t2 ? t1 : t2));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best1 = 1e30f, best2 = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        CK(cudaMemcpy(k0, hkey.data(), n * 8, cudaMemcpyHostToDevice));
        kb = cub::DoubleBuffer<unsigned long long>(k0, k1);
        cudaEventRecord(a);
        CK(cub::DeviceRadixSort::SortKeys(tmp, t1, kb, (int)n, 0, end_bit));
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); if (rep) best1 = ms < best1 ? ms : best1;
        CK(cudaMemcpy(c0, hcol.data(), n * 4, cudaMemcpyHostToDevice));
        cudaEventRecord(a);
        CK(cub::DeviceSegmentedSort::SortKeys(tmp, t2, c0, c1, (int)n, (int)N, doff, doff + 1));
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b); if (rep) best2 = ms < best2 ? ms : best2;
    }
    printf("{\"items\": %ld, \"rows\": %ld, \"key_bits\": %d, \"radix64_ms\": %.3f, \"segmented32_ms\": %.3f}\n", n, N, end_bit,
           best1, best2);
    return 0;
}
