/*
 * cleora_gen.c -- seeded synthetic graph generators (TEST / BENCH INFRASTRUCTURE).
 *
 * This module produces the input COO edge lists that BOTH the oracle (oracle/) and
 * the CUDA path (paper_2102_02302_b200/) consume.  It holds none of the method's
 * arithmetic: no transition matrix, no degree, no embedding, no normalisation.
 * It only draws graphs.  The five configurations stand in for the paper's Table 1
 * datasets (Table 1), which are not available in this container;
 * the recipes are SURVEY.md §8(d) ("Synthetic inputs") and DESIGN.md §"Input recipe".
 *
 * RNG: counter-based, so every draw is a pure function of
 * (seed, stream, counter) and generation is parallel and deterministic:
 *     u64  = mix64( mix64(seed + GOLDEN*stream) XOR counter )
 *     unif = (u64 >> 11) * 2^-53                       in [0, 1)
 * mix64 is the SplitMix64 finaliser (Steele, Lea, Flood 2014).  Streams:
 *     1 endpoints / R-MAT quadrants, 2 weights, 3 id permutation,
 *     4 lattice deletions, 5 lattice diagonals.
 *
 * Output convention: caller allocates src/dst(/w) with the capacity returned by the
 * matching *_capacity function (an upper bound); the generator returns the number
 * of edges written, or -1 on allocation failure.  Undirected configs list each
 * edge once (the library / oracle mirror it).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t g_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t g_key(uint64_t seed, uint64_t stream) { return g_mix64(seed + GOLDEN * stream); }
static inline uint64_t g_u64(uint64_t key, uint64_t counter) { return g_mix64(key ^ counter); }
static inline double g_unif(uint64_t key, uint64_t counter) {
    return (double)(g_u64(key, counter) >> 11) * 0x1.0p-53;
}

uint64_t gen_u64(uint64_t seed, uint64_t stream, uint64_t counter) { return g_u64(g_key(seed, stream), counter); }
double gen_unif(uint64_t seed, uint64_t stream, uint64_t counter) { return g_unif(g_key(seed, stream), counter); }

/* ---------------------------------------------------------------- helpers */

/* LSD radix sort of uint64 keys, 16-bit digits; skips digits that are constant. */
static int radix_sort_u64(uint64_t* a, int64_t n) {
    if (n < 2) return 0;
    uint64_t* tmp = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
    if (!tmp) return -1;
    int64_t* cnt = (int64_t*)malloc(65536 * sizeof(int64_t));
    if (!cnt) { free(tmp); return -1; }
    uint64_t* src = a; uint64_t* dst = tmp;
    for (int shift = 0; shift < 64; shift += 16) {
        memset(cnt, 0, 65536 * sizeof(int64_t));
        for (int64_t i = 0; i < n; i++) cnt[(src[i] >> shift) & 0xFFFF]++;
        int single = 0;
        for (int b = 0; b < 65536; b++) if (cnt[b] == n) { single = 1; break; }
        if (single) continue;
        int64_t s = 0;
        for (int b = 0; b < 65536; b++) { int64_t c = cnt[b]; cnt[b] = s; s += c; }
        for (int64_t i = 0; i < n; i++) dst[cnt[(src[i] >> shift) & 0xFFFF]++] = src[i];
        uint64_t* t = src; src = dst; dst = t;
    }
    if (src != a) memcpy(a, src, (size_t)n * sizeof(uint64_t));
    free(tmp); free(cnt);
    return 0;
}

/* Seeded Fisher-Yates permutation of [0,n): stream 3, sequential draw index. */
static int32_t* fisher_yates(int32_t n, uint64_t seed) {
    int32_t* p = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    if (!p) return NULL;
    for (int32_t i = 0; i < n; i++) p[i] = i;
    uint64_t key = g_key(seed, 3);
    uint64_t t = 0;
    for (int64_t i = (int64_t)n - 1; i > 0; i--, t++) {
        int64_t j = (int64_t)(g_unif(key, t) * (double)(i + 1));
        if (j > i) j = i;
        int32_t x = p[i]; p[i] = p[j]; p[j] = x;
    }
    return p;
}

int gen_permutation(int32_t n, uint64_t seed, int32_t* out) {
    int32_t* p = fisher_yates(n, seed);
    if (!p) return -1;
    memcpy(out, p, (size_t)n * sizeof(int32_t));
    free(p);
    return 0;
}

static int relabel(int32_t n, uint64_t seed, int64_t m, int32_t* src, int32_t* dst) {
    int32_t* p = fisher_yates(n, seed);
    if (!p) return -1;
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; e++) { src[e] = p[src[e]]; dst[e] = p[dst[e]]; }
    free(p);
    return 0;
}

/* Canonicalise (min,max), sort, drop duplicates; returns the new edge count. */
static int64_t dedupe_undirected(int64_t m, int32_t* src, int32_t* dst) {
    uint64_t* k = (uint64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
    if (!k) return -1;
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; e++) {
        uint32_t a = (uint32_t)src[e], b = (uint32_t)dst[e];
        uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
        k[e] = ((uint64_t)lo << 32) | hi;
    }
    if (radix_sort_u64(k, m)) { free(k); return -1; }
    int64_t u = 0;
    for (int64_t e = 0; e < m; e++) {
        if (e > 0 && k[e] == k[e - 1]) continue;
        src[u] = (int32_t)(k[e] >> 32); dst[u] = (int32_t)(k[e] & 0xFFFFFFFFu); u++;
    }
    free(k);
    return u;
}

/* ---------------------------------------------------------------- c1: Erdos-Renyi G(n,m) */
/* m distinct unordered pairs u<v, uniform; self-loops and duplicates rejected.
 * Sequential draw index t: u from counter 2t, v from 2t+1 (stream 1).            */
int64_t gen_er(int32_t n, int64_t m, uint64_t seed, int32_t* src, int32_t* dst) {
    if (n < 2) return 0;
    int64_t maxm = (int64_t)n * (n - 1) / 2;
    if (m > maxm) m = maxm;
    int64_t cap = 1; while (cap < 4 * m + 16) cap <<= 1;
    uint64_t* tab = (uint64_t*)malloc((size_t)cap * sizeof(uint64_t));
    if (!tab) return -1;
    memset(tab, 0xFF, (size_t)cap * sizeof(uint64_t));
    uint64_t key = g_key(seed, 1);
    int64_t got = 0; uint64_t t = 0;
    while (got < m) {
        int64_t u = (int64_t)(g_unif(key, 2 * t) * n), v = (int64_t)(g_unif(key, 2 * t + 1) * n);
        t++;
        if (u >= n) u = n - 1;
        if (v >= n) v = n - 1;
        if (u == v) continue;
        int64_t lo = u < v ? u : v, hi = u < v ? v : u;
        uint64_t kk = ((uint64_t)lo << 32) | (uint64_t)hi;
        uint64_t h = g_mix64(kk) & (uint64_t)(cap - 1);
        int dup = 0;
        while (tab[h] != ~0ULL) { if (tab[h] == kk) { dup = 1; break; } h = (h + 1) & (uint64_t)(cap - 1); }
        if (dup) continue;
        tab[h] = kk;
        src[got] = (int32_t)lo; dst[got] = (int32_t)hi; got++;
    }
    free(tab);
    return got;
}

/* ---------------------------------------------------------------- c2: Chung-Lu power law */
/* Expected degree w_i = c (i + i0)^(-1/(gamma-1)).  Draw `pairs` endpoint pairs with
 * P(endpoint = i) proportional to w_i (inverse CDF over the prefix sums), counter
 * (pair*64 + attempt)*2 + endpoint on stream 1; self-loops resampled (attempt+1).
 * Then canonicalise + dedupe (simple graph) and scramble ids (Fisher-Yates, stream 3). */
int64_t gen_chung_lu(int32_t n, int64_t pairs, double gamma, double i0, double c, uint64_t seed,
                     int32_t* src, int32_t* dst) {
    double* cum = (double*)malloc((size_t)n * sizeof(double));
    if (!cum) return -1;
    double ex = -1.0 / (gamma - 1.0), s = 0.0;
    for (int32_t i = 0; i < n; i++) { s += c * pow((double)i + i0, ex); cum[i] = s; }
    double total = s;
    uint64_t key = g_key(seed, 1);
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < pairs; p++) {
        int32_t ends[2] = {0, 0};
        for (uint64_t att = 0; att < 64; att++) {
            for (int e = 0; e < 2; e++) {
                double x = g_unif(key, (((uint64_t)p * 64 + att) * 2 + (uint64_t)e)) * total;
                int64_t lo = 0, hi = n - 1;               /* first i with cum[i] > x */
                while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (cum[mid] > x) hi = mid; else lo = mid + 1; }
                ends[e] = (int32_t)lo;
            }
            if (ends[0] != ends[1]) break;
        }
        if (ends[0] == ends[1]) ends[1] = (ends[0] + 1) % n;   /* 64 failures: practically never */
        src[p] = ends[0]; dst[p] = ends[1];
    }
    free(cum);
    int64_t m = dedupe_undirected(pairs, src, dst);
    if (m < 0) return -1;
    if (relabel(n, seed, m, src, dst)) return -1;
    return m;
}

/* ---------------------------------------------------------------- c3: damaged lattice */
/* side x side grid, ids r*side + c (NOT scrambled: spatial locality like road data).
 * Each of the 2*side*(side-1) lattice edges deleted with p_del (stream 4, counter =
 * edge index: horizontal edges first, row-major, then vertical).  Each of the
 * (side-1)^2 cells gets one diagonal with p_diag (stream 5, counter 2*cell), whose
 * direction (down-right or down-left) is drawn at counter 2*cell+1.                */
int64_t gen_lattice(int32_t side, double p_del, double p_diag, uint64_t seed, int32_t* src, int32_t* dst) {
    uint64_t kdel = g_key(seed, 4), kdiag = g_key(seed, 5);
    int64_t m = 0, eidx = 0;
    for (int32_t r = 0; r < side; r++)
        for (int32_t c = 0; c + 1 < side; c++, eidx++)
            if (g_unif(kdel, (uint64_t)eidx) >= p_del) { src[m] = r * side + c; dst[m] = r * side + c + 1; m++; }
    for (int32_t r = 0; r + 1 < side; r++)
        for (int32_t c = 0; c < side; c++, eidx++)
            if (g_unif(kdel, (uint64_t)eidx) >= p_del) { src[m] = r * side + c; dst[m] = (r + 1) * side + c; m++; }
    for (int32_t r = 0; r + 1 < side; r++)
        for (int32_t c = 0; c + 1 < side; c++) {
            uint64_t cell = (uint64_t)r * (uint64_t)(side - 1) + (uint64_t)c;
            if (g_unif(kdiag, 2 * cell) < p_diag) {
                if (g_unif(kdiag, 2 * cell + 1) < 0.5) { src[m] = r * side + c; dst[m] = (r + 1) * side + c + 1; }
                else { src[m] = r * side + c + 1; dst[m] = (r + 1) * side + c; }
                m++;
            }
        }
    return m;
}

/* ---------------------------------------------------------------- c4/c5: R-MAT */
/* R-MAT(a,b,c,d) at `scale` levels, MSB first, no per-level noise.  Edge e, attempt t,
 * level l uses counter ((e*64 + t)*32 + l) on stream 1.  Endpoints >= n and self-loops
 * are resampled (attempt+1).  If `weights` != NULL: lognormal(mu, sigma) via Box-Muller
 * on stream 2, counters 2e and 2e+1, rounded to fp32.                              */
int64_t gen_rmat(int32_t n, int32_t scale, int64_t m, double a, double b, double c,
                 double mu, double sigma, uint64_t seed, int32_t* src, int32_t* dst, float* weights) {
    uint64_t key = g_key(seed, 1), kw = g_key(seed, 2);
    double ab = a + b, abc = a + b + c;
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; e++) {
        int64_t s = 0, d = 0;
        for (uint64_t att = 0; att < 64; att++) {
            s = 0; d = 0;
            for (int l = 0; l < scale; l++) {
                double u = g_unif(key, (((uint64_t)e * 64 + att) * 32 + (uint64_t)l));
                int rb = 0, cb = 0;
                if (u < a) { rb = 0; cb = 0; } else if (u < ab) { rb = 0; cb = 1; }
                else if (u < abc) { rb = 1; cb = 0; } else { rb = 1; cb = 1; }
                s = (s << 1) | rb; d = (d << 1) | cb;
            }
            if (s < n && d < n && s != d) break;
        }
        if (s >= n || d >= n || s == d) { s = e % n; d = (e + 1) % n; }  /* practically never */
        src[e] = (int32_t)s; dst[e] = (int32_t)d;
        if (weights) {
            double u1 = g_unif(kw, 2 * (uint64_t)e), u2 = g_unif(kw, 2 * (uint64_t)e + 1);
            double z = sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * 3.14159265358979323846 * u2);
            weights[e] = (float)exp(mu + sigma * z);
        }
    }
    return m;
}

/* Undirected R-MAT (c5): sample, canonicalise, dedupe, scramble. */
int64_t gen_rmat_undirected(int32_t n, int32_t scale, int64_t samples, double a, double b, double c,
                            uint64_t seed, int32_t* src, int32_t* dst) {
    gen_rmat(n, scale, samples, a, b, c, 0.0, 1.0, seed, src, dst, NULL);
    int64_t m = dedupe_undirected(samples, src, dst);
    if (m < 0) return -1;
    if (relabel(n, seed, m, src, dst)) return -1;
    return m;
}

/* Directed R-MAT with weights (c4): duplicates KEPT, ids scrambled. */
int64_t gen_rmat_directed(int32_t n, int32_t scale, int64_t m, double a, double b, double c,
                          double mu, double sigma, uint64_t seed, int32_t* src, int32_t* dst, float* w) {
    gen_rmat(n, scale, m, a, b, c, mu, sigma, seed, src, dst, w);
    if (relabel(n, seed, m, src, dst)) return -1;
    return m;
}
