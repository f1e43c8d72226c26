/*
 * cleora_oracle.c -- the CPU ORACLE for Cleora's hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this.  The product path (paper_2102_02302_b200/) never does, and the
 * two share no code: no headers, helpers, constants generators or kernels.
 *
 * It is the plain definition of the method, written out slowly and obviously:
 *   Rychalska et al., "Cleora: A Simple, Strong and Scalable Graph Embedding Scheme",
 *   arXiv 2102.02302, §3.2 "Embedding" and Algorithm 1
 *   with Q = 1 chunk:
 *       M_ab = e_ab / deg(v_a)
 *       T_0 ~ U(-1, 1)
 *       for i = 1..I:  T_i = M . T_{i-1};  L2-normalise rows
 * Readings where the paper is silent are SURVEY.md §8(c) points 1-12/Z, listed in
 * DESIGN.md §"Readings of the paper"; each step below names the one it uses.
 *
 * Precision: accumulate in fp64, store fp32 once per iteration (4-byte storage of T,
 * PAPER.md:174 "2 x d x |V| objects of 4 bytes").  Accumulation order: ascending
 * column within a row, then ascending j for the sum of squares (reading 8).
 *
 * Parallelism: rows are independent (Alg. 1 line 5 is a row-wise product), so
 * OpenMP splits rows across host threads; each row is computed sequentially, hence
 * the result does not depend on the thread count.  No blocking, no fusion.
 *
 * Error codes mirror include/cleora.h (2 usage, 3 data) but are defined here again on
 * purpose (no shared header).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EUSAGE 2
#define OR_EDATA 3
#define OR_ENOMEM 4

/* ------------------------------------------------------------------ B1-B4: M in CSR */

typedef struct {
    int32_t src, dst;
    int64_t pos;   /* position in the entry list: originals 0..E-1, mirrors E.. */
    double w;      /* the edge weight (1.0 when unweighted)                     */
} or_entry;

static int or_cmp(const void* pa, const void* pb) {
    const or_entry* a = (const or_entry*)pa;
    const or_entry* b = (const or_entry*)pb;
    if (a->src != b->src) return a->src < b->src ? -1 : 1;
    if (a->dst != b->dst) return a->dst < b->dst ? -1 : 1;
    /* ties broken by list position => qsort becomes a STABLE sort (reading B1) */
    if (a->pos != b->pos) return a->pos < b->pos ? -1 : 1;
    return 0;
}

typedef struct {
    int32_t n;
    int64_t nnz;
    int64_t* row_ptr;  /* [n+1] */
    int32_t* col;      /* [nnz] */
    float* val;        /* [nnz]  M_ab = fp32_rn(e_ab / deg(a))  */
    double* e;         /* [nnz]  e_ab (merged weight, fp64)     */
    double* deg;       /* [n]    deg(a) = sum_b e_ab            */
} oracle_csr;

void oracle_csr_free(oracle_csr* m) {
    if (!m) return;
    free(m->row_ptr); free(m->col); free(m->val); free(m->e); free(m->deg); free(m);
}

/*
 * Build M = D^-1 A (Alg. 1 line 3).
 *   B1 entry list: the input edges in input order; if undirected, then one mirror
 *      (v,u,w) per edge with u != v, in input order (a self-loop appears once:
 *      reading 5; "count an edge in both directions").  Stable sort
 *      by (src, dst).
 *   B2 e_ab = fp64 sum, left to right in that order, of the weights of all entries
 *      equal to (a,b): "e_ab is the number of edges running from node a to b ... If
 *      edges have attached weights, e_ab is the sum of the weights".
 *   B3 deg(a) = fp64 sum of e_ab over ascending b: the weighted out-degree, so M is
 *      row-stochastic (reading 2; directed rows use out-edges, reading 3).
 *   B4 M_ab = (float)(e_ab / deg(a)), one fp64 division rounded once to fp32.
 * Validation (§8(b)): 0 <= id < n, weight finite and > 0.
 */
int oracle_build(const int32_t* src, const int32_t* dst, const float* w, int64_t n_edges,
                 int32_t n, int32_t directed, oracle_csr** out) {
    *out = NULL;
    if (!src || !dst || n <= 0 || n_edges <= 0) return OR_EUSAGE;
    for (int64_t i = 0; i < n_edges; i++) {
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) return OR_EDATA;
        if (w && !(isfinite(w[i]) && w[i] > 0.0f)) return OR_EDATA;
    }
    /* B1 */
    int64_t cap = directed ? n_edges : 2 * n_edges;
    or_entry* ent = (or_entry*)malloc((size_t)cap * sizeof(or_entry));
    if (!ent) return OR_ENOMEM;
    int64_t m = 0;
    for (int64_t i = 0; i < n_edges; i++) {
        ent[m].src = src[i]; ent[m].dst = dst[i]; ent[m].pos = m;
        ent[m].w = w ? (double)w[i] : 1.0; m++;
    }
    if (!directed) {
        for (int64_t i = 0; i < n_edges; i++) {
            if (src[i] == dst[i]) continue;
            ent[m].src = dst[i]; ent[m].dst = src[i]; ent[m].pos = m;
            ent[m].w = w ? (double)w[i] : 1.0; m++;
        }
    }
    qsort(ent, (size_t)m, sizeof(or_entry), or_cmp);

    oracle_csr* M = (oracle_csr*)calloc(1, sizeof(oracle_csr));
    if (!M) { free(ent); return OR_ENOMEM; }
    M->n = n;
    /* B2: merge equal (a,b) by summing weights in stable order */
    int64_t nnz = 0;
    for (int64_t i = 0; i < m; i++)
        if (i == 0 || ent[i].src != ent[i - 1].src || ent[i].dst != ent[i - 1].dst) nnz++;
    M->nnz = nnz;
    M->row_ptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    M->col = (int32_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
    M->val = (float*)malloc((size_t)(nnz ? nnz : 1) * sizeof(float));
    M->e = (double*)malloc((size_t)(nnz ? nnz : 1) * sizeof(double));
    M->deg = (double*)calloc((size_t)n, sizeof(double));
    int32_t* row = (int32_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
    if (!M->row_ptr || !M->col || !M->val || !M->e || !M->deg || !row) {
        free(row); free(ent); oracle_csr_free(M); return OR_ENOMEM;
    }
    int64_t k = -1;
    for (int64_t i = 0; i < m; i++) {
        if (i == 0 || ent[i].src != ent[i - 1].src || ent[i].dst != ent[i - 1].dst) {
            k++;
            row[k] = ent[i].src; M->col[k] = ent[i].dst; M->e[k] = 0.0;
        }
        M->e[k] = M->e[k] + ent[i].w;
    }
    free(ent);
    /* row pointer: count entries per row, exclusive prefix sum */
    for (int64_t q = 0; q < nnz; q++) M->row_ptr[row[q] + 1]++;
    for (int32_t a = 0; a < n; a++) M->row_ptr[a + 1] += M->row_ptr[a];
    free(row);
    /* B3: deg(a) = sum over ascending b of e_ab (entries of a row are sorted by b) */
    for (int32_t a = 0; a < n; a++) {
        double s = 0.0;
        for (int64_t q = M->row_ptr[a]; q < M->row_ptr[a + 1]; q++) s = s + M->e[q];
        M->deg[a] = s;
    }
    /* B4: M_ab = e_ab / deg(a), rounded once to fp32 */
    for (int32_t a = 0; a < n; a++)
        for (int64_t q = M->row_ptr[a]; q < M->row_ptr[a + 1]; q++)
            M->val[q] = (float)(M->e[q] / M->deg[a]);
    *out = M;
    return OR_OK;
}

int64_t oracle_csr_nnz(const oracle_csr* m) { return m->nnz; }
int32_t oracle_csr_n(const oracle_csr* m) { return m->n; }

void oracle_csr_copy(const oracle_csr* m, int64_t* row_ptr, int32_t* col, float* val, double* e, double* deg) {
    if (row_ptr) memcpy(row_ptr, m->row_ptr, ((size_t)m->n + 1) * sizeof(int64_t));
    if (col) memcpy(col, m->col, (size_t)m->nnz * sizeof(int32_t));
    if (val) memcpy(val, m->val, (size_t)m->nnz * sizeof(float));
    if (e) memcpy(e, m->e, (size_t)m->nnz * sizeof(double));
    if (deg) memcpy(deg, m->deg, (size_t)m->n * sizeof(double));
}

/* ------------------------------------------------------------------ I1: T_0 */

/* SplitMix64 output function (Steele, Lea, Flood 2014), all arithmetic mod 2^64. */
static uint64_t or_splitmix64_mix(uint64_t z) {
    z = z ^ (z >> 30);
    z = z * 0xBF58476D1CE4E5B9ULL;
    z = z ^ (z >> 27);
    z = z * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    return z;
}

/*
 * T_0[v][j] = H(seed, v, j)  -- "T_0 ~ U(-1, 1)" (Alg. 1 line 4
 * ); BASELINE.json: "initialised deterministically from a hash of
 * (node id, dimension) into [-1,1]".  Reading 1:
 *     s = mix(seed + 0x9E3779B97F4A7C15)
 *     h = mix(s XOR (v << 32 | j))
 *     T_0 = ((int)(h >> 40) - 2^23) * 2^-23   in [-1, 1 - 2^-23], exact in fp32.
 * The paper fixes only the distribution, so exact values are parity-unpinned BY THE
 * PAPER; the distribution is pinned by tests (range, mean, variance, pairwise cos).
 */
float oracle_hash_value(uint64_t seed, int64_t v, int64_t j) {
    uint64_t s = or_splitmix64_mix(seed + 0x9E3779B97F4A7C15ULL);
    uint64_t h = or_splitmix64_mix(s ^ (((uint64_t)v << 32) | (uint64_t)j));
    int64_t top24 = (int64_t)(h >> 40);                 /* 0 .. 2^24-1 */
    double x = (double)(top24 - 8388608) / 8388608.0;   /* exact */
    return (float)x;
}

void oracle_hash_init(uint64_t seed, int64_t row_begin, int64_t row_end, int32_t d, float* out) {
    #pragma omp parallel for schedule(static)
    for (int64_t v = row_begin; v < row_end; v++)
        for (int32_t j = 0; j < d; j++)
            out[(v - row_begin) * (int64_t)d + j] = oracle_hash_value(seed, v, j);
}

/* ------------------------------------------------------------------ O1: one iteration */

/*
 * T_out[a] = normalize( sum_b M_ab T_in[b] )  for rows a in [r0, r1)
 * Alg. 1 lines 6-7: "T_i = M . T_{i-1}; L2 normalize rows of T_i".
 *   acc[j] = sum_k (double)val[k] * (double)T_in[col[k]][j],  k ascending
 *   ss     = sum_j acc[j]^2                                     j ascending
 *   T_out[a][j] = ss == 0 ? 0 : (float)(acc[j] / sqrt(ss))
 * Reading Z: a row without out-edges gives the zero vector and stays zero.
 * Reading 6: exact ss == 0 test, no epsilon.  Reading 10: normalise ROWS.
 * T_out rows are written at (a - r0) * d.
 */
void oracle_step_rows(const oracle_csr* M, int32_t d, const float* T_in, float* T_out, int64_t r0, int64_t r1) {
    #pragma omp parallel
    {
        double* acc = (double*)malloc((size_t)d * sizeof(double));
        #pragma omp for schedule(dynamic, 1024)
        for (int64_t a = r0; a < r1; a++) {
            for (int32_t j = 0; j < d; j++) acc[j] = 0.0;
            for (int64_t k = M->row_ptr[a]; k < M->row_ptr[a + 1]; k++) {
                double mv = (double)M->val[k];
                const float* tb = T_in + (int64_t)M->col[k] * d;
                for (int32_t j = 0; j < d; j++) acc[j] = acc[j] + mv * (double)tb[j];
            }
            double ss = 0.0;
            for (int32_t j = 0; j < d; j++) ss = ss + acc[j] * acc[j];
            float* o = T_out + (a - r0) * (int64_t)d;
            if (ss == 0.0) {
                for (int32_t j = 0; j < d; j++) o[j] = 0.0f;
            } else {
                double nrm = sqrt(ss);
                for (int32_t j = 0; j < d; j++) o[j] = (float)(acc[j] / nrm);
            }
        }
        free(acc);
    }
}

/* Whole Algorithm 1 with Q = 1: T_0 from the hash, then `iters` steps.  T (n x d) in/out:
 * on return holds T_iters.  `work` is caller scratch of n*d floats. */
void oracle_embed(const oracle_csr* M, int32_t d, uint64_t seed, int32_t iters, float* T, float* work) {
    oracle_hash_init(seed, 0, M->n, d, T);
    float* a = T; float* b = work;
    for (int32_t i = 0; i < iters; i++) {
        oracle_step_rows(M, d, a, b, 0, M->n);
        float* t = a; a = b; b = t;
    }
    if (a != T) memcpy(T, a, (size_t)M->n * (size_t)d * sizeof(float));
}

/* ------------------------------------------------------------------ f1: chunks (Q > 1) */

/*
 * Algorithm 1 line 1: "Divide graph G into Q chunks.  Let G_q be the q-th chunk
 * with edge set E_q".  The paper does not say how; reading R13: edge i of the
 * input list goes to chunk
 *     q(i) = floor(Q * (h_i >> 32) / 2^32),   h_i = mix(mix(chunk_seed + 0x9E3779B97F4A7C15) XOR i)
 * (mix = the SplitMix64 output function above), so every edge is in exactly one chunk and the
 * assignment is deterministic and order-free ("deterministic hash-based edge
 * assignment").
 */
int32_t oracle_chunk_of_edge(uint64_t chunk_seed, int64_t i, int32_t Q) {
    uint64_t s = or_splitmix64_mix(chunk_seed + 0x9E3779B97F4A7C15ULL);
    uint64_t h = or_splitmix64_mix(s ^ (uint64_t)i);
    return (int32_t)(((h >> 32) * (uint64_t)Q) >> 32);
}

void oracle_chunk_assign(uint64_t chunk_seed, int64_t n_edges, int32_t Q, int32_t* out) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_edges; i++) out[i] = oracle_chunk_of_edge(chunk_seed, i, Q);
}

/*
 * Algorithm 1 lines 10-12:
 *     T_v = sum_q w_qv T^q_v,   w_qv = |n in V_q : n = n_v| / sum_k |n in V_k : n = n_v|
 * Reading R14: |n in V_q : n = n_v| = occurrences of v as an endpoint of the edges of E_q
 * (occ[q*n + v]; an edge contributes one occurrence to each of its two endpoints, a self-loop
 * two).  A node that occurs in no chunk gets the zero row.  No normalisation after the merge
 * (Algorithm 1 performs none).  Arithmetic: w = (double)occ / (double)total, one fp64 division;
 * acc = acc + w * (double)T^q[v][j] in fp64 over ascending q; one rounding to fp32 at the end.
 * Tq[q] points to chunk q's N x d fp32 embedding.
 */
void oracle_merge(const float* const* Tq, const int64_t* occ, int32_t Q, int32_t n, int32_t d, float* out) {
    #pragma omp parallel for schedule(static)
    for (int32_t v = 0; v < n; v++) {
        int64_t tot = 0;
        for (int32_t q = 0; q < Q; q++) tot += occ[(int64_t)q * n + v];
        float* o = out + (int64_t)v * d;
        for (int32_t j = 0; j < d; j++) {
            double acc = 0.0;
            if (tot > 0)
                for (int32_t q = 0; q < Q; q++) {
                    double w = (double)occ[(int64_t)q * n + v] / (double)tot;
                    acc = acc + w * (double)Tq[q][(int64_t)v * d + j];
                }
            o[j] = (float)acc;
        }
    }
}

/* Threads the oracle will use (for reporting cpu_baseline.cores). */
int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
