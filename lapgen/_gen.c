/*
 * lapgen/_gen.c -- seeded synthetic-graph generators (INPUT GENERATION ONLY).
 *
 * This file holds none of the solver method's arithmetic.  It produces the
 * edge lists that stand in for the paper's graphs (BASELINE.json configs 4/5,
 * SURVEY.md §8(d) M1); both the CPU oracle and the CUDA library read the
 * CSR that lapgen/__init__.py builds from these edges.
 *
 * Random numbers: a counter-based stream  r(k) = sm64(stream_seed + k*GOLDEN)
 * where sm64 is the SplitMix64 finaliser.  This is the generator's own copy;
 * the method's hash (O-S11) is implemented separately in oracle/ and csrc/.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t gen_sm64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* uniform integer in [0, m) from a 64-bit word (multiply-high reduction) */
static inline uint64_t gen_below(uint64_t r, uint64_t m) {
    return (uint64_t)(((unsigned __int128)r * (unsigned __int128)m) >> 64);
}

/*
 * Barabasi-Albert preferential attachment (BASELINE.json configs[3]).
 * Start: clique on vertices 0..m (m+1 vertices).  For t = m+1 .. n-1 choose m
 * DISTINCT targets by uniform sampling from the endpoint list of the existing
 * edges (probability proportional to degree), rejecting repeats.
 * Outputs the undirected edges (u[e] < v[e] not guaranteed; u = new vertex).
 * Returns the number of edges written, or -1 if cap is too small.
 */
int64_t gen_barabasi_albert(int64_t n, int32_t m, uint64_t seed,
                            int32_t *eu, int32_t *ev, int64_t cap) {
    int64_t ne = 0;
    int64_t k0 = (int64_t)m + 1;
    if (n < k0) k0 = n;
    int64_t max_edges = k0 * (k0 - 1) / 2 + (n - k0) * (int64_t)m;
    if (cap < max_edges) return -1;
    int32_t *ends = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)max_edges);
    if (!ends) return -1;
    int64_t nends = 0;
    for (int64_t a = 0; a < k0; a++)
        for (int64_t b = a + 1; b < k0; b++) {
            eu[ne] = (int32_t)a; ev[ne] = (int32_t)b; ne++;
            ends[nends++] = (int32_t)a; ends[nends++] = (int32_t)b;
        }
    uint64_t stream = gen_sm64(seed ^ 0x4241424152414241ULL); /* "BABARABA" */
    uint64_t ctr = 0;
    int32_t tg[64];
    for (int64_t t = k0; t < n; t++) {
        int got = 0;
        while (got < m) {
            uint64_t r = gen_sm64(stream + (ctr++) * 0x9E3779B97F4A7C15ULL);
            int32_t c = ends[gen_below(r, (uint64_t)nends)];
            int dup = 0;
            for (int q = 0; q < got; q++) if (tg[q] == c) { dup = 1; break; }
            if (!dup) tg[got++] = c;
        }
        for (int q = 0; q < m; q++) {
            eu[ne] = (int32_t)t; ev[ne] = tg[q]; ne++;
            ends[nends++] = (int32_t)t; ends[nends++] = tg[q];
        }
    }
    free(ends);
    return ne;
}

/*
 * R-MAT edge generator with counter-based randoms (for scales too large for
 * numpy; BASELINE.json configs[4]).  Per edge and per bit level, one uniform
 * double picks a quadrant with probabilities (a,b,c,d): the u-bit is set for
 * quadrants c and d, the v-bit for b and d (Graph500 convention, no noise).
 * Edge e uses words r(e*scale + level).  Parallel over edges with OpenMP if
 * compiled with it; the output is independent of the thread count.
 */
void gen_rmat(int32_t scale, int64_t nedges, double a, double b, double c,
              uint64_t seed, int64_t *eu, int64_t *ev) {
    uint64_t stream = gen_sm64(seed ^ 0x524D4154524D4154ULL); /* "RMATRMAT" */
    double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < nedges; e++) {
        int64_t u = 0, v = 0;
        for (int32_t l = 0; l < scale; l++) {
            uint64_t r = gen_sm64(stream + (uint64_t)(e * scale + l) * 0x9E3779B97F4A7C15ULL);
            double x = (double)(r >> 11) * 0x1.0p-53;
            int ub = 0, vb = 0;
            if (x < a) { }
            else if (x < ab) { vb = 1; }
            else if (x < abc) { ub = 1; }
            else { ub = 1; vb = 1; }
            u = (u << 1) | ub;
            v = (v << 1) | vb;
        }
        eu[e] = u; ev[e] = v;
    }
}

/*
 * Symmetric CSR from an undirected edge list (u[e], v[e], w[e]), u != v, no
 * duplicate pairs: both directions are stored, columns ascending per row.
 * row_ptr has n+1 entries; col/val have 2*ne entries.  Counting sort by row,
 * then insertion/shell sort of each row by column (rows are short on average).
 */
static void gen_sort_row(int32_t *c, double *x, int64_t len) {
    /* shell sort on (c, x) by c; stable order is irrelevant (no duplicates) */
    static const int64_t gaps[] = {701, 301, 132, 57, 23, 10, 4, 1};
    for (int g = 0; g < 8; g++) {
        int64_t gap = gaps[g];
        for (int64_t i = gap; i < len; i++) {
            int32_t tc = c[i]; double tx = x[i];
            int64_t j = i;
            while (j >= gap && c[j - gap] > tc) { c[j] = c[j - gap]; x[j] = x[j - gap]; j -= gap; }
            c[j] = tc; x[j] = tx;
        }
    }
}

static int gen_cmp_pair(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

void gen_csr_from_edges(int64_t n, int64_t ne, const int64_t *u, const int64_t *v,
                        const double *w, int64_t *row_ptr, int32_t *col, double *val) {
    memset(row_ptr, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t e = 0; e < ne; e++) { row_ptr[u[e] + 1]++; row_ptr[v[e] + 1]++; }
    for (int64_t i = 0; i < n; i++) row_ptr[i + 1] += row_ptr[i];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    memcpy(fill, row_ptr, sizeof(int64_t) * (size_t)n);
    for (int64_t e = 0; e < ne; e++) {
        int64_t p = fill[u[e]]++; col[p] = (int32_t)v[e]; val[p] = w ? w[e] : 1.0;
        int64_t q = fill[v[e]]++; col[q] = (int32_t)u[e]; val[q] = w ? w[e] : 1.0;
    }
    free(fill);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++) {
        int64_t len = row_ptr[i + 1] - row_ptr[i];
        if (len > 4096) {
            /* long rows: sort (col,val) pairs packed as 16-byte records */
            struct { int32_t c; int32_t pad; double x; } *tmp = malloc(16 * (size_t)len);
            for (int64_t k = 0; k < len; k++) { tmp[k].c = col[row_ptr[i] + k]; tmp[k].pad = 0; tmp[k].x = val[row_ptr[i] + k]; }
            qsort(tmp, (size_t)len, 16, gen_cmp_pair);
            for (int64_t k = 0; k < len; k++) { col[row_ptr[i] + k] = tmp[k].c; val[row_ptr[i] + k] = tmp[k].x; }
            free(tmp);
        } else {
            gen_sort_row(col + row_ptr[i], val + row_ptr[i], len);
        }
    }
}

/*
 * R-MAT at scales numpy cannot handle (BASELINE.json configs[4], scale 26,
 * 2^30 generated edges): the whole pipeline of lapgen.rmat_large in C/OpenMP,
 * producing the same CSR as gen_rmat + dedup_undirected + csr_from_edges +
 * largest_component (checked at small scales in tests/test_lapgen.py):
 *   1. edges from gen_rmat's counter stream, self loops dropped, key =
 *      (min << 32) | max;
 *   2. parallel LSD radix sort of the keys, duplicates dropped;
 *   3. union-find over the unique edges, the largest component kept (ties:
 *      the smallest root label as numpy's argmax over bincount picks the
 *      first maximum of the component labels ordered by smallest vertex),
 *      vertices relabelled by ascending original id;
 *   4. symmetric CSR, columns ascending, unit weights (w not materialised).
 * Two calls: gen_rmat_lcc_build() returns a handle with n and nnz; then
 * gen_rmat_lcc_fetch() copies row_ptr/col out and frees the handle.
 */
typedef struct { int64_t n, nnz; int64_t *row_ptr; int32_t *col; } gen_csr_t;

static void gen_radix_sort_u64(uint64_t *a, uint64_t *tmp, int64_t n, int bits) {
    const int R = 11, B = 1 << R;
    int nth = 1;
#ifdef _OPENMP
    nth = omp_get_max_threads();
#endif
    int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * (size_t)B * (size_t)nth);
    uint64_t *src = a, *dst = tmp;
    for (int sh = 0; sh < bits; sh += R) {
        memset(hist, 0, sizeof(int64_t) * (size_t)B * (size_t)nth);
#pragma omp parallel num_threads(nth)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            int64_t lo = n * t / nth, hi = n * (t + 1) / nth;
            int64_t *h = hist + (size_t)t * B;
            for (int64_t i = lo; i < hi; i++) h[(src[i] >> sh) & (B - 1)]++;
#pragma omp barrier
#pragma omp single
            {
                int64_t run = 0;
                for (int d = 0; d < B; d++)
                    for (int q = 0; q < nth; q++) {
                        int64_t c = hist[(size_t)q * B + d];
                        hist[(size_t)q * B + d] = run;
                        run += c;
                    }
            }
            for (int64_t i = lo; i < hi; i++) dst[h[(src[i] >> sh) & (B - 1)]++] = src[i];
        }
        uint64_t *x = src; src = dst; dst = x;
    }
    if (src != a) memcpy(a, src, sizeof(uint64_t) * (size_t)n);
    free(hist);
}

static int64_t gen_uf_find(int64_t *p, int64_t x) {
    while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
    return x;
}

void *gen_rmat_lcc_build(int32_t scale, int64_t nedges, double a, double b, double c, uint64_t seed,
                         int64_t *n_out, int64_t *nnz_out) {
    const int64_t N = (int64_t)1 << scale;
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)nedges);
    uint64_t stream = gen_sm64(seed ^ 0x524D4154524D4154ULL); /* same stream as gen_rmat */
    double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < nedges; e++) {
        int64_t u = 0, v = 0;
        for (int32_t l = 0; l < scale; l++) {
            uint64_t r = gen_sm64(stream + (uint64_t)(e * scale + l) * 0x9E3779B97F4A7C15ULL);
            double x = (double)(r >> 11) * 0x1.0p-53;
            int ub = 0, vb = 0;
            if (x < a) { }
            else if (x < ab) { vb = 1; }
            else if (x < abc) { ub = 1; }
            else { ub = 1; vb = 1; }
            u = (u << 1) | ub;
            v = (v << 1) | vb;
        }
        uint64_t lo = (uint64_t)(u < v ? u : v), hi = (uint64_t)(u < v ? v : u);
        key[e] = (u == v) ? UINT64_MAX : ((lo << 32) | hi);   /* self loops sort last, dropped below */
    }
    uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)nedges);
    gen_radix_sort_u64(key, tmp, nedges, 64);
    free(tmp);
    /* unique, self loops (UINT64_MAX) dropped */
    int64_t m = 0;
    for (int64_t e = 0; e < nedges; e++) {
        if (key[e] == UINT64_MAX) break;
        if (m == 0 || key[e] != key[m - 1]) key[m++] = key[e];
    }
    /* components */
    int64_t *par = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    for (int64_t i = 0; i < N; i++) par[i] = i;
    for (int64_t e = 0; e < m; e++) {
        int64_t x = gen_uf_find(par, (int64_t)(key[e] >> 32)), y = gen_uf_find(par, (int64_t)(key[e] & 0xFFFFFFFFULL));
        if (x != y) { if (x < y) par[y] = x; else par[x] = y; }   /* root = smallest vertex of the component */
    }
    int64_t *size = (int64_t *)calloc((size_t)N, sizeof(int64_t));
    for (int64_t i = 0; i < N; i++) size[gen_uf_find(par, i)]++;
    int64_t best = 0;
    for (int64_t i = 1; i < N; i++) if (size[i] > size[best]) best = i;   /* first maximum: smallest root */
    free(size);
    int32_t *nid = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
    int64_t n = 0;
    for (int64_t i = 0; i < N; i++) nid[i] = (par[i] == i ? i : gen_uf_find(par, i)) == best ? (int32_t)n++ : -1;
    free(par);
    gen_csr_t *g = (gen_csr_t *)malloc(sizeof(gen_csr_t));
    g->n = n;
    g->row_ptr = (int64_t *)calloc((size_t)(n + 1), sizeof(int64_t));
    for (int64_t e = 0; e < m; e++) {
        int32_t u = nid[key[e] >> 32], v = nid[key[e] & 0xFFFFFFFFULL];
        if (u < 0) continue;
        g->row_ptr[u + 1]++;
        g->row_ptr[v + 1]++;
    }
    for (int64_t i = 0; i < n; i++) g->row_ptr[i + 1] += g->row_ptr[i];
    g->nnz = g->row_ptr[n];
    g->col = (int32_t *)malloc(sizeof(int32_t) * (size_t)(g->nnz + 1));
    /* keys are sorted by (min, max): a row's smaller neighbours (key max = row)
     * arrive in ascending min, its larger ones (key min = row) in ascending max,
     * and every smaller one precedes every larger one in key order */
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    memcpy(fill, g->row_ptr, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t e = 0; e < m; e++) {
        int32_t u = nid[key[e] >> 32], v = nid[key[e] & 0xFFFFFFFFULL];
        if (u < 0) continue;
        g->col[fill[v]++] = u;   /* u < v: a smaller neighbour of v */
    }
    /* larger neighbours after the smaller ones: second pass in key order */
    for (int64_t e = 0; e < m; e++) {
        int32_t u = nid[key[e] >> 32], v = nid[key[e] & 0xFFFFFFFFULL];
        if (u < 0) continue;
        g->col[fill[u]++] = v;
    }
    free(fill);
    free(nid);
    free(key);
    *n_out = g->n;
    *nnz_out = g->nnz;
    return g;
}

void gen_rmat_lcc_fetch(void *h, int64_t *row_ptr, int32_t *col) {
    gen_csr_t *g = (gen_csr_t *)h;
    memcpy(row_ptr, g->row_ptr, sizeof(int64_t) * (size_t)(g->n + 1));
    memcpy(col, g->col, sizeof(int32_t) * (size_t)g->nnz);
    free(g->row_ptr);
    free(g->col);
    free(g);
}
