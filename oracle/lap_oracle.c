/*
 * oracle/lap_oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY; see header).
 *
 * Plain C99 + GCC __int128, compiled with -ffp-contract=off so every
 * floating operation below is one IEEE-754 round-to-nearest-even operation in
 * the order written.  Optional OpenMP ("all host cores ...
 * bitwise identical to the 1-thread run"): only loops whose iterations are
 * independent (one row, one entry, one aggregate each) are parallel; integer
 * counters are atomic; every floating sum keeps one fixed order whatever the
 * thread count (per-row / per-aggregate loops in ascending index order, dot
 * products in fixed 4096-element chunks, CanonSums exact).  The result does
 * not depend on the number of threads (tests/test_oracle_threads.py).  Each function cites the PAPER.md (P:)
 * passage it follows and the SURVEY.md §8(c) reading (O-Rxx / O-Sxx) that
 * resolves what the paper leaves open.
 *
 * Nothing here is shared with the CUDA library: it has its own hash, its own
 * canonical sum, its own solver.  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline leg may load it.
 */
#include "lap_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* number of OpenMP threads the oracle uses (1 without OpenMP) */
void orc_set_threads(int32_t t) {
#ifdef _OPENMP
    omp_set_num_threads(t > 0 ? t : 1);
#else
    (void)t;
#endif
}
int32_t orc_get_threads(void) {
#ifdef _OPENMP
    return (int32_t)omp_get_max_threads();
#else
    return 1;
#endif
}

typedef __int128 i128;
typedef unsigned __int128 u128;

enum { ST_DECIDED = 0, ST_UNDECIDED = 1, ST_SEED = 2 };  /* rank order */

void orc_params_default(orc_params *p) {
    p->tol = 1e-8;
    p->max_iters = 500;
    p->cheby_degree = 2;
    p->cheby_lo = 0.3;
    p->cheby_hi = 1.1;
    p->lanczos_steps = 10;
    p->elim_max_degree = 4;
    p->elim_enable = 1;
    p->n_test_vectors = 4;
    p->tv_sweeps = 3;
    p->tv_omega = 2.0 / 3.0;  /* O-R6 */
    p->vote_rounds = 10;
    p->vote_threshold = 8;    /* P:619 (>=), O-R8 */
    p->coarse_nnz = 1000;
    p->max_levels = 40;
    p->seed = 0;
    p->random_order = 1;
    p->affinity_power = 1;    /* O-R5 */
    p->cycle = 0;             /* V-cycle by default */
    p->kcycle_inner = 2;      /* S:525 / S:562 (paper: "a number of") */
    p->elim_rounds = 1;       /* "one iteration is sufficient" */
}

/* ======================================================================== */
/* O-S11 canonical arithmetic                                               */
/* ======================================================================== */

/* SplitMix64 output function (Steele, Lea & Flood 2014); bijective. O-S11 */
uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    return z;
}

/* salt_k = mix64(seed XOR k*0x9E3779B97F4A7C15); k=1 perm, 2 elim hash,
 * 3 test vectors, 4 Lanczos (O-S11). */
uint64_t orc_salt(uint64_t seed, uint64_t k) {
    return orc_mix64(seed ^ (k * 0x9E3779B97F4A7C15ULL));
}

static uint64_t unxorshift(uint64_t z, int s) {
    uint64_t x = z;
    for (int i = 0; i < 64 / s + 1; i++) x = z ^ (x >> s);
    return x;
}

static uint64_t inv_mul(uint64_t a) {
    /* Newton iteration for the inverse of an odd number mod 2^64 */
    uint64_t x = a;
    for (int i = 0; i < 6; i++) x *= 2 - a * x;
    return x;
}

uint64_t orc_mix64_inverse(uint64_t z) {
    z = unxorshift(z, 31);
    z *= inv_mul(0x94D049BB133111EBULL);
    z = unxorshift(z, 27);
    z *= inv_mul(0xBF58476D1CE4E5B9ULL);
    z = unxorshift(z, 30);
    return z;
}

/* ilogb for finite nonzero x; 0 -> a very small sentinel */
int32_t orc_ilogb(double x) {
    if (x == 0.0) return -2000;
    return (int32_t)ilogb(x);
}

static int32_t bitlen64(uint64_t k) {
    int32_t c = 0;
    while (k) { c++; k >>= 1; }
    return c;
}

/* E_lo = e_max + ceil(log2(K+1)) - 125 ; ceil(log2(K+1)) = bit length of K. */
int32_t orc_canon_elo(int32_t e_max, int64_t K) {
    return e_max + bitlen64((uint64_t)K) - 125;
}

/* q(t) = round-half-even(t * 2^-E_lo) as an exact integer (O-S11). */
static i128 canon_quant(double t, int32_t E_lo) {
    if (t == 0.0) return 0;
    uint64_t bits;
    memcpy(&bits, &t, 8);
    int neg = (int)(bits >> 63);
    int ex = (int)((bits >> 52) & 0x7FF);
    uint64_t man = bits & 0xFFFFFFFFFFFFFULL;
    int e;
    if (ex == 0) e = -1074;
    else { man |= 1ULL << 52; e = ex - 1075; }
    /* |t| = man * 2^e ; t * 2^-E_lo = man * 2^(e - E_lo) */
    int sh = e - E_lo;
    u128 q;
    if (sh >= 0) {
        q = (u128)man << sh;   /* caller guarantees no overflow (|t| <= 2^e_max) */
    } else {
        int r = -sh;
        if (r >= 54) {
            q = 0;             /* man*2^-r < 2^53*2^-54 = 1/2 strictly */
        } else {
            uint64_t hi = man >> r;
            uint64_t rem = man & ((1ULL << r) - 1);
            uint64_t half = 1ULL << (r - 1);
            if (rem > half || (rem == half && (hi & 1))) hi++;
            q = hi;
        }
    }
    return neg ? -(i128)q : (i128)q;
}

/* round-half-even(Q) to fp64, times 2^E_lo (O-S11; done by hand). */
static double canon_to_double(i128 Q, int32_t E_lo) {
    if (Q == 0) return 0.0;
    int neg = Q < 0;
    u128 a = neg ? (u128)0 - (u128)Q : (u128)Q;
    int p = 127;
    while (!((a >> p) & 1)) p--;
    uint64_t m;
    int e = 0;
    if (p <= 52) {
        m = (uint64_t)a;
    } else {
        int s = p - 52;
        u128 hi = a >> s;
        u128 rem = a - (hi << s);
        u128 half = (u128)1 << (s - 1);
        if (rem > half || (rem == half && (hi & 1))) hi++;
        if (hi >> 53) { hi >>= 1; s++; }
        m = (uint64_t)hi;
        e = s;
    }
    double r = ldexp((double)m, e + E_lo);
    return neg ? -r : r;
}

/* CanonSum of cnt terms for an operation instance (e_max, K).  O-S11/O-R23 */
double orc_canon_sum(const double *t, int64_t cnt, int32_t e_max, int64_t K) {
    int32_t E_lo = orc_canon_elo(e_max, K);
    i128 Q = 0;
    for (int64_t k = 0; k < cnt; k++) Q += canon_quant(t[k], E_lo);
    return canon_to_double(Q, E_lo);
}

static double max_abs(const double *v, int64_t n) {
    double m = 0.0;
    #pragma omp parallel for reduction(max:m) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double a = fabs(v[i]);
        if (a > m) m = a;
    }
    return m;
}

/* CanonSum of fl(a_i * b_i) (b = NULL: of a_i) over a long vector; the int128
 * sum is exact, so the thread partials may be added in any order. */
static double canon_dot(const double *a, const double *b, int64_t n, int32_t e_max, int64_t K) {
    int32_t E_lo = orc_canon_elo(e_max, K);
    i128 Q = 0;
    #pragma omp parallel
    {
        i128 q = 0;
        #pragma omp for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            double t = b ? a[i] * b[i] : a[i];
            q += canon_quant(t, E_lo);
        }
        #pragma omp critical
        Q += q;
    }
    return canon_to_double(Q, E_lo);
}

/* ======================================================================== */
/* O-S0 validation                            */
/* ======================================================================== */

static int64_t find_in_row(const int64_t *row_ptr, const int32_t *col, int64_t i, int32_t j) {
    int64_t lo = row_ptr[i], hi = row_ptr[i + 1];
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (col[mid] < j) lo = mid + 1;
        else hi = mid;
    }
    if (lo < row_ptr[i + 1] && col[lo] == j) return lo;
    return -1;
}

int orc_validate(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w) {
    if (n < 1 || !row_ptr) return ORC_EINVAL;
    if (row_ptr[0] != 0) return ORC_EGRAPH;
    for (int64_t i = 0; i < n; i++) if (row_ptr[i + 1] < row_ptr[i]) return ORC_EGRAPH;
    int bad = 0;
    #pragma omp parallel for schedule(dynamic, 1024) reduction(|:bad)
    for (int64_t i = 0; i < n; i++) {
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1] && !bad; k++) {
            int32_t j = col[k];
            if (j < 0 || j >= n || j == i) { bad = 1; break; }              /* range, self loop */
            if (k > row_ptr[i] && col[k - 1] >= j) { bad = 1; break; }       /* sorted, unique */
            double wk = w ? w[k] : 1.0;
            if (!(wk > 0.0) || !isfinite(wk)) { bad = 1; break; }           /* w > 0 */
            int64_t t = find_in_row(row_ptr, col, j, (int32_t)i);
            if (t < 0) { bad = 1; break; }                                  /* symmetric pattern */
            if (w && memcmp(&w[t], &wk, 8) != 0) { bad = 1; break; }        /* w_ij == w_ji bitwise */
        }
    }
    if (bad) return ORC_EGRAPH;
    /* connectivity by BFS ("we assume that the graph G is connected") */
    int64_t *queue = malloc(sizeof(int64_t) * (size_t)n);
    uint8_t *seen = calloc((size_t)n, 1);
    int64_t head = 0, tail = 0;
    queue[tail++] = 0;
    seen[0] = 1;
    while (head < tail) {
        int64_t i = queue[head++];
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++)
            if (!seen[col[k]]) { seen[col[k]] = 1; queue[tail++] = col[k]; }
    }
    free(queue);
    free(seen);
    return tail == n ? ORC_OK : ORC_EDISCONNECTED;
}

/* ======================================================================== */
/* O-S1 random vertex ordering (O-R31)                           */
/* ======================================================================== */

static const uint64_t *g_sort_keys;
static int cmp_by_key(const void *a, const void *b) {
    uint64_t ka = g_sort_keys[*(const int64_t *)a], kb = g_sort_keys[*(const int64_t *)b];
    return (ka > kb) - (ka < kb);
}

/* perm[i] = rank of mix64(i XOR salt_1) in ascending order (keys distinct). */
void orc_random_perm(int64_t n, uint64_t seed, int64_t *perm) {
    uint64_t s1 = orc_salt(seed, 1);
    uint64_t *keys = malloc(sizeof(uint64_t) * (size_t)n);
    int64_t *order = malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; i++) { keys[i] = orc_mix64((uint64_t)i ^ s1); order[i] = i; }
    g_sort_keys = keys;
    qsort(order, (size_t)n, sizeof(int64_t), cmp_by_key);
    for (int64_t r = 0; r < n; r++) perm[order[r]] = r;
    free(keys);
    free(order);
}

/* d_i = CanonSum_j w_ij  (P:72-75 row sums; O-R23, O-R37). e_max from max w, K = nnz. */
void orc_row_sums(int64_t n, const int64_t *row_ptr, const double *w, double *d) {
    int64_t nnz = row_ptr[n];
    int32_t e_max = orc_ilogb(max_abs(w, nnz)) + 1;
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++)
        d[i] = orc_canon_sum(w + row_ptr[i], row_ptr[i + 1] - row_ptr[i], e_max, nnz);
}

/* ======================================================================== */
/* H1: y = L x = d o x - A x  (the (+,x) instance of P:351)       */
/* ======================================================================== */

void orc_spmv(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
              const double *d, const double *x, double *y) {
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) s += w[k] * x[col[k]];
        y[i] = d[i] * x[i] - s;
    }
}

/* ======================================================================== */
/* O-S2 elimination: Alg. 2, oplus_elim/otimes_elim P:403-421   */
/* ======================================================================== */

/* cand_i = deg_i <= max_degree (O-R19).  z_i = candidate of smallest
 * (hash, index) over the closed neighbourhood {i} u N(i) -- the diagonal of L
 * puts i in its own neighbourhood.  F = {i : cand_i and z_i = i}.
 * hash(j) = mix64(j XOR salt_2) (O-R17), or hash_override[j] in tests.
 * Non-candidates are skipped instead of mapped to the infinity sentinel
 * (O-R18).  Returns |F|. */
uint64_t orc_elim_hash(uint64_t j, uint64_t seed) { return orc_mix64(j ^ orc_salt(seed, 2)); }

int64_t orc_elim_select(int64_t n, const int64_t *row_ptr, const int32_t *col,
                        int32_t max_degree, uint64_t seed, const uint64_t *hash_override,
                        uint8_t *F) {
    int64_t nF = 0;
    #pragma omp parallel for reduction(+:nF) schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; i++) {
        F[i] = 0;
        if (row_ptr[i + 1] - row_ptr[i] > max_degree) continue;      /* not a candidate */
        /* z_i = oplus over the closed neighbourhood of candidates */
        int64_t zj = i;
        uint64_t zh = hash_override ? hash_override[i] : orc_elim_hash((uint64_t)i, seed);
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
            int64_t j = col[k];
            if (row_ptr[j + 1] - row_ptr[j] > max_degree) continue;  /* otimes -> empty */
            uint64_t hj = hash_override ? hash_override[j] : orc_elim_hash((uint64_t)j, seed);
            if (hj < zh || (hj == zh && j < zj)) { zh = hj; zj = j; }
        }
        if (zj == i) { F[i] = 1; nF++; }                              /* line 430 */
    }
    return nF;
}

/* coarse (C) numbering: order-preserving compaction (O-R22); F -> -1-slot */
static int64_t make_fmap(int64_t n, const uint8_t *F, int32_t *fmap) {
    int64_t nc = 0, nf = 0;
    for (int64_t i = 0; i < n; i++) {
        if (F[i]) fmap[i] = (int32_t)(-1 - nf++);
        else fmap[i] = (int32_t)nc++;
    }
    return nc;
}

typedef struct { int32_t c; int32_t pad; double v; } term_t;
static int cmp_term(const void *a, const void *b) {
    int32_t x = ((const term_t *)a)->c, y = ((const term_t *)b)->c;
    return (x > y) - (x < y);
}

/* gather the Schur terms of C-row i (coarse ids) into buf; returns count */
static int64_t schur_row_terms(const int64_t *row_ptr, const int32_t *col, const double *w,
                               const double *d, const uint8_t *F, const int32_t *fmap,
                               int64_t i, term_t *buf) {
    int64_t cnt = 0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
        int32_t j = col[k];
        if (!F[j]) {                       /* L_CC entry: w_ab */
            if (buf) { buf[cnt].c = fmap[j]; buf[cnt].v = w[k]; }
            cnt++;
        } else {                           /* fill through f = j: fl(fl(w_fa*w_fb)/d_f), O-R25 */
            int64_t f = j;
            int64_t kfa = find_in_row(row_ptr, col, f, (int32_t)i);
            double wfa = w[kfa];
            for (int64_t q = row_ptr[f]; q < row_ptr[f + 1]; q++) {
                int32_t b = col[q];
                if (b == i) continue;
                if (buf) {
                    double prod = wfa * w[q];
                    buf[cnt].c = fmap[b];
                    buf[cnt].v = prod / d[f];
                }
                cnt++;
            }
        }
    }
    return cnt;
}

int64_t orc_schur_count(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint8_t *F) {
    /* upper bound on terms per C row, used only for scratch sizing */
    int64_t mx = 0;
    for (int64_t i = 0; i < n; i++) {
        if (F[i]) continue;
        int64_t c = 0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
            int32_t j = col[k];
            c += F[j] ? (row_ptr[j + 1] - row_ptr[j] - 1) : 1;
        }
        if (c > mx) mx = c;
    }
    return mx;
}

/* Schur complement L_{l+1} = L_CC - L_FC^T L_FF^-1 L_FC, entry
 * by entry: W'[a,b] = CanonSum({w_ab} u {fl(fl(w_fa w_fb)/d_f) : f in F,
 * f~a, f~b}) for a != b (O-S2, O-R25); d'_a = CanonSum_b W'[a,b] (O-R24).
 * Canonical-sum instance: e_max = ilogb(max w)+1, K = 4*nnz (every fill term
 * <= min(w_fa, w_fb) since d_f >= w_fa + w_fb; at most 3 fill terms per
 * stored entry because deg_f <= 4).  Returns nnz of the new level; nrow_ptr
 * must hold nc+1, ncol/nw the new nnz (call with ncol=NULL to count). */
int64_t orc_schur(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                  const double *d, const uint8_t *F, int32_t *fmap,
                  int64_t *nrow_ptr, int32_t *ncol, double *nw, double *nd) {
    int64_t nnz = row_ptr[n];
    int64_t nc = make_fmap(n, F, fmap);
    int32_t e_max = orc_ilogb(max_abs(w, nnz)) + 1;
    int64_t K = 4 * nnz;
    int64_t mx = orc_schur_count(n, row_ptr, col, F);
    int64_t *cid = malloc(sizeof(int64_t) * (size_t)(nc + 1));       /* C row a -> fine vertex */
    for (int64_t i = 0; i < n; i++) if (!F[i]) cid[fmap[i]] = i;
    int64_t *rl = calloc((size_t)(nc + 1), sizeof(int64_t));          /* row lengths of the new level */
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1 && !ncol) break;
        #pragma omp parallel
        {
            term_t *buf = malloc(sizeof(term_t) * (size_t)(mx + 1));
            double *tv = malloc(sizeof(double) * (size_t)(mx + 1));
            #pragma omp for schedule(dynamic, 256)
            for (int64_t a = 0; a < nc; a++) {
                int64_t i = cid[a];
                int64_t cnt = schur_row_terms(row_ptr, col, w, d, F, fmap, i, buf);
                qsort(buf, (size_t)cnt, sizeof(term_t), cmp_term);
                int64_t out = pass ? nrow_ptr[a] : 0, s = 0;
                while (s < cnt) {
                    int64_t e = s;
                    while (e < cnt && buf[e].c == buf[s].c) { tv[e - s] = buf[e].v; e++; }
                    if (pass) {
                        ncol[out] = buf[s].c;
                        nw[out] = orc_canon_sum(tv, e - s, e_max, K);
                    }
                    out++;
                    s = e;
                }
                if (!pass) rl[a] = out;
            }
            free(buf);
            free(tv);
        }
        if (pass == 0 && nrow_ptr) {
            nrow_ptr[0] = 0;
            for (int64_t a = 0; a < nc; a++) nrow_ptr[a + 1] = nrow_ptr[a] + rl[a];
        }
    }
    int64_t tot = 0;
    for (int64_t a = 0; a < nc; a++) tot += rl[a];
    free(cid);
    free(rl);
    if (ncol && nd) orc_row_sums(nc, nrow_ptr, nw, nd);
    return tot;
}

/* ======================================================================== */
/* O-S3 strength of connection                                  */
/* ======================================================================== */

/* uniform [0,1) from a 64-bit word: (u >> 11) * 2^-53 */
static double u01(uint64_t u) { return (double)(u >> 11) * 0x1.0p-53; }

/* X0[i,k] = 2*((U(l,i,k) >> 11) 2^-53) - 1,
 * U(l,i,k) = mix64(mix64(salt_3 XOR (2l + attempt)) XOR (4i + k))   (O-R7, O-R33) */
static void init_test_vectors(int64_t n, uint64_t seed, int32_t level, int32_t attempt, double *X) {
    uint64_t base = orc_mix64(orc_salt(seed, 3) ^ (uint64_t)(2 * level + attempt));
    for (int64_t i = 0; i < n; i++)
        for (int k = 0; k < 4; k++)
            X[4 * i + k] = 2.0 * u01(orc_mix64(base ^ (uint64_t)(4 * i + k))) - 1.0;
}

/* `sweeps` damped-Jacobi sweeps on L x = 0 for each of the 4 columns
 * ("smooth on Ly = 0"; "three iterations of Jacobi smoothing"):
 *   s_ik = CanonSum_j fl(w_ij x_jk)
 *   x_ik <- fl(x_ik - fl(omega * fl(fl(fl(d_i x_ik) - s_ik) / d_i)))
 * One canonical-sum instance per sweep: e_max = ilogb(max w) + ilogb(max|X|) + 2,
 * K = nnz (O-S3).  Synchronous (Jacobi): the new X is built from the old. */
void orc_test_vectors_from(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                           const double *d, int32_t sweeps, double omega, double *X) {
    int64_t nnz = row_ptr[n];
    double *Xn = malloc(sizeof(double) * 4 * (size_t)n);
    int64_t maxdeg = 0;
    for (int64_t i = 0; i < n; i++)
        if (row_ptr[i + 1] - row_ptr[i] > maxdeg) maxdeg = row_ptr[i + 1] - row_ptr[i];
    double *t = malloc(sizeof(double) * (size_t)(maxdeg + 1));
    int32_t ew = orc_ilogb(max_abs(w, nnz));
    free(t);
    for (int sw = 0; sw < sweeps; sw++) {
        double mx = max_abs(X, 4 * n);
        int32_t e_max = (mx > 0.0) ? ew + orc_ilogb(mx) + 2 : ew + 1;
        #pragma omp parallel
        {
            double *tt = malloc(sizeof(double) * (size_t)(maxdeg + 1));
            #pragma omp for schedule(dynamic, 1024)
            for (int64_t i = 0; i < n; i++) {
                for (int k = 0; k < 4; k++) {
                    int64_t c = 0;
                    for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++) tt[c++] = w[q] * X[4 * (int64_t)col[q] + k];
                    double s = orc_canon_sum(tt, c, e_max, nnz);
                    double xi = X[4 * i + k];
                    double dx = d[i] * xi;
                    double rr = dx - s;
                    double qq = rr / d[i];
                    double om = omega * qq;
                    Xn[4 * i + k] = xi - om;
                }
            }
            free(tt);
        }
        memcpy(X, Xn, sizeof(double) * 4 * (size_t)n);
    }
    free(Xn);
}

void orc_test_vectors(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                      const double *d, uint64_t seed, int32_t level, int32_t attempt,
                      int32_t sweeps, double omega, double *X) {
    init_test_vectors(n, seed, level, attempt, X);
    orc_test_vectors_from(n, row_ptr, col, w, d, sweeps, omega, X);
}

/* C_ij on the stored pattern, 0 diagonal by construction:
 *   g  = ((x_i0 x_j0 + x_i1 x_j1) + x_i2 x_j2) + x_i3 x_j3   (left to right)
 *   n_i = same expression over x_ik^2
 *   power 1 (O-R5, LAMG affinity): C = fl(fl(g g) / fl(n_i n_j))
 *   power 2 (literal P:564-565):   C = fl(fl(g g) / fl(fl(n_i n_i) fl(n_j n_j)))
 * C = 0 when the denominator is 0. */
static double dot4(const double *a, const double *b) {
    double s = a[0] * b[0];
    s = s + a[1] * b[1];
    s = s + a[2] * b[2];
    s = s + a[3] * b[3];
    return s;
}

void orc_affinity(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *X,
                  int32_t power, double *C) {
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++) {
        double ni = dot4(X + 4 * i, X + 4 * i);
        for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++) {
            int64_t j = col[q];
            double nj = dot4(X + 4 * j, X + 4 * j);
            double g = dot4(X + 4 * i, X + 4 * j);
            double num = g * g;
            double den;
            if (power == 2) { double a = ni * ni; double b = nj * nj; den = a * b; }
            else den = ni * nj;
            C[q] = (den > 0.0) ? num / den : 0.0;
        }
    }
}

/* S_ij = C_ij / max(max_s C_is, max_s C_sj); entry dropped (stored
 * as 0) when that maximum is 0 (O-R16).  C is symmetric, so the column max of
 * j is the row max of j. */
void orc_normalize_strength(int64_t n, const int64_t *row_ptr, const int32_t *col,
                            const double *C, double *S) {
    double *M = malloc(sizeof(double) * (size_t)n);
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++) {
        double m = 0.0;
        for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++) if (C[q] > m) m = C[q];
        M[i] = m;
    }
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++)
        for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++) {
            double den = M[i] > M[col[q]] ? M[i] : M[col[q]];
            S[q] = den > 0.0 ? C[q] / den : 0.0;
        }
    free(M);
}

/* ======================================================================== */
/* O-S4 vote-based aggregation: Alg. 3                 */
/* ======================================================================== */

/* status_i = (Undecided, i), votes = 0.  Round t = 1..rounds,
 * filter 2^-t (O-R13).  For every Undecided i (O-R9):
 *   d_i = oplus_agg over j in N(i) with S_ij >= 2^-t and S_ij != 0 of
 *         (state_j, j, S_ij) under the total order (rank(state), S, -j)
 *         (P:597-612 with the index tie-break of O-R10); Decided neighbours
 *         never win against a Seed/Undecided one and are skipped (O-R12).
 *   Seed  -> status'_i = (Decided, j)
 *   Undec -> votes_j += 1
 * then every i with status'_i = (Undecided, i) and votes_i >= threshold
 * becomes (Seed, i) (">= 8" per P:619, O-R8).  Synchronous
 * rounds (O-R11).  Afterwards roots = Seed u Undecided, numbered by ascending
 * vertex id (O-R14, O-R15); agg_i = id(root(i)).  Returns m. */
int64_t orc_aggregate(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *S,
                      int32_t rounds, int32_t threshold, int32_t *agg,
                      int8_t *state_out, int32_t *votes_out) {
    int8_t *st = malloc((size_t)n), *nst = malloc((size_t)n);
    int32_t *idx = malloc(sizeof(int32_t) * (size_t)n), *nidx = malloc(sizeof(int32_t) * (size_t)n);
    int32_t *votes = calloc((size_t)n, sizeof(int32_t));
    for (int64_t i = 0; i < n; i++) { st[i] = ST_UNDECIDED; idx[i] = (int32_t)i; }
    for (int32_t t = 1; t <= rounds; t++) {
        double filt = ldexp(1.0, -t);
        memcpy(nst, st, (size_t)n);
        memcpy(nidx, idx, sizeof(int32_t) * (size_t)n);
        #pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t i = 0; i < n; i++) {
            if (st[i] != ST_UNDECIDED) continue;
            int br = -1; double bs = 0.0; int64_t bj = -1;
            for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++) {
                double s = S[q];
                if (s == 0.0 || s < filt) continue;
                int64_t j = col[q];
                int r = st[j];
                if (r == ST_DECIDED) continue;
                if (r > br || (r == br && (s > bs || (s == bs && j < bj)))) { br = r; bs = s; bj = j; }
            }
            if (bj < 0) continue;
            if (br == ST_SEED) { nst[i] = ST_DECIDED; nidx[i] = (int32_t)bj; }
            else {
                #pragma omp atomic
                votes[bj] += 1;                                 /* integer: exact in any order */
            }
        }
        for (int64_t i = 0; i < n; i++)
            if (nst[i] == ST_UNDECIDED && votes[i] >= threshold) nst[i] = ST_SEED;
        memcpy(st, nst, (size_t)n);
        memcpy(idx, nidx, sizeof(int32_t) * (size_t)n);
    }
    int32_t *id = malloc(sizeof(int32_t) * (size_t)n);
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++) id[i] = (st[i] != ST_DECIDED) ? (int32_t)m++ : -1;
    for (int64_t i = 0; i < n; i++) agg[i] = (st[i] != ST_DECIDED) ? id[i] : id[idx[i]];
    if (state_out) memcpy(state_out, st, (size_t)n);
    if (votes_out) memcpy(votes_out, votes, sizeof(int32_t) * (size_t)n);
    free(st); free(nst); free(idx); free(nidx); free(votes); free(id);
    return m;
}

/* ======================================================================== */
/* O-S5 Galerkin coarse operator L_{l+1} = R L P                */
/* ======================================================================== */

/* W_c[a,b] = CanonSum{ w_ij : agg_i = a, agg_j = b } for a != b; the
 * within-aggregate entries cancel against the diagonal (R L P of a Laplacian
 * is a Laplacian); d_c = CanonSum of the coarse row (O-R24).  Instance:
 * e_max = ilogb(max w)+1, K = nnz(fine).  Returns coarse nnz; with
 * ccol == NULL only counts. */
static int64_t galerkin_impl(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                             const int32_t *agg, int64_t m, int64_t *crow_ptr, int32_t *ccol,
                             double *cw, double *cd) {
    int64_t nnz = row_ptr[n];
    /* bucket fine entries by coarse row a (the order inside a bucket is
     * irrelevant: the row is sorted by coarse column and every entry is a
     * CanonSum, which does not depend on the order of its terms) */
    int64_t *cnt = calloc((size_t)(m + 1), sizeof(int64_t));
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++)
        for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++)
            if (agg[i] != agg[col[q]]) {
                #pragma omp atomic
                cnt[agg[i] + 1]++;
            }
    for (int64_t a = 0; a < m; a++) cnt[a + 1] += cnt[a];
    int64_t tot = cnt[m];
    term_t *buf = malloc(sizeof(term_t) * (size_t)(tot + 1));
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(m + 1));
    memcpy(fill, cnt, sizeof(int64_t) * (size_t)(m + 1));
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++)
        for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++) {
            int32_t a = agg[i], b = agg[col[q]];
            if (a != b) {
                int64_t pos;
                #pragma omp atomic capture
                pos = fill[a]++;
                buf[pos].c = b;
                buf[pos].v = w[q];
            }
        }
    int32_t e_max = orc_ilogb(max_abs(w, nnz)) + 1;
    int64_t mxrow = 0;
    for (int64_t a = 0; a < m; a++) if (cnt[a + 1] - cnt[a] > mxrow) mxrow = cnt[a + 1] - cnt[a];
    int64_t *rl = calloc((size_t)(m + 1), sizeof(int64_t));
    #pragma omp parallel for schedule(dynamic, 256)
    for (int64_t a = 0; a < m; a++) {                              /* sort each coarse row, count distinct */
        term_t *r = buf + cnt[a];
        int64_t len = cnt[a + 1] - cnt[a];
        qsort(r, (size_t)len, sizeof(term_t), cmp_term);
        int64_t u = 0;
        for (int64_t e = 0; e < len; e++) if (e == 0 || r[e].c != r[e - 1].c) u++;
        rl[a] = u;
    }
    int64_t out = 0;
    for (int64_t a = 0; a < m; a++) out += rl[a];
    if (crow_ptr) {
        crow_ptr[0] = 0;
        for (int64_t a = 0; a < m; a++) crow_ptr[a + 1] = crow_ptr[a] + rl[a];
    }
    if (ccol) {
        #pragma omp parallel
        {
            double *tv = malloc(sizeof(double) * (size_t)(mxrow + 1));
            #pragma omp for schedule(dynamic, 256)
            for (int64_t a = 0; a < m; a++) {
                term_t *r = buf + cnt[a];
                int64_t len = cnt[a + 1] - cnt[a], o = crow_ptr[a], s = 0;
                while (s < len) {
                    int64_t e = s;
                    while (e < len && r[e].c == r[s].c) { tv[e - s] = r[e].v; e++; }
                    ccol[o] = r[s].c;
                    cw[o] = orc_canon_sum(tv, e - s, e_max, nnz);
                    o++;
                    s = e;
                }
            }
            free(tv);
        }
    }
    free(cnt); free(buf); free(fill); free(rl);
    if (ccol && cd) orc_row_sums(m, crow_ptr, cw, cd);
    return out;
}

int64_t orc_galerkin_count(int64_t n, const int64_t *row_ptr, const int32_t *col,
                           const int32_t *agg, int64_t m) {
    double *w = malloc(sizeof(double) * (size_t)(row_ptr[n] + 1));
    for (int64_t k = 0; k < row_ptr[n]; k++) w[k] = 1.0;
    int64_t r = galerkin_impl(n, row_ptr, col, w, agg, m, NULL, NULL, NULL, NULL);
    free(w);
    return r;
}

int64_t orc_galerkin(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                     const int32_t *agg, int64_t m, int64_t *crow_ptr, int32_t *ccol,
                     double *cw, double *cd) {
    return galerkin_impl(n, row_ptr, col, w, agg, m, crow_ptr, ccol, cw, cd);
}

/* ======================================================================== */
/* O-S6 lambda-hat: 10 Lanczos steps on B = D^-1/2 L D^-1/2 (O-R3)    */
/* ======================================================================== */

/* largest eigenvalue of the symmetric tridiagonal (alpha[0..k-1], beta[0..k-2])
 * by bisection on the Sturm count. */
double orc_tridiag_max_eig(int32_t k, const double *alpha, const double *beta) {
    if (k <= 0) return 0.0;
    double lo = alpha[0], hi = alpha[0];
    for (int i = 0; i < k; i++) {
        double r = 0.0;
        if (i > 0) r += fabs(beta[i - 1]);
        if (i < k - 1) r += fabs(beta[i]);
        if (alpha[i] - r < lo) lo = alpha[i] - r;
        if (alpha[i] + r > hi) hi = alpha[i] + r;
    }
    for (int it = 0; it < 200; it++) {
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        /* number of eigenvalues > mid = k - #(eigenvalues <= mid) */
        int cnt_le = 0;
        double q = 1.0;
        for (int i = 0; i < k; i++) {
            double b2 = (i > 0) ? beta[i - 1] * beta[i - 1] : 0.0;
            q = (alpha[i] - mid) - ((i > 0) ? b2 / q : 0.0);
            if (q == 0.0) q = -1e-300;
            if (q < 0.0) cnt_le++;
        }
        if (cnt_le == k) hi = mid;  /* all eigenvalues below mid */
        else lo = mid;
    }
    return hi;
}

/* Lanczos start vector before normalisation (O-S6, reading R-U' of DESIGN.md):
 *   v_i = 2 U'(l,i) - 1,  U'(l,i) = u01(mix64(mix64(salt_4 XOR 2l) XOR i)). */
void orc_lanczos_start(int64_t n, uint64_t seed, int32_t level, double *v) {
    uint64_t base = orc_mix64(orc_salt(seed, 4) ^ (uint64_t)(2 * level));
    for (int64_t i = 0; i < n; i++) v[i] = 2.0 * u01(orc_mix64(base ^ (uint64_t)i)) - 1.0;
}

/* exponent of an exact bound: every |t| < 2^(e(m)+1) for |t| <= m (m finite);
 * m = 0 -> a sentinel far below any term (all terms are then exactly 0). */
static int32_t ebound(double m) { return m > 0.0 ? orc_ilogb(m) : -1000; }

/* 10 Lanczos steps on B = D^-1/2 L D^-1/2 (O-R3, O-S6), no
 * reorthogonalisation, stop when beta_j <= 1e-14 |alpha_j|.  Every sum is a
 * CanonSum (O-S11; reading R-lambda of DESIGN.md: O-R23 extended to lambda-hat,
 * so lambda-hat is a deterministic function of the level, bit-identical on
 * the GPU), with these exact exponent bounds (|v_i| < 2 always: v = y / ||y||):
 *   ||v0||^2 : terms v_i^2 <= 1                          e_max = 1,  K = n
 *   (L u)_i  : s_i = CanonSum_j fl(w_ij u_j), |u| < 2 max(rs)
 *                                    e_max = e(max w) + e(max rs) + 3,  K = nnz
 *   alpha    : terms fl(y_i v_i), |.| < 2^(e(max|y|)+1) * 2 e_max = e(max|y|) + 2, K = n
 *   beta^2   : y' = fl(y - fl(alpha v)), |y'| < 2^(max(e(max|y|)+1, e(alpha)+2)+1)
 *              (+1 for the rounding)   e_max = 2 (max(e(max|y|)+1, e(alpha)+2) + 2), K = n
 * Each scalar step is one IEEE rounding:
 *   rs_i = fl(1 / fl(sqrt(d_i))), u_i = fl(rs_i v_i),
 *   y_i = fl(fl(rs_i fl(fl(d_i u_i) - s_i)) - fl(beta_prev vp_i)),
 *   v_i = fl(y_i / beta). */
double orc_lanczos(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                   const double *d, uint64_t seed, int32_t level, int32_t steps,
                   double *alpha_out, double *beta_out, int32_t *k_out) {
    int64_t nnz = row_ptr[n];
    double *v = malloc(sizeof(double) * (size_t)n), *vp = calloc((size_t)n, sizeof(double));
    double *u = malloc(sizeof(double) * (size_t)n), *y = malloc(sizeof(double) * (size_t)n);
    double *rs = malloc(sizeof(double) * (size_t)n), *t = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int64_t maxdeg = 0;
    for (int64_t i = 0; i < n; i++)
        if (row_ptr[i + 1] - row_ptr[i] > maxdeg) maxdeg = row_ptr[i + 1] - row_ptr[i];
    double alpha[64], beta[64];
    orc_lanczos_start(n, seed, level, v);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) rs[i] = 1.0 / sqrt(d[i]);
    double nv = sqrt(canon_dot(v, v, n, 1, n));
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) v[i] = v[i] / nv;
    const int32_t e_spmv = ebound(max_abs(w, nnz)) + ebound(max_abs(rs, n)) + 3;
    int32_t k = 0;
    double bprev = 0.0;
    for (int32_t j = 0; j < steps; j++) {
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) u[i] = rs[i] * v[i];
        #pragma omp parallel
        {
            double *tr = malloc(sizeof(double) * (size_t)(maxdeg + 1));
            #pragma omp for schedule(dynamic, 1024)
            for (int64_t i = 0; i < n; i++) {                        /* y = D^-1/2 L D^-1/2 v - beta vp */
                int64_t c = 0;
                for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++) tr[c++] = w[q] * u[col[q]];
                double si = orc_canon_sum(tr, c, e_spmv, nnz);
                double li = d[i] * u[i] - si;
                double bv = bprev * vp[i];
                y[i] = rs[i] * li - bv;
            }
            free(tr);
        }
        int32_t ey = ebound(max_abs(y, n));
        double a = canon_dot(y, v, n, ey + 2, n);
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) { double av = a * v[i]; y[i] = y[i] - av; }
        int32_t ea = ebound(fabs(a));
        int32_t eb = 2 * ((ey + 1 > ea + 2 ? ey + 1 : ea + 2) + 2);
        double b = sqrt(canon_dot(y, y, n, eb, n));
        alpha[k] = a;
        beta[k] = b;
        k++;
        if (b <= 1e-14 * fabs(a)) break;
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) { vp[i] = v[i]; v[i] = y[i] / b; }
        bprev = b;
    }
    double lam = orc_tridiag_max_eig(k, alpha, beta);
    if (alpha_out) memcpy(alpha_out, alpha, sizeof(double) * (size_t)k);
    if (beta_out) memcpy(beta_out, beta, sizeof(double) * (size_t)k);
    if (k_out) *k_out = k;
    free(v); free(vp); free(u); free(y); free(rs); free(t);
    return lam;
}

/* ======================================================================== */
/* O-S10 coarsest level: dense L^+ (O-R26)               */
/* ======================================================================== */

/* Ground the last vertex, invert the (n-1)x(n-1) SPD block by Cholesky, and
 * project: L^+ = (I - J/n) [[A^-1, 0], [0, 0]] (I - J/n)  (equals the
 * Moore-Penrose inverse for a connected graph). */
int orc_coarse_pinv(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                    const double *d, double *pinv) {
    memset(pinv, 0, sizeof(double) * (size_t)(n * n));
    if (n <= 1) return ORC_OK;
    int64_t g = n - 1;
    double *A = calloc((size_t)(g * g), sizeof(double));
    for (int64_t i = 0; i < g; i++) {
        A[i * g + i] = d[i];
        for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++)
            if (col[q] < g) A[i * g + col[q]] = -w[q];
    }
    /* Cholesky A = R^T R (upper R stored in A) */
    for (int64_t j = 0; j < g; j++) {
        double s = A[j * g + j];
        for (int64_t k = 0; k < j; k++) s -= A[k * g + j] * A[k * g + j];
        if (!(s > 0.0)) { free(A); return ORC_EDISCONNECTED; }
        double r = sqrt(s);
        A[j * g + j] = r;
        for (int64_t i = j + 1; i < g; i++) {
            double t = A[j * g + i];
            for (int64_t k = 0; k < j; k++) t -= A[k * g + j] * A[k * g + i];
            A[j * g + i] = t / r;
        }
    }
    /* Ainv = R^-1 R^-T, column by column */
    double *G = calloc((size_t)(n * n), sizeof(double));
    double *e = malloc(sizeof(double) * (size_t)g);
    for (int64_t c = 0; c < g; c++) {
        for (int64_t i = 0; i < g; i++) e[i] = (i == c) ? 1.0 : 0.0;
        for (int64_t i = 0; i < g; i++) {          /* R^T y = e */
            double t = e[i];
            for (int64_t k = 0; k < i; k++) t -= A[k * g + i] * e[k];
            e[i] = t / A[i * g + i];
        }
        for (int64_t i = g - 1; i >= 0; i--) {     /* R x = y */
            double t = e[i];
            for (int64_t k = i + 1; k < g; k++) t -= A[i * g + k] * e[k];
            e[i] = t / A[i * g + i];
        }
        for (int64_t i = 0; i < g; i++) G[i * n + c] = e[i];
    }
    /* P G P with P = I - J/n */
    double *rm = calloc((size_t)n, sizeof(double)), *cm = calloc((size_t)n, sizeof(double));
    double tot = 0.0;
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < n; j++) { rm[i] += G[i * n + j]; cm[j] += G[i * n + j]; tot += G[i * n + j]; }
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < n; j++)
            pinv[i * n + j] = G[i * n + j] - rm[i] / n - cm[j] / n + tot / ((double)n * n);
    free(A); free(G); free(e); free(rm); free(cm);
    return ORC_OK;
}

/* ======================================================================== */
/* O-S6 Chebyshev smoother in D^-1 L on [lo*lam, hi*lam]    */
/* ======================================================================== */

/* Standard Chebyshev acceleration with D^-1 as preconditioner (O-R1, O-R4):
 *   theta=(b+a)/2, delta=(b-a)/2, sigma=theta/delta, rho_old=1/sigma
 *   r = b - L x ; dv = D^-1 r / theta ; x += dv
 *   for k=1..K-1: r = b - L x ; rho = 1/(2 sigma - rho_old)
 *                 dv = rho rho_old dv + (2 rho/delta) D^-1 r ; x += dv */
void orc_chebyshev(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                   const double *d, double lambda, double lo, double hi, int32_t degree,
                   const double *b, double *x, int32_t x_is_zero) {
    double a = lo * lambda, bb = hi * lambda;
    double theta = 0.5 * (bb + a), delta = 0.5 * (bb - a);
    double sigma = theta / delta, rho_old = 1.0 / sigma;
    double *r = malloc(sizeof(double) * (size_t)n), *dv = malloc(sizeof(double) * (size_t)n);
    if (x_is_zero) { for (int64_t i = 0; i < n; i++) { x[i] = 0.0; r[i] = b[i]; } }
    else {
        orc_spmv(n, row_ptr, col, w, d, x, r);
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) r[i] = b[i] - r[i];
    }
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) { dv[i] = r[i] / d[i] / theta; x[i] += dv[i]; }
    for (int32_t k = 1; k < degree; k++) {
        orc_spmv(n, row_ptr, col, w, d, x, r);
        double rho = 1.0 / (2.0 * sigma - rho_old);
        double c1 = rho * rho_old, c2 = 2.0 * rho / delta;
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            r[i] = b[i] - r[i];
            dv[i] = c1 * dv[i] + c2 * (r[i] / d[i]);
            x[i] += dv[i];
        }
        rho_old = rho;
    }
    free(r); free(dv);
}

/* ======================================================================== */
/* O-S9 hierarchy setup (O-R21, O-R27, O-R28)                */
/* ======================================================================== */

static void level_free(orc_level *L) {
    free(L->row_ptr); free(L->col); free(L->w); free(L->d);
    free(L->agg); free(L->S); free(L->fmap); free(L->pinv);
    free(L->mem_ptr); free(L->members); free(L->ct_ptr); free(L->ct_q); free(L->ct_f);
    memset(L, 0, sizeof(*L));
}

void orc_free(orc_hier *h) {
    if (!h) return;
    for (int l = 0; l < h->nlev; l++) level_free(&h->lev[l]);
    free(h->perm);
    free(h);
}

/* O-S1: the relabelled level 0, Pi L Pi^T: new row r = old row
 * inv[r], columns perm[col] in ascending order; w = NULL means unit weights.
 * out_row_ptr[n+1], out_col/out_w[nnz]. */
void orc_relabel(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w, const int64_t *perm,
                 int64_t *out_row_ptr, int32_t *out_col, double *out_w) {
    int64_t *inv = malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; i++) inv[perm[i]] = i;
    out_row_ptr[0] = 0;
    for (int64_t r = 0; r < n; r++) out_row_ptr[r + 1] = out_row_ptr[r] + (row_ptr[inv[r] + 1] - row_ptr[inv[r]]);
    int64_t mx = 0;
    for (int64_t i = 0; i < n; i++) if (row_ptr[i + 1] - row_ptr[i] > mx) mx = row_ptr[i + 1] - row_ptr[i];
    #pragma omp parallel
    {
        term_t *tmp = malloc(sizeof(term_t) * (size_t)(mx + 1));
        #pragma omp for schedule(dynamic, 1024)
        for (int64_t r = 0; r < n; r++) {
            int64_t i = inv[r], len = row_ptr[i + 1] - row_ptr[i];
            for (int64_t k = 0; k < len; k++) {
                tmp[k].c = (int32_t)perm[col[row_ptr[i] + k]];
                tmp[k].v = w ? w[row_ptr[i] + k] : 1.0;
            }
            qsort(tmp, (size_t)len, sizeof(term_t), cmp_term);
            for (int64_t k = 0; k < len; k++) { out_col[out_row_ptr[r] + k] = tmp[k].c; out_w[out_row_ptr[r] + k] = tmp[k].v; }
        }
        free(tmp);
    }
    free(inv);
}

int orc_setup(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
              const orc_params *pp, orc_hier **out) {
    *out = NULL;
    orc_params p;
    if (pp) p = *pp; else orc_params_default(&p);
    int rc = orc_validate(n, row_ptr, col, w);
    if (rc != ORC_OK) return rc;
    orc_hier *h = calloc(1, sizeof(orc_hier));
    h->p = p;
    h->n0 = n;
    h->perm = malloc(sizeof(int64_t) * (size_t)n);
    int64_t nnz = row_ptr[n];

    /* O-S1: level 0 = Pi_rand L Pi_rand^T (input only) */
    if (p.random_order) orc_random_perm(n, p.seed, h->perm);
    else for (int64_t i = 0; i < n; i++) h->perm[i] = i;
    orc_level *L0 = &h->lev[0];
    L0->n = n; L0->nnz = nnz;
    L0->row_ptr = calloc((size_t)(n + 1), sizeof(int64_t));
    L0->col = malloc(sizeof(int32_t) * (size_t)(nnz + 1));
    L0->w = malloc(sizeof(double) * (size_t)(nnz + 1));
    L0->d = malloc(sizeof(double) * (size_t)n);
    orc_relabel(n, row_ptr, col, w, h->perm, L0->row_ptr, L0->col, L0->w);
    orc_row_sums(n, L0->row_ptr, L0->w, L0->d);

    int elim_run = 0;   /* elimination levels in a row just above (O-R21; P:485-486 elim_rounds) */
    int l = 0;
    for (;;) {
        orc_level *L = &h->lev[l];
        int64_t nl = L->n, z = L->nnz;
        if (nl + z <= p.coarse_nnz || l == p.max_levels - 1 || l == 63) {      /* O-R27 */
            L->kind = ORC_COARSEST;
            break;
        }
        if (p.elim_enable && elim_run < p.elim_rounds) {                      /* O-R21 */
            uint8_t *F = malloc((size_t)nl);
            int64_t nF = orc_elim_select(nl, L->row_ptr, L->col, p.elim_max_degree, p.seed, NULL, F);
            if (20 * nF > nl) {                                                /* O-R20 */
                orc_level *N = &h->lev[l + 1];
                L->kind = ORC_ELIM;
                L->nF = nF;
                L->fmap = malloc(sizeof(int32_t) * (size_t)nl);
                int64_t nc = nl - nF;
                N->n = nc;
                N->row_ptr = malloc(sizeof(int64_t) * (size_t)(nc + 1));
                int64_t cn = orc_schur(nl, L->row_ptr, L->col, L->w, L->d, F, L->fmap, N->row_ptr, NULL, NULL, NULL);
                N->nnz = cn;
                N->col = malloc(sizeof(int32_t) * (size_t)(cn + 1));
                N->w = malloc(sizeof(double) * (size_t)(cn + 1));
                N->d = malloc(sizeof(double) * (size_t)(nc + 1));
                orc_schur(nl, L->row_ptr, L->col, L->w, L->d, F, L->fmap, N->row_ptr, N->col, N->w, N->d);
                free(F);
                elim_run++;
                l++;
                continue;
            }
            free(F);
        }
        /* aggregation level */
        L->kind = ORC_AGG;
        L->lambda = orc_lanczos(nl, L->row_ptr, L->col, L->w, L->d, p.seed, l, p.lanczos_steps, NULL, NULL, NULL);
        L->agg = malloc(sizeof(int32_t) * (size_t)nl);
        L->S = malloc(sizeof(double) * (size_t)(z + 1));
        double *X = malloc(sizeof(double) * 4 * (size_t)nl);
        double *C = malloc(sizeof(double) * (size_t)(z + 1));
        int64_t m = nl;
        for (int attempt = 0; attempt < 2 && m == nl; attempt++) {            /* O-S9 stall retry */
            orc_test_vectors(nl, L->row_ptr, L->col, L->w, L->d, p.seed, l, attempt, p.tv_sweeps, p.tv_omega, X);
            orc_affinity(nl, L->row_ptr, L->col, X, p.affinity_power, C);
            orc_normalize_strength(nl, L->row_ptr, L->col, C, L->S);
            m = orc_aggregate(nl, L->row_ptr, L->col, L->S, p.vote_rounds, p.vote_threshold, L->agg, NULL, NULL);
        }
        free(X); free(C);
        if (m == nl) {                                                        /* stalled twice */
            free(L->agg); L->agg = NULL;
            free(L->S); L->S = NULL;
            L->kind = ORC_COARSEST;
            h->status = ORC_ESTALL;
            if (nl > 8192) { h->nlev = l + 1; orc_free(h); return ORC_ESTALL; }
            break;
        }
        L->m = m;
        orc_level *N = &h->lev[l + 1];
        N->n = m;
        N->row_ptr = malloc(sizeof(int64_t) * (size_t)(m + 1));
        int64_t cn = orc_galerkin_count(nl, L->row_ptr, L->col, L->agg, m);
        N->nnz = cn;
        N->col = malloc(sizeof(int32_t) * (size_t)(cn + 1));
        N->w = malloc(sizeof(double) * (size_t)(cn + 1));
        N->d = malloc(sizeof(double) * (size_t)(m + 1));
        orc_galerkin(nl, L->row_ptr, L->col, L->w, L->agg, m, N->row_ptr, N->col, N->w, N->d);
        elim_run = 0;
        l++;
    }
    h->nlev = l + 1;
    for (int32_t t = 0; t < l; t++) {                  /* transfer lists (ascending fine index) */
        orc_level *T = &h->lev[t];
        if (T->kind == ORC_AGG) {
            T->mem_ptr = calloc((size_t)(T->m + 1), sizeof(int64_t));
            T->members = malloc(sizeof(int32_t) * (size_t)(T->n + 1));
            for (int64_t i = 0; i < T->n; i++) T->mem_ptr[T->agg[i] + 1]++;
            for (int64_t a = 0; a < T->m; a++) T->mem_ptr[a + 1] += T->mem_ptr[a];
            int64_t *cur = malloc(sizeof(int64_t) * (size_t)(T->m + 1));
            memcpy(cur, T->mem_ptr, sizeof(int64_t) * (size_t)(T->m + 1));
            for (int64_t i = 0; i < T->n; i++) T->members[cur[T->agg[i]]++] = (int32_t)i;
            free(cur);
        } else if (T->kind == ORC_ELIM) {
            int64_t nc = h->lev[t + 1].n, tot = 0;
            T->ct_ptr = calloc((size_t)(nc + 1), sizeof(int64_t));
            for (int64_t f = 0; f < T->n; f++) {
                if (T->fmap[f] >= 0) continue;
                for (int64_t q = T->row_ptr[f]; q < T->row_ptr[f + 1]; q++) { T->ct_ptr[T->fmap[T->col[q]] + 1]++; tot++; }
            }
            for (int64_t c = 0; c < nc; c++) T->ct_ptr[c + 1] += T->ct_ptr[c];
            T->ct_q = malloc(sizeof(int64_t) * (size_t)(tot + 1));
            T->ct_f = malloc(sizeof(int32_t) * (size_t)(tot + 1));
            int64_t *cur = malloc(sizeof(int64_t) * (size_t)(nc + 1));
            memcpy(cur, T->ct_ptr, sizeof(int64_t) * (size_t)(nc + 1));
            for (int64_t f = 0; f < T->n; f++) {
                if (T->fmap[f] >= 0) continue;
                for (int64_t q = T->row_ptr[f]; q < T->row_ptr[f + 1]; q++) {
                    int64_t c = T->fmap[T->col[q]];
                    T->ct_q[cur[c]] = q;
                    T->ct_f[cur[c]] = (int32_t)f;
                    cur[c]++;
                }
            }
            free(cur);
        }
    }
    orc_level *Lc = &h->lev[l];
    Lc->pinv = malloc(sizeof(double) * (size_t)(Lc->n * Lc->n));
    rc = orc_coarse_pinv(Lc->n, Lc->row_ptr, Lc->col, Lc->w, Lc->d, Lc->pinv);
    if (rc != ORC_OK) { orc_free(h); return rc; }
    *out = h;
    return h->status;
}

int32_t orc_nlev(const orc_hier *h) { return h->nlev; }
const orc_level *orc_get_level(const orc_hier *h, int32_t l) { return &h->lev[l]; }

/* ======================================================================== */
/* O-S7 V-cycle: Alg. 1 with gamma = 1, elimination levels as    */
/* the exact additive 2-level transfer of P:463-477 (no smoothing)    */
/* ======================================================================== */

/* b' = P^T b on an elimination level:
 *   b'_idx(c) = b_c + sum_{f~c} fl(w_fc / d_f) b_f, the f in ascending order */
static void elim_restrict(const orc_level *L, int64_t nc, const double *b, double *bc) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < L->n; i++) if (L->fmap[i] >= 0) bc[L->fmap[i]] = b[i];
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t c = 0; c < nc; c++)
        for (int64_t t = L->ct_ptr[c]; t < L->ct_ptr[c + 1]; t++) {
            int64_t f = L->ct_f[t], q = L->ct_q[t];
            bc[c] += (L->w[q] / L->d[f]) * b[f];
        }
}
/* x = P x' + F-smoother: x_c = x'_idx(c); x_f = (b_f + sum w_fc x'_idx(c)) / d_f */
static void elim_prolong(const orc_level *L, const double *b, const double *xc, double *x) {
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < L->n; i++) {
        if (L->fmap[i] >= 0) { x[i] = xc[L->fmap[i]]; continue; }
        double s = b[i];
        for (int64_t q = L->row_ptr[i]; q < L->row_ptr[i + 1]; q++) s += L->w[q] * xc[L->fmap[L->col[q]]];
        x[i] = s / L->d[i];
    }
}
/* r_c[a] = sum_{agg_i = a} r_i, the members in ascending order */
static void agg_restrict(const orc_level *L, const double *r, double *rc) {
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t a = 0; a < L->m; a++) {
        double s = 0.0;
        for (int64_t t = L->mem_ptr[a]; t < L->mem_ptr[a + 1]; t++) s += r[L->members[t]];
        rc[a] = s;
    }
}

void orc_vcycle(const orc_hier *h, int32_t l, const double *b, double *x) {
    const orc_level *L = &h->lev[l];
    int64_t n = L->n;
    if (L->kind == ORC_COARSEST) {                   /* x = L_c^+ (b - mean b) */
        #pragma omp parallel for schedule(static) if (n > 64)
        for (int64_t i = 0; i < n; i++) {
            double s = 0.0;
            for (int64_t j = 0; j < n; j++) s += L->pinv[i * n + j] * b[j];
            x[i] = s;
        }
        return;
    }
    if (L->kind == ORC_ELIM) {
        int64_t nc = h->lev[l + 1].n;
        double *bc = malloc(sizeof(double) * (size_t)(nc + 1)), *xc = malloc(sizeof(double) * (size_t)(nc + 1));
        /* b' = P^T b:  b'_idx(c) = b_c + sum_{f~c} (w_fc/d_f) b_f */
        elim_restrict(L, nc, b, bc);
        orc_vcycle(h, l + 1, bc, xc);
        /* x = P x' + Fsmooth(b): x_c = x'_idx(c); x_f = (b_f + sum w_fc x'_idx(c)) / d_f */
        elim_prolong(L, b, xc, x);
        free(bc); free(xc);
        return;
    }
    /* aggregation level */
    const orc_params *p = &h->p;
    int64_t m = L->m;
    double *r = malloc(sizeof(double) * (size_t)n);
    double *rc = calloc((size_t)(m + 1), sizeof(double)), *xc = malloc(sizeof(double) * (size_t)(m + 1));
    orc_chebyshev(n, L->row_ptr, L->col, L->w, L->d, L->lambda, p->cheby_lo, p->cheby_hi,
                  p->cheby_degree, b, x, 1);                                 /* pre-smooth from 0 */
    orc_spmv(n, L->row_ptr, L->col, L->w, L->d, x, r);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) r[i] = b[i] - r[i];                      /* residual */
    agg_restrict(L, r, rc);                                                  /* R r */
    orc_vcycle(h, l + 1, rc, xc);                                            /* coarse */
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) x[i] += xc[L->agg[i]];                   /* x += P x_c */
    orc_chebyshev(n, L->row_ptr, L->col, L->w, L->d, L->lambda, p->cheby_lo, p->cheby_hi,
                  p->cheby_degree, b, x, 0);                                 /* post-smooth */
    free(r); free(rc); free(xc);
}

/* Solve-phase dot products and sums in fixed 4096-element chunks: each chunk
 * summed left to right, then the chunk sums left to right (SURVEY §8(d) M5:
 * the same rounding for any number of threads; the solve phase's parity is by
 * tolerance, O-S11).  b = NULL: sum of a. */
#define ORC_CHUNK 4096
static double chunked_sum(const double *a, const double *b, int64_t n) {
    int64_t nc = (n + ORC_CHUNK - 1) / ORC_CHUNK;
    double stackp[64];
    double *part = nc <= 64 ? stackp : malloc(sizeof(double) * (size_t)nc);
    #pragma omp parallel for schedule(static) if (nc > 4)
    for (int64_t c = 0; c < nc; c++) {
        int64_t e = (c + 1) * ORC_CHUNK < n ? (c + 1) * ORC_CHUNK : n;
        double s = 0.0;
        if (b) for (int64_t i = c * ORC_CHUNK; i < e; i++) s += a[i] * b[i];
        else for (int64_t i = c * ORC_CHUNK; i < e; i++) s += a[i];
        part[c] = s;
    }
    double s = 0.0;
    for (int64_t c = 0; c < nc; c++) s += part[c];
    if (part != stackp) free(part);
    return s;
}
static double dotp(const double *a, const double *b, int64_t n) { return chunked_sum(a, b, n); }

/* ======================================================================== */
/* N2 K-cycle (Notay & Vassilevski's recursive Krylov cycle):     */
/* at each aggregation level below the finest, kcycle_inner FCG iterations    */
/* with the rest of the hierarchy as the preconditioner; elimination levels  */
/* are not accelerated.  Smoothing, transfers and the coarsest   */
/* solve are those of the V-cycle above.                                      */
/* ======================================================================== */

void orc_kcycle(const orc_hier *h, int32_t l, const double *b, double *x) {
    const orc_level *L = &h->lev[l];
    int64_t n = L->n;
    if (L->kind == ORC_COARSEST) { orc_vcycle(h, l, b, x); return; }
    if (L->kind == ORC_ELIM) {
        int64_t nc = h->lev[l + 1].n;
        double *bc = malloc(sizeof(double) * (size_t)(nc + 1)), *xc = malloc(sizeof(double) * (size_t)(nc + 1));
        elim_restrict(L, nc, b, bc);
        orc_kcoarse(h, l + 1, bc, xc);                                       /* coarse problem */
        elim_prolong(L, b, xc, x);
        free(bc); free(xc);
        return;
    }
    const orc_params *p = &h->p;
    int64_t m = L->m;
    double *r = malloc(sizeof(double) * (size_t)n);
    double *rc = calloc((size_t)(m + 1), sizeof(double)), *xc = malloc(sizeof(double) * (size_t)(m + 1));
    orc_chebyshev(n, L->row_ptr, L->col, L->w, L->d, L->lambda, p->cheby_lo, p->cheby_hi,
                  p->cheby_degree, b, x, 1);                                 /* pre-smooth from 0 */
    orc_spmv(n, L->row_ptr, L->col, L->w, L->d, x, r);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) r[i] = b[i] - r[i];                      /* residual */
    agg_restrict(L, r, rc);                                                  /* R r */
    orc_kcoarse(h, l + 1, rc, xc);                                           /* coarse problem */
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) x[i] += xc[L->agg[i]];                   /* x += P x_c */
    orc_chebyshev(n, L->row_ptr, L->col, L->w, L->d, L->lambda, p->cheby_lo, p->cheby_hi,
                  p->cheby_degree, b, x, 0);                                 /* post-smooth */
    free(r); free(rc); free(xc);
}

/* FCG(1) (Notay 2000, truncation 1) from x = 0, k = 1..kcycle_inner:
 *   z = B r ;  p = z  (k = 1) ,  p = z - (z.q_prev / p_prev.q_prev) p_prev  (k > 1)
 *   q = L p ;  alpha = (p.r) / (p.q) ;  x += alpha p ;  r -= alpha q
 * with B = orc_kcycle(l).  A direction with p.q = 0 (a zero right-hand side)
 * takes alpha = 0 and beta = 0 (reading R-K2). */
void orc_kcoarse(const orc_hier *h, int32_t l, const double *b, double *x) {
    const orc_level *L = &h->lev[l];
    int64_t n = L->n;
    if (L->kind != ORC_AGG) { orc_kcycle(h, l, b, x); return; }
    double *r = malloc(sizeof(double) * (size_t)n), *z = malloc(sizeof(double) * (size_t)n);
    double *pv = malloc(sizeof(double) * (size_t)n), *q = malloc(sizeof(double) * (size_t)n);
    memcpy(r, b, sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; i++) x[i] = 0.0;
    double pq_prev = 0.0;
    for (int32_t k = 1; k <= h->p.kcycle_inner; k++) {
        orc_kcycle(h, l, r, z);
        if (k == 1) {
            memcpy(pv, z, sizeof(double) * (size_t)n);
        } else {
            double beta = pq_prev != 0.0 ? -dotp(z, q, n) / pq_prev : 0.0;   /* q = L p_prev here */
            for (int64_t i = 0; i < n; i++) pv[i] = z[i] + beta * pv[i];
        }
        orc_spmv(n, L->row_ptr, L->col, L->w, L->d, pv, q);
        double pq = dotp(pv, q, n);
        double alpha = pq != 0.0 ? dotp(pv, r, n) / pq : 0.0;
        for (int64_t i = 0; i < n; i++) { x[i] += alpha * pv[i]; r[i] -= alpha * q[i]; }
        pq_prev = pq;
    }
    free(r); free(z); free(pv); free(q);
}

/* ======================================================================== */
/* O-S8 PCG preconditioned by one V-cycle      */
/* ======================================================================== */

static void project_mean(double *v, int64_t n) {
    double s = chunked_sum(v, NULL, n);
    s /= (double)n;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) v[i] -= s;
}

int orc_solve(const orc_hier *h, const double *b_in, double *x_out, double tol,
              int32_t *iters, double *rel_residual) {
    const orc_level *L0 = &h->lev[0];
    int64_t n = L0->n;
    int32_t max_iters = h->p.max_iters;
    double *b = malloc(sizeof(double) * (size_t)n), *x = calloc((size_t)n, sizeof(double));
    double *r = malloc(sizeof(double) * (size_t)n), *z = malloc(sizeof(double) * (size_t)n);
    double *pv = malloc(sizeof(double) * (size_t)n), *q = malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; i++) b[h->perm[i]] = b_in[i];                 /* b' = Pi b */
    project_mean(b, n);
    double bn = sqrt(dotp(b, b, n));
    int rc = ORC_OK;
    int32_t k = 0;
    double rel = 0.0;
    if (bn == 0.0) {
        for (int64_t i = 0; i < n; i++) x_out[i] = 0.0;
        *iters = 0; *rel_residual = 0.0;
        goto done;
    }
    memcpy(r, b, sizeof(double) * (size_t)n);
    int conv = 0;
    if (h->p.cycle == 1) {
        /* N2: FCG(1) preconditioned by the K-cycle ("FCG when using
         * K-cycles"); same projection and stopping rules as the PCG below */
        orc_kcycle(h, 0, r, z);
        project_mean(z, n);
        memcpy(pv, z, sizeof(double) * (size_t)n);
        for (k = 1; k <= max_iters; k++) {
            orc_spmv(n, L0->row_ptr, L0->col, L0->w, L0->d, pv, q);
            double pq = dotp(pv, q, n);
            double alpha = dotp(pv, r, n) / pq;
            for (int64_t i = 0; i < n; i++) { x[i] += alpha * pv[i]; r[i] -= alpha * q[i]; }
            if (sqrt(dotp(r, r, n)) / bn <= tol) {                           /* O-R30 */
                orc_spmv(n, L0->row_ptr, L0->col, L0->w, L0->d, x, z);
                for (int64_t i = 0; i < n; i++) z[i] = b[i] - z[i];
                if (sqrt(dotp(z, z, n)) / bn <= tol) { conv = 1; break; }
                memcpy(r, z, sizeof(double) * (size_t)n);
            }
            orc_kcycle(h, 0, r, z);
            project_mean(z, n);                                              /* O-R29 */
            double beta = -dotp(z, q, n) / pq;
            for (int64_t i = 0; i < n; i++) pv[i] = z[i] + beta * pv[i];
        }
    } else {
    orc_vcycle(h, 0, r, z);
    project_mean(z, n);
    memcpy(pv, z, sizeof(double) * (size_t)n);
    double rho = dotp(r, z, n);
    for (k = 1; k <= max_iters; k++) {
        orc_spmv(n, L0->row_ptr, L0->col, L0->w, L0->d, pv, q);
        double alpha = rho / dotp(pv, q, n);
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) { x[i] += alpha * pv[i]; r[i] -= alpha * q[i]; }
        if (sqrt(dotp(r, r, n)) / bn <= tol) {                               /* O-R30 */
            orc_spmv(n, L0->row_ptr, L0->col, L0->w, L0->d, x, q);
            for (int64_t i = 0; i < n; i++) q[i] = b[i] - q[i];
            if (sqrt(dotp(q, q, n)) / bn <= tol) { conv = 1; break; }
            memcpy(r, q, sizeof(double) * (size_t)n);
        }
        orc_vcycle(h, 0, r, z);
        project_mean(z, n);                                                  /* O-R29 */
        double rho2 = dotp(r, z, n);
        double beta = rho2 / rho;
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) pv[i] = z[i] + beta * pv[i];
        rho = rho2;
    }
    }
    if (!conv) { k = max_iters; rc = ORC_ENOCONV; }
    project_mean(x, n);
    orc_spmv(n, L0->row_ptr, L0->col, L0->w, L0->d, x, q);
    for (int64_t i = 0; i < n; i++) q[i] = b[i] - q[i];
    rel = sqrt(dotp(q, q, n)) / bn;
    for (int64_t i = 0; i < n; i++) x_out[i] = x[h->perm[i]];               /* x = Pi^T x' */
    *iters = k;
    *rel_residual = rel;
done:
    free(b); free(x); free(r); free(z); free(pv); free(q);
    return rc;
}
