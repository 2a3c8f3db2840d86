/*
 * oracle/lap_oracle.h -- CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * A plain, slow, single-threaded C implementation of the unsmoothed-
 * aggregation multigrid method for graph Laplacians of Konolige & Brown,
 * "A Parallel Solver for Graph Laplacians" (arXiv 1705.06266), written from
 * PAPER.md and the readings in SURVEY.md §8(c) / DESIGN.md §Readings.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1705_06266_b200/, liblap.so) never links, imports or calls it, and
 * the two share no source, header, table or helper.
 *
 * Citations: P:NNN = /root/reference/PAPER.md line NNN; S:NNN = SPEC.md line;
 * O-xx = SURVEY.md §8(c) row.
 *
 * Pins: every function below is pinned by tests/test_oracle_*.py and
 * tests/test_golden_streams.py against something other than itself (SPEC /
 * SURVEY worked examples and goldens, closed forms, brute force on tiny
 * graphs, dense library routines); the K-cycle (orc_kcycle / orc_kcoarse,
 * N2) by the FCG Gram-system identity and the V-cycle/PCG special cases
 * (tests/test_oracle_kcycle.py).  No function is parity-unpinned.  What has
 * no external truth (SURVEY O-P16) is only the OUTPUT of these pinned
 * functions on the five BASELINE.json configs as a whole (nobody publishes
 * the aggregates of a 4M-vertex graph): there the check is the invariants
 * at full size plus "oracle == GPU bit for bit".
 */
#ifndef LAP_ORACLE_H
#define LAP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EGRAPH = 2, ORC_EDISCONNECTED = 3,
       ORC_ENOMEM = 4, ORC_ENOCONV = 7, ORC_ESTALL = 8 };

enum { ORC_AGG = 0, ORC_ELIM = 1, ORC_COARSEST = 2 };

typedef struct {
    double  tol;             /* 1e-8                    */
    int32_t max_iters;       /* 500            S:547, O-R43             */
    int32_t cheby_degree;    /* 2                    */
    double  cheby_lo;        /* 0.3            P:643, O-R2              */
    double  cheby_hi;        /* 1.1            P:643, O-R2              */
    int32_t lanczos_steps;   /* 10             P:643, O-R3              */
    int32_t elim_max_degree; /* 4                */
    int32_t elim_enable;     /* 1                                       */
    int32_t n_test_vectors;  /* 4 (fixed)                    */
    int32_t tv_sweeps;       /* 3                    */
    double  tv_omega;        /* 2/3            O-R6                     */
    int32_t vote_rounds;     /* 10             */
    int32_t vote_threshold;  /* 8 (>=)         P:619, O-R8              */
    int64_t coarse_nnz;      /* 1000           P:672, O-R27             */
    int32_t max_levels;      /* 40             S:467, O-R28             */
    uint64_t seed;           /* 0              O-S11                    */
    int32_t random_order;    /* 1                */
    int32_t affinity_power;  /* 1 (LAMG, O-R5); 2 = literal P:564-565   */
    int32_t cycle;           /* 0 V-cycle + PCG (default);
                                1 K-cycle + FCG (N2)         */
    int32_t kcycle_inner;    /* 2 inner FCG iterations   */
    int32_t elim_rounds;     /* 1: elimination levels in a row */
} orc_params;

typedef struct {
    int32_t kind;            /* ORC_AGG / ORC_ELIM / ORC_COARSEST       */
    int64_t n, nnz;          /* vertices, stored off-diagonal entries   */
    int64_t *row_ptr;        /* n+1                                     */
    int32_t *col;            /* nnz, ascending per row                  */
    double  *w;              /* nnz, > 0 (L_ij = -w_ij)                 */
    double  *d;              /* n, diag(L) = CanonSum of the row        */
    /* aggregation level */
    double   lambda;         /* lambda-hat of D^-1 L (O-S6)             */
    int64_t  m;              /* number of aggregates (= next n)         */
    int32_t *agg;            /* n: aggregate id                         */
    double  *S;              /* nnz: strength (aligned with col)        */
    /* elimination level */
    int64_t  nF;             /* |F|                                     */
    int32_t *fmap;           /* n: C -> coarse index >= 0; F -> -1-fslot */
    /* coarsest */
    double  *pinv;           /* n*n row-major L^+                       */
    /* transfer lists (derived at the end of setup; fix the summation order
     * of R r and P^T b to ascending fine index, whatever the thread count) */
    int64_t *mem_ptr;        /* agg: m+1, members of aggregate a ascending */
    int32_t *members;        /* agg: n                                  */
    int64_t *ct_ptr;         /* elim: nc+1, F neighbours of C vertex c ascending */
    int64_t *ct_q;           /* elim: entry index q of (f, c) in row f  */
    int32_t *ct_f;           /* elim: the F vertex f                    */
} orc_level;

typedef struct {
    int32_t nlev;
    int32_t status;          /* ORC_OK or ORC_ESTALL                    */
    int64_t n0;
    int64_t *perm;           /* n0: new id of input vertex (Pi_rand)    */
    orc_level lev[64];
    orc_params p;
} orc_hier;

void     orc_params_default(orc_params *p);
void     orc_set_threads(int32_t t);   /* OpenMP threads (results do not depend on it) */
int32_t  orc_get_threads(void);

/* --- canonical arithmetic (O-S11) ---------------------------------------- */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_salt(uint64_t seed, uint64_t k);
uint64_t orc_mix64_inverse(uint64_t z);
int32_t  orc_canon_elo(int32_t e_max, int64_t K);
double   orc_canon_sum(const double *t, int64_t cnt, int32_t e_max, int64_t K);
int32_t  orc_ilogb(double x);

/* --- O-S0 / O-S1 ---------------------------------------------------------- */
int  orc_validate(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w);
void orc_random_perm(int64_t n, uint64_t seed, int64_t *perm);
void orc_row_sums(int64_t n, const int64_t *row_ptr, const double *w, double *d);
void orc_relabel(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w, const int64_t *perm,
                 int64_t *out_row_ptr, int32_t *out_col, double *out_w);

/* --- primitives (each pinned in tests) ------------------------------------ */
void orc_spmv(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
              const double *d, const double *x, double *y);
/* h(j) = mix64(j XOR salt_2) (O-R17) */
uint64_t orc_elim_hash(uint64_t j, uint64_t seed);
int64_t orc_elim_select(int64_t n, const int64_t *row_ptr, const int32_t *col,
                        int32_t max_degree, uint64_t seed, const uint64_t *hash_override,
                        uint8_t *F);
/* Schur complement (star-mesh): returns new nnz; out arrays sized by caller
 * from orc_schur_count.  fmap filled as in orc_level. */
int64_t orc_schur_count(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint8_t *F);
int64_t orc_schur(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                  const double *d, const uint8_t *F, int32_t *fmap,
                  int64_t *nrow_ptr, int32_t *ncol, double *nw, double *nd);
void orc_test_vectors(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                      const double *d, uint64_t seed, int32_t level, int32_t attempt,
                      int32_t sweeps, double omega, double *X /* n*4 row-major, in: ignored */);
void orc_test_vectors_from(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                           const double *d, int32_t sweeps, double omega, double *X /* in/out */);
void orc_affinity(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *X,
                  int32_t power, double *C);
void orc_normalize_strength(int64_t n, const int64_t *row_ptr, const int32_t *col,
                            const double *C, double *S);
int64_t orc_aggregate(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *S,
                      int32_t rounds, int32_t threshold, int32_t *agg,
                      int8_t *state_out, int32_t *votes_out);
int64_t orc_galerkin_count(int64_t n, const int64_t *row_ptr, const int32_t *col,
                           const int32_t *agg, int64_t m);
int64_t orc_galerkin(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                     const int32_t *agg, int64_t m, int64_t *crow_ptr, int32_t *ccol,
                     double *cw, double *cd);
double orc_lanczos(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                   const double *d, uint64_t seed, int32_t level, int32_t steps,
                   double *alpha_out, double *beta_out, int32_t *k_out);
void orc_lanczos_start(int64_t n, uint64_t seed, int32_t level, double *v /* n, unnormalised */);
double orc_tridiag_max_eig(int32_t k, const double *alpha, const double *beta);
int  orc_coarse_pinv(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                     const double *d, double *pinv);
void orc_chebyshev(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                   const double *d, double lambda, double lo, double hi, int32_t degree,
                   const double *b, double *x, int32_t x_is_zero);

/* --- hierarchy + solve (O-S7..O-S9) --------------------------------------- */
int  orc_setup(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
               const orc_params *p, orc_hier **out);
void orc_free(orc_hier *h);
/* V-cycle on the permuted (internal) numbering, level l */
void orc_vcycle(const orc_hier *h, int32_t l, const double *b, double *x);
/* K-cycle (N2): as the V-cycle, but the coarse problem of an
 * aggregation level is handed to orc_kcoarse instead of one recursive cycle */
void orc_kcycle(const orc_hier *h, int32_t l, const double *b, double *x);
/* x = kcycle_inner FCG(1) iterations on L_l x = b from x = 0, preconditioned
 * by orc_kcycle(l) when level l is an aggregation level; orc_kcycle(l) itself
 * otherwise (elimination levels are not accelerated) */
void orc_kcoarse(const orc_hier *h, int32_t l, const double *b, double *x);
/* PCG (cycle 0) or FCG(1) + K-cycle (cycle 1) on the caller's numbering;
 * returns ORC_OK / ORC_ENOCONV */
int  orc_solve(const orc_hier *h, const double *b, double *x, double tol,
               int32_t *iters, double *rel_residual);
/* accessors for ctypes */
int32_t orc_nlev(const orc_hier *h);
const orc_level *orc_get_level(const orc_hier *h, int32_t l);

#ifdef __cplusplus
}
#endif
#endif
