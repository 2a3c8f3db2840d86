/*
 * include/lap.h -- C ABI of liblap.so, the B200-native (sm_100a) hot path of
 * the unsmoothed-aggregation multigrid solver for graph Laplacians of
 * Konolige & Brown, "A Parallel Solver for Graph Laplacians" (arXiv
 * 1705.06266).  Citations: P:NNN = PAPER.md line, S:NNN = SPEC.md line,
 * O-xx = SURVEY.md §8(c) reading.
 *
 * Problem: given a connected, positively weighted,
 * undirected graph G = (V, E, w) with Laplacian L = D - A, compute x with
 * L x = b for b projected orthogonal to the constant vector.
 *
 * Two calls carry the method:
 *   lap_setup  -- builds the multigrid hierarchy on the GPU:
 *                 random vertex order, low-degree elimination levels
 *                 (Alg. 2 + Schur complement), aggregation levels (affinity
 *                 strength, Alg. 3 voting, Galerkin R L P), lambda-hat by
 *                 Lanczos, dense coarsest pseudo-inverse.
 *   lap_solve  -- PCG preconditioned by one V-cycle (Alg. 1, gamma = 1) with
 *                 degree-2 Chebyshev/Jacobi smoothing.
 *
 * Conventions for every function:
 *   - Return value is a lap_status; LAP_OK = 0.  No C++ exception crosses
 *     the ABI.  On failure, *out pointers are set to NULL and
 *     lap_last_error() returns a thread-local message.
 *   - `cuda_stream` is a cudaStream_t (NULL = legacy default stream).  All
 *     device work is enqueued on it.  Calls that return host-visible scalars
 *     (lap_setup, lap_solve, lap_level_*) synchronise that stream.
 *   - Vector arguments of lap_solve / lap_spmv / lap_vcycle may be host
 *     (pageable or pinned) or device pointers on the current device; the
 *     library detects which with cudaPointerGetAttributes and copies host
 *     data itself.  The caller owns them; the library never retains them.
 *   - The hierarchy owns all its device memory until lap_free.  One solve
 *     may be in flight per hierarchy at a time (work vectors live in it).
 *   - Everything computes in IEEE fp64.  Setup reductions that feed discrete
 *     decisions use the order-independent canonical sum of O-S11 (int128
 *     fixed point), so hierarchies are bit-identical to the CPU oracle.
 */
#ifndef LAP_H
#define LAP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LAP_OK = 0,
    LAP_EINVAL = 1,        /* bad argument / parameter                               */
    LAP_EGRAPH = 2,        /* asymmetric, self loop, w<=0/NaN, unsorted/duplicate col */
    LAP_EDISCONNECTED = 3, /* graph not connected                      */
    LAP_ENOMEM = 4,        /* device allocation failed                               */
    LAP_ECUDA = 5,         /* CUDA runtime error                                     */
    LAP_ENCCL = 6,         /* reserved: collective failure                           */
    LAP_ENOCONV = 7,       /* PCG hit max_iters; x holds the last iterate    */
    LAP_ESTALL = 8         /* warning: aggregation stalled twice, coarsest is large  */
} lap_status;

/* Symmetric off-diagonal adjacency of G in CSR (the Laplacian is implied:
 * L_ij = -w_ij, L_ii = sum_j w_ij).  n >= 1; row_ptr[0] = 0; col strictly
 * ascending within each row, no i == i entries; w_ij == w_ji bitwise, finite,
 * > 0; w == NULL means unit weights.  on_device: 0 = host arrays,
 * 1 = device arrays on the current device.  lap_setup deep-copies. */
typedef struct {
    int64_t n;
    const int64_t *row_ptr;   /* n+1 */
    const int32_t *col;       /* row_ptr[n] */
    const double *w;          /* row_ptr[n] or NULL */
    int32_t on_device;
} lap_graph;

/* Parameters; lap_params_default() sets the paper's values. */
typedef struct {
    double tol;               /* 1e-8 relative residual        */
    int32_t max_iters;        /* 500                              S:547, O-R43 */
    int32_t cheby_degree;     /* 2 (pre and post)        */
    double cheby_lo;          /* 0.3 * lambda-hat                 P:643, O-R2  */
    double cheby_hi;          /* 1.1 * lambda-hat                 P:643, O-R2  */
    int32_t lanczos_steps;    /* 10                               P:643, O-R3  */
    int32_t elim_max_degree;  /* 4    */
    int32_t elim_enable;      /* 1        */
    int32_t n_test_vectors;   /* 4 (only 4 supported)        */
    int32_t tv_sweeps;        /* 3 Jacobi sweeps        */
    double tv_omega;          /* 2/3                              O-R6         */
    int32_t vote_rounds;      /* 10   */
    int32_t vote_threshold;   /* 8, seed iff votes >= 8           P:619, O-R8  */
    int64_t coarse_nnz;       /* 1000: coarsest iff n+nnz <= this P:672, O-R27 */
    int32_t max_levels;       /* 40        */
    uint64_t seed;            /* 0: salts of O-S11                             */
    int32_t random_order;     /* 1: Pi_rand on the input only    */
    int32_t affinity_power;   /* 1 = LAMG affinity (O-R5); 2 = literal P:564   */
    int32_t keep_strength;    /* 1: retain S per aggregation level (tests)     */
    int32_t use_graphs;       /* 1: capture the V-cycle as a CUDA graph        */
    int64_t replicate_nnz;    /* multi-GPU: levels with nnz >= this are sharded,
                                 the rest replicated; 0 = nnz(L_0) / (32 P)    */
    int32_t cycle;            /* 0: PCG + V-cycle (default);
                                 1: FCG(1) + K-cycle,
                                 single-GPU only                               */
    int32_t kcycle_inner;     /* 2: FCG iterations per aggregation level below
                                 the finest (paper: "a number of")      */
    int32_t elim_rounds;      /* 1: at most this many elimination levels in a
                                 row before an aggregation level ("we can run
                                 low-degree elimination multiple times in a
                                 row"; one is the paper's choice)   */
    int32_t keep_logical;     /* -1: release a level's logical CSR once its solve
                                 storage exists when nnz >= 2^28 (cfg 5 memory);
                                 1: always keep (lap_level_export needs it);
                                 0: always release                             */
} lap_params;

typedef struct lap_hierarchy lap_hierarchy;
typedef struct lap_comm lap_comm;

void lap_params_default(lap_params *p);
const char *lap_last_error(void);
const char *lap_version(void);

/* Build the hierarchy (SURVEY O-S0..O-S10).
 * Validates the graph (LAP_EGRAPH / LAP_EDISCONNECTED); returns LAP_ESTALL
 * (with a usable hierarchy) if aggregation stalled twice (O-R28). */
lap_status lap_setup(const lap_graph *g, const lap_params *p, void *cuda_stream,
                     lap_hierarchy **out);

/* Solve L x = b to relative residual tol (<= 0: use params.tol) with PCG +
 * V-cycle (O-S8), or FCG(1) + K-cycle when the hierarchy
 * was built with params.cycle = 1.  b, x: length n in the caller's
 * numbering.  A copy of b is projected to mean zero; x is returned mean-zero.
 * *iters = number of L p products; *rel_residual = ||b - L x|| / ||b||
 * recomputed at the end.  b = const -> x = 0, iters = 0, LAP_OK.
 * LAP_ENOCONV if max_iters was reached (x = last iterate). */
lap_status lap_solve(lap_hierarchy *h, const double *b, double *x, double tol,
                     int32_t *iters, double *rel_residual, void *cuda_stream);

void lap_free(lap_hierarchy *h);   /* NULL-safe */

/* A hierarchy given as files (SURVEY §8(b) interchange format; the CPU oracle
 * writes it, oracle.Hierarchy.export): the solve then runs on exactly those
 * operators, maps and lambda-hats (parity isolation; checkpoint / resume of a
 * setup).  Directory layout, little-endian raw arrays + flat JSON:
 *   meta.json            {"format": "lap-hierarchy-v1", "nlev": L, "n0": n, ...}
 *   perm.i64             n: internal (level-0) id of caller vertex i (Pi_rand)
 *   L<l>/meta.json       {"kind": 0 agg | 1 elim | 2 coarsest, "n", "nnz",
 *                         "lambda" and "m" (kind 0)}
 *   L<l>/row_ptr.i64 (n+1), col.i32 (nnz), w.f64 (nnz), d.f64 (n)
 *   L<l>/agg.i32 (kind 0) | fmap.i32 (kind 1: C -> order-preserving coarse id,
 *                         F -> -1 - slot, slots ascending) | coarse_pinv.f64
 *                         (kind 2, n*n row-major L^+)
 * Sizes are checked against meta.json and the level chain (n_{l+1} = m or
 * n - |F|; the last level, and only it, is the coarsest); any mismatch or
 * unreadable file -> LAP_EINVAL.  p: solve parameters (cheby_lo/hi, cycle,
 * use_graphs, tol, max_iters); the setup parameters are not used. */
lap_status lap_import_hierarchy(const char *dir, const lap_params *p, void *cuda_stream, lap_hierarchy **out);

/* Device memory: liblap allocates from a stream-ordered pool of its own (never
 * the device's default pool, so PyTorch's caching allocator and NCCL are not
 * starved).  When the last live hierarchy is freed the pool is trimmed down to
 * `bytes` of reservation (default 0: everything goes back to the device).  A
 * caller that runs setups in a loop may retain the reservation (e.g. 2^40) to
 * avoid re-mapping gigabytes at every setup; lap_pool_retain(0) releases it. */
void lap_pool_retain(uint64_t bytes);

/* ---- introspection (host output buffers sized from lap_level_info) ------ */
lap_status lap_num_levels(const lap_hierarchy *h, int32_t *nlev);
/* kind: 0 aggregation, 1 elimination, 2 coarsest.  lambda_hat only for kind 0. */
lap_status lap_level_info(const lap_hierarchy *h, int32_t l, int32_t *kind, int64_t *n,
                          int64_t *nnz_off, double *lambda_hat);
/* Copies level l to host arrays (any may be NULL): row_ptr[n+1], col[nnz],
 * w[nnz], d[n], map[n] = agg[] (kind 0) or fmap[] (kind 1: coarse index for
 * C vertices, -1-slot for F vertices).  LAP_EINVAL if row_ptr/col/w are asked
 * for and the level's logical CSR was released (params.keep_logical); use
 * lap_level_rows then. */
lap_status lap_level_export(const lap_hierarchy *h, int32_t l, int64_t *row_ptr, int32_t *col,
                            double *w, double *d, int32_t *map);
/* Rows rows[0..k) of level l's logical CSR (ascending columns, the logical
 * numbering the oracle sees), rebuilt from the solve storage, so it works also
 * when the logical copy was released.  Two calls: with col == NULL only
 * row_ptr[k+1] (host, exclusive offsets) is filled; then col/w (host,
 * row_ptr[k] entries).  Parity hook for graphs too big to export whole. */
lap_status lap_level_rows(const lap_hierarchy *h, int32_t l, int64_t k, const int64_t *rows, int64_t *row_ptr,
                          int32_t *col, double *w);
/* Strength S[nnz] of aggregation level l (requires params.keep_strength). */
lap_status lap_level_strength(const lap_hierarchy *h, int32_t l, double *S);
/* Coarsest pseudo-inverse, n*n row-major (host buffer). */
lap_status lap_coarse_pinv(const lap_hierarchy *h, double *pinv);
/* perm[i] = internal (level-0) id of caller vertex i (Pi_rand). */
lap_status lap_perm(const lap_hierarchy *h, int64_t *perm);
/* y = L_l x on level l, internal numbering (H1). */
lap_status lap_spmv(const lap_hierarchy *h, int32_t l, const double *x, double *y, void *cuda_stream);
/* k right-hand sides at once (P:102-118 -- eigenvector / embedding
 * uses solve many systems with one Laplacian).  Column j of B (n x k,
 * column-major, caller numbering, host or device) is solved exactly as
 * lap_solve would (its own projection, PCG + V-cycle, stopping rule; O-S8),
 * but the k solves advance together so every pass over a level's matrix
 * serves all columns (SpMM).  1 <= k <= 32 (k <= 8: a thread per row, K values
 * per gather; 9..16: two such blocks of <= 8 columns one after the other;
 * 17..32: 32 lanes per row, one coalesced gather per neighbour).  X: n x k column-major, mean-zero
 * columns.  iters[j], rel_residual[j]: per column (length k).  LAP_ENOCONV if
 * any column reached max_iters.  Single-GPU hierarchies only. */
lap_status lap_solve_block(lap_hierarchy *h, int32_t k, const double *B, double *X, double tol,
                           int32_t *iters, double *rel_residual, void *cuda_stream);
/* z = V(0, r): one V-cycle on the internal (permuted) level-0 numbering (O-S7). */
lap_status lap_vcycle(lap_hierarchy *h, const double *r, double *z, void *cuda_stream);
/* z = K(l, r): one K-cycle at level l: the V-cycle's
 * smoothing and transfers, with the coarse problem of every aggregation level
 * below l solved by params.kcycle_inner FCG(1) iterations preconditioned by
 * the K-cycle there (elimination levels are not accelerated).
 * r, z: length n_l, internal (storage-independent, level-l) numbering, host
 * or device.  with_fcg = 1 applies the FCG iterations at level l itself
 * (l >= 1 aggregation levels; the "coarse solve" orc_kcoarse of the oracle).
 * Any single-GPU hierarchy; LAP_EINVAL for a bad level or a sharded one. */
lap_status lap_kcycle(lap_hierarchy *h, int32_t l, int32_t with_fcg, const double *r, double *z,
                      void *cuda_stream);

/* ---- multi-GPU: 2D-sharded solve ------------------------------
 * The fine levels (nnz >= params.replicate_nnz) are distributed as a 2D edge
 * partition over a pr x pc process grid: rank r sits at grid
 * position (r / pc, r % pc) and owns one piece of every sharded level's rows
 * (block-cyclic over the storage order); per SpMV the column communicator
 * allgathers x and the row communicator reduce-scatters A x (NCCL).  The
 * coarse levels are replicated on every rank.  Setup is the single-
 * GPU setup run identically on each rank (deterministic, O-R23).
 * lap_solve on such a hierarchy takes the FULL b and returns the FULL x on
 * every rank; all ranks must call it together (collectives inside). */
/* 128-byte ncclUniqueId for rank 0 to broadcast (e.g. via torch.distributed). */
lap_status lap_nccl_unique_id(uint8_t id[128]);
/* One rank per process/GPU; grid_rows * grid_cols == nranks <= 16.  Creates the
 * NCCL world communicator and its row / column splits.  LAP_ENCCL on failure. */
lap_status lap_comm_create(const uint8_t nccl_id[128], int32_t rank, int32_t nranks, int32_t grid_rows,
                           int32_t grid_cols, lap_comm **out);
/* The whole pr x pc grid inside this process on the current device: every
 * rank's shard is held here and the collectives are device copies and
 * fixed-order sums (used to validate the sharded data path on one GPU). */
lap_status lap_comm_create_virtual(int32_t grid_rows, int32_t grid_cols, lap_comm **out);
lap_status lap_comm_info(const lap_comm *c, int32_t *rank, int32_t *nranks, int32_t *grid_rows, int32_t *grid_cols,
                         int32_t *is_virtual);
void lap_comm_free(lap_comm *c);  /* NULL-safe; after every hierarchy using it is freed */
/* lap_setup + sharding over the communicator's grid (the comm must outlive h). */
lap_status lap_setup_dist(const lap_graph *g, const lap_params *p, lap_comm *c, void *cuda_stream,
                          lap_hierarchy **out);
/* Host-only (no GPU needed): the piece map of a sharded level with n rows over
 * nranks pieces: dist[t] = piece * piece_size + slot of storage row rows[t]
 * (block-cyclic in blocks of 256 rows); *piece_size = padded piece length. */
/* SURVEY N1 (distributed setup): lap_setup_dist splits every
 * coarse-operator term build (Galerkin R L P, Schur complement, relabel of a
 * big graph) by output rows over the communicator's ranks, each range
 * holding about 1/P of the terms, and gathers the ranges on every rank (the
 * result is the single-GPU operator bit for bit).  This is the split rule,
 * host-only: cum[0..nout] = terms of the output rows before row o
 * (non-decreasing); bounds[0..nranks]: rank r builds rows [bounds[r],
 * bounds[r+1]), bounds[r] = the first o with cum[o] * nranks >= r * cum[nout].
 * LAP_EINVAL on a decreasing or negative cum. */
lap_status lap_setup_split(int64_t nout, const int64_t *cum, int32_t nranks, int64_t *bounds);
lap_status lap_dist_index(int64_t n, int32_t nranks, int64_t m, const int64_t *rows, int64_t *dist,
                          int64_t *piece_size);

/* Test hook: the method's counter-based random streams (SURVEY O-S11, O-R17,
 * O-R7/O-R33, O-S6), evaluated on the device by the same functions the setup
 * kernels use, copied to the HOST buffer `out`:
 *   which = 0: out[i] = h(i) = mix64(i XOR salt_2)          (uint64, n)
 *   which = 1: out[4i+k] = X0[i,k] of (level, attempt)      (double, 4n)
 *   which = 2: out[i] = Lanczos start v_i of `level`, before normalisation
 *              (2 u01(mix64(mix64(salt_4 XOR 2 level) XOR i)) - 1; double, n) P:643
 *   which = 3: out[i] = mix64(i)                            (uint64, n)
 * LAP_EINVAL for a bad `which` / negative sizes. */
lap_status lap_random_stream(int32_t which, uint64_t seed, int32_t level, int32_t attempt, int64_t n, void *out,
                             void *cuda_stream);

/* ---- counters for the benchmark ----------------------------------------- */
typedef struct {
    int64_t kernel_launches;  /* kernels launched by the last lap_solve / lap_setup   */
    int64_t spmv_edges;       /* sum of nnz_off over SpMV-shaped passes (last call)   */
    int64_t spmv_bytes;       /* algorithmic HBM bytes of those passes    */
    double  setup_ms;         /* device time of the last lap_setup (CUDA events)      */
    double  solve_ms;         /* device time of the last lap_solve (CUDA events)      */
    int32_t vcycles;          /* V-cycles applied by the last lap_solve               */
} lap_stats;
lap_status lap_get_stats(const lap_hierarchy *h, lap_stats *s);

/* Time `reps` back-to-back launches of one solve-phase operation on
 * `cuda_stream` with CUDA events; ms[reps] (host) receives per-launch times in
 * milliseconds.  V-cycles (which = 2) are timed one graph launch each; single
 * kernels (which = 0, 1) are captured `reps` at a time into one CUDA graph (as
 * the solve runs them) and every ms[i] is the mean per launch of a timed
 * graph launch.
 *   which = 0: y = L_l x on level l (H1)
 *   which = 1: one fused Chebyshev/Jacobi step on aggregation level l (H2)
 *   which = 2: one V-cycle z = V(0, r) (H16, Alg. 1; l ignored; graph launch)
 * *bytes = algorithmic HBM bytes per launch (12 nnz + 32 n for H1,
 * 12 nnz + 56 n for H2, the sum over the cycle's kernels for a V-cycle);
 * *edges = nonzeros traversed per launch.  Work vectors of the hierarchy are
 * overwritten (zeros).  LAP_EINVAL for a bad level / kind. */
lap_status lap_bench_op(lap_hierarchy *h, int32_t which, int32_t l, int32_t reps, void *cuda_stream,
                        double *ms, double *bytes, int64_t *edges);

/* The M3 "second ceiling": CUDA-event time (ms[reps], host) of
 * one kernel doing m random 8-byte gathers x[col[k]] from an x of nx doubles
 * (uniform counter-hash columns, no locality) with the SpMV's col (int32) and
 * w (fp64) streams -- the SpMV of a random-ordered power-law level without its
 * epilogue.  Allocates its own buffers; 1 <= nx < 2^31. */
lap_status lap_bench_gather(int64_t nx, int64_t m, int32_t reps, void *cuda_stream, double *ms);

#ifdef __cplusplus
}
#endif
#endif
