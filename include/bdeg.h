/* bdeg.h — C ABI of libbdeg.so: exact degree of the C*-solution set of a
 * Laurent binomial system on NVIDIA B200 (sm_100a).
 *
 * Method: Chen & Mehta, arXiv 1501.02237.  The CPU front end
 * computes the Smith Normal Form of the exponent matrix, which
 * fixes the dimension d = n - rank A, the component count |prod d_j|
 * (Prop. 1) and the parametrisation matrix P_0 (eq. rank-decomp).
 * The degree of each component is the normalised volume
 *     deg V = d! Vol_d(conv{p_0^(1), ..., p_0^(n), 0})      (Prop. 4)
 * computed as the sum of |det| over the cells of the regular simplicial
 * subdivision induced by a lifting omega: a (d+1)-subset is a
 * cell iff the lower-face system I(a_0..a_d) (eq. lower-face) is
 * (strictly) feasible.  The GPU enumerates every K-subset of the lifted
 * point configuration by combinatorial rank (the brute force of P:798-800,
 * made practical by prefix-shared fraction-free elimination).
 *
 * Conventions for every entry point:
 *   - Nothing throws across the ABI; every call returns a bdeg_status.
 *   - On error the output structs are left untouched; bdeg_last_error(plan)
 *     (or bdeg_last_error(NULL) for errors before a plan exists) returns a
 *     human-readable message valid until the next call on that plan.
 *   - The caller owns every input array; bdeg_plan* copies what it needs.
 *   - A plan is used by one host thread at a time; plans are independent.
 *   - Device work is enqueued on options.stream (a cudaStream_t; NULL = the
 *     legacy default stream) of options.device.
 *   - There is NO CPU fallback: without a usable sm_100 device the device
 *     entry points return BDEG_E_CUDA.
 */
#ifndef BDEG_H
#define BDEG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bdeg_plan_s *bdeg_plan_t;

typedef enum {
    BDEG_OK = 0,
    BDEG_E_INVALID = 1,       /* bad argument (shape, NULL pointer, range)            */
    BDEG_E_INCONSISTENT = 2,  /* b^{Q_0} != 1: empty solution set         */
    BDEG_E_DEGENERATE = 3,    /* lifting not generic ("almost all"); user-given
                                 lifting, or max_relift generated liftings exhausted  */
    BDEG_E_IO = 4,            /* reserved (SPEC exit code 4)                           */
    BDEG_E_TOO_LARGE = 5,     /* N > 128, K > 32, or an exact value exceeds 2^125      */
    BDEG_E_CUDA = 6,          /* CUDA runtime error / no sm_100 device                 */
    BDEG_E_COMM = 7           /* reserved for the multi-GPU combine                    */
} bdeg_status;

/* x^A = b (eq. standard-form). */
typedef struct {
    int32_t n;               /* number of variables (rows of A), n >= 1              */
    int32_t m;               /* number of binomials (columns of A), m >= 0           */
    const int64_t *A;        /* n*m, ROW-major: A[i*m + j]; column j = alpha_j - beta_j */
    const double *b_re;      /* m entries (real part of b_j = -c_{j,2}/c_{j,1}), or NULL => b = 1 */
    const double *b_im;      /* m entries or NULL (=> imaginary parts 0)             */
    const int64_t *lifting;  /* n+1 values: omega per variable, last = the origin;
                                NULL => generated from options.seed (SplitMix64,
                                values in [0, 2^lift_bits)).            */
} bdeg_problem;

/* options.flags */
#define BDEG_FLAG_NO_LLL            0x1u  /* keep the SNF basis of P_0 (no LLL reduction)     */
#define BDEG_FLAG_NO_HOMOG_SHORTCUT 0x2u  /* always K = d+1 with the origin (no pyramid K = d)  */
#define BDEG_FLAG_FORCE_TIER0       0x4u  /* start in tier 0: int32 values, int64 products            */
#define BDEG_FLAG_FORCE_TIER1       0x8u  /* start in tier 1: int32 V rows / int64 lift row, int64 products */
#define BDEG_FLAG_FORCE_TIER2       0x20u /* tier 2 only: int64 values, checked int128 products       */
#define BDEG_FLAG_NO_RELIFT         0x10u /* report BDEG_E_DEGENERATE instead of re-lifting       */
#define BDEG_FLAG_DEGREE_ONLY       0x40u /* skip cell-dead subtrees (a point of the prefix span
                                             lies strictly below: no cell); degree,
                                             cells, candidates stay exact, singular becomes an
                                             upper bound (singular_complete = 0)              */
#define BDEG_FLAG_NATURAL_ORDER     0x80u /* system plans (bdeg_plan): keep the points in first-
                                             occurrence order.  By default they are sorted by
                                             ascending lifting residual (the lifting minus its
                                             least-squares linear fit; stable) -- the order changes the
                                             rank space and the work, never a result (DESIGN.md
                                             reading O); bdeg_plan_points_get returns the order
                                             in use, and ranks and cell masks refer to it     */

typedef struct {
    uint64_t seed;           /* seed of the generated lifting (and of re-lifts)      */
    int32_t lift_bits;       /* generated omega in [0, 2^lift_bits); default 20      */
    int32_t max_relift;      /* re-lift attempts for generated liftings; default 32  */
    int32_t device;          /* CUDA device ordinal; default 0                       */
    int32_t rank, world;     /* this process's shard of rank space (default 0, 1)    */
    void *stream;            /* cudaStream_t for every launch/copy; NULL = default   */
    uint32_t flags;          /* BDEG_FLAG_*                                          */
    int32_t inner_levels;    /* register-resident DFS depth S in 0..7; -1 = auto     */
    int32_t ctas_per_sm;     /* persistent CTAs per SM; 0 = auto                     */
} bdeg_options;

typedef struct {
    /* front end (bdeg_plan / bdeg_plan_info) */
    int32_t n, rank, dim;    /* dim = n - rank (Prop. 1)                             */
    int32_t K, N;            /* subset size and number of lifted points              */
    int32_t tier;            /* arithmetic tier the enumeration started in (0, 1, 2) */
    int32_t homogeneous;     /* 1 if 1^T A = 0 (K = d, pyramid reading)              */
    int32_t inner_levels;    /* S used by the kernel                                 */
    uint64_t comp_lo, comp_hi;        /* |prod d_j| as unsigned 128-bit      */
    /* enumeration (bdeg_degree / bdeg_finalize) */
    uint64_t deg_lo; int64_t deg_hi;  /* degree of each component, signed 128-bit    */
    uint64_t candidates;     /* K-subsets examined (= C(N,K) for a full run)         */
    uint64_t cells;          /* cells of the regular subdivision (lifting-dependent) */
    uint64_t singular;       /* K-subsets with det = 0 (lifting-independent)         */
    uint64_t ties;           /* would-be cells with a zero facet value (degenerate)  */
    uint64_t overflow_reruns;/* items re-run in tier 2 (int64) after leaving tier 0/1 */
    uint64_t updates;        /* fraction-free elimination updates executed          */
    uint64_t leaves;         /* (K-1)-prefixes tested (each = one warp-wide facet test) */
    uint64_t dead_leaves;    /* of which inside cell-dead subtrees (singular count only) */
    int32_t relifts;         /* re-lift attempts used                                */
    int32_t consistent;      /* 0 if b^{Q_0} != 1                                    */
    int32_t singular_complete; /* 1 unless BDEG_FLAG_DEGREE_ONLY                      */
    uint64_t seed_used;      /* seed of the lifting that produced the result         */
    uint64_t total_candidates; /* C(N,K)                                             */
    double plan_ms, kernel_ms, total_ms;
    uint64_t wide_reruns;    /* items re-run in the int128-value tier after leaving int64 */
    int32_t dead_full;       /* 1: the planner sampled a degenerate configuration (>= 25 % singular
                                K-subsets) and full mode detects cell-dead subtrees,
                                whose leaves then only count singular candidates */
} bdeg_result;

#define BDEG_NSLOTS 16       /* int64 partial-result slots combined by one all-reduce(SUM) */

/* Fill *o with the defaults listed above. */
void bdeg_default_options(bdeg_options *o);

/* Front end + planner (CPU) for x^A = b.  Copies the inputs.  Returns
 * BDEG_E_INCONSISTENT for an empty solution set, BDEG_E_TOO_LARGE when the
 * point configuration exceeds N <= 128, K <= 32 (N > 64: the walk only), a
 * coordinate or lifting reaches 2^62, or Hadamard's bound on the lifted
 * minors reaches 2^125 (beyond the int128 tier), BDEG_E_INVALID on bad
 * shapes.  d = 0 plans are valid (degree 1, no device work). */
bdeg_status bdeg_plan(const bdeg_problem *prob, const bdeg_options *opt, bdeg_plan_t *out);

/* Plan directly on a lifted vector configuration: K-vectors V (N*K,
 * POINT-major, V[l*K + t]) with lifting (N values, or NULL => generated).
 * Cells are K-subsets sigma with sign det[[V_sig, v_l],[w_sig, w_l]] =
 * sign det V_sig for every other l (lower facets of the lifted cone).  For an
 * affine point set a_l in Z^{K-1} pass v_l = (1, a_l). */
bdeg_status bdeg_plan_points(int32_t K, int32_t N, const int64_t *V, const int64_t *lifting,
                             const bdeg_options *opt, bdeg_plan_t *out);

/* Front-end fields of the result (no device work). */
bdeg_status bdeg_plan_info(bdeg_plan_t plan, bdeg_result *out);

/* The lifted configuration the plan currently enumerates (host copies): V
 * (N*K int64, POINT-major, in the plan's point order — system plans: the
 * distinct non-zero columns of P_0 and, unless homogeneous, the origin
 * (Prop. 4), sorted by ascending lifting residual (or in variable order with
 * BDEG_FLAG_NATURAL_ORDER); point plans: the caller's order.  Colex ranks,
 * work items and cell masks refer to this order) and omega (N int64: the lifting in use after any
 * bdeg_relift, and for N > 64 the basis-seeded lifting).  Either
 * pointer may be NULL.  BDEG_E_INVALID for a d = 0 plan (no points). */
bdeg_status bdeg_plan_points_get(bdeg_plan_t plan, int64_t *V, int64_t *omega);

/* Device workspace: bytes needed, and an optional caller-owned device buffer
 * (e.g. a torch.uint8 CUDA tensor) that must outlive the plan's device work.
 * Without it the plan allocates with cudaMalloc on first use. */
size_t bdeg_workspace_bytes(bdeg_plan_t plan);
bdeg_status bdeg_set_workspace(bdeg_plan_t plan, void *d_ptr, size_t bytes);

/* Whole rank space on one GPU, synchronous (returns after the D2H read of
 * the result).  Handles overflow re-runs and, for generated liftings,
 * re-lifts on degeneracy.  BDEG_E_DEGENERATE for a degenerate user lifting. */
bdeg_status bdeg_degree(bdeg_plan_t plan, bdeg_result *out);

/* Same over the colex ranks [begin, end) of K-subsets (rank = sum_i
 * C(c_i, i+1), c_0 < ... < c_{K-1}); no re-lift (ties are reported). */
bdeg_status bdeg_degree_range(bdeg_plan_t plan, uint64_t begin, uint64_t end, bdeg_result *out);

/* Work decomposition of the rank space (host only).  Item i is
 * the i-th position of the plan's work queue: a tuple of the largest subset
 * indices whose candidates are the contiguous colex ranks [*begin, *end).
 * Items partition [0, C(N,K)) and are listed largest-first: with world > 1,
 * base-depth items larger than a quarter of a warp's share (C(N,K) / (world
 * x SMs x resident warps)) are split one or more levels deeper.  Sharding
 * rule of bdeg_degree_partial: rank r of world W takes the positions
 * r, r + W, r + 2W, ... below n_static; the positions from n_static on are
 * taken from the cross-GPU stealing counter (bdeg_steal_attach), `grab` per
 * atomic, or, without it, by the same interleave (n_static = num_items). */
uint64_t bdeg_num_items(bdeg_plan_t plan);
bdeg_status bdeg_item_range(bdeg_plan_t plan, uint64_t item, uint64_t *begin, uint64_t *end);
/* Queue shape: total positions, how many of them are split (finer-depth)
 * items (they come first, sorted by size), the static prefix and the tail
 * grab size.  Any pointer may be NULL. */
bdeg_status bdeg_queue_info(bdeg_plan_t plan, uint64_t *n_items, uint64_t *n_split, uint64_t *n_static,
                            uint64_t *grab);

/* Result slots (int64, summed by the all-reduce): [0..3] the degree as four
 * 32-bit limbs (value = sum_i slot[i] << 32i), [4] cells, [5] singular,
 * [6] candidates, [7] ties, [8] items re-run in tier 2, [9] values beyond
 * the int128 tier (fatal), [10] unused (0), [11] items, [12] updates,
 * [13] leaves, [14] dead leaves, [15] items re-run in the int128 tier. */

/* This process's shard (options.rank of options.world) accumulated into the
 * caller's DEVICE buffer d_slots (BDEG_NSLOTS int64, zeroed here), async on
 * the stream.  Combine with one all-reduce(SUM) and call bdeg_finalize. */
bdeg_status bdeg_degree_partial(bdeg_plan_t plan, int64_t *d_slots);

/* cell emission: the cells of the subdivision among the colex
 * ranks [begin, end), as (mask, |det|) pairs into h_out (HOST, 2*capacity
 * uint64): bit l of mask = point l (bdeg_plan_info's point order).  *count =
 * cells found (may exceed capacity; only capacity pairs are written). */
bdeg_status bdeg_cells(bdeg_plan_t plan, uint64_t begin, uint64_t end, uint64_t *h_out, uint64_t capacity,
                       uint64_t *count);

/* The lifted hyperplane of a cell (host): h with h . v_c = omega_c for the K
 * points c of the cell, returned as h = h_num / den (h_num: K int64, den =
 * +-det V_sigma).  In the paper's notation the cell's
 * inner normal is alpha^ = (alpha, 1) with, for the generic formulation
 * v = (1, a): h = (<a^_0, alpha^>, -alpha).  BDEG_E_TOO_LARGE beyond int64. */
bdeg_status bdeg_cell_normal(bdeg_plan_t plan, uint64_t mask_lo, uint64_t mask_hi, int64_t *h_num, int64_t *den);

/* output-sensitive degree: walk the regular subdivision cell to
 * cell across ridges (the paper's pivoting, and its graph view,
 * P:1068-1132), each pivot an exact warp-wide ridge test, cells deduplicated
 * in a device hash set, volumes summed exactly.  Work ~ cells x K
 * instead of C(N,K).  Result: degree and cells exact (same subdivision as
 * bdeg_degree for the same lifting); candidates/singular are not enumerated
 * (singular_complete = 0); leaves = ridge tests, dead_leaves = boundary ridges.
 * Re-lifts generated liftings on ties like bdeg_degree.
 * Memory: device buffers allocated by the call itself (cudaMalloc, freed on
 * return) — a hash set of 16-byte cell masks + 1-byte level tags that holds
 * only the breadth-first window of levels L-1..L+1 (adjacent cells' levels
 * differ by <= 1), plus two frontier buffers; it grows to the free device
 * memory and fails with BDEG_E_TOO_LARGE when two consecutive levels no
 * longer fit.  N <= 128 points (N > 64 needs a generated lifting: the start
 * cell is a basis lifted at 0).  Tier-0 plans use int32 working storage
 * (cells whose values leave int32 are redone in int64, exact either way). */
bdeg_status bdeg_degree_walk(bdeg_plan_t plan, bdeg_result *out);

/* the walk with its hash set SHARDED over the ranks (the
 * paper's KnownNodes table shared by its GPUs, rebuilt as
 * owner-computes over NVLink): cell m is owned by rank hash(m) mod world
 * (options.rank / options.world of the plan); each rank keeps only its cells
 * (breadth-first window of levels L-1..L+1), expands its frontier, and the
 * neighbours owned elsewhere are exchanged after every level by one
 * all-to-all; volumes are summed by the owner and combined by one all-reduce.
 * Every rank calls it with the same plan (same lifting) and a bdeg_comm whose
 * callbacks implement the collectives over the caller's process group:
 *   allreduce_sum(ctx, vals, n): host int64[n], SUM in place;
 *   alltoall_counts(ctx, send, recv): host uint64[world] each;
 *   alltoall_cells(ctx, d_send, send_counts, d_recv, recv_counts): DEVICE
 *     buffers of 16-byte cells, segment per rank, complete on return.
 * A callback returns 0 on success (else BDEG_E_COMM).  Ties abort every rank
 * (BDEG_E_DEGENERATE; generated liftings are re-lifted collectively). */
typedef struct {
    void *ctx;
    int (*allreduce_sum)(void *ctx, int64_t *vals, int32_t n);
    int (*alltoall_counts)(void *ctx, const uint64_t *send, uint64_t *recv);
    int (*alltoall_cells)(void *ctx, const void *d_send, const uint64_t *send_counts, void *d_recv,
                          const uint64_t *recv_counts);
} bdeg_comm;
bdeg_status bdeg_degree_walk_sharded(bdeg_plan_t plan, const bdeg_comm *comm, bdeg_result *out);

/* Cross-GPU dynamic work stealing.  One process (rank 0)
 * creates a pair of tail counters in its GPU's memory and exports them as a
 * CUDA IPC handle (BDEG_STEAL_HANDLE_BYTES bytes); every rank (rank 0 included,
 * via the same handle in another process, or its own) attaches them to its
 * plan.  bdeg_degree_partial then takes its static interleaved share of the
 * queue's first n_static positions (bdeg_queue_info) and the remaining
 * positions from the ONE global counter, `grab` per system-scope atomic over
 * NVLink; the counters alternate by step parity and rank 0's launch zeroes
 * the idle one, so all ranks must call bdeg_degree_partial once per step,
 * separated by the result all-reduce (which orders the steps). */
#define BDEG_STEAL_HANDLE_BYTES 64
bdeg_status bdeg_steal_create(int32_t device, uint8_t *out_handle);
bdeg_status bdeg_steal_attach(bdeg_plan_t plan, const uint8_t *handle);

/* front end at scale (no plan needed).  Rank of A (n x m,
 * ROW-major int64) modulo a prime < 2^31 by GPU Gaussian row reduction (the
 * paper's GPU row reduction; one cooperative kernel, no host
 * round trip per column).  rank_p(A) <= rank_Q(A), equal
 * unless p divides every maximal non-zero minor.  bdeg_dimension_modp returns
 * n - max(rank_p) over the primes 2^31-1 and 2^31-19 (probabilistic, pinned by
 * the paper's Tables 1-2; the exact dimension comes from bdeg_plan's SNF). */
bdeg_status bdeg_rank_modp(int32_t n, int32_t m, const int64_t *A, uint32_t prime, int32_t device, void *stream,
                           int64_t *rank);
bdeg_status bdeg_dimension_modp(int32_t n, int32_t m, const int64_t *A, int32_t device, int32_t *dim);

/* EXACT rank and component count at scale (no plan needed).
 * One cooperative GPU kernel eliminates A (n x m, ROW-major int64) over Z
 * with unit pivots only (+-1 entries: each is an invariant factor 1 of the
 * Smith form); the rows never used x the columns left without a
 * unit pivot form a residual block whose Smith form the host finishes
 * exactly (Euclidean, checked int128).  Returns rank A (dimension n - rank,
 * Prop. 1), |prod d_j| (the number of components) as two 64-bit
 * halves, and how many unit pivots the GPU found.  BDEG_E_TOO_LARGE when an
 * entry would pass 2^61 or the residual exceeds 4e6 entries. */
bdeg_status bdeg_smith_gpu(int32_t n, int32_t m, const int64_t *A, int32_t device, void *stream, int64_t *rank,
                           uint64_t *comp_lo, uint64_t *comp_hi, int64_t *unit_pivots);

/* Carry-normalise summed slots (HOST memory) into *out. */
bdeg_status bdeg_finalize(bdeg_plan_t plan, const int64_t *h_slots, bdeg_result *out);

/* Replace a generated lifting with the one for re-lift attempt `attempt`
 * (seed derived from options.seed); BDEG_E_INVALID for a user lifting. */
bdeg_status bdeg_relift(bdeg_plan_t plan, int32_t attempt);

const char *bdeg_last_error(bdeg_plan_t plan);
const char *bdeg_status_str(bdeg_status s);
void bdeg_destroy(bdeg_plan_t plan);

/* Number of kernels this process has launched through libbdeg (evidence for
 * bench.py's gpu_launches). */
uint64_t bdeg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* BDEG_H */
