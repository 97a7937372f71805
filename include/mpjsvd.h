/*
 * mpjsvd.h -- C-ABI of the B200-native mixed-precision one-sided Jacobi SVD.
 *
 * Computes the full SVD A = U * diag(S) * V^T of a dense real m x n fp64
 * matrix with m >= n (Alg. 3 "Require A ... with m >= n,
 * Ensure the full singular value decomposition A = U Sigma V^*"), by the
 * paper's four stages:
 *   (1) preconditioning: [m > n] Householder QR A = Q_tall R1,
 *       column-pivoted QR A1 P = Q_p R, LQ R = L Q_2 and
 *       X = L (reading c-7);
 *   (2) fp32 one-sided block Jacobi on fl32(X 2^-e) computing U_low only
 *       (Alg. 1) -- or, under
 *       path = AUTO, the gates of Alg. 3 and possibly the fp32 QR SVD
 *       (DESIGN.md c-15, c-24);
 *   (3) precision switch (U-route, the paper's Alg. 3 l.446-447): Q from the
 *       Householder QR of X^T working(U_low), Y = X Q (
 *       DESIGN.md c-11; switch_u = 0 selects the V-route CholeskyQR of V32);
 *   (4) fp64 one-sided block Jacobi on (Y, V := Q) to eps_tol (or the sec. 3.4
 *       V formation, refine_v = 1, DESIGN.md c-23), then sigma_j = ||y_j||,
 *       U_X = Y diag(1/sigma), descending sort;
 * and assembles U = Q_tall Q_p U_X, V = P Q_t V_X.
 *
 * Conventions (all entry points):
 *   - Matrices are column-major fp64.  A is m x n with leading dimension lda,
 *     U is m x n (ldu), S has n entries (descending, > 0), V is n x n (ldv).
 *   - Pointers may be DEVICE pointers on the handle's device (the fast path;
 *     nothing crosses PCIe) or HOST pointers (pageable or pinned): the library
 *     detects host memory with cudaPointerGetAttributes and stages it through
 *     device buffers inside the call (that is the end-to-end path bench.py
 *     times).  A may not alias U, S or V.
 *   - Ownership: the caller owns A (never modified), U, S and V.  The handle
 *     owns every device workspace, stream event and NCCL object; they are
 *     freed by mpjsvd_destroy.  Workspaces are (re)allocated on the first call
 *     for a given (m, n) and reused after that.
 *   - Threading: one mpjsvd_factor at a time per handle; distinct handles may
 *     be used concurrently from different host threads.
 *   - The call is stream-ordered on options.stream (NULL: a stream owned by
 *     the handle) and synchronises the host once per Jacobi sweep (16-byte
 *     convergence read-back) and once at exit.
 *   - No C++ exception, abort or exit crosses this boundary.  Errors are
 *     negative return codes; mpjsvd_strerror() maps any code to a static
 *     string.
 */
#ifndef MPJSVD_H
#define MPJSVD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPJSVD_VERSION 150   /* 1.5: option l2_order */
#define MPJSVD_COMM_ID_BYTES 128

/* return codes */
#define MPJSVD_OK 0
#define MPJSVD_WARN_NOT_CONVERGED 1   /* outputs filled; fp64 stage hit max_sweeps64 */
#define MPJSVD_ERR_INVALID_ARG (-1)   /* null pointer, m < n, n < 2, lda < m, ldu < m, ldv < n, bad option */
#define MPJSVD_ERR_NONFINITE (-2)     /* A contains NaN or Inf */
#define MPJSVD_ERR_RANK_DEFICIENT (-3)/* zero R diagonal / zero column / singular V^T V */
#define MPJSVD_ERR_CUDA (-4)          /* CUDA runtime error (see mpjsvd_last_cuda_error) */
#define MPJSVD_ERR_NCCL (-5)          /* NCCL missing or failed (see mpjsvd_last_cuda_error) */
#define MPJSVD_ERR_OUT_OF_MEMORY (-6)
#define MPJSVD_ERR_NOT_SUPPORTED (-7) /* e.g. num_gpus != 1, block_cols unsupported, n > 8192, m > 16384 */
#define MPJSVD_ERR_BREAKDOWN (-8)     /* finite input, non-finite intermediate (fp32 stage overflow, switch) */

/* path (Alg. 3 gates; reading c-15) */
#define MPJSVD_PATH_FORCE_MIXED 0     /* always run the fp32 Jacobi stage (default) */
#define MPJSVD_PATH_AUTO 1            /* Alg. 3 gates decide (DESIGN.md c-15):
                                         cond gate -> tail gate -> orth gate -> fp32 Jacobi if orth <= tol_alg,
                                         else the fp32 QR-SVD branch */
#define MPJSVD_PATH_FORCE_FP64 2      /* skip the fp32 stage: Q = I, Y = X */

/* stats.path_taken: 0 fp32 Jacobi (forced or AUTO), 2 fp64 only (forced), and under AUTO:
   3 fp64 only (cond gate: scaled cond(R) <= tol_cond and cond(D) > cond_d_min),
   4 fp64 only (tail gate: >= tail_frac n columns of X below 2^tail_cut_log2 max),
   5 fp64 only (orth gate: ||X_t^T X_t - I||_max <= tol_orth),
   6 fp32 QR-SVD (orth > tol_alg) */
#define MPJSVD_TAKEN_JACOBI 0
#define MPJSVD_TAKEN_FP64 2
#define MPJSVD_TAKEN_SKIP_COND 3
#define MPJSVD_TAKEN_SKIP_TAIL 4
#define MPJSVD_TAKEN_SKIP_ORTH 5
#define MPJSVD_TAKEN_QRSVD 6

typedef struct mpjsvd_handle_s* mpjsvd_handle;

typedef struct {
    int32_t num_gpus;          /* must be 1: one handle per process/GPU; multi-GPU via mpjsvd_comm_init */
    int32_t device_id;         /* CUDA device ordinal (default: current device) */
    int32_t block_cols;        /* b, columns per Jacobi block: 8, 16 or 32 (default 32) */
    double tol_mult32;         /* eps_tol32 = tol_mult32 * sqrt(n) * 2^-24 (default 4) */
    double tol_mult64;         /* eps_tol64 = tol_mult64 * sqrt(n) * 2^-53 (default 4) */
    int32_t inner_tol_div;     /* 2b x 2b inner solve runs to eps_tol / inner_tol_div (default 8) */
    int32_t max_sweeps32;      /* default 20 (+ stagnation exit, reading c-10) */
    int32_t max_sweeps64;      /* default 30 */
    int32_t max_inner;         /* inner sweeps cap (default 30) */
    int32_t path;              /* MPJSVD_PATH_* (default FORCE_MIXED) */
    int32_t x_from_lq;         /* 1 (default): X = L; 0: X = R (ablation) */
    int32_t compute_gates;     /* 1 (default): report orth / tail / cond measures */
    void* stream;              /* cudaStream_t on device_id, or NULL */
    int32_t virtual_shards;    /* G >= 1 (default 1): run the sharded Jacobi engine with G shards
                                  emulated on this one GPU -- shard buffers, per-round block
                                  exchange as device copies, one kernel over all shards' pairs
                                  (the multi-GPU data path, testable on one device) */
    int32_t split_rows;        /* > 0: rows per Gram row-split (fixes the fp summation order across
                                  shard counts); 0 (default): chosen per launch for SM fill */
    int32_t fp32_tensor_cores; /* 1 (default): the fp32 stage's Gram and update products (b = 32) run on
                                  the tcgen05 TF32 tensor cores with a hi/lo split (~2^-21 relative per
                                  product, fp32 accumulation; reading c-20); 0: FFMA SIMT */
    int32_t pdl_overlap;       /* 1 (default): the Jacobi update (fp64 DMMA; fp32 with fp32_tensor_cores) is a persistent kernel
                                  launched as a programmatic dependent of the inner solve and drains the
                                  pairs in the order their solves finish (overlaps the solve's tail) */
    int32_t mp_rrqr;           /* 1: mixed-precision RRQR (Alg. 4): the column permutation
                                  from an fp32 QRP of fl32(A1 2^-e), then fp64 Householder QR of A1 P;
                                  0 (default): fp64 column-pivoted QR (Businger-Golub).  On B200 the fp32
                                  QRP costs about as much as the fp64 one (reading c-22) */
    int32_t max_inner32;       /* inner sweeps cap of the fp32 stage's 2b x 2b solves (default 1; the fp64
                                  stage uses max_inner); reading c-5 */
    int32_t switch_u;          /* 1 (default): U-route precision switch, the paper's Alg. 3 choice (PAPER.md:446-447,
                                  542-545, 563-573): the fp32 stage does not accumulate V; Q = qr(X^T working(U_low))
                                  by fp64 Householder QR (diag(R2) >= 0).  0: V-route, the fp32 stage accumulates V32
                                  and Q = qr(fl64(V32)) by CholeskyQR (reading c-11) */
    /* AUTO gates (path = MPJSVD_PATH_AUTO; reading c-15) */
    double tol_orth;           /* orth gate, default 1e-5 (PAPER.md:643-644 footnote) */
    double tol_alg;            /* Jacobi if orth <= tol_alg, else the fp32 QR-SVD branch; default +inf */
    double tol_cond_mult;      /* tol_cond = tol_cond_mult * n^(1/4) ("O(n^{1/4})"), default 1 */
    double cond_d_min;         /* "condition number of D extremely large": max/min column norm > this, default 1e15 */
    double tail_frac;          /* tail gate: at least ceil(tail_frac n) small columns, default 1/3 */
    int32_t tail_cut_log2;     /* "small": ||x_j|| < 2^tail_cut_log2 max_j ||x_j||, default -60 */
    /* kernel-variant switches (defaults = the measured best; the alternatives are kept for the
       bitwise-equality tests and for experiments) */
    int32_t gram_tma;          /* fp32 tcgen05 Gram operand loads: 2 (default) TMA 2-D boxes into 128-byte-swizzled
                                  operands; 1 TMA 4-D boxes into the SWIZZLE_NONE canonical layout (round 1);
                                  0 cp.async.  All three issue the same MMAs (bitwise equal on equal row slabs) */
    int32_t gram_kt;           /* rows per TMA Gram stage: 0 (default) auto (32 for >= 6144 rows, else 64), 32, 64 */
    int32_t gram_variant;      /* Gram stage variant: with gram_tma = 0 the cp.async variant 0..5; with gram_tma = 1:
                                  8 / 9 warp-specialised; 10..13 the swizzled kernel with 3 / 4 / 6 / 8 stages, 14 / 15
                                  with 256 threads, 16 / 17 warp-specialised swizzled kernel with 4 / 6 stages, 18 / 19
                                  the same with the A operand [H ; L] in tensor memory (8 / 6 stages of raw columns
                                  only), 20..26 measured shapes of 18 (2 CTAs/SM with 6 A buffers, refill lag, two
                                  conversion warp groups); 0 (default): 18.  10..26 are bitwise
                                  equal on equal row slabs */
    int32_t update_tpc;        /* tiles per work item of the overlapped fp32 update; 0 (default): ~3 items per SM */
    int32_t skip_unchanged;    /* 1 (default): skip the Gram and solve of a pair whose blocks did not rotate since
                                  its previous evaluation (exact); 0: evaluate every pair */
    int32_t qr_panel_mode;     /* blocked Householder QR panels: 0 (default) flag-chained with look-ahead,
                                  1 cooperative grid-barrier kernel, 2 flag-chained without look-ahead */
    int32_t diag_timing;       /* diagnostics to stderr, bit mask: 1 QRP phases, 2 fp32/fp64 solve phases,
                                  4 cp.async Gram phases, 8 batched inner-solve phases (default 0) */
    int32_t refine_v;          /* V of the fp64 refinement: 0 (default) accumulate rotations from V := Q (reading c-12);
                                  1: PAPER.md:599-615 (sec. 3.4, reading c-23): refine Y without V, U_X = Y diag(1/||y_j||),
                                  V_X = qr(X^T U_X) by fp64 Householder QR, then one accumulating refinement from
                                  (X V_X, V := V_X) ("always converges in one sweep") */
    int32_t update_variant;    /* fp32 tcgen05 update: 1 (default) A operand (W hi/lo) in tensor memory (tcgen05.mma
                                  A-from-TMEM, double buffered; C5 fp32 stage 569 -> 534 ms); 0 in shared memory
                                  (round 1).  Bitwise equal */
    int32_t qrp_panel_stages;  /* column-pivoted QR end-of-panel update: -1 (default) auto (a per-thread cp.async ring of
                                  2 stages when it fits in shared memory), 0 register path (round 1), 2..4 forced.
                                  Bitwise equal */
    int32_t gram_pdl;          /* 1 (default): each Jacobi round's solve is a programmatic dependent of its Gram and
                                  starts a pair as soon as that pair's row-slab partials are counted (per-pair counters),
                                  overlapping the Gram's last wave; 0: the solve waits for the whole Gram.  Bitwise
                                  equal */
    int32_t l2_order;          /* fp32 tcgen05 stage, L2-aware traversal (experiment switch): the Gram CTAs take
                                  interleaved 32-row tiles (all pairs walk the rows top -> bottom in step) and the
                                  update claims its tile groups bottom group first, so each kernel starts on the rows
                                  the previous one touched last.  0 (default) off: contiguous row slabs, pair-major
                                  update (measured on B200: no gain at C5); 1 on; -1 on when fp32 X
                                  exceeds 96 MB and split_rows = 0.  The interleaved Gram sums its row-slab partials
                                  over different row sets: results differ from 0 in rounding only (same parity bar) */
} mpjsvd_options;

typedef struct {
    int32_t path_taken;        /* MPJSVD_TAKEN_*: 0 fp32 Jacobi, 2 fp64 only (forced), 3/4/5 fp64 only by the AUTO
                                  cond / tail / orth gate, 6 fp32 QR SVD (AUTO, orth > tol_alg) */
    int32_t sweeps32, sweeps64, converged;
    double stage_ms[8];        /* qr_tall, qrp, lq, gates, fp32, lift, fp64, assemble (CUDA events) */
    double total_ms;           /* device time from entry to outputs written */
    double orth_measure;       /* ||X_t^T X_t - I||_max, X_t = fl32(X) D^-1 */
    double tail_fraction;      /* fraction of columns of X with norm < 2^-60 max */
    double cond_estimate;      /* max_k R_kk / min_k R_kk */
    double final_off32, final_off64;
    double off_trace32[32], off_trace64[32];   /* per-sweep max normalised off-diagonal */
    int32_t upd_trace32[32], upd_trace64[32];  /* per-sweep number of updated block pairs */
    int64_t kernel_launches;   /* kernels launched by this call */
    int32_t inner_max_trace32[32], inner_max_trace64[32];  /* per sweep: most inner sweeps of one pair */
    int32_t inner_sum_trace32[32], inner_sum_trace64[32];  /* per sweep: inner sweeps summed over pairs */
    int32_t skip_trace32[32], skip_trace64[32];  /* per sweep: pairs whose Gram and solve were skipped because
                                                    neither block rotated since their previous evaluation
                                                    (exact: same Gram, same metric, no rotation) */
    double cond_scaled;        /* kappa_1(R diag(1/c)), c_k = ||A1(:, perm_k)|| = ||R(:,k)||: the column-scaled
                                  cond_R of the AUTO cond gate (Alg. 3 l.423; DESIGN.md c-15); NaN unless AUTO */
    double cond_d;             /* max_j ||A1(:,j)|| / min_j ||A1(:,j)|| (cond(D) of A = B D); NaN unless AUTO */
    int32_t v_sweeps64;        /* fp64 sweeps that accumulated V (the last v_sweeps64 of sweeps64; < sweeps64 only with
                                  refine_v = 1) */
} mpjsvd_stats;

/* Fill *opts with the defaults above. */
void mpjsvd_default_options(mpjsvd_options* opts);

/* Create a handle bound to opts->device_id (opts may be NULL: defaults).
   Returns 0 or a negative error code; *h is NULL on error. */
int mpjsvd_create(mpjsvd_handle* h, const mpjsvd_options* opts);

/* The SVD.  See the conventions above.  stats may be NULL.  Sizes: n <= 8192 (the column-pivoted QR keeps the
   n-row pivot column in shared memory and 16 rows per thread in registers), m <= 16384 (m > n: a Householder QR
   first); larger sizes return MPJSVD_ERR_NOT_SUPPORTED before any work. */
int mpjsvd_factor(mpjsvd_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                  double* U, int64_t ldu, double* S, double* V, int64_t ldv,
                  mpjsvd_stats* stats);

/* Free every resource of the handle.  Safe on NULL. */
int mpjsvd_destroy(mpjsvd_handle h);

/* Static description of a return code. */
const char* mpjsvd_strerror(int code);

/* Last CUDA error string recorded by the library (static storage). */
const char* mpjsvd_last_cuda_error(void);

int mpjsvd_version(void);

/* ------------------------------------------------------------------------
 * Multi-GPU: one process per GPU,
 * each with its own handle.  Rank 0 calls mpjsvd_comm_unique_id and hands
 * the MPJSVD_COMM_ID_BYTES bytes to every rank (e.g. a torch.distributed
 * broadcast); every rank then calls mpjsvd_comm_init with its rank and the
 * world size (this creates the handle's NCCL communicator; NCCL is loaded
 * with dlopen, MPJSVD_ERR_NCCL if unavailable).  Afterwards every rank calls
 * mpjsvd_factor with the same m and n (checked: MPJSVD_ERR_INVALID_ARG on all
 * ranks otherwise): rank 0 passes A, U, S, V; the others may pass NULL for
 * all four (their ld arguments are ignored).  Preconditioning, lift and
 * assembly run on rank 0; both Jacobi stages run sharded: rank g holds the
 * column blocks of k = M/(2G) pairs and exchanges <= 2 blocks with its
 * neighbours after every round (ncclSend/ncclRecv), with one max/sum
 * all-reduce of the convergence counters per sweep.  The block count M is
 * padded to a multiple of 2G with empty blocks.  Outputs are written on
 * rank 0 only; the sweep statistics on every rank.  Collective: every rank
 * must make the same sequence of calls.
 * ------------------------------------------------------------------------ */
int mpjsvd_comm_unique_id(uint8_t* id /* MPJSVD_COMM_ID_BYTES */);
int mpjsvd_comm_init(mpjsvd_handle h, int32_t rank, int32_t world, const uint8_t* id);
/* rank / world size of the handle (0 / 1 without a communicator) */
int mpjsvd_comm_info(mpjsvd_handle h, int32_t* rank, int32_t* world);

/* The shard plan (host only, no GPU needed): the schedule and the block
 * exchanges the sharded engine performs, exported so that tests can drive
 * the same exchange logic over another transport.  nblk column blocks over
 * `world` ranks (world = 1: the single-GPU layout, buffer j = block j).
 *   plan_info:    M positions (padded), k pairs per rank, nbuf buffers per rank
 *   plan_pairs:   out[4t..4t+3] = (buf0, buf1, blk0, blk1) of rank's local
 *                 pair t in the current round (blk0 < blk1; blk >= nblk is
 *                 an empty bye block); returns k
 *   plan_advance: apply one round's shift; writes up to cap inter-rank moves
 *                 (blk, src_rank, src_buf, dst_rank, dst_buf), 5 int32 each,
 *                 in the canonical order every rank posts them; returns the
 *                 move count
 *   plan_locate:  current (rank, buffer) of block blk                     */
typedef struct mpjsvd_plan_s* mpjsvd_plan;
int mpjsvd_plan_create(mpjsvd_plan* plan, int32_t nblk, int32_t world);
int mpjsvd_plan_info(mpjsvd_plan plan, int32_t* M, int32_t* k, int32_t* nbuf);
int mpjsvd_plan_pairs(mpjsvd_plan plan, int32_t rank, int32_t* out);
int mpjsvd_plan_advance(mpjsvd_plan plan, int32_t* moves, int32_t cap);
int mpjsvd_plan_locate(mpjsvd_plan plan, int32_t blk, int32_t* rank, int32_t* buf);
int mpjsvd_plan_destroy(mpjsvd_plan plan);

/* Per-kernel timing for benchmarking.  mpjsvd_set_profiling(h, 1) clears the
   accumulators and brackets every subsequent kernel launch of the Jacobi
   rounds (pair_gram / pair_solve / pair_update, fp32 and fp64) and each
   stage-level launch group (qrp_coop, lq_coop, qr_coop_tall, gates_orth,
   lift_cholqr, rv_gemm, assemble_wy) with CUDA events on the handle's
   stream; mpjsvd_get_profile(h, idx, ...) returns the number of entries and
   fills entry idx (name, summed device ms, launch count).  idx < 0: count
   only.  Profiling adds two event records per launch and no synchronisation. */
int mpjsvd_set_profiling(mpjsvd_handle h, int32_t on);
int mpjsvd_get_profile(mpjsvd_handle h, int32_t idx, char* name, int32_t name_len, double* total_ms,
                       int64_t* launches);

/* ------------------------------------------------------------------------
 * Step-level entry points (used by the parity tests to compare one step of
 * the path with the oracle's same step).  Same conventions: column-major,
 * device or host pointers, stream-ordered on the handle's stream.
 * Unlike mpjsvd_factor, these take DEVICE pointers only.
 * ------------------------------------------------------------------------ */

/* One-sided block round-robin Jacobi in fp64 on X (m x n, ldx), accumulating
   into V (nv x n, ldv; may be NULL) -- the refinement stage (PAPER.md:452-454,
   575-597) run on an injected X.  tol / tol_in as in the options.  Returns
   sweeps (> 0 converged, < 0 not converged) through *sweeps and the traces
   through stats (sweeps64, off_trace64, upd_trace64). */
int mpjsvd_block_jacobi_f64(mpjsvd_handle h, double* X, int64_t m, int64_t n, int64_t ldx,
                            double* V, int64_t nv, int64_t ldv, double tol, double tol_in,
                            int32_t max_sweeps, int32_t* sweeps, mpjsvd_stats* stats);

/* Same in fp32 (the low-precision stage), with the
   stagnation exit of reading c-10 when `stagnation` != 0. */
int mpjsvd_block_jacobi_f32(mpjsvd_handle h, float* X, int64_t m, int64_t n, int64_t ldx,
                            float* V, int64_t nv, int64_t ldv, float tol, float tol_in,
                            int32_t max_sweeps, int32_t stagnation, int32_t* sweeps,
                            mpjsvd_stats* stats);

/* Inner 2b x 2b solve on `count` independent symmetric matrices G (w x w
   each, packed back to back, ld = w): two-sided round-robin Jacobi to
   tol_in (reading c-5); on exit G holds the rotated matrix and E = V_blk - I.
   fp64 when is_f64 != 0 (double*), else fp32 (float*).  w <= 64. */
int mpjsvd_inner_solve(mpjsvd_handle h, int32_t is_f64, void* G, void* E, int32_t w, int32_t count,
                       double tol_in, int32_t max_inner, int32_t* rotations);

/* Column-pivoted Householder QR A P = Q R in place (n x n or m x n, lda):
   on exit R in the upper triangle (diag >= 0), reflectors below, tau[n],
   perm[n] (0-based original column at position k).  pivot = 0: plain QR
   (perm = identity); 1: fp64 QRP (lazy cooperative kernel); 2: fp64 QRP
   (unblocked kernel); 3: mixed-precision RRQR, Alg. 4 (fp32 QRP pivots of
   fl32(A 2^-e), then fp64 QR of A P).  PAPER.md:332-335 / 416-420 / 496-512. */
int mpjsvd_qr(mpjsvd_handle h, double* A, int64_t m, int64_t n, int64_t lda, double* tau,
              int32_t* perm, int32_t pivot);

/* Precision lift: Q = V * Rv^-1, Rv = chol(V^T V),
   V = fl64(V32) (n x n, ldv32 / ldq). */
int mpjsvd_lift(mpjsvd_handle h, const float* V32, int64_t n, int64_t ldv32, double* Q, int64_t ldq);

/* U-route precision switch (Alg. 3 l.446-447): Z = X^T Ulow in fp64, Householder QR
   Z = Q R2 with diag(R2) >= 0, Q = H_0 ... H_{n-1} I written to Q.  X, Ulow, Q are n x n column-major
   fp64 (ldx, ldu, ldq >= n), device or host pointers (copied through handle workspaces; X and Ulow are
   not modified).  x_lower != 0 declares X lower triangular (its upper part is then not read).  In exact
   arithmetic Q = V_X when X = U_X S V_X^T and Ulow = U_X.  Errors: INVALID_ARG (null, n < 1, ld < n),
   CUDA, OUT_OF_MEMORY. */
int mpjsvd_switch_u(mpjsvd_handle h, const double* X, int64_t n, int64_t ldx, const double* Ulow, int64_t ldu,
                    double* Q, int64_t ldq, int32_t x_lower);

/* Step-level: the fp32 QR SVD of the AUTO branch ("QR SVD algorithm in the
   lower precision ... without generating V_low"; reading c-24): fp32 Householder bidiagonalisation,
   fp32 implicit-shift QR on the bidiagonal, left rotations and reflectors accumulated in fp64.  X32: n x n
   fp32 (ldx >= n, device or host; not modified).  U: n x n fp64 (ldu >= n) receives U_low, columns in
   descending singular value order; S (n floats, may be NULL) the singular values.  Errors: INVALID_ARG,
   RANK_DEFICIENT (an exact zero singular value), CUDA (incl. no convergence in 6 n^2 QR steps),
   OUT_OF_MEMORY, NOT_SUPPORTED (n > 16384). */
int mpjsvd_qrsvd32(mpjsvd_handle h, const float* X32, int64_t n, int64_t ldx, double* U, int64_t ldu, float* S);

/* C <- Q C with Q = H_0 ... H_{k-1} packed as returned by mpjsvd_qr (rows m). */
int mpjsvd_apply_q(mpjsvd_handle h, const double* Vr, int64_t m, int64_t k, int64_t ldv,
                   const double* tau, double* C, int64_t ldc, int64_t ncols);

/* C = alpha op(A) op(B) + beta C, fp64, column-major (the library GEMM used by
   the lift, R*V product and assembly).  transa/transb: 0 = N, 1 = T. */
int mpjsvd_gemm_f64(mpjsvd_handle h, int32_t transa, int32_t transb, int64_t M, int64_t N, int64_t K,
                    double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                    double beta, double* C, int64_t ldc);

#ifdef __cplusplus
}
#endif
#endif
