/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, sequential CPU oracle for the mixed-precision one-sided Jacobi
 * SVD of arXiv 2209.04626 ("Mixed precision Jacobi SVD algorithm").  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code, header, table or
 * constant generator with the CUDA path (paper_2209_04626_b200/csrc).
 *
 * Two oracles:
 *   O-MIX  om_*  : Algorithm 3 step by step, with the
 *                  block round-robin ordering and every reading fixed in
 *                  DESIGN.md sec. "Readings".
 *   O-CYC  oc_*  : textbook Algorithm 1 in fp64 with the
 *                  row-cyclic order of eq. (2.1).
 *
 * All matrices are column-major.  Return codes: 0 ok, 1 not converged
 * (outputs filled), -1 invalid argument, -2 non-finite input, -3 rank
 * deficient.
 *
 * Parity pins: see tests/test_oracle_pins.py.  Every function below is
 * pinned by at least one test that does not re-type its formula.
 */
#ifndef MPJSVD_ORACLE_H
#define MPJSVD_ORACLE_H
#include <stdint.h>

#define OM_PATH_FORCE_MIXED 0
#define OM_PATH_AUTO 1
#define OM_PATH_FORCE_FP64 2
/* path_taken under AUTO (Alg. 3 gates; DESIGN.md c-15) */
#define OM_TAKEN_SKIP_COND 3
#define OM_TAKEN_SKIP_TAIL 4
#define OM_TAKEN_SKIP_ORTH 5
#define OM_TAKEN_QRSVD 6

typedef struct {
    int32_t b;              /* block width (columns per block) */
    double tol_mult32;      /* eps_tol = tol_mult * sqrt(n) * u  (reading c-1) */
    double tol_mult64;
    int32_t inner_tol_div;  /* inner solve threshold = eps_tol / inner_tol_div (c-5) */
    int32_t max_sweeps32;
    int32_t max_sweeps64;
    int32_t max_inner;      /* inner sweeps cap (c-5) */
    int32_t path;           /* OM_PATH_* */
    int32_t x_from_lq;      /* 1: X = L (default, F1); 0: X = R */
    int32_t nthreads;       /* OpenMP threads over disjoint pairs (0 = default) */
    int32_t mp_rrqr;        /* 1: mixed-precision RRQR, Alg. 4; 0 (default): fp64 QRP (c-22) */
    int32_t max_inner32;    /* inner sweeps cap of the fp32 stage (c-5; default 1) */
    int32_t switch_u;       /* 1: U-route switch (Alg. 3 l.446-447): the fp32 stage
                               does not accumulate V; Q = qr(X^T U_low) (default); 0: V-route (c-11) */
    double tol_orth, tol_alg, tol_cond_mult, cond_d_min, tail_frac;   /* AUTO gates (c-15) */
    int32_t tail_cut_log2;
    int32_t refine_v;       /* 0 (default): the fp64 refinement accumulates V from V := Q (c-12);
                               1: PAPER.md:599-615 (sec. 3.4, reading c-23): refine without V, V_X = qr(X^T U_X),
                               then one accumulating refinement from (X V_X, V := V_X) */
} om_opts;

typedef struct {
    int32_t sweeps32, sweeps64, converged, path_taken;
    double orth_measure, tail_fraction, cond_estimate;
    double final_off32, final_off64;
    double off_trace32[64], off_trace64[64];
    int32_t upd_trace32[64], upd_trace64[64];
    int32_t perm[1];        /* unused placeholder (keeps layout simple) */
    double cond_scaled;     /* kappa_1(R diag(1/||R(:,k)||)) (AUTO only, else NaN) */
    double cond_d;          /* max/min column norm of A1 (cond(D) of A = B D; AUTO only, else NaN) */
    int32_t v_sweeps64;     /* fp64 sweeps that accumulated V (the last v_sweeps64 of sweeps64) */
} om_stats;

/* The low-precision QR SVD of the AUTO branch (qrsvd.c, reading c-24):
   fp32 Householder bidiagonalisation + fp32 implicit-shift QR on the bidiagonal, left rotations and
   reflectors accumulated into U (n x n fp64, ldu; columns in descending singular value order); S the
   singular values (fp32, descending).  X32 (ldx) is not modified.  0 ok, 1 no convergence, -3 a zero
   diagonal of B (rank deficient). */
int om_qrsvd32(const float* X32, int64_t n, int64_t ldx, double* U, int64_t ldu, float* S);

void om_default_opts(om_opts* o);

/* --- building blocks (exported for step-level parity tests) ------------- */
/* Householder reflector of x[0..len-1] with beta = +||x|| >= 0 (c-13):
   on exit x[0] = beta, x[1..] = v[1..] (v[0] = 1 implicit), returns tau. */
double om_house(double* x, int64_t len);
/* Unpivoted Householder QR in place, diag(R) >= 0.  PAPER.md:416-420. */
int om_qr(double* A, int64_t m, int64_t n, int64_t lda, double* tau);
/* Businger-Golub column-pivoted QR (LAPACK xGEQP3 semantics, diag(R) >= 0,
   pivot = largest partial norm, ties -> lowest index).  PAPER.md:332-335. */
int om_qrp(double* A, int64_t m, int64_t n, int64_t lda, int32_t* perm, double* tau);
/* The same Businger-Golub QRP carried out entirely in fp32 (Alg. 4 line 2, "RRQR in a lower precision"). */
int om_qrp_f32(float* A, int64_t m, int64_t n, int64_t lda, int32_t* perm, float* tau);
/* Mixed-precision RRQR (Alg. 4) of the m x n A in place: P from om_qrp_f32 on
   fl32(A 2^-e) (e = frexp exponent of max|A|, reading c-9), then om_qr of A P. Same outputs as om_qrp. */
int om_mprrqr(double* A, int64_t m, int64_t n, int64_t lda, int32_t* perm, double* tau);
/* C <- Q*C with Q = H_0 H_1 ... H_{k-1} stored as in om_qr (rows m). */
void om_apply_q(const double* Vr, int64_t m, int64_t k, int64_t ldv, const double* tau,
                double* C, int64_t ldc, int64_t ncols);
/* 2b x 2b inner solve (c-5): two-sided round-robin Jacobi on symmetric G
   (w x w, full storage, ld = w), E = V_blk - I on exit (ld = w).
   Returns the number of rotations; *inner_sweeps receives the sweeps used. */
int64_t om_inner_solve_f64(double* G, int32_t w, double tol_in, int32_t max_inner,
                           double* E, int32_t* inner_sweeps);
int64_t om_inner_solve_f32(float* G, int32_t w, float tol_in, int32_t max_inner,
                           float* E, int32_t* inner_sweeps);
/* Block round-robin one-sided Jacobi (Alg. 1 in block form, c-4..c-6, c-10).
   X is m x n (ldx), V is nv x n (ldv) or NULL.  Returns sweeps (negative if
   not converged within max_sweeps).  off_trace/upd_trace may be NULL. */
int32_t om_block_jacobi_f64(double* X, int64_t m, int64_t n, int64_t ldx,
                            double* V, int64_t nv, int64_t ldv, int32_t b,
                            double tol, double tol_in, int32_t max_sweeps, int32_t max_inner,
                            double* off_trace, int32_t* upd_trace, int32_t nthreads);
int32_t om_block_jacobi_f32(float* X, int64_t m, int64_t n, int64_t ldx,
                            float* V, int64_t nv, int64_t ldv, int32_t b,
                            float tol, float tol_in, int32_t max_sweeps, int32_t max_inner,
                            int32_t stagnation,
                            double* off_trace, int32_t* upd_trace, int32_t nthreads);
/* Precision lift (c-11): Q = V * Rv^-1 with Rv = chol(V^T V), V = fl64(V32). */
int om_lift(const float* V32, int64_t n, int64_t ldv32, double* Q, int64_t ldq);

/* U-route precision switch (Alg. 3 l.446-447 "Q R2 = X^T working(U_low)"):
   Z = X^T Ulow in fp64, Householder QR Z = Q R2 with diag(R2) >= 0 (c-13), Q formed explicitly
   (Q = H_0 ... H_{n-1} I).  X, Ulow, Q n x n.  In exact arithmetic Q = V_X when X = U_X S V_X^T and
   Ulow = U_X.  Returns -3 when a diagonal of R2 is zero. */
int om_switch_u(const double* X, int64_t n, int64_t ldx, const double* Ulow, int64_t ldu,
                double* Q, int64_t ldq);

/* --- the whole method ------------------------------------------------- */
/* Gate measures of Alg. 3 (DESIGN.md c-15), on X n x n (ldx) / upper R:
   orth = ||X_t^T X_t - I||_max (fp32; work: n*n floats), tail = fraction of columns with norm below
   2^cut_log2 max, cond_scaled = kappa_1(R diag(1/c)), cond_d = max/min of cn[0..n). */
double om_gate_orth(const double* X, int64_t n, int64_t ldx, float* work);
double om_gate_tail(const double* X, int64_t n, int64_t ldx, int32_t cut_log2);
double om_gate_cond_scaled(const double* R, int64_t n, int64_t ldr, const double* c);
double om_gate_cond_d(const double* cn, int64_t n);
int om_mixed_svd(const double* A, int64_t m, int64_t n, int64_t lda, const om_opts* opts,
                 double* U, int64_t ldu, double* S, double* V, int64_t ldv, om_stats* st);

/* --- O-CYC: textbook Algorithm 1, fp64, row-cyclic order eq. (2.1) ---- */
/* On exit X holds X*V_X (unnormalised), V (n x n, ldv) the accumulated
   rotations (V seeded by the caller).  Returns sweeps (<0: not converged). */
int32_t oc_cyclic_jacobi(double* X, int64_t m, int64_t n, int64_t ldx, double* V, int64_t ldv,
                         double tol, int32_t max_sweeps, int64_t* rotations);

#endif
