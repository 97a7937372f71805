/*
 * omix.c -- TEST INFRASTRUCTURE ONLY.  O-MIX: plain, slow, sequential CPU
 * implementation of the mixed-precision Jacobi SVD (Alg. 3)
 * exactly as read in DESIGN.md ("Readings").
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline,
 * --impl reference) may load it.  It shares no code with the CUDA path.
 *
 * Built with gcc -O2 -ffp-contract=off (reading c-14): IEEE round-to-nearest,
 * correctly rounded sqrt, no FMA contraction.  OpenMP (optional) only runs
 * disjoint block pairs / independent columns concurrently; results do not
 * depend on the thread count.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include "oracle.h"

#define U64 1.1102230246251565e-16   /* 2^-53, PAPER.md:584-585 (reading c-2) */
#define U32 5.9604644775390625e-08   /* 2^-24 */

/* ---- block Jacobi, instantiated for fp32 and fp64 -------------------- */
#define REAL float
#define SFX f32
#define RSQRT_U 4096.0f              /* 1/sqrt(2^-24) */
#include "bj_impl.inc"
#undef REAL
#undef SFX
#undef RSQRT_U
#define REAL double
#define SFX f64
#define RSQRT_U 94906265.62425156    /* 1/sqrt(2^-53) */
#include "bj_impl.inc"
#undef REAL
#undef SFX
#undef RSQRT_U

int32_t om_block_jacobi_f64(double* X, int64_t m, int64_t n, int64_t ldx, double* V, int64_t nv,
                            int64_t ldv, int32_t b, double tol, double tol_in, int32_t max_sweeps,
                            int32_t max_inner, double* off_trace, int32_t* upd_trace, int32_t nthreads) {
    return block_jacobi_f64(X, m, n, ldx, V, nv, ldv, b, tol, tol_in, max_sweeps, max_inner, 0,
                            off_trace, upd_trace, nthreads);
}

int32_t om_block_jacobi_f32(float* X, int64_t m, int64_t n, int64_t ldx, float* V, int64_t nv,
                            int64_t ldv, int32_t b, float tol, float tol_in, int32_t max_sweeps,
                            int32_t max_inner, int32_t stagnation, double* off_trace,
                            int32_t* upd_trace, int32_t nthreads) {
    return block_jacobi_f32(X, m, n, ldx, V, nv, ldv, b, tol, tol_in, max_sweeps, max_inner,
                            stagnation, off_trace, upd_trace, nthreads);
}

void om_default_opts(om_opts* o) {
    o->b = 32;
    o->tol_mult32 = 4.0;
    o->tol_mult64 = 4.0;
    o->inner_tol_div = 8;
    o->max_sweeps32 = 20;
    o->max_sweeps64 = 30;
    o->max_inner = 30;
    o->path = OM_PATH_FORCE_MIXED;
    o->x_from_lq = 1;
    o->nthreads = 0;
    o->mp_rrqr = 0;
    o->max_inner32 = 1;
    o->switch_u = 1;
    o->tol_orth = 1e-5;
    o->tol_alg = INFINITY;
    o->tol_cond_mult = 1.0;
    o->cond_d_min = 1e15;
    o->tail_frac = 1.0 / 3.0;
    o->tail_cut_log2 = -60;
    o->refine_v = 0;
}


/* ---- Householder ------------------------------------------------------ */
/* GVL Alg. 5.1.1 with beta = +||x|| (diag(R) >= 0, reading c-13). */
double om_house(double* x, int64_t len) {
    double alpha = x[0];
    double sigma = 0.0;
    for (int64_t i = 1; i < len; ++i) sigma += x[i] * x[i];
    if (sigma == 0.0) {
        if (alpha >= 0.0) return 0.0;          /* H = I */
        x[0] = -alpha;                          /* H = I - 2 e1 e1^T */
        return 2.0;
    }
    double mu = sqrt(alpha * alpha + sigma);
    double v0 = alpha <= 0.0 ? alpha - mu : -sigma / (alpha + mu);
    double tau = 2.0 * v0 * v0 / (sigma + v0 * v0);
    for (int64_t i = 1; i < len; ++i) x[i] /= v0;
    x[0] = mu;
    return tau;
}

/* apply H = I - tau v v^T (v = [1; x[1..len-1]]) to column c[0..len-1] */
static void apply_h(const double* v, int64_t len, double tau, double* c) {
    if (tau == 0.0) return;
    double w = c[0];
    for (int64_t i = 1; i < len; ++i) w += v[i] * c[i];
    w *= tau;
    c[0] -= w;
    for (int64_t i = 1; i < len; ++i) c[i] -= w * v[i];
}

int om_qr(double* A, int64_t m, int64_t n, int64_t lda, double* tau) {
    /* PAPER.md:416-420 (Alg. 3 "A = Q R1"), 472-476 (sec. 3.1) */
    int rc = 0;
    for (int64_t k = 0; k < n; ++k) {
        double* ak = A + k * lda + k;
        tau[k] = om_house(ak, m - k);
        if (ak[0] == 0.0) rc = -3;
#pragma omp parallel for schedule(static)
        for (int64_t j = k + 1; j < n; ++j) apply_h(ak, m - k, tau[k], A + j * lda + k);
    }
    return rc;
}

static double plain_norm(const double* x, int64_t len) {
    double s = 0.0;
    for (int64_t i = 0; i < len; ++i) s += x[i] * x[i];
    return sqrt(s);
}

int om_qrp(double* A, int64_t m, int64_t n, int64_t lda, int32_t* perm, double* tau) {
    /* Businger-Golub RRQR, AP = Q1 R (Alg. 2 line 1);
       partial-norm downdating with recompute as LAPACK xLAQP2 (reading c-20). */
    const double tol3z = sqrt(U64);
    double* vn1 = (double*)malloc(sizeof(double) * (size_t)n);
    double* vn2 = (double*)malloc(sizeof(double) * (size_t)n);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)m);
    int rc = 0;
    for (int64_t j = 0; j < n; ++j) {
        perm[j] = (int32_t)j;
        vn1[j] = plain_norm(A + j * lda, m);
        vn2[j] = vn1[j];
    }
    for (int64_t k = 0; k < n && k < m; ++k) {
        int64_t pvt = k;
        for (int64_t j = k + 1; j < n; ++j)
            if (vn1[j] > vn1[pvt]) pvt = j;          /* ties -> lowest index */
        if (pvt != k) {
            memcpy(tmp, A + pvt * lda, sizeof(double) * (size_t)m);
            memcpy(A + pvt * lda, A + k * lda, sizeof(double) * (size_t)m);
            memcpy(A + k * lda, tmp, sizeof(double) * (size_t)m);
            int32_t ip = perm[pvt]; perm[pvt] = perm[k]; perm[k] = ip;
            vn1[pvt] = vn1[k];
            vn2[pvt] = vn2[k];
        }
        double* ak = A + k * lda + k;
        tau[k] = om_house(ak, m - k);
        if (ak[0] == 0.0) rc = -3;
#pragma omp parallel for schedule(static)
        for (int64_t j = k + 1; j < n; ++j) {
            double* aj = A + j * lda;
            apply_h(ak, m - k, tau[k], aj + k);
            if (vn1[j] != 0.0) {
                double r = fabs(aj[k]) / vn1[j];
                double temp = 1.0 - r * r;
                if (temp < 0.0) temp = 0.0;
                double q = vn1[j] / vn2[j];
                double temp2 = temp * q * q;
                if (temp2 <= tol3z) {
                    if (k + 1 < m) {
                        vn1[j] = plain_norm(aj + k + 1, m - k - 1);
                        vn2[j] = vn1[j];
                    } else {
                        vn1[j] = 0.0;
                        vn2[j] = 0.0;
                    }
                } else {
                    vn1[j] *= sqrt(temp);
                }
            }
        }
    }
    free(vn1);
    free(vn2);
    free(tmp);
    return rc;
}

/* ---- fp32 QRP (Alg. 4 line 2) ------------------------------------------
   om_house / apply_h / plain_norm / om_qrp written out again in float: every
   operation rounds to fp32; tol3z = sqrt(u32) (LAPACK xLAQP2 in single). */
static float house_f32(float* x, int64_t len) {
    float alpha = x[0];
    float sigma = 0.0f;
    for (int64_t i = 1; i < len; ++i) sigma += x[i] * x[i];
    if (sigma == 0.0f) {
        if (alpha >= 0.0f) return 0.0f;
        x[0] = -alpha;
        return 2.0f;
    }
    float mu = sqrtf(alpha * alpha + sigma);
    float v0 = alpha <= 0.0f ? alpha - mu : -sigma / (alpha + mu);
    float tau = 2.0f * v0 * v0 / (sigma + v0 * v0);
    for (int64_t i = 1; i < len; ++i) x[i] /= v0;
    x[0] = mu;
    return tau;
}

static void apply_h_f32(const float* v, int64_t len, float tau, float* c) {
    if (tau == 0.0f) return;
    float w = c[0];
    for (int64_t i = 1; i < len; ++i) w += v[i] * c[i];
    w *= tau;
    c[0] -= w;
    for (int64_t i = 1; i < len; ++i) c[i] -= w * v[i];
}

static float plain_norm_f32(const float* x, int64_t len) {
    float s = 0.0f;
    for (int64_t i = 0; i < len; ++i) s += x[i] * x[i];
    return sqrtf(s);
}

int om_qrp_f32(float* A, int64_t m, int64_t n, int64_t lda, int32_t* perm, float* tau) {
    const float tol3z = sqrtf((float)U32);
    float* vn1 = (float*)malloc(sizeof(float) * (size_t)n);
    float* vn2 = (float*)malloc(sizeof(float) * (size_t)n);
    float* tmp = (float*)malloc(sizeof(float) * (size_t)m);
    int rc = 0;
    for (int64_t j = 0; j < n; ++j) {
        perm[j] = (int32_t)j;
        vn1[j] = plain_norm_f32(A + j * lda, m);
        vn2[j] = vn1[j];
    }
    for (int64_t k = 0; k < n && k < m; ++k) {
        int64_t pvt = k;
        for (int64_t j = k + 1; j < n; ++j)
            if (vn1[j] > vn1[pvt]) pvt = j;          /* ties -> lowest index */
        if (pvt != k) {
            memcpy(tmp, A + pvt * lda, sizeof(float) * (size_t)m);
            memcpy(A + pvt * lda, A + k * lda, sizeof(float) * (size_t)m);
            memcpy(A + k * lda, tmp, sizeof(float) * (size_t)m);
            int32_t ip = perm[pvt]; perm[pvt] = perm[k]; perm[k] = ip;
            vn1[pvt] = vn1[k];
            vn2[pvt] = vn2[k];
        }
        float* ak = A + k * lda + k;
        tau[k] = house_f32(ak, m - k);
        if (ak[0] == 0.0f) rc = -3;
#pragma omp parallel for schedule(static)
        for (int64_t j = k + 1; j < n; ++j) {
            float* aj = A + j * lda;
            apply_h_f32(ak, m - k, tau[k], aj + k);
            if (vn1[j] != 0.0f) {
                float r = fabsf(aj[k]) / vn1[j];
                float temp = 1.0f - r * r;
                if (temp < 0.0f) temp = 0.0f;
                float q = vn1[j] / vn2[j];
                float temp2 = temp * q * q;
                if (temp2 <= tol3z) {
                    if (k + 1 < m) {
                        vn1[j] = plain_norm_f32(aj + k + 1, m - k - 1);
                        vn2[j] = vn1[j];
                    } else {
                        vn1[j] = 0.0f;
                        vn2[j] = 0.0f;
                    }
                } else {
                    vn1[j] *= sqrtf(temp);
                }
            }
        }
    }
    free(vn1);
    free(vn2);
    free(tmp);
    return rc;
}

/* Mixed-precision RRQR, PAPER.md:496-512 (Alg. 4):
   line 1  A_low = lower(A)                 (fl32 of A 2^-e: exact power-of-two scale, c-9)
   line 2  A_low P = Q_low R_low in fp32    (om_qrp_f32; only P is kept)
   line 3  A <- A P
   line 4  A = Q R in the working precision (om_qr, fp64 Householder). */
int om_mprrqr(double* A, int64_t m, int64_t n, int64_t lda, int32_t* perm, double* tau) {
    double mx = 0.0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) { double v = fabs(A[i + j * lda]); if (v > mx) mx = v; }
    int e = 0;
    frexp(mx, &e);
    const double scale = ldexp(1.0, -e);
    float* A32 = (float*)malloc(sizeof(float) * (size_t)m * (size_t)n);
    float* tau32 = (float*)malloc(sizeof(float) * (size_t)n);
    double* Ap = (double*)malloc(sizeof(double) * (size_t)m * (size_t)n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) A32[i + j * m] = (float)(A[i + j * lda] * scale);
    om_qrp_f32(A32, m, n, m, perm, tau32);
    for (int64_t k = 0; k < n; ++k) memcpy(Ap + k * m, A + (int64_t)perm[k] * lda, sizeof(double) * (size_t)m);
    for (int64_t k = 0; k < n; ++k) memcpy(A + k * lda, Ap + k * m, sizeof(double) * (size_t)m);
    int rc = om_qr(A, m, n, lda, tau);
    free(A32);
    free(tau32);
    free(Ap);
    return rc;
}

void om_apply_q(const double* Vr, int64_t m, int64_t k, int64_t ldv, const double* tau, double* C,
                int64_t ldc, int64_t ncols) {
    /* Q = H_0 H_1 ... H_{k-1}: apply H_{k-1} first. */
    for (int64_t i = k - 1; i >= 0; --i) {
        const double* v = Vr + i * ldv + i;
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < ncols; ++j) apply_h(v, m - i, tau[i], C + j * ldc + i);
    }
}

/* ---- precision lift (reading c-11) ------------------ */
int om_lift(const float* V32, int64_t n, int64_t ldv32, double* Q, int64_t ldq) {
    double* V = (double*)malloc(sizeof(double) * (size_t)n * n);
    double* G = (double*)malloc(sizeof(double) * (size_t)n * n);
    double* R = (double*)calloc((size_t)n * n, sizeof(double));
    int rc = 0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) V[i + j * n] = (double)V32[i + j * ldv32];
    /* G = V^T V */
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i <= j; ++i) {
            double acc = 0.0;
            for (int64_t r = 0; r < n; ++r) acc += V[r + i * n] * V[r + j * n];
            G[i + j * n] = acc;
            G[j + i * n] = acc;
        }
    /* Cholesky G = R^T R, R upper with positive diagonal */
    for (int64_t j = 0; j < n; ++j) {
        double d = G[j + j * n];
        for (int64_t k = 0; k < j; ++k) d -= R[k + j * n] * R[k + j * n];
        if (!(d > 0.0)) { rc = -3; d = DBL_MIN; }
        double rjj = sqrt(d);
        R[j + j * n] = rjj;
#pragma omp parallel for schedule(static)
        for (int64_t i = j + 1; i < n; ++i) {
            double s = G[j + i * n];
            for (int64_t k = 0; k < j; ++k) s -= R[k + j * n] * R[k + i * n];
            R[j + i * n] = s / rjj;
        }
    }
    /* Q = V R^-1: row-wise forward substitution (rows independent) */
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r) {
        for (int64_t j = 0; j < n; ++j) {
            double s = V[r + j * n];
            for (int64_t i = 0; i < j; ++i) s -= Q[r + i * ldq] * R[i + j * n];
            Q[r + j * ldq] = s / R[j + j * n];
        }
    }
    free(V);
    free(G);
    free(R);
    return rc;
}

/* ---- U-route precision switch (Alg. 3 l.446-447) --- */
int om_switch_u(const double* X, int64_t n, int64_t ldx, const double* Ulow, int64_t ldu,
                double* Q, int64_t ldq) {
    double* Z = (double*)malloc(sizeof(double) * (size_t)n * n);
    double* tau = (double*)malloc(sizeof(double) * (size_t)n);
    /* Z = X^T Ulow: z_ij = sum_r x_ri u_rj, ascending r */
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int64_t r = 0; r < n; ++r) acc += X[r + i * ldx] * Ulow[r + j * ldu];
            Z[i + j * n] = acc;
        }
    /* Z = Q R2, Householder, diag(R2) >= 0 */
    int rc = om_qr(Z, n, n, n, tau);
    /* Q = H_0 ... H_{n-1} I */
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) Q[i + j * ldq] = i == j ? 1.0 : 0.0;
    om_apply_q(Z, n, n, n, tau, Q, ldq, n);
    free(Z);
    free(tau);
    return rc;
}

/* overflow-safe two-pass norm: scale by max|x|, then sum squares */
static double safe_norm(const double* x, int64_t len) {
    double mx = 0.0;
    for (int64_t i = 0; i < len; ++i) if (fabs(x[i]) > mx) mx = fabs(x[i]);
    if (mx == 0.0) return 0.0;
    double s = 0.0;
    for (int64_t i = 0; i < len; ++i) { double y = x[i] / mx; s += y * y; }
    return mx * sqrt(s);
}

/* stable descending argsort by key (ties -> lower index) */
static void argsort_desc(const double* key, int64_t n, int64_t* idx) {
    for (int64_t i = 0; i < n; ++i) idx[i] = i;
    /* insertion-free merge via rank counting: O(n^2) but obviously stable */
    int64_t* rank = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
        int64_t rk = 0;
        for (int64_t k = 0; k < n; ++k)
            if (key[k] > key[j] || (key[k] == key[j] && k < j)) ++rk;
        rank[j] = rk;
    }
    for (int64_t j = 0; j < n; ++j) idx[rank[j]] = j;
    free(rank);
}

/* Y = X Q (n x n, all column-major, ld n): y_j = sum_k x_k q_kj in ascending k */
static void times_q(const double* X, const double* Q, double* Y, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
        double* yj = Y + j * n;
        for (int64_t i = 0; i < n; ++i) yj[i] = 0.0;
        for (int64_t k = 0; k < n; ++k) {
            double q = Q[k + j * n];
            const double* xk = X + k * n;
            for (int64_t i = 0; i < n; ++i) yj[i] += xk[i] * q;
        }
    }
}

/* ---- gate measures of Alg. 3 (reading c-15) -------------------------
   Each is a plain loop over its definition; pinned in tests/test_oracle_pins.py (exact constructions,
   closed forms, invariances, LAPACK). */

/* orth = || X_t^T X_t - I ||_max with X_t = lower(X) D^-1, D_jj the 2-norm of column j of lower(X)
   (PAPER.md:429-431): lower(X) = fl32(X); ||fl32(x_j)|| is summed in fp64 and rounded to fp32; the Gram
   X_t^T X_t is "one matrix-matrix multiplication in the lower precision": fp32 products
   accumulated in fp32 in ascending row order (reading c-17).  work: n*n floats. */
double om_gate_orth(const double* X, int64_t n, int64_t ldx, float* Xt) {
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) { float f = (float)X[i + j * ldx]; s += (double)f * (double)f; }
        float d = (float)sqrt(s);
        for (int64_t i = 0; i < n; ++i) Xt[i + j * n] = d > 0 ? (float)X[i + j * ldx] / d : 0.0f;
    }
    double orth = 0.0;
#pragma omp parallel for schedule(dynamic, 4) reduction(max : orth)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i <= j; ++i) {
            float acc = 0.0f;
            for (int64_t r = 0; r < n; ++r) acc += Xt[r + i * n] * Xt[r + j * n];
            double dev = fabs((double)acc - (i == j ? 1.0 : 0.0));
            if (dev > orth) orth = dev;
        }
    return orth;
}

/* fraction of "small" columns of X: ||x_j|| < 2^cut_log2 max_k ||x_k|| (reading c-15) */
double om_gate_tail(const double* X, int64_t n, int64_t ldx, int32_t cut_log2) {
    double mxn = 0.0;
    double* cn = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) { cn[j] = safe_norm(X + j * ldx, n); if (cn[j] > mxn) mxn = cn[j]; }
    int64_t small = 0;
    for (int64_t j = 0; j < n; ++j) if (cn[j] < ldexp(mxn, cut_log2)) ++small;
    free(cn);
    return (double)small / (double)n;
}

/* cond_R of Alg. 3 l.423 / kappa(R) of PAPER.md:629-634 for the column-scaled R: kappa_1(R_s) =
   ||R_s||_1 ||R_s^-1||_1, R_s = R diag(1/c) (R = upper triangle of R, ldr; c_k > 0 the column scales).
   R_s^-1 = diag(c) R^-1; column j of R^-1 by back substitution R z = e_j. */
double om_gate_cond_scaled(const double* R, int64_t n, int64_t ldr, const double* c) {
    double nrm = 0.0, inv = 0.0;
    for (int64_t k = 0; k < n; ++k) {
        if (!(c[k] > 0.0) || R[k + k * ldr] == 0.0) return INFINITY;
        double s = 0.0;
        for (int64_t i = 0; i <= k; ++i) s += fabs(R[i + k * ldr]);
        s /= c[k];
        if (s > nrm) nrm = s;
    }
#pragma omp parallel for schedule(dynamic, 8) reduction(max : inv)
    for (int64_t j = 0; j < n; ++j) {
        double* z = (double*)malloc(sizeof(double) * (size_t)(j + 1));
        z[j] = 1.0 / R[j + j * ldr];
        for (int64_t i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int64_t l = i + 1; l <= j; ++l) s += R[i + l * ldr] * z[l];
            z[i] = -s / R[i + i * ldr];
        }
        double cs = 0.0;
        for (int64_t i = 0; i <= j; ++i) cs += c[i] * fabs(z[i]);
        if (cs > inv) inv = cs;
        free(z);
    }
    return nrm * inv;
}

/* condition number of D in A = B D (Alg. 3 l.423-424): max/min column norm */
double om_gate_cond_d(const double* cn, int64_t n) {
    double dmx = 0.0, dmn = INFINITY;
    for (int64_t k = 0; k < n; ++k) {
        if (cn[k] > dmx) dmx = cn[k];
        if (cn[k] < dmn) dmn = cn[k];
    }
    return dmn > 0.0 ? dmx / dmn : INFINITY;
}

/* ---- Algorithm 3 ------------------------------------------------------- */
int om_mixed_svd(const double* A, int64_t m, int64_t n, int64_t lda, const om_opts* opts,
                 double* U, int64_t ldu, double* S, double* Vout, int64_t ldv, om_stats* st) {
    om_opts o;
    if (opts) o = *opts; else om_default_opts(&o);
    om_stats dummy;
    if (!st) st = &dummy;
    memset(st, 0, sizeof(*st));
    /* step 1: validate ("m >= n") */
    if (!A || !U || !S || !Vout || n < 2 || m < n || lda < m || ldu < m || ldv < n || o.b < 1 || o.b > 1024)
        return -1;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i)
            if (!isfinite(A[i + j * lda])) return -2;
#ifdef _OPENMP
    if (o.nthreads > 0) omp_set_num_threads(o.nthreads);
#endif
    int rc = 0;
    const int64_t nn = n * n;
    double* Aw = (double*)malloc(sizeof(double) * (size_t)m * n);
    double* tau_tall = (double*)malloc(sizeof(double) * (size_t)n);
    double* A1 = (double*)calloc((size_t)nn, sizeof(double));
    double* tau_p = (double*)malloc(sizeof(double) * (size_t)n);
    int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    double* Rt = (double*)calloc((size_t)nn, sizeof(double));
    double* tau_t = (double*)malloc(sizeof(double) * (size_t)n);
    double* X = (double*)calloc((size_t)nn, sizeof(double));
    float* X32 = (float*)malloc(sizeof(float) * (size_t)nn);
    float* V32 = (float*)calloc((size_t)nn, sizeof(float));
    double* Q = (double*)calloc((size_t)nn, sizeof(double));
    double* Y = (double*)calloc((size_t)nn, sizeof(double));
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    double* key = (double*)malloc(sizeof(double) * (size_t)n);
    double* tmpm = (double*)malloc(sizeof(double) * (size_t)nn);
    double* a1n = NULL;

    for (int64_t j = 0; j < n; ++j) memcpy(Aw + j * m, A + j * lda, sizeof(double) * (size_t)m);

    /* step 2: tall case A = Q R1, A1 = R1 */
    if (m > n) {
        if (om_qr(Aw, m, n, m, tau_tall) != 0) { /* zero diagonal: rank deficient */ }
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i <= j; ++i) A1[i + j * n] = Aw[i + j * m];
    } else {
        for (int64_t j = 0; j < n; ++j) memcpy(A1 + j * n, Aw + j * m, sizeof(double) * (size_t)n);
    }

    /* column norms of A1 = D of A = B D (the cond gate's cond(D)) */
    a1n = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) a1n[j] = safe_norm(A1 + j * n, n);

    /* step 3: RRQR A1 P = Q_p R, by the mixed-precision RRQR of
       PAPER.md:494-495 ("We use this mixed precision algorithm ... in the preconditioning stage") */
    if ((o.mp_rrqr ? om_mprrqr(A1, n, n, n, perm, tau_p) : om_qrp(A1, n, n, n, perm, tau_p)) != 0) {
        rc = -3;
        goto done;
    }

    /* step 4: R = L Q2 via QR of R^T; X = L (F1) */
    if (o.x_from_lq) {
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i <= j; ++i) Rt[j + i * n] = A1[i + j * n];   /* Rt = R^T */
        if (om_qr(Rt, n, n, n, tau_t) != 0) { rc = -3; goto done; }
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = j; i < n; ++i) X[i + j * n] = Rt[j + i * n];    /* L = (R_t)^T */
    } else {
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i <= j; ++i) X[i + j * n] = A1[i + j * n];
    }

    /* step 5: gate measures, report only (c-15) */
    {
        double mnr = INFINITY, mxr = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double rjj = fabs(A1[j + j * n]);
            if (rjj > mxr) mxr = rjj;
            if (rjj < mnr) mnr = rjj;
        }
        st->cond_estimate = mnr > 0 ? mxr / mnr : INFINITY;
        st->tail_fraction = om_gate_tail(X, n, n, -60);
        st->orth_measure = om_gate_orth(X, n, n, X32);
    }

    /* gate quantities of AUTO (reading c-15): cond_scaled = kappa_1 of R diag(1/c), c_k = ||R(:,k)|| =
       ||A1(:, perm_k)||; cond_d = max/min column norm of A1.  Computed under AUTO only (O(n^3)). */
    st->cond_scaled = NAN;
    st->cond_d = NAN;
    if (o.path == OM_PATH_AUTO) {
        for (int64_t k = 0; k < n; ++k) key[k] = a1n[perm[k]];
        st->cond_scaled = om_gate_cond_scaled(A1, n, n, key);
        st->cond_d = om_gate_cond_d(a1n, n);
    }
    int32_t taken = o.path == OM_PATH_FORCE_FP64 ? OM_PATH_FORCE_FP64 : OM_PATH_FORCE_MIXED;
    if (o.path == OM_PATH_AUTO) {
        /* Alg. 3 order: cond gate, tail gate (654-663), orth gate (428-433),
           then Jacobi if orth <= tol_alg else the QR SVD (435-445) */
        const double tol_cond = o.tol_cond_mult * pow((double)n, 0.25);
        double mxn = 0.0;
        int64_t small = 0;
        for (int64_t j = 0; j < n; ++j) { key[j] = safe_norm(X + j * n, n); if (key[j] > mxn) mxn = key[j]; }
        for (int64_t j = 0; j < n; ++j) if (key[j] < ldexp(mxn, o.tail_cut_log2)) ++small;
        if (st->cond_scaled <= tol_cond && st->cond_d > o.cond_d_min) taken = OM_TAKEN_SKIP_COND;
        else if ((double)small >= ceil(o.tail_frac * (double)n)) taken = OM_TAKEN_SKIP_TAIL;
        else if (st->orth_measure <= o.tol_orth) taken = OM_TAKEN_SKIP_ORTH;
        else if (st->orth_measure <= o.tol_alg) taken = OM_PATH_FORCE_MIXED;
        else taken = OM_TAKEN_QRSVD;
    }
    if (taken == OM_TAKEN_QRSVD) {
        /* lower(X) = U_low S_low V_low^* by the QR SVD in fp32, U only; then the
           U-route switch Q R2 = X^T working(U_low) (446-447) and Y = X Q */
        st->path_taken = OM_TAKEN_QRSVD;
        double mx = 0.0;
        for (int64_t i = 0; i < nn; ++i) if (fabs(X[i]) > mx) mx = fabs(X[i]);
        int e = 0;
        frexp(mx, &e);
        for (int64_t i = 0; i < nn; ++i) X32[i] = (float)ldexp(X[i], -e);
        float* S32 = (float*)malloc(sizeof(float) * (size_t)n);
        const int lrc = om_qrsvd32(X32, n, n, tmpm, n, S32);   /* qrsvd.c: U_low (fp64, sorted) */
        free(S32);
        if (lrc != 0) { rc = lrc < 0 ? -3 : 1; goto done; }
        if (om_switch_u(X, n, n, tmpm, n, Q, n) != 0) { rc = -3; goto done; }
        times_q(X, Q, Y, n);
    } else if (taken != OM_PATH_FORCE_MIXED) {
        /* Q = I, Y = X */
        st->path_taken = taken;
        for (int64_t j = 0; j < n; ++j) Q[j + j * n] = 1.0;
        memcpy(Y, X, sizeof(double) * (size_t)nn);
    } else {
        st->path_taken = OM_PATH_FORCE_MIXED;
        /* step 6: X32 = fl32(X 2^-e), max|X| 2^-e in [0.5, 1) (c-9); V32 = I (V-route only) */
        double mx = 0.0;
        for (int64_t i = 0; i < nn; ++i) if (fabs(X[i]) > mx) mx = fabs(X[i]);
        int e = 0;
        frexp(mx, &e);
        for (int64_t i = 0; i < nn; ++i) X32[i] = (float)ldexp(X[i], -e);
        memset(V32, 0, sizeof(float) * (size_t)nn);
        for (int64_t j = 0; j < n; ++j) V32[j + j * n] = 1.0f;

        /* step 7: fp32 block Jacobi (c-10).  The U-route computes U_low only
           (PAPER.md:542-545): no V accumulation */
        float tol32 = (float)(o.tol_mult32 * sqrt((double)n) * U32);
        float tol32_in = tol32 / (float)o.inner_tol_div;
        int32_t sw32 = om_block_jacobi_f32(X32, n, n, n, o.switch_u ? NULL : V32, o.switch_u ? 0 : n, n, o.b,
                                           tol32, tol32_in, o.max_sweeps32, o.max_inner32, 1, st->off_trace32,
                                           st->upd_trace32, o.nthreads);
        st->sweeps32 = sw32 < 0 ? -sw32 : sw32;
        st->final_off32 = st->sweeps32 > 0 && st->sweeps32 <= 64 ? st->off_trace32[st->sweeps32 - 1] : 0;

        /* step 8: sigma32 = column norms, stable descending sort (Alg. 1 l.309) */
        for (int64_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (int64_t i = 0; i < n; ++i) s += (double)X32[i + j * n] * (double)X32[i + j * n];
            key[j] = sqrt(s);
        }
        argsort_desc(key, n, idx);
        if (o.switch_u) {
            /* step 9u: U_low = working(X32 Sigma32^-1), columns in sigma32-descending order;
               Q = qr(X^T U_low) */
            for (int64_t j = 0; j < n; ++j) {
                if (!(key[idx[j]] > 0.0)) { rc = -3; goto done; }
                for (int64_t i = 0; i < n; ++i) tmpm[i + j * n] = (double)X32[i + idx[j] * n] / key[idx[j]];
            }
            if (om_switch_u(X, n, n, tmpm, n, Q, n) != 0) { rc = -3; goto done; }
        } else {
            /* step 9: permute V32; lift Q = qr(fl64(V32)) by CholeskyQR (c-11) */
            float* Vs = X32;  /* reuse: X32 no longer needed */
            for (int64_t j = 0; j < n; ++j) memcpy(Vs + j * n, V32 + idx[j] * n, sizeof(float) * (size_t)n);
            if (om_lift(Vs, n, n, Q, n) != 0) { rc = -3; goto done; }
        }

        /* step 10: Y = X Q */
        times_q(X, Q, Y, n);
    }

    /* step 11: fp64 refinement, V := Q (c-12) */
    if (!o.refine_v) {
        double tol64 = o.tol_mult64 * sqrt((double)n) * U64;
        double tol64_in = tol64 / (double)o.inner_tol_div;
        int32_t sw64 = om_block_jacobi_f64(Y, n, n, n, Q, n, n, o.b, tol64, tol64_in, o.max_sweeps64,
                                           o.max_inner, st->off_trace64, st->upd_trace64, o.nthreads);
        st->converged = sw64 > 0;
        st->sweeps64 = sw64 < 0 ? -sw64 : sw64;
        st->v_sweeps64 = st->sweeps64;
        st->final_off64 = st->sweeps64 > 0 && st->sweeps64 <= 64 ? st->off_trace64[st->sweeps64 - 1] : 0;
        if (!st->converged) rc = 1;
    } else {
        /* step 11' (sec. 3.4; reading c-23): "we first compute U_X without accumulating
           V_X" -- refinement of Y alone; U_X = Y diag(1/||y_j||); "we form V_X from the QR factorization of
           X^* U_X" (Householder, diag(R2) >= 0: om_switch_u); Y = X V_X; "another round of the one-sided
           Jacobi SVD algorithm by accumulating Jacobi rotations" from (Y, V := V_X), which "always converges
           in one sweep".  Traces: the first stage's sweeps, then the accumulating stage's. */
        double tol64 = o.tol_mult64 * sqrt((double)n) * U64;
        double tol64_in = tol64 / (double)o.inner_tol_div;
        int32_t swa = om_block_jacobi_f64(Y, n, n, n, NULL, 0, n, o.b, tol64, tol64_in, o.max_sweeps64,
                                          o.max_inner, st->off_trace64, st->upd_trace64, o.nthreads);
        int32_t na = swa < 0 ? -swa : swa;
        for (int64_t j = 0; j < n; ++j) {
            double s = safe_norm(Y + j * n, n);
            if (!(s > 0.0)) { rc = -3; goto done; }
            for (int64_t i = 0; i < n; ++i) tmpm[i + j * n] = Y[i + j * n] / s;
        }
        if (om_switch_u(X, n, n, tmpm, n, Q, n) != 0) { rc = -3; goto done; }
        times_q(X, Q, Y, n);
        int32_t swb = om_block_jacobi_f64(Y, n, n, n, Q, n, n, o.b, tol64, tol64_in, o.max_sweeps64,
                                          o.max_inner, st->off_trace64 + na, st->upd_trace64 + na, o.nthreads);
        int32_t nb = swb < 0 ? -swb : swb;
        st->converged = swa > 0 && swb > 0;
        st->sweeps64 = na + nb;
        st->v_sweeps64 = nb;
        st->final_off64 = st->sweeps64 > 0 && st->sweeps64 <= 64 ? st->off_trace64[st->sweeps64 - 1] : 0;
        if (!st->converged) rc = 1;
    }

    /* step 12: sigma = ||y_j||, U_X = Y / sigma, stable descending sort (Alg. 1 l.305-310) */
    for (int64_t j = 0; j < n; ++j) {
        key[j] = safe_norm(Y + j * n, n);
        if (!(key[j] > 0.0)) { rc = -3; goto done; }
    }
    argsort_desc(key, n, idx);
    /* U_X into tmpm (n x n), V_X into X (reuse) */
    for (int64_t j = 0; j < n; ++j) {
        int64_t s = idx[j];
        S[j] = key[s];
        for (int64_t i = 0; i < n; ++i) tmpm[i + j * n] = Y[i + s * n] / key[s];
        memcpy(X + j * n, Q + s * n, sizeof(double) * (size_t)n);
    }

    /* step 13: U = Q_tall [Q_p U_X]; V = P Q_t V_X */
    om_apply_q(A1, n, n, n, tau_p, tmpm, n, n);
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i < n; ++i) U[i + j * ldu] = tmpm[i + j * n];
        for (int64_t i = n; i < m; ++i) U[i + j * ldu] = 0.0;
    }
    if (m > n) om_apply_q(Aw, m, n, m, tau_tall, U, ldu, n);
    if (o.x_from_lq) om_apply_q(Rt, n, n, n, tau_t, X, n, n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t k = 0; k < n; ++k) Vout[perm[k] + j * ldv] = X[k + j * n];

done:
    free(Aw); free(tau_tall); free(A1); free(tau_p); free(perm); free(Rt); free(tau_t);
    free(X); free(X32); free(V32); free(Q); free(Y); free(idx); free(key); free(tmpm); free(a1n);
    return rc;
}
