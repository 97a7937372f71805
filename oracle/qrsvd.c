/*
 * qrsvd.c -- TEST INFRASTRUCTURE ONLY.  The "QR SVD algorithm in the lower precision" of Alg. 3's
 * AUTO branch ("Apply QR SVD algorithm in the lower precision to obtain
 * lower(X) = U_low Sigma_low V_low^* without generating V_low explicitly"), written out step by step as
 * DESIGN.md reading c-24 fixes it:
 *
 *   1. Householder bidiagonalisation X32 = Q_B B P_B^T in fp32 (GVL Alg. 5.4.2): for k = 0..n-1 a left
 *      reflector of column k (d_k = +||x||), then a right reflector of row k over columns k+1..n-1
 *      (e_k = +||y||).  Products accumulated in fp32 in ascending index order.
 *   2. Implicit-shift QR on the upper-bidiagonal B in fp32 (Golub-Kahan step, bulge chased downward):
 *      shift = the smaller singular value of the trailing 2 x 2 of the active block; a right rotation
 *      on columns (i, i+1) then a left rotation on rows (i, i+1) per position; e_i is set to 0 when
 *      |e_i| <= u32 (|d_i| + |d_{i+1}|).  The active block is the bottom-most unreduced one.
 *   3. The left rotations are accumulated into U_B (= I at the start) in fp64:
 *      u_i <- c u_i + s u_{i+1}, u_{i+1} <- -s u_i + c u_{i+1}  (B_new = G B, U <- U G^T).
 *   4. U_low = Q_B U_B in fp64 (the fp32 reflectors applied as exact fp64 values; Alg. 3 converts U_low
 *      to the working precision anyway).
 *   5. sigma_j = |d_j|, stable descending sort, columns of U_low permuted alike.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may load it.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

#define U32F 5.9604644775390625e-08f   /* 2^-24 */

/* fp32 Householder, GVL Alg. 5.1.1 with beta = +||x||: x <- (beta, v_1..v_{len-1}), v_0 = 1; returns tau */
static float house32(float* x, int64_t len, int64_t inc) {
    float alpha = x[0];
    float sigma = 0.0f;
    for (int64_t i = 1; i < len; ++i) sigma += x[i * inc] * x[i * inc];
    if (sigma == 0.0f) {
        if (alpha >= 0.0f) return 0.0f;
        x[0] = -alpha;
        return 2.0f;
    }
    float mu = sqrtf(alpha * alpha + sigma);
    float v0 = alpha <= 0.0f ? alpha - mu : -sigma / (alpha + mu);
    float tau = 2.0f * v0 * v0 / (sigma + v0 * v0);
    for (int64_t i = 1; i < len; ++i) x[i * inc] /= v0;
    x[0] = mu;
    return tau;
}

/* (c, s, r) with [c s; -s c] [f; g] = [r; 0] (LAPACK xLARTG convention, r = hypot(f, g)) */
static void givens32(float f, float g, float* c, float* s, float* r) {
    if (g == 0.0f) { *c = 1.0f; *s = 0.0f; *r = f; return; }
    if (f == 0.0f) { *c = 0.0f; *s = 1.0f; *r = g; return; }
    float rr = hypotf(f, g);
    *c = f / rr;
    *s = g / rr;
    *r = rr;
}

/* smaller singular value of [[f, g], [0, h]] (xLAS2 closed form) */
static float sv_min_2x2(float f, float g, float h) {
    float fa = fabsf(f), ga = fabsf(g), ha = fabsf(h);
    float fhmn = fminf(fa, ha), fhmx = fmaxf(fa, ha);
    if (fhmn == 0.0f) return 0.0f;
    if (ga < fhmx) {
        float as = 1.0f + fhmn / fhmx, at = (fhmx - fhmn) / fhmx, au = (ga / fhmx) * (ga / fhmx);
        float c = 2.0f / (sqrtf(as * as + au) + sqrtf(at * at + au));
        return fhmn * c;
    }
    float au = fhmx / ga;
    if (au == 0.0f) return (fhmn * fhmx) / ga;
    float as = 1.0f + fhmn / fhmx, at = (fhmx - fhmn) / fhmx;
    float c = 1.0f / (sqrtf(1.0f + (as * au) * (as * au)) + sqrtf(1.0f + (at * au) * (at * au)));
    return (fhmn * c) * au * 2.0f;
}

int om_qrsvd32(const float* X32, int64_t n, int64_t ldx, double* U, int64_t ldu, float* S) {
    float* A = (float*)malloc(sizeof(float) * (size_t)n * n);
    float* tau = (float*)malloc(sizeof(float) * (size_t)n);
    float* d = (float*)malloc(sizeof(float) * (size_t)n);
    float* e = (float*)calloc((size_t)(n > 1 ? n : 2), sizeof(float));
    double* UB = (double*)calloc((size_t)n * n, sizeof(double));
    double* P = (double*)calloc((size_t)n * n, sizeof(double));
    double* tau64 = (double*)malloc(sizeof(double) * (size_t)n);
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int rc = 0;
    for (int64_t j = 0; j < n; ++j) memcpy(A + j * n, X32 + j * ldx, sizeof(float) * (size_t)n);

    /* 1. bidiagonalisation */
    for (int64_t k = 0; k < n; ++k) {
        float* ak = A + k * n + k;
        tau[k] = house32(ak, n - k, 1);
        d[k] = ak[0];
        for (int64_t j = k + 1; j < n; ++j) {          /* A(k:, j) -= tau v (v^T A(k:, j)) */
            float* aj = A + j * n + k;
            float w = aj[0];
            for (int64_t i = 1; i < n - k; ++i) w += ak[i] * aj[i];
            w *= tau[k];
            aj[0] -= w;
            for (int64_t i = 1; i < n - k; ++i) aj[i] -= w * ak[i];
        }
        if (k + 1 < n) {
            float* rk = A + (k + 1) * n + k;          /* row k, columns k+1..n-1, stride n */
            float pi = house32(rk, n - k - 1, n);
            e[k] = rk[0];
            for (int64_t i = k + 1; i < n; ++i) {     /* A(i, k+1:) -= pi (A(i, k+1:) u) u^T */
                float w = A[i + (k + 1) * n];
                for (int64_t l = 1; l < n - k - 1; ++l) w += A[i + (k + 1 + l) * n] * rk[l * n];
                w *= pi;
                A[i + (k + 1) * n] -= w;
                for (int64_t l = 1; l < n - k - 1; ++l) A[i + (k + 1 + l) * n] -= w * rk[l * n];
            }
        }
    }

    /* 2.-3. implicit-shift QR on B, left rotations accumulated into U_B (fp64) */
    for (int64_t j = 0; j < n; ++j) UB[j + j * n] = 1.0;
    const int64_t maxit = 6 * n * n + 60;
    int64_t it = 0;
    int64_t hi = n - 1;
    while (hi > 0) {
        for (int64_t i = 0; i < hi; ++i)
            if (fabsf(e[i]) <= U32F * (fabsf(d[i]) + fabsf(d[i + 1]))) e[i] = 0.0f;
        while (hi > 0 && e[hi - 1] == 0.0f) --hi;
        if (hi == 0) break;
        int64_t lo = hi - 1;
        while (lo > 0 && e[lo - 1] != 0.0f) --lo;
        for (int64_t i = lo; i <= hi; ++i)
            if (d[i] == 0.0f) { rc = -3; goto out; }   /* rank deficient (reading c-18) */
        if (++it > maxit) { rc = 1; goto out; }
        float shift = sv_min_2x2(d[hi - 1], e[hi - 1], d[hi]);
        float dmax = 0.0f;
        for (int64_t i = lo; i <= hi; ++i) dmax = fmaxf(dmax, fabsf(d[i]));
        if ((shift / dmax) * (shift / dmax) < U32F) shift = 0.0f;
        float f = (fabsf(d[lo]) - shift) * ((d[lo] >= 0.0f ? 1.0f : -1.0f) + shift / d[lo]);
        float g = e[lo];
        for (int64_t i = lo; i < hi; ++i) {
            float cr, sr, r, cl, sl;
            givens32(f, g, &cr, &sr, &r);                 /* right rotation, columns (i, i+1) */
            if (i > lo) e[i - 1] = r;
            f = cr * d[i] + sr * e[i];
            e[i] = cr * e[i] - sr * d[i];
            g = sr * d[i + 1];
            d[i + 1] = cr * d[i + 1];
            givens32(f, g, &cl, &sl, &r);                 /* left rotation, rows (i, i+1) */
            d[i] = r;
            f = cl * e[i] + sl * d[i + 1];
            d[i + 1] = cl * d[i + 1] - sl * e[i];
            if (i + 1 < hi) {
                g = sl * e[i + 1];
                e[i + 1] = cl * e[i + 1];
            }
            const double c = (double)cl, s = (double)sl;
            double* ui = UB + i * n;
            double* uj = UB + (i + 1) * n;
            for (int64_t r2 = 0; r2 < n; ++r2) {
                const double a = ui[r2], b = uj[r2];
                ui[r2] = c * a + s * b;
                uj[r2] = -s * a + c * b;
            }
        }
        e[hi - 1] = f;
    }
    for (int64_t j = 0; j < n; ++j)
        if (d[j] == 0.0f) { rc = -3; goto out; }       /* an exact zero singular value: rank deficient */

    /* 4. U_low = Q_B U_B in fp64 (reflectors of step 1, fp32 values) */
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i < n; ++i) P[i + j * n] = (double)A[i + j * n];
        tau64[j] = (double)tau[j];
    }
    om_apply_q(P, n, n, n, tau64, UB, n, n);

    /* 5. sigma = |d|, stable descending order */
    for (int64_t j = 0; j < n; ++j) idx[j] = j;
    for (int64_t a = 1; a < n; ++a) {                 /* insertion sort: stable */
        int64_t t = idx[a], b = a;
        while (b > 0 && fabsf(d[idx[b - 1]]) < fabsf(d[t])) { idx[b] = idx[b - 1]; --b; }
        idx[b] = t;
    }
    for (int64_t j = 0; j < n; ++j) {
        S[j] = fabsf(d[idx[j]]);
        memcpy(U + j * ldu, UB + idx[j] * n, sizeof(double) * (size_t)n);
    }
out:
    free(A); free(tau); free(d); free(e); free(UB); free(P); free(tau64); free(idx);
    return rc;
}
