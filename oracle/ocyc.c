/*
 * ocyc.c -- TEST INFRASTRUCTURE ONLY.  O-CYC: the textbook one-sided Jacobi
 * SVD, Algorithm 1 of the paper, in fp64 with the
 * row-cyclic pair order of eq. (2.1):
 *   (1,2),(1,3),...,(1,n),(2,3),...,(n-1,n).
 * Scalar plane rotations, the closest-to-identity choice
 * (footnote).  Shares no code with omix.c (the block
 * algorithm) nor with the CUDA path.
 */
#include <math.h>
#include <stdint.h>
#include "oracle.h"

static double dot(const double* x, const double* y, int64_t m) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += x[i] * y[i];
    return s;
}

int32_t oc_cyclic_jacobi(double* X, int64_t m, int64_t n, int64_t ldx, double* V, int64_t ldv,
                         double tol, int32_t max_sweeps, int64_t* rotations) {
    int64_t nrot = 0;
    for (int32_t iter = 1; iter <= max_sweeps; ++iter) {
        int converged = 1;                                   /* Alg. 1 line 4 */
        for (int64_t p = 0; p < n - 1; ++p) {
            for (int64_t q = p + 1; q < n; ++q) {            /* eq. (2.1) */
                double* xp = X + p * ldx;
                double* xq = X + q * ldx;
                double a = dot(xp, xp, m);                   /* ||x_p||^2 */
                double b = dot(xq, xq, m);                   /* ||x_q||^2 */
                double c = dot(xq, xp, m);                   /* x_q^T x_p */
                if (!(a > 0.0) || !(b > 0.0)) continue;
                if (fabs(c) > tol * sqrt(a) * sqrt(b)) {     /* Alg. 1 line 6 */
                    double zeta = (b - a) / (2.0 * c);
                    double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    double cs = 1.0 / sqrt(1.0 + t * t);
                    double sn = t * cs;
                    for (int64_t i = 0; i < m; ++i) {        /* X <- X J */
                        double u = xp[i], w = xq[i];
                        xp[i] = cs * u - sn * w;
                        xq[i] = sn * u + cs * w;
                    }
                    if (V) {                                 /* V_X <- V_X J */
                        double* vp = V + p * ldv;
                        double* vq = V + q * ldv;
                        for (int64_t i = 0; i < n; ++i) {
                            double u = vp[i], w = vq[i];
                            vp[i] = cs * u - sn * w;
                            vq[i] = sn * u + cs * w;
                        }
                    }
                    converged = 0;
                    ++nrot;
                }
            }
        }
        if (converged) {
            if (rotations) *rotations = nrot;
            return iter;
        }
    }
    if (rotations) *rotations = nrot;
    return -max_sweeps;
}
