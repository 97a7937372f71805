// k_linalg.cu -- dense fp64 building blocks of the precision switch
// (QR of V by CholeskyQR, reading c-11), the R*V product
// ("Y <- X Q") and the assembly U = Q_p U_X, V = P Q_t V_X
// by blocked compact-WY reflector application.
#include <cuda_runtime.h>
#include "common.cuh"
#include "jacobi.h"

namespace mpj {

// ------------------------------------------------------------------------
// fp64 GEMM: C = alpha op(A) op(B) + beta C (column-major).  64 x 64 tile,
// BK = 16, 256 threads, 4 x 4 register tile per thread, FP64 FMA pipe.
// ------------------------------------------------------------------------
constexpr int GB_M = 64, GB_N = 64, GB_K = 16;

__global__ void __launch_bounds__(256) k_gemm_f64(int ta, int tb, long long M, long long N, long long K,
                                                  double alpha, const double* __restrict__ A, long long lda,
                                                  const double* __restrict__ B, long long ldb, double beta,
                                                  double* __restrict__ C, long long ldc) {
    __shared__ __align__(16) double As[2][GB_K][GB_M + 2];
    __shared__ __align__(16) double Bs[2][GB_K][GB_N + 2];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const long long i0 = (long long)blockIdx.x * GB_M, j0 = (long long)blockIdx.y * GB_N;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    double ra[4], rb[4];
    auto fetch = [&](long long k0) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            int e = tid + 256 * t;
            int ii, kk;
            if (!ta) { ii = e & 63; kk = e >> 6; } else { kk = e & 15; ii = e >> 4; }
            long long gi = i0 + ii, gk = k0 + kk;
            double v = 0.0;
            if (gi < M && gk < K) v = ta ? A[gk + gi * lda] : A[gi + gk * lda];
            ra[t] = v;
            int jj, kb;
            if (!tb) { kb = e & 15; jj = e >> 4; } else { jj = e & 63; kb = e >> 6; }
            long long gj = j0 + jj, gkb = k0 + kb;
            double w = 0.0;
            if (gj < N && gkb < K) w = tb ? B[gj + gkb * ldb] : B[gkb + gj * ldb];
            rb[t] = w;
        }
    };
    auto store = [&](int st) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            int e = tid + 256 * t;
            int ii, kk;
            if (!ta) { ii = e & 63; kk = e >> 6; } else { kk = e & 15; ii = e >> 4; }
            As[st][kk][ii] = ra[t];
            int jj, kb;
            if (!tb) { kb = e & 15; jj = e >> 4; } else { jj = e & 63; kb = e >> 6; }
            Bs[st][kb][jj] = rb[t];
        }
    };
    const long long nk = (K + GB_K - 1) / GB_K;
    if (nk > 0) { fetch(0); store(0); }
    __syncthreads();
    for (long long kt = 0; kt < nk; ++kt) {
        const int st = kt & 1;
        if (kt + 1 < nk) fetch((kt + 1) * GB_K);
#pragma unroll
        for (int kk = 0; kk < GB_K; ++kk) {
            const double2 a01 = *reinterpret_cast<const double2*>(&As[st][kk][ty * 4]);
            const double2 a23 = *reinterpret_cast<const double2*>(&As[st][kk][ty * 4 + 2]);
            const double2 b01 = *reinterpret_cast<const double2*>(&Bs[st][kk][tx * 4]);
            const double2 b23 = *reinterpret_cast<const double2*>(&Bs[st][kk][tx * 4 + 2]);
            const double av[4] = {a01.x, a01.y, a23.x, a23.y};
            const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
        if (kt + 1 < nk) store(st ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        long long gj = j0 + tx * 4 + j;
        if (gj >= N) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            long long gi = i0 + ty * 4 + i;
            if (gi >= M) continue;
            double* c = C + gi + gj * ldc;
            *c = beta == 0.0 ? alpha * acc[i][j] : alpha * acc[i][j] + beta * *c;
        }
    }
}

int gemm_f64(int ta, int tb, long long M, long long N, long long K, double alpha, const double* A, long long lda,
             const double* B, long long ldb, double beta, double* C, long long ldc, cudaStream_t st) {
    if (M <= 0 || N <= 0) return 0;
    dim3 grid((unsigned)ceil_div(M, GB_M), (unsigned)ceil_div(N, GB_N));
    k_gemm_f64<<<grid, 256, 0, st>>>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// ------------------------------------------------------------------------
// Cholesky G = R^T R (upper, in place), right-looking, panel width 32.
// ------------------------------------------------------------------------
constexpr int CH_NB = 32;

__global__ void k_potrf_diag(double* G, long long ldg, int k0, int kb, int* bad) {
    __shared__ double a[CH_NB][CH_NB + 1];
    const int tid = threadIdx.x;
    for (int e = tid; e < kb * kb; e += blockDim.x) {
        int r = e % kb, c = e / kb;
        a[r][c] = r <= c ? G[(k0 + r) + (long long)(k0 + c) * ldg] : 0.0;
    }
    __syncthreads();
    for (int j = 0; j < kb; ++j) {
        if (tid == 0) {
            double d = a[j][j];
            if (!(d > 0.0)) { atomicOr(bad, 1); d = 2.2250738585072014e-308; }
            a[j][j] = sqrt(d);
        }
        __syncthreads();
        for (int c = j + 1 + tid; c < kb; c += blockDim.x) a[j][c] /= a[j][j];
        __syncthreads();
        for (int e = tid; e < kb * kb; e += blockDim.x) {
            int r = e % kb, c = e / kb;
            if (r > j && r <= c) a[r][c] -= a[j][r] * a[j][c];
        }
        __syncthreads();
    }
    for (int e = tid; e < kb * kb; e += blockDim.x) {
        int r = e % kb, c = e / kb;
        if (r <= c) G[(k0 + r) + (long long)(k0 + c) * ldg] = a[r][c];
    }
}

// U12 = U11^-T A12 : each column of A12 (kb rows) solved by one thread
__global__ void k_potrf_panel(double* G, long long ldg, int k0, int kb, int n) {
    __shared__ double u[CH_NB][CH_NB + 1];
    for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
        int r = e % kb, c = e / kb;
        u[r][c] = r <= c ? G[(k0 + r) + (long long)(k0 + c) * ldg] : 0.0;
    }
    __syncthreads();
    long long c = (long long)k0 + kb + blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= n) return;
    double x[CH_NB];
    double* col = G + k0 + c * ldg;
#pragma unroll
    for (int j = 0; j < CH_NB; ++j) x[j] = j < kb ? col[j] : 0.0;
#pragma unroll
    for (int j = 0; j < CH_NB; ++j) {
        if (j < kb) {
            double s = x[j];
#pragma unroll
            for (int i = 0; i < CH_NB; ++i)
                if (i < j) s -= u[i][j] * x[i];
            x[j] = s / u[j][j];
        }
    }
#pragma unroll
    for (int j = 0; j < CH_NB; ++j)
        if (j < kb) col[j] = x[j];
}

int potrf_upper(double* G, long long ldg, int n, int* bad, cudaStream_t st) {
    for (int k0 = 0; k0 < n; k0 += CH_NB) {
        int kb = n - k0 < CH_NB ? n - k0 : CH_NB;
        k_potrf_diag<<<1, 256, 0, st>>>(G, ldg, k0, kb, bad);
        MPJ_LAUNCHED();
        int rest = n - k0 - kb;
        if (rest > 0) {
            k_potrf_panel<<<(unsigned)ceil_div(rest, 128), 128, 0, st>>>(G, ldg, k0, kb, n);
            MPJ_LAUNCHED();
            const double* U12 = G + k0 + (long long)(k0 + kb) * ldg;
            double* A22 = G + (k0 + kb) + (long long)(k0 + kb) * ldg;
            int rc = gemm_f64(1, 0, rest, rest, kb, -1.0, U12, ldg, U12, ldg, 1.0, A22, ldg, st);
            if (rc) return rc;
        }
    }
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// ------------------------------------------------------------------------
// Q <- Q R^-1 (R upper), column blocks of 64: GEMM for the coupling, then a
// per-row forward substitution with the diagonal block in shared memory.
// ------------------------------------------------------------------------
constexpr int TR_NB = 64;

__global__ void k_trsm_rows(const double* R, long long ldr, double* Q, long long ldq, long long nrows, int j0,
                            int jb) {
    __shared__ double r[TR_NB][TR_NB + 1];
    for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
        int a = e % jb, c = e / jb;
        r[a][c] = R[(j0 + a) + (long long)(j0 + c) * ldr];
    }
    __syncthreads();
    long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (row >= nrows) return;
    double x[TR_NB];
#pragma unroll
    for (int c = 0; c < TR_NB; ++c) x[c] = c < jb ? Q[row + (long long)(j0 + c) * ldq] : 0.0;
#pragma unroll
    for (int c = 0; c < TR_NB; ++c) {
        if (c < jb) {
            double s = x[c];
#pragma unroll
            for (int i = 0; i < TR_NB; ++i)
                if (i < c) s -= x[i] * r[i][c];
            x[c] = s / r[c][c];
        }
    }
#pragma unroll
    for (int c = 0; c < TR_NB; ++c)
        if (c < jb) Q[row + (long long)(j0 + c) * ldq] = x[c];
}

int trsm_right_upper(const double* R, long long ldr, double* Q, long long ldq, long long nrows, int n,
                     cudaStream_t st) {
    for (int j0 = 0; j0 < n; j0 += TR_NB) {
        int jb = n - j0 < TR_NB ? n - j0 : TR_NB;
        if (j0 > 0) {
            int rc = gemm_f64(0, 0, nrows, jb, j0, -1.0, Q, ldq, R + (long long)j0 * ldr, ldr, 1.0,
                              Q + (long long)j0 * ldq, ldq, st);
            if (rc) return rc;
        }
        k_trsm_rows<<<(unsigned)ceil_div(nrows, 128), 128, 0, st>>>(R, ldr, Q, ldq, nrows, j0, jb);
        MPJ_LAUNCHED();
    }
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// ------------------------------------------------------------------------
// Blocked compact-WY application C <- Q C, Q = H_0 ... H_{k-1}.
// Panels of WY_NB reflectors in reverse order; for each:
//   Vp explicit (unit diagonal), S = Vp^T Vp, T (LAPACK xLARFT 'F','C'),
//   W1 = Vp^T C, W2 = T W1, C -= Vp W2.
// ------------------------------------------------------------------------
constexpr int WY_NB = 64;

__global__ void k_make_panel(const double* Vr, long long ldv, long long m, int j0, int kb, double* Vp,
                             long long ldp) {
    const int c = blockIdx.y;
    const long long rows = m - j0;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
        double v;
        if (c >= kb) v = 0.0;
        else if (r == c) v = 1.0;
        else if (r < c) v = 0.0;
        else v = Vr[(j0 + r) + (long long)(j0 + c) * ldv];
        Vp[r + (long long)c * ldp] = v;
    }
}

__global__ void k_larft(const double* S, int kb, const double* tau, int j0, double* T) {
    // S, T: WY_NB x WY_NB column-major (ld WY_NB); T upper triangular
    __shared__ double t[WY_NB][WY_NB + 1];
    const int r = threadIdx.x;
    for (int e = r; e < WY_NB * WY_NB; e += blockDim.x) t[e % WY_NB][e / WY_NB] = 0.0;
    __syncthreads();
    for (int i = 0; i < kb; ++i) {
        const double ti = tau[j0 + i];
        double val = 0.0;
        if (r < i) {
            double s = 0.0;
            for (int c = r; c < i; ++c) s += t[r][c] * S[c + i * WY_NB];
            val = -ti * s;
        }
        __syncthreads();
        if (r < i) t[r][i] = val;
        if (r == i) t[i][i] = ti;
        __syncthreads();
    }
    for (int e = r; e < WY_NB * WY_NB; e += blockDim.x) T[e] = t[e % WY_NB][e / WY_NB];
}

size_t apply_q_work_elems(long long m, long long ncols) {
    return (size_t)m * WY_NB + 2 * WY_NB * WY_NB + 2 * (size_t)WY_NB * ncols;
}

int apply_q_wy(const double* Vr, long long m, int k, long long ldv, const double* tau, double* C, long long ldc,
               long long ncols, double* work, cudaStream_t st) {
    double* Vp = work;                                  // m x WY_NB (ld m)
    double* S = Vp + (size_t)m * WY_NB;                 // WY_NB x WY_NB
    double* T = S + WY_NB * WY_NB;
    double* W1 = T + WY_NB * WY_NB;                     // WY_NB x ncols
    double* W2 = W1 + (size_t)WY_NB * ncols;
    const int npan = (k + WY_NB - 1) / WY_NB;
    for (int pnl = npan - 1; pnl >= 0; --pnl) {
        const int j0 = pnl * WY_NB;
        const int kb = k - j0 < WY_NB ? k - j0 : WY_NB;
        const long long rows = m - j0;
        const long long ldp = m;
        int gx = (int)ceil_div(rows, 256);
        if (gx > 128) gx = 128;
        k_make_panel<<<dim3(gx, WY_NB), 256, 0, st>>>(Vr, ldv, m, j0, kb, Vp, ldp);
        MPJ_LAUNCHED();
        int rc = gemm_f64(1, 0, WY_NB, WY_NB, rows, 1.0, Vp, ldp, Vp, ldp, 0.0, S, WY_NB, st);
        if (rc) return rc;
        k_larft<<<1, WY_NB, 0, st>>>(S, kb, tau, j0, T);
        MPJ_LAUNCHED();
        rc = gemm_f64(1, 0, WY_NB, ncols, rows, 1.0, Vp, ldp, C + j0, ldc, 0.0, W1, WY_NB, st);
        if (rc) return rc;
        rc = gemm_f64(0, 0, WY_NB, ncols, WY_NB, 1.0, T, WY_NB, W1, WY_NB, 0.0, W2, WY_NB, st);
        if (rc) return rc;
        rc = gemm_f64(0, 0, rows, ncols, WY_NB, -1.0, Vp, ldp, W2, WY_NB, 1.0, C + j0, ldc, st);
        if (rc) return rc;
    }
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mpj
