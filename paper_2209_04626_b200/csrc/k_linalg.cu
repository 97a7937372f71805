// k_linalg.cu -- dense fp64 building blocks of the precision switch
// (QR of V by CholeskyQR, reading c-11), the R*V product
// ("Y <- X Q") and the assembly U = Q_p U_X, V = P Q_t V_X
// by blocked compact-WY reflector application.
#include <cuda_runtime.h>
#include "common.cuh"
#include "jacobi.h"

namespace mpj {

// ------------------------------------------------------------------------
// fp64 GEMM on the FP64 tensor pipe (DMMA, mma.sync.m8n8k4.f64):
// C = alpha op(A) op(B) + beta C, column-major, any M, N, K, lda, ldb.
// CTA tile 128 x 64, k-tile 16, 8 warps (4 x 2) with 32 x 32 warp tiles
// (4 x 4 DMMA tiles, 32 fp64 accumulators per thread), 3-stage cp.async
// pipeline.  Both operands are staged k-major (As[k][m], Bs[k][n]) with row
// strides 132 / 68 doubles (= 4 mod 16): the 16-lane phases of every
// fragment load hit 16 distinct 8-byte banks.  Contiguous, aligned runs are
// copied with 16-byte cp.async, everything else (transposed operands,
// ragged edges) with 8-byte cp.async; out-of-range elements are zero-filled.
// ------------------------------------------------------------------------
#ifndef MPJ_GM_BK
#define MPJ_GM_BK 16
#endif
#ifndef MPJ_GM_ST
#define MPJ_GM_ST 3
#endif
constexpr int GM_BM = 128, GM_BN = 64, GM_BK = MPJ_GM_BK, GM_ST = MPJ_GM_ST;
constexpr int GM_SA = GM_BM + 4, GM_SB = GM_BN + 4;

__device__ __forceinline__ void dmma884_l(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void cpa8(double* dst, const double* src, bool valid) {
    unsigned saddr = (unsigned)__cvta_generic_to_shared(dst);
    int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cpa16(double* dst, const double* src, int valid_elems) {
    unsigned saddr = (unsigned)__cvta_generic_to_shared(dst);
    int sz = valid_elems * 8;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(src), "r"(sz));
}

// Stage a (rows x 16) k-slab of op(A) (rows = M direction).  KF = false: the operand is r-fast in memory
// (element (r, k) at P[r + k*ld]) and lands k-major, S[k][r] (row stride SROW); KF = true: it is k-fast
// (element (r, k) at P[k + r*ld]) and lands r-major, S[r][k] (row stride GM_SK), so that both layouts move
// 16-byte runs (round 1 scattered k-fast operands into S[k][r] with one 8-byte cp.async per element).
constexpr int GM_SK = GM_BK + 4;   // = 4 mod 16 doubles: conflict-free fragment loads along k
template <int ROWS, int SROW, bool KF>
__device__ __forceinline__ void gm_stage(double* S, const double* __restrict__ P, long long ld, bool vec_ok,
                                         long long r0, long long k0, long long R, long long K) {
    const int tid = threadIdx.x;
    if (!KF && vec_ok) {
        // 16-byte chunks along r: ROWS/2 chunks per k
        for (int v = tid; v < GM_BK * (ROWS / 2); v += 256) {
            const int kk = v / (ROWS / 2), rr = (v % (ROWS / 2)) * 2;
            const long long gr = r0 + rr, gk = k0 + kk;
            int valid = (gk < K) ? (int)max(0LL, min(2LL, R - gr)) : 0;
            const double* src = valid ? P + gr + gk * ld : P;
            cpa16(&S[kk * SROW + rr], src, valid);
        }
    } else if (!KF) {
        for (int v = tid; v < GM_BK * ROWS; v += 256) {
            const int kk = v / ROWS, rr = v % ROWS;
            const long long gr = r0 + rr, gk = k0 + kk;
            const bool valid = gr < R && gk < K;
            cpa8(&S[kk * SROW + rr], valid ? P + gr + gk * ld : P, valid);
        }
    } else if (vec_ok) {
        // 16-byte chunks along k: GM_BK/2 chunks per row
        for (int v = tid; v < ROWS * (GM_BK / 2); v += 256) {
            const int rr = v / (GM_BK / 2), kk = (v % (GM_BK / 2)) * 2;
            const long long gr = r0 + rr, gk = k0 + kk;
            int valid = (gr < R) ? (int)max(0LL, min(2LL, K - gk)) : 0;
            const double* src = valid ? P + gk + gr * ld : P;
            cpa16(&S[rr * GM_SK + kk], src, valid);
        }
    } else {
        for (int v = tid; v < GM_BK * ROWS; v += 256) {
            const int kk = v % GM_BK, rr = v / GM_BK;
            const long long gr = r0 + rr, gk = k0 + kk;
            const bool valid = gr < R && gk < K;
            cpa8(&S[rr * GM_SK + kk], valid ? P + gk + gr * ld : P, valid);
        }
    }
}

template <bool AKF, bool BKF>
constexpr size_t gemm_smem() {
    return sizeof(double) * (size_t)GM_ST * ((AKF ? GM_BM * GM_SK : GM_BK * GM_SA) + (BKF ? GM_BN * GM_SK : GM_BK * GM_SB));
}

// AKF: op(A) is k-fast in memory (ta == 1); BKF: op(B) is k-fast (tb == 0)
template <bool AKF, bool BKF>
__global__ void __launch_bounds__(256) k_gemm_f64(long long M, long long N, long long K,
                                                  double alpha, const double* __restrict__ A, long long lda,
                                                  const double* __restrict__ B, long long ldb, double beta,
                                                  double* __restrict__ C, long long ldc, int vec_a, int vec_b,
                                                  long long kchunk, double* __restrict__ part, int shape) {
    constexpr int ASZ = AKF ? GM_BM * GM_SK : GM_BK * GM_SA, BSZ = BKF ? GM_BN * GM_SK : GM_BK * GM_SB;
    extern __shared__ __align__(16) unsigned char gm_smem[];
    double* As = reinterpret_cast<double*>(gm_smem);                  // [ST][ASZ]
    double* Bs = As + GM_ST * ASZ;                                    // [ST][BSZ]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;                          // 4 x 2 warps
    const long long i0 = (long long)blockIdx.x * GM_BM, j0 = (long long)blockIdx.y * GM_BN;
    // shape bit 0: only the upper triangle of C is wanted -> skip tiles strictly below the diagonal
    if ((shape & 1) && j0 + GM_BN <= i0) return;
    // shape bit 1: op(A) is lower triangular -> op(A)(i, k) = 0 for k > i: K range ends at the tile's last row
    if ((shape & 2) && kchunk == 0 && K > i0 + GM_BM) K = i0 + GM_BM;
    // shape bit 2: op(A) is upper triangular -> op(A)(i, k) = 0 for k < i: K range starts at the tile's first row
    if ((shape & 4) && kchunk == 0) {
        const long long k0 = min(K, (i0 / GM_BK) * GM_BK);
        if (!AKF) A += k0 * lda; else A += k0;
        if (BKF) B += k0; else B += k0 * ldb;
        K -= k0;
    }
    // split-K: this CTA covers k in [kb, kb + kchunk) of op(A)/op(B); partial results go to part
    const long long kb = (long long)blockIdx.z * kchunk;
    if (kchunk > 0) {
        const long long ke = min(K, kb + kchunk);
        if (!AKF) A += kb * lda; else A += kb;
        if (BKF) B += kb; else B += kb * ldb;
        K = ke - kb;
    }
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const long long nk = (K + GM_BK - 1) / GM_BK;
    // op(A) (i,k): ta == 0 -> A[i + k lda] (i fast); ta == 1 -> A[k + i lda]
    // op(B) (k,j): tb == 0 -> B[k + j ldb] (k fast); tb == 1 -> B[j + k ldb] (j fast)
    auto stage = [&](long long kt, int st) {
        gm_stage<GM_BM, GM_SA, AKF>(As + st * ASZ, A, lda, vec_a, i0, kt * GM_BK, M, K);
        gm_stage<GM_BN, GM_SB, BKF>(Bs + st * BSZ, B, ldb, vec_b, j0, kt * GM_BK, N, K);
    };
#pragma unroll
    for (int s0 = 0; s0 < GM_ST - 1; ++s0) {
        if (s0 < nk) stage(s0, s0);
        asm volatile("cp.async.commit_group;\n" ::);
    }
    for (long long kt = 0; kt < nk; ++kt) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(GM_ST - 2));
        __syncthreads();
        if (kt + GM_ST - 1 < nk) stage(kt + GM_ST - 1, (int)((kt + GM_ST - 1) % GM_ST));
        asm volatile("cp.async.commit_group;\n" ::);
        const double* as = As + (kt % GM_ST) * ASZ;
        const double* bs = Bs + (kt % GM_ST) * BSZ;
#pragma unroll
        for (int k0 = 0; k0 < GM_BK; k0 += 4) {
            double fa[4], fb[4];
            const int kq = k0 + (lane & 3);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int m = wm * 32 + 8 * i + (lane >> 2);
                fa[i] = AKF ? as[m * GM_SK + kq] : as[kq * GM_SA + m];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int nn = wn * 32 + 8 * j + (lane >> 2);
                fb[j] = BKF ? bs[nn * GM_SK + kq] : bs[kq * GM_SB + nn];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884_l(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const long long gi = i0 + wm * 32 + 8 * i + (lane >> 2);
        if (gi >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const long long gj = j0 + wn * 32 + 8 * j + 2 * (lane & 3) + h;
                if (gj >= N) continue;
                if (part) {
                    part[((long long)blockIdx.z * N + gj) * M + gi] = acc[i][j][h];
                } else {
                    double* c = C + gi + gj * ldc;
                    *c = beta == 0.0 ? alpha * acc[i][j][h] : alpha * acc[i][j][h] + beta * *c;
                }
            }
        }
    }
}

// deterministic split-K reduction: C = alpha sum_s part_s + beta C (fixed order)
__global__ void k_splitk_reduce(const double* __restrict__ part, int nsplit, long long M, long long N, double alpha,
                                double beta, double* __restrict__ C, long long ldc) {
    const long long total = M * N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const long long i = e % M, j = e / M;
        double s = 0.0;
        for (int z = 0; z < nsplit; ++z) s += part[(long long)z * total + e];
        double* c = C + i + j * ldc;
        *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
    }
}

static thread_local double* g_gemm_ws = nullptr;
static thread_local size_t g_gemm_ws_elems = 0;
void gemm_set_workspace(double* ws, size_t elems) {
    g_gemm_ws = ws;
    g_gemm_ws_elems = elems;
}

template <bool AKF, bool BKF>
static int gemm_launch(long long M, long long N, long long K, double alpha, const double* A, long long lda,
                       const double* B, long long ldb, double beta, double* C, long long ldc, int shape,
                       cudaStream_t st) {
    constexpr size_t smem = gemm_smem<AKF, BKF>();
    MPJ_CUDA_TRY(set_smem(k_gemm_f64<AKF, BKF>, smem));
    const int vec_a = (lda % 2 == 0) && (((uintptr_t)A & 15) == 0);
    const int vec_b = (ldb % 2 == 0) && (((uintptr_t)B & 15) == 0);
    dim3 grid((unsigned)ceil_div(M, GM_BM), (unsigned)ceil_div(N, GM_BN));
    // split K when the output tiles cannot fill the GPU (skinny WY / Gram products)
    const long long tiles = (long long)grid.x * grid.y;
    long long nsplit = 1;
    if (tiles < 148 && K >= 1024 && g_gemm_ws && shape == 0) {
        nsplit = ceil_div(2 * 148, tiles);
        nsplit = min(nsplit, K / 256);
        nsplit = min(nsplit, (long long)(g_gemm_ws_elems / (size_t)(M * N)));
        nsplit = min(nsplit, 64LL);
    }
    if (nsplit > 1) {
        const long long kchunk = round_up(ceil_div(K, nsplit), GM_BK);
        nsplit = ceil_div(K, kchunk);
        grid.z = (unsigned)nsplit;
        k_gemm_f64<AKF, BKF><<<grid, 256, smem, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, vec_a, vec_b,
                                                      kchunk, g_gemm_ws, 0);
        MPJ_LAUNCHED();
        long long gr = ceil_div(M * N, 256);
        if (gr > 4096) gr = 4096;
        k_splitk_reduce<<<(unsigned)gr, 256, 0, st>>>(g_gemm_ws, (int)nsplit, M, N, alpha, beta, C, ldc);
        MPJ_LAUNCHED();
    } else {
        k_gemm_f64<AKF, BKF><<<grid, 256, smem, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, vec_a, vec_b,
                                                      0, nullptr, shape);
        MPJ_LAUNCHED();
    }
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

int gemm_f64_ex(int ta, int tb, long long M, long long N, long long K, double alpha, const double* A, long long lda,
                const double* B, long long ldb, double beta, double* C, long long ldc, int shape, cudaStream_t st) {
    if (M <= 0 || N <= 0) return 0;
    if (ta == 0 && tb == 1) return gemm_launch<false, false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, shape, st);
    if (ta == 0 && tb == 0) return gemm_launch<false, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, shape, st);
    if (ta == 1 && tb == 1) return gemm_launch<true, false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, shape, st);
    return gemm_launch<true, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, shape, st);
}

int gemm_f64(int ta, int tb, long long M, long long N, long long K, double alpha, const double* A, long long lda,
             const double* B, long long ldb, double beta, double* C, long long ldc, cudaStream_t st) {
    return gemm_f64_ex(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 0, st);
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
            int rc = gemm_f64_ex(1, 0, rest, rest, kb, -1.0, U12, ldg, U12, ldg, 1.0, A22, ldg, 1, st);   // upper only
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
constexpr int WY_NB = WY_PANEL;   // panel of the WY application / blocked QR
constexpr int LT_NB = 64;    // block of the T formation (k_larft)

__global__ void k_make_panel(const double* Vr, long long ldv, long long m, int j0, int kb, double* Vp,
                             long long ldp) {
    const int c = blockIdx.y;
    const long long rows = m - j0;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < ldp; r += (long long)gridDim.x * blockDim.x) {
        double v;
        if (c >= kb || r >= rows) v = 0.0;
        else if (r == c) v = 1.0;
        else if (r < c) v = 0.0;
        else v = Vr[(j0 + r) + (long long)(j0 + c) * ldv];
        Vp[r + (long long)c * ldp] = v;
    }
}

// T of the compact WY form (LAPACK xLARFT 'F','C'): column i of T is
// -tau_i T[0:i, 0:i] S[0:i, i], T[i][i] = tau_i.  S (the strict upper part of
// Vp^T Vp) and tau are staged in shared memory first, so the kb dependent
// steps run on shared memory only.
__global__ void k_larft(const double* S, int kb_all, const double* tau, double* T) {
    // CTA z forms the diagonal block z (reflectors z LT_NB .. z LT_NB + kb - 1) of the panel's T
    const int j0 = blockIdx.x * LT_NB;
    const int kb = kb_all - j0 < LT_NB ? kb_all - j0 : LT_NB;
    S += j0 + (long long)j0 * WY_NB;
    T += j0 + (long long)j0 * WY_NB;
    // S, T: LT_NB x LT_NB blocks of ld WY_NB matrices (column-major); T upper triangular.
    // LT_NB x 8 threads: row r = tid / 8, the 8 lanes of a row split the dot product T[r, r:i] S[r:i, i].
    // Step i reads columns < i of t and writes column i, so one barrier per step suffices.
    extern __shared__ double lsm[];
    double* t = lsm;                                  // [LT_NB][LT_NB + 1]: t[r * (LT_NB + 1) + c]
    double* sv = t + LT_NB * (LT_NB + 1);             // [LT_NB][LT_NB + 1]: S
    double* ts = sv + LT_NB * (LT_NB + 1);            // tau
    constexpr int LS = LT_NB + 1;
    const int tid = threadIdx.x, r = tid >> 3, q = tid & 7;
    for (int e = tid; e < LT_NB * LT_NB; e += blockDim.x) {
        const int a = e % LT_NB, c = e / LT_NB;
        t[a * LS + c] = 0.0;
        sv[a * LS + c] = S[a + (long long)c * WY_NB];
    }
    if (tid < kb) ts[tid] = tau[j0 + tid];
    __syncthreads();
    for (int i = 0; i < kb; ++i) {
        double s = 0.0;
        if (r < i)
            for (int c = r + q; c < i; c += 8) s += t[r * LS + c] * sv[c * LS + i];
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        if (q == 0) {
            if (r < i) t[r * LS + i] = -ts[i] * s;
            else if (r == i) t[i * LS + i] = ts[i];
        }
        __syncthreads();
    }
    for (int e = tid; e < LT_NB * LT_NB; e += blockDim.x) T[(e % LT_NB) + (long long)(e / LT_NB) * WY_NB] = t[(e % LT_NB) * LS + e / LT_NB];
}
static size_t larft_smem() { return sizeof(double) * (2 * (size_t)LT_NB * (LT_NB + 1) + LT_NB); }

size_t apply_q_work_elems(long long m, long long ncols) {
    return (size_t)round_up(m, 32) * WY_NB + 3 * WY_NB * WY_NB + 2 * (size_t)WY_NB * ncols;
}

// C <- H C with H = H_0 ... H_{kb-1} (trans = 0) or H^T (trans = 1) for ONE
// panel of kb <= WY_NB reflectors stored below the diagonal of P (rows
// `rows`, ld ldp; reflector i has its unit at row i).
static int apply_panel(const double* P, long long ldp, long long rows, int kb, const double* tau, double* C,
                       long long ldc, long long ncols, int trans, double* work, cudaStream_t st,
                       const double* t_in = nullptr, double* t_out = nullptr, bool reuse = false) {
    const long long ldw = round_up(rows, 32);
    double* Vp = work;                                  // rows x WY_NB (ld ldw)
    double* S = Vp + (size_t)ldw * WY_NB;               // WY_NB x WY_NB
    double* T = S + WY_NB * WY_NB;
    double* T12w = T + WY_NB * WY_NB;                   // WY_NB x WY_NB scratch (recursive T)
    double* W1 = T12w + WY_NB * WY_NB;                  // WY_NB x ncols
    double* W2 = W1 + (size_t)WY_NB * ncols;
    int gx = (int)ceil_div(rows, 256);
    if (gx > 128) gx = 128;
    int rc = 0;
    if (reuse) goto apply;                              // Vp and T of this panel are still in work
    k_make_panel<<<dim3(gx, WY_NB), 256, 0, st>>>(P, ldp, rows, 0, kb, Vp, ldw);
    MPJ_LAUNCHED();
    if (t_in) {
        // T of this panel was formed by the factorisation that produced the reflectors
        MPJ_CUDA_TRY(cudaMemcpyAsync(T, t_in, sizeof(double) * WY_NB * WY_NB, cudaMemcpyDeviceToDevice, st));
        goto apply;
    }
    rc = gemm_f64(1, 0, WY_NB, WY_NB, rows, 1.0, Vp, ldw, Vp, ldw, 0.0, S, WY_NB, st);
    if (rc) return rc;
    MPJ_CUDA_TRY(set_smem(k_larft, (size_t)(larft_smem())));
    // T in LT_NB blocks: diagonal blocks by k_larft, then the recursive coupling
    // T[0:a, a:b] = -T[0:a, 0:a] S[0:a, a:b] T[a:b, a:b] (LAPACK xLARFT, recursive form)
    MPJ_CUDA_TRY(cudaMemsetAsync(T, 0, sizeof(double) * WY_NB * WY_NB, st));
    k_larft<<<(unsigned)ceil_div(kb, LT_NB), LT_NB * 8, larft_smem(), st>>>(S, kb, tau, T);   // diagonal blocks
    MPJ_LAUNCHED();
    for (int b0 = LT_NB; b0 < kb; b0 += LT_NB) {
        const int bk = kb - b0 < LT_NB ? kb - b0 : LT_NB;
        {
            // W = S[0:b0, b0:b0+bk] T22 ; T12 = -T11 W
            rc = gemm_f64(0, 0, b0, bk, bk, 1.0, S + (long long)b0 * WY_NB, WY_NB, T + b0 + (long long)b0 * WY_NB,
                          WY_NB, 0.0, T12w, WY_NB, st);
            if (rc) return rc;
            rc = gemm_f64(0, 0, b0, bk, b0, -1.0, T, WY_NB, T12w, WY_NB, 0.0, T + (long long)b0 * WY_NB, WY_NB, st);
            if (rc) return rc;
        }
    }
    if (t_out) MPJ_CUDA_TRY(cudaMemcpyAsync(t_out, T, sizeof(double) * WY_NB * WY_NB, cudaMemcpyDeviceToDevice, st));
    if (!C) return 0;                                   // T only (wy_tfactors)
apply:
    // transposed products keep the long dimension (ncols) in the GEMM's M: W1^T = C^T Vp,
    // W2^T = W1^T T^(T) (T^T for trans), C -= Vp W2 = Vp (W2^T)^T
    rc = gemm_f64(1, 0, ncols, WY_NB, rows, 1.0, C, ldc, Vp, ldw, 0.0, W1, ncols, st);
    if (rc) return rc;
    rc = gemm_f64(0, trans ? 0 : 1, ncols, WY_NB, WY_NB, 1.0, W1, ncols, T, WY_NB, 0.0, W2, ncols, st);
    if (rc) return rc;
    rc = gemm_f64(0, 1, rows, ncols, WY_NB, -1.0, Vp, ldw, W2, ncols, 1.0, C, ldc, st);
    return rc;
}

// T factors of every WY panel of Q = H_0 ... H_{k-1} (reflectors as left by qr_blocked / the QRP), for a later
// apply_q_wy with tcache (all panels cached); work as for apply_q_wy with ncols = 0
int wy_tfactors(const double* Vr, long long m, int k, long long ldv, const double* tau, double* tcache, double* work,
                cudaStream_t st) {
    const int npan = (k + WY_NB - 1) / WY_NB;
    for (int pnl = 0; pnl < npan; ++pnl) {
        const int j0 = pnl * WY_NB;
        const int kb = k - j0 < WY_NB ? k - j0 : WY_NB;
        int rc = apply_panel(Vr + j0 + (long long)j0 * ldv, ldv, m - j0, kb, tau + j0, nullptr, 1, 0, 0, work, st,
                             nullptr, tcache + (size_t)pnl * WY_NB * WY_NB);
        if (rc) return rc;
    }
    return 0;
}

int apply_q_wy(const double* Vr, long long m, int k, long long ldv, const double* tau, double* C, long long ldc,
               long long ncols, double* work, cudaStream_t st, const double* tcache, int ncached) {
    const int npan = (k + WY_NB - 1) / WY_NB;
    for (int pnl = npan - 1; pnl >= 0; --pnl) {
        const int j0 = pnl * WY_NB;
        const int kb = k - j0 < WY_NB ? k - j0 : WY_NB;
        const double* tin = tcache && pnl < ncached ? tcache + (size_t)pnl * WY_NB * WY_NB : nullptr;
        int rc = apply_panel(Vr + j0 + (long long)j0 * ldv, ldv, m - j0, kb, tau + j0, C + j0, ldc, ncols, 0, work, st,
                             tin);
        if (rc) return rc;
    }
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// Q = H_0 ... H_{k-1} I formed in place on C (m x m, must hold the identity on entry; LAPACK xORGQR
// order): panels are applied last to first, and before panel j0 is applied C is the identity outside
// C[j0:, j0:], so the panel only touches that trailing block (4/3 m^3 instead of 2 m^3 flops).
int form_q_wy(const double* Vr, long long m, int k, long long ldv, const double* tau, double* C, long long ldc,
              double* work, cudaStream_t st, const double* tcache, int ncached) {
    const int npan = (k + WY_NB - 1) / WY_NB;
    for (int pnl = npan - 1; pnl >= 0; --pnl) {
        const int j0 = pnl * WY_NB;
        const int kb = k - j0 < WY_NB ? k - j0 : WY_NB;
        const double* tin = tcache && pnl < ncached ? tcache + (size_t)pnl * WY_NB * WY_NB : nullptr;
        int rc = apply_panel(Vr + j0 + (long long)j0 * ldv, ldv, m - j0, kb, tau + j0, C + j0 + (long long)j0 * ldc,
                             ldc, m - j0, 0, work, st, tin);
        if (rc) return rc;
    }
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// Blocked Householder QR (LAPACK xGEQRF structure): panels of WY_NB columns
// factored by the cooperative unblocked kernel (one CTA per column), trailing
// matrix updated with the panel's compact-WY form Q^T = I - V T^T V^T on the
// DMMA GEMM.  Used for the tall QR and the LQ of R
// (QR of R^T).  Same reflectors / R as the unblocked algorithm
// up to rounding.
static int factor_panel(double* Pn, long long lda, int rows, int kb, double* tau, QrWork& w, cudaStream_t st) {
    if (w.ready) return qr_panel_chain(Pn, lda, rows, kb, tau, w.ready, st);
    QrWork wp = w;
    int grid = 0;
    int rc = qr_coop_grid(rows, &grid);
    if (rc) return rc;
    wp.grid = grid < kb ? grid : kb;
    return qr_coop(Pn, lda, rows, kb, tau, 0, wp, nullptr, st);
}

int qr_blocked(double* A, long long lda, int m, int n, double* tau, QrWork& w, double* work, cudaStream_t st,
               double* tcache) {
    if (w.ready && w.la_stream && n > WY_NB) {
        // look-ahead (LAPACK-style): panel p's reflectors update panel p+1's columns first; panel p+1 is then
        // factored on la_stream while the rest of p's trailing update runs here
        int rc = factor_panel(A, lda, m, n < WY_NB ? n : WY_NB, tau, w, st);
        if (rc) return rc;
        for (int j0 = 0; j0 < n; j0 += WY_NB) {
            const int kb = n - j0 < WY_NB ? n - j0 : WY_NB;
            double* Pn = A + j0 + (long long)j0 * lda;
            if (j0 > 0) MPJ_CUDA_TRY(cudaStreamWaitEvent(st, w.la_ev1, 0));
            const int j1 = j0 + kb;
            if (j1 >= n) break;
            const int kb1 = n - j1 < WY_NB ? n - j1 : WY_NB;
            double* tslot = tcache ? tcache + (size_t)(j0 / WY_NB) * WY_NB * WY_NB : nullptr;
            rc = apply_panel(Pn, lda, m - j0, kb, tau + j0, Pn + (long long)kb * lda, lda, kb1, 1, work, st, nullptr,
                             tslot);
            if (rc) return rc;
            MPJ_CUDA_TRY(cudaEventRecord(w.la_ev0, st));
            MPJ_CUDA_TRY(cudaStreamWaitEvent(w.la_stream, w.la_ev0, 0));
            rc = factor_panel(A + j1 + (long long)j1 * lda, lda, m - j1, kb1, tau + j1, w, w.la_stream);
            if (rc) return rc;
            MPJ_CUDA_TRY(cudaEventRecord(w.la_ev1, w.la_stream));
            if (j1 + kb1 < n) {
                rc = apply_panel(Pn, lda, m - j0, kb, tau + j0, Pn + (long long)(kb + kb1) * lda, lda, n - j1 - kb1, 1,
                                 work, st, nullptr, nullptr, true);
                if (rc) return rc;
            }
        }
        MPJ_CUDA_TRY(cudaGetLastError());
        return 0;
    }
    for (int j0 = 0; j0 < n; j0 += WY_NB) {
        const int kb = n - j0 < WY_NB ? n - j0 : WY_NB;
        double* Pn = A + j0 + (long long)j0 * lda;
        int rc = factor_panel(Pn, lda, m - j0, kb, tau + j0, w, st);
        if (rc) return rc;
        if (j0 + kb < n) {
            rc = apply_panel(Pn, lda, m - j0, kb, tau + j0, Pn + (long long)kb * lda, lda, n - j0 - kb, 1, work, st,
                             nullptr, tcache ? tcache + (size_t)(j0 / WY_NB) * WY_NB * WY_NB : nullptr);
            if (rc) return rc;
        }
    }
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mpj
