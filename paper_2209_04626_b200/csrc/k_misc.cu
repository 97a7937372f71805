// k_misc.cu -- bandwidth-bound kernels of the path: input validation, layout
// moves between the factorisation stages, the fp32 downcast (reading c-9),
// column norms / descending sort (Alg. 1),
// finalisation and the permutation of V, gate measures
// (PAPER.md:429-431).
#include <cuda_runtime.h>
#include <float.h>
#include "common.cuh"
#include "jacobi.h"

namespace mpj {

static inline dim3 grid2d(long long rows, long long cols, int bx = 256) {
    long long gx = ceil_div(rows, bx);
    if (gx > 64) gx = 64;
    long long gy = cols > 65535 ? 65535 : cols;
    return dim3((unsigned)gx, (unsigned)gy);
}

__global__ void k_check_finite(const double* A, long long lda, long long m, long long n, int* bad) {
    int found = 0;
    for (long long j = blockIdx.y; j < n; j += gridDim.y)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
            if (!isfinite(A[i + j * lda])) found = 1;
    if (__syncthreads_or(found) && threadIdx.x == 0) atomicOr(bad, 1);
}
int check_finite(const double* A, long long lda, long long m, long long n, int* bad, cudaStream_t st) {
    k_check_finite<<<grid2d(m, n), 256, 0, st>>>(A, lda, m, n, bad);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

__global__ void k_copy(const double* src, long long lds, double* dst, long long ldd, long long rows, long long cols) {
    for (long long j = blockIdx.y; j < cols; j += gridDim.y)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows; i += (long long)gridDim.x * blockDim.x)
            dst[i + j * ldd] = src[i + j * lds];
}
int copy_matrix(const double* src, long long lds, double* dst, long long ldd, long long rows, long long cols,
                cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return 0;
    k_copy<<<grid2d(rows, cols), 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

template <typename T>
__global__ void k_set_identity(T* A, long long lda, long long rows_pad, long long n) {
    for (long long j = blockIdx.y; j < n; j += gridDim.y)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows_pad; i += (long long)gridDim.x * blockDim.x)
            A[i + j * lda] = i == j ? T(1) : T(0);
}
template <typename T>
int set_identity(T* A, long long lda, long long rows_pad, long long n, cudaStream_t st) {
    k_set_identity<T><<<grid2d(rows_pad, n), 256, 0, st>>>(A, lda, rows_pad, n);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}
template int set_identity<float>(float*, long long, long long, long long, cudaStream_t);
template int set_identity<double>(double*, long long, long long, long long, cudaStream_t);

// Rt = R^T for the upper triangle of R (zeros elsewhere, padding rows zero)
__global__ void k_transpose_upper(const double* R, long long ldr, double* Rt, long long ldt, int n, long long rows_pad) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;   // tile of Rt: rows bx.., cols by..
    const int tx = threadIdx.x, ty = threadIdx.y;           // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        int rr = by + tx, cc = bx + k;                      // coalesced read of R[rr][cc] (-> Rt[cc][rr])
        double v = 0.0;
        if (rr < n && cc < n && rr <= cc) v = R[rr + (long long)cc * ldr];
        tile[k][tx] = v;                                    // tile[k][t] = R[by+t][bx+k]
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        long long row = bx + tx, col = by + k;              // Rt[row][col] = R[col][row]
        if (row < rows_pad && col < n) Rt[row + col * ldt] = (row < n) ? tile[tx][k] : 0.0;
    }
}
int transpose_upper(const double* R, long long ldr, double* Rt, long long ldt, int n, long long rows_pad,
                    cudaStream_t st) {
    dim3 g((unsigned)ceil_div(rows_pad, 32), (unsigned)ceil_div(n, 32));
    k_transpose_upper<<<g, dim3(32, 8), 0, st>>>(R, ldr, Rt, ldt, n, rows_pad);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// X = L = (upper(Rt))^T : X[i][j] = Rt[j][i] for i >= j, else 0
__global__ void k_lower_from_rt(const double* Rt, long long ldt, double* X, long long ldx, int n, long long rows_pad) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;   // tile of X: rows bx.., cols by..
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int k = ty; k < 32; k += 8) {
        int rr = by + tx, cc = bx + k;                      // coalesced read of Rt[rr][cc] (-> X[cc][rr])
        double v = 0.0;
        if (rr < n && cc < n && rr <= cc) v = Rt[rr + (long long)cc * ldt];
        tile[k][tx] = v;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        long long row = bx + tx, col = by + k;
        if (row < rows_pad && col < n) X[row + col * ldx] = (row < n) ? tile[tx][k] : 0.0;
    }
}
int lower_from_rt(const double* Rt, long long ldt, double* X, long long ldx, int n, long long rows_pad,
                  cudaStream_t st) {
    dim3 g((unsigned)ceil_div(rows_pad, 32), (unsigned)ceil_div(n, 32));
    k_lower_from_rt<<<g, dim3(32, 8), 0, st>>>(Rt, ldt, X, ldx, n, rows_pad);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

__global__ void k_upper_of(const double* A, long long lda, double* R, long long ldr, int n, long long rows_pad) {
    for (long long j = blockIdx.y; j < n; j += gridDim.y)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows_pad; i += (long long)gridDim.x * blockDim.x)
            R[i + j * ldr] = (i <= j && i < n) ? A[i + j * lda] : 0.0;
}
int upper_of(const double* A, long long lda, double* R, long long ldr, int n, long long rows_pad, cudaStream_t st) {
    k_upper_of<<<grid2d(rows_pad, n), 256, 0, st>>>(A, lda, R, ldr, n, rows_pad);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

__global__ void k_maxabs(const double* A, long long lda, long long rows, long long cols, double* out) {
    __shared__ double red[32];
    double mx = 0.0;
    for (long long j = blockIdx.y; j < cols; j += gridDim.y)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows; i += (long long)gridDim.x * blockDim.x)
            mx = fmax(mx, fabs(A[i + j * lda]));
    mx = block_max(mx, red);
    if (threadIdx.x == 0) atomic_max_nonneg(out, mx);
}
int maxabs(const double* A, long long lda, long long rows, long long cols, double* out, cudaStream_t st) {
    MPJ_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st));
    dim3 g = grid2d(rows, cols);
    if (g.y > 2048) g.y = 2048;
    k_maxabs<<<g, 256, 0, st>>>(A, lda, rows, cols, out);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// X32 = fl32(X 2^-e), e = exponent of max|X| (max 2^-e in [0.5, 1)), reading c-9
__global__ void k_downcast(const double* X, long long ldx, float* X32, long long ld32, long long rows_pad, int n,
                           const double* mx) {
    int e = 0;
    frexp(*mx, &e);
    for (long long j = blockIdx.y; j < n; j += gridDim.y)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows_pad; i += (long long)gridDim.x * blockDim.x)
            X32[i + j * ld32] = (float)ldexp(X[i + j * ldx], -e);
}
int downcast_scaled(const double* X, long long ldx, float* X32, long long ld32, long long rows_pad, int n,
                    const double* maxabs_dev, cudaStream_t st) {
    k_downcast<<<grid2d(rows_pad, n), 256, 0, st>>>(X, ldx, X32, ld32, rows_pad, n, maxabs_dev);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// column norms in fp64: safe = two-pass scaled (overflow-free), else plain
template <typename T>
__global__ void k_col_norms(const T* X, long long ldx, long long rows, double* out, int safe) {
    __shared__ double red[32];
    const T* col = X + (long long)blockIdx.x * ldx;
    double scale = 1.0;
    if (safe) {
        double mx = 0.0;
        for (long long i = threadIdx.x; i < rows; i += blockDim.x) mx = fmax(mx, fabs((double)col[i]));
        mx = block_max(mx, red);
        if (mx == 0.0) { if (threadIdx.x == 0) out[blockIdx.x] = 0.0; return; }
        scale = mx;
    }
    double s = 0.0;
    for (long long i = threadIdx.x; i < rows; i += blockDim.x) {
        double y = safe ? (double)col[i] / scale : (double)col[i];
        s += y * y;
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[blockIdx.x] = safe ? scale * sqrt(s) : sqrt(s);
}
template <typename T>
int col_norms(const T* X, long long ldx, long long rows, int n, double* out, int safe, cudaStream_t st) {
    k_col_norms<T><<<n, 256, 0, st>>>(X, ldx, rows, out, safe);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}
template int col_norms<float>(const float*, long long, long long, int, double*, int, cudaStream_t);
template int col_norms<double>(const double*, long long, long long, int, double*, int, cudaStream_t);

// stable descending rank: rank_j = #{k : key_k > key_j or (key_k == key_j and k < j)}
__global__ void k_rank_desc(const double* key, int n, int* rank) {
    __shared__ double tile[1024];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const double kj = j < n ? key[j] : 0.0;
    int r = 0;
    for (int base = 0; base < n; base += 1024) {
        __syncthreads();
        for (int t = threadIdx.x; t < 1024; t += blockDim.x) tile[t] = base + t < n ? key[base + t] : -1.0;
        __syncthreads();
        const int lim = min(1024, n - base);
        for (int t = 0; t < lim; ++t) {
            const double kk = tile[t];
            const int k = base + t;
            r += (kk > kj || (kk == kj && k < j)) ? 1 : 0;
        }
    }
    if (j < n) rank[j] = r;
}
int rank_desc(const double* key, int n, int* rank, cudaStream_t st) {
    k_rank_desc<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(key, n, rank);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// V[:, rank_j] = fl64(V32[:, j])
__global__ void k_sort_upcast(const float* V32, long long ld32, const int* rank, double* V, long long ldv,
                              long long rows_pad, int n) {
    for (long long j = blockIdx.y; j < n; j += gridDim.y) {
        const long long dj = rank[j];
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows_pad; i += (long long)gridDim.x * blockDim.x)
            V[i + dj * ldv] = (double)V32[i + j * ld32];
    }
}
int sort_upcast_v(const float* V32, long long ld32, const int* rank, double* V, long long ldv, long long rows_pad,
                  int n, cudaStream_t st) {
    k_sort_upcast<<<grid2d(rows_pad, n), 256, 0, st>>>(V32, ld32, rank, V, ldv, rows_pad, n);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// U-route: U_low[:, rank_j] = fl64(X32[:, j]) / sigma32_j (sigma32_j = ||X32[:, j]||, fp64);
// a zero column sets *bad (rank deficient, reading c-18)
__global__ void k_sort_upcast_scale(const float* X32, long long ld32, const int* rank, const double* sig,
                                    double* U, long long ldu, long long rows_pad, int n, int* bad) {
    for (long long j = blockIdx.y; j < n; j += gridDim.y) {
        const long long dj = rank[j];
        const double s = sig[j];
        if (!(s > 0.0)) {
            if (blockIdx.x == 0 && threadIdx.x == 0) *bad = 1;
            continue;
        }
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows_pad; i += (long long)gridDim.x * blockDim.x)
            U[i + dj * ldu] = (double)X32[i + j * ld32] / s;
    }
}
int sort_upcast_scale(const float* X32, long long ld32, const int* rank, const double* sig, double* U, long long ldu,
                      long long rows_pad, int n, int* bad, cudaStream_t st) {
    k_sort_upcast_scale<<<grid2d(rows_pad, n), 256, 0, st>>>(X32, ld32, rank, sig, U, ldu, rows_pad, n, bad);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// U_X[:, rank_j] = Y[:, j] / sigma_j ; V_X[:, rank_j] = Q[:, j] ; S[rank_j] = sigma_j
__global__ void k_finalize(const double* Y, long long ldy, const double* Q, long long ldq, const double* sig,
                           const int* rank, double* UX, long long ldu, double* VX, long long ldvx, double* S,
                           long long rows_pad, int n) {
    for (long long j = blockIdx.y; j < n; j += gridDim.y) {
        const long long dj = rank[j];
        const double s = sig[j];
        if (blockIdx.x == 0 && threadIdx.x == 0) S[dj] = s;
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows_pad; i += (long long)gridDim.x * blockDim.x) {
            UX[i + dj * ldu] = Y[i + j * ldy] / s;
            VX[i + dj * ldvx] = Q[i + j * ldq];
        }
    }
}
int finalize(const double* Y, long long ldy, const double* Q, long long ldq, const double* sig, const int* rank,
             double* UX, long long ldu, double* VX, long long ldvx, double* S, long long rows_pad, int n,
             cudaStream_t st) {
    k_finalize<<<grid2d(rows_pad, n), 256, 0, st>>>(Y, ldy, Q, ldq, sig, rank, UX, ldu, VX, ldvx, S, rows_pad, n);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// U_X = Y diag(1/sig) in place order (sec. 3.4 V formation); sig_j = 0 -> rank deficient
__global__ void k_scale_cols(const double* Y, long long ldy, const double* sig, double* UX, long long ldu,
                             long long rows_pad, int n, int* bad) {
    for (long long j = blockIdx.y; j < n; j += gridDim.y) {
        const double s = sig[j];
        if (!(s > 0.0)) {
            if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(bad, 1);
            continue;
        }
        const double r = 1.0 / s;
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows_pad; i += (long long)gridDim.x * blockDim.x)
            UX[i + j * ldu] = Y[i + j * ldy] * r;
    }
}
int scale_cols(const double* Y, long long ldy, const double* sig, double* UX, long long ldu, long long rows_pad,
               int n, int* bad, cudaStream_t st) {
    k_scale_cols<<<grid2d(rows_pad, n), 256, 0, st>>>(Y, ldy, sig, UX, ldu, rows_pad, n, bad);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// V[perm[k]][:] = M[k][:]
__global__ void k_scatter_rows(const double* M, long long ldm, const int* perm, double* V, long long ldv, int n) {
    for (long long j = blockIdx.y; j < n; j += gridDim.y)
        for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
            V[perm[k] + j * ldv] = M[k + j * ldm];
}
int scatter_rows_perm(const double* M, long long ldm, const int* perm, double* V, long long ldv, int n,
                      cudaStream_t st) {
    k_scatter_rows<<<grid2d(n, n), 256, 0, st>>>(M, ldm, perm, V, ldv, n);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// out2[0] = max_k R_kk, out2[1] = min_k R_kk ; bad if some R_kk <= 0
__global__ void k_diag_stats(const double* R, long long ldr, int n, double* out2, int* bad) {
    __shared__ double red[32];
    double mx = 0.0, mn = DBL_MAX;
    int z = 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        double d = R[k + (long long)k * ldr];
        mx = fmax(mx, d);
        mn = fmin(mn, d);
        if (!(d > 0.0)) z = 1;
    }
    mx = block_max(mx, red);
    mn = -block_max(-mn, red);
    if (__syncthreads_or(z) && threadIdx.x == 0) atomicOr(bad, 1);
    if (threadIdx.x == 0) { out2[0] = mx; out2[1] = mn; }
}
int diag_stats(const double* R, long long ldr, int n, double* out2, int* bad, cudaStream_t st) {
    k_diag_stats<<<1, 1024, 0, st>>>(R, ldr, n, out2, bad);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// ---- gate measure orth = || X_t^T X_t - I ||_max (fp32), PAPER.md:429-431 --
__global__ void k_gate_scale(const double* X, long long ldx, long long rows_pad, int n, float* Xt, long long ldt) {
    __shared__ double red[32];
    const long long j = blockIdx.x;
    double s = 0.0;
    for (long long i = threadIdx.x; i < rows_pad; i += blockDim.x) {
        float f = (float)X[i + j * ldx];
        s += (double)f * (double)f;
    }
    s = block_sum(s, red);
    const float d = (float)sqrt(s);
    for (long long i = threadIdx.x; i < rows_pad; i += blockDim.x)
        Xt[i + j * ldt] = d > 0.0f ? (float)X[i + j * ldx] / d : 0.0f;
}

// 128 x 128 tiles of X_t^T X_t (lower tiles only), max |g - delta| -> out.  256 threads, 8 x 8 outputs per
// thread (rows ty*4 + {0..3} and 64 + ty*4 + {0..3}, likewise columns: float4 shared-memory reads), 16-row
// K chunks double-buffered in shared memory with the next chunk prefetched into registers.
constexpr int GO_T = 128, GO_K = 16, GO_LD = GO_T + 4;
__global__ void __launch_bounds__(256) k_gate_orth(const float* __restrict__ Xt, long long ldt, long long rows_pad,
                                                   int n, double* out) {
    const int bi = blockIdx.x, bj = blockIdx.y;
    if (bj > bi) return;
    __shared__ __align__(16) float As[2][GO_K][GO_LD];
    __shared__ __align__(16) float Bs[2][GO_K][GO_LD];
    __shared__ double red[32];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    // loader: column lc = tid / 2 of the tile, rows lr .. lr + 7 of the chunk
    const int lc = tid >> 1, lr = (tid & 1) * 8;
    const long long ci = (long long)bi * GO_T + lc, cj = (long long)bj * GO_T + lc;
    const float* pa = Xt + ci * ldt + lr;
    const float* pb = Xt + cj * ldt + lr;
    const bool va = ci < n, vb = cj < n;
    float4 ra0, ra1, rb0, rb1;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    auto load = [&](long long k0) {
        ra0 = va ? __ldg(reinterpret_cast<const float4*>(pa + k0)) : z4;
        ra1 = va ? __ldg(reinterpret_cast<const float4*>(pa + k0 + 4)) : z4;
        rb0 = vb ? __ldg(reinterpret_cast<const float4*>(pb + k0)) : z4;
        rb1 = vb ? __ldg(reinterpret_cast<const float4*>(pb + k0 + 4)) : z4;
    };
    auto store = [&](int buf) {
        const float a[8] = {ra0.x, ra0.y, ra0.z, ra0.w, ra1.x, ra1.y, ra1.z, ra1.w};
        const float b[8] = {rb0.x, rb0.y, rb0.z, rb0.w, rb1.x, rb1.y, rb1.z, rb1.w};
#pragma unroll
        for (int r = 0; r < 8; ++r) { As[buf][lr + r][lc] = a[r]; Bs[buf][lr + r][lc] = b[r]; }
    };
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    load(0);
    store(0);
    __syncthreads();
    int buf = 0;
    for (long long k0 = 0; k0 < rows_pad; k0 += GO_K) {
        const bool more = k0 + GO_K < rows_pad;
        if (more) load(k0 + GO_K);
#pragma unroll
        for (int kk = 0; kk < GO_K; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (more) store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const long long gi = (long long)bi * GO_T + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
            const long long gj = (long long)bj * GO_T + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
            if (gi < n && gj < n) mx = fmax(mx, fabs((double)acc[i][j] - (gi == gj ? 1.0 : 0.0)));
        }
    mx = block_max(mx, red);
    if (tid == 0) atomic_max_nonneg(out, mx);
}

int gates_orth(const double* X, long long ldx, long long rows_pad, int n, float* Xt, long long ldt, double* out,
               cudaStream_t st) {
    k_gate_scale<<<n, 256, 0, st>>>(X, ldx, rows_pad, n, Xt, ldt);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st));
    if (ldt % 4 || rows_pad % GO_K || ((uintptr_t)Xt & 15)) return -1;   // MPJSVD_ERR_INVALID_ARG
    dim3 g((unsigned)ceil_div(n, GO_T), (unsigned)ceil_div(n, GO_T));
    k_gate_orth<<<g, 256, 0, st>>>(Xt, ldt, rows_pad, n, out);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

// ---- cond gate of AUTO (Alg. 3 l.423; DESIGN.md c-15): kappa_1(R diag(1/c)) with
// c_k = ||A1(:, perm_k)|| = ||R(:,k)||.  Z = diag(c) R^-1 = R_s^-1 comes from the triangular solve; these
// kernels give the column scales and the two 1-norms (max over columns of the absolute column sums).
__global__ void k_gate_scales(const double* a1n, const int* perm, int n, double* c, double* Z, long long ldz,
                              long long rows_pad) {
    for (long long j = blockIdx.y; j < n; j += gridDim.y) {
        const double cj = a1n[perm[j]];
        if (blockIdx.x == 0 && threadIdx.x == 0) c[j] = cj;
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows_pad; i += (long long)gridDim.x * blockDim.x)
            Z[i + j * ldz] = i == j ? cj : 0.0;
    }
}
// out = max_j (sum_{i < rows_j} |Z_ij|) / (c ? c_j : 1), rows_j = j + 1 (upper) or rows
__global__ void k_col_abs_sum_max(const double* Z, long long ldz, long long rows, int n, const double* c, int upper,
                                  double* out) {
    __shared__ double red[32];
    for (int j = blockIdx.x; j < n; j += gridDim.x) {
        const long long r = upper ? (long long)j + 1 : rows;
        double s = 0.0;
        for (long long i = threadIdx.x; i < r; i += blockDim.x) s += fabs(Z[i + (long long)j * ldz]);
        s = block_sum(s, red);
        if (threadIdx.x == 0) atomic_max_nonneg(out, c ? s / c[j] : s);
    }
}
int gate_cond_scaled(const double* R, long long ldr, const double* a1n, const int* perm, int n, double* c,
                     double* Z, long long ldz, long long rows_pad, double* out2, cudaStream_t st) {
    MPJ_CUDA_TRY(cudaMemsetAsync(out2, 0, 2 * sizeof(double), st));
    k_gate_scales<<<grid2d(rows_pad, n), 256, 0, st>>>(a1n, perm, n, c, Z, ldz, rows_pad);
    MPJ_LAUNCHED();
    k_col_abs_sum_max<<<n < 1184 ? n : 1184, 256, 0, st>>>(R, ldr, n, n, c, 1, out2);   // ||R_s||_1
    MPJ_LAUNCHED();
    int rc = trsm_right_upper(R, ldr, Z, ldz, rows_pad, n, st);                        // Z = diag(c) R^-1
    if (rc) return rc;
    k_col_abs_sum_max<<<n < 1184 ? n : 1184, 256, 0, st>>>(Z, ldz, n, n, nullptr, 0, out2 + 1);   // ||R_s^-1||_1
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mpj
