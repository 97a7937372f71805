// k_qr.cu -- Householder QR with optional Businger-Golub column pivoting as
// ONE persistent cooperative kernel ("AP = Q1 R", 350;
// 416-420 "A = Q R1"; 354 "R = L Q2" via QR of R^T).
//
// Design: physical column p is owned by CTA p % G and
// never moves; logical order lives in per-CTA copies of phys[]/pos[] that
// every CTA updates identically.  Per step k there is ONE grid barrier:
//   1. every CTA reduces the G per-CTA pivot candidates (largest partial
//      norm, ties -> lowest logical index) and swaps phys/pos;
//   2. every CTA recomputes the same reflector of the pivot column
//      (identical code + fixed reduction tree -> identical bits), so no CTA
//      waits for an owner to publish it;
//   3. each CTA applies H_k to its unprocessed owned columns (one column at a
//      time, register resident), downdates the partial norms (LAPACK xLAQP2
//      rule, reading R3) and posts its next candidate;
//   4. grid barrier.
// The owner writes v / R_kk back one step later (other CTAs are still
// reading the pivot column during step k).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <float.h>
#include <atomic>
#include "common.cuh"
#include "jacobi.h"

namespace cg = cooperative_groups;

namespace mpj {

struct QrArgs {
    double* A;
    long long lda;
    int m, n, pivot;
    double* tau;
    QrWork w;
};

// block-wide argmax of (value desc, pos asc); returns the winning col to all threads
__device__ __forceinline__ int block_argmax(double v, int p, int c, double* red) {
    int* redi = reinterpret_cast<int*>(red + 16);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        int p2 = __shfl_xor_sync(0xffffffffu, p, o);
        int c2 = __shfl_xor_sync(0xffffffffu, c, o);
        if (c2 >= 0 && (c < 0 || v2 > v || (v2 == v && p2 < p))) { v = v2; p = p2; c = c2; }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) { red[wid] = v; redi[2 * wid] = p; redi[2 * wid + 1] = c; }
    __syncthreads();
    if (wid == 0) {
        v = lane < nw ? red[lane] : -1.0;
        p = lane < nw ? redi[2 * lane] : 0x7fffffff;
        c = lane < nw ? redi[2 * lane + 1] : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double v2 = __shfl_xor_sync(0xffffffffu, v, o);
            int p2 = __shfl_xor_sync(0xffffffffu, p, o);
            int c2 = __shfl_xor_sync(0xffffffffu, c, o);
            if (c2 >= 0 && (c < 0 || v2 > v || (v2 == v && p2 < p))) { v = v2; p = p2; c = c2; }
        }
        if (lane == 0) redi[0] = c;
    }
    __syncthreads();
    int res = redi[0];
    __syncthreads();
    return res;
}

constexpr int QR_NT = 512;

template <int RPT>
__global__ void __launch_bounds__(QR_NT, 1) k_qr_coop(QrArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double vs[];            // v of the current step (rows k..m-1), then red[32]
    double* red = vs + a.m;
    __shared__ double s_alpha;
    __shared__ int s_piv;
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const int m = a.m, n = a.n;
    const long long lda = a.lda;
    volatile int* phys = a.w.phys_all + (long long)cta * n;   // volatile: written by tid 0, read by all
    volatile int* pos = a.w.pos_all + (long long)cta * n;
    const double tol3z = sqrt(1.1102230246251565e-16);

    for (int j = tid; j < n; j += QR_NT) { phys[j] = j; pos[j] = j; }
    // initial column norms of owned columns + first candidate
    double best = -1.0;
    int best_pos = 0x7fffffff, best_col = -1;
    for (int p = cta; p < n; p += G) {
        const double* col = a.A + (long long)p * lda;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            int i = tid + QR_NT * j;
            if (i < m) { double x = __ldcg(col + i); s += x * x; }
        }
        s = block_sum(s, red);
        double nrm = sqrt(s);
        if (tid == 0) { a.w.vn1[p] = nrm; a.w.vn2[p] = nrm; }
        if (nrm > best || (nrm == best && p < best_pos)) { best = nrm; best_pos = p; best_col = p; }
    }
    if (tid == 0) {
        a.w.cand_val[cta] = best;
        a.w.cand_pos[cta] = best_pos;
        a.w.cand_col[cta] = best_col;
    }
    __syncthreads();
    grid.sync();

    int prev_piv = -1, prev_k = -1;
    double prev_mu = 0.0;
    for (int k = 0; k < n; ++k) {
        const int buf = k & 1;
        // ---- owner writes back the previous reflector (v, R_kk)
        if (prev_piv >= 0 && prev_piv % G == cta) {
            double* col = a.A + (long long)prev_piv * lda;
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                int i = prev_k + 1 + tid + QR_NT * j;
                if (i < m) col[i] = vs[i];
            }
            if (tid == 0) col[prev_k] = prev_mu;
        }
        __syncthreads();
        // ---- 1. pivot
        int piv = k;
        if (a.pivot) {
            double bv = -1.0;
            int bp = 0x7fffffff, bc = -1;
            for (int g = tid; g < G; g += QR_NT) {
                int pc = __ldcg(a.w.cand_col + buf * G + g);
                if (pc < 0) continue;
                double v = __ldcg(a.w.cand_val + buf * G + g);
                int ps = __ldcg(a.w.cand_pos + buf * G + g);
                if (v > bv || (v == bv && ps < bp)) { bv = v; bp = ps; bc = pc; }
            }
            bc = block_argmax(bv, bp, bc, red);
            if (tid == 0) s_piv = bc;
            __syncthreads();
            piv = s_piv;
            __syncthreads();
            // swap logical positions k <-> pos[piv] (identical in every CTA)
            if (tid == 0) {
                int pk = phys[k], pj = pos[piv];
                phys[k] = piv; phys[pj] = pk;
                pos[piv] = k; pos[pk] = pj;
            }
            __syncthreads();
        }
        // ---- 2. reflector of the pivot column (computed redundantly)
        const double* pcol = a.A + (long long)piv * lda;
        double x[RPT];
        double sig = 0.0;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            int i = k + 1 + tid + QR_NT * j;
            x[j] = i < m ? __ldcg(pcol + i) : 0.0;
            sig += x[j] * x[j];
        }
        if (tid == 0) s_alpha = __ldcg(pcol + k);
        sig = block_sum(sig, red);       // also orders s_alpha
        const double alpha = s_alpha;
        double tau, v0, mu;
        bool scale_v = true;
        if (sig == 0.0) {
            scale_v = false;
            if (alpha >= 0.0) { tau = 0.0; mu = alpha; v0 = 1.0; }
            else { tau = 2.0; mu = -alpha; v0 = 1.0; }
        } else {
            mu = sqrt(alpha * alpha + sig);
            v0 = alpha <= 0.0 ? alpha - mu : -sig / (alpha + mu);
            tau = 2.0 * v0 * v0 / (sig + v0 * v0);
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            int i = k + 1 + tid + QR_NT * j;
            if (i < m) vs[i] = scale_v ? x[j] / v0 : x[j];
        }
        if (tid == 0) vs[k] = 1.0;
        if (cta == 0 && tid == 0) a.tau[k] = tau;
        __syncthreads();
        // ---- 3. apply H_k to the owned, unprocessed columns
        best = -1.0; best_pos = 0x7fffffff; best_col = -1;
        for (int p = cta; p < n; p += G) {
            if (p == piv) continue;
            if (a.pivot) { if (pos[p] <= k) continue; }
            else if (p <= k) continue;
            double* col = a.A + (long long)p * lda;
            double y[RPT];
            double d = 0.0;
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                int i = k + tid + QR_NT * j;
                y[j] = i < m ? __ldcg(col + i) : 0.0;
                d += (i < m ? vs[i] : 0.0) * y[j];
            }
            d = block_sum(d, red);
            const double wv = tau * d;
            double s2 = 0.0;
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                int i = k + tid + QR_NT * j;
                if (i < m) {
                    y[j] -= wv * vs[i];
                    col[i] = y[j];
                    if (i > k) s2 += y[j] * y[j];
                }
            }
            if (a.pivot) {
                // partial-norm downdate (LAPACK xLAQP2, reading R3)
                __shared__ double s_rkp;
                if (tid == 0) s_rkp = y[0];       // row k lives in thread 0, j = 0
                __syncthreads();
                double v1 = __ldcg(a.w.vn1 + p), v2 = __ldcg(a.w.vn2 + p);
                bool recompute = false;
                if (v1 != 0.0) {
                    double r = fabs(s_rkp) / v1;
                    double temp = 1.0 - r * r;
                    temp = temp < 0.0 ? 0.0 : temp;
                    double q = v1 / v2;
                    double temp2 = temp * q * q;
                    if (temp2 <= tol3z) recompute = true;
                    else v1 = v1 * sqrt(temp);
                }
                if (recompute) {              // block-uniform branch
                    s2 = block_sum(s2, red);
                    if (k + 1 < m) { v1 = sqrt(s2); v2 = v1; }
                    else { v1 = 0.0; v2 = 0.0; }
                }
                __syncthreads();
                if (tid == 0) { a.w.vn1[p] = v1; a.w.vn2[p] = v2; }
                const int ps = pos[p];
                if (v1 > best || (v1 == best && ps < best_pos)) { best = v1; best_pos = ps; best_col = p; }
            }
        }
        if (tid == 0) {
            const int nb = buf ^ 1;
            a.w.cand_val[nb * G + cta] = best;
            a.w.cand_pos[nb * G + cta] = best_pos;
            a.w.cand_col[nb * G + cta] = best_col;
        }
        prev_piv = piv; prev_k = k; prev_mu = mu;
        grid.sync();
    }
    // final write-back of the last reflector
    if (prev_piv >= 0 && prev_piv % G == cta) {
        double* col = a.A + (long long)prev_piv * lda;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            int i = prev_k + 1 + tid + QR_NT * j;
            if (i < m) col[i] = vs[i];
        }
        if (tid == 0) col[prev_k] = prev_mu;
    }
}

template <int RPT>
static void* qr_kernel_ptr() { return (void*)k_qr_coop<RPT>; }

static int rpt_for(int m) {
    int r = 1;
    while (r * QR_NT < m) r <<= 1;
    return r;
}

static void* qr_kernel_for(int rpt) {
    switch (rpt) {
        case 1: return qr_kernel_ptr<1>();
        case 2: return qr_kernel_ptr<2>();
        case 4: return qr_kernel_ptr<4>();
        case 8: return qr_kernel_ptr<8>();
        case 16: return qr_kernel_ptr<16>();
        case 32: return qr_kernel_ptr<32>();
        default: return nullptr;
    }
}

int qr_coop_grid(int m, int* grid) {
    int rpt = rpt_for(m);
    void* fn = qr_kernel_for(rpt);
    if (!fn) return -7;
    size_t smem = sizeof(double) * ((size_t)m + 32);
    MPJ_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, nsm = 0, per = 0;
    MPJ_CUDA_TRY(cudaGetDevice(&dev));
    MPJ_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    MPJ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, QR_NT, smem));
    if (per < 1) return -7;
    *grid = nsm * per;
    return 0;
}

int qr_coop(double* A, long long lda, int m, int n, double* tau, int pivot, QrWork& w, int* phys_out,
            cudaStream_t st) {
    int rpt = rpt_for(m);
    void* fn = qr_kernel_for(rpt);
    if (!fn) return -7;
    size_t smem = sizeof(double) * ((size_t)m + 32);
    QrArgs args;
    args.A = A;
    args.lda = lda;
    args.m = m;
    args.n = n;
    args.pivot = pivot;
    args.tau = tau;
    args.w = w;
    void* params[] = {&args};
    MPJ_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(w.grid), dim3(QR_NT), params, smem, st));
    MPJ_LAUNCHED();
    if (phys_out)
        MPJ_CUDA_TRY(cudaMemcpyAsync(phys_out, w.phys_all, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
    return 0;
}

// ------------------------------------------------------------------------
// Unpivoted panel QR (the panels of qr_blocked) without grid barriers.
// CTA z owns the CPC panel columns c0 = z CPC .. c0 + CPC - 1 for the whole
// kernel, register resident (rows tid + QR_NT j).  It applies H_0 .. H_{c0-1}
// in order, each as soon as its reflector is published, then forms its own
// reflectors one after the other (same formulas as k_qr_coop), applying each
// to its later columns locally, writes v and tau, and releases the flags
// ready[c0 ..] = epoch.  The chain therefore crosses CTAs (flag + L2 round
// trip) once per CPC columns instead of a grid-wide barrier per column, and
// the kernel is safe to run beside other kernels (no co-residency
// requirement: a CTA only waits for lower-numbered CTAs).
// ------------------------------------------------------------------------
template <int CPC>
__device__ __forceinline__ void block_sum_vec(double (&v)[CPC], double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < CPC; ++q) {
        v[q] = warp_sum(v[q]);
        if (lane == 0) red[q * 32 + wid] = v[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < CPC; ++q) v[q] = warp_sum(lane < nw ? red[q * 32 + lane] : 0.0);
    __syncthreads();
}

template <int RPT, int CPC>
__global__ void __launch_bounds__(QR_NT, 1) k_qr_panel(double* __restrict__ A, long long lda, int m, int n,
                                                       double* __restrict__ tau, int* ready, int epoch) {
    extern __shared__ double vsh[];           // v of the current step at this thread's rows
    __shared__ double red[32 * CPC];
    __shared__ double s_alpha;
    const int c0 = blockIdx.x * CPC, tid = threadIdx.x;
    const int nc = n - c0 < CPC ? n - c0 : CPC;
    double y[CPC][RPT];
#pragma unroll
    for (int q = 0; q < CPC; ++q)
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int i = tid + QR_NT * j;
            y[q][j] = (q < nc && i < m) ? A[(long long)(c0 + q) * lda + i] : 0.0;
        }
    for (int k = 0; k < c0; ++k) {
        if (tid == 0)
            while (ld_acquire_gpu(ready + k) != epoch) { }
        __syncthreads();
        const double* vk = A + (long long)k * lda;
        const double tk = __ldcg(tau + k);
        double d[CPC];
#pragma unroll
        for (int q = 0; q < CPC; ++q) d[q] = 0.0;
        if constexpr (RPT * (CPC + 1) <= 48) {
            // v at this thread's rows stays in registers (no shared-memory round trip on the chain)
            double vr[RPT];
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const int i = tid + QR_NT * j;
                vr[j] = (i > k && i < m) ? __ldcg(vk + i) : (i == k ? 1.0 : 0.0);
            }
#pragma unroll
            for (int j = 0; j < RPT; ++j)
#pragma unroll
                for (int q = 0; q < CPC; ++q) d[q] += vr[j] * y[q][j];
            block_sum_vec<CPC>(d, red);
#pragma unroll
            for (int q = 0; q < CPC; ++q) {
                const double wv = tk * d[q];
#pragma unroll
                for (int j = 0; j < RPT; ++j) y[q][j] -= wv * vr[j];
            }
        } else {
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const int i = tid + QR_NT * j;
                double v = 0.0;
                if (i > k && i < m) v = __ldcg(vk + i);
                else if (i == k) v = 1.0;
                vsh[tid + QR_NT * j] = v;
#pragma unroll
                for (int q = 0; q < CPC; ++q) d[q] += v * y[q][j];
            }
            block_sum_vec<CPC>(d, red);
#pragma unroll
            for (int q = 0; q < CPC; ++q) {
                const double wv = tk * d[q];
#pragma unroll
                for (int j = 0; j < RPT; ++j) y[q][j] -= wv * vsh[tid + QR_NT * j];
            }
        }
    }
    double mus[CPC];
#pragma unroll
    for (int q = 0; q < CPC; ++q) {
        mus[q] = 0.0;
        if (q >= nc) break;
        const int c = c0 + q;
        // own reflector H_c of y_q(c:m)
        double sig = 0.0;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int i = tid + QR_NT * j;
            if (i == c) s_alpha = y[q][j];
            if (i > c && i < m) sig += y[q][j] * y[q][j];
        }
        sig = block_sum(sig, red);            // also orders s_alpha
        const double alpha = s_alpha;
        double tk, v0, mu;
        bool scale_v = true;
        if (sig == 0.0) {
            scale_v = false;
            if (alpha >= 0.0) { tk = 0.0; mu = alpha; v0 = 1.0; }
            else { tk = 2.0; mu = -alpha; v0 = 1.0; }
        } else {
            mu = sqrt(alpha * alpha + sig);
            v0 = alpha <= 0.0 ? alpha - mu : -sig / (alpha + mu);
            tk = 2.0 * v0 * v0 / (sig + v0 * v0);
        }
        mus[q] = mu;
        double* col = A + (long long)c * lda;
        // v = x / v0 as x * (1 / v0) (RPT divisions per thread were a visible share of the column step);
        // the exact quotient where 1 / v0 would leave the normal range
        const bool recip = fabs(v0) > 1e-290 && fabs(v0) < 1e290;
        const double rv0 = 1.0 / v0;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int i = tid + QR_NT * j;
            if (i > c && i < m) {
                if (scale_v) y[q][j] = recip ? y[q][j] * rv0 : y[q][j] / v0;
                col[i] = y[q][j];
            }
        }
        if (tid == 0) tau[c] = tk;
        // release column c at once (the next CTA applies H_c while this one forms its next reflector);
        // one fence by the releasing thread after the barrier (cumulative)
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release_gpu(ready + c, epoch);
        }
        // H_c applied to this CTA's later columns (v_c = 1, v = y_q below row c)
#pragma unroll
        for (int q2 = q + 1; q2 < CPC; ++q2) {
            if (q2 >= nc) break;
            double d = 0.0;
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const int i = tid + QR_NT * j;
                const double v = (i > c && i < m) ? y[q][j] : (i == c ? 1.0 : 0.0);
                d += v * y[q2][j];
            }
            d = block_sum(d, red);
            const double wv = tk * d;
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const int i = tid + QR_NT * j;
                const double v = (i > c && i < m) ? y[q][j] : (i == c ? 1.0 : 0.0);
                y[q2][j] -= wv * v;
            }
        }
    }
    // R(0:c, c) is read only by later kernels
#pragma unroll
    for (int q = 0; q < CPC; ++q) {
        if (q >= nc) break;
        const int c = c0 + q;
        double* col = A + (long long)c * lda;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int i = tid + QR_NT * j;
            if (i <= c) col[i] = i < c ? y[q][j] : mus[q];
        }
    }
}

template <int RPT, int CPC>
static void* panel_kernel_ptr() { return (void*)k_qr_panel<RPT, CPC>; }

// columns per CTA: 2 while two register-resident columns fit (RPT <= 16), else 1
static void* panel_kernel_for(int rpt, int* cpc) {
    *cpc = rpt <= 16 ? 2 : 1;
    switch (rpt) {
        case 1: return panel_kernel_ptr<1, 2>();
        case 2: return panel_kernel_ptr<2, 2>();
        case 4: return panel_kernel_ptr<4, 2>();
        case 8: return panel_kernel_ptr<8, 2>();
        case 16: return panel_kernel_ptr<16, 2>();
        case 32: return panel_kernel_ptr<32, 1>();
        default: return nullptr;
    }
}

int qr_panel_chain(double* A, long long lda, int m, int n, double* tau, int* ready, cudaStream_t st) {
    static std::atomic<int> epoch{0};
    if (n <= 0) return 0;
    const int rpt = rpt_for(m);
    int cpc = 1;
    void* fn = panel_kernel_for(rpt, &cpc);
    if (!fn || n > 1024) return -7;
    const size_t smem = sizeof(double) * (size_t)QR_NT * rpt;
    MPJ_CUDA_TRY(mpj_set_smem(reinterpret_cast<const void*>(fn), smem));
    int ep = ++epoch;
    if (ep <= 0) { epoch = 1; ep = 1; }
    void* params[] = {&A, &lda, &m, &n, &tau, &ready, &ep};
    MPJ_CUDA_TRY(cudaLaunchKernel(fn, dim3((n + cpc - 1) / cpc), dim3(QR_NT), params, smem, st));
    MPJ_LAUNCHED();
    return 0;
}

__global__ void k_gather_cols(const double* A, long long lda, const int* perm, double* out, long long ldo,
                              long long rows) {
    const int k = blockIdx.y;
    const double* src = A + (long long)perm[k] * lda;
    double* dst = out + (long long)k * ldo;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int gather_cols(const double* A, long long lda, const int* perm, double* out, long long ldo, long long rows,
                int n, cudaStream_t st) {
    int gx = (int)((rows + 255) / 256);
    if (gx > 64) gx = 64;
    k_gather_cols<<<dim3(gx, n), 256, 0, st>>>(A, lda, perm, out, ldo, rows);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mpj
