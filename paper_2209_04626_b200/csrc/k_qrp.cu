// k_qrp.cu -- column-pivoted Householder QR, A P = Q R (PAPER.md:332-335,
// Alg. 2 line 1; 350), Businger-Golub pivoting with the LAPACK xLAQP2 partial
// norm downdate (reading R3), as ONE persistent cooperative kernel
// with xLAQPS-style lazy updates.
//
// Physical column p is owned by CTA p % G and never moves (logical order in
// per-CTA copies of phys/pos).  Step k (jj = k mod NB inside a panel of NB
// steps):
//   pass 1 (all CTAs, row slices): bring the pivot column up to date with the
//     panel's pending reflectors, x = a_piv - V_panel F(piv,:)^T, and
//     accumulate slice partials of sum x_i^2 (i > k) and z_t = v_t^T x;
//   grid barrier;
//   every CTA: reflector (mu, v0, tau) from the fixed-order reduction of the
//     partials, auxv_t = -tau (v_t(k) + z_t / v0);
//   pass 2 (owners, columns): F(p, jj) = tau v^T a_p + F(p, :) auxv  (a READ
//     of the stale trailing column: the GEMV half of QRP), row k of p updated
//     with all panel reflectors, partial norm downdated; a column whose norm
//     must be recomputed is updated eagerly (its F row zeroed);
//   end of panel: owners apply the panel to their trailing columns
//     (a_p -= V_panel F(p,:)^T, rows below the panel);
//   grid barrier.
// The trailing matrix is read once per step and written once per panel
// (the unblocked algorithm reads AND writes it every step).  Reflectors are
// stored unnormalised (x) during the factorisation and scaled by 1/v0 at the
// end (R_kk = mu >= 0, reading c-13).
#include <algorithm>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include "common.cuh"
#include "jacobi.h"

namespace cg = cooperative_groups;

namespace mpj {

constexpr int QP_NT = 512;
constexpr int QP_NB = 32;
constexpr int QP_PE_G = 4;      // columns per group of the end-of-panel ring
constexpr int QP_PART_PT = 12;
constexpr int QP_CAND_PL = 6;    // candidates per lane of the pivot warp: G <= 32 QP_CAND_PL   // partials per thread in the reflector reduction: G (QP_NB + 1) <= QP_NT QP_PART_PT

template <typename T>
struct QrpArgs {
    T* A;
    long long lda;
    int m, n;
    T* tau;
    QrWork w;
    T* F;       // n x QP_NB (row p: pending panel coefficients of column p)
    T* part;    // G x (QP_NB + 1)
    T* v0g;     // n
    T* mug;     // n
    int nown;        // max owned columns per CTA
    int pe_st;       // stages of the end-of-panel cp.async ring (0: register path)
    long long* dbg;  // optional phase timers (CTA 0), MPJSVD_QRP_TIMING=1
};

template <typename T>
__device__ __forceinline__ int qp_argmax(T v, int p, int c, T* red) {
    int* redi = reinterpret_cast<int*>(red + 16);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T v2 = __shfl_xor_sync(0xffffffffu, v, o);
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
            T v2 = __shfl_xor_sync(0xffffffffu, v, o);
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

// warp-wide argmax under the total order (value desc, logical position asc); c < 0: no candidate
template <typename T>
__device__ __forceinline__ void warp_argmax(T& v, int& p, int& c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T v2 = __shfl_xor_sync(0xffffffffu, v, o);
        int p2 = __shfl_xor_sync(0xffffffffu, p, o);
        int c2 = __shfl_xor_sync(0xffffffffu, c, o);
        if (c2 >= 0 && (c < 0 || v2 > v || (v2 == v && p2 < p))) { v = v2; p = p2; c = c2; }
    }
}

// block-wide sums of NV values (fixed tree); red needs 32 * NV doubles
template <int NV, typename T>
__device__ __forceinline__ void block_sum_n(T (&v)[NV], T* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) red[q * 32 + wid] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        T r = lane < nw ? red[q * 32 + lane] : 0.0;
        v[q] = warp_sum(r);
    }
    __syncthreads();
}

template <typename T, int RPT>
__global__ void __launch_bounds__(QP_NT, 1) k_qrp_lazy(QrpArgs<T> a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char qsm_raw[];
    T* qsm = reinterpret_cast<T*>(qsm_raw);
    const int m = a.m, n = a.n, nown = a.nown;
    T* vs = qsm;                               // m: current reflector v (rows k..m-1); also the
                                               // staging of the G x (QP_NB + 1) partials (vsz >= both)
    const int vsz = max(m, (int)gridDim.x * (QP_NB + 1));
    T* Fown = vs + vsz;                        // nown x QP_NB
    T* vn1s = Fown + (size_t)nown * QP_NB;     // nown
    T* vn2s = vn1s + nown;                     // nown
    T* red = vn2s + nown;                      // 33 * 32 (>= 32 * (QP_NB + 1))
    T* auxv = red + 32 * (QP_NB + 1);          // QP_NB
    T* vk = auxv + QP_NB;                      // QP_NB: v_t(k)
    T* v0p = vk + QP_NB;                       // QP_NB: 1 / v0 of the panel reflectors
    T* fpiv = v0p + QP_NB;                     // QP_NB: F(piv, :)
    T* scal = fpiv + QP_NB;                    // 8 scalars
    T* dsm = scal + 8;                         // nown: v^T a_p of the owned columns
    T* ykp = dsm + nown;                       // nown: a(k, p) before the row update
    T* dsm2 = ykp + nown;                      // 2 nown: per-half partial dots
    int* pcol = reinterpret_cast<int*>(dsm2 + 2 * nown); // QP_NB
    int* rflag = pcol + QP_NB;                      // nown: recompute flags
    int* own = rflag + nown;                        // nown: physical column of owned slot s (-1: none); the
                                                    // live columns are re-dealt round-robin at every panel end
    // 16-bit (n <= 16384): the shared-memory footprint sets the L1 left for the GEMV's loads in flight
    unsigned short* phys = reinterpret_cast<unsigned short*>(own + nown);   // n: column at logical position (this CTA's copy)
    unsigned short* pos = phys + n;                 // n: logical position of physical column
    int* lsl = reinterpret_cast<int*>(pos + n);     // nown: live owned slots at a panel end (2n shorts: 4-byte aligned)
    // end-of-panel ring: stage s, column u of a group, thread t at ring[(s QP_PE_G + u) QP_NT + t]
    T* ring = reinterpret_cast<T*>(qsm_raw + ((reinterpret_cast<size_t>(lsl + nown) - reinterpret_cast<size_t>(qsm_raw) + 15) & ~size_t(15)));
    __shared__ int s_anyrec, s_piv, s_nl;
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const long long lda = a.lda;
    const T tol3z = sqrt(sizeof(T) == 8 ? T(1.1102230246251565e-16) : T(5.9604644775390625e-08));

    for (int j = tid; j < n; j += QP_NT) { phys[j] = j; pos[j] = j; }
    if (tid == 0) s_anyrec = 0;
    for (int e = tid; e < nown * QP_NB; e += QP_NT) Fown[e] = 0.0;
    for (int sl = tid; sl < nown; sl += QP_NT) {
        const int p = cta + G * sl;
        own[sl] = p < n ? p : -1;                    // -1: no column in this slot
        rflag[sl] = 0;
    }
    // logical position of the column in owned slot sl (-1: empty slot)
    auto lp = [&](int sl) -> int { return own[sl] >= 0 ? pos[own[sl]] : -1; };
    T best = -1.0;
    int best_pos = 0x7fffffff, best_col = -1;
    for (int p = cta, s = 0; p < n; p += G, ++s) {
        const T* col = a.A + (long long)p * lda;
        T sq[1] = {0.0};
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            int i = tid + QP_NT * j;
            if (i < m) { T x = __ldcg(col + i); sq[0] += x * x; }
        }
        block_sum_n<1, T>(sq, red);
        const T nrm = sqrt(sq[0]);
        if (tid == 0) { vn1s[s] = nrm; vn2s[s] = nrm; }
        if (nrm > best || (nrm == best && p < best_pos)) { best = nrm; best_pos = p; best_col = p; }
        for (int t = tid; t < QP_NB; t += QP_NT) a.F[(long long)p * QP_NB + t] = 0.0;
    }
    if (tid == 0) {
        a.w.cand_val[cta] = (double)best;
        a.w.cand_pos[cta] = best_pos;
        a.w.cand_col[cta] = best_col;
    }
    __syncthreads();
    grid.sync();

    long long tph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tlast = clock64();
    auto tmark = [&](int ph) {
        if (a.dbg && tid == 0) {
            long long t = clock64();
            tph[ph] += t - tlast;
            tlast = t;
        }
    };
    for (int k = 0; k < n; ++k) {
        const int buf = k & 1;
        const int jj = k % QP_NB;
        tmark(7);
        // pass 1's row slice and its first rows of the panel's reflectors do not depend on the pivot: their loads
        // are issued before the pivot is chosen (they overlap warp 0's candidate reduction)
        constexpr int RS = QP_NT / 32;
        const long long p1_S = (m - k + G - 1) / G;
        const long long p1_r0 = k + (long long)cta * p1_S, p1_r1 = min((long long)m, p1_r0 + p1_S);
        const int p1_lane = tid & 31, p1_wid = tid >> 5;
        const T* pcl = p1_lane < jj ? a.A + (long long)pcol[p1_lane] * lda : nullptr;
        const T rvl = p1_lane < jj ? v0p[p1_lane] : T(0);
        T vpre[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long i = p1_r0 + p1_wid + u * RS;
            vpre[u] = (p1_lane < jj && i < p1_r1) ? __ldcg(pcl + i) * rvl : T(0);
        }
        // ---------------- pivot (largest partial norm, ties -> lowest logical index): warp 0
        if (tid < 32) {
            T bv = -1.0;
            int bp = 0x7fffffff, bc = -1;
            int pcv[QP_CAND_PL], psv[QP_CAND_PL];
            double vv[QP_CAND_PL];
#pragma unroll
            for (int j = 0; j < QP_CAND_PL; ++j) {       // every candidate load in flight at once
                const int g = tid + 32 * j;
                pcv[j] = g < G ? __ldcg(a.w.cand_col + buf * G + g) : -1;
                vv[j] = g < G ? __ldcg(a.w.cand_val + buf * G + g) : -1.0;
                psv[j] = g < G ? __ldcg(a.w.cand_pos + buf * G + g) : 0x7fffffff;
            }
#pragma unroll
            for (int j = 0; j < QP_CAND_PL; ++j) {
                if (pcv[j] < 0) continue;
                const T v = (T)vv[j];
                if (v > bv || (v == bv && psv[j] < bp)) { bv = v; bp = psv[j]; bc = pcv[j]; }
            }
            warp_argmax(bv, bp, bc);
            int pv = __shfl_sync(0xffffffffu, bc, 0);
            // no finite candidate (NaN partial norms): keep the column in place instead of indexing
            // with -1 (the host returns MPJSVD_ERR_NONFINITE before the QRP; this guards direct calls)
            if (pv < 0) pv = phys[k];
            if (tid < jj) fpiv[tid] = __ldcg(a.F + (long long)pv * QP_NB + tid);
            if (tid == 0) {
                s_piv = pv;
                int pk = phys[k], pj = pos[pv];
                phys[k] = pv; phys[pj] = pk;
                pos[pv] = k; pos[pk] = pj;
                pcol[jj] = pv;
            }
        }
        __syncthreads();
        const int piv = s_piv;
        tmark(0);
        // ---------------- pass 1: pivot column rows k..m-1 in row slices.
        // A warp takes one row at a time; lane t < jj holds v_t(i) (panel reflector t,
        // unnormalised x_t times 1/v0_t) so the pending update is a warp reduction and
        // lane t accumulates z_t = sum_i v_t(i) x_i directly.
        {
            const long long r0 = p1_r0, r1 = p1_r1;
            const int lane = p1_lane, wid = p1_wid;
            T* pc = a.A + (long long)piv * lda;
            const T fl = lane < jj ? fpiv[lane] : 0.0;
            T zl = 0.0, sx2 = 0.0;
            for (long long ib = r0 + wid; ib < r1; ib += 4 * RS) {
                T vtv[4], xv[4];
                const bool first = ib == r0 + wid;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const long long i = ib + u * RS;
                    vtv[u] = first ? vpre[u] : ((lane < jj && i < r1) ? __ldcg(pcl + i) * rvl : T(0));
                    xv[u] = i < r1 ? __ldcg(pc + i) : T(0);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const long long i = ib + u * RS;
                    if (i >= r1) break;
                    const T upd = warp_sum(vtv[u] * fl);
                    const T x = xv[u] - upd;
                    if (lane == 0) pc[i] = x;
                    if (i > k) {
                        zl += vtv[u] * x;
                        sx2 += x * x;
                    }
                }
            }
            // lane t of every warp holds a partial z_t; sx2 identical in all lanes of a warp
            red[wid * 33 + lane] = zl;
            if (lane == 0) red[wid * 33 + 32] = sx2;
            __syncthreads();
            if (tid <= QP_NB) {
                T sacc = 0.0;
                for (int w = 0; w < QP_NT / 32; ++w) sacc += red[w * 33 + tid];
                const int q = tid == 32 ? QP_NB : tid;
                // slot-major layout part[slot][G], slot 0 = sigma, slot t + 1 = z_t: the jj + 1 live slots of
                // this step are one contiguous prefix (the reduction below loads only those)
                if (q < jj || q == QP_NB) a.part[(long long)(q == QP_NB ? 0 : q + 1) * G + cta] = sacc;
            }
            __syncthreads();
        }
        tmark(1);
        grid.sync();
        tmark(2);
        // ---------------- reflector (identical in every CTA)
        T colv[RPT];                  // pivot column rows k+1.. (pass 1 output), loaded with the partials
        T alpha_r = 0.0, vk_r = 0.0;
        {
            // value q (z_t for t < jj, sigma at q = QP_NB) summed over the G CTAs: the (jj + 1) x G live
            // partials (slot-major) are staged in shared memory (every load in flight at once), then warp w
            // sums q = w, w + 16, ... with lanes striding over g (fixed tree)
            const int lane = tid & 31, wid = tid >> 5;
            const int tot = G * (jj + 1);
            T pv[QP_PART_PT];
#pragma unroll
            for (int j = 0; j < QP_PART_PT; ++j) {
                const int e = tid + QP_NT * j;
                pv[j] = e < tot ? __ldcg(a.part + e) : T(0);
            }
            {
                const T* pcp = a.A + (long long)piv * lda;
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    const int i = k + 1 + tid + QP_NT * j;
                    colv[j] = i < m ? __ldcg(pcp + i) : T(0);
                }
                if (tid == 0) alpha_r = __ldcg(pcp + k);
                if (tid < jj) vk_r = __ldcg(a.A + (long long)pcol[tid] * lda + k);
            }
#pragma unroll
            for (int j = 0; j < QP_PART_PT; ++j) {
                const int e = tid + QP_NT * j;
                if (e < tot) vs[e] = pv[j];
            }
            __syncthreads();
            for (int q = wid; q <= QP_NB; q += QP_NT / 32) {
                if (q < jj || q == QP_NB) {
                    const int slot = q == QP_NB ? 0 : q + 1;
                    T sacc = 0.0;
                    for (int g = lane; g < G; g += 32) sacc += vs[slot * G + g];
                    sacc = warp_sum(sacc);
                    if (lane == 0) red[q] = sacc;
                }
            }
        }
        if (tid == 0) scal[0] = alpha_r;   // alpha
        if (tid < jj) vk[tid] = vk_r * v0p[tid];
        __syncthreads();
        const T sig = red[QP_NB], alpha = scal[0];
        T tau, v0, mu;
        if (sig == 0.0) {
            v0 = 1.0;
            if (alpha >= 0.0) { tau = 0.0; mu = alpha; } else { tau = 2.0; mu = -alpha; }
        } else {
            mu = sqrt(alpha * alpha + sig);
            v0 = alpha <= 0.0 ? alpha - mu : -sig / (alpha + mu);
            tau = 2.0 * v0 * v0 / (sig + v0 * v0);
        }
        const T rv0 = 1.0 / v0;
        if (tid < jj) auxv[tid] = -tau * (vk[tid] + red[tid] * rv0);
        if (cta == 0 && tid == 0) { a.tau[k] = tau; a.v0g[k] = v0; a.mug[k] = mu; }
        {
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                int i = k + 1 + tid + QP_NT * j;
                if (i < m) vs[i] = colv[j] * rv0;
            }
            if (tid == 0) vs[k] = 1.0;
        }
        __syncthreads();
        tmark(3);
        if (tid == 0) { v0p[jj] = rv0; vk[jj] = 1.0; }
        // ---------------- pass 2a: v^T a_p for the owned unprocessed columns (read-only GEMV).
        // Work items (owned column, row half) are streamed by independent warps (no CTA
        // barrier inside the loop); each item's partial dot goes to dsm2[2 s + h].
        const bool panel_end = (jj == QP_NB - 1) || (k == n - 1);
        {
            const int lane = tid & 31, wid = tid >> 5;
            const long long rows = m - k;
            const long long L = (rows + 1) / 2;
            // the sweep over the owned columns alternates direction from step to step, so the
            // columns read last (still in L2) are read first by the next step
            const bool rev = (k & 1) != 0;
            for (int it = wid; it < 2 * nown; it += QP_NT / 32) {
                const int sl = rev ? nown - 1 - (it >> 1) : (it >> 1), h = it & 1;
                if (lp(sl) <= k) continue;
                const T* col = a.A + (long long)own[sl] * lda;
                const long long rb = k + h * L, re = min((long long)m, rb + L);
                T acc0 = 0.0, acc1 = 0.0;
                long long i = rb + lane;
                for (; i + 96 < re; i += 128) {
                    const T y0v = __ldcg(col + i), y1v = __ldcg(col + i + 32);
                    const T y2v = __ldcg(col + i + 64), y3v = __ldcg(col + i + 96);
                    acc0 += vs[i] * y0v;
                    acc1 += vs[i + 32] * y1v;
                    acc0 += vs[i + 64] * y2v;
                    acc1 += vs[i + 96] * y3v;
                }
                for (; i < re; i += 32) acc0 += vs[i] * __ldcg(col + i);
                const T dp = warp_sum(acc0 + acc1);
                if (lane == 0) {
                    dsm2[2 * sl + h] = dp;
                    if (h == 0) ykp[sl] = __ldcg(col + k);
                }
            }
        }
        __syncthreads();
        for (int sl = tid; sl < nown; sl += QP_NT) dsm[sl] = dsm2[2 * sl] + dsm2[2 * sl + 1];
        __syncthreads();
        // ---------------- pass 2b: one thread per owned column: F(p, jj), row k, norm downdate
        T cbest = -1.0;
        int cpos = 0x7fffffff, ccol = -1;
        for (int sl = tid; sl < nown; sl += QP_NT) {
            if (lp(sl) <= k) continue;
            const int p = own[sl];
            T* Fs = Fown + (size_t)sl * QP_NB;
            T f = tau * dsm[sl];
            for (int t = 0; t < jj; ++t) f += Fs[t] * auxv[t];
            T akp = ykp[sl];
            for (int t = 0; t < jj; ++t) akp -= vk[t] * Fs[t];
            akp -= f;
            a.A[(long long)p * lda + k] = akp;
            Fs[jj] = f;
            a.F[(long long)p * QP_NB + jj] = f;
            // partial-norm downdate (LAPACK xLAQP2)
            const T v1 = vn1s[sl], v2 = vn2s[sl];
            int rec = 0;
            if (v1 != 0.0) {
                const T r = fabs(akp) / v1;
                T temp = 1.0 - r * r;
                temp = temp < 0.0 ? 0.0 : temp;
                const T q = v1 / v2;
                if (temp * q * q <= tol3z) rec = 1;
                else vn1s[sl] = v1 * sqrt(temp);
            }
            rflag[sl] = rec;
            if (rec) s_anyrec = 1;
        }
        __syncthreads();
        tmark(4);
        // ---------------- eager recompute of flagged columns (rare)
        const bool anyrec = s_anyrec != 0;
        for (int sl = 0; anyrec && sl < nown; ++sl) {
            if (!rflag[sl]) continue;                  // flags are only set for live columns
            const int p = own[sl];
            T* col = a.A + (long long)p * lda;
            const T* Fs = Fown + (size_t)sl * QP_NB;
            T sq[1] = {0.0};
            for (long long i = k + 1 + tid; i < m; i += QP_NT) {
                T yv = __ldcg(col + i);
                for (int t = 0; t <= jj; ++t) {
                    const T vt = t == jj ? vs[i] : __ldcg(a.A + (long long)pcol[t] * lda + i) * v0p[t];
                    yv -= vt * Fs[t];
                }
                col[i] = yv;
                sq[0] += yv * yv;
            }
            block_sum_n<1, T>(sq, red);
            if (tid == 0) {
                const T nv = k + 1 < m ? sqrt(sq[0]) : 0.0;
                vn1s[sl] = nv;
                vn2s[sl] = nv;
                rflag[sl] = 0;
            }
            for (int t = tid; t <= jj; t += QP_NT) {
                Fown[(size_t)sl * QP_NB + t] = 0.0;
                a.F[(long long)p * QP_NB + t] = 0.0;
            }
            __syncthreads();
        }
        if (anyrec) {
            __syncthreads();
            if (tid == 0) s_anyrec = 0;
        }
        tmark(8);
        // ---------------- end of panel: apply the panel to the owned trailing columns
        if (panel_end) {
          if (a.pe_st >= 2) {
            // Every thread streams its own row of the live owned columns, QP_PE_G columns per group,
            // through a private cp.async ring of pe_st stages (pe_st - 1 groups in flight while one is
            // updated): the update is bound by the bytes in flight, which registers alone cap at one group.
            if (tid == 0) {
                int nl = 0;
                for (int sl = 0; sl < nown; ++sl)
                    if (lp(sl) > k) lsl[nl++] = sl;
                s_nl = nl;
            }
            __syncthreads();
            const int nl = s_nl, ngr = (nl + QP_PE_G - 1) / QP_PE_G, S = a.pe_st;
            const unsigned rbase = (unsigned)__cvta_generic_to_shared(ring + tid);
            // row chunks in a CTA-rotated order: every CTA reads the same panel columns (vt), and CTAs walking
            // the rows in lockstep would all hit the same L2 lines at once
            const long long nch = (m - k - 1 + QP_NT - 1) / QP_NT;
            for (long long c = 0; c < nch; ++c) {
                const long long i0 = k + 1 + ((c + cta) % nch) * QP_NT;
                const long long i = i0 + tid;
                const bool rowok = i < m;
                auto issue = [&](int g) {
                    if (g < ngr && rowok) {
                        const int st = g % S;
#pragma unroll
                        for (int u = 0; u < QP_PE_G; ++u) {
                            const int q = g * QP_PE_G + u;
                            if (q < nl) {
                                const T* src = a.A + (long long)own[lsl[q]] * lda + i;
                                const unsigned dst = rbase + (unsigned)(((st * QP_PE_G + u) * QP_NT) * sizeof(T));
                                if constexpr (sizeof(T) == 8)
                                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
                                else
                                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
                            }
                        }
                    }
                    asm volatile("cp.async.commit_group;\n" ::: "memory");
                };
                for (int g = 0; g < S - 1; ++g) issue(g);
                T vt[QP_NB];
#pragma unroll
                for (int t = 0; t < QP_NB; ++t) {
                    vt[t] = 0.0;
                    if (rowok && t <= jj) vt[t] = (t == jj) ? vs[i] : __ldcg(a.A + (long long)pcol[t] * lda + i) * v0p[t];
                }
                for (int g = 0; g < ngr; ++g) {
                    issue(g + S - 1);
                    // S - 1 newer groups may stay pending; group g has landed (each thread reads only its own copies)
                    if (S == 4) asm volatile("cp.async.wait_group 3;\n" ::: "memory");
                    else if (S == 3) asm volatile("cp.async.wait_group 2;\n" ::: "memory");
                    else asm volatile("cp.async.wait_group 1;\n" ::: "memory");
                    if (!rowok) continue;
                    const T* rs = ring + (g % S) * QP_PE_G * QP_NT + tid;
                    T y[QP_PE_G];
                    const T* Fs[QP_PE_G];
#pragma unroll
                    for (int u = 0; u < QP_PE_G; ++u) {
                        const int q = g * QP_PE_G + u;
                        Fs[u] = Fown + (size_t)lsl[q < nl ? q : 0] * QP_NB;
                        y[u] = q < nl ? rs[u * QP_NT] : T(0);
                    }
#pragma unroll
                    for (int t = 0; t < QP_NB; ++t)            // vt[t] = 0 for t > jj
#pragma unroll
                        for (int u = 0; u < QP_PE_G; ++u) y[u] -= vt[t] * Fs[u][t];
#pragma unroll
                    for (int u = 0; u < QP_PE_G; ++u) {
                        const int q = g * QP_PE_G + u;
                        if (q < nl) a.A[(long long)own[lsl[q]] * lda + i] = y[u];
                    }
                }
                asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            }
          } else {
            for (long long i0 = k + 1; i0 < m; i0 += QP_NT) {
                const long long i = i0 + tid;
                if (i < m) {
                    T vt[QP_NB];
#pragma unroll
                    for (int t = 0; t < QP_NB; ++t) {
                        vt[t] = 0.0;
                        if (t <= jj) vt[t] = (t == jj) ? vs[i] : __ldcg(a.A + (long long)pcol[t] * lda + i) * v0p[t];
                    }
                    for (int s0 = 0; s0 < nown; s0 += 4) {
                        T yv[4];
                        bool lv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            lv[u] = (s0 + u < nown) && lp(s0 + u) > k;
                            yv[u] = lv[u] ? __ldcg(a.A + (long long)own[s0 + u] * lda + i) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            if (!lv[u]) continue;
                            const T* Fs = Fown + (size_t)(s0 + u) * QP_NB;
#pragma unroll
                            for (int t = 0; t < QP_NB; ++t)
                                if (t <= jj) yv[u] -= vt[t] * Fs[t];
                            a.A[(long long)own[s0 + u] * lda + i] = yv[u];
                        }
                    }
                }
            }
          }
            __syncthreads();
            for (int e = tid; e < nown * QP_NB; e += QP_NT) {
                const int sl = e / QP_NB;
                Fown[e] = 0.0;
                if (own[sl] >= 0) a.F[(long long)own[sl] * QP_NB + (e % QP_NB)] = 0.0;
            }
            if (k + 1 < n) {
                // re-deal the live columns round-robin in logical order (CTA imbalance grows as pivots
                // leave unevenly); no panel state is pending, only the partial norms move (via global memory)
                for (int sl = tid; sl < nown; sl += QP_NT)
                    if (lp(sl) > k) { a.w.vn1[own[sl]] = (double)vn1s[sl]; a.w.vn2[own[sl]] = (double)vn2s[sl]; }
                grid.sync();
                for (int sl = tid; sl < nown; sl += QP_NT) {
                    const long long j = (long long)k + 1 + cta + (long long)G * sl;
                    const int p = j < n ? phys[j] : -1;
                    own[sl] = p;
                    if (p >= 0) { vn1s[sl] = (T)__ldcg(a.w.vn1 + p); vn2s[sl] = (T)__ldcg(a.w.vn2 + p); }
                    rflag[sl] = 0;
                }
                __syncthreads();
            }
        }
        tmark(5);
        // ---------------- candidate for the next step (argmax over the owned columns): warp 0
        if (tid < 32) {
            for (int sl = tid; sl < nown; sl += 32) {
                const int ps = lp(sl);
                if (ps <= k) continue;
                const T v1 = vn1s[sl];
                if (v1 > cbest || (v1 == cbest && ps < cpos)) { cbest = v1; cpos = ps; ccol = own[sl]; }
            }
            warp_argmax(cbest, cpos, ccol);
            if (tid == 0) {
                const int nb = buf ^ 1;
                a.w.cand_val[nb * G + cta] = ccol >= 0 ? (double)cbest : -1.0;
                a.w.cand_pos[nb * G + cta] = ccol >= 0 ? cpos : 0x7fffffff;
                a.w.cand_col[nb * G + cta] = ccol;
            }
        }
        __syncthreads();
        tmark(6);
        grid.sync();
    }
    if (a.dbg && tid == 0)
        for (int q = 0; q < 10; ++q) {
            if (cta == 0) a.dbg[q] = tph[q];
            a.dbg[16 + 10 * cta + q] = tph[q];
        }
    if (cta == 0)
        for (int j = tid; j < n; j += QP_NT) a.w.phys_all[j] = phys[j];
    // ---------------- normalise the stored reflectors, R_kk = mu
    for (int p = cta; p < n; p += G) {
        const int k = pos[p];
        const T rv0 = 1.0 / __ldcg(a.v0g + k), mu = __ldcg(a.mug + k);
        T* col = a.A + (long long)p * lda;
        for (long long i = k + 1 + tid; i < m; i += QP_NT) col[i] = col[i] * rv0;
        if (tid == 0) col[k] = mu;
    }
}

template <typename T, int RPT>
static void* qrp_kernel_ptr() { return (void*)k_qrp_lazy<T, RPT>; }

template <typename T>
static void* qrp_kernel_for(int m) {
    int r = 1;
    while (r * QP_NT < m) r <<= 1;
    switch (r) {
        case 1: return qrp_kernel_ptr<T, 1>();
        case 2: return qrp_kernel_ptr<T, 2>();
        case 4: return qrp_kernel_ptr<T, 4>();
        case 8: return qrp_kernel_ptr<T, 8>();
        case 16: return qrp_kernel_ptr<T, 16>();
        default: return nullptr;
    }
}

template <typename T>
static size_t qrp_smem(int m, int n, int nown, int grid) {
    const size_t vsz = std::max((size_t)m, (size_t)grid * (QP_NB + 1));
    return sizeof(T) * (vsz + (size_t)nown * QP_NB + 6 * (size_t)nown + 33 * 32 + 4 * QP_NB + 8) +
           sizeof(int) * (QP_NB + 3 * (size_t)nown + (size_t)n) + 64;
}

// bytes of the end-of-panel ring with pe_st stages (after the 16-byte alignment of qrp_smem's layout)
template <typename T>
static size_t qrp_ring_bytes(int pe_st) {
    return pe_st >= 2 ? 16 + sizeof(T) * (size_t)pe_st * QP_PE_G * QP_NT : 0;
}

template <typename T>
static int qrp_lazy_grid_t(int m, int n, int* grid, int* nown, int* pe_st = nullptr) {
    void* fn = qrp_kernel_for<T>(m);
    if (!fn) return -7;
    int dev = 0, nsm = 0, per = 0;
    MPJ_CUDA_TRY(cudaGetDevice(&dev));
    MPJ_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    int g = nsm;
    int no = (n + g - 1) / g;
    if (n > 65535) return -7;   // 16-bit phys / pos
    if (g * (QP_NB + 1) > QP_NT * QP_PART_PT || g > 32 * QP_CAND_PL) return -7;
    size_t smem = qrp_smem<T>(m, n, no, g);
    if (smem > 227 * 1024) return -7;
    // end-of-panel ring: 2 stages by default (measured, C5 panel phase 75 -> 67 ms; 3 or 4 stages take L1 from
    // the GEMV pass: 226 -> 229 / 287 ms), or the forced count
    int st = 0;
    if (g_mpj_qrp_pe < 0) {
        st = smem + qrp_ring_bytes<T>(2) <= 227 * 1024 ? 2 : 0;
    } else if (g_mpj_qrp_pe >= 2 && smem + qrp_ring_bytes<T>(g_mpj_qrp_pe) <= 227 * 1024) {
        st = g_mpj_qrp_pe;
    }
    smem += qrp_ring_bytes<T>(st);
    if (pe_st) *pe_st = st;
    MPJ_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // the smallest shared-memory carveout that holds the kernel: the rest of the 256 KB is L1, which stages the
    // GEMV's loads in flight (measured: +48 KB of shared memory slowed the C5 GEMV pass 226 -> 287 ms)
    const int pct = (int)std::min<size_t>(100, (smem + 1024 + 228 * 1024 / 100 - 1) * 100 / (228 * 1024));
    MPJ_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    MPJ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, QP_NT, smem));
    if (per < 1) return -7;
    *grid = g;
    *nown = no;
    return 0;
}

int qrp_lazy_grid(int m, int n, int* grid, int* nown) { return qrp_lazy_grid_t<double>(m, n, grid, nown); }

size_t qrp_lazy_work_doubles(int n, int grid) {
    return (size_t)n * QP_NB + (size_t)grid * (QP_NB + 1) + 2 * (size_t)n;
}

template <typename T>
static int qrp_lazy_t(T* A, long long lda, int m, int n, T* tau, QrWork& w, T* work, int* phys_out,
                      cudaStream_t st) {
    int grid = 0, nown = 0, pe_st = 0;
    int rc = qrp_lazy_grid_t<T>(m, n, &grid, &nown, &pe_st);
    if (rc) return rc;
    void* fn = qrp_kernel_for<T>(m);
    QrpArgs<T> args;
    args.A = A;
    args.lda = lda;
    args.m = m;
    args.n = n;
    args.tau = tau;
    args.w = w;
    args.w.grid = grid;
    args.F = work;
    args.part = work + (size_t)n * QP_NB;
    args.v0g = args.part + (size_t)grid * (QP_NB + 1);
    args.mug = args.v0g + n;
    args.nown = nown;
    args.pe_st = pe_st;
    args.dbg = nullptr;
    static long long* dbg = nullptr;
    if (g_mpj_diag & 1) {
        if (!dbg) cudaMalloc(&dbg, (16 + 10 * 1024) * sizeof(long long));
        args.dbg = dbg;
    }
    void* params[] = {&args};
    MPJ_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(QP_NT), params, qrp_smem<T>(m, n, nown, grid) + qrp_ring_bytes<T>(pe_st), st));
    MPJ_LAUNCHED();
    if (phys_out)
        MPJ_CUDA_TRY(cudaMemcpyAsync(phys_out, w.phys_all, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
    if (args.dbg) {
        static long long h[16 + 10 * 1024];
        cudaMemcpyAsync(h, args.dbg, sizeof(long long) * (16 + 10 * grid), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        const char* names[10] = {"pivot", "pass1", "sync1", "reflector", "pass2", "panel", "cand", "sync2", "recompute", "?"};
        fprintf(stderr, "[qrp timing m=%d n=%d G=%d] ", m, n, grid);
        for (int q = 0; q < 9; ++q) fprintf(stderr, "%s=%.1fms ", names[q], h[q] / 1.965e6);
        fprintf(stderr, "\n[qrp timing over CTAs min/mean/max ms] ");
        for (int q = 0; q < 9; ++q) {
            double mn = 1e30, mx = 0, sm = 0;
            for (int g = 0; g < grid; ++g) {
                const double v = h[16 + 10 * g + q] / 1.965e6;
                mn = v < mn ? v : mn; mx = v > mx ? v : mx; sm += v;
            }
            fprintf(stderr, "%s=%.1f/%.1f/%.1f ", names[q], mn, sm / grid, mx);
        }
        fprintf(stderr, "\n");
    }
    return 0;
}

int qrp_lazy(double* A, long long lda, int m, int n, double* tau, QrWork& w, double* work, int* phys_out,
             cudaStream_t st) {
    return qrp_lazy_t<double>(A, lda, m, n, tau, w, work, phys_out, st);
}
int qrp_lazy_f32(float* A, long long lda, int m, int n, float* tau, QrWork& w, float* work, int* phys_out,
                 cudaStream_t st) {
    return qrp_lazy_t<float>(A, lda, m, n, tau, w, work, phys_out, st);
}

}  // namespace mpj
