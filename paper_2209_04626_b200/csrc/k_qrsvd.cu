// k_qrsvd.cu -- the "QR SVD algorithm in the lower precision" of Alg. 3's AUTO branch (PAPER.md:441-445,
// 515-545: lower(X) = U_low Sigma_low V_low^* "without generating V_low explicitly"), hand-written for
// sm_100a in the steps of DESIGN.md reading c-24:
//   1. k_bidiag32: Householder bidiagonalisation X32 = Q_B B P_B^T in fp32, one persistent cooperative
//      kernel (one CTA per SM, columns dealt round-robin to CTAs; per step: left reflector by the column's
//      owner, its application to the owned columns, the right reflector of row k computed redundantly by
//      every CTA from the updated row, the product (A u) as per-CTA partial sums reduced by row slices,
//      the rank-1 right update; four grid barriers per step);
//   2. k_bdqr32: implicit-shift QR on the upper-bidiagonal B in fp32 (Golub-Kahan step, bulge chased down,
//      shift = smaller singular value of the trailing 2 x 2), one warp: lane 0 runs the dependent rotation
//      chain, the warp does the deflation scans; the left rotations of every step are logged;
//   3. k_rot_apply: the logged left rotations applied to U_B (= I) in fp64, one thread per row (rows
//      across a warp are contiguous in the column-major U: coalesced), steps in log order;
//   4. U_low = Q_B U_B by the fp64 compact-WY application (apply_q_wy) of the fp32 reflectors;
//   5. sigma = |d|, stable descending order, columns of U_low permuted alike.
// The log is processed in chunks (the QR kernel stops when the rotation buffer is full and resumes from
// its saved state), so the buffer is bounded independently of the iteration count.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "jacobi.h"

namespace cg = cooperative_groups;

#define QS_TRY(x)               \
    do {                        \
        int _r = (x);           \
        if (_r != 0) return _r; \
    } while (0)

namespace mpj {

constexpr int BD_NT = 512;
constexpr float U32F = 5.9604644775390625e-08f;   // 2^-24

struct BidiagArgs {
    float* A;
    long long lda;
    int n;
    float* d;        // [n]   diagonal of B
    float* e;        // [n]   superdiagonal of B (e[n-1] = 0)
    float* tau;      // [n]   left reflector scalars (v_k below the diagonal of column k, v_k(0) = 1)
    float* rowbuf;   // [n]   row k of the trailing matrix after the left update
    float* ppart;    // [G][n] per-CTA partial sums of (A u)
    float* p;        // [n]   pi * (A u)
};

// block-wide deterministic sum over BD_NT threads (fixed tree); all threads receive the result
__device__ __forceinline__ float bd_block_sum(float v, float* red) {
    return block_sum(v, red);
}

__global__ void __launch_bounds__(BD_NT, 1) k_bidiag32(BidiagArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ float bd_sm[];
    float* u = bd_sm;                   // right reflector of the current row (n floats)
    __shared__ float red[32];
    __shared__ float s_scal[4];
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NW = BD_NT / 32;
    const int n = a.n;
    const long long lda = a.lda;
    float* A = a.A;
    for (int k = 0; k < n; ++k) {
        // ---- left reflector of column k (owner only; its column is up to date in this CTA)
        if (k % G == cta) {
            float* ak = A + (long long)k * lda;
            const float alpha = ak[k];          // read before the block sum's barriers (tid 0 writes it below)
            float sg = 0.f;
            for (int i = k + 1 + tid; i < n; i += BD_NT) sg += ak[i] * ak[i];
            sg = bd_block_sum(sg, red);
            float tk, mu, v0 = 1.f;
            if (sg == 0.f) {
                tk = alpha >= 0.f ? 0.f : 2.f;
                mu = alpha >= 0.f ? alpha : -alpha;
            } else {
                mu = sqrtf(alpha * alpha + sg);
                v0 = alpha <= 0.f ? alpha - mu : -sg / (alpha + mu);
                tk = 2.f * v0 * v0 / (sg + v0 * v0);
                for (int i = k + 1 + tid; i < n; i += BD_NT) ak[i] = ak[i] / v0;
            }
            if (tid == 0) {
                ak[k] = mu;
                a.d[k] = mu;
                a.tau[k] = tk;
            }
        }
        grid.sync();
        // ---- apply H_k = I - tau v v^T to the owned columns j > k; row k of the result -> rowbuf
        {
            const float tk = __ldcg(a.tau + k);
            const float* v = A + (long long)k * lda;
            int j0 = k + 1 + ((cta - (k + 1) % G) + G) % G;   // first owned column > k
            for (int j = j0 + wid * G; j < n; j += NW * G) {
                float* aj = A + (long long)j * lda;
                float w = 0.f;
                if (tk != 0.f) {
                    for (int i = k + 1 + lane; i < n; i += 32) w += __ldcg(v + i) * aj[i];
                    w = warp_sum(w);
                    w = (aj[k] + w) * tk;
                    for (int i = k + 1 + lane; i < n; i += 32) aj[i] -= w * __ldcg(v + i);
                }
                __syncwarp();
                if (lane == 0) {
                    aj[k] -= w;
                    a.rowbuf[j] = aj[k];
                }
            }
        }
        grid.sync();
        if (k + 1 >= n) break;
        // ---- right reflector of row k over columns k+1..n-1 (every CTA, same fixed-order reduction)
        const int len = n - k - 1;
        float sg = 0.f;
        for (int l = 1 + tid; l < len; l += BD_NT) {
            const float y = __ldcg(a.rowbuf + k + 1 + l);
            sg += y * y;
        }
        sg = bd_block_sum(sg, red);
        if (tid == 0) {
            const float alpha = __ldcg(a.rowbuf + k + 1);
            float pi, mu, v0 = 1.f;
            if (sg == 0.f) {
                pi = alpha >= 0.f ? 0.f : 2.f;
                mu = alpha >= 0.f ? alpha : -alpha;
            } else {
                mu = sqrtf(alpha * alpha + sg);
                v0 = alpha <= 0.f ? alpha - mu : -sg / (alpha + mu);
                pi = 2.f * v0 * v0 / (sg + v0 * v0);
            }
            s_scal[0] = pi;
            s_scal[1] = v0;
            if (cta == 0) a.e[k] = mu;
        }
        __syncthreads();
        const float pi = s_scal[0], v0 = s_scal[1];
        if (pi == 0.f) continue;   // H = I: no right update (same decision in every CTA)
        for (int l = tid; l < len; l += BD_NT) u[l] = l == 0 ? 1.f : __ldcg(a.rowbuf + k + 1 + l) / v0;
        __syncthreads();
        // partial (A u)_i over the owned columns j >= k+1, rows i > k (thread per row: coalesced)
        {
            int j0 = k + 1 + ((cta - (k + 1) % G) + G) % G;
            float* pp = a.ppart + (long long)cta * n;
            for (int i = k + 1 + tid; i < n; i += BD_NT) {
                float acc = 0.f;
                for (int j = j0; j < n; j += G) acc += A[i + (long long)j * lda] * u[j - k - 1];
                pp[i] = acc;
            }
        }
        grid.sync();
        // reduce the partials over CTAs for this CTA's row slice (fixed CTA order)
        {
            const int rows = n - k - 1;
            const int per = (rows + G - 1) / G;
            const int r0 = k + 1 + cta * per, r1 = min(n, r0 + per);
            for (int i = r0 + tid; i < r1; i += BD_NT) {
                float s = 0.f;
                for (int g = 0; g < G; ++g) s += __ldcg(a.ppart + (long long)g * n + i);
                a.p[i] = pi * s;
            }
        }
        grid.sync();
        // A(i, j) -= p_i u_{j-k-1} on the owned columns
        {
            int j0 = k + 1 + ((cta - (k + 1) % G) + G) % G;
            for (int j = j0 + wid * G; j < n; j += NW * G) {
                float* aj = A + (long long)j * lda;
                const float uj = u[j - k - 1];
                for (int i = k + 1 + lane; i < n; i += 32) aj[i] -= __ldcg(a.p + i) * uj;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------------------
struct BdqrState {
    int hi;            // bottom of the unreduced part (n - 1 at the start)
    int rc;            // 0 running/ok, -3 exact zero on the diagonal, 1 no convergence
    int done;
    int nsteps;        // steps logged in this chunk
    long long nrot;    // rotations logged in this chunk
    long long it;      // total QR steps so far
};

// The rotation chain of the bidiagonal QR is one dependent sequence: r = sqrt(f^2 + g^2) and one reciprocal
// instead of hypotf and two divisions (the scaled X keeps |f|, |g| <= ~1, so f^2 + g^2 cannot overflow; below
// 2^-60 the scaled hypotf avoids underflow).  A few ulp from the oracle's hypotf / division (reading c-24).
__device__ __forceinline__ void givens32(float f, float g, float& c, float& s, float& r) {
    if (g == 0.f) { c = 1.f; s = 0.f; r = f; return; }
    if (f == 0.f) { c = 0.f; s = 1.f; r = g; return; }
    float rr = __fsqrt_rn(__fmaf_rn(f, f, __fmul_rn(g, g)));
    if (rr < 8.6736174e-19f) rr = hypotf(f, g);
    const float ri = __frcp_rn(rr);
    c = f * ri;
    s = g * ri;
    r = rr;
}

__device__ __forceinline__ float sv_min_2x2(float f, float g, float h) {
    const float fa = fabsf(f), ga = fabsf(g), ha = fabsf(h);
    const float fhmn = fminf(fa, ha), fhmx = fmaxf(fa, ha);
    if (fhmn == 0.f) return 0.f;
    if (ga < fhmx) {
        const float as = 1.f + fhmn / fhmx, at = (fhmx - fhmn) / fhmx, au = (ga / fhmx) * (ga / fhmx);
        const float c = 2.f / (sqrtf(as * as + au) + sqrtf(at * at + au));
        return fhmn * c;
    }
    const float au = fhmx / ga;
    if (au == 0.f) return (fhmn * fhmx) / ga;
    const float as = 1.f + fhmn / fhmx, at = (fhmx - fhmn) / fhmx;
    const float c = 1.f / (sqrtf(1.f + (as * au) * (as * au)) + sqrtf(1.f + (at * au) * (at * au)));
    return (fhmn * c) * au * 2.f;
}

// One warp.  Runs QR steps until B is diagonal, a rotation buffer chunk is full, or an error.
__global__ void __launch_bounds__(32, 1) k_bdqr32(float* dg, float* eg, int n, BdqrState* stp, float2* rot,
                                                   int2* steps, long long cap_rot, int cap_steps, long long maxit) {
    extern __shared__ float q_sm[];
    float* d = q_sm;
    float* e = q_sm + n;
    const int lane = threadIdx.x;
    for (int i = lane; i < n; i += 32) { d[i] = dg[i]; e[i] = eg[i]; }
    __shared__ int s_hi, s_lo, s_stop, s_zero;
    __shared__ float s_dmax;
    BdqrState st = *stp;
    if (lane == 0) { s_hi = st.hi; s_stop = 0; }
    long long nrot = 0;
    int nsteps = 0;
    __syncwarp();
    while (true) {
        int hi = s_hi;
        if (hi <= 0) break;
        // deflation: e_i = 0 when |e_i| <= u32 (|d_i| + |d_{i+1}|), i < hi
        for (int i = lane; i < hi; i += 32)
            if (fabsf(e[i]) <= U32F * (fabsf(d[i]) + fabsf(d[i + 1]))) e[i] = 0.f;
        __syncwarp();
        if (lane == 0) {
            while (hi > 0 && e[hi - 1] == 0.f) --hi;
            int lo = hi > 0 ? hi - 1 : 0;
            while (lo > 0 && e[lo - 1] != 0.f) --lo;
            s_hi = hi;
            s_lo = lo;
        }
        __syncwarp();
        hi = s_hi;
        if (hi <= 0) break;
        const int lo = s_lo;
        int zero = 0;
        float dmax = 0.f;
        for (int i = lo + lane; i <= hi; i += 32) {
            zero |= d[i] == 0.f;
            dmax = fmaxf(dmax, fabsf(d[i]));
        }
        zero = __any_sync(0xffffffffu, zero);
        dmax = warp_max(dmax);
        if (zero) { if (lane == 0) st.rc = -3; break; }
        if (nrot + (hi - lo) > cap_rot || nsteps >= cap_steps) break;      // chunk full: resume later
        if (st.it + 1 > maxit) { if (lane == 0) st.rc = 1; break; }
        st.it += 1;
        if (lane == 0) {
            float shift = sv_min_2x2(d[hi - 1], e[hi - 1], d[hi]);
            if ((shift / dmax) * (shift / dmax) < U32F) shift = 0.f;
            float f = (fabsf(d[lo]) - shift) * ((d[lo] >= 0.f ? 1.f : -1.f) + shift / d[lo]);
            float g = e[lo];
            float2* rp = rot + nrot;
            for (int i = lo; i < hi; ++i) {
                float cr, sr, r, cl, sl;
                givens32(f, g, cr, sr, r);
                if (i > lo) e[i - 1] = r;
                f = cr * d[i] + sr * e[i];
                e[i] = cr * e[i] - sr * d[i];
                g = sr * d[i + 1];
                d[i + 1] = cr * d[i + 1];
                givens32(f, g, cl, sl, r);
                d[i] = r;
                f = cl * e[i] + sl * d[i + 1];
                d[i + 1] = cl * d[i + 1] - sl * e[i];
                if (i + 1 < hi) {
                    g = sl * e[i + 1];
                    e[i + 1] = cl * e[i + 1];
                }
                rp[i - lo] = make_float2(cl, sl);
            }
            e[hi - 1] = f;
            steps[nsteps] = make_int2(lo, hi);
        }
        nrot += hi - lo;
        ++nsteps;
        __syncwarp();
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) { dg[i] = d[i]; eg[i] = e[i]; }
    if (lane == 0) {
        st.hi = s_hi;
        st.nsteps = nsteps;
        st.nrot = nrot;
        st.done = (st.rc != 0 || s_hi <= 0) ? 1 : 0;
        if (st.rc == 0 && s_hi <= 0)
            for (int j = 0; j < n; ++j)
                if (d[j] == 0.f) { st.rc = -3; break; }   // an exact zero singular value
        *stp = st;
    }
}

// U(:, [i i+1]) <- U(:, [i i+1]) [[c, -s], [s, c]] for the logged steps, one thread per row (fp64)
__global__ void k_rot_apply(double* U, long long ldu, int n, const float2* __restrict__ rot,
                            const int2* __restrict__ steps, int nsteps) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    double* ur = U + r;
    const float2* rp = rot;
    for (int s = 0; s < nsteps; ++s) {
        const int2 sp = steps[s];
        double carry = ur[(long long)sp.x * ldu];
        int i = sp.x;
#pragma unroll 4
        for (; i < sp.y; ++i) {
            const float2 cs = rp[i - sp.x];
            const double b = ur[(long long)(i + 1) * ldu];
            const double c = cs.x, sn = cs.y;
            ur[(long long)i * ldu] = c * carry + sn * b;
            carry = c * b - sn * carry;
        }
        ur[(long long)sp.y * ldu] = carry;
        rp += sp.y - sp.x;
    }
}

// The same rotations, RB consecutive steps per pass over a row (wavefront): at outer position p step s applies
// its rotation at i = p - s, so a row keeps a window of RB + 1 elements in registers and every element is read
// and written once per RB steps instead of once per step.  Positions outside a step's [lo, hi) are identity.
// Identical arithmetic per rotation as k_rot_apply (same order of the two FMAs per element).
template <int RB>
__global__ void k_rot_apply_wave(double* U, long long ldu, int n, const float2* __restrict__ rot,
                                 const int2* __restrict__ steps, const long long* __restrict__ offs, int nsteps) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    double* ur = U + r;
    for (int s0 = 0; s0 < nsteps; s0 += RB) {
        int lo[RB], hi[RB];
        long long of[RB];
        int lmin = 1 << 30, hmax = -1;
#pragma unroll
        for (int s = 0; s < RB; ++s) {
            if (s0 + s < nsteps) {
                const int2 sp = steps[s0 + s];
                lo[s] = sp.x;
                hi[s] = sp.y;
                of[s] = offs[s0 + s] - sp.x;
            } else {
                lo[s] = 1 << 30;
                hi[s] = -1;
                of[s] = 0;
            }
            lmin = min(lmin, lo[s]);
            hmax = max(hmax, hi[s]);
        }
        // window w[j] = u[p - RB + 1 + j], j = 0..RB, at outer position p
        double w[RB + 1];
#pragma unroll
        for (int j = 0; j < RB; ++j) w[j] = 0.0;
        w[RB - 1] = ur[(long long)lmin * ldu];
        const int pend = hmax - 1 + RB - 1;
        for (int p = lmin; p <= pend; ++p) {
            w[RB] = (p + 1 <= hmax) ? ur[(long long)(p + 1) * ldu] : 0.0;
#pragma unroll
            for (int s = 0; s < RB; ++s) {
                const int i = p - s;
                if (i >= lo[s] && i < hi[s]) {
                    const float2 cs = rot[of[s] + i];
                    const double c = cs.x, sn = cs.y;
                    const double a = w[RB - 1 - s], b = w[RB - s];
                    w[RB - 1 - s] = c * a + sn * b;
                    w[RB - s] = c * b - sn * a;
                }
            }
            const int q = p - RB + 1;                 // element leaving the window: final for this batch
            if (q >= lmin) ur[(long long)q * ldu] = w[0];
#pragma unroll
            for (int j = 0; j < RB; ++j) w[j] = w[j + 1];
        }
        // the window still holds u[pend - RB + 2 .. pend + 1] in w[0 .. RB - 1]
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            const int q = pend - RB + 2 + j;
            if (q >= lmin && q <= hmax) ur[(long long)q * ldu] = w[j];
        }
    }
}

__global__ void k_step_offsets(const int2* steps, int nsteps, long long* offs) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        long long o = 0;
        for (int s = 0; s < nsteps; ++s) {
            offs[s] = o;
            o += steps[s].y - steps[s].x;
        }
    }
}

// packed fp64 copy of the fp32 reflectors (for the WY application) and |d| as fp64 sort keys
__global__ void k_qrsvd_prep(const float* A, long long lda, const float* tau, const float* d, int n, double* P,
                             long long ldp, double* tau64, double* keys) {
    for (long long j = blockIdx.y; j < n; j += gridDim.y) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            tau64[j] = (double)tau[j];
            keys[j] = (double)fabsf(d[j]);
        }
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ldp; i += (long long)gridDim.x * blockDim.x)
            P[i + j * ldp] = i < n ? (double)A[i + j * lda] : 0.0;
    }
}

// dst(:, rank[j]) = src(:, j); S_out[rank[j]] = keys[j] (optional)
__global__ void k_permute_cols(const double* src, long long lds, const int* rank, double* dst, long long ldd,
                               long long rows, const double* keys, float* S_out) {
    const long long j = blockIdx.y;
    const long long dj = rank[j];
    if (S_out && blockIdx.x == 0 && threadIdx.x == 0) S_out[dj] = (float)keys[j];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows; i += (long long)gridDim.x * blockDim.x)
        dst[i + dj * ldd] = src[i + j * lds];
}

size_t qrsvd32_work_bytes(int n) {
    const long long cap_rot = std::min<long long>((long long)n * n + 64, 16LL << 20);
    const long long cap_steps = 4LL * n + 64;
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    size_t b = 0;
    b += sizeof(float) * (size_t)n * 4;                 // d, e, tau, rowbuf
    b += sizeof(float) * (size_t)n;                     // p
    b += sizeof(float) * (size_t)nsm * n;               // ppart
    b += sizeof(float2) * (size_t)cap_rot + (sizeof(int2) + sizeof(long long)) * (size_t)cap_steps + 512;
    b += sizeof(double) * (size_t)n * 2 + sizeof(int) * (size_t)n + 1024;
    return b;
}

int qrsvd32(float* X32, long long ldx, int n, double* U, long long ldu, double* UB, double* P, long long ldp,
            void* work, double* wy_work, int* bad, cudaStream_t st, float* S_out) {
    if (n < 1) return -1;
    int dev = 0, nsm = 148, per = 0;
    MPJ_CUDA_TRY(cudaGetDevice(&dev));
    MPJ_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const long long cap_rot = std::min<long long>((long long)n * n + 64, 16LL << 20);
    const int cap_steps = 4 * n + 64;
    char* w = reinterpret_cast<char*>(work);
    auto take = [&](size_t bytes) { char* p = w; w += (bytes + 255) & ~size_t(255); return (void*)p; };
    float* d = (float*)take(sizeof(float) * n);
    float* e = (float*)take(sizeof(float) * n);
    float* tau = (float*)take(sizeof(float) * n);
    float* rowbuf = (float*)take(sizeof(float) * n);
    float* p = (float*)take(sizeof(float) * n);
    float* ppart = (float*)take(sizeof(float) * (size_t)nsm * n);
    float2* rot = (float2*)take(sizeof(float2) * (size_t)cap_rot);
    int2* steps = (int2*)take(sizeof(int2) * (size_t)cap_steps);
    long long* offs = (long long*)take(sizeof(long long) * (size_t)cap_steps);
    BdqrState* bst = (BdqrState*)take(sizeof(BdqrState));
    double* tau64 = (double*)take(sizeof(double) * n);
    double* keys = (double*)take(sizeof(double) * n);
    int* rank = (int*)take(sizeof(int) * n);

    // 1. bidiagonalisation (cooperative, one CTA per SM)
    const size_t smem = sizeof(float) * (size_t)n;
    MPJ_CUDA_TRY(set_smem(k_bidiag32, smem));
    MPJ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bidiag32, BD_NT, smem));
    if (per < 1) return -7;
    MPJ_CUDA_TRY(cudaMemsetAsync(e, 0, sizeof(float) * n, st));
    BidiagArgs ba{X32, ldx, n, d, e, tau, rowbuf, ppart, p};
    void* params[] = {&ba};
    MPJ_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_bidiag32, dim3(nsm), dim3(BD_NT), params, smem, st));
    MPJ_LAUNCHED();

    // 2.-3. QR on B in chunks, rotations applied to U_B = I after each chunk
    QS_TRY(set_identity<double>(UB, ldu, ldu, n, st));
    BdqrState h0{};
    h0.hi = n - 1;
    MPJ_CUDA_TRY(cudaMemcpyAsync(bst, &h0, sizeof(h0), cudaMemcpyHostToDevice, st));
    const size_t qsm = sizeof(float) * 2 * (size_t)n;
    MPJ_CUDA_TRY(set_smem(k_bdqr32, qsm));
    const long long maxit = 6LL * n * n + 60;
    BdqrState hs{};
    for (int chunk = 0; chunk < 1 << 20; ++chunk) {
        k_bdqr32<<<1, 32, qsm, st>>>(d, e, n, bst, rot, steps, cap_rot, cap_steps, maxit);
        MPJ_LAUNCHED();
        MPJ_CUDA_TRY(cudaMemcpyAsync(&hs, bst, sizeof(hs), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
        if (hs.nsteps > 0) {
            k_step_offsets<<<1, 32, 0, st>>>(steps, hs.nsteps, offs);
            MPJ_LAUNCHED();
            k_rot_apply_wave<8><<<(unsigned)ceil_div(n, 32), 32, 0, st>>>(UB, ldu, n, rot, steps, offs, hs.nsteps);
            MPJ_LAUNCHED();
        }
        if (hs.done) break;
        if (hs.nsteps == 0) return -4;   // no progress: cannot happen unless a chunk cannot hold one step
    }
    if (hs.rc == -3) { MPJ_CUDA_TRY(cudaMemsetAsync(bad, 0xff, sizeof(int), st)); return 0; }
    if (hs.rc != 0) {
        mpj_record_cuda_error(cudaErrorUnknown, "fp32 QR SVD: bidiagonal QR did not converge in 6 n^2 steps",
                              __FILE__, __LINE__);
        return -4;
    }

    // 4. U_low = Q_B U_B (fp64 WY application of the fp32 reflectors)
    k_qrsvd_prep<<<dim3((unsigned)ceil_div(ldp, 256) < 64 ? (unsigned)ceil_div(ldp, 256) : 64, (unsigned)n), 256, 0, st>>>(
        X32, ldx, tau, d, n, P, ldp, tau64, keys);
    MPJ_LAUNCHED();
    QS_TRY(apply_q_wy(P, n, n, ldp, tau64, UB, ldu, n, wy_work, st));
    // 5. stable descending order of |d|, columns permuted alike
    QS_TRY(rank_desc(keys, n, rank, st));
    k_permute_cols<<<dim3((unsigned)ceil_div(ldu, 256) < 64 ? (unsigned)ceil_div(ldu, 256) : 64, (unsigned)n), 256, 0, st>>>(
        UB, ldu, rank, U, ldu, ldu, keys, S_out);
    MPJ_LAUNCHED();
    MPJ_CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace mpj
