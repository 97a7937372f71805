// k_jacobi.cu -- block round-robin one-sided Jacobi kernels (fp32 and fp64).
//
// One Jacobi *round* (Alg. 1, in block form; DESIGN.md
// "Block Jacobi") processes the N_b/2 disjoint block pairs (I, J) of the
// circle-method schedule at once:
//   k_pair_gram   : partial Gram G = W^T W, W = [X_I X_J] (m x w), split over
//                   row slabs -> partial[pair][split][W][W]
//   k_pair_solve  : fixed-order reduction of the partials, pair metric
//                   max |g_pq| / sqrt(g_pp g_qq), and -- if it exceeds eps_tol
//                   -- the 2b x 2b two-sided inner Jacobi solve giving
//                   E = V_blk - I (reading c-5)
//   k_pair_update : W <- W + W E and V_IJ <- V_IJ + V_IJ E (delta form, F3)
// Columns of X / V never move on one GPU: block ids index column slabs.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include "common.cuh"
#include "jacobi.h"

namespace mpj {

template <typename T> struct RealTraits;
template <> struct RealTraits<float> {
    static constexpr float rsqrt_u = 4096.0f;              // 1/sqrt(2^-24)
};
template <> struct RealTraits<double> {
    static constexpr double rsqrt_u = 94906265.62425156;   // 1/sqrt(2^-53)
};

// pointer to pair-local column c (c < w0 + w1) of X (v = false) or V (v = true)
template <typename T>
__device__ __forceinline__ T* pair_col(const PairDesc<T>& d, int c, bool v, long long ld) {
    return c < d.w0 ? (v ? d.v0 : d.x0) + (long long)c * ld : (v ? d.v1 : d.x1) + (long long)(c - d.w0) * ld;
}

// ------------------------------------------------------------------------
// k_pair_gram: grid (nsplit, npairs), 64 threads (8 x 8), thread tile
// (W/8) x (W/8) of G.  Row slab [split*R, min((split+1)*R, m_pad)) in k-tiles
// of KT rows, natural column-major staging in shared memory.
// ------------------------------------------------------------------------
template <typename T, int W>
__global__ void __launch_bounds__(64) k_pair_gram(JacobiRound<T> a) {
    reset_publication(a);
    if (pair_unchanged(a, a.pd[blockIdx.y])) return;
    constexpr int KT = 32;
    constexpr int VEC = 16 / sizeof(T);       // elements per 16-byte vector
    constexpr int S = KT + VEC;               // padded column stride (conflict-free)
    constexpr int TP = W / 8;
    __shared__ __align__(16) T Ws[2][W * S];
    __shared__ const T* colp[W];

    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
    const PairDesc<T> pd = a.pd[pair];
    const int w = pd.w0 + pd.w1;
    if (tid < W) colp[tid] = tid < w ? pair_col(pd, tid, false, a.ldx) : nullptr;
    __syncthreads();

    const long long rbeg = (long long)split * a.rows_per_split;
    const long long rend = min(rbeg + (long long)a.rows_per_split, (long long)a.m_pad);
    const int ntile = (int)((rend - rbeg + KT - 1) / KT);

    T acc[TP][TP];
#pragma unroll
    for (int i = 0; i < TP; ++i)
#pragma unroll
        for (int j = 0; j < TP; ++j) acc[i][j] = T(0);

    constexpr int VPC = KT / VEC;                       // vectors per column per tile
    constexpr int NV = (W * VPC + 63) / 64;             // vectors per thread
    auto load_tile = [&](int t, int stage) {
        const long long r0 = rbeg + (long long)t * KT;
#pragma unroll
        for (int u = 0; u < NV; ++u) {
            int v = tid + 64 * u;
            if (v < W * VPC) {
                int c = v / VPC, ch = v % VPC;
                T* dst = &Ws[stage][c * S + ch * VEC];
                const T* cp = colp[c];
                if (cp != nullptr && r0 + ch * VEC < rend) {
                    const T* src = cp + r0 + ch * VEC;
                    unsigned saddr = (unsigned)__cvta_generic_to_shared(dst);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(src));
                } else {
                    *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };

    if (ntile > 0) load_tile(0, 0);
    for (int t = 0; t < ntile; ++t) {
        const int st = t & 1;
        if (t + 1 < ntile) {
            load_tile(t + 1, st ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();
        const T* ws = Ws[st];
#pragma unroll
        for (int kk = 0; kk < KT; kk += VEC) {
            T av[TP][VEC], bv[TP][VEC];
#pragma unroll
            for (int i = 0; i < TP; ++i) {
                const float4 x = *reinterpret_cast<const float4*>(&ws[(ty + 8 * i) * S + kk]);
                const float4 y = *reinterpret_cast<const float4*>(&ws[(tx + 8 * i) * S + kk]);
                *reinterpret_cast<float4*>(&av[i][0]) = x;
                *reinterpret_cast<float4*>(&bv[i][0]) = y;
            }
#pragma unroll
            for (int v = 0; v < VEC; ++v)
#pragma unroll
                for (int i = 0; i < TP; ++i)
#pragma unroll
                    for (int j = 0; j < TP; ++j) acc[i][j] = fma(av[i][v], bv[j][v], acc[i][j]);
        }
        __syncthreads();
    }
    T* out = a.partial + ((long long)pair * a.nsplit + split) * (W * W);
#pragma unroll
    for (int i = 0; i < TP; ++i)
#pragma unroll
        for (int j = 0; j < TP; ++j) out[(ty + 8 * i) * W + (tx + 8 * j)] = acc[i][j];
}

// ------------------------------------------------------------------------
// Inner 2b x 2b solve (reading c-5), one CTA per pair, G and E in shared
// memory.  The circle-method schedule of the 2b indices is tabulated once per
// CTA (pairs of a round, pair and partner of an index).  The rotation
// parameters are the oracle's (c-3) formulas with IEEE div/sqrt; inactive
// pairs carry the identity (c, s) = (1, 0).  See inner_solve_dev for the
// thread organisation.
// ------------------------------------------------------------------------
// Inner-solve thread layout (see inner_solve_dev): NB_MAX pair-pair blocks of
// G, W/2 pairs x W/8 eight-row chunks of E, and one warp for the rotations.
template <int W>
constexpr int inner_nb_max() { return (W / 2) * (W / 2 + 1) / 2; }
template <int W>
constexpr int inner_g_threads() { return (inner_nb_max<W>() + 31) / 32 * 32; }
template <int W>
constexpr int inner_e_items() { return (W / 2) * (W / 8); }
// two leading "critical" warps: per round they update the diagonal blocks and the blocks that hold the
// off-diagonal element of a next-round pair, then release the rotation warp (named barrier 1)
constexpr int INNER_CRIT = 64;
template <int W>
constexpr int inner_nt() { return INNER_CRIT + inner_g_threads<W>() + (inner_e_items<W>() + 31) / 32 * 32 + 32; }

// rotation of one pair: (c, s), c - 1 and an active flag, read with one vector load
template <typename T>
struct __align__(4 * sizeof(T)) Rot4 {
    T c, s, cm1, act;
};

template <typename T, int W>
struct InnerSmem {
    static constexpr int GS = W + 1;
    static constexpr int R = W - 1;                    // max rounds per inner sweep
    T G[W * (W + 1)];
    // fp32: E stored by columns (E[row][col] at E[col * ES + row]) and updated with 16-byte vectors;
    // fp64: by rows (E[row * ES + col]), which measured faster for the 8-byte element
    static constexpr bool ECOL = sizeof(T) == 4;
    static constexpr int EV = 16 / sizeof(T);          // elements per 16-byte vector
    static constexpr int ES = ECOL ? W + EV : W + 1;
    alignas(16) T E[W * ES];
    static __device__ __forceinline__ int eidx(int row, int col) { return ECOL ? col * ES + row : row * ES + col; }
    Rot4<T> rot[2][W / 2];                             // current / next round
    T rt[2][W / 2], rg[2][W / 2], rpp[2][W / 2], rqq[2][W / 2];   // exact 2x2 diagonal update
    unsigned short spq[R][W / 2];                      // pair k of round r: p | q << 8 (p < q; q may be the bye)
    unsigned char knx[R][W];                           // pair of index i in round r
    short crit[R][W / 2];                              // round r: block (kA | kB << 8) holding next-round pair k' (-1: none / duplicate)
    unsigned cmask[R][(W / 2 * (W / 2 + 1) / 2 + 31) / 32];   // round r: bitmask of those blocks
    int nrot[2];
    T red[32];
    long long dbg_t[2][32];                            // per-warp phase end clocks (debug timing only)
};

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

// (x, y) <- (c x - s y, s x + c y); identity exactly when (c, s) = (1, 0)
template <typename T>
__device__ __forceinline__ void rot2(T c, T s, T& x, T& y) {
    const T nx = fma_rn(c, x, -mul_rn(s, y));
    const T ny = fma_rn(s, x, mul_rn(c, y));
    x = nx;
    y = ny;
}

// reciprocal and reciprocal square root: MUFU approximation + two Newton steps (fp64)
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    return y * fma(-h * y, y, 1.5);
}

// rotation parameters from the pair's Gram entries (indices p < q): (c, s), t, c - 1; returns active
template <typename T>
__device__ __forceinline__ int rotation_from(bool valid, T gpp, T gqq, T gpq, T tol_in, T& c, T& sn, T& t, T& cm1) {
    c = T(1); sn = T(0); t = T(0); cm1 = T(0);
    // Alg. 1 guard |x_q^T x_p| > eps ||x_p|| ||x_q||
    if (!(valid && gpp > T(0) && gqq > T(0) && fabs(gpq) > tol_in * sqrt(gpp) * sqrt(gqq))) return 0;
    // closest-to-identity rotation (reading c-3)
    if constexpr (sizeof(T) == 4) {
        // fp32 stage (an initial guess refined in fp64): MUFU rsqrt / fast
        // division, a few ulp from the IEEE formulas (DESIGN.md c-14)
        const float zeta = __fdividef(gqq - gpp, 2.0f * gpq);
        if (fabsf(zeta) > RealTraits<float>::rsqrt_u) {
            t = __fdividef(0.5f, zeta);
        } else {
            const float r1 = fmaf(zeta, zeta, 1.0f);
            const float sq = r1 * rsqrtf(r1);
            t = __fdividef(zeta >= 0.0f ? 1.0f : -1.0f, fabsf(zeta) + sq);
        }
        const float r2 = fmaf(t, t, 1.0f);
        c = rsqrtf(r2);
        sn = t * c;
        cm1 = -__fdividef(t * t * c, 1.0f + r2 * c);
    } else {
        // fp64: the same formulas with MUFU reciprocal / rsqrt refined by two Newton steps (<= 2 ulp
        // from the IEEE quotients and roots; the refinement's accuracy is set by the outer fp64
        // Gram and update, the rotation only has to be orthogonal to u64: c^2 + s^2 = 1 + O(u64))
        const double zeta = (gqq - gpp) * rcp_nr(2.0 * gpq);
        if (fabs(zeta) > RealTraits<double>::rsqrt_u) {
            t = 0.5 * rcp_nr(zeta);
        } else {
            const double r1 = fma(zeta, zeta, 1.0);
            const double sq = r1 * rsqrt_nr(r1);
            t = (zeta >= 0.0 ? 1.0 : -1.0) * rcp_nr(fabs(zeta) + sq);
        }
        const double r2 = fma(t, t, 1.0);
        c = rsqrt_nr(r2);
        sn = t * c;
        cm1 = -(t * t * c) * rcp_nr(1.0 + r2 * c);
    }
    return 1;
}

// rotation parameters of pair k (indices p < q) into buffer `buf`; returns active
template <typename T, int W>
__device__ __forceinline__ int set_rotation(InnerSmem<T, W>& sm, int buf, int k, int q, int w, T gpp, T gqq, T gpq,
                                            T tol_in) {
    T c, sn, t, cm1;
    const int active = rotation_from<T>(q < w, gpp, gqq, gpq, tol_in, c, sn, t, cm1);
    Rot4<T> r4;
    r4.c = c;
    r4.s = sn;
    r4.cm1 = cm1;
    r4.act = active ? T(1) : T(0);
    sm.rot[buf][k] = r4;
    sm.rt[buf][k] = t;
    sm.rg[buf][k] = gpq;
    sm.rpp[buf][k] = gpp;
    sm.rqq[buf][k] = gqq;
    return active;
}

// Inner solve, two phases per round of the circle method on the w2 indices
// (pairs k = 0..P-1 of round r are (sp[r][k], sq[r][k]), p < q, q = w the bye
// when w is odd).  G is kept as its upper triangle G[min][max] (+ diagonal):
//   phase A  thread t < NB = P(P+1)/2 owns the pair-pair block (kA, kB),
//            kA <= kB (fixed for the whole solve): the 2 x 2 block
//            G[{p_A,q_A}][{p_B,q_B}] <- R_A^T G R_B (B's column rotation first,
//            then A's row rotation; kA == kB: the exact 2 x 2 diagonal update).
//            Every element of G is written by exactly one thread.
//   barrier
//   phase B  the last warp: lane kn computes the rotation of pair kn of the
//            next round from the fresh G (reading c-3); the threads between
//            NB and the last warp apply the current rotations to E's columns
//            (E <- (I + E) J - I, delta form).
//   barrier (OR-reduced at the end of an inner sweep: stop when no rotation)
// Rotations of one round act on disjoint index pairs, so the result is that
// of the oracle's sequential loop up to the rounding order of the two
// rotations applied to an off-diagonal block (reading c-5).
// Does any pair (p < q < w) pass the rotation guard of set_rotation (reading
// c-3)?  Upper-triangle storage; this thread's share of the pairs.
template <typename T, int W>
__device__ __forceinline__ int any_pair_above(const InnerSmem<T, W>& sm, int w, T tol_in) {
    constexpr int GS = InnerSmem<T, W>::GS;
    int f = 0;
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
        const int p = e / w, q = e - (e / w) * w;
        if (p < q) {
            const T gpp = sm.G[p * GS + p], gqq = sm.G[q * GS + q], gpq = sm.G[p * GS + q];
            f |= (gpp > T(0) && gqq > T(0) && fabs(gpq) > tol_in * sqrt(gpp) * sqrt(gqq)) ? 1 : 0;
        }
    }
    return f;
}

template <typename T, int W>
__device__ int inner_solve_dev(InnerSmem<T, W>& sm, int w, T tol_in, int max_inner, int* sweeps_used,
                               long long* dbg = nullptr) {
    constexpr int GS = InnerSmem<T, W>::GS;
    constexpr int NG = inner_g_threads<W>();
    constexpr int NCH = W / 8;                          // eight-row chunks of E per pair
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31;
    const int w2 = w + (w & 1);
    const int P = w2 / 2, NR = w2 - 1;
    const int NB = P * (P + 1) / 2;
    const int pwarp0 = nt - 32;                         // first thread of the rotation warp
    constexpr int NCW = (W / 2 * (W / 2 + 1) / 2 + 31) / 32;
    for (int e = tid; e < NR * P; e += nt) {
        const int r = e / P, k = e - (e / P) * P;
        const int x = rr_slot(r, k, w2), y = rr_slot(r, w2 - 1 - k, w2);
        sm.spq[r][k] = (unsigned short)(min(x, y) | (max(x, y) << 8));
        sm.knx[r][x] = (unsigned char)k;
        sm.knx[r][y] = (unsigned char)k;
    }
    for (int e = tid; e < NR * NCW; e += nt) sm.cmask[e / NCW][e % NCW] = 0u;
    __syncthreads();
    // critical blocks of round r: the block (min(kx, ky), max(kx, ky)) of round r that holds the element
    // (x, y) of next-round pair k' (kx, ky: the round-r pairs of x and y); first claimer keeps it
    for (int e = tid; e < NR * P; e += nt) {
        const int r = e / P, k = e - (e / P) * P;
        const int rn = r + 1 < NR ? r + 1 : 0;
        const unsigned pq = sm.spq[rn][k];
        const int x = pq & 255, y = pq >> 8;
        short blk = -1;
        if (y < w && NR > 1) {
            const int kx = sm.knx[r][x], ky = sm.knx[r][y];
            const int a0 = min(kx, ky), b0 = max(kx, ky);
            const int id = a0 * P - a0 * (a0 - 1) / 2 + (b0 - a0);
            const unsigned bit = 1u << (id & 31);
            if (a0 != b0 && !(atomicOr(&sm.cmask[r][id >> 5], bit) & bit)) blk = (short)(a0 | (b0 << 8));
        }
        sm.crit[r][k] = blk;
    }
    constexpr int EV = InnerSmem<T, W>::EV, ES = InnerSmem<T, W>::ES;
    for (int i = tid; i < W * ES; i += nt) sm.E[i] = T(0);
    if (tid < 2) sm.nrot[tid] = 0;
    // fixed roles: pair-pair block (kA, kB) of G, or (pair kE, row chunk cE) of E: chunk c holds the
    // rows (j NCH + c) EV .. + EV - 1, j < 8 / EV, so that the NCH lanes of a pair read a contiguous
    // run of every column with 16-byte accesses
    int kA = -1, kB = -1, kE = -1, r0E = 0, myblk = -1;
    const int gt = tid - INNER_CRIT;                    // non-critical G thread index
    if (tid >= INNER_CRIT && gt < NB) {
        int rem = gt, row = 0;
        while (rem >= P - row) { rem -= P - row; ++row; }
        kA = row;
        kB = row + rem;
        myblk = gt;
    } else if (gt >= NG && gt < NG + P * NCH) {
        kE = (gt - NG) / NCH;
        r0E = (gt - NG) % NCH;                         // chunk index c
        // row-major E: rows c, c + NCH, ..., c + 7 NCH (interleaved, so that the NCH lanes of a pair hit
        // distinct banks; 8-row blocks put them only 0 or 8 double-words apart)
    }
    __syncthreads();
    if (max_inner < 1) { if (sweeps_used) *sweeps_used = 0; return 0; }
    int f_cur = 0, f_next = 0, my_cnt = 0;
    if (tid >= pwarp0 && lane < P) {
        const unsigned pq = sm.spq[0][lane];
        const int p = pq & 255, q = pq >> 8;
        const T gpp = sm.G[p * GS + p];
        const T gqq = q < w ? sm.G[q * GS + q] : T(0);
        const T gpq = q < w ? sm.G[p * GS + q] : T(0);
        f_cur = set_rotation<T, W>(sm, 0, lane, q, w, gpp, gqq, gpq, tol_in);
    }
    __syncthreads();
    int sweep = 0, r = 0, buf = 0;
    if (!__syncthreads_or(any_pair_above<T, W>(sm, w, tol_in))) {   // already converged: the check sweep only
        if (sweeps_used) *sweeps_used = 1;
        return 0;
    }
    long long t_start = 0;
    const int warp = tid >> 5;
    while (true) {
        const bool last = (r == NR - 1);
        const int rn = last ? 0 : r + 1;
        if (dbg && tid == 0) t_start = clock64();
        // One phase per round.  The critical warps update the diagonal blocks and the blocks holding the
        // next round's off-diagonal elements, then release the rotation warp (named barrier 1), which
        // computes the next round's rotations while the other G warps finish the remaining blocks and the
        // E warps apply this round's rotations to E; one CTA barrier ends the round.
        auto g_block = [&](const int kA, const int kB) {
            const Rot4<T> RA = sm.rot[buf][kA];
            const unsigned pqa = sm.spq[r][kA];
            const int pa = pqa & 255, qa = pqa >> 8;
            if (kA == kB) {
                if (RA.act != T(0)) {
                    const T t = sm.rt[buf][kA], g = sm.rg[buf][kA];
                    sm.G[pa * GS + pa] = fma_rn(-t, g, sm.rpp[buf][kA]);
                    sm.G[qa * GS + qa] = fma_rn(t, g, sm.rqq[buf][kA]);
                    sm.G[pa * GS + qa] = T(0);
                    ++my_cnt;
                }
            } else {
                const Rot4<T> RB = sm.rot[buf][kB];
                if (RA.act != T(0) || RB.act != T(0)) {
                    const unsigned pqb = sm.spq[r][kB];
                    const int pb = pqb & 255, qb = pqb >> 8;
                    const bool qav = qa < w, qbv = qb < w;
                    // p_A < q_A and p_B < q_B; the block's canonical positions
                    const int i00 = pa < pb ? pa * GS + pb : pb * GS + pa;
                    const int i01 = pa < qb ? pa * GS + qb : qb * GS + pa;
                    const int i10 = qa < pb ? qa * GS + pb : pb * GS + qa;
                    const int i11 = qa < qb ? qa * GS + qb : qb * GS + qa;
                    T x00 = sm.G[i00];
                    T x01 = qbv ? sm.G[i01] : T(0);
                    T x10 = qav ? sm.G[i10] : T(0);
                    T x11 = (qav && qbv) ? sm.G[i11] : T(0);
                    rot2(RB.c, RB.s, x00, x01); rot2(RB.c, RB.s, x10, x11);     // columns (p_B, q_B)
                    rot2(RA.c, RA.s, x00, x10); rot2(RA.c, RA.s, x01, x11);     // rows (p_A, q_A)
                    sm.G[i00] = x00;
                    if (qbv) sm.G[i01] = x01;
                    if (qav) sm.G[i10] = x10;
                    if (qav && qbv) sm.G[i11] = x11;
                }
            }
        };
        if (tid < INNER_CRIT) {
            int ka = -1, kb = -1;
            if (tid < 32) {
                if (tid < P) ka = kb = tid;
            } else if (tid - 32 < P) {
                const int cb = sm.crit[r][tid - 32];
                if (cb >= 0) { ka = cb & 255; kb = cb >> 8; }
            }
            if (ka >= 0) g_block(ka, kb);
            // release the other G and E warps (barrier 2), then the rotation warp (barrier 1): the critical
            // blocks get the shared-memory pipe to themselves
            asm volatile("bar.arrive 2, %0;\n" ::"r"(pwarp0) : "memory");
            asm volatile("bar.sync 1, %0;\n" ::"r"(INNER_CRIT + 32) : "memory");
        } else if (tid >= pwarp0) {
            asm volatile("bar.sync 1, %0;\n" ::"r"(INNER_CRIT + 32) : "memory");
            if (lane < P) {
                const unsigned pq = sm.spq[rn][lane];
                const int x = pq & 255, y = pq >> 8;
                const T gxx = sm.G[x * GS + x];
                const T gyy = y < w ? sm.G[y * GS + y] : T(0);
                const T gxy = y < w ? sm.G[x * GS + y] : T(0);
                const int act = set_rotation<T, W>(sm, buf ^ 1, lane, y, w, gxx, gyy, gxy, tol_in);
                if (last) f_next |= act; else f_cur |= act;
            }
        } else {
          // G warps wait for the critical blocks; the E warps (which do not touch G) also arrive, and start at once
          if (tid < INNER_CRIT + NG) asm volatile("bar.sync 2, %0;\n" ::"r"(pwarp0) : "memory");
          else asm volatile("bar.arrive 2, %0;\n" ::"r"(pwarp0) : "memory");
          if (kA >= 0) {
            if (kA != kB && !((sm.cmask[r][myblk >> 5] >> (myblk & 31)) & 1u)) g_block(kA, kB);
          } else if (kE >= 0) {
            const Rot4<T> R4 = sm.rot[buf][kE];
            if (R4.act != T(0)) {
                const unsigned pq = sm.spq[r][kE];
                const int pa = pq & 255, qa = pq >> 8;
                if constexpr (InnerSmem<T, W>::ECOL) {
                    T* cp = sm.E + pa * ES;
                    T* cq = sm.E + qa * ES;
                    T ep[8], eq[8];
#pragma unroll
                    for (int j = 0; j < 8 / EV; ++j) {
                        const int row0 = (j * NCH + r0E) * EV;
                        *reinterpret_cast<float4*>(&ep[j * EV]) = *reinterpret_cast<const float4*>(cp + row0);
                        *reinterpret_cast<float4*>(&eq[j * EV]) = *reinterpret_cast<const float4*>(cq + row0);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) rot2(R4.c, R4.s, ep[u], eq[u]);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int row = ((u / EV) * NCH + r0E) * EV + (u % EV);
                        if (row == pa) { ep[u] += R4.cm1; eq[u] += R4.s; }
                        if (row == qa) { ep[u] -= R4.s; eq[u] += R4.cm1; }
                    }
#pragma unroll
                    for (int j = 0; j < 8 / EV; ++j) {
                        const int row0 = (j * NCH + r0E) * EV;
                        *reinterpret_cast<float4*>(cp + row0) = *reinterpret_cast<const float4*>(&ep[j * EV]);
                        *reinterpret_cast<float4*>(cq + row0) = *reinterpret_cast<const float4*>(&eq[j * EV]);
                    }
                } else {
                    T ep[8], eq[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        ep[u] = sm.E[(r0E + NCH * u) * ES + pa];
                        eq[u] = sm.E[(r0E + NCH * u) * ES + qa];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) rot2(R4.c, R4.s, ep[u], eq[u]);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int row = r0E + NCH * u;
                        if (row == pa) { ep[u] += R4.cm1; eq[u] += R4.s; }
                        if (row == qa) { ep[u] -= R4.s; eq[u] += R4.cm1; }
                        sm.E[row * ES + pa] = ep[u];
                        sm.E[row * ES + qa] = eq[u];
                    }
                }
            }
        }
        }
        if (dbg) {
            // per-warp end clocks of this round's work: [0] critical warps 0-1, [1] rotation warp,
            // [2] slowest other G warp, [3] slowest E warp (all from the round start)
            __syncwarp();
            if (lane == 0) sm.dbg_t[0][tid >> 5] = clock64();
            __syncthreads();
            if (tid == 0) {
                long long mc = 0, mr = 0, mg = 0, me = 0;
                const int nw = nt >> 5, gw0 = INNER_CRIT >> 5, gw1 = (INNER_CRIT + NG) >> 5;
                for (int q = 0; q < nw; ++q) {
                    const long long v = sm.dbg_t[0][q] - t_start;
                    if (q < gw0) mc = max(mc, v);
                    else if (q == nw - 1) mr = v;
                    else if (q < gw1) mg = max(mg, v);
                    else me = max(me, v);
                }
                dbg[0] += mc; dbg[1] += mr; dbg[2] += mg; dbg[3] += me; dbg[4] += 1;
            }
        }
        if (last) {
            const int any = __syncthreads_or(f_cur);
            f_cur = f_next;
            f_next = 0;
            if (!any || sweep + 1 >= max_inner) break;
            ++sweep;
            // A sweep without rotations leaves G unchanged, so its rounds would take exactly the
            // decisions of one parallel pass over all pairs now: if none exceeds the threshold,
            // that (check) sweep is counted and skipped.
            if (!__syncthreads_or(any_pair_above<T, W>(sm, w, tol_in))) break;
        } else {
            __syncthreads();
        }
        r = rn;
        buf ^= 1;
    }
    if (sweeps_used) *sweeps_used = sweep + 1;
    // mirror the upper triangle (callers read G as a full symmetric matrix)
    for (int e = tid; e < w * w; e += nt) {
        const int x = e / w, y = e - (e / w) * w;
        if (x > y) sm.G[x * GS + y] = sm.G[y * GS + x];
    }
    // total rotations: warp sums, then one shared atomic per warp
    const int wsum = __reduce_add_sync(0xffffffffu, (unsigned)my_cnt);
    if (lane == 0) atomicAdd(&sm.nrot[0], wsum);
    __syncthreads();
    const int total = sm.nrot[0];
    __syncthreads();
    return total;
}

// ------------------------------------------------------------------------
// k_pair_solve: one CTA per pair.
// ------------------------------------------------------------------------
__device__ long long* g_solve_dbg = nullptr;   // phase clocks of k_pair_solve, CTA 0 (MPJSVD_SOLVE_TIMING=1)

// ---- pieces of a pair solve (k_pair_solve) ------------------------------------------------------------
// exact skip: the pair's Gram equals the one of a sweep ago (same metric, no rotation); returns true if skipped
template <typename T>
__device__ __forceinline__ bool solve_skip_unchanged(const JacobiRound<T>& a, int pair) {
    if (!pair_unchanged(a, a.pd[pair])) return false;
    if (threadIdx.x == 0) {
        atomic_max_nonneg(a.sweep_off, a.pair_off[pair]);
        atomicAdd(a.sweep_skip, 1);
        a.flag[pair] = 0;
        if (a.dlist) {
            __threadfence();
            const int pos = atomicAdd(a.dctr, 1);
            st_release_gpu(a.dlist + pos, pair);
        }
    }
    return true;
}

// the pair's Gram: wait for its row-slab partials (gram_pdl), fixed-order reduction into G (full symmetric,
// row stride GS), pair metric max_{p<q} |g_pq| / (sqrt(g_pp) sqrt(g_qq)), flags / sweep statistics; returns
// whether the pair rotates.  dsq: w scratch values, red: 32.
template <typename T, int W, int NT>
__device__ __forceinline__ bool solve_prologue(const JacobiRound<T>& a, int pair, int w, T* G, int GS, T* dsq, T* red) {
    const int tid = threadIdx.x;
    if (a.gram_pdl) {
        // launched beside the Gram: wait until every row slab of this pair has been counted
        if (tid == 0) {
            unsigned long long t0 = 0;
            while (ld_acquire_gpu(a.gcnt + pair) < a.nsplit) {
                __nanosleep(64);
                const unsigned long long t = global_ns();
                if (t0 == 0) t0 = t;
                else if (t - t0 > MPJ_SPIN_TIMEOUT_NS) { atomicExch(a.dctr + 2, 1); break; }
            }
            a.gcnt[pair] = 0;      // next use: the next round's Gram, after this kernel
        }
        __syncthreads();
    }
    // fixed-order reduction over row slabs (deterministic)
    const T* part = a.partial + (long long)pair * a.nsplit * (W * W);
    {
        // each thread owns up to RE elements; the split loop is outermost so that the RE loads of one split
        // are in flight together (same summation order per element: split 0, 1, ...)
        constexpr int RE = (W * W + NT - 1) / NT;
        T acc[RE];
#pragma unroll
        for (int u = 0; u < RE; ++u) acc[u] = T(0);
        for (int sp = 0; sp < a.nsplit; ++sp) {
            const T* ps = part + (long long)sp * (W * W);
#pragma unroll
            for (int u = 0; u < RE; ++u) {
                const int e = tid + u * NT;
                if (e < W * W) acc[u] += __ldcg(ps + e);
            }
        }
#pragma unroll
        for (int u = 0; u < RE; ++u) {
            const int e = tid + u * NT;
            const int p = e / W, q = e - (e / W) * W;
            if (e < W * W && p < w && q < w && p >= q) {      // partials hold (at least) the lower triangle
                G[p * GS + q] = acc[u];
                G[q * GS + p] = acc[u];
            }
        }
    }
    __syncthreads();
    for (int p = tid; p < w; p += NT) dsq[p] = sqrt(G[p * GS + p]);
    __syncthreads();
    T off = T(0);
    for (int e = tid; e < w * w; e += NT) {
        const int p = e / w, q = e - (e / w) * w;
        if (p < q) {
            T gpp = G[p * GS + p], gqq = G[q * GS + q];
            if (gpp > T(0) && gqq > T(0)) {
                T v = fabs(G[p * GS + q]) / (dsq[p] * dsq[q]);
                off = v > off ? v : off;
            }
        }
    }
    off = block_max(off, red);
    const bool rotate = off > a.tol;
    if (tid == 0) {
        atomic_max_nonneg(a.sweep_off, (double)off);
        if (rotate) atomicAdd(a.sweep_upd, 1);
        a.flag[pair] = rotate ? 1 : 0;
        if (a.skip) {
            a.pair_off[pair] = (double)off;
            if (rotate) {
                a.last_mod[a.pd[pair].b0] = a.gidx;
                a.last_mod[a.pd[pair].b1] = a.gidx;
            }
        }
    }
    return rotate;
}

// inner-solve statistics and publication of the solved pair (E and flag complete)
template <typename T>
__device__ __forceinline__ void solve_epilogue(const JacobiRound<T>& a, int pair, bool rotate, int used) {
    if (rotate && threadIdx.x == 0) {
        atomicMax(a.sweep_inner, used);
        atomicAdd(a.sweep_inner + 1, used);
    }
    if (a.dlist) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const int pos = atomicAdd(a.dctr, 1);
            st_release_gpu(a.dlist + pos, pair);
        }
    }
}

template <typename T, int W>
__global__ void __launch_bounds__(inner_nt<W>()) k_pair_solve(JacobiRound<T> a) {
    long long* sdbg = (blockIdx.x == 0 && threadIdx.x == 0) ? g_solve_dbg : nullptr;
    const long long c0 = sdbg ? clock64() : 0;
    constexpr int GS = InnerSmem<T, W>::GS;
    extern __shared__ __align__(16) unsigned char smraw[];
    InnerSmem<T, W>& sm = *reinterpret_cast<InnerSmem<T, W>*>(smraw);
    const int pair = blockIdx.x, tid = threadIdx.x;
    if (a.pdl) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");   // the update may start
    const int w = a.pd[pair].w0 + a.pd[pair].w1;
    if (solve_skip_unchanged(a, pair)) return;
    const bool rotate = solve_prologue<T, W, inner_nt<W>()>(a, pair, w, sm.G, GS, sm.E, sm.red);   // E: scratch
    const long long c1 = sdbg ? clock64() : 0;
    int used = 0;
    if (rotate) {
        inner_solve_dev<T, W>(sm, w, a.tol_in, a.max_inner, &used);
        if (sdbg) { sdbg[1] += clock64() - c1; sdbg[3] += 1; }
        T* E = a.E + (long long)pair * (W * W);
        for (int e = tid; e < W * W; e += blockDim.x) {
            const int k = e / W, j = e - (e / W) * W;
            E[e] = (k < w && j < w) ? sm.E[InnerSmem<T, W>::eidx(k, j)] : T(0);   // E[k][j] row-major
        }
    }
    if (sdbg) { sdbg[0] += c1 - c0; sdbg[2] += clock64() - c0; sdbg[4] += 1; }
    solve_epilogue(a, pair, rotate, used);
}

// ------------------------------------------------------------------------
// k_pair_update: grid (row chunks of 64, npairs, 2 [X, V]); 64 threads.
// out = W + W E on a 64-row slab; thread tile 8 rows x (W/8) columns.
// ------------------------------------------------------------------------
template <typename T, int W>
__global__ void __launch_bounds__(64) k_pair_update(JacobiRound<T> a) {
    constexpr int RC = 64;
    constexpr int VEC = 16 / sizeof(T);
    constexpr int SW = RC + VEC;           // Ws[k][rho] stride
    constexpr int SE = W + VEC;            // Es[k][j] stride
    constexpr int TP = W / 8;
    extern __shared__ __align__(16) unsigned char upd_smem[];
    T* Ws = reinterpret_cast<T*>(upd_smem);              // W * SW
    T* Es = Ws + W * SW;                                   // W * SE
    T** colp = reinterpret_cast<T**>(Es + W * SE);
    const int pair = blockIdx.y, which = blockIdx.z;
    if (!a.flag[pair]) return;
    if (which && !a.has_v) return;
    const long long ld = which ? a.ldv : a.ldx;
    const long long rows_pad = which ? a.nv_pad : a.m_pad;
    const long long row0 = (long long)blockIdx.x * RC;
    if (row0 >= rows_pad) return;
    const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
    const PairDesc<T> pd = a.pd[pair];
    const int w = pd.w0 + pd.w1;
    if (tid < W) colp[tid] = tid < w ? pair_col(pd, tid, which != 0, ld) : nullptr;
    const T* Eg = a.E + (long long)pair * (W * W);
    for (int e = tid; e < W * W; e += 64) {
        const int k = e / W, j = e - (e / W) * W;
        Es[k * SE + j] = Eg[e];
    }
    __syncthreads();
    const long long nrow = min((long long)RC, rows_pad - row0);   // multiple of 32
    constexpr int VPC = RC / VEC;
    for (int v = tid; v < W * VPC; v += 64) {
        const int k = v / VPC, ch = v % VPC;
        T* dst = &Ws[k * SW + ch * VEC];
        if (colp[k] != nullptr && ch * VEC < nrow)
            *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(colp[k] + row0 + ch * VEC);
        else
            *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    T acc[8][TP];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TP; ++j) acc[i][j] = T(0);
    for (int k = 0; k < w; ++k) {
        T av[8], bv[TP];
#pragma unroll
        for (int i = 0; i < 8; i += VEC)
            *reinterpret_cast<float4*>(&av[i]) = *reinterpret_cast<const float4*>(&Ws[k * SW + ty * 8 + i]);
#pragma unroll
        for (int j = 0; j < TP; j += (VEC < TP ? VEC : TP)) {
            if constexpr (TP >= VEC) {
                *reinterpret_cast<float4*>(&bv[j]) = *reinterpret_cast<const float4*>(&Es[k * SE + tx * TP + j]);
            } else {
#pragma unroll
                for (int jj = 0; jj < TP; ++jj) bv[jj] = Es[k * SE + tx * TP + jj];
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < TP; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int j = 0; j < TP; ++j) {
        const int col = tx * TP + j;
        if (col >= w) continue;
        T* dstc = colp[col] + row0 + ty * 8;
        if (ty * 8 >= nrow) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) dstc[i] = Ws[col * SW + ty * 8 + i] + acc[i][j];
    }
}



// ========================================================================
// FP64 tensor-pipe (DMMA) versions: mma.sync.aligned.m8n8k4.row.col.f64.
// B200 has no tcgen05 kind::f64; DMMA runs on the FP64 pipe (measured 36.9
// TFLOP/s, profiles/peaks.json).  Fragment layout (PTX ISA, m8n8k4 f64):
//   A (8x4, row): lane l holds A[l>>2][l&3];  B (4x8, col): B[l&3][l>>2];
//   C/D (8x8): lane l holds D[l>>2][2(l&3)], D[l>>2][2(l&3)+1].
// ========================================================================
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// lower-triangle tile t -> (i, j), i >= j, row-major over the lower triangle
__host__ __device__ constexpr int tri_i(int t) {
    int ii = 0;
    while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
    return ii;
}
__host__ __device__ constexpr int tri_j(int t) { return t - tri_i(t) * (tri_i(t) + 1) / 2; }

constexpr int GRAM_KT = 32, GRAM_S = GRAM_KT + 4, GRAM_STAGES = 3, GRAM_NWARP = 4;

// The k-loop of one warp with a compile-time tile list (tiles WARP, WARP+4, ...)
template <int W, int WARP>
__device__ __forceinline__ void gram_warp(const double* const* colp, double* Wsm,
                                          long long rbeg, int ntile, double* out) {
    constexpr int KT = GRAM_KT, S = GRAM_S, STAGES = GRAM_STAGES, NTI = W / 8;
    constexpr int NTILE = NTI * (NTI + 1) / 2;
    constexpr int TPW = (NTILE - WARP + GRAM_NWARP - 1) / GRAM_NWARP;
    const int tid = threadIdx.x, lane = tid & 31;
    double acc[TPW > 0 ? TPW : 1][2];
#pragma unroll
    for (int u = 0; u < TPW; ++u) acc[u][0] = acc[u][1] = 0.0;
    constexpr int CH = KT / 2;
    auto load_tile = [&](int t, int stage) {
        const long long r0 = rbeg + (long long)t * KT;
        double* ws = Wsm + stage * (W * S);
        for (int v = tid; v < W * CH; v += 128) {
            const int c = v / CH, ch = v % CH;
            double* dst = &ws[c * S + ch * 2];
            const double* cp = colp[c];
            if (cp != nullptr) cp_async16(dst, cp + r0 + ch * 2);
            else *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
        }
    };
#pragma unroll
    for (int s0 = 0; s0 < STAGES - 1; ++s0) {
        if (s0 < ntile) load_tile(s0, s0);
        cp_async_commit();
    }
    for (int t = 0; t < ntile; ++t) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        if (t + STAGES - 1 < ntile) load_tile(t + STAGES - 1, (t + STAGES - 1) % STAGES);
        cp_async_commit();
        const double* ws = Wsm + (t % STAGES) * (W * S);
#pragma unroll
        for (int k0 = 0; k0 < KT; k0 += 4) {
            double f[NTI];
#pragma unroll
            for (int i = 0; i < NTI; ++i) f[i] = ws[(8 * i + (lane >> 2)) * S + k0 + (lane & 3)];
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                constexpr int dummy = 0;
                (void)dummy;
                const int tt = WARP + GRAM_NWARP * u;
                dmma884(acc[u][0], acc[u][1], f[tri_i(tt)], f[tri_j(tt)]);
            }
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
        const int tt = WARP + GRAM_NWARP * u;
        const int row = 8 * tri_i(tt) + (lane >> 2), col = 8 * tri_j(tt) + 2 * (lane & 3);
        *reinterpret_cast<double2*>(&out[row * W + col]) = make_double2(acc[u][0], acc[u][1]);
    }
}

// ------------------------------------------------------------------------
// k_pair_gram_dmma: grid (nsplit, npairs), 128 threads (4 warps).  The CTA
// streams its row slab of W = [X_I X_J] through a 3-stage cp.async pipeline
// (k-tile 32 rows, column-major staging, column stride 36 doubles: the
// 16-lane phases of an m8n8k4 fragment load hit 16 distinct 8-byte banks).
// Per 4-row k-step every warp loads the W/8 fragments (they serve as both A
// and B: G = W^T W) and issues one DMMA per lower-triangle tile it owns
// (tiles warp, warp+4, ...: 9 of the 36 at W = 64).  Writes the lower
// triangle of the partial Gram.
// ------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(128) k_pair_gram_dmma(JacobiRound<double> a) {
    reset_publication(a);
    gram_pdl_begin(a);
    if (pair_unchanged(a, a.pd[blockIdx.y])) return;
    extern __shared__ __align__(16) unsigned char gram_smem[];
    double* Wsm = reinterpret_cast<double*>(gram_smem);
    const double** colp = reinterpret_cast<const double**>(Wsm + GRAM_STAGES * W * GRAM_S);
    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5;
    const PairDesc<double> pd = a.pd[pair];
    const int w = pd.w0 + pd.w1;
    if (tid < W) colp[tid] = tid < w ? pair_col(pd, tid, false, a.ldx) : nullptr;
    __syncthreads();
    const long long rbeg = (long long)split * a.rows_per_split;
    const long long rend = min(rbeg + (long long)a.rows_per_split, (long long)a.m_pad);
    const int ntile = (int)((rend - rbeg) / GRAM_KT);
    double* out = a.partial + ((long long)pair * a.nsplit + split) * (W * W);
    switch (warp) {
        case 0: gram_warp<W, 0>(colp, Wsm, rbeg, ntile, out); break;
        case 1: gram_warp<W, 1>(colp, Wsm, rbeg, ntile, out); break;
        case 2: gram_warp<W, 2>(colp, Wsm, rbeg, ntile, out); break;
        default: gram_warp<W, 3>(colp, Wsm, rbeg, ntile, out); break;
    }
    gram_pdl_end(a, pair);
}
static size_t gram_dmma_smem(int W) { return sizeof(double) * (size_t)GRAM_STAGES * W * GRAM_S + sizeof(long long) * W; }

// ------------------------------------------------------------------------
// k_pair_gram_f32t: fp32 Gram (W = 64) on the FFMA pipe, symmetric at 16 x 16
// block granularity.  The lower triangle of the 4 x 4 grid of 16 x 16 blocks
// (6 off-diagonal + 4 diagonal blocks) is cut into 40 uniform 8 x 8 tiles
// (90 % of the products are needed, no lane divergence: every thread runs the
// same 8 x 8 outer product on its own columns).  Grid (nsplit, npairs), 160
// threads = 4 row groups x 40 tiles; the CTA's row slab streams through a
// 3-stage cp.async pipeline of 32-row k-tiles and row group g takes the
// 4-row chunks 2g, 2g+1 of every k-tile (float4 fragments).  The row groups'
// partial tiles are summed in shared memory; the lower triangle is written.
// Shared layout: 16-byte chunk (column c, rows 4rc..4rc+3) at chunk index
// 8c + (rc ^ (c >> 3)): the column groups of one LDS.128 hit distinct banks.
// ------------------------------------------------------------------------
constexpr int G32_KT = 32, G32_ST = 6, G32_NT = 160;

__device__ __forceinline__ int g32_chunk(int c, int rc) { return 8 * c + (rc ^ ((c >> 3) & 7)); }

__global__ void __launch_bounds__(G32_NT, 3) k_pair_gram_f32t(JacobiRound<float> a) {
    reset_publication(a);
    if (pair_unchanged(a, a.pd[blockIdx.y])) return;
    constexpr int W = 64;
    extern __shared__ __align__(16) unsigned char g32_smem[];
    float4* Ws = reinterpret_cast<float4*>(g32_smem);            // [ST][W*8] chunks
    float* red = reinterpret_cast<float*>(g32_smem);               // [W*W] partial sums (aliases the stages)
    __shared__ const float* colp[W];
    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x;
    const PairDesc<float> pd = a.pd[pair];
    const int w = pd.w0 + pd.w1;
    if (tid < W) colp[tid] = tid < w ? pair_col(pd, tid, false, a.ldx) : nullptr;
    __syncthreads();
    const long long rbeg = (long long)split * a.rows_per_split;
    const long long rend = min(rbeg + (long long)a.rows_per_split, (long long)a.m_pad);
    const int ntile = (int)((rend - rbeg) / G32_KT);
    // tile of this thread: 16x16 block (BI >= BJ), 8x8 sub-tile (sa, sb)
    const int tile = tid % 40, rg = tid / 40;
    int BI, BJ, sa, sb;
    if (tile < 24) {                                   // off-diagonal blocks (1,0),(2,0),(2,1),(3,0),(3,1),(3,2)
        const int blk = tile >> 2;
        BI = blk < 1 ? 1 : (blk < 3 ? 2 : 3);
        BJ = blk - (BI * (BI - 1)) / 2;
        sa = (tile >> 1) & 1; sb = tile & 1;
    } else {                                           // diagonal blocks, full squares
        const int t2 = tile - 24;
        BI = BJ = t2 >> 2;
        sa = (t2 >> 1) & 1; sb = t2 & 1;
    }
    const int ca = 16 * BI + 8 * sa, cb = 16 * BJ + 8 * sb;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    auto load_tile = [&](int t, int st) {
        const long long r0 = rbeg + (long long)t * G32_KT;
        float4* dst = Ws + st * W * 8;
        for (int v = tid; v < W * 8; v += G32_NT) {
            const int c = v >> 3, rc = v & 7;
            float4* d = dst + g32_chunk(c, rc);
            if (colp[c] != nullptr) cp_async16(d, colp[c] + r0 + rc * 4);
            else *d = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
#pragma unroll
    for (int s0 = 0; s0 < G32_ST - 1; ++s0) {
        if (s0 < ntile) load_tile(s0, s0);
        cp_async_commit();
    }
    for (int t = 0; t < ntile; ++t) {
        cp_async_wait<G32_ST - 2>();
        __syncthreads();
        if (t + G32_ST - 1 < ntile) load_tile(t + G32_ST - 1, (t + G32_ST - 1) % G32_ST);
        cp_async_commit();
        const float4* ws = Ws + (t % G32_ST) * W * 8;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rc = 2 * rg + h;
            const float4* wa = ws + 8 * ca + (rc ^ (ca >> 3));
            const float4* wb = ws + 8 * cb + (rc ^ (cb >> 3));
            float4 fa[8], fb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                fa[u] = wa[8 * u];
                fb[u] = wb[8 * u];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    acc[i][j] = fmaf(fa[i].x, fb[j].x, acc[i][j]);
                    acc[i][j] = fmaf(fa[i].y, fb[j].y, acc[i][j]);
                    acc[i][j] = fmaf(fa[i].z, fb[j].z, acc[i][j]);
                    acc[i][j] = fmaf(fa[i].w, fb[j].w, acc[i][j]);
                }
        }
    }
    cp_async_wait<0>();
    __syncthreads();                                   // staging buffers become the reduction buffer
    // ---- sum the four row groups' partial tiles (fixed order) and write the lower triangle
    for (int g = 0; g < 4; ++g) {
        __syncthreads();
        if (rg == g) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float* d = &red[(ca + i) * W + cb + j];
                    *d = g == 0 ? acc[i][j] : *d + acc[i][j];
                }
        }
    }
    __syncthreads();
    float* out = a.partial + ((long long)pair * a.nsplit + split) * (W * W);
    for (int e = tid; e < W * W; e += G32_NT) {
        const int p = e / W, q = e % W;
        if (p >= q) out[e] = red[e];
    }
}

// ------------------------------------------------------------------------
// k_pair_update_dmma: grid (tile groups, npairs, 2 [X, V]), 512 threads (16
// warps); out = W + W E on UD_RC-row tiles, UD_TPC tiles per CTA.  E^T is
// staged once per CTA (column stride W+4: conflict-free fragment loads); the
// tiles are double-buffered (cp.async of tile t+1 overlaps the DMMAs of tile
// t; column stride 132).  Each warp owns (128/8) x (W/2) of the output and
// runs K = w/4 DMMA k-steps; the result is added in place into the staged
// tile and stored back with coalesced 16-byte stores.
// ------------------------------------------------------------------------
#ifndef MPJ_UD_RC
#define MPJ_UD_RC 64
#endif
#ifndef MPJ_UD_MINB
#define MPJ_UD_MINB 2
#endif
constexpr int UD_NT = 256, UD_RC = MPJ_UD_RC, UD_TPC = 1024 / MPJ_UD_RC;   // 2 CTAs per SM (smem ~104 KB each)
constexpr int UD_MINB = MPJ_UD_MINB;
template <int W> constexpr int ud_rc() { return W >= 64 ? UD_RC : 64; }   // 8 rows per row-group warp at least
template <int W> constexpr int ud_tpc() { return 1024 / ud_rc<W>(); }
template <int W>
constexpr size_t update_dmma_smem() {
    return sizeof(double) * ((size_t)2 * W * (ud_rc<W>() + 4) + (size_t)W * (W + 4)) + sizeof(double*) * W;
}

template <int W>
__global__ void __launch_bounds__(UD_NT, UD_MINB) k_pair_update_dmma(JacobiRound<double> a) {
    constexpr int RC = ud_rc<W>(), SW = RC + 4, SE = W + 4, UD_TPC = ud_tpc<W>();
    constexpr int WC = W >= 64 ? 2 : 1, WR = (UD_NT / 32) / WC;
    constexpr int TM = RC / WR / 8, TN = W / WC / 8;
    extern __shared__ __align__(16) unsigned char upd_smem[];
    double* Wbuf = reinterpret_cast<double*>(upd_smem);     // [2][W][SW]  (column k, row rho)
    double* Et = Wbuf + 2 * W * SW;                          // [W][SE]     (Et[j][k] = E[k][j])
    double** colp = reinterpret_cast<double**>(Et + W * SE);
    const int pair = blockIdx.y, which = blockIdx.z;
    if (!a.flag[pair]) return;
    if (which && !a.has_v) return;
    const long long ld = which ? a.ldv : a.ldx;
    const long long rows_pad = which ? a.nv_pad : a.m_pad;
    const long long row_lo = (long long)blockIdx.x * UD_TPC * RC;
    if (row_lo >= rows_pad) return;
    const long long row_hi = min(rows_pad, row_lo + (long long)UD_TPC * RC);
    const int ntile = (int)((row_hi - row_lo + RC - 1) / RC);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const auto pd = a.pd[pair];
    const int w = pd.w0 + pd.w1;
    if (tid < W) colp[tid] = tid < w ? pair_col(pd, tid, which != 0, ld) : nullptr;
    __syncthreads();
    auto issue = [&](int t) {
        double* Ws = Wbuf + (t & 1) * (W * SW);
        const long long row0 = row_lo + (long long)t * RC;
        const int nrow = (int)min((long long)RC, rows_pad - row0);    // multiple of 32
        for (int v = tid; v < W * (RC / 2); v += UD_NT) {
            const int c = v / (RC / 2), ch = v % (RC / 2);
            double* dst = &Ws[c * SW + ch * 2];
            if (colp[c] != nullptr && ch * 2 < nrow) cp_async16(dst, colp[c] + row0 + ch * 2);
            else *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
        }
        cp_async_commit();
    };
    issue(0);
    const double* Eg = a.E + (long long)pair * (W * W);
    for (int e = tid; e < W * W; e += UD_NT) {
        const int k = e / W, j = e - (e / W) * W;
        Et[j * SE + k] = Eg[e];
    }
    const int wr = warp / WC, wc = warp % WC;
    const int rb = wr * (RC / WR), cb = wc * (W / WC);
    const int kend = (w + 3) & ~3;
    for (int t = 0; t < ntile; ++t) {
        if (t + 1 < ntile) { issue(t + 1); cp_async_wait<1>(); }
        else cp_async_wait<0>();
        __syncthreads();                                      // tile t (and E) visible
        double* Ws = Wbuf + (t & 1) * (W * SW);
        double acc[TM][TN][2];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int k0 = 0; k0 < kend; k0 += 4) {
            double fa[TM], fb[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) fa[i] = Ws[(k0 + (lane & 3)) * SW + rb + 8 * i + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < TN; ++j) fb[j] = Et[(cb + 8 * j + (lane >> 2)) * SE + k0 + (lane & 3)];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma884(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
        }
        __syncthreads();                                      // all fragment reads done before the in-place add
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int rho = rb + 8 * i + (lane >> 2);
                const int col = cb + 8 * j + 2 * (lane & 3);
                Ws[col * SW + rho] += acc[i][j][0];
                Ws[(col + 1) * SW + rho] += acc[i][j][1];
            }
        __syncthreads();
        const long long row0 = row_lo + (long long)t * RC;
        const int nrow = (int)min((long long)RC, rows_pad - row0);
        for (int v = tid; v < W * (RC / 2); v += UD_NT) {
            const int c = v / (RC / 2), ch = v % (RC / 2);
            if (c < w && ch * 2 < nrow)
                *reinterpret_cast<double2*>(colp[c] + row0 + ch * 2) =
                    *reinterpret_cast<const double2*>(&Ws[c * SW + ch * 2]);
        }
        __syncthreads();                                      // buffer t & 1 free for tile t + 2
    }
}

// ------------------------------------------------------------------------
// k_pair_update_dmma_pdl: k_pair_update_dmma as a persistent kernel (one CTA
// per SM) launched as a programmatic dependent of the round's solve: work
// items (completion position p, X or V, group of UD_TPC tiles) come from a
// global counter in completion order, item p waits (acquire) for the p-th
// published pair (k_pair_solve) and skips pairs that did not rotate.
// ------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(UD_NT, UD_MINB) k_pair_update_dmma_pdl(JacobiRound<double> a, int ngroups) {
    constexpr int RC = ud_rc<W>(), SW = RC + 4, SE = W + 4, UD_TPC = ud_tpc<W>();
    constexpr int WC = W >= 64 ? 2 : 1, WR = (UD_NT / 32) / WC;
    constexpr int TM = RC / WR / 8, TN = W / WC / 8;
    extern __shared__ __align__(16) unsigned char upd_smem[];
    double* Wbuf = reinterpret_cast<double*>(upd_smem);
    double* Et = Wbuf + 2 * W * SW;
    double** colp = reinterpret_cast<double**>(Et + W * SE);
    __shared__ int item[3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = warp / WC, wc = warp % WC;
    const int rb = wr * (RC / WR), cb = wc * (W / WC);
    const long long total = (long long)a.npairs * 2 * ngroups;
    while (true) {
        if (tid == 0) {
            int pair = -1, which = 0, grp = 0;
            while (true) {
                const long long wk = atomicAdd(a.dctr + 1, 1);
                if (wk >= total) break;
                const int p = (int)(wk / (2 * ngroups)), rem = (int)(wk % (2 * ngroups));
                which = rem / ngroups;
                grp = rem % ngroups;
                int pr = ld_acquire_gpu(a.dlist + p);
                unsigned long long t0 = 0;
                while (pr < 0) {
                    __nanosleep(256);
                    pr = ld_acquire_gpu(a.dlist + p);
                    if (pr >= 0) break;
                    const unsigned long long t = global_ns();
                    if (t0 == 0) t0 = t;
                    else if (t - t0 > MPJ_SPIN_TIMEOUT_NS) { atomicExch(a.dctr + 2, 1); break; }
                }
                if (pr < 0) { pair = -1; break; }
                if (!a.flag[pr] || (which && !a.has_v)) continue;
                const long long rows_pad = which ? a.nv_pad : a.m_pad;
                if ((long long)grp * UD_TPC * RC >= rows_pad) continue;
                pair = pr;
                break;
            }
            item[0] = pair; item[1] = which; item[2] = grp;
        }
        __syncthreads();
        const int pair = item[0], which = item[1], grp = item[2];
        if (pair < 0) break;
        const long long ld = which ? a.ldv : a.ldx;
        const long long rows_pad = which ? a.nv_pad : a.m_pad;
        const long long row_lo = (long long)grp * UD_TPC * RC;
        const long long row_hi = min(rows_pad, row_lo + (long long)UD_TPC * RC);
        const int ntile = (int)((row_hi - row_lo + RC - 1) / RC);
        const auto pd = a.pd[pair];
        const int w = pd.w0 + pd.w1;
        if (tid < W) colp[tid] = tid < w ? pair_col(pd, tid, which != 0, ld) : nullptr;
        __syncthreads();
        auto issue = [&](int t) {
            double* Ws = Wbuf + (t & 1) * (W * SW);
            const long long row0 = row_lo + (long long)t * RC;
            const int nrow = (int)min((long long)RC, rows_pad - row0);
            for (int v = tid; v < W * (RC / 2); v += UD_NT) {
                const int c = v / (RC / 2), ch = v % (RC / 2);
                double* dst = &Ws[c * SW + ch * 2];
                if (colp[c] != nullptr && ch * 2 < nrow) cp_async16(dst, colp[c] + row0 + ch * 2);
                else *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
            }
            cp_async_commit();
        };
        issue(0);
        const double* Eg = a.E + (long long)pair * (W * W);
        for (int e = tid; e < W * W; e += UD_NT) {
            const int k = e / W, j = e - (e / W) * W;
            Et[j * SE + k] = Eg[e];
        }
        const int kend = (w + 3) & ~3;
        for (int t = 0; t < ntile; ++t) {
            if (t + 1 < ntile) { issue(t + 1); cp_async_wait<1>(); }
            else cp_async_wait<0>();
            __syncthreads();
            double* Ws = Wbuf + (t & 1) * (W * SW);
            double acc[TM][TN][2];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            for (int k0 = 0; k0 < kend; k0 += 4) {
                double fa[TM], fb[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) fa[i] = Ws[(k0 + (lane & 3)) * SW + rb + 8 * i + (lane >> 2)];
#pragma unroll
                for (int j = 0; j < TN; ++j) fb[j] = Et[(cb + 8 * j + (lane >> 2)) * SE + k0 + (lane & 3)];
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) dmma884(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                    const int rho = rb + 8 * i + (lane >> 2);
                    const int col = cb + 8 * j + 2 * (lane & 3);
                    Ws[col * SW + rho] += acc[i][j][0];
                    Ws[(col + 1) * SW + rho] += acc[i][j][1];
                }
            __syncthreads();
            const long long row0 = row_lo + (long long)t * RC;
            const int nrow = (int)min((long long)RC, rows_pad - row0);
            for (int v = tid; v < W * (RC / 2); v += UD_NT) {
                const int c = v / (RC / 2), ch = v % (RC / 2);
                if (c < w && ch * 2 < nrow)
                    *reinterpret_cast<double2*>(colp[c] + row0 + ch * 2) =
                        *reinterpret_cast<const double2*>(&Ws[c * SW + ch * 2]);
            }
            __syncthreads();
        }
    }
}

template <int W>
static int launch_update_dmma_pdl(const JacobiRound<double>& a, cudaStream_t st) {
    const size_t dsm = update_dmma_smem<W>();
    MPJ_CUDA_TRY(set_smem(k_pair_update_dmma_pdl<W>, (size_t)(dsm)));
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long rows_pad = a.m_pad > a.nv_pad ? a.m_pad : a.nv_pad;
    const int ngroups = (int)((rows_pad + 1023) / 1024);
    const long long items = (long long)a.npairs * 2 * ngroups;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(items < UD_MINB * nsm ? items : UD_MINB * nsm));   // UD_MINB CTAs per SM
    cfg.blockDim = dim3(UD_NT);
    cfg.dynamicSmemBytes = dsm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_pair_update_dmma_pdl<W>, a, ngroups);
    MPJ_LAUNCHED();
    if (e != cudaSuccess) {
        mpj_record_cuda_error(e, "cudaLaunchKernelEx(update dmma pdl)", __FILE__, __LINE__);
        return -4;
    }
    return 0;
}

// ------------------------------------------------------------------------
// k_pair_update_f32: fp32 SIMT version of the update (FFMA pipe).  Grid
// (row chunks of 128, npairs, 2), 256 threads; thread tile 8 rows x (W/16)
// columns of out = W + W E; slab and E staged in shared memory (16-byte
// vector reads: 3 LDS.128 per 32 FFMA at W = 64), result added in place in
// the staged slab and stored with coalesced 16-byte stores.
// ------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(256) k_pair_update_f32(JacobiRound<float> a) {
    constexpr int RC = 128, SW = RC + 4, SE = W + 4, TN = W / 16;
    extern __shared__ __align__(16) unsigned char upd_smem[];
    float* Ws = reinterpret_cast<float*>(upd_smem);     // [W][SW]  (column k, row rho)
    float* Es = Ws + W * SW;                            // [W][SE]  (Es[k][j] = E[k][j])
    float** colp = reinterpret_cast<float**>(Es + W * SE);
    const int pair = blockIdx.y, which = blockIdx.z;
    if (!a.flag[pair]) return;
    if (which && !a.has_v) return;
    const long long ld = which ? a.ldv : a.ldx;
    const long long rows_pad = which ? a.nv_pad : a.m_pad;
    const long long row0 = (long long)blockIdx.x * RC;
    if (row0 >= rows_pad) return;
    const int nrow = (int)min((long long)RC, rows_pad - row0);
    const int tid = threadIdx.x;
    const auto pd = a.pd[pair];
    const int w = pd.w0 + pd.w1;
    if (tid < W) colp[tid] = tid < w ? pair_col(pd, tid, which != 0, ld) : nullptr;
    __syncthreads();
    for (int v = tid; v < W * (RC / 4); v += 256) {
        const int c = v / (RC / 4), ch = v % (RC / 4);
        float* dst = &Ws[c * SW + ch * 4];
        if (colp[c] != nullptr && ch * 4 < nrow) cp_async16(dst, colp[c] + row0 + ch * 4);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    cp_async_commit();
    const float* Eg = a.E + (long long)pair * (W * W);
    for (int e = tid * 4; e < W * W; e += 256 * 4) {
        const int k = e / W, j = e - (e / W) * W;
        *reinterpret_cast<float4*>(&Es[k * SE + j]) = *reinterpret_cast<const float4*>(&Eg[e]);
    }
    cp_async_wait<0>();
    __syncthreads();
    const int cg = tid & 15, rg = tid >> 4;          // 16 column groups x 16 row groups
    const int rb = rg * 8, cb = cg * TN;
    float acc[8][TN];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
    for (int k = 0; k < w; ++k) {
        float av[8], bv[TN];
        *reinterpret_cast<float4*>(&av[0]) = *reinterpret_cast<const float4*>(&Ws[k * SW + rb]);
        *reinterpret_cast<float4*>(&av[4]) = *reinterpret_cast<const float4*>(&Ws[k * SW + rb + 4]);
        if constexpr (TN == 4) {
            *reinterpret_cast<float4*>(&bv[0]) = *reinterpret_cast<const float4*>(&Es[k * SE + cb]);
        } else {
#pragma unroll
            for (int j = 0; j < TN; ++j) bv[j] = Es[k * SE + cb + j];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) Ws[(cb + j) * SW + rb + i] += acc[i][j];
    __syncthreads();
    for (int v = tid; v < W * (RC / 4); v += 256) {
        const int c = v / (RC / 4), ch = v % (RC / 4);
        if (c < w && ch * 4 < nrow)
            *reinterpret_cast<float4*>(colp[c] + row0 + ch * 4) =
                *reinterpret_cast<const float4*>(&Ws[c * SW + ch * 4]);
    }
}

// ------------------------------------------------------------------------
// k_inner_solve_batch: test entry (mpjsvd_inner_solve): count matrices.
// ------------------------------------------------------------------------
__device__ long long* g_inner_dbg_f = nullptr;   // phase timers of the batch kernel (MPJSVD_INNER_TIMING=1)
__device__ long long* g_inner_dbg_d = nullptr;

template <typename T, int W>
__global__ void __launch_bounds__(inner_nt<W>()) k_inner_solve_batch(T* G, T* E, int w, T tol_in, int max_inner, int* rot) {
    constexpr int GS = InnerSmem<T, W>::GS;
    extern __shared__ __align__(16) unsigned char smraw[];
    InnerSmem<T, W>& sm = *reinterpret_cast<InnerSmem<T, W>*>(smraw);
    T* g = G + (long long)blockIdx.x * w * w;
    T* e = E + (long long)blockIdx.x * w * w;
    for (int i = threadIdx.x; i < w * w; i += blockDim.x) sm.G[(i % w) * GS + i / w] = g[i];
    __syncthreads();
    long long* dbgp = sizeof(T) == 4 ? g_inner_dbg_f : g_inner_dbg_d;
    int nr = inner_solve_dev<T, W>(sm, w, tol_in, max_inner, nullptr, blockIdx.x == 0 ? dbgp : nullptr);
    for (int i = threadIdx.x; i < w * w; i += blockDim.x) {
        g[i] = sm.G[(i % w) * GS + i / w];
        e[i] = sm.E[InnerSmem<T, W>::eidx(i % w, i / w)];   // column-major out: e[row + col*w] = E[row][col]
    }
    if (threadIdx.x == 0) rot[blockIdx.x] = nr;
}

// ------------------------------------------------------------------------
// host launchers
// ------------------------------------------------------------------------
template <typename T> struct KName;
template <> struct KName<float> {
    static constexpr const char* gram = "pair_gram_f32";
    static constexpr const char* solve = "pair_solve_f32";
    static constexpr const char* update = "pair_update_f32";
};
template <> struct KName<double> {
    static constexpr const char* gram = "pair_gram_f64";
    static constexpr const char* solve = "pair_solve_f64";
    static constexpr const char* update = "pair_update_f64";
};

template <typename T, int W>
static int launch_round_w(const JacobiRound<T>& a0, cudaStream_t st, const ProfHook* hook) {
    // Gram -> solve overlap only behind the Gram kernels that count their partials (gram_pdl_end)
    JacobiRound<T> a = a0;
    a.gram_pdl = a0.gram_pdl && (sizeof(T) == 8 || (W == 64 && a0.use_tc && a0.smap && a0.gram_variant >= 10 &&
                                                     a0.gram_variant <= 26)) ? 1 : 0;
    if (hook) hook->begin(hook->ctx, KName<T>::gram);
    if constexpr (sizeof(T) == 8) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_dmma<W>, (size_t)(gram_dmma_smem(W))));
        k_pair_gram_dmma<W><<<dim3(a.nsplit, a.npairs), 128, gram_dmma_smem(W), st>>>(a);
    } else if constexpr (W == 64) {
        if (a.use_tc) {
            launch_gram_tc(a, st);
            if (hook) hook->end(hook->ctx, KName<T>::gram);
            goto solve;
        }
        const size_t g32 = sizeof(float4) * G32_ST * 64 * 8;
        MPJ_CUDA_TRY(set_smem(k_pair_gram_f32t, (size_t)(g32)));
        k_pair_gram_f32t<<<dim3(a.nsplit, a.npairs), G32_NT, g32, st>>>(a);
    } else {
        k_pair_gram<T, W><<<dim3(a.nsplit, a.npairs), 64, 0, st>>>(a);
    }
    MPJ_LAUNCHED();
    if (hook) hook->end(hook->ctx, KName<T>::gram);
solve:
    const size_t sms = sizeof(InnerSmem<T, W>);
    MPJ_CUDA_TRY(set_smem(k_pair_solve<T, W>, sms));
    // overlapped update (fp32 tcgen05 with programmatic dependent launch): no event may sit
    // between the solve and the update, so one bracket covers both
    const bool overlap = a.pdl && (sizeof(T) == 8 || (W == 64 && a.use_tc));
    const char* both = sizeof(T) == 4 ? "pair_solve_update_f32" : "pair_solve_update_f64";
    if (hook) hook->begin(hook->ctx, overlap ? both : KName<T>::solve);
    {
        // a programmatic dependent of the Gram under gram_pdl (per-pair counters, solve_prologue)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)a.npairs);
        cfg.blockDim = dim3(inner_nt<W>());
        cfg.dynamicSmemBytes = sms;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = a.gram_pdl ? 1 : 0;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_pair_solve<T, W>, a);
        if (e != cudaSuccess) {
            mpj_record_cuda_error(e, "cudaLaunchKernelEx(solve)", __FILE__, __LINE__);
            return -4;
        }
    }
    MPJ_LAUNCHED();
    if (overlap) {
        int rc = 0;
        if constexpr (sizeof(T) == 4) rc = launch_update_tc_pdl(a, st);
        else rc = launch_update_dmma_pdl<W>(a, st);
        if (rc) return rc;
        if (hook) hook->end(hook->ctx, both);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            mpj_record_cuda_error(e, "jacobi round launch", __FILE__, __LINE__);
            return -4;
        }
        return 0;
    }
    if (hook) hook->end(hook->ctx, KName<T>::solve);
    const long long rows_pad = a.m_pad > a.nv_pad ? a.m_pad : a.nv_pad;
    constexpr int VEC = 16 / sizeof(T);
    const size_t usm = sizeof(T) * (size_t)W * ((64 + VEC) + (W + VEC)) + sizeof(long long) * W;
    MPJ_CUDA_TRY(set_smem(k_pair_update<T, W>, usm));
    if (hook) hook->begin(hook->ctx, KName<T>::update);
    if constexpr (sizeof(T) == 8) {
        const size_t dsm = update_dmma_smem<W>();
        MPJ_CUDA_TRY(set_smem(k_pair_update_dmma<W>, (size_t)(dsm)));
        k_pair_update_dmma<W><<<dim3((unsigned)ceil_div(rows_pad, 1024LL), a.npairs, a.has_v ? 2 : 1),
                                UD_NT, dsm, st>>>(a);
    } else if (W == 64 && a.use_tc) {
        if constexpr (sizeof(T) == 4) launch_update_tc(a, st);
    } else {
        const size_t fsm = sizeof(float) * (size_t)W * ((128 + 4) + (W + 4)) + sizeof(long long) * W;
        MPJ_CUDA_TRY(set_smem(k_pair_update_f32<W>, (size_t)(fsm)));
        (void)usm;
        k_pair_update_f32<W><<<dim3((unsigned)ceil_div(rows_pad, 128), a.npairs, a.has_v ? 2 : 1), 256, fsm, st>>>(a);
    }
    MPJ_LAUNCHED();
    if (hook) hook->end(hook->ctx, KName<T>::update);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        mpj_record_cuda_error(e, "jacobi round launch", __FILE__, __LINE__);
        return -4;
    }
    return 0;
}

// resident CTAs per SM of the Gram kernel used for (T, W) (for the split choice)
template <typename T>
int gram_ctas_per_sm(int W, int use_tc, long long rows_pad, int tma, int kt, int variant) {
    int per = 1;
    if constexpr (sizeof(T) == 8) {
        const size_t smem = gram_dmma_smem(W);
        if (W == 64) {
            cudaFuncSetAttribute(k_pair_gram_dmma<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pair_gram_dmma<64>, 128, smem);
        } else if (W == 32) {
            cudaFuncSetAttribute(k_pair_gram_dmma<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pair_gram_dmma<32>, 128, smem);
        } else {
            cudaFuncSetAttribute(k_pair_gram_dmma<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pair_gram_dmma<16>, 128, smem);
        }
    } else {
        if (W == 64 && use_tc) {
            per = gram_tc_ctas_per_sm(rows_pad, tma, kt, variant);
        } else if (W == 64) {
            const size_t g32 = sizeof(float4) * G32_ST * 64 * 8;
            cudaFuncSetAttribute(k_pair_gram_f32t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g32);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pair_gram_f32t, G32_NT, g32);
        } else if (W == 32) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pair_gram<float, 32>, 64, 0);
        } else {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pair_gram<float, 16>, 64, 0);
        }
    }
    cudaGetLastError();
    return per < 1 ? 1 : per;
}
template int gram_ctas_per_sm<float>(int, int, long long, int, int, int);
template int gram_ctas_per_sm<double>(int, int, long long, int, int, int);

void solve_timing_report(const char* tag, int sweep) {
    static long long* dbg = nullptr;
    if (!(g_mpj_diag & 2)) return;
    if (!dbg) {
        cudaMalloc(&dbg, 8 * sizeof(long long));
        cudaMemset(dbg, 0, 8 * sizeof(long long));
        cudaMemcpyToSymbol(g_solve_dbg, &dbg, sizeof(dbg));
        return;
    }
    long long hv[8];
    cudaMemcpy(hv, dbg, sizeof(hv), cudaMemcpyDeviceToHost);
    const double nl = hv[4] > 0 ? (double)hv[4] : 1.0, ns = hv[3] > 0 ? (double)hv[3] : 1.0;
    fprintf(stderr, "[solve timing %s sweep %d] launches=%lld solves=%lld per launch (cycles): prologue=%.0f total=%.0f; per solve: inner=%.0f\n",
            tag, sweep, hv[4], hv[3], hv[0] / nl, hv[2] / nl, hv[1] / ns);
    cudaMemset(dbg, 0, 8 * sizeof(long long));
}

template <typename T>
int launch_jacobi_round(const JacobiRound<T>& a, int W, cudaStream_t st, const ProfHook* hook) {
    switch (W) {
        case 16: return launch_round_w<T, 16>(a, st, hook);
        case 32: return launch_round_w<T, 32>(a, st, hook);
        case 64: return launch_round_w<T, 64>(a, st, hook);
        default: return -7;
    }
}
template int launch_jacobi_round<float>(const JacobiRound<float>&, int, cudaStream_t, const ProfHook*);
template int launch_jacobi_round<double>(const JacobiRound<double>&, int, cudaStream_t, const ProfHook*);

template <typename T, int W>
static int inner_batch_w(T* G, T* E, int w, T tol_in, int max_inner, int count, int* rot, cudaStream_t st) {
    const size_t sms = sizeof(InnerSmem<T, W>);
    MPJ_CUDA_TRY(set_smem(k_inner_solve_batch<T, W>, sms));
    static long long* dbg = nullptr;
    const bool timing = (g_mpj_diag & 8) != 0;
    if (timing) {
        if (!dbg) cudaMalloc(&dbg, 8 * sizeof(long long));
        cudaMemsetAsync(dbg, 0, 8 * sizeof(long long), st);
        if (sizeof(T) == 4) cudaMemcpyToSymbolAsync(g_inner_dbg_f, &dbg, sizeof(dbg), 0, cudaMemcpyHostToDevice, st);
        else cudaMemcpyToSymbolAsync(g_inner_dbg_d, &dbg, sizeof(dbg), 0, cudaMemcpyHostToDevice, st);
    }
    k_inner_solve_batch<T, W><<<count, inner_nt<W>(), sms, st>>>(G, E, w, tol_in, max_inner, rot);
    MPJ_LAUNCHED();
    if (timing) {
        long long hv[8];
        long long* zero = nullptr;
        cudaMemcpyAsync(hv, dbg, sizeof(hv), cudaMemcpyDeviceToHost, st);
        if (sizeof(T) == 4) cudaMemcpyToSymbolAsync(g_inner_dbg_f, &zero, sizeof(zero), 0, cudaMemcpyHostToDevice, st);
        else cudaMemcpyToSymbolAsync(g_inner_dbg_d, &zero, sizeof(zero), 0, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
        const double rounds = hv[4] > 0 ? (double)hv[4] : 1.0;
        fprintf(stderr, "[inner timing %s w=%d] rounds=%lld per round (cycles from round start): critical=%.0f rotation=%.0f G=%.0f E=%.0f\n",
                sizeof(T) == 4 ? "f32" : "f64", w, hv[4], hv[0] / rounds, hv[1] / rounds, hv[2] / rounds, hv[3] / rounds);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

template <typename T>
int launch_inner_batch(T* G, T* E, int w, T tol_in, int max_inner, int count, int* rot, cudaStream_t st) {
    if (w <= 16) return inner_batch_w<T, 16>(G, E, w, tol_in, max_inner, count, rot, st);
    if (w <= 32) return inner_batch_w<T, 32>(G, E, w, tol_in, max_inner, count, rot, st);
    if (w <= 64) return inner_batch_w<T, 64>(G, E, w, tol_in, max_inner, count, rot, st);
    return -7;
}
template int launch_inner_batch<float>(float*, float*, int, float, int, int, int*, cudaStream_t);
template int launch_inner_batch<double>(double*, double*, int, double, int, int, int*, cudaStream_t);

}  // namespace mpj
