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

struct PairCols {
    int I, J, wI, wJ;
};

__device__ __forceinline__ PairCols pair_cols(int r, int i, int M, int nblk, int b, int n) {
    int a = rr_slot(r, i, M), c = rr_slot(r, M - 1 - i, M);
    PairCols pc;
    pc.I = min(a, c);
    pc.J = max(a, c);
    pc.wI = pc.I < nblk ? min(b, n - pc.I * b) : 0;
    pc.wJ = pc.J < nblk ? min(b, n - pc.J * b) : 0;
    return pc;
}

// global column of pair-local column c (c < wI + wJ)
__device__ __forceinline__ int pair_gcol(const PairCols& pc, int c, int b) {
    return c < pc.wI ? pc.I * b + c : pc.J * b + (c - pc.wI);
}

// ------------------------------------------------------------------------
// k_pair_gram: grid (nsplit, npairs), 64 threads (8 x 8), thread tile
// (W/8) x (W/8) of G.  Row slab [split*R, min((split+1)*R, m_pad)) in k-tiles
// of KT rows, natural column-major staging in shared memory.
// ------------------------------------------------------------------------
template <typename T, int W>
__global__ void __launch_bounds__(64) k_pair_gram(JacobiRound<T> a) {
    constexpr int KT = 32;
    constexpr int VEC = 16 / sizeof(T);       // elements per 16-byte vector
    constexpr int S = KT + VEC;               // padded column stride (conflict-free)
    constexpr int TP = W / 8;
    __shared__ __align__(16) T Ws[2][W * S];
    __shared__ long long colofs[W];

    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
    PairCols pc = pair_cols(a.round, pair, a.M, a.nblk, a.b, a.n);
    const int w = pc.wI + pc.wJ;
    if (tid < W) colofs[tid] = tid < w ? (long long)pair_gcol(pc, tid, a.b) * a.ldx : -1;
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
                long long off = colofs[c];
                if (off >= 0 && r0 + ch * VEC < rend) {
                    const T* src = a.X + off + r0 + ch * VEC;
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
// Inner 2b x 2b solve (reading c-5), one CTA.  G (w x w, stride GS) and
// E in shared memory.  Each inner round: phase A computes the P = w2/2
// rotations of the circle-method round (disjoint pairs, so their parameters
// do not depend on each other); phase B applies J^T G J blockwise on the
// 2 x 2 blocks (writing each block and its mirror from the same numbers, so
// G stays exactly symmetric) and E <- (I + E) J - I in delta form.
// Returns the number of rotations; *sweeps_used receives inner sweeps.
// ------------------------------------------------------------------------
template <typename T, int W>
struct InnerSmem {
    static constexpr int GS = W + 1;
    T G[W * (W + 1)];
    T E[W * (W + 1)];
    T rc[W / 2], rs[W / 2], rt[W / 2], rm[W / 2], rg[W / 2], rpp[W / 2], rqq[W / 2];
    int pp[W / 2], qq[W / 2], act[W / 2];
    int nrot;
    T red[32];
};

template <typename T, int W>
__device__ int inner_solve_dev(InnerSmem<T, W>& sm, int w, T tol_in, int max_inner, int* sweeps_used) {
    constexpr int GS = InnerSmem<T, W>::GS;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int w2 = w + (w & 1);
    const int P = w2 / 2;
    int total = 0, used = 0;
    for (int i = tid; i < W * GS; i += nt) sm.E[i] = T(0);
    for (int isw = 0; isw < max_inner; ++isw) {
        if (tid == 0) sm.nrot = 0;
        __syncthreads();
        used = isw + 1;
        for (int ir = 0; ir < w2 - 1; ++ir) {
            // ---- phase A: rotation parameters
            if (tid < P) {
                int x = rr_slot(ir, tid, w2), y = rr_slot(ir, w2 - 1 - tid, w2);
                int p = min(x, y), q = max(x, y);
                sm.pp[tid] = p;
                sm.qq[tid] = q;
                int active = 0;
                if (q < w) {
                    T gpp = sm.G[p * GS + p], gqq = sm.G[q * GS + q], gpq = sm.G[p * GS + q];
                    // Alg. 1 guard |x_q^T x_p| > eps ||x_p|| ||x_q||
                    if (gpp > T(0) && gqq > T(0) && fabs(gpq) > tol_in * sqrt(gpp) * sqrt(gqq)) {
                        // closest-to-identity rotation (reading c-3)
                        T zeta = (gqq - gpp) / (T(2) * gpq);
                        T t;
                        if (fabs(zeta) > RealTraits<T>::rsqrt_u) {
                            t = T(1) / (T(2) * zeta);
                        } else {
                            T sg = zeta >= T(0) ? T(1) : T(-1);
                            t = sg / (fabs(zeta) + sqrt(T(1) + zeta * zeta));
                        }
                        T rt = sqrt(T(1) + t * t);
                        T c = T(1) / rt;
                        sm.rc[tid] = c;
                        sm.rs[tid] = t * c;
                        sm.rt[tid] = t;
                        sm.rm[tid] = -(t * t * c) / (T(1) + rt);
                        sm.rg[tid] = gpq;
                        sm.rpp[tid] = gpp;
                        sm.rqq[tid] = gqq;
                        active = 1;
                        atomicAdd(&sm.nrot, 1);
                    }
                }
                sm.act[tid] = active;
            }
            __syncthreads();
            // ---- phase B1: G <- J^T G J on 2x2 blocks (A <= B)
            for (int idx = tid; idx < P * P; idx += nt) {
                const int A = idx / P, B = idx - (idx / P) * P;
                if (A > B) continue;
                const int aA = sm.act[A], aB = sm.act[B];
                const int pa = sm.pp[A], qa = sm.qq[A], pb = sm.pp[B], qb = sm.qq[B];
                if (A == B) {
                    if (aA) {
                        const T t = sm.rt[A], g = sm.rg[A];
                        sm.G[pa * GS + pa] = sm.rpp[A] - t * g;
                        sm.G[qa * GS + qa] = sm.rqq[A] + t * g;
                        sm.G[pa * GS + qa] = T(0);
                        sm.G[qa * GS + pa] = T(0);
                    }
                    continue;
                }
                if (!aA && !aB) continue;
                const bool qav = qa < w, qbv = qb < w;
                T x00 = sm.G[pa * GS + pb];
                T x01 = qbv ? sm.G[pa * GS + qb] : T(0);
                T x10 = qav ? sm.G[qa * GS + pb] : T(0);
                T x11 = (qav && qbv) ? sm.G[qa * GS + qb] : T(0);
                if (aB) {   // columns (pb, qb) <- (c x_p - s x_q, s x_p + c x_q)
                    const T c = sm.rc[B], s = sm.rs[B];
                    T y00 = c * x00 - s * x01, y01 = s * x00 + c * x01;
                    T y10 = c * x10 - s * x11, y11 = s * x10 + c * x11;
                    x00 = y00; x01 = y01; x10 = y10; x11 = y11;
                }
                if (aA) {   // rows (pa, qa)
                    const T c = sm.rc[A], s = sm.rs[A];
                    T z00 = c * x00 - s * x10, z10 = s * x00 + c * x10;
                    T z01 = c * x01 - s * x11, z11 = s * x01 + c * x11;
                    x00 = z00; x01 = z01; x10 = z10; x11 = z11;
                }
                sm.G[pa * GS + pb] = x00; sm.G[pb * GS + pa] = x00;
                if (qbv) { sm.G[pa * GS + qb] = x01; sm.G[qb * GS + pa] = x01; }
                if (qav) { sm.G[qa * GS + pb] = x10; sm.G[pb * GS + qa] = x10; }
                if (qav && qbv) { sm.G[qa * GS + qb] = x11; sm.G[qb * GS + qa] = x11; }
            }
            // ---- phase B2: E <- (I + E) J - I (delta form)
            for (int idx = tid; idx < P * w; idx += nt) {
                const int k = idx / w, rho = idx - (idx / w) * w;
                if (!sm.act[k]) continue;
                const int p = sm.pp[k], q = sm.qq[k];
                const T c = sm.rc[k], s = sm.rs[k], cm1 = sm.rm[k];
                const T ep = sm.E[rho * GS + p], eq = sm.E[rho * GS + q];
                T np = c * ep - s * eq, nq = s * ep + c * eq;
                if (rho == p) { np += cm1; nq += s; }
                if (rho == q) { np -= s; nq += cm1; }
                sm.E[rho * GS + p] = np;
                sm.E[rho * GS + q] = nq;
            }
            __syncthreads();
        }
        const int nr = sm.nrot;
        total += nr;
        __syncthreads();
        if (nr == 0) break;
    }
    if (sweeps_used) *sweeps_used = used;
    return total;
}

// ------------------------------------------------------------------------
// k_pair_solve: one CTA per pair.
// ------------------------------------------------------------------------
template <typename T, int W>
__global__ void __launch_bounds__(256) k_pair_solve(JacobiRound<T> a) {
    constexpr int GS = InnerSmem<T, W>::GS;
    extern __shared__ __align__(16) unsigned char smraw[];
    InnerSmem<T, W>& sm = *reinterpret_cast<InnerSmem<T, W>*>(smraw);
    const int pair = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    PairCols pc = pair_cols(a.round, pair, a.M, a.nblk, a.b, a.n);
    const int w = pc.wI + pc.wJ;
    // fixed-order reduction over row slabs (deterministic)
    const T* part = a.partial + (long long)pair * a.nsplit * (W * W);
    for (int e = tid; e < W * W; e += nt) {
        const int p = e / W, q = e - (e / W) * W;
        if (p < w && q < w && p <= q) {
            T s = T(0);
            for (int sp = 0; sp < a.nsplit; ++sp) s += part[(long long)sp * (W * W) + p * W + q];
            sm.G[p * GS + q] = s;
            sm.G[q * GS + p] = s;
        }
    }
    __syncthreads();
    // pair metric: max_{p<q} |g_pq| / (sqrt(g_pp) sqrt(g_qq))
    T off = T(0);
    for (int e = tid; e < w * w; e += nt) {
        const int p = e / w, q = e - (e / w) * w;
        if (p < q) {
            T gpp = sm.G[p * GS + p], gqq = sm.G[q * GS + q];
            if (gpp > T(0) && gqq > T(0)) {
                T v = fabs(sm.G[p * GS + q]) / (sqrt(gpp) * sqrt(gqq));
                off = v > off ? v : off;
            }
        }
    }
    off = block_max(off, sm.red);
    const bool rotate = off > a.tol;
    if (tid == 0) {
        atomic_max_nonneg(a.sweep_off, (double)off);
        if (rotate) atomicAdd(a.sweep_upd, 1);
        a.flag[pair] = rotate ? 1 : 0;
    }
    if (!rotate) return;
    inner_solve_dev<T, W>(sm, w, a.tol_in, a.max_inner, nullptr);
    T* E = a.E + (long long)pair * (W * W);
    for (int e = tid; e < W * W; e += nt) {
        const int k = e / W, j = e - (e / W) * W;
        E[e] = (k < w && j < w) ? sm.E[k * GS + j] : T(0);   // E[k][j] row-major
    }
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
    long long* colofs = reinterpret_cast<long long*>(Es + W * SE);
    const int pair = blockIdx.y, which = blockIdx.z;
    if (!a.flag[pair]) return;
    T* Mx = which ? a.V : a.X;
    if (Mx == nullptr) return;
    const long long ld = which ? a.ldv : a.ldx;
    const long long rows_pad = which ? a.nv_pad : a.m_pad;
    const long long row0 = (long long)blockIdx.x * RC;
    if (row0 >= rows_pad) return;
    const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
    PairCols pc = pair_cols(a.round, pair, a.M, a.nblk, a.b, a.n);
    const int w = pc.wI + pc.wJ;
    if (tid < W) colofs[tid] = tid < w ? (long long)pair_gcol(pc, tid, a.b) * ld : -1;
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
        if (colofs[k] >= 0 && ch * VEC < nrow)
            *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(Mx + colofs[k] + row0 + ch * VEC);
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
        T* dstc = Mx + colofs[col] + row0 + ty * 8;
        if (ty * 8 >= nrow) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) dstc[i] = Ws[col * SW + ty * 8 + i] + acc[i][j];
    }
}

// ------------------------------------------------------------------------
// k_inner_solve_batch: test entry (mpjsvd_inner_solve): count matrices.
// ------------------------------------------------------------------------
template <typename T, int W>
__global__ void __launch_bounds__(256) k_inner_solve_batch(T* G, T* E, int w, T tol_in, int max_inner, int* rot) {
    constexpr int GS = InnerSmem<T, W>::GS;
    extern __shared__ __align__(16) unsigned char smraw[];
    InnerSmem<T, W>& sm = *reinterpret_cast<InnerSmem<T, W>*>(smraw);
    T* g = G + (long long)blockIdx.x * w * w;
    T* e = E + (long long)blockIdx.x * w * w;
    for (int i = threadIdx.x; i < w * w; i += blockDim.x) sm.G[(i % w) * GS + i / w] = g[i];
    __syncthreads();
    int nr = inner_solve_dev<T, W>(sm, w, tol_in, max_inner, nullptr);
    for (int i = threadIdx.x; i < w * w; i += blockDim.x) {
        g[i] = sm.G[(i % w) * GS + i / w];
        e[i] = sm.E[(i % w) * GS + i / w];   // column-major out: e[row + col*w] = E[row][col]
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
static int launch_round_w(const JacobiRound<T>& a, cudaStream_t st, const ProfHook* hook) {
    if (hook) hook->begin(hook->ctx, KName<T>::gram);
    k_pair_gram<T, W><<<dim3(a.nsplit, a.npairs), 64, 0, st>>>(a);
    MPJ_LAUNCHED();
    if (hook) hook->end(hook->ctx, KName<T>::gram);
    const size_t sms = sizeof(InnerSmem<T, W>);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_pair_solve<T, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sms);
        attr_set = true;
    }
    if (hook) hook->begin(hook->ctx, KName<T>::solve);
    k_pair_solve<T, W><<<a.npairs, 256, sms, st>>>(a);
    MPJ_LAUNCHED();
    if (hook) hook->end(hook->ctx, KName<T>::solve);
    const long long rows_pad = a.m_pad > a.nv_pad ? a.m_pad : a.nv_pad;
    constexpr int VEC = 16 / sizeof(T);
    const size_t usm = sizeof(T) * (size_t)W * ((64 + VEC) + (W + VEC)) + sizeof(long long) * W;
    static bool attr_u = false;
    if (!attr_u) {
        cudaFuncSetAttribute(k_pair_update<T, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm);
        attr_u = true;
    }
    if (hook) hook->begin(hook->ctx, KName<T>::update);
    k_pair_update<T, W><<<dim3((unsigned)ceil_div(rows_pad, 64), a.npairs, a.V ? 2 : 1), 64, usm, st>>>(a);
    MPJ_LAUNCHED();
    if (hook) hook->end(hook->ctx, KName<T>::update);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        mpj_record_cuda_error(e, "jacobi round launch", __FILE__, __LINE__);
        return -4;
    }
    return 0;
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
    cudaFuncSetAttribute(k_inner_solve_batch<T, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sms);
    k_inner_solve_batch<T, W><<<count, 256, sms, st>>>(G, E, w, tol_in, max_inner, rot);
    MPJ_LAUNCHED();
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
