// k_tc.cu -- tcgen05 (5th-generation tensor core) kernels of the fp32 Jacobi
// stage (reading c-20).
//
// The fp32 block Jacobi's two dense contractions run on the TF32 tensor cores
// with fp32 operands split as x = hi + lo (hi = x with the low 13 mantissa
// bits cleared, i.e. exactly representable in tf32; lo = x - hi exactly),
// accumulating in TMEM in fp32:
//   k_pair_gram_tc    G = W^T W of a row slab of W = [X_I X_J] (n x 64):
//                     A = [W_hi^T ; W_lo^T] (128 x K), B_hi = W_hi^T, B_lo = W_lo^T,
//                     D = A B_hi^T + A B_lo^T (M = 128, N = 64), so that
//                     G = D[0:64] + D[64:128] = (hi + lo)^T (hi + lo);
//   k_pair_update_tc  out = W + W E on 128-row tiles:
//                     D = W_hi E_hi + W_lo E_hi + W_hi E_lo (3 passes, K = 64).
// Per-product error ~2^-21 relative (the lo parts are tf32-truncated by the
// MMA), against 2^-24 for FFMA: the fp32 stage only produces the initial
// guess the fp64 refinement corrects (reading c-20).
//
// Operands are staged by the threads into shared memory in the canonical
// K-major SWIZZLE_NONE layout (core matrices of 8 rows x 16 B; LBO = 128 B
// between the two k-halves of a K = 8 step, SBO between 8-row groups); one
// elected thread issues tcgen05.mma, completion is signalled through
// tcgen05.commit -> mbarrier, and the epilogue reads TMEM with tcgen05.ld
// (warp w owns TMEM lanes 32w..32w+31).  Validated by tools/tc_probe.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include "common.cuh"
#include "jacobi.h"

namespace mpj {

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// shared-memory matrix descriptor: SWIZZLE_NONE, version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// instruction descriptor kind::tf32, fp32 accumulate, both operands K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(mbar)));
}
__device__ __forceinline__ void mbar_init(uint64_t* mbar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(mbar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(mbar)), "r"(parity));
    }
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n"); }

template <int NCOL>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst) {   // one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst)), "n"(NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
template <int NCOL>
__device__ __forceinline__ void tmem_free(uint32_t base) {     // the allocating warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(NCOL));
}
// 32 lanes x 16 columns of fp32 (thread = lane, v[j] = column c0 + j)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ float hi_part(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ float4 hi4(float4 v) { return make_float4(hi_part(v.x), hi_part(v.y), hi_part(v.z), hi_part(v.w)); }
__device__ __forceinline__ float4 lo4(float4 v, float4 h) { return make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w); }

// byte offset of element (r, k) in a K-major SWIZZLE_NONE operand with KK columns
__device__ __forceinline__ uint32_t koff(int r, int k, int KK) {
    return (uint32_t)(((r >> 3) * (KK >> 2) + (k >> 2)) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

// 4 x 4 transpose inside each quad of lanes: lane i holds row i of a 4 x 4
// block in v (v.x = column 0 ...) and ends with column i (two butterfly
// stages; each swaps the elements whose index bit differs from the lane's).
__device__ __forceinline__ float4 quad_transpose(float4 v, int lane) {
    const bool b0 = lane & 1, b1 = (lane >> 1) & 1;
    float x = b0 ? v.x : v.y, y = b0 ? v.z : v.w;
    float rx = __shfl_xor_sync(0xffffffffu, x, 1), ry = __shfl_xor_sync(0xffffffffu, y, 1);
    if (b0) { v.x = rx; v.z = ry; } else { v.y = rx; v.w = ry; }
    x = b1 ? v.x : v.z;
    y = b1 ? v.y : v.w;
    rx = __shfl_xor_sync(0xffffffffu, x, 2);
    ry = __shfl_xor_sync(0xffffffffu, y, 2);
    if (b1) { v.x = rx; v.y = ry; } else { v.z = rx; v.w = ry; }
    return v;
}

}  // namespace tc

// ------------------------------------------------------------------------
// k_pair_gram_tc: grid (nsplit, npairs), 128 threads.  The CTA's row slab
// streams through GT_ST shared stages of GT_KT rows.  A stage holds the
// operand A = [H^T ; L^T] (128 x GT_KT, K-major): rows 0..63 are the raw fp32
// W chunks, copied from global memory with cp.async (the tensor core
// truncates them to tf32: exactly the hi part H), rows 64..127 the lo parts
// L = W - H written by the thread that copied the chunk.  One MMA per K = 8
// step, D = A H (M = 128, N = 64), gives D[0:64] = H^T H and D[64:128] = L^T H,
// and G = H^T H + L^T H + (L^T H)^T (the lo x lo term, ~2^-22, is dropped).
// ------------------------------------------------------------------------
constexpr int GT_NT = 128;
template <int KT, int ST>
constexpr size_t gram_tc_smem() { return (size_t)ST * (128 * KT * 4) + 1024; }

__device__ __forceinline__ void cp16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ long long* g_gram_dbg = nullptr;   // phase timers (MPJSVD_GRAM_TIMING=1, tools only)

template <int GT_KT, int GT_ST, int MINB>
__global__ void __launch_bounds__(GT_NT, MINB) k_pair_gram_tc(JacobiRound<float> a) {
    constexpr int GT_STAGE_BYTES = 128 * GT_KT * 4;
    constexpr int GT_CHUNKS = 64 * (GT_KT / 4) / GT_NT;   // 16-byte chunks per thread per tile
    reset_publication(a);
    if (pair_unchanged(a, a.pd[blockIdx.y])) return;
    extern __shared__ __align__(1024) unsigned char gt_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gt_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t mbar[GT_ST + 1];
    __shared__ uint32_t tmem_base;
    __shared__ const float* colp[64];
    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5;
    const PairDesc<float> pd = a.pd[pair];
    const int w = pd.w0 + pd.w1;
    if (tid < 64) colp[tid] = tid < w ? (tid < pd.w0 ? pd.x0 + (long long)tid * a.ldx : pd.x1 + (long long)(tid - pd.w0) * a.ldx) : nullptr;
    if (warp == 0) tc::tmem_alloc<64>(&tmem_base);
    if (tid == 0) {
        for (int s = 0; s <= GT_ST; ++s) tc::mbar_init(&mbar[s]);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;
    const long long rbeg = (long long)split * a.rows_per_split;
    const long long rend = min(rbeg + (long long)a.rows_per_split, (long long)a.m_pad);
    const int ntile = (int)((rend - rbeg + GT_KT - 1) / GT_KT);
    constexpr uint32_t SBO = (GT_KT / 4) * 128;         // 2048 B between 8-row groups
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    const uint32_t sbase = tc::smem_u32(sm);
    // chunk f = tid + 128 u: column c = 8 (f / (8 KT/4)) + (f & 7), rows 4 k4 .. + 3, k4 = (f >> 3) % (KT/4)
    const float* src[GT_CHUNKS];
    uint32_t soff[GT_CHUNKS];
    int krow[GT_CHUNKS];
#pragma unroll
    for (int u = 0; u < GT_CHUNKS; ++u) {
        const int f = tid + GT_NT * u;
        const int cg = f / (8 * (GT_KT / 4)), k4 = (f >> 3) % (GT_KT / 4), c8 = f & 7;
        const int c = 8 * cg + c8;
        src[u] = colp[c] ? colp[c] + 4 * k4 : nullptr;
        krow[u] = 4 * k4;
        soff[u] = (uint32_t)((cg * (GT_KT / 4) + k4) * 128 + c8 * 16);
    }
    auto issue = [&](int t) {               // raw chunks of tile t -> stage t % GT_ST (rows 0..63)
        unsigned char* st = sm + (size_t)(t % GT_ST) * GT_STAGE_BYTES;
        const long long r0 = rbeg + (long long)t * GT_KT;
#pragma unroll
        for (int u = 0; u < GT_CHUNKS; ++u) {
            if (src[u] && r0 + krow[u] < rend) cp16(sbase + (uint32_t)((t % GT_ST) * GT_STAGE_BYTES) + soff[u], src[u] + r0);
            else *reinterpret_cast<float4*>(st + soff[u]) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
#pragma unroll
    for (int t = 0; t < GT_ST - 1; ++t) {
        if (t < ntile) issue(t);
        cp_commit();
    }
    long long* dbg = g_gram_dbg;
    long long tw[6] = {0, 0, 0, 0, 0, 0};
    for (int t = 0; t < ntile; ++t) {
        const int s = t % GT_ST;
        unsigned char* st = sm + (size_t)s * GT_STAGE_BYTES;
        long long c0 = dbg ? clock64() : 0;
        cp_wait<GT_ST - 2>();                           // this thread's chunks of tile t have landed
        long long c1 = dbg ? clock64() : 0;
#pragma unroll
        for (int u = 0; u < GT_CHUNKS; ++u) {
            const float4 x = *reinterpret_cast<const float4*>(st + soff[u]);
            *reinterpret_cast<float4*>(st + soff[u] + 8 * SBO) = tc::lo4(x, tc::hi4(x));
        }
        tc::fence_async_smem();
        long long c2 = dbg ? clock64() : 0;
        __syncthreads();
        long long c3 = dbg ? clock64() : 0;
        if (tid == 0) {
            tc::fence_after();
            const uint32_t base = sbase + (uint32_t)(s * GT_STAGE_BYTES);
#pragma unroll
            for (int ks = 0; ks < GT_KT / 8; ++ks) {
                const uint64_t ad = tc::sdesc(base + ks * 256, 128, SBO);
                tc::mma(tmem, ad, ad, idesc, (t > 0 || ks > 0) ? 1u : 0u);   // B = rows 0..63 = H^T
            }
            tc::commit(&mbar[s]);
        }
        // refill: tile t + GT_ST - 1 goes to the stage of tile t - 1 once its MMAs are done
        const int tn = t + GT_ST - 1;
        long long c4 = dbg ? clock64() : 0, c5 = c4;
        if (tn < ntile) {
            if (t >= 1) tc::mbar_wait(&mbar[(t - 1) % GT_ST], (uint32_t)(((t - 1) / GT_ST) & 1));
            c5 = dbg ? clock64() : 0;
            issue(tn);
        }
        cp_commit();
        if (dbg) {
            const long long c6 = clock64();
            tw[0] += c1 - c0; tw[1] += c2 - c1; tw[2] += c3 - c2; tw[3] += c4 - c3; tw[4] += c5 - c4; tw[5] += c6 - c5;
        }
    }
    if (dbg && tid == 32) {
        for (int i = 0; i < 6; ++i) atomicAdd((unsigned long long*)(dbg + i), (unsigned long long)tw[i]);
        atomicAdd((unsigned long long*)(dbg + 6), (unsigned long long)ntile);
    }
    float* out = a.partial + ((long long)pair * a.nsplit + split) * (64 * 64);
    float* red = reinterpret_cast<float*>(sm);           // 2 x 64 x 65 floats (stages are free after the last MMA)
    cp_wait<0>();
    if (ntile > 0) {
        if (tid == 0) tc::commit(&mbar[GT_ST]);
        tc::mbar_wait(&mbar[GT_ST], 0);
        tc::fence_after();
        // every thread: TMEM lane tid (row tid of D) -> red[tid / 64][tid % 64][:]
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
            float v[16];
            tc::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) red[tid * 65 + c0 + j] = v[j];
        }
        __syncthreads();
        // G[p][q] = (H^T H)[p][q] + (L^T H)[p][q] + (L^T H)[q][p]
        for (int e = tid; e < 64 * 64; e += GT_NT) {
            const int p = e >> 6, q = e & 63;
            out[e] = red[p * 65 + q] + red[(64 + p) * 65 + q] + red[(64 + q) * 65 + p];
        }
    } else {
        for (int e = tid; e < 64 * 64; e += GT_NT) out[e] = 0.f;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<64>(tmem);
}

// ------------------------------------------------------------------------
// k_pair_gram_tma: k_pair_gram_tc with the raw W chunks loaded by TMA.  A
// 4-D tensor view of X (r4 = 4 consecutive rows, c8 = 8 columns at stride ld,
// kq = row groups of 4 at stride 16 B, cg = column groups of 8) makes one box
// {4, 8, KT/4, 4} = 32 columns x KT rows land in shared memory exactly in the
// canonical K-major SWIZZLE_NONE layout (core matrix (cg, kq) at cg SBO + kq
// 128 B): X_I fills M-groups 0..3, X_J 4..7 of the stage, one elected thread
// issues both boxes (mbarrier complete_tx), so no thread issues per-chunk
// copies.  The 128 threads then write the lo parts (M-groups 8..15) from the
// landed chunks, thread 0 issues the MMAs and refills the stage of tile t - 1
// after its MMAs complete.  Rows past the matrix and columns past its last
// column are zero-filled by the TMA unit.
// ------------------------------------------------------------------------
template <int GM_KT, int GM_ST>
constexpr size_t gram_tma_smem() { return (size_t)GM_ST * (128 * GM_KT * 4) + 1024; }

__device__ __forceinline__ void tma_load_4d(uint32_t sdst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
        ::"r"(sdst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(tc::smem_u32(mbar))
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tc::smem_u32(mbar)), "r"(bytes)
                 : "memory");
}

template <int GM_KT, int GM_ST, int MINB>
__global__ void __launch_bounds__(GT_NT, MINB) k_pair_gram_tma(JacobiRound<float> a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int STAGE = 128 * GM_KT * 4;              // raw (64 x KT) + lo (64 x KT)
    constexpr uint32_t SBO = (GM_KT / 4) * 128;         // 2048 B between 8-row (M) groups
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    reset_publication(a);
    if (pair_unchanged(a, a.pd[blockIdx.y])) return;
    extern __shared__ __align__(1024) unsigned char gm_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gm_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[GM_ST], done[GM_ST], fin;
    __shared__ uint32_t tmem_base;
    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5;
    const PairDesc<float> pd = a.pd[pair];
    const int cI = (int)((pd.x0 - a.tbase) / a.tld), cJ = (int)((pd.x1 - a.tbase) / a.tld);
    const bool hasJ = pd.w1 > 0;
    const uint32_t tx = hasJ ? 2u * 32u * GM_KT * 4u : 32u * GM_KT * 4u;
    if (warp == 0) tc::tmem_alloc<64>(&tmem_base);
    if (tid == 0) {
        for (int s = 0; s < GM_ST; ++s) { tc::mbar_init(&full[s]); tc::mbar_init(&done[s]); }
        tc::mbar_init(&fin);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    if (!hasJ) {   // bye pair: M-groups 4..7 stay zero in every stage
        for (int s = 0; s < GM_ST; ++s)
            for (int i = tid; i < 4 * (int)SBO / 16; i += GT_NT)
                reinterpret_cast<float4*>(sm + (size_t)s * STAGE + 4 * SBO)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        tc::fence_async_smem();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;
    const long long rbeg = (long long)split * a.rows_per_split;
    const long long rend = min(rbeg + (long long)a.rows_per_split, (long long)a.m_pad);
    const int ntile = (int)((rend - rbeg + GM_KT - 1) / GM_KT);
    const uint32_t sbase = tc::smem_u32(sm);
    auto issue = [&](int t) {                // thread 0: both boxes of tile t -> stage t % GM_ST
        const int s = t % GM_ST;
        const int kq = (int)((rbeg + (long long)t * GM_KT) >> 2);
        mbar_expect_tx(&full[s], tx);
        tma_load_4d(sbase + (uint32_t)(s * STAGE), &tmap, 0, 0, kq, cI >> 3, &full[s]);
        if (hasJ) tma_load_4d(sbase + (uint32_t)(s * STAGE) + 4 * SBO, &tmap, 0, 0, kq, cJ >> 3, &full[s]);
    };
    if (tid == 0)
        for (int t = 0; t < GM_ST && t < ntile; ++t) issue(t);
    for (int t = 0; t < ntile; ++t) {
        const int s = t % GM_ST;
        unsigned char* st = sm + (size_t)s * STAGE;
        tc::mbar_wait(&full[s], (uint32_t)((t / GM_ST) & 1));
        // lo parts of the landed raw chunks: 1024 16-byte chunks, 8 per thread, linear (conflict-free)
#pragma unroll
        for (int u = 0; u < GM_KT / 8; ++u) {
            const int f = tid + GT_NT * u;
            const float4 x = reinterpret_cast<const float4*>(st)[f];
            reinterpret_cast<float4*>(st + 8 * SBO)[f] = tc::lo4(x, tc::hi4(x));
        }
        tc::fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            const uint32_t base = sbase + (uint32_t)(s * STAGE);
#pragma unroll
            for (int ks = 0; ks < GM_KT / 8; ++ks) {
                const uint64_t ad = tc::sdesc(base + ks * 256, 128, SBO);
                tc::mma(tmem, ad, ad, idesc, (t > 0 || ks > 0) ? 1u : 0u);
            }
            tc::commit(&done[s]);
            // refill the stage of tile t - 1 once its MMAs have read it
            if (t >= 1 && t - 1 + GM_ST < ntile) {
                const int sp = (t - 1) % GM_ST;
                tc::mbar_wait(&done[sp], (uint32_t)(((t - 1) / GM_ST) & 1));
                issue(t - 1 + GM_ST);
            }
        }
    }
    float* out = a.partial + ((long long)pair * a.nsplit + split) * (64 * 64);
    float* red = reinterpret_cast<float*>(sm);
    if (ntile > 0) {
        if (tid == 0) tc::commit(&fin);
        tc::mbar_wait(&fin, 0);
        tc::fence_after();
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
            float v[16];
            tc::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) red[tid * 65 + c0 + j] = v[j];
        }
        __syncthreads();
        for (int e = tid; e < 64 * 64; e += GT_NT) {
            const int p = e >> 6, q = e & 63;
            out[e] = red[p * 65 + q] + red[(64 + p) * 65 + q] + red[(64 + q) * 65 + p];
        }
    } else {
        for (int e = tid; e < 64 * 64; e += GT_NT) out[e] = 0.f;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<64>(tmem);
}

// k_pair_gram_tma_ws: the TMA Gram with warp specialisation.  Lane 0 of warp 0 is the producer and the MMA
// issuer (TMA of tile t + ST - 1 into the stage of tile t - 1 once that tile's MMAs completed; the MMAs of tile
// t once its lo parts are written); warps 1..3 write the lo parts of each landed stage and arrive on the
// stage's lo_ready barrier (96 arrivals) -- no CTA-wide barrier per tile, so the lo work of the next tile
// overlaps the producer's waits.  Same operand layout, MMA sequence and epilogue as k_pair_gram_tma (bitwise
// equal results).
__device__ __forceinline__ void mbar_init_n(uint64_t* mbar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tc::smem_u32(mbar)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tc::smem_u32(mbar)) : "memory");
}

template <int GM_KT, int GM_ST, int MINB>
__global__ void __launch_bounds__(GT_NT, MINB) k_pair_gram_tma_ws(JacobiRound<float> a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int STAGE = 128 * GM_KT * 4;
    constexpr uint32_t SBO = (GM_KT / 4) * 128;
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    constexpr int RAW4 = 64 * GM_KT / 4;                // float4 chunks of the raw half of a stage
    reset_publication(a);
    if (pair_unchanged(a, a.pd[blockIdx.y])) return;
    extern __shared__ __align__(1024) unsigned char gw_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gw_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[GM_ST], lor[GM_ST], done[GM_ST], fin;
    __shared__ uint32_t tmem_base;
    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5;
    const PairDesc<float> pd = a.pd[pair];
    const int cI = (int)((pd.x0 - a.tbase) / a.tld), cJ = (int)((pd.x1 - a.tbase) / a.tld);
    const bool hasJ = pd.w1 > 0;
    const uint32_t tx = hasJ ? 2u * 32u * GM_KT * 4u : 32u * GM_KT * 4u;
    if (warp == 0) tc::tmem_alloc<64>(&tmem_base);
    if (tid == 0) {
        for (int s = 0; s < GM_ST; ++s) {
            tc::mbar_init(&full[s]);
            mbar_init_n(&lor[s], GT_NT - 32);
            tc::mbar_init(&done[s]);
        }
        tc::mbar_init(&fin);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    if (!hasJ) {
        for (int s = 0; s < GM_ST; ++s)
            for (int i = tid; i < 4 * (int)SBO / 16; i += GT_NT)
                reinterpret_cast<float4*>(sm + (size_t)s * STAGE + 4 * SBO)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        tc::fence_async_smem();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;
    const long long rbeg = (long long)split * a.rows_per_split;
    const long long rend = min(rbeg + (long long)a.rows_per_split, (long long)a.m_pad);
    const int ntile = (int)((rend - rbeg + GM_KT - 1) / GM_KT);
    const uint32_t sbase = tc::smem_u32(sm);
    if (warp == 0) {
        if (tid == 0) {
            auto issue = [&](int t) {
                const int s = t % GM_ST;
                const int kq = (int)((rbeg + (long long)t * GM_KT) >> 2);
                mbar_expect_tx(&full[s], tx);
                tma_load_4d(sbase + (uint32_t)(s * STAGE), &tmap, 0, 0, kq, cI >> 3, &full[s]);
                if (hasJ) tma_load_4d(sbase + (uint32_t)(s * STAGE) + 4 * SBO, &tmap, 0, 0, kq, cJ >> 3, &full[s]);
            };
            for (int t = 0; t < GM_ST && t < ntile; ++t) issue(t);
            for (int t = 0; t < ntile; ++t) {
                const int s = t % GM_ST;
                tc::mbar_wait(&lor[s], (uint32_t)((t / GM_ST) & 1));
                tc::fence_after();
                const uint32_t base = sbase + (uint32_t)(s * STAGE);
#pragma unroll
                for (int ks = 0; ks < GM_KT / 8; ++ks) {
                    const uint64_t ad = tc::sdesc(base + ks * 256, 128, SBO);
                    tc::mma(tmem, ad, ad, idesc, (t > 0 || ks > 0) ? 1u : 0u);
                }
                tc::commit(&done[s]);
                if (t >= 1 && t - 1 + GM_ST < ntile) {
                    const int sp = (t - 1) % GM_ST;
                    tc::mbar_wait(&done[sp], (uint32_t)(((t - 1) / GM_ST) & 1));
                    issue(t - 1 + GM_ST);
                }
            }
            if (ntile > 0) tc::commit(&fin);
        }
        __syncwarp();
    } else {
        const int lt = tid - 32;
        for (int t = 0; t < ntile; ++t) {
            const int s = t % GM_ST;
            unsigned char* st = sm + (size_t)s * STAGE;
            tc::mbar_wait(&full[s], (uint32_t)((t / GM_ST) & 1));
            for (int f = lt; f < RAW4; f += GT_NT - 32) {
                const float4 x = reinterpret_cast<const float4*>(st)[f];
                reinterpret_cast<float4*>(st + 8 * SBO)[f] = tc::lo4(x, tc::hi4(x));
            }
            tc::fence_async_smem();
            mbar_arrive(&lor[s]);
        }
    }
    float* out = a.partial + ((long long)pair * a.nsplit + split) * (64 * 64);
    float* red = reinterpret_cast<float*>(sm);
    if (ntile > 0) {
        tc::mbar_wait(&fin, 0);
        tc::fence_after();
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
            float v[16];
            tc::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) red[tid * 65 + c0 + j] = v[j];
        }
        __syncthreads();
        for (int e = tid; e < 64 * 64; e += GT_NT) {
            const int p = e >> 6, q = e & 63;
            out[e] = red[p * 65 + q] + red[(64 + p) * 65 + q] + red[(64 + q) * 65 + p];
        }
    } else {
        for (int e = tid; e < 64 * 64; e += GT_NT) out[e] = 0.f;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<64>(tmem);
}

// k_pair_gram_sw: the TMA Gram on 128-byte-swizzled operands.  One 2-D box of 32 rows x 32 columns per block
// (a 128-byte inner run per column instead of the 16-byte runs of the 4-D canonical view) lands column c of the
// block as M-row c of a K-major SWIZZLE_128B operand (8-row atoms of 1024 B, K = 32 rows per stage); X_I fills
// M-rows 0..31, X_J 32..63, the lo parts (written at the same offsets + 8 KB, so with the same swizzle)
// 64..127.  The MMA descriptors use layout type SWIZZLE_128B (SBO = 1024 B) and advance 32 B per K = 8 step.
// Same K order and MMA sequence as k_pair_gram_tma at KT = 32: bitwise equal partial Grams.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void tma_load_2d_g(uint32_t sdst, const CUtensorMap* map, int c0, int c1, uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(sdst), "l"(map), "r"(c0), "r"(c1), "r"(tc::smem_u32(mbar))
        : "memory");
}

template <int GM_ST, int MINB, int NT = GT_NT>
__global__ void __launch_bounds__(NT, MINB) k_pair_gram_sw(JacobiRound<float> a, const __grid_constant__ CUtensorMap smap) {
    constexpr int KT = 32;
    constexpr int STAGE = 128 * KT * 4;                 // 16 KB: raw I | raw J | lo I | lo J, 4 KB each
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    reset_publication(a);
    gram_pdl_begin(a);
    if (pair_unchanged(a, a.pd[blockIdx.y])) return;
    extern __shared__ __align__(1024) unsigned char gs_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gs_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[GM_ST], done[GM_ST], fin;
    __shared__ uint32_t tmem_base;
    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5;
    const PairDesc<float> pd = a.pd[pair];
    const int cI = (int)((pd.x0 - a.tbase) / a.tld), cJ = (int)((pd.x1 - a.tbase) / a.tld);
    const bool hasJ = pd.w1 > 0;
    const uint32_t tx = hasJ ? 2u * 32u * KT * 4u : 32u * KT * 4u;
    if (warp == 0) tc::tmem_alloc<64>(&tmem_base);
    if (tid == 0) {
        for (int s = 0; s < GM_ST; ++s) { tc::mbar_init(&full[s]); tc::mbar_init(&done[s]); }
        tc::mbar_init(&fin);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    if (!hasJ) {   // bye pair: M-rows 32..63 (raw J) stay zero in every stage
        for (int s = 0; s < GM_ST; ++s)
            for (int i = tid; i < 4096 / 16; i += NT)
                reinterpret_cast<float4*>(sm + (size_t)s * STAGE + 4096)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        tc::fence_async_smem();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;
    const long long rbeg = (long long)split * a.rows_per_split;
    const long long rend = min(rbeg + (long long)a.rows_per_split, (long long)a.m_pad);
    const int ntile = (int)((rend - rbeg + KT - 1) / KT);
    const uint32_t sbase = tc::smem_u32(sm);
    auto issue = [&](int t) {
        const int s = t % GM_ST;
        const int r0 = (int)(rbeg + (long long)t * KT);
        mbar_expect_tx(&full[s], tx);
        tma_load_2d_g(sbase + (uint32_t)(s * STAGE), &smap, r0, cI, &full[s]);
        if (hasJ) tma_load_2d_g(sbase + (uint32_t)(s * STAGE) + 4096, &smap, r0, cJ, &full[s]);
    };
    if (tid == 0)
        for (int t = 0; t < GM_ST && t < ntile; ++t) issue(t);
    for (int t = 0; t < ntile; ++t) {
        const int s = t % GM_ST;
        unsigned char* st = sm + (size_t)s * STAGE;
        tc::mbar_wait(&full[s], (uint32_t)((t / GM_ST) & 1));
#pragma unroll
        for (int u = 0; u < 512 / NT; ++u) {     // 512 raw float4 chunks, linear
            const int f = tid + NT * u;
            const float4 x = reinterpret_cast<const float4*>(st)[f];
            reinterpret_cast<float4*>(st + 8192)[f] = tc::lo4(x, tc::hi4(x));
        }
        tc::fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            const uint32_t base = sbase + (uint32_t)(s * STAGE);
#pragma unroll
            for (int ks = 0; ks < KT / 8; ++ks) {
                const uint64_t ad = sdesc_sw128(base + ks * 32);
                tc::mma(tmem, ad, ad, idesc, (t > 0 || ks > 0) ? 1u : 0u);
            }
            tc::commit(&done[s]);
            if (t >= 1 && t - 1 + GM_ST < ntile) {
                const int sp = (t - 1) % GM_ST;
                tc::mbar_wait(&done[sp], (uint32_t)(((t - 1) / GM_ST) & 1));
                issue(t - 1 + GM_ST);
            }
        }
    }
    float* out = a.partial + ((long long)pair * a.nsplit + split) * (64 * 64);
    float* red = reinterpret_cast<float*>(sm);
    if (ntile > 0) {
        if (tid == 0) tc::commit(&fin);
        tc::mbar_wait(&fin, 0);
        tc::fence_after();
        if (tid < 128) {                         // TMEM lanes 0..127: warps 0..3
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 16) {
                float v[16];
                tc::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) red[tid * 65 + c0 + j] = v[j];
            }
        }
        __syncthreads();
        for (int e = tid; e < 64 * 64; e += NT) {
            const int p = e >> 6, q = e & 63;
            out[e] = red[p * 65 + q] + red[(64 + p) * 65 + q] + red[(64 + q) * 65 + p];
        }
    } else {
        for (int e = tid; e < 64 * 64; e += NT) out[e] = 0.f;
    }
    gram_pdl_end(a, pair);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<64>(tmem);
}

// k_pair_gram_sw_ws: k_pair_gram_sw with the work split by warps instead of a CTA barrier per tile.  Warp 0
// (one lane) issues the TMA boxes and the MMAs; warps 1..4 (128 threads) write the lo parts of each stage as
// soon as its boxes land and arrive on the stage's lo barrier (128 arrivals).  The lo warps run up to GM_ST
// tiles ahead of the MMA lane, whose waits (lo parts, the previous tile's MMAs before a refill) no longer
// hold them.  Same operand layout, MMA sequence and epilogue as k_pair_gram_sw: bitwise equal.
template <int GM_ST, int MINB>
__global__ void __launch_bounds__(160, MINB) k_pair_gram_sw_ws(JacobiRound<float> a, const __grid_constant__ CUtensorMap smap) {
    constexpr int KT = 32, NT = 160;
    constexpr int STAGE = 128 * KT * 4;                 // 16 KB: raw I | raw J | lo I | lo J, 4 KB each
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    reset_publication(a);
    gram_pdl_begin(a);
    if (pair_unchanged(a, a.pd[blockIdx.y])) return;
    extern __shared__ __align__(1024) unsigned char gs_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gs_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[GM_ST], done[GM_ST], lo_ready[GM_ST], fin;
    __shared__ uint32_t tmem_base;
    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5;
    const PairDesc<float> pd = a.pd[pair];
    const int cI = (int)((pd.x0 - a.tbase) / a.tld), cJ = (int)((pd.x1 - a.tbase) / a.tld);
    const bool hasJ = pd.w1 > 0;
    const uint32_t tx = hasJ ? 2u * 32u * KT * 4u : 32u * KT * 4u;
    if (warp == 0) tc::tmem_alloc<64>(&tmem_base);
    if (tid == 0) {
        for (int s = 0; s < GM_ST; ++s) {
            tc::mbar_init(&full[s]);
            tc::mbar_init(&done[s]);
            mbar_init_n(&lo_ready[s], 128);
        }
        tc::mbar_init(&fin);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    if (!hasJ) {   // bye pair: M-rows 32..63 (raw J) stay zero in every stage
        for (int s = 0; s < GM_ST; ++s)
            for (int i = tid; i < 4096 / 16; i += NT)
                reinterpret_cast<float4*>(sm + (size_t)s * STAGE + 4096)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        tc::fence_async_smem();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;
    // row tiles of this CTA: its contiguous row slab, or (gram_il, DESIGN.md sec. 8 "L2-aware traversal") the
    // tiles split, split + nsplit, ... of the whole row range, so that all CTAs walk the rows top -> bottom in step
    const bool il = a.gram_il != 0;
    const long long rbeg = il ? (long long)split * KT : (long long)split * a.rows_per_split;
    const long long rend = il ? (long long)a.m_pad : min(rbeg + (long long)a.rows_per_split, (long long)a.m_pad);
    const long long rstep = il ? (long long)a.nsplit * KT : (long long)KT;
    const int ntile = rend > rbeg ? (int)((rend - rbeg + rstep - 1) / rstep) : 0;
    const uint32_t sbase = tc::smem_u32(sm);
    auto issue = [&](int t) {
        const int s = t % GM_ST;
        const int r0 = (int)(rbeg + (long long)t * rstep);
        mbar_expect_tx(&full[s], tx);
        tma_load_2d_g(sbase + (uint32_t)(s * STAGE), &smap, r0, cI, &full[s]);
        if (hasJ) tma_load_2d_g(sbase + (uint32_t)(s * STAGE) + 4096, &smap, r0, cJ, &full[s]);
    };
    if (warp == 0) {
        if (tid == 0) {
            for (int t = 0; t < GM_ST && t < ntile; ++t) issue(t);
            for (int t = 0; t < ntile; ++t) {
                const int s = t % GM_ST;
                tc::mbar_wait(&lo_ready[s], (uint32_t)((t / GM_ST) & 1));
                tc::fence_after();
                const uint32_t base = sbase + (uint32_t)(s * STAGE);
#pragma unroll
                for (int ks = 0; ks < KT / 8; ++ks) {
                    const uint64_t ad = sdesc_sw128(base + ks * 32);
                    tc::mma(tmem, ad, ad, idesc, (t > 0 || ks > 0) ? 1u : 0u);
                }
                tc::commit(&done[s]);
                if (t >= 1 && t - 1 + GM_ST < ntile) {
                    const int sp = (t - 1) % GM_ST;
                    tc::mbar_wait(&done[sp], (uint32_t)(((t - 1) / GM_ST) & 1));
                    issue(t - 1 + GM_ST);
                }
            }
            if (ntile > 0) tc::commit(&fin);
        }
        __syncwarp();
    } else {
        const int lt = tid - 32;                  // 0..127
        for (int t = 0; t < ntile; ++t) {
            const int s = t % GM_ST;
            unsigned char* st = sm + (size_t)s * STAGE;
            tc::mbar_wait(&full[s], (uint32_t)((t / GM_ST) & 1));
#pragma unroll
            for (int u = 0; u < 512 / 128; ++u) {     // 512 raw float4 chunks, linear
                const int f = lt + 128 * u;
                const float4 x = reinterpret_cast<const float4*>(st)[f];
                reinterpret_cast<float4*>(st + 8192)[f] = tc::lo4(x, tc::hi4(x));
            }
            tc::fence_async_smem();
            mbar_arrive(&lo_ready[s]);
        }
    }
    float* out = a.partial + ((long long)pair * a.nsplit + split) * (64 * 64);
    float* red = reinterpret_cast<float*>(sm);
    if (ntile > 0) {
        tc::mbar_wait(&fin, 0);
        tc::fence_after();
        __syncthreads();                           // every stage consumed before red (stage 0) is overwritten
        if (tid < 128) {                           // TMEM lanes 0..127: warps 0..3
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 16) {
                float v[16];
                tc::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) red[tid * 65 + c0 + j] = v[j];
            }
        }
        __syncthreads();
        for (int e = tid; e < 64 * 64; e += NT) {
            const int p = e >> 6, q = e & 63;
            out[e] = red[p * 65 + q] + red[(64 + p) * 65 + q] + red[(64 + q) * 65 + p];
        }
    } else {
        for (int e = tid; e < 64 * 64; e += NT) out[e] = 0.f;
    }
    gram_pdl_end(a, pair);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<64>(tmem);
}

// rows per stage of the TMA Gram (MPJSVD_GRAM_KT = 32 or 64): KT = 64 -> 3 x 32 KB stages, 2 CTAs per SM;
// KT = 32 -> 3 x 16 KB stages, 4 CTAs per SM
// Default by row count (measured on B200): 32 for >= 6144 rows (C5: Gram 237 -> 217 ms), 64 below (C3: 33 vs 35 ms)
int gram_tma_kt(long long rows_pad, int forced) {
    if (forced == 32 || forced == 64) return forced;
    return rows_pad >= 6144 ? 32 : 64;
}

int make_gram_tmap(void* out, const float* base, long long ld, long long rows_pad, long long cols, int kt) {
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(f);
    }
    if (!fn || cols % 8 != 0 || rows_pad % 4 != 0 || ld % 4 != 0) return -1;
    const cuuint64_t gdim[4] = {4, 8, (cuuint64_t)(rows_pad / 4), (cuuint64_t)(cols / 8)};
    const cuuint64_t gstride[3] = {(cuuint64_t)ld * 4, 16, (cuuint64_t)ld * 4 * 8};
    const cuuint32_t box[4] = {4, 8, (cuuint32_t)(kt / 4), 4};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = fn(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                          const_cast<float*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

// ------------------------------------------------------------------------
// k_pair_update_tc: grid (tile groups, npairs, 2 [X, V]), 256 threads;
// out = W + W E on 128-row tiles.  Raw tiles (column-major 128 x 64 fp32)
// stream into a UT_NR-deep cp.async ring; per tile the threads transpose
// from shared memory (thread: row tid % 128, columns 32 (tid / 128) .. + 31;
// a warp reads 32 consecutive rows of a column: conflict-free), split into
// A_hi / A_lo (K-major) and write the exact W row into TMEM accumulator
// t % 2 (tcgen05.st); thread 0 issues D += W_hi E_hi + W_lo E_hi + W_hi E_lo
// (24 MMAs, commit -> mbar[t % 2]); the epilogue of tile t - 1 then drains
// accumulator (t-1) % 2 (tcgen05.ld, one coalesced 128-byte store per warp and
// column) while the MMAs of tile t run.  E^T is staged once per CTA.
// ------------------------------------------------------------------------
constexpr int UT_NT = 256, UT_TM = 128, UT_NR = 4;
constexpr int UT_RAW_BYTES = UT_TM * 64 * 4;          // 32 KB
constexpr size_t update_tc_smem() {
    return (size_t)2 * 64 * 64 * 4 + (size_t)2 * UT_TM * 64 * 4 + (size_t)UT_NR * UT_RAW_BYTES + 1024;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])));
}

__global__ void __launch_bounds__(UT_NT, 1) k_pair_update_tc(JacobiRound<float> a, int tiles_per_cta) {
    extern __shared__ __align__(1024) unsigned char ut_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(ut_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char* Bh = sm;                       // E^T hi: 64 x 64 K-major (16 KB)
    unsigned char* Bl = sm + 16384;               // E^T lo
    unsigned char* Ah = sm + 32768;               // W tile hi: 128 x 64 K-major (32 KB)
    unsigned char* Al = sm + 65536;               // W tile lo
    float* ring = reinterpret_cast<float*>(sm + 98304);   // UT_NR raw tiles [64 cols][128 rows]
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ uint32_t tmem_base;
    __shared__ float* colp[64];
    const int pair = blockIdx.y, which = blockIdx.z;
    if (!a.flag[pair]) return;
    if (which && !a.has_v) return;
    const long long ld = which ? a.ldv : a.ldx;
    const long long rows_pad = which ? a.nv_pad : a.m_pad;
    const long long row_lo = (long long)blockIdx.x * tiles_per_cta * UT_TM;
    if (row_lo >= rows_pad) return;
    const long long row_hi = min(rows_pad, row_lo + (long long)tiles_per_cta * UT_TM);
    const int ntile = (int)((row_hi - row_lo + UT_TM - 1) / UT_TM);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int trow = tid & 127, half = tid >> 7;  // tile row (= TMEM lane) and column half of this thread
    const PairDesc<float> pd = a.pd[pair];
    const int w = pd.w0 + pd.w1;
    float* const s0 = which ? pd.v0 : pd.x0;
    float* const s1 = which ? pd.v1 : pd.x1;
    if (tid < 64) colp[tid] = tid < w ? (tid < pd.w0 ? s0 + (long long)tid * ld : s1 + (long long)(tid - pd.w0) * ld) : nullptr;
    if (warp == 0) tc::tmem_alloc<128>(&tmem_base);
    if (tid == 0) {
        tc::mbar_init(&mbar[0]);
        tc::mbar_init(&mbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    __syncthreads();                              // colp visible
    // raw tile t: 64 columns x 32 chunks of 4 rows; thread: 8 chunks (c = (tid + 256 u) / 32, rows 4 ((tid + 256 u) % 32))
    const uint32_t rbase = tc::smem_u32(ring);
    auto issue = [&](int t) {
        const int slot = t % UT_NR;
        const long long r0 = row_lo + (long long)t * UT_TM;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int f = tid + UT_NT * u;
            const int c = f >> 5, r4 = 4 * (f & 31);
            const float* p = colp[c];
            float* dst = ring + (size_t)slot * (UT_TM * 64) + c * UT_TM + r4;
            if (p && r0 + r4 < rows_pad) cp16(rbase + (uint32_t)(((size_t)slot * (UT_TM * 64) + c * UT_TM + r4) * 4), p + r0 + r4);
            else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
#pragma unroll
    for (int t = 0; t < UT_NR - 1; ++t) {
        if (t < ntile) issue(t);
        cp_commit();
    }
    // B = E^T: B[n][k] = E[k][n]; item (n, k4): float4 over k
    const float* Eg = a.E + (long long)pair * (64 * 64);
    for (int it = tid; it < 64 * 16; it += UT_NT) {
        const int n = it & 63, k4 = it >> 6;
        float4 v = make_float4(Eg[(4 * k4 + 0) * 64 + n], Eg[(4 * k4 + 1) * 64 + n], Eg[(4 * k4 + 2) * 64 + n],
                               Eg[(4 * k4 + 3) * 64 + n]);
        const uint32_t o = tc::koff(n, 4 * k4, 64);
        const float4 h = tc::hi4(v);
        *reinterpret_cast<float4*>(Bh + o) = h;
        *reinterpret_cast<float4*>(Bl + o) = tc::lo4(v, h);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    constexpr uint32_t SBO = 16 * 128;                  // 64 columns: 2048 B between 8-row groups
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    auto epilogue = [&](int t) {
        const long long row = row_lo + (long long)t * UT_TM + trow;
        const bool rok = row < rows_pad;
        const uint32_t acc = tmem + (uint32_t)(64 * (t & 1));
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += 16) {
            float d[16];
            tc::tmem_ld16(acc + lane_base + (uint32_t)(32 * half + c0), d);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int c = 32 * half + c0 + j;
                if (rok && c < w) {
                    float* p = c < pd.w0 ? s0 + (long long)c * ld : s1 + (long long)(c - pd.w0) * ld;
                    p[row] = d[j];
                }
            }
        }
    };
    for (int t = 0; t < ntile; ++t) {
        const int b = t & 1;
        cp_wait<UT_NR - 2>();                      // this thread's chunks of tile t
        __syncthreads();                           // everyone's chunks of tile t
        if (t >= 1) tc::mbar_wait(&mbar[b ^ 1], (uint32_t)(((t - 1) >> 1) & 1));   // MMAs of t - 1 done: A free
        tc::fence_after();
        // ---- transpose from the raw tile, split, W row -> TMEM accumulator b
        const float* raw = ring + (size_t)(t % UT_NR) * (UT_TM * 64);
#pragma unroll
        for (int g = 0; g < 2; ++g) {              // 16 columns at a time
            float wv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) wv[j] = raw[(32 * half + 16 * g + j) * UT_TM + trow];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 x = make_float4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
                const uint32_t o = tc::koff(trow, 32 * half + 16 * g + 4 * q, 64);
                const float4 h = tc::hi4(x);
                *reinterpret_cast<float4*>(Ah + o) = h;
                *reinterpret_cast<float4*>(Al + o) = tc::lo4(x, h);
            }
            tmem_st16(tmem + (uint32_t)(64 * b) + lane_base + (uint32_t)(32 * half + 16 * g), wv);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
        tc::fence_async_smem();
        tc::fence_before();
        __syncthreads();                           // A, TMEM b written; raw slot t % NR consumed
        // refill the ring: tile t + NR - 1 -> slot (t - 1) % NR (consumed last iteration)
        if (t + UT_NR - 1 < ntile) issue(t + UT_NR - 1);
        cp_commit();
        if (tid == 0) {
            tc::fence_after();
            const uint32_t ah = tc::smem_u32(Ah), al = tc::smem_u32(Al), bh = tc::smem_u32(Bh), bl = tc::smem_u32(Bl);
            const uint32_t acc = tmem + (uint32_t)(64 * b);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                tc::mma(acc, tc::sdesc(ah + ks * 256, 128, SBO), tc::sdesc(bh + ks * 256, 128, SBO), idesc, 1u);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                tc::mma(acc, tc::sdesc(al + ks * 256, 128, SBO), tc::sdesc(bh + ks * 256, 128, SBO), idesc, 1u);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                tc::mma(acc, tc::sdesc(ah + ks * 256, 128, SBO), tc::sdesc(bl + ks * 256, 128, SBO), idesc, 1u);
            tc::commit(&mbar[b]);
        }
        // ---- epilogue of tile t - 1 (accumulator b ^ 1) while the MMAs of tile t run
        if (t >= 1) epilogue(t - 1);
        tc::fence_before();
    }
    cp_wait<0>();
    if (ntile >= 1) {
        const int t = ntile - 1;
        tc::mbar_wait(&mbar[t & 1], (uint32_t)((t >> 1) & 1));
        tc::fence_after();
        epilogue(t);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<128>(tmem);
}

// ------------------------------------------------------------------------
// k_pair_update_tc_pdl: the update of k_pair_update_tc as a persistent
// kernel (one CTA per SM) launched as a programmatic dependent of the round's
// solve, so that it starts while slow pairs are still solving.  Work items
// (completion position p, X or V, group of UT_TPC tiles) are taken from a
// global counter in completion order; item p waits (acquire) until the p-th
// solved pair is published (k_pair_solve: E and flag written, then release),
// skips pairs that did not rotate, and runs the same pipeline as
// k_pair_update_tc on its rows.  mbarrier phases are tracked per CTA across
// items.  A consumer that waits too long sets dctr[2] and gives up (no hang).
// ------------------------------------------------------------------------
constexpr int UT_TPC = 16;

__device__ __forceinline__ void tma_load_2d(uint32_t sdst, const CUtensorMap* map, int c0, int c1, uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(sdst), "l"(map), "r"(c0), "r"(c1), "r"(tc::smem_u32(mbar))
        : "memory");
}



// TMA = true (U-route, X only): the raw tiles arrive by TMA (two 2-D boxes of 128 rows x 32 columns per tile,
// mbarrier complete_tx, ring slots tracked by a per-CTA running tile count) instead of 2048 16-byte cp.async
// per tile; columns / rows past the matrix are zero-filled (a bye block is addressed past the last column)
template <bool TMA>
__global__ void __launch_bounds__(UT_NT, 1) k_pair_update_tc_pdl(JacobiRound<float> a, int ngroups, int tpc,
                                                                  const __grid_constant__ CUtensorMap umap) {
    extern __shared__ __align__(1024) unsigned char ut_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(ut_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char* Bh = sm;
    unsigned char* Bl = sm + 16384;
    unsigned char* Ah = sm + 32768;
    unsigned char* Al = sm + 65536;
    float* ring = reinterpret_cast<float*>(sm + 98304);
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ __align__(8) uint64_t rfull[UT_NR];
    __shared__ uint32_t tmem_base;
    __shared__ float* colp[64];
    __shared__ int item[3];                     // pair, which, group (pair < 0: stop)
    const int tid = threadIdx.x, warp = tid >> 5;
    const int trow = tid & 127, half = tid >> 7;
    if (warp == 0) tc::tmem_alloc<128>(&tmem_base);
    if (tid == 0) {
        tc::mbar_init(&mbar[0]);
        tc::mbar_init(&mbar[1]);
        for (int q = 0; q < UT_NR; ++q) tc::mbar_init(&rfull[q]);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    constexpr uint32_t SBO = 16 * 128;
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    const uint32_t rbase = tc::smem_u32(ring);
    const long long total = (long long)a.npairs * 2 * ngroups;
    uint32_t ph[2] = {0u, 0u};                  // completed waits per accumulator barrier
    long long gt0 = 0;                          // TMA: raw tiles of the previous items (ring slot / parity)
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
                if ((long long)grp * tpc * UT_TM >= rows_pad) continue;
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
        const long long row_lo = (long long)grp * tpc * UT_TM;
        const long long row_hi = min(rows_pad, row_lo + (long long)tpc * UT_TM);
        const int ntile = (int)((row_hi - row_lo + UT_TM - 1) / UT_TM);
        const PairDesc<float> pd = a.pd[pair];
        const int w = pd.w0 + pd.w1;
        float* const s0 = which ? pd.v0 : pd.x0;
        float* const s1 = which ? pd.v1 : pd.x1;
        if (tid < 64) colp[tid] = tid < w ? (tid < pd.w0 ? s0 + (long long)tid * ld : s1 + (long long)(tid - pd.w0) * ld) : nullptr;
        __syncthreads();
        const int cI = TMA ? (int)((pd.x0 - a.tbase) / a.tld) : 0;
        const int cJ = TMA ? (pd.w1 > 0 ? (int)((pd.x1 - a.tbase) / a.tld) : (1 << 30)) : 0;
        auto issue = [&](int t) {
            if constexpr (TMA) {
                if (tid == 0) {
                    const int slot = (int)((gt0 + t) % UT_NR);
                    const int r0 = (int)(row_lo + (long long)t * UT_TM);
                    const uint32_t dst = rbase + (uint32_t)((size_t)slot * (UT_TM * 64) * 4);
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic reads of the slot done
                    mbar_expect_tx(&rfull[slot], (uint32_t)UT_RAW_BYTES);
                    tma_load_2d(dst, &umap, r0, cI, &rfull[slot]);
                    tma_load_2d(dst + 32 * UT_TM * 4, &umap, r0, cJ, &rfull[slot]);
                }
                return;
            }
            const int slot = t % UT_NR;
            const long long r0 = row_lo + (long long)t * UT_TM;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int f = tid + UT_NT * u;
                const int c = f >> 5, r4 = 4 * (f & 31);
                const float* p = colp[c];
                float* dst = ring + (size_t)slot * (UT_TM * 64) + c * UT_TM + r4;
                if (p && r0 + r4 < rows_pad) cp16(rbase + (uint32_t)(((size_t)slot * (UT_TM * 64) + c * UT_TM + r4) * 4), p + r0 + r4);
                else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
#pragma unroll
        for (int t = 0; t < UT_NR - 1; ++t) {
            if (t < ntile) issue(t);
            if constexpr (!TMA) cp_commit();
        }
        const float* Eg = a.E + (long long)pair * (64 * 64);
        for (int it = tid; it < 64 * 16; it += UT_NT) {
            const int n = it & 63, k4 = it >> 6;
            float4 v = make_float4(Eg[(4 * k4 + 0) * 64 + n], Eg[(4 * k4 + 1) * 64 + n], Eg[(4 * k4 + 2) * 64 + n],
                                   Eg[(4 * k4 + 3) * 64 + n]);
            const uint32_t o = tc::koff(n, 4 * k4, 64);
            const float4 h = tc::hi4(v);
            *reinterpret_cast<float4*>(Bh + o) = h;
            *reinterpret_cast<float4*>(Bl + o) = tc::lo4(v, h);
        }
        auto epilogue = [&](int t) {
            const long long row = row_lo + (long long)t * UT_TM + trow;
            const bool rok = row < rows_pad;
            const uint32_t acc = tmem + (uint32_t)(64 * (t & 1));
#pragma unroll
            for (int c0 = 0; c0 < 32; c0 += 16) {
                float d[16];
                tc::tmem_ld16(acc + lane_base + (uint32_t)(32 * half + c0), d);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int c = 32 * half + c0 + j;
                    if (rok && c < w) {
                        float* p = c < pd.w0 ? s0 + (long long)c * ld : s1 + (long long)(c - pd.w0) * ld;
                        p[row] = d[j];
                    }
                }
            }
        };
        for (int t = 0; t < ntile; ++t) {
            const int b = t & 1;
            if constexpr (TMA) {
                tc::mbar_wait(&rfull[(gt0 + t) % UT_NR], (uint32_t)(((gt0 + t) / UT_NR) & 1));
            } else {
                cp_wait<UT_NR - 2>();
                tc::fence_before();
                __syncthreads();
            }
            if (t >= 1) { tc::mbar_wait(&mbar[b ^ 1], ph[b ^ 1] & 1u); ++ph[b ^ 1]; }
            tc::fence_after();
            const float* raw = ring + (size_t)(TMA ? (gt0 + t) % UT_NR : t % UT_NR) * (UT_TM * 64);
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                float wv[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) wv[j] = raw[(32 * half + 16 * g + j) * UT_TM + trow];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 x = make_float4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
                    const uint32_t o = tc::koff(trow, 32 * half + 16 * g + 4 * q, 64);
                    const float4 h = tc::hi4(x);
                    *reinterpret_cast<float4*>(Ah + o) = h;
                    *reinterpret_cast<float4*>(Al + o) = tc::lo4(x, h);
                }
                tmem_st16(tmem + (uint32_t)(64 * b) + lane_base + (uint32_t)(32 * half + 16 * g), wv);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n");
            tc::fence_async_smem();
            tc::fence_before();
            __syncthreads();
            if (t + UT_NR - 1 < ntile) issue(t + UT_NR - 1);
            if constexpr (!TMA) cp_commit();
            if (tid == 0) {
                tc::fence_after();
                const uint32_t ah = tc::smem_u32(Ah), al = tc::smem_u32(Al), bh = tc::smem_u32(Bh), bl = tc::smem_u32(Bl);
                const uint32_t acc = tmem + (uint32_t)(64 * b);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    tc::mma(acc, tc::sdesc(ah + ks * 256, 128, SBO), tc::sdesc(bh + ks * 256, 128, SBO), idesc, 1u);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    tc::mma(acc, tc::sdesc(al + ks * 256, 128, SBO), tc::sdesc(bh + ks * 256, 128, SBO), idesc, 1u);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    tc::mma(acc, tc::sdesc(ah + ks * 256, 128, SBO), tc::sdesc(bl + ks * 256, 128, SBO), idesc, 1u);
                tc::commit(&mbar[b]);
            }
            if (t >= 1) epilogue(t - 1);
        }
        cp_wait<0>();
        if (ntile >= 1) {
            const int t = ntile - 1;
            tc::mbar_wait(&mbar[t & 1], ph[t & 1] & 1u);
            ++ph[t & 1];
            tc::fence_after();
            epilogue(t);
        }
        tc::fence_before();
        __syncthreads();                        // item done: smem, TMEM free for the next item
        gt0 += ntile;
    }
    if (warp == 0) tc::tmem_free<128>(tmem);
}

// ------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------
int launch_gram_sw_ta(const JacobiRound<float>& a, cudaStream_t st);   // TMEM-A Gram, defined with its kernel below
// Gram variants (KT rows per stage, ST stages, CTAs per SM); MPJSVD_GRAM_VARIANT selects one (experiments)
struct GramVariant {
    void (*fn)(JacobiRound<float>);
    size_t smem;
    int per_sm;
};
static const GramVariant g_gram_variants[] = {
    {k_pair_gram_tc<64, 3, 2>, gram_tc_smem<64, 3>(), 2},
    {k_pair_gram_tc<64, 6, 1>, gram_tc_smem<64, 6>(), 1},
    {k_pair_gram_tc<32, 6, 2>, gram_tc_smem<32, 6>(), 2},
    {k_pair_gram_tc<128, 3, 1>, gram_tc_smem<128, 3>(), 1},
    {k_pair_gram_tc<32, 4, 3>, gram_tc_smem<32, 4>(), 3},
    {k_pair_gram_tc<64, 4, 1>, gram_tc_smem<64, 4>(), 1},
};
static const GramVariant& gram_variant(int v) {
    if (v < 0 || v >= (int)(sizeof(g_gram_variants) / sizeof(g_gram_variants[0]))) v = 0;
    return g_gram_variants[v];
}

int make_update_tmap(void* out, const float* base, long long ld, long long rows_pad, long long cols) {
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(f);
    }
    if (!fn || ld % 4 != 0) return -1;
    const cuuint64_t gdim[2] = {(cuuint64_t)rows_pad, (cuuint64_t)cols};
    const cuuint64_t gstride[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {UT_TM, 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base),
                          gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

int make_gram_tmap_sw128(void* out, const float* base, long long ld, long long rows_pad, long long cols) {
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(f);
    }
    if (!fn || ld % 4 != 0) return -1;
    const cuuint64_t gdim[2] = {(cuuint64_t)rows_pad, (cuuint64_t)cols};
    const cuuint64_t gstride[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base),
                          gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

int launch_gram_tc(const JacobiRound<float>& a, cudaStream_t st) {
    if (a.smap && a.gram_variant >= 18 && a.gram_variant <= 26) return launch_gram_sw_ta(a, st);
    if (a.smap && a.gram_variant >= 10 && a.gram_variant <= 17) {
        const CUtensorMap& sm = *reinterpret_cast<const CUtensorMap*>(a.smap);
        switch (a.gram_variant) {
            case 11:
                MPJ_CUDA_TRY(set_smem(k_pair_gram_sw<4, 3>, gram_tma_smem<32, 4>()));
                k_pair_gram_sw<4, 3><<<dim3(a.nsplit, a.npairs), GT_NT, gram_tma_smem<32, 4>(), st>>>(a, sm);
                break;
            case 12:
                MPJ_CUDA_TRY(set_smem(k_pair_gram_sw<6, 2>, gram_tma_smem<32, 6>()));
                k_pair_gram_sw<6, 2><<<dim3(a.nsplit, a.npairs), GT_NT, gram_tma_smem<32, 6>(), st>>>(a, sm);
                break;
            case 13:
                MPJ_CUDA_TRY(set_smem(k_pair_gram_sw<8, 1>, gram_tma_smem<32, 8>()));
                k_pair_gram_sw<8, 1><<<dim3(a.nsplit, a.npairs), GT_NT, gram_tma_smem<32, 8>(), st>>>(a, sm);
                break;
            case 14:
                MPJ_CUDA_TRY(set_smem(k_pair_gram_sw<4, 3, 256>, gram_tma_smem<32, 4>()));
                k_pair_gram_sw<4, 3, 256><<<dim3(a.nsplit, a.npairs), 256, gram_tma_smem<32, 4>(), st>>>(a, sm);
                break;
            case 15:
                MPJ_CUDA_TRY(set_smem(k_pair_gram_sw<3, 4, 256>, gram_tma_smem<32, 3>()));
                k_pair_gram_sw<3, 4, 256><<<dim3(a.nsplit, a.npairs), 256, gram_tma_smem<32, 3>(), st>>>(a, sm);
                break;
            case 16:
                MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ws<4, 3>, gram_tma_smem<32, 4>()));
                k_pair_gram_sw_ws<4, 3><<<dim3(a.nsplit, a.npairs), 160, gram_tma_smem<32, 4>(), st>>>(a, sm);
                break;
            case 17:
                MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ws<6, 2>, gram_tma_smem<32, 6>()));
                k_pair_gram_sw_ws<6, 2><<<dim3(a.nsplit, a.npairs), 160, gram_tma_smem<32, 6>(), st>>>(a, sm);
                break;
            default:
                MPJ_CUDA_TRY(set_smem(k_pair_gram_sw<3, 4>, gram_tma_smem<32, 3>()));
                k_pair_gram_sw<3, 4><<<dim3(a.nsplit, a.npairs), GT_NT, gram_tma_smem<32, 3>(), st>>>(a, sm);
        }
        MPJ_LAUNCHED();
        return 0;
    }
    if (a.tmap) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_tma<64, 3, 2>, gram_tma_smem<64, 3>()));
        MPJ_CUDA_TRY(set_smem(k_pair_gram_tma<32, 3, 4>, gram_tma_smem<32, 3>()));
        if (a.gram_variant == 8 || a.gram_variant == 9) {
            // experiment: warp-specialised TMA Gram (8: 3 stages, 9: 4 stages at KT = 32 / 3 at KT = 64)
            const CUtensorMap& tm = *reinterpret_cast<const CUtensorMap*>(a.tmap);
            if (a.gram_kt == 32 && a.gram_variant == 9) {
                MPJ_CUDA_TRY(set_smem(k_pair_gram_tma_ws<32, 4, 3>, gram_tma_smem<32, 4>()));
                k_pair_gram_tma_ws<32, 4, 3><<<dim3(a.nsplit, a.npairs), GT_NT, gram_tma_smem<32, 4>(), st>>>(a, tm);
            } else if (a.gram_kt == 32) {
                MPJ_CUDA_TRY(set_smem(k_pair_gram_tma_ws<32, 3, 4>, gram_tma_smem<32, 3>()));
                k_pair_gram_tma_ws<32, 3, 4><<<dim3(a.nsplit, a.npairs), GT_NT, gram_tma_smem<32, 3>(), st>>>(a, tm);
            } else {
                MPJ_CUDA_TRY(set_smem(k_pair_gram_tma_ws<64, 3, 2>, gram_tma_smem<64, 3>()));
                k_pair_gram_tma_ws<64, 3, 2><<<dim3(a.nsplit, a.npairs), GT_NT, gram_tma_smem<64, 3>(), st>>>(a, tm);
            }
            MPJ_LAUNCHED();
            return 0;
        }
        if (a.gram_kt == 32)
            k_pair_gram_tma<32, 3, 4><<<dim3(a.nsplit, a.npairs), GT_NT, gram_tma_smem<32, 3>(), st>>>(
                a, *reinterpret_cast<const CUtensorMap*>(a.tmap));
        else
            k_pair_gram_tma<64, 3, 2><<<dim3(a.nsplit, a.npairs), GT_NT, gram_tma_smem<64, 3>(), st>>>(
                a, *reinterpret_cast<const CUtensorMap*>(a.tmap));
        MPJ_LAUNCHED();
        return 0;
    }
    const GramVariant& gv = gram_variant(a.gram_variant);
    MPJ_CUDA_TRY(set_smem(gv.fn, (size_t)(gv.smem)));
    static long long* dbg = nullptr;
    static long long calls = 0;
    const bool timing = (a.diag & 4) != 0;
    if (timing && !dbg) {
        cudaMalloc(&dbg, 8 * sizeof(long long));
        cudaMemset(dbg, 0, 8 * sizeof(long long));
        cudaMemcpyToSymbol(g_gram_dbg, &dbg, sizeof(dbg));
    }
    gv.fn<<<dim3(a.nsplit, a.npairs), GT_NT, gv.smem, st>>>(a);
    MPJ_LAUNCHED();
    if (timing && ++calls % 500 == 0) {
        long long hv[8];
        cudaMemcpy(hv, dbg, sizeof(hv), cudaMemcpyDeviceToHost);
        const double nt = hv[6] > 0 ? (double)hv[6] : 1.0;
        fprintf(stderr, "[gram timing] tiles=%lld per tile (cycles, warp 1): cp_wait=%.0f lo=%.0f bar=%.0f mma_issue=%.0f mbar_wait=%.0f refill=%.0f\n",
                hv[6], hv[0] / nt, hv[1] / nt, hv[2] / nt, hv[3] / nt, hv[4] / nt, hv[5] / nt);
    }
    return 0;
}

int launch_update_tc(const JacobiRound<float>& a, cudaStream_t st) {
    MPJ_CUDA_TRY(set_smem(k_pair_update_tc, (size_t)(update_tc_smem())));
    const long long rows_pad = a.m_pad > a.nv_pad ? a.m_pad : a.nv_pad;
    const long long tiles = (rows_pad + UT_TM - 1) / UT_TM;
    const int tpc = tiles >= 16 ? 16 : (int)tiles;
    const unsigned gx = (unsigned)((tiles + tpc - 1) / tpc);
    k_pair_update_tc<<<dim3(gx, a.npairs, a.has_v ? 2 : 1), UT_NT, update_tc_smem(), st>>>(a, tpc);
    MPJ_LAUNCHED();
    return 0;
}

int gram_tc_ctas_per_sm(long long rows_pad, int tma, int kt, int variant) {
    if (tma) {
        const int k = gram_tma_kt(rows_pad, kt);
        if ((variant == 9 && k == 32) || variant == 11 || variant == 14 || variant == 16 || variant == 18 || variant == 22 || variant == 23 || variant == 25) return 3;
        if (variant == 10 || variant == 15 || variant == 19) return 4;
        if (variant == 12 || variant == 17 || variant == 20 || variant == 21 || variant == 24 || variant == 26) return 2;
        if (variant == 13) return 1;
        return k == 32 ? 4 : 2;
    }
    // shared memory bound: (stages + alignment + static) per CTA of 228 KB per SM
    const GramVariant& gv = gram_variant(variant);
    const int per = (int)((228 * 1024) / (gv.smem + 2048));
    return per < gv.per_sm ? per : gv.per_sm;
}

}  // namespace mpj


namespace mpj {

// tcgen05.mma with the A operand in tensor memory (the "TS" form: A K-major, lane = M-row, one column per K element)
__device__ __forceinline__ void mma_ts(uint32_t dtmem, uint32_t atmem, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "r"(atmem), "l"(bd), "r"(idesc), "r"(acc));
}

// ------------------------------------------------------------------------
// k_pair_gram_sw_ta: the warp-specialised swizzled Gram (k_pair_gram_sw_ws) with the A operand [H ; L] in TENSOR
// MEMORY.  k_pair_gram_sw_ws is bound by shared-memory traffic (per 32-row tile: 8 KB landed by TMA, 8 KB read and
// 8 KB of lo parts written by the lo warps, 24 KB read by the MMAs: A = [H ; L] 16 KB + B = H 8 KB).  Here a stage is
// only the 8 KB of raw columns (B = H, read by the MMA through the same SWIZZLE_128B descriptor): thread m of the
// four conversion warps owns TMEM lane m = M-row m of A, reads its column's 32 rows (one swizzled 128-byte row,
// conflict-free 16-byte chunks), and writes hi (m < 64) or lo = x - hi (m >= 64) into the tile's A buffer with
// tcgen05.st (column = K element); the MMAs are the A-from-TMEM form (mma_ts).  No lo parts in shared memory, no
// async-proxy fence: 32 KB of shared-memory traffic per tile instead of 48, and GM_ST stages of 8 KB instead of
// 16 KB (twice the tiles in flight in the same footprint).  A is double buffered (TMEM columns 64..95 / 96..127
// next to the 64 accumulator columns; 128 allocated): the conversion of tile t waits for the MMAs of tile t - 2.
// Same products in the same order as k_pair_gram_sw_ws: bitwise equal on equal row sets.
// ------------------------------------------------------------------------
template <int GM_ST, int MINB, int NA, int LAG = 1, int CG = 1>
__global__ void __launch_bounds__(32 + 128 * CG, MINB) k_pair_gram_sw_ta(JacobiRound<float> a, const __grid_constant__ CUtensorMap smap) {
    constexpr int KT = 32, NT = 32 + 128 * CG;          // warp 0: TMA + MMA lane; CG groups of 4 conversion warps
    constexpr int STAGE = 64 * KT * 4;                  // 8 KB: raw I | raw J, 4 KB each
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    reset_publication(a);
    gram_pdl_begin(a);
    if (pair_unchanged(a, a.pd[blockIdx.y])) return;
    extern __shared__ __align__(1024) unsigned char gta_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gta_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[GM_ST], done[GM_ST], a_ready[NA], fin;
    __shared__ uint32_t tmem_base;
    const int pair = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5;
    const PairDesc<float> pd = a.pd[pair];
    const int cI = (int)((pd.x0 - a.tbase) / a.tld), cJ = (int)((pd.x1 - a.tbase) / a.tld);
    const bool hasJ = pd.w1 > 0;
    const uint32_t tx = hasJ ? 2u * 32u * KT * 4u : 32u * KT * 4u;
    constexpr int TCOLS = 64 + 32 * NA <= 128 ? 128 : 256;   // accumulator + NA A buffers of 32 columns
    static_assert(64 + 32 * NA <= 256, "TMEM columns");
    if (warp == 0) tc::tmem_alloc<TCOLS>(&tmem_base);
    if (tid == 0) {
        for (int s = 0; s < GM_ST; ++s) {
            tc::mbar_init(&full[s]);
            tc::mbar_init(&done[s]);
        }
        for (int q = 0; q < NA; ++q) mbar_init_n(&a_ready[q], 128);
        tc::mbar_init(&fin);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    if (!hasJ) {   // bye pair: N-rows 32..63 (raw J) stay zero in every stage
        for (int s = 0; s < GM_ST; ++s)
            for (int i = tid; i < 4096 / 16; i += NT)
                reinterpret_cast<float4*>(sm + (size_t)s * STAGE + 4096)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        tc::fence_async_smem();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;                    // columns [0, 64): accumulator; then NA A buffers of 32
    const bool il = a.gram_il != 0;
    const long long rbeg = il ? (long long)split * KT : (long long)split * a.rows_per_split;
    const long long rend = il ? (long long)a.m_pad : min(rbeg + (long long)a.rows_per_split, (long long)a.m_pad);
    const long long rstep = il ? (long long)a.nsplit * KT : (long long)KT;
    const int ntile = rend > rbeg ? (int)((rend - rbeg + rstep - 1) / rstep) : 0;
    const uint32_t sbase = tc::smem_u32(sm);
    auto issue = [&](int t) {
        const int s = t % GM_ST;
        const int r0 = (int)(rbeg + (long long)t * rstep);
        mbar_expect_tx(&full[s], tx);
        tma_load_2d_g(sbase + (uint32_t)(s * STAGE), &smap, r0, cI, &full[s]);
        if (hasJ) tma_load_2d_g(sbase + (uint32_t)(s * STAGE) + 4096, &smap, r0, cJ, &full[s]);
    };
    if (warp == 0) {
        if (tid == 0) {
            for (int t = 0; t < GM_ST && t < ntile; ++t) issue(t);
            for (int t = 0; t < ntile; ++t) {
                const int s = t % GM_ST, ab = t % NA;
                tc::mbar_wait(&a_ready[ab], (uint32_t)((t / NA) & 1));
                tc::fence_after();
                const uint32_t base = sbase + (uint32_t)(s * STAGE);
                const uint32_t abuf = tmem + 64u + 32u * (uint32_t)ab;
#pragma unroll
                for (int ks = 0; ks < KT / 8; ++ks)
                    mma_ts(tmem, abuf + (uint32_t)(8 * ks), sdesc_sw128(base + ks * 32), idesc, (t > 0 || ks > 0) ? 1u : 0u);
                tc::commit(&done[s]);
                // refill the stage of tile t - LAG: with LAG = 1 this lane waits for the completion of the MMAs it
                // issued one iteration ago (issue -> mbarrier latency on the critical path of every tile); LAG >= 2
                // finds them complete, at the price of LAG - 1 tiles of prefetch distance
                if (t >= LAG && t - LAG + GM_ST < ntile) {
                    const int sp = (t - LAG) % GM_ST;
                    tc::mbar_wait(&done[sp], (uint32_t)(((t - LAG) / GM_ST) & 1));
                    issue(t - LAG + GM_ST);
                }
            }
            if (ntile > 0) tc::commit(&fin);
        }
        __syncwarp();
    } else {
        // conversion warps (CG groups of four; group g takes the tiles t = g, g + CG, ...): warp w may touch TMEM
        // lanes 32 (w % 4) .. + 31
        const int grp = (warp - 1) >> 2;
        const int m = 32 * (warp & 3) + (tid & 31);       // M-row of A = TMEM lane
        const int c = m & 63;                             // column of W = [X_I X_J]
        const bool lo = m >= 64;
        const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
        for (int t = grp; t < ntile; t += CG) {
            const int s = t % GM_ST, ab = t % NA;
            const unsigned char* row = sm + (size_t)s * STAGE + c * 128;
            if (t >= NA) {                                // the MMAs of tile t - NA have read this A buffer
                tc::mbar_wait(&done[(t - NA) % GM_ST], (uint32_t)(((t - NA) / GM_ST) & 1));
                tc::fence_after();
            }
            tc::mbar_wait(&full[s], (uint32_t)((t / GM_ST) & 1));
            float4 x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = *reinterpret_cast<const float4*>(row + ((j ^ (c & 7)) << 4));
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                float v[16];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 xv = x[4 * g + j];
                    const float4 h = tc::hi4(xv);
                    const float4 o = lo ? tc::lo4(xv, h) : h;
                    v[4 * j + 0] = o.x; v[4 * j + 1] = o.y; v[4 * j + 2] = o.z; v[4 * j + 3] = o.w;
                }
                tmem_st16(tmem + lane_base + 64u + 32u * (uint32_t)ab + 16u * (uint32_t)g, v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n");
            tc::fence_before();
            mbar_arrive(&a_ready[ab]);
        }
    }
    float* out = a.partial + ((long long)pair * a.nsplit + split) * (64 * 64);
    float* red = reinterpret_cast<float*>(sm);
    if (ntile > 0) {
        tc::mbar_wait(&fin, 0);
        tc::fence_after();
        __syncthreads();                           // every stage consumed before red (stage 0..) is overwritten
        if (tid < 128) {                           // TMEM lanes 0..127: warps 0..3
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 16) {
                float v[16];
                tc::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) red[tid * 65 + c0 + j] = v[j];
            }
        }
        __syncthreads();
        for (int e = tid; e < 64 * 64; e += NT) {
            const int p = e >> 6, q = e & 63;
            out[e] = red[p * 65 + q] + red[(64 + p) * 65 + q] + red[(64 + q) * 65 + p];
        }
    } else {
        for (int e = tid; e < 64 * 64; e += NT) out[e] = 0.f;
    }
    gram_pdl_end(a, pair);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<TCOLS>(tmem);
}

template <int ST>
constexpr size_t gram_ta_smem() { return (size_t)ST * 8192 + 1024; }

// launcher of the TMEM-A Gram (gram_variant 18: 8 stages at 3 CTAs/SM, 2 A buffers; 19: 6 stages at 4 CTAs/SM;
// 20 / 21: 12 / 8 stages at 2 CTAs/SM with 6 A buffers (256 TMEM columns))
int launch_gram_sw_ta(const JacobiRound<float>& a, cudaStream_t st) {
    const CUtensorMap& sm = *reinterpret_cast<const CUtensorMap*>(a.smap);
    if (a.gram_variant == 19) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ta<6, 4, 2>, gram_ta_smem<6>()));
        k_pair_gram_sw_ta<6, 4, 2><<<dim3(a.nsplit, a.npairs), 160, gram_ta_smem<6>(), st>>>(a, sm);
    } else if (a.gram_variant == 20) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ta<12, 2, 6>, gram_ta_smem<12>()));
        k_pair_gram_sw_ta<12, 2, 6><<<dim3(a.nsplit, a.npairs), 160, gram_ta_smem<12>(), st>>>(a, sm);
    } else if (a.gram_variant == 21) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ta<8, 2, 6>, gram_ta_smem<8>()));
        k_pair_gram_sw_ta<8, 2, 6><<<dim3(a.nsplit, a.npairs), 160, gram_ta_smem<8>(), st>>>(a, sm);
    } else if (a.gram_variant == 22) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ta<8, 3, 2, 2>, gram_ta_smem<8>()));
        k_pair_gram_sw_ta<8, 3, 2, 2><<<dim3(a.nsplit, a.npairs), 160, gram_ta_smem<8>(), st>>>(a, sm);
    } else if (a.gram_variant == 23) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ta<8, 3, 2, 3>, gram_ta_smem<8>()));
        k_pair_gram_sw_ta<8, 3, 2, 3><<<dim3(a.nsplit, a.npairs), 160, gram_ta_smem<8>(), st>>>(a, sm);
    } else if (a.gram_variant == 25) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ta<8, 3, 2, 1, 2>, gram_ta_smem<8>()));
        k_pair_gram_sw_ta<8, 3, 2, 1, 2><<<dim3(a.nsplit, a.npairs), 288, gram_ta_smem<8>(), st>>>(a, sm);
    } else if (a.gram_variant == 26) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ta<12, 2, 6, 1, 2>, gram_ta_smem<12>()));
        k_pair_gram_sw_ta<12, 2, 6, 1, 2><<<dim3(a.nsplit, a.npairs), 288, gram_ta_smem<12>(), st>>>(a, sm);
    } else if (a.gram_variant == 24) {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ta<12, 2, 6, 3>, gram_ta_smem<12>()));
        k_pair_gram_sw_ta<12, 2, 6, 3><<<dim3(a.nsplit, a.npairs), 160, gram_ta_smem<12>(), st>>>(a, sm);
    } else {
        MPJ_CUDA_TRY(set_smem(k_pair_gram_sw_ta<8, 3, 2>, gram_ta_smem<8>()));
        k_pair_gram_sw_ta<8, 3, 2><<<dim3(a.nsplit, a.npairs), 160, gram_ta_smem<8>(), st>>>(a, sm);
    }
    MPJ_LAUNCHED();
    return 0;
}

// ------------------------------------------------------------------------
// k_pair_update_tc_ts: k_pair_update_tc_pdl with the A operand (W_hi, W_lo) in TENSOR MEMORY instead of shared
// memory (tcgen05.mma ... [d], [a_tmem], b_desc: the "TS" form, A K-major, lane = row, one column per
// K element).  Each thread already holds its row of the tile after the transposition read, so it writes
// W_hi, W_lo and the exact W with tcgen05.st (no shared-memory A, no async-proxy fence for it); A is double
// buffered in TMEM (2 x 128 columns next to the 2 x 64 accumulator columns, 512 allocated), so tile t + 1 is
// transposed while the MMAs of tile t run and the MMAs of tile t - 1 are only waited for right before the
// epilogue of t - 1.  Shared memory holds only E^T (hi, lo) and a UTS_NR-deep raw ring.  Same products in the
// same order as k_pair_update_tc_pdl (bitwise equal).
// ------------------------------------------------------------------------
constexpr int UTS_NR = 6;
constexpr size_t update_ts_smem() { return 32768 + (size_t)UTS_NR * UT_RAW_BYTES + 1024; }


template <bool TMA>
__global__ void __launch_bounds__(UT_NT, 1) k_pair_update_tc_ts(JacobiRound<float> a, int ngroups, int tpc,
                                                                 const __grid_constant__ CUtensorMap umap) {
    extern __shared__ __align__(1024) unsigned char uts_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(uts_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char* Bh = sm;
    unsigned char* Bl = sm + 16384;
    float* ring = reinterpret_cast<float*>(sm + 32768);
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ __align__(8) uint64_t rfull[UTS_NR];
    __shared__ uint32_t tmem_base;
    __shared__ float* colp[64];
    __shared__ int item[3];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int trow = tid & 127, half = tid >> 7;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
    if (tid == 0) {
        tc::mbar_init(&mbar[0]);
        tc::mbar_init(&mbar[1]);
        for (int q = 0; q < UTS_NR; ++q) tc::mbar_init(&rfull[q]);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base;                 // columns [0, 128): accumulators; [128, 384): A buffers
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    constexpr uint32_t SBO = 16 * 128;
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    const uint32_t rbase = tc::smem_u32(ring);
    const long long total = (long long)a.npairs * 2 * ngroups;
    uint32_t ph[2] = {0u, 0u};
    long long gt0 = 0;
    while (true) {
        if (tid == 0) {
            int pair = -1, which = 0, grp = 0;
            while (true) {
                const long long wk = atomicAdd(a.dctr + 1, 1);
                if (wk >= total) break;
                int p, rem;
                if (a.upd_order) {   // tile group major, bottom group first (the rows the Gram read last)
                    p = (int)(wk % a.npairs);
                    rem = (int)(wk / a.npairs);
                    which = rem / ngroups;
                    grp = ngroups - 1 - rem % ngroups;
                } else {
                    p = (int)(wk / (2 * ngroups));
                    rem = (int)(wk % (2 * ngroups));
                    which = rem / ngroups;
                    grp = rem % ngroups;
                }
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
                if ((long long)grp * tpc * UT_TM >= rows_pad) continue;
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
        const long long row_lo = (long long)grp * tpc * UT_TM;
        const long long row_hi = min(rows_pad, row_lo + (long long)tpc * UT_TM);
        const int ntile = (int)((row_hi - row_lo + UT_TM - 1) / UT_TM);
        const PairDesc<float> pd = a.pd[pair];
        const int w = pd.w0 + pd.w1;
        float* const s0 = which ? pd.v0 : pd.x0;
        float* const s1 = which ? pd.v1 : pd.x1;
        if (tid < 64) colp[tid] = tid < w ? (tid < pd.w0 ? s0 + (long long)tid * ld : s1 + (long long)(tid - pd.w0) * ld) : nullptr;
        __syncthreads();
        const int cI = TMA ? (int)((pd.x0 - a.tbase) / a.tld) : 0;
        const int cJ = TMA ? (pd.w1 > 0 ? (int)((pd.x1 - a.tbase) / a.tld) : (1 << 30)) : 0;
        auto issue = [&](int t) {
            if constexpr (TMA) {
                if (tid == 0) {
                    const int slot = (int)((gt0 + t) % UTS_NR);
                    const int r0 = (int)(row_lo + (long long)t * UT_TM);
                    const uint32_t dst = rbase + (uint32_t)((size_t)slot * (UT_TM * 64) * 4);
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    mbar_expect_tx(&rfull[slot], (uint32_t)UT_RAW_BYTES);
                    tma_load_2d(dst, &umap, r0, cI, &rfull[slot]);
                    tma_load_2d(dst + 32 * UT_TM * 4, &umap, r0, cJ, &rfull[slot]);
                }
                return;
            }
            const int slot = t % UTS_NR;
            const long long r0 = row_lo + (long long)t * UT_TM;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int f = tid + UT_NT * u;
                const int c = f >> 5, r4 = 4 * (f & 31);
                const float* p = colp[c];
                float* dst = ring + (size_t)slot * (UT_TM * 64) + c * UT_TM + r4;
                if (p && r0 + r4 < rows_pad) cp16(rbase + (uint32_t)(((size_t)slot * (UT_TM * 64) + c * UT_TM + r4) * 4), p + r0 + r4);
                else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
#pragma unroll
        for (int t = 0; t < UTS_NR - 1; ++t) {
            if (t < ntile) issue(t);
            if constexpr (!TMA) cp_commit();
        }
        const float* Eg = a.E + (long long)pair * (64 * 64);
        {
            // all 16 loads of a thread in flight before the first conversion (one L2 latency per item, not four)
            constexpr int EQ = 64 * 16 / UT_NT;
            float4 v[EQ];
#pragma unroll
            for (int q = 0; q < EQ; ++q) {
                const int it = tid + UT_NT * q, n = it & 63, k4 = it >> 6;
                v[q] = make_float4(__ldcg(Eg + (4 * k4 + 0) * 64 + n), __ldcg(Eg + (4 * k4 + 1) * 64 + n),
                                   __ldcg(Eg + (4 * k4 + 2) * 64 + n), __ldcg(Eg + (4 * k4 + 3) * 64 + n));
            }
#pragma unroll
            for (int q = 0; q < EQ; ++q) {
                const int it = tid + UT_NT * q, n = it & 63, k4 = it >> 6;
                const uint32_t o = tc::koff(n, 4 * k4, 64);
                const float4 h = tc::hi4(v[q]);
                *reinterpret_cast<float4*>(Bh + o) = h;
                *reinterpret_cast<float4*>(Bl + o) = tc::lo4(v[q], h);
            }
        }
        tc::fence_async_smem();                  // E^T (generic stores) -> visible to the MMA (async proxy)
        auto epilogue = [&](int t) {
            const long long row = row_lo + (long long)t * UT_TM + trow;
            const bool rok = row < rows_pad;
            const uint32_t acc = tmem + (uint32_t)(64 * (t & 1));
#pragma unroll
            for (int c0 = 0; c0 < 32; c0 += 16) {
                float d[16];
                tc::tmem_ld16(acc + lane_base + (uint32_t)(32 * half + c0), d);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int c = 32 * half + c0 + j;
                    if (rok && c < w) {
                        float* p = c < pd.w0 ? s0 + (long long)c * ld : s1 + (long long)(c - pd.w0) * ld;
                        p[row] = d[j];
                    }
                }
            }
        };
        for (int t = 0; t < ntile; ++t) {
            const int b = t & 1;
            if constexpr (TMA) {
                tc::mbar_wait(&rfull[(gt0 + t) % UTS_NR], (uint32_t)(((gt0 + t) / UTS_NR) & 1));
            } else {
                cp_wait<UTS_NR - 2>();
                __syncthreads();
            }
            const float* raw = ring + (size_t)(TMA ? (gt0 + t) % UTS_NR : t % UTS_NR) * (UT_TM * 64);
            const uint32_t ahi = tmem + 128u + 128u * (uint32_t)b, alo = ahi + 64u;
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                float wv[16], hv[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) wv[j] = raw[(32 * half + 16 * g + j) * UT_TM + trow];
                const uint32_t col = lane_base + (uint32_t)(32 * half + 16 * g);
                tmem_st16(tmem + (uint32_t)(64 * b) + col, wv);     // exact W: D = W + W E
#pragma unroll
                for (int j = 0; j < 16; ++j) hv[j] = tc::hi_part(wv[j]);
                tmem_st16(ahi + col, hv);
#pragma unroll
                for (int j = 0; j < 16; ++j) wv[j] -= hv[j];
                tmem_st16(alo + col, wv);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n");
            tc::fence_before();
            __syncthreads();                    // A, W of tile t in TMEM; raw slot of tile t - 1 free
            if (t + UTS_NR - 1 < ntile) issue(t + UTS_NR - 1);
            if constexpr (!TMA) cp_commit();
            if (tid == 0) {
                tc::fence_after();
                const uint32_t bh = tc::smem_u32(Bh), bl = tc::smem_u32(Bl);
                const uint32_t acc = tmem + (uint32_t)(64 * b);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    mma_ts(acc, ahi + (uint32_t)(8 * ks), tc::sdesc(bh + ks * 256, 128, SBO), idesc, 1u);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    mma_ts(acc, alo + (uint32_t)(8 * ks), tc::sdesc(bh + ks * 256, 128, SBO), idesc, 1u);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    mma_ts(acc, ahi + (uint32_t)(8 * ks), tc::sdesc(bl + ks * 256, 128, SBO), idesc, 1u);
                tc::commit(&mbar[b]);
            }
            if (t >= 1) {
                tc::mbar_wait(&mbar[b ^ 1], ph[b ^ 1] & 1u);
                ++ph[b ^ 1];
                tc::fence_after();
                epilogue(t - 1);
            }
        }
        if constexpr (!TMA) cp_wait<0>();
        if (ntile >= 1) {
            const int t = ntile - 1;
            tc::mbar_wait(&mbar[t & 1], ph[t & 1] & 1u);
            ++ph[t & 1];
            tc::fence_after();
            epilogue(t);
        }
        tc::fence_before();
        __syncthreads();
        gt0 += ntile;
    }
    if (warp == 0) tc::tmem_free<512>(tmem);
}

}  // namespace mpj

namespace mpj {
int launch_update_tc_pdl(const JacobiRound<float>& a, cudaStream_t st) {
    const bool ts = a.update_ts != 0;
    if (ts) {
        MPJ_CUDA_TRY(set_smem(k_pair_update_tc_ts<true>, update_ts_smem()));
        MPJ_CUDA_TRY(set_smem(k_pair_update_tc_ts<false>, update_ts_smem()));
    } else {
        MPJ_CUDA_TRY(set_smem(k_pair_update_tc_pdl<true>, (size_t)(update_tc_smem())));
        MPJ_CUDA_TRY(set_smem(k_pair_update_tc_pdl<false>, (size_t)(update_tc_smem())));
    }
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long rows_pad = a.m_pad > a.nv_pad ? a.m_pad : a.nv_pad;
    // tiles per work item: the largest power of two <= UT_TPC that still gives every SM about three items
    // (the dynamic claim then balances the CTAs; smaller items cost a pipeline ramp each).  Measured on
    // B200: C3 (64 pairs x 4096 rows) 16 -> 4 tiles: 0.453 -> 0.437 s; C5 keeps 16
    int tpc = UT_TPC;
    while (tpc > 2 && (long long)a.npairs * (a.has_v ? 2 : 1) * ((rows_pad + (long long)tpc * UT_TM - 1) / ((long long)tpc * UT_TM)) < 3LL * nsm)
        tpc >>= 1;
    if (a.update_tpc > 0) tpc = a.update_tpc;    // options.update_tpc (experiments)
    const int ngroups = (int)((rows_pad + (long long)tpc * UT_TM - 1) / ((long long)tpc * UT_TM));
    const long long items = (long long)a.npairs * 2 * ngroups;
    const unsigned grid = (unsigned)(items < nsm ? items : nsm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(UT_NT);
    cfg.dynamicSmemBytes = update_tc_smem();
    cfg.stream = st;
    cudaLaunchAttribute attr1[1];
    attr1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr1[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr1;
    cfg.numAttrs = 1;
    CUtensorMap dummy;
    memset(&dummy, 0, sizeof(dummy));
    cudaError_t e;
    if (ts) {
        cfg.dynamicSmemBytes = update_ts_smem();
        if (a.umap && !a.has_v)
            e = cudaLaunchKernelEx(&cfg, k_pair_update_tc_ts<true>, a, ngroups, tpc, *reinterpret_cast<const CUtensorMap*>(a.umap));
        else
            e = cudaLaunchKernelEx(&cfg, k_pair_update_tc_ts<false>, a, ngroups, tpc, dummy);
    } else if (a.umap && !a.has_v)
        e = cudaLaunchKernelEx(&cfg, k_pair_update_tc_pdl<true>, a, ngroups, tpc, *reinterpret_cast<const CUtensorMap*>(a.umap));
    else
        e = cudaLaunchKernelEx(&cfg, k_pair_update_tc_pdl<false>, a, ngroups, tpc, dummy);
    MPJ_LAUNCHED();
    if (e != cudaSuccess) {
        mpj_record_cuda_error(e, "cudaLaunchKernelEx(update pdl)", __FILE__, __LINE__);
        return -4;
    }
    return 0;
}
}  // namespace mpj
