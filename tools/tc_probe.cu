// tc_probe.cu -- validates the tcgen05 (kind::tf32) building blocks used by
// the fp32 Jacobi kernels: shared-memory matrix descriptors (SWIZZLE_NONE,
// K-major and MN-major canonical layouts), the instruction descriptor, TMEM
// alloc / 32x32b loads, and tcgen05.commit -> mbarrier completion.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu && tools/tc_probe
//
// D[m][n] = sum_k A[m][k] B[n][k] for M = 128, N = 64, K = 64 (one CTA, 128
// threads), operands staged from fp32 by the threads in either layout; the
// result is compared with a double reference on tf32-truncated inputs.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
    uint64_t d = (uint64_t)layout << 61;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;                 // descriptor version 1 (sm_100)
    return d;                               // base offset 0, SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

// layout offsets (bytes) of element (r, k) of an R x KK operand
__device__ __forceinline__ uint32_t off_kmajor(int r, int k, int KK) {   // core 8 rows x 4 k (16 B rows)
    return (uint32_t)(((r >> 3) * (KK >> 2) + (k >> 2)) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint32_t off_mnmajor(int r, int k, int R) {   // core 4 r (16 B) x 8 k
    return (uint32_t)((r >> 2) * 128 + (k >> 3) * (R >> 2) * 128 + (k & 7) * 16 + (r & 3) * 4);
}

// MN-major SWIZZLE_128B: atom = 8 k-rows x 128 B (32 elements along MN), 16 B chunks XOR (k % 8);
// MN atoms at stride LBO = 1024 B, k atoms (8 k) at stride SBO = (R/32) * 1024 B
__device__ __forceinline__ uint32_t off_mn_sw128(int r, int k, int R) {
    return (uint32_t)((r >> 5) * 1024 + (k >> 3) * (R >> 5) * 1024 + (k & 7) * 128 + ((((r & 31) >> 2) ^ (k & 7)) << 4) +
                      (r & 3) * 4);
}

__global__ void k_probe(const float* A, const float* B, float* D, int mode) {
    const int mn_major = mode > 0;
    extern __shared__ __align__(1024) float dyn_raw[];
    float* dyn = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(dyn_raw) + 1023) & ~(uintptr_t)1023);
    float* As = dyn;
    float* Bs = dyn + M * K;
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    char* as = reinterpret_cast<char*>(As);
    char* bs = reinterpret_cast<char*>(Bs);
    for (int e = tid; e < M * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        const uint32_t o = mode == 3 ? off_mn_sw128(r, k, M) : mn_major ? off_mnmajor(r, k, M) : off_kmajor(r, k, K);
        *reinterpret_cast<float*>(as + o) = A[r * K + k];
    }
    for (int e = tid; e < N * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        const uint32_t o = mode == 3 ? off_mn_sw128(r, k, N) : mn_major ? off_mnmajor(r, k, N) : off_kmajor(r, k, K);
        *reinterpret_cast<float*>(bs + o) = B[r * K + k];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "n"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = idesc_tf32(M, N, mn_major, mn_major);
        for (int ks = 0; ks < K / 8; ++ks) {
            uint64_t ad, bd;
            if (mn_major) {
                // SBO: stride between 4-element groups along M/N (128 B); LBO: between 8-k groups
                if (mode == 3) {
                    ad = make_sdesc(smem_u32(as) + ks * (M / 32) * 1024, 1024, (M / 32) * 1024, 2);
                    bd = make_sdesc(smem_u32(bs) + ks * (N / 32) * 1024, 1024, (N / 32) * 1024, 2);
                } else if (mode == 1) {
                    ad = make_sdesc(smem_u32(as) + ks * (M / 4) * 128, (M / 4) * 128, 128);
                    bd = make_sdesc(smem_u32(bs) + ks * (N / 4) * 128, (N / 4) * 128, 128);
                } else {
                    ad = make_sdesc(smem_u32(as) + ks * (M / 4) * 128, 128, (M / 4) * 128);
                    bd = make_sdesc(smem_u32(bs) + ks * (N / 4) * 128, 128, (N / 4) * 128);
                }
            } else {
                // LBO: stride between the two 4-k core matrices (128 B); SBO: between 8-row groups
                ad = make_sdesc(smem_u32(as) + ks * 256, 128, (K / 4) * 128);
                bd = make_sdesc(smem_u32(bs) + ks * 256, 128, (K / 4) * 128);
            }
            mma_tf32(tbase, ad, bd, idesc, ks > 0);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&mbar)));
    }
    // wait for the MMA
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                : "=r"(done)
                : "r"(smem_u32(&mbar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // lane = row: warp w reads rows 32w..32w+31, 16 columns at a time
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        for (int j = 0; j < 16; ++j) D[tid * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(64));
}

// M = 64 probe: A rows 0..63 only; read all 128 TMEM lanes x 64 columns
__global__ void k_probe_m64(const float* A, const float* B, float* D) {
    extern __shared__ __align__(1024) float dyn_raw[];
    float* dyn = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(dyn_raw) + 1023) & ~(uintptr_t)1023);
    float* As = dyn;
    float* Bs = dyn + 64 * K;
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    char* as = reinterpret_cast<char*>(As);
    char* bs = reinterpret_cast<char*>(Bs);
    for (int e = tid; e < 64 * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<float*>(as + off_kmajor(r, k, K)) = A[r * K + k];
    }
    for (int e = tid; e < N * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<float*>(bs + off_kmajor(r, k, K)) = B[r * K + k];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = tmem_base;
    // zero the accumulator region first (all 128 lanes) so untouched lanes read 0
    for (int c0 = 0; c0 < N; c0 += 16) {
        const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + c0;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr), "r"(0u));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (tid == 0) {
        const uint32_t idesc = idesc_tf32(64, N, 0, 0);
        for (int ks = 0; ks < K / 8; ++ks) {
            uint64_t ad = make_sdesc(smem_u32(as) + ks * 256, 128, (K / 4) * 128);
            uint64_t bd = make_sdesc(smem_u32(bs) + ks * 256, 128, (K / 4) * 128);
            mma_tf32(tbase, ad, bd, idesc, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)));
    }
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        for (int j = 0; j < 16; ++j) D[tid * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(64));
}

static float tf32_trunc(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xffffe000u;
    float y;
    memcpy(&y, &u, 4);
    return y;
}

int main() {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    srand(1);
    for (auto& x : A) x = (float)rand() / RAND_MAX - 0.5f;
    for (auto& x : B) x = (float)rand() / RAND_MAX - 0.5f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    int fails = 0;
    for (int mn = 0; mn < 4; ++mn) {
        cudaMemset(dD, 0, D.size() * 4);
        cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (M + N) * K * 4 + 1024);
        k_probe<<<1, 128, (M + N) * K * 4 + 1024>>>(dA, dB, dD, mn);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("layout %s: CUDA error %s\n", mn ? "MN" : "K", cudaGetErrorString(e)); return 2; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0, maxerr_t = 0, scale = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0, reft = 0;
                for (int k = 0; k < K; ++k) {
                    ref += (double)A[m * K + k] * B[n * K + k];
                    reft += (double)tf32_trunc(A[m * K + k]) * tf32_trunc(B[n * K + k]);
                }
                maxerr = fmax(maxerr, fabs(D[m * N + n] - ref));
                maxerr_t = fmax(maxerr_t, fabs(D[m * N + n] - reft));
                scale = fmax(scale, fabs(ref));
            }
        printf("mode %d layout %s-major: max|D-ref| = %.3e  max|D-ref(tf32-truncated)| = %.3e  (scale %.3f)  D[0]=%g D[last]=%g\n",
               mn, mn ? "MN" : "K", maxerr, maxerr_t, scale, D[0], D[M * N - 1]);
        if (!(maxerr_t < 1e-4 * scale)) ++fails;
    }
    // M = 64: where does row i of D land?
    {
        cudaMemset(dD, 0, D.size() * 4);
        cudaFuncSetAttribute(k_probe_m64, cudaFuncAttributeMaxDynamicSharedMemorySize, (64 + N) * K * 4 + 1024);
        k_probe_m64<<<1, 128, (64 + N) * K * 4 + 1024>>>(dA, dB, dD);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("m64: CUDA error %s\n", cudaGetErrorString(e)); return 2; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int found = 0;
        for (int lane = 0; lane < 128; ++lane) {
            // match lane's row against reference rows of A (tf32)
            int match = -1;
            for (int i = 0; i < 64 && match < 0; ++i) {
                double err = 0, sc = 0;
                for (int n = 0; n < N; ++n) {
                    double ref = 0;
                    for (int k = 0; k < K; ++k) ref += (double)tf32_trunc(A[i * K + k]) * tf32_trunc(B[n * K + k]);
                    err = fmax(err, fabs(D[lane * N + n] - ref)); sc = fmax(sc, fabs(ref));
                }
                if (err < 1e-4 * sc) match = i;
            }
            if (match >= 0) ++found;
            if (lane % 8 == 0 || match >= 0 && lane < 40) printf("m64 lane %3d -> row %d (D[0]=%g)\n", lane, match, D[lane * N]);
        }
        printf("m64: %d lanes matched a row\n", found);
    }
    printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
    return fails ? 1 : 0;
}
