// bw_pattern.cu -- read bandwidth of the Gram's access pattern (tools only, not product code):
// a column-major fp32 matrix (rows x cols, ld = rows); CTA (split, pair) streams rows
// [split * rps, (split + 1) * rps) of 64 columns (two 32-column slabs) in tiles of KT rows,
// reading 16-byte chunks with cp.async into an ST-stage ring (no compute), like k_pair_gram_tc.
// Usage: bw_pattern  -> prints GB/s per (KT, ST, CTAs/SM, nsplit)
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int KT, int ST, int NT>
__global__ void k_read(const float* X, long long ld, long long rps, int npairs, float* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int pair = blockIdx.y, split = blockIdx.x, tid = threadIdx.x;
    const long long r0 = split * rps;
    const int ntile = (int)(rps / KT);
    constexpr int CH = 64 * (KT / 4) / NT;      // 16-byte chunks per thread per tile
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    auto issue = [&](int t) {
#pragma unroll
        for (int u = 0; u < CH; ++u) {
            const int f = tid + NT * u;
            const int c = f / (KT / 4), k4 = f % (KT / 4);
            const int col = c < 32 ? pair * 32 + c : (npairs + pair) * 32 + (c - 32);
            cp16(sb + (uint32_t)((t % ST) * (64 * KT * 4) + f * 16), X + col * ld + r0 + (long long)t * KT + 4 * k4);
        }
    };
    for (int t = 0; t < ST - 1; ++t) { if (t < ntile) issue(t); commit(); }
    float acc = 0.f;
    for (int t = 0; t < ntile; ++t) {
        waitg<ST - 2>();
        __syncthreads();
        acc += reinterpret_cast<const float*>(sm + (t % ST) * (64 * KT * 4))[tid];
        __syncthreads();
        if (t + ST - 1 < ntile) issue(t + ST - 1);
        commit();
    }
    if (acc == 12345.f) sink[0] = acc;
}

template <int KT, int ST, int NT>
void run(const float* X, long long rows, int npairs, int nsplit, float* sink) {
    const size_t smem = (size_t)ST * 64 * KT * 4;
    cudaFuncSetAttribute(k_read<KT, ST, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long rps = rows / nsplit;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) k_read<KT, ST, NT><<<dim3(nsplit, npairs), NT, smem>>>(X, rows, rps, npairs, sink);
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) k_read<KT, ST, NT><<<dim3(nsplit, npairs), NT, smem>>>(X, rows, rps, npairs, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)rows * 64 * npairs * 4;
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_read<KT, ST, NT>, NT, smem);
    printf("KT=%3d ST=%d NT=%d nsplit=%2d ctas/sm=%d  %.1f us  %.0f GB/s  (%s)\n", KT, ST, NT, nsplit, per,
           ms / reps * 1e3, bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const long long rows = 8192;
    const int n = 8192, npairs = 128;
    float* X;
    float* sink;
    cudaMalloc(&X, sizeof(float) * rows * n);
    cudaMalloc(&sink, 4);
    cudaMemset(X, 0, sizeof(float) * rows * n);
    for (int ns : {2, 4, 8}) {
        run<64, 3, 128>(X, rows, npairs, ns, sink);
        run<64, 6, 128>(X, rows, npairs, ns, sink);
        run<128, 3, 128>(X, rows, npairs, ns, sink);
        run<128, 4, 256>(X, rows, npairs, ns, sink);
        run<256, 3, 256>(X, rows, npairs, ns, sink);
        run<32, 8, 128>(X, rows, npairs, ns, sink);
    }
    return 0;
}
