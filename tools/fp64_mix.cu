// fp64_mix.cu -- do the FP64 DMMA (mma.sync m8n8k4) and DFMA pipes of B200 add up?  One kernel whose warps run
// a DMMA loop or a DFMA loop (fraction of DFMA warps swept); reports the aggregate fp64 TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix tools/fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_mix(double* out, int iters_mma, int iters_fma, int fma_warps_per8) {
    const int warp = threadIdx.x >> 5;
    double s = 0;
    if ((warp & 7) < fma_warps_per8) {
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
        const double a = 0.999, b = 1e-3;
        for (int i = 0; i < iters_fma; ++i) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s += x[k];
    } else {
        double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
        double c[8][2];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
        for (int i = 0; i < iters_mma; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    }
    if (s == -1.2345) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 256;
    // per warp: DMMA loop does iters_mma * 8 * 512 flops; DFMA loop iters_fma * 32 * 32 * 2 flops
    for (int fw = 0; fw <= 8; ++fw) {
        const int im = 2048, ifm = 2048;
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_mix<<<blocks, threads>>>(out, im, ifm, fw);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        const double warps = (double)blocks * threads / 32;
        const double fma_w = warps * fw / 8, mma_w = warps - fma_w;
        const double flops = mma_w * im * 8 * 512.0 + fma_w * ifm * 32 * 32 * 2.0;
        printf("dfma warps %d/8: %.3f ms  %.1f TFLOP/s (dmma part %.1f, dfma part %.1f)\n", fw, best,
               flops / (best * 1e-3) / 1e12, mma_w * im * 8 * 512.0 / (best * 1e-3) / 1e12,
               fma_w * ifm * 32 * 32 * 2.0 / (best * 1e-3) / 1e12);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
