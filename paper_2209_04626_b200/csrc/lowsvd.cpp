// lowsvd.cpp -- the fp32 QR SVD of the AUTO branch ("Apply QR SVD algorithm in
// the lower precision ... without generating V_low"), through cuSOLVER's sgesvd (Golub-Kahan
// bidiagonalisation + implicit-shift QR, LAPACK xGESVD semantics), loaded with dlopen so that the library
// runs without it; the branch fails with MPJSVD_ERR_NOT_SUPPORTED when libcusolver is absent.  The default
// path (fp32 one-sided Jacobi) never calls it.
#include <cusolverDn.h>
#include <dlfcn.h>
#include <stdio.h>

#include <mutex>

#include <cuda_runtime.h>

namespace mpj {

namespace {

struct SolverApi {
    bool ok = false;
    decltype(&cusolverDnCreate) Create = nullptr;
    decltype(&cusolverDnDestroy) Destroy = nullptr;
    decltype(&cusolverDnSetStream) SetStream = nullptr;
    decltype(&cusolverDnSgesvd_bufferSize) BufferSize = nullptr;
    decltype(&cusolverDnSgesvd) Gesvd = nullptr;
};
SolverApi g_api;
std::once_flag g_once;
char g_err[256] = "no error";

void load_api() {
    const char* names[] = {"libcusolver.so.11", "libcusolver.so", "/usr/local/cuda/lib64/libcusolver.so.11"};
    void* h = nullptr;
    for (const char* nm : names) {
        h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
        if (h) break;
    }
    if (!h) {
        snprintf(g_err, sizeof(g_err), "libcusolver not found (%s)", dlerror());
        return;
    }
    g_api.Create = reinterpret_cast<decltype(g_api.Create)>(dlsym(h, "cusolverDnCreate"));
    g_api.Destroy = reinterpret_cast<decltype(g_api.Destroy)>(dlsym(h, "cusolverDnDestroy"));
    g_api.SetStream = reinterpret_cast<decltype(g_api.SetStream)>(dlsym(h, "cusolverDnSetStream"));
    g_api.BufferSize = reinterpret_cast<decltype(g_api.BufferSize)>(dlsym(h, "cusolverDnSgesvd_bufferSize"));
    g_api.Gesvd = reinterpret_cast<decltype(g_api.Gesvd)>(dlsym(h, "cusolverDnSgesvd"));
    g_api.ok = g_api.Create && g_api.Destroy && g_api.SetStream && g_api.BufferSize && g_api.Gesvd;
    if (!g_api.ok) snprintf(g_err, sizeof(g_err), "libcusolver lacks a gesvd symbol");
}

}  // namespace

const char* lowsvd_last_error() { return g_err; }

// X32 (n x n, ld ldx; destroyed) = U S V^T in fp32; U (n x n, ld ldu), S[n] descending.  work: device
// scratch of at least lowsvd_work_bytes(n) bytes.  0 ok, -7 library missing, -4 failure.
size_t lowsvd_work_bytes(int n) {
    std::call_once(g_once, load_api);
    if (!g_api.ok) return 0;
    cusolverDnHandle_t hd = nullptr;
    if (g_api.Create(&hd) != CUSOLVER_STATUS_SUCCESS) return 0;
    int lwork = 0;
    g_api.BufferSize(hd, n, n, &lwork);
    g_api.Destroy(hd);
    return sizeof(float) * ((size_t)lwork + (size_t)n) + 64;
}

int lowsvd_sgesvd(float* X32, int n, long long ldx, float* S, float* U, long long ldu, void* work, size_t work_bytes,
                  cudaStream_t st) {
    std::call_once(g_once, load_api);
    if (!g_api.ok) return -7;
    cusolverDnHandle_t hd = nullptr;
    if (g_api.Create(&hd) != CUSOLVER_STATUS_SUCCESS) {
        snprintf(g_err, sizeof(g_err), "cusolverDnCreate failed");
        return -4;
    }
    g_api.SetStream(hd, st);
    int lwork = 0;
    g_api.BufferSize(hd, n, n, &lwork);
    int* info = reinterpret_cast<int*>(work);
    float* wk = reinterpret_cast<float*>(reinterpret_cast<char*>(work) + 64);
    float* rwork = wk + lwork;
    int rc = 0;
    if (sizeof(float) * ((size_t)lwork + (size_t)n) + 64 > work_bytes) {
        snprintf(g_err, sizeof(g_err), "gesvd workspace too small");
        rc = -4;
    } else {
        const cusolverStatus_t s = g_api.Gesvd(hd, 'A', 'N', n, n, X32, (int)ldx, S, U, (int)ldu, nullptr, 1, wk, lwork,
                                               rwork, info);
        if (s != CUSOLVER_STATUS_SUCCESS) {
            snprintf(g_err, sizeof(g_err), "cusolverDnSgesvd status %d", (int)s);
            rc = -4;
        }
    }
    cudaStreamSynchronize(st);
    g_api.Destroy(hd);
    return rc;
}

}  // namespace mpj
