// mpjsvd.cu -- the C-ABI (include/mpjsvd.h) and the single-GPU engine that
// drives the kernels of the mixed-precision Jacobi SVD (PAPER.md:405-458,
// Alg. 3) in the order of DESIGN.md "Path".  No exception crosses the ABI;
// every step returns an int code.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "../../include/mpjsvd.h"
#include "common.cuh"
#include "jacobi.h"

thread_local int64_t g_mpj_launches = 0;
static thread_local char g_last_cuda_err[512] = "no error";

void mpj_record_cuda_error(cudaError_t e, const char* what, const char* file, int line) {
    snprintf(g_last_cuda_err, sizeof(g_last_cuda_err), "%s (%d) in %s at %s:%d", cudaGetErrorString(e), (int)e,
             what, file, line);
}

#define MPJ_TRY(x)                  \
    do {                            \
        int _r = (x);               \
        if (_r != 0) return _r;     \
    } while (0)

using namespace mpj;

namespace {

enum Slot {
    S_A, S_A1, S_A1L, S_RT, S_X, S_Q, S_Y, S_G, S_WY, S_UX, S_VX, S_UBIG, S_VOUT,
    S_X32, S_V32, S_TAU_T0, S_TAU_P, S_TAU_T, S_PERM, S_RANK, S_KEYS, S_FLAGS, S_SCAL,
    S_PART, S_E, S_JFLAG, S_SWEEP, S_QR_PHYS, S_QR_POS, S_QR_VN1, S_QR_VN2, S_QR_CV, S_QR_CP, S_QR_CC,
    S_IOTA, S_TMP1, S_TMP2, S_SOUT, S_GEMMWS, S_QRPW, S_COUNT
};

constexpr double U64 = 1.1102230246251565e-16;
constexpr double U32 = 5.9604644775390625e-08;

}  // namespace

// Per-kernel CUDA-event timing (bench profiling, mpjsvd_set_profiling).
struct Profiler {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    struct Pending { const char* name; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> open;     // begin event of the launch in flight
    std::map<std::string, std::pair<double, long long>> acc;
    cudaStream_t st = nullptr;
    cudaEvent_t get() {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
    void begin(const char* name) {
        (void)name;
        cudaEvent_t e = get();
        cudaEventRecord(e, st);
        open.push_back(e);
    }
    void end(const char* name) {
        cudaEvent_t e = get();
        cudaEventRecord(e, st);
        pending.push_back({name, open.back(), e});
        open.pop_back();
    }
    void resolve() {   // after a stream synchronisation
        for (auto& p : pending) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, p.a, p.b);
            auto& x = acc[p.name];
            x.first += ms;
            x.second += 1;
        }
        pending.clear();
        open.clear();
        used = 0;
    }
    static void hb(void* c, const char* n) { static_cast<Profiler*>(c)->begin(n); }
    static void he(void* c, const char* n) { static_cast<Profiler*>(c)->end(n); }
};

struct mpjsvd_handle_s {
    Profiler prof;
    mpjsvd_options opts;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    void* buf[S_COUNT] = {};
    size_t cap[S_COUNT] = {};
    void* host_pinned = nullptr;   // sweep read-back
    cudaEvent_t ev[10] = {};
};

namespace {

int ensure(mpjsvd_handle h, Slot s, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (h->cap[s] >= bytes) return 0;
    if (h->buf[s]) cudaFree(h->buf[s]);
    h->buf[s] = nullptr;
    h->cap[s] = 0;
    cudaError_t e = cudaMalloc(&h->buf[s], bytes);
    if (e != cudaSuccess) {
        mpj_record_cuda_error(e, "cudaMalloc", __FILE__, __LINE__);
        cudaGetLastError();
        return MPJSVD_ERR_OUT_OF_MEMORY;
    }
    h->cap[s] = bytes;
    return 0;
}
template <typename T>
T* P(mpjsvd_handle h, Slot s) { return reinterpret_cast<T*>(h->buf[s]); }

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

struct JacobiResult {
    int sweeps = 0;
    bool converged = false;
    double off[64] = {};
    int upd[64] = {};
};

// Block round-robin Jacobi stage (fp32 or fp64) on padded device buffers.
template <typename T>
int run_block_jacobi(mpjsvd_handle h, T* X, long long ldx, long long m_pad, int n, T* V, long long ldv,
                     long long nv_pad, int b, T tol, T tol_in, int max_sweeps, int max_inner, bool stagnation,
                     JacobiResult& res) {
    cudaStream_t st = h->stream;
    const int W = 2 * b;
    if (W != 16 && W != 32 && W != 64) return MPJSVD_ERR_NOT_SUPPORTED;
    const int nblk = (int)ceil_div(n, b);
    int M = nblk + (nblk & 1);
    if (nblk == 1) M = 2;
    const int npairs = M / 2;
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, h->device);
    // Row splits of the Gram: minimise waves(npairs * nsplit) / nsplit (wave quantisation of
    // the resident CTA slots), preferring fewer splits (smaller partial reduction) on ties.
    const long long slots = (long long)dev_sms * gram_ctas_per_sm<T>(W);
    const long long maxsplit = std::max(1LL, std::min(m_pad / 32, 64LL));
    long long nsplit = 1;
    double best = 1e30;
    for (long long ns = 1; ns <= maxsplit; ++ns) {
        const long long rps_ = round_up(ceil_div(m_pad, ns), 32);
        const long long ns_eff = ceil_div(m_pad, rps_);
        const double cost = (double)ceil_div(npairs * ns_eff, slots) * (rps_ + 96) + 16.0 * ns_eff;
        if (cost < best - 1e-9) { best = cost; nsplit = ns_eff; }
    }
    long long rps = round_up(ceil_div(m_pad, nsplit), 32);
    nsplit = ceil_div(m_pad, rps);
    MPJ_TRY(ensure(h, S_PART, sizeof(T) * (size_t)npairs * nsplit * W * W));
    MPJ_TRY(ensure(h, S_E, sizeof(T) * (size_t)npairs * W * W));
    MPJ_TRY(ensure(h, S_JFLAG, sizeof(int) * (size_t)npairs));
    MPJ_TRY(ensure(h, S_SWEEP, 64 * (sizeof(double) + sizeof(int))));
    double* d_off = P<double>(h, S_SWEEP);
    int* d_upd = reinterpret_cast<int*>(d_off + 64);
    MPJ_CUDA_TRY(cudaMemsetAsync(d_off, 0, 64 * (sizeof(double) + sizeof(int)), st));

    JacobiRound<T> a;
    a.X = X; a.ldx = ldx; a.m_pad = m_pad; a.n = n;
    a.V = V; a.ldv = ldv; a.nv_pad = V ? nv_pad : 0;
    a.b = b; a.nblk = nblk; a.M = M; a.npairs = npairs;
    a.nsplit = (int)nsplit; a.rows_per_split = rps;
    a.partial = P<T>(h, S_PART); a.E = P<T>(h, S_E); a.flag = P<int>(h, S_JFLAG);
    a.tol = tol; a.tol_in = tol_in; a.max_inner = max_inner;

    double* hp = reinterpret_cast<double*>(h->host_pinned);
    double prev = -1.0;
    res = JacobiResult();
    for (int sw = 1; sw <= max_sweeps && sw <= 64; ++sw) {
        a.sweep_off = d_off + (sw - 1);
        a.sweep_upd = d_upd + (sw - 1);
        ProfHook hook{&h->prof, &Profiler::hb, &Profiler::he};
        for (int r = 0; r < M - 1; ++r) {
            a.round = r;
            MPJ_TRY(launch_jacobi_round<T>(a, W, st, h->prof.on ? &hook : nullptr));
        }
        MPJ_CUDA_TRY(cudaMemcpyAsync(hp, d_off + (sw - 1), sizeof(double), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(hp + 1, d_upd + (sw - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
        if (h->prof.on) h->prof.resolve();
        const double off = hp[0];
        int upd = 0;
        memcpy(&upd, hp + 1, sizeof(int));
        res.sweeps = sw;
        res.off[sw - 1] = off;
        res.upd[sw - 1] = upd;
        if (upd == 0) { res.converged = true; break; }
        // fp32 stagnation exit (reading c-10)
        if (stagnation && sw >= 3 && off <= 1e-4 && prev >= 0 && off > 0.25 * prev) { res.converged = true; break; }
        prev = off;
    }
    return 0;
}

int ensure_qr_work(mpjsvd_handle h, int m, int n, QrWork& w) {
    int grid = 0;
    MPJ_TRY(qr_coop_grid(m, &grid));
    MPJ_TRY(ensure(h, S_QR_PHYS, sizeof(int) * (size_t)grid * n));
    MPJ_TRY(ensure(h, S_QR_POS, sizeof(int) * (size_t)grid * n));
    MPJ_TRY(ensure(h, S_QR_VN1, sizeof(double) * (size_t)n));
    MPJ_TRY(ensure(h, S_QR_VN2, sizeof(double) * (size_t)n));
    MPJ_TRY(ensure(h, S_QR_CV, sizeof(double) * 2 * (size_t)grid));
    MPJ_TRY(ensure(h, S_QR_CP, sizeof(int) * 2 * (size_t)grid));
    MPJ_TRY(ensure(h, S_QR_CC, sizeof(int) * 2 * (size_t)grid));
    w.phys_all = P<int>(h, S_QR_PHYS);
    w.pos_all = P<int>(h, S_QR_POS);
    w.vn1 = P<double>(h, S_QR_VN1);
    w.vn2 = P<double>(h, S_QR_VN2);
    w.cand_val = P<double>(h, S_QR_CV);
    w.cand_pos = P<int>(h, S_QR_CP);
    w.cand_col = P<int>(h, S_QR_CC);
    w.grid = grid;
    return 0;
}

// Precision lift on the padded n x n buffer Q (holding fl64(V32)):
// G = Q^T Q, G = R^T R, Q <- Q R^-1  (reading c-11)
int lift_inplace(mpjsvd_handle h, double* Q, long long ldq, int n, int* bad) {
    cudaStream_t st = h->stream;
    const long long n_pad = round_up(n, 32);
    MPJ_TRY(ensure(h, S_G, sizeof(double) * (size_t)n_pad * n));
    double* G = P<double>(h, S_G);
    MPJ_TRY(gemm_f64(1, 0, n, n, n, 1.0, Q, ldq, Q, ldq, 0.0, G, n_pad, st));
    MPJ_TRY(potrf_upper(G, n_pad, n, bad, st));
    MPJ_TRY(trsm_right_upper(G, n_pad, Q, ldq, n, n, st));
    return 0;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

#define PROF_B(name) do { if (h->prof.on) h->prof.begin(name); } while (0)
#define PROF_E(name) do { if (h->prof.on) h->prof.end(name); } while (0)

int factor_impl(mpjsvd_handle h, const double* A, int64_t m, int64_t n, int64_t lda, double* U, int64_t ldu,
                double* S, double* V, int64_t ldv, mpjsvd_stats* stats) {
    const mpjsvd_options& o = h->opts;
    h->prof.st = h->stream;
    cudaStream_t st = h->stream;
    const long long m_pad = round_up(m, 32), n_pad = round_up(n, 32);
    const bool a_dev = is_device_ptr(A), u_dev = is_device_ptr(U), s_dev = is_device_ptr(S),
               v_dev = is_device_ptr(V);
    mpjsvd_stats local;
    mpjsvd_stats& s = stats ? *stats : local;
    memset(&s, 0, sizeof(s));
    g_mpj_launches = 0;

    const size_t nn = (size_t)n_pad * n;
    MPJ_TRY(ensure(h, S_A, sizeof(double) * (size_t)m_pad * n));
    MPJ_TRY(ensure(h, S_A1, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_A1L, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_RT, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_X, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_Q, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_Y, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_UX, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_VX, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_VOUT, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_X32, sizeof(float) * nn));
    MPJ_TRY(ensure(h, S_V32, sizeof(float) * nn));
    MPJ_TRY(ensure(h, S_TAU_T0, sizeof(double) * n));
    MPJ_TRY(ensure(h, S_TAU_P, sizeof(double) * n));
    MPJ_TRY(ensure(h, S_TAU_T, sizeof(double) * n));
    MPJ_TRY(ensure(h, S_PERM, sizeof(int) * n));
    MPJ_TRY(ensure(h, S_RANK, sizeof(int) * n));
    MPJ_TRY(ensure(h, S_KEYS, sizeof(double) * n));
    MPJ_TRY(ensure(h, S_SOUT, sizeof(double) * n));
    MPJ_TRY(ensure(h, S_FLAGS, sizeof(int) * 8));
    MPJ_TRY(ensure(h, S_SCAL, sizeof(double) * 8));
    MPJ_TRY(ensure(h, S_WY, sizeof(double) * apply_q_work_elems(m_pad, n)));
    if (m > n) MPJ_TRY(ensure(h, S_UBIG, sizeof(double) * (size_t)m_pad * n));
    MPJ_TRY(ensure(h, S_GEMMWS, sizeof(double) * (size_t)8 * 64 * n_pad + sizeof(double) * 64 * 64 * 64));
    gemm_set_workspace(P<double>(h, S_GEMMWS), h->cap[S_GEMMWS] / sizeof(double));

    double* dA = P<double>(h, S_A);
    double* dA1 = P<double>(h, S_A1);
    double* dA1L = P<double>(h, S_A1L);
    double* dRt = P<double>(h, S_RT);
    double* dX = P<double>(h, S_X);
    double* dQ = P<double>(h, S_Q);
    double* dY = P<double>(h, S_Y);
    double* dUX = P<double>(h, S_UX);
    double* dVX = P<double>(h, S_VX);
    double* dVout = P<double>(h, S_VOUT);
    float* dX32 = P<float>(h, S_X32);
    float* dV32 = P<float>(h, S_V32);
    int* flags = P<int>(h, S_FLAGS);    // [0] nonfinite [1] rank deficient [2] cholesky
    double* scal = P<double>(h, S_SCAL);  // [0] maxabs [1..2] diag stats [3] orth
    cudaEvent_t* ev = h->ev;

    MPJ_CUDA_TRY(cudaEventRecord(ev[0], st));
    MPJ_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int) * 8, st));
    // ---- input -> padded device copy (host memory is staged here: e2e path)
    MPJ_CUDA_TRY(cudaMemsetAsync(dA, 0, sizeof(double) * (size_t)m_pad * n, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(dA, sizeof(double) * m_pad, A, sizeof(double) * lda, sizeof(double) * m, n,
                                   a_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    MPJ_TRY(check_finite(dA, m_pad, m, n, flags + 0, st));

    // ---- stage 0: tall QR  A = Q_tall R1
    QrWork qw;
    if (m > n) {
        MPJ_TRY(ensure_qr_work(h, (int)m, (int)n, qw));
        PROF_B("qr_coop_tall");
        MPJ_TRY(qr_blocked(dA, m_pad, (int)m, (int)n, P<double>(h, S_TAU_T0), qw, P<double>(h, S_WY), st));
        PROF_E("qr_coop_tall");
        MPJ_TRY(upper_of(dA, m_pad, dA1, n_pad, (int)n, n_pad, st));
    } else {
        MPJ_TRY(copy_matrix(dA, m_pad, dA1, n_pad, n_pad, n, st));
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[1], st));
    // ---- stage 1: column-pivoted QR  A1 P = Q_p R
    MPJ_TRY(ensure_qr_work(h, (int)n, (int)n, qw));
    PROF_B("qrp_coop");
    {
        int g = 0, no = 0;
        MPJ_TRY(qrp_lazy_grid((int)n, (int)n, &g, &no));
        MPJ_TRY(ensure(h, S_QRPW, sizeof(double) * qrp_lazy_work_doubles((int)n, g)));
        MPJ_TRY(qrp_lazy(dA1, n_pad, (int)n, (int)n, P<double>(h, S_TAU_P), qw, P<double>(h, S_QRPW), P<int>(h, S_PERM), st));
    }
    PROF_E("qrp_coop");
    MPJ_TRY(gather_cols(dA1, n_pad, P<int>(h, S_PERM), dA1L, n_pad, n_pad, (int)n, st));
    MPJ_TRY(diag_stats(dA1L, n_pad, (int)n, scal + 1, flags + 1, st));
    MPJ_CUDA_TRY(cudaEventRecord(ev[2], st));
    // ---- stage 2: R = L Q_2 via QR of R^T; X = L
    if (o.x_from_lq) {
        MPJ_TRY(transpose_upper(dA1L, n_pad, dRt, n_pad, (int)n, n_pad, st));
        PROF_B("lq_coop");
        MPJ_TRY(qr_blocked(dRt, n_pad, (int)n, (int)n, P<double>(h, S_TAU_T), qw, P<double>(h, S_WY), st));
        PROF_E("lq_coop");
        MPJ_TRY(lower_from_rt(dRt, n_pad, dX, n_pad, (int)n, n_pad, st));
    } else {
        MPJ_TRY(upper_of(dA1L, n_pad, dX, n_pad, (int)n, n_pad, st));
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[3], st));
    // ---- stage 3: gate measures, report only
    std::vector<double> xnorms;
    if (o.compute_gates) {
        PROF_B("gates_orth");
        MPJ_TRY(gates_orth(dX, n_pad, n_pad, (int)n, dX32, n_pad, scal + 3, st));
        PROF_E("gates_orth");
        MPJ_TRY(col_norms<double>(dX, n_pad, n_pad, (int)n, P<double>(h, S_KEYS), 1, st));
        xnorms.resize(n);
        MPJ_CUDA_TRY(cudaMemcpyAsync(xnorms.data(), P<double>(h, S_KEYS), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[4], st));
    // ---- stage 4: fp32 block Jacobi
    JacobiResult r32, r64;
    if (o.path != MPJSVD_PATH_FORCE_FP64) {
        MPJ_TRY(maxabs(dX, n_pad, n_pad, n, scal + 0, st));
        MPJ_TRY(downcast_scaled(dX, n_pad, dX32, n_pad, n_pad, (int)n, scal + 0, st));
        MPJ_TRY(set_identity<float>(dV32, n_pad, n_pad, n, st));
        const float tol32 = (float)(o.tol_mult32 * sqrt((double)n) * U32);
        const float tol32_in = tol32 / (float)o.inner_tol_div;
        MPJ_TRY(run_block_jacobi<float>(h, dX32, n_pad, n_pad, (int)n, dV32, n_pad, n_pad, o.block_cols, tol32,
                                        tol32_in, o.max_sweeps32, o.max_inner, true, r32));
        // sort by sigma32 (descending, stable) and upcast V32 -> Q
        MPJ_TRY(col_norms<float>(dX32, n_pad, n_pad, (int)n, P<double>(h, S_KEYS), 0, st));
        MPJ_TRY(rank_desc(P<double>(h, S_KEYS), (int)n, P<int>(h, S_RANK), st));
        MPJ_TRY(sort_upcast_v(dV32, n_pad, P<int>(h, S_RANK), dQ, n_pad, n_pad, (int)n, st));
        MPJ_CUDA_TRY(cudaEventRecord(ev[5], st));
        // ---- stage 5: lift Q = qr(fl64(V32)), Y = X Q
        PROF_B("lift_cholqr");
        MPJ_TRY(lift_inplace(h, dQ, n_pad, (int)n, flags + 2));
        PROF_E("lift_cholqr");
        PROF_B("rv_gemm");
        MPJ_TRY(gemm_f64(0, 0, n_pad, n, n, 1.0, dX, n_pad, dQ, n_pad, 0.0, dY, n_pad, st));
        PROF_E("rv_gemm");
        s.path_taken = MPJSVD_PATH_FORCE_MIXED;
    } else {
        MPJ_CUDA_TRY(cudaEventRecord(ev[5], st));
        MPJ_TRY(set_identity<double>(dQ, n_pad, n_pad, n, st));
        MPJ_TRY(copy_matrix(dX, n_pad, dY, n_pad, n_pad, n, st));
        s.path_taken = MPJSVD_PATH_FORCE_FP64;
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[6], st));
    // ---- stage 6: fp64 refinement with V := Q
    {
        const double tol64 = o.tol_mult64 * sqrt((double)n) * U64;
        MPJ_TRY(run_block_jacobi<double>(h, dY, n_pad, n_pad, (int)n, dQ, n_pad, n_pad, o.block_cols, tol64,
                                         tol64 / o.inner_tol_div, o.max_sweeps64, o.max_inner, false, r64));
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[7], st));
    // ---- stage 7: sigma, U_X, sort; U = Q_tall Q_p U_X; V = P Q_t V_X
    MPJ_TRY(col_norms<double>(dY, n_pad, n_pad, (int)n, P<double>(h, S_SOUT), 1, st));
    MPJ_TRY(rank_desc(P<double>(h, S_SOUT), (int)n, P<int>(h, S_RANK), st));
    MPJ_TRY(finalize(dY, n_pad, dQ, n_pad, P<double>(h, S_SOUT), P<int>(h, S_RANK), dUX, n_pad, dVX, n_pad,
                     P<double>(h, S_KEYS) /* sorted sigma */, n_pad, (int)n, st));
    PROF_B("assemble_wy");
    MPJ_TRY(apply_q_wy(dA1L, n, (int)n, n_pad, P<double>(h, S_TAU_P), dUX, n_pad, n, P<double>(h, S_WY), st));
    double* Ufin = dUX;
    long long ldUf = n_pad;
    if (m > n) {
        double* dUB = P<double>(h, S_UBIG);
        MPJ_CUDA_TRY(cudaMemsetAsync(dUB, 0, sizeof(double) * (size_t)m_pad * n, st));
        MPJ_TRY(copy_matrix(dUX, n_pad, dUB, m_pad, n, n, st));
        MPJ_TRY(apply_q_wy(dA, m, (int)n, m_pad, P<double>(h, S_TAU_T0), dUB, m_pad, n, P<double>(h, S_WY), st));
        Ufin = dUB;
        ldUf = m_pad;
    }
    if (o.x_from_lq)
        MPJ_TRY(apply_q_wy(dRt, n, (int)n, n_pad, P<double>(h, S_TAU_T), dVX, n_pad, n, P<double>(h, S_WY), st));
    MPJ_TRY(scatter_rows_perm(dVX, n_pad, P<int>(h, S_PERM), dVout, n_pad, (int)n, st));
    PROF_E("assemble_wy");
    MPJ_CUDA_TRY(cudaEventRecord(ev[8], st));
    // ---- outputs (device -> device, or device -> host on the e2e path)
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(U, sizeof(double) * ldu, Ufin, sizeof(double) * ldUf, sizeof(double) * m, n,
                                   u_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(V, sizeof(double) * ldv, dVout, sizeof(double) * n_pad, sizeof(double) * n, n,
                                   v_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaMemcpyAsync(S, P<double>(h, S_KEYS), sizeof(double) * n,
                                 s_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaEventRecord(ev[9], st));
    // ---- small read-backs for stats and error flags
    int hflags[8];
    double hscal[8];
    MPJ_CUDA_TRY(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaMemcpyAsync(hscal, scal, sizeof(hscal), cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    if (h->prof.on) h->prof.resolve();
    if (hflags[0]) return MPJSVD_ERR_NONFINITE;
    if (hflags[1] || hflags[2]) return MPJSVD_ERR_RANK_DEFICIENT;

    s.sweeps32 = r32.sweeps;
    s.sweeps64 = r64.sweeps;
    s.converged = r64.converged ? 1 : 0;
    for (int i = 0; i < 32; ++i) {
        s.off_trace32[i] = r32.off[i]; s.upd_trace32[i] = r32.upd[i];
        s.off_trace64[i] = r64.off[i]; s.upd_trace64[i] = r64.upd[i];
    }
    s.final_off32 = r32.sweeps ? r32.off[r32.sweeps - 1] : 0.0;
    s.final_off64 = r64.sweeps ? r64.off[r64.sweeps - 1] : 0.0;
    s.cond_estimate = hscal[2] > 0 ? hscal[1] / hscal[2] : INFINITY;
    s.orth_measure = o.compute_gates ? hscal[3] : NAN;
    s.tail_fraction = NAN;
    if (o.compute_gates) {
        // fraction of "small" columns of X: ||x_j|| < 2^-60 max_j ||x_j|| (reading c-15)
        double mx = 0.0;
        for (double v : xnorms) mx = v > mx ? v : mx;
        long long small = 0;
        for (double v : xnorms) small += v < ldexp(mx, -60) ? 1 : 0;
        s.tail_fraction = (double)small / (double)n;
    }
    s.stage_ms[0] = elapsed(ev[0], ev[1]);
    s.stage_ms[1] = elapsed(ev[1], ev[2]);
    s.stage_ms[2] = elapsed(ev[2], ev[3]);
    s.stage_ms[3] = elapsed(ev[3], ev[4]);
    s.stage_ms[4] = elapsed(ev[4], ev[5]);
    s.stage_ms[5] = elapsed(ev[5], ev[6]);
    s.stage_ms[6] = elapsed(ev[6], ev[7]);
    s.stage_ms[7] = elapsed(ev[7], ev[9]);
    s.total_ms = elapsed(ev[0], ev[9]);
    s.kernel_launches = g_mpj_launches;
    // sigma of a zero column (rank deficiency that survived QR) is an error too
    {
        double smin = 0.0;
        const double* Sd = S;
        if (!s_dev) smin = Sd[n - 1];
        else cudaMemcpy(&smin, Sd + (n - 1), sizeof(double), cudaMemcpyDeviceToHost);
        if (!(smin > 0.0)) return MPJSVD_ERR_RANK_DEFICIENT;
    }
    return r64.converged ? MPJSVD_OK : MPJSVD_WARN_NOT_CONVERGED;
}

}  // namespace

// ==========================================================================
// C-ABI
// ==========================================================================
template <typename T>
static int jacobi_entry(mpjsvd_handle h, T* X, int64_t m, int64_t n, int64_t ldx, T* V, int64_t nv, int64_t ldv,
                        T tol, T tol_in, int32_t max_sweeps, bool stagnation, int32_t* sweeps, mpjsvd_stats* stats,
                        bool is64) {
    if (!h || !X || m < 1 || n < 1 || ldx < m || (V && ldv < nv) || max_sweeps < 1) return MPJSVD_ERR_INVALID_ARG;
    cudaStream_t st = h->stream;
    const long long m_pad = round_up(m, 32), nv_pad = round_up(nv > 0 ? nv : 1, 32);
    MPJ_TRY(ensure(h, S_TMP1, sizeof(T) * (size_t)m_pad * n));
    if (V) MPJ_TRY(ensure(h, S_TMP2, sizeof(T) * (size_t)nv_pad * n));
    T* Xw = P<T>(h, S_TMP1);
    T* Vw = V ? P<T>(h, S_TMP2) : nullptr;
    MPJ_CUDA_TRY(cudaMemsetAsync(Xw, 0, sizeof(T) * (size_t)m_pad * n, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(Xw, sizeof(T) * m_pad, X, sizeof(T) * ldx, sizeof(T) * m, n, cudaMemcpyDefault, st));
    if (V) {
        MPJ_CUDA_TRY(cudaMemsetAsync(Vw, 0, sizeof(T) * (size_t)nv_pad * n, st));
        MPJ_CUDA_TRY(cudaMemcpy2DAsync(Vw, sizeof(T) * nv_pad, V, sizeof(T) * ldv, sizeof(T) * nv, n, cudaMemcpyDefault, st));
    }
    JacobiResult r;
    g_mpj_launches = 0;
    MPJ_TRY(run_block_jacobi<T>(h, Xw, m_pad, m_pad, (int)n, Vw, nv_pad, nv_pad, h->opts.block_cols, tol, tol_in,
                                max_sweeps, h->opts.max_inner, stagnation, r));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(X, sizeof(T) * ldx, Xw, sizeof(T) * m_pad, sizeof(T) * m, n, cudaMemcpyDefault, st));
    if (V)
        MPJ_CUDA_TRY(cudaMemcpy2DAsync(V, sizeof(T) * ldv, Vw, sizeof(T) * nv_pad, sizeof(T) * nv, n, cudaMemcpyDefault, st));
    MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    if (sweeps) *sweeps = r.converged ? r.sweeps : -r.sweeps;
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        for (int i = 0; i < 32; ++i) {
            if (is64) { stats->off_trace64[i] = r.off[i]; stats->upd_trace64[i] = r.upd[i]; }
            else { stats->off_trace32[i] = r.off[i]; stats->upd_trace32[i] = r.upd[i]; }
        }
        if (is64) stats->sweeps64 = r.sweeps; else stats->sweeps32 = r.sweeps;
        stats->converged = r.converged;
        stats->kernel_launches = g_mpj_launches;
    }
    return 0;
}

extern "C" {

void mpjsvd_default_options(mpjsvd_options* o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->num_gpus = 1;
    o->device_id = -1;
    o->block_cols = 32;
    o->tol_mult32 = 4.0;
    o->tol_mult64 = 4.0;
    o->inner_tol_div = 8;
    o->max_sweeps32 = 20;
    o->max_sweeps64 = 30;
    o->max_inner = 30;
    o->path = MPJSVD_PATH_FORCE_MIXED;
    o->x_from_lq = 1;
    o->compute_gates = 1;
    o->stream = nullptr;
}

int mpjsvd_create(mpjsvd_handle* out, const mpjsvd_options* opts) {
    if (!out) return MPJSVD_ERR_INVALID_ARG;
    *out = nullptr;
    mpjsvd_options o;
    if (opts) o = *opts; else mpjsvd_default_options(&o);
    if (o.num_gpus != 1) return MPJSVD_ERR_NOT_SUPPORTED;
    if (o.block_cols != 8 && o.block_cols != 16 && o.block_cols != 32) return MPJSVD_ERR_NOT_SUPPORTED;
    if (!(o.tol_mult32 > 0) || !(o.tol_mult64 > 0) || o.inner_tol_div < 1 || o.max_sweeps32 < 1 ||
        o.max_sweeps64 < 1 || o.max_inner < 1 || (o.path != 0 && o.path != 2))
        return MPJSVD_ERR_INVALID_ARG;
    mpjsvd_handle h = new (std::nothrow) mpjsvd_handle_s();
    if (!h) return MPJSVD_ERR_OUT_OF_MEMORY;
    h->opts = o;
    int dev = o.device_id;
    if (dev < 0) {
        if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); delete h; return MPJSVD_ERR_CUDA; }
    }
    h->device = dev;
    if (cudaSetDevice(dev) != cudaSuccess) {
        mpj_record_cuda_error(cudaGetLastError(), "cudaSetDevice", __FILE__, __LINE__);
        delete h;
        return MPJSVD_ERR_CUDA;
    }
    if (o.stream) {
        h->stream = (cudaStream_t)o.stream;
    } else {
        if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            delete h;
            return MPJSVD_ERR_CUDA;
        }
        h->own_stream = true;
    }
    for (auto& e : h->ev) cudaEventCreate(&e);
    if (cudaMallocHost(&h->host_pinned, 64) != cudaSuccess) {
        cudaGetLastError();
        mpjsvd_destroy(h);
        return MPJSVD_ERR_OUT_OF_MEMORY;
    }
    *out = h;
    return MPJSVD_OK;
}

int mpjsvd_destroy(mpjsvd_handle h) {
    if (!h) return MPJSVD_OK;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (int i = 0; i < S_COUNT; ++i)
        if (h->buf[i]) cudaFree(h->buf[i]);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : h->prof.pool) cudaEventDestroy(e);
    if (h->host_pinned) cudaFreeHost(h->host_pinned);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
    cudaGetLastError();
    return MPJSVD_OK;
}

const char* mpjsvd_strerror(int code) {
    switch (code) {
        case MPJSVD_OK: return "ok";
        case MPJSVD_WARN_NOT_CONVERGED: return "warning: fp64 refinement did not converge within max_sweeps64 (outputs filled)";
        case MPJSVD_ERR_INVALID_ARG: return "invalid argument";
        case MPJSVD_ERR_NONFINITE: return "input contains NaN or Inf";
        case MPJSVD_ERR_RANK_DEFICIENT: return "rank deficient input (zero R diagonal or zero column)";
        case MPJSVD_ERR_CUDA: return "CUDA error (see mpjsvd_last_cuda_error)";
        case MPJSVD_ERR_NCCL: return "NCCL error";
        case MPJSVD_ERR_OUT_OF_MEMORY: return "out of device memory";
        case MPJSVD_ERR_NOT_SUPPORTED: return "not supported in this build";
        default: return "unknown error code";
    }
}

const char* mpjsvd_last_cuda_error(void) { return g_last_cuda_err; }

int mpjsvd_version(void) { return MPJSVD_VERSION; }

int mpjsvd_set_profiling(mpjsvd_handle h, int32_t on) {
    if (!h) return MPJSVD_ERR_INVALID_ARG;
    h->prof.on = on != 0;
    h->prof.acc.clear();
    h->prof.pending.clear();
    h->prof.open.clear();
    h->prof.used = 0;
    return 0;
}

int mpjsvd_get_profile(mpjsvd_handle h, int32_t idx, char* name, int32_t name_len, double* total_ms,
                       int64_t* launches) {
    if (!h) return MPJSVD_ERR_INVALID_ARG;
    const int count = (int)h->prof.acc.size();
    if (idx < 0) return count;
    if (idx >= count) return MPJSVD_ERR_INVALID_ARG;
    auto it = h->prof.acc.begin();
    std::advance(it, idx);
    if (name && name_len > 0) {
        strncpy(name, it->first.c_str(), (size_t)name_len - 1);
        name[name_len - 1] = 0;
    }
    if (total_ms) *total_ms = it->second.first;
    if (launches) *launches = it->second.second;
    return count;
}

int mpjsvd_factor(mpjsvd_handle h, const double* A, int64_t m, int64_t n, int64_t lda, double* U, int64_t ldu,
                  double* S, double* V, int64_t ldv, mpjsvd_stats* stats) {
    if (!h || !A || !U || !S || !V) return MPJSVD_ERR_INVALID_ARG;
    if (n < 2 || m < n || lda < m || ldu < m || ldv < n) return MPJSVD_ERR_INVALID_ARG;
    if (m > 16384 || n > 16384) return MPJSVD_ERR_NOT_SUPPORTED;
    if (cudaSetDevice(h->device) != cudaSuccess) { cudaGetLastError(); return MPJSVD_ERR_CUDA; }
    int rc = factor_impl(h, A, m, n, lda, U, ldu, S, V, ldv, stats);
    if (rc == MPJSVD_ERR_CUDA || rc == MPJSVD_ERR_OUT_OF_MEMORY) cudaGetLastError();
    return rc;
}

int mpjsvd_gemm_f64(mpjsvd_handle h, int32_t transa, int32_t transb, int64_t M, int64_t N, int64_t K, double alpha,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
    if (!h || !A || !B || !C) return MPJSVD_ERR_INVALID_ARG;
    MPJ_TRY(ensure(h, S_GEMMWS, sizeof(double) * (size_t)(M > 0 ? M : 1) * (N > 0 ? N : 1) * 16));
    gemm_set_workspace(P<double>(h, S_GEMMWS), h->cap[S_GEMMWS] / sizeof(double));
    int rc = gemm_f64(transa, transb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, h->stream);
    if (rc) return rc;
    return cudaStreamSynchronize(h->stream) == cudaSuccess ? 0 : MPJSVD_ERR_CUDA;
}

int mpjsvd_inner_solve(mpjsvd_handle h, int32_t is_f64, void* G, void* E, int32_t w, int32_t count, double tol_in,
                       int32_t max_inner, int32_t* rotations) {
    if (!h || !G || !E || w < 1 || w > 64 || count < 1) return MPJSVD_ERR_INVALID_ARG;
    MPJ_TRY(ensure(h, S_TMP1, sizeof(int) * (size_t)count));
    int rc = is_f64 ? launch_inner_batch<double>((double*)G, (double*)E, w, tol_in, max_inner, count,
                                                  P<int>(h, S_TMP1), h->stream)
                    : launch_inner_batch<float>((float*)G, (float*)E, w, (float)tol_in, max_inner, count,
                                                 P<int>(h, S_TMP1), h->stream);
    if (rc) return rc;
    if (rotations)
        MPJ_CUDA_TRY(cudaMemcpyAsync(rotations, P<int>(h, S_TMP1), sizeof(int) * count, cudaMemcpyDeviceToHost,
                                     h->stream));
    MPJ_CUDA_TRY(cudaStreamSynchronize(h->stream));
    return 0;
}

int mpjsvd_block_jacobi_f64(mpjsvd_handle h, double* X, int64_t m, int64_t n, int64_t ldx, double* V, int64_t nv,
                            int64_t ldv, double tol, double tol_in, int32_t max_sweeps, int32_t* sweeps,
                            mpjsvd_stats* stats) {
    return jacobi_entry<double>(h, X, m, n, ldx, V, nv, ldv, tol, tol_in, max_sweeps, false, sweeps, stats, true);
}

int mpjsvd_block_jacobi_f32(mpjsvd_handle h, float* X, int64_t m, int64_t n, int64_t ldx, float* V, int64_t nv,
                            int64_t ldv, float tol, float tol_in, int32_t max_sweeps, int32_t stagnation,
                            int32_t* sweeps, mpjsvd_stats* stats) {
    return jacobi_entry<float>(h, X, m, n, ldx, V, nv, ldv, tol, tol_in, max_sweeps, stagnation != 0, sweeps, stats,
                               false);
}

int mpjsvd_qr(mpjsvd_handle h, double* A, int64_t m, int64_t n, int64_t lda, double* tau, int32_t* perm,
              int32_t pivot) {
    if (!h || !A || !tau || m < n || n < 1 || lda < m) return MPJSVD_ERR_INVALID_ARG;
    gemm_set_workspace(nullptr, 0);
    cudaStream_t st = h->stream;
    const long long m_pad = round_up(m, 32);
    MPJ_TRY(ensure(h, S_TMP1, sizeof(double) * (size_t)m_pad * n));
    MPJ_TRY(ensure(h, S_TMP2, sizeof(double) * (size_t)m_pad * n));
    MPJ_TRY(ensure(h, S_IOTA, sizeof(int) * (size_t)n));
    double* Aw = P<double>(h, S_TMP1);
    MPJ_CUDA_TRY(cudaMemsetAsync(Aw, 0, sizeof(double) * (size_t)m_pad * n, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(Aw, sizeof(double) * m_pad, A, sizeof(double) * lda, sizeof(double) * m, n,
                                   cudaMemcpyDefault, st));
    QrWork qw;
    MPJ_TRY(ensure_qr_work(h, (int)m, (int)n, qw));
    int* phys = P<int>(h, S_IOTA);
    if (pivot == 2) {                 // unblocked reference kernel (tests)
        MPJ_TRY(qr_coop(Aw, m_pad, (int)m, (int)n, tau, 1, qw, phys, st));
    } else if (pivot) {
        int g = 0, no = 0;
        MPJ_TRY(qrp_lazy_grid((int)m, (int)n, &g, &no));
        MPJ_TRY(ensure(h, S_QRPW, sizeof(double) * qrp_lazy_work_doubles((int)n, g)));
        MPJ_TRY(qrp_lazy(Aw, m_pad, (int)m, (int)n, tau, qw, P<double>(h, S_QRPW), phys, st));
    } else {
        MPJ_TRY(ensure(h, S_WY, sizeof(double) * apply_q_work_elems(m_pad, n)));
        MPJ_TRY(qr_blocked(Aw, m_pad, (int)m, (int)n, tau, qw, P<double>(h, S_WY), st));
        std::vector<int> iota(n);
        for (int i = 0; i < n; ++i) iota[i] = i;
        MPJ_CUDA_TRY(cudaMemcpyAsync(phys, iota.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
    }
    double* out = Aw;
    if (pivot) {
        MPJ_TRY(gather_cols(Aw, m_pad, phys, P<double>(h, S_TMP2), m_pad, m_pad, (int)n, st));
        out = P<double>(h, S_TMP2);
    }
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(A, sizeof(double) * lda, out, sizeof(double) * m_pad, sizeof(double) * m, n,
                                   cudaMemcpyDefault, st));
    if (perm) MPJ_CUDA_TRY(cudaMemcpyAsync(perm, phys, sizeof(int) * n, cudaMemcpyDefault, st));
    MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    return 0;
}

int mpjsvd_lift(mpjsvd_handle h, const float* V32, int64_t n, int64_t ldv32, double* Q, int64_t ldq) {
    if (!h || !V32 || !Q || n < 1 || ldv32 < n || ldq < n) return MPJSVD_ERR_INVALID_ARG;
    gemm_set_workspace(nullptr, 0);
    cudaStream_t st = h->stream;
    const long long n_pad = round_up(n, 32);
    MPJ_TRY(ensure(h, S_TMP1, sizeof(float) * (size_t)n_pad * n));
    MPJ_TRY(ensure(h, S_TMP2, sizeof(double) * (size_t)n_pad * n));
    MPJ_TRY(ensure(h, S_IOTA, sizeof(int) * (size_t)n));
    MPJ_TRY(ensure(h, S_FLAGS, sizeof(int) * 8));
    float* Vw = P<float>(h, S_TMP1);
    double* Qw = P<double>(h, S_TMP2);
    MPJ_CUDA_TRY(cudaMemsetAsync(Vw, 0, sizeof(float) * (size_t)n_pad * n, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(Vw, sizeof(float) * n_pad, V32, sizeof(float) * ldv32, sizeof(float) * n, n,
                                   cudaMemcpyDefault, st));
    std::vector<int> iota(n);
    for (int i = 0; i < n; ++i) iota[i] = i;
    MPJ_CUDA_TRY(cudaMemcpyAsync(P<int>(h, S_IOTA), iota.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
    MPJ_CUDA_TRY(cudaMemsetAsync(P<int>(h, S_FLAGS), 0, sizeof(int) * 8, st));
    MPJ_TRY(sort_upcast_v(Vw, n_pad, P<int>(h, S_IOTA), Qw, n_pad, n_pad, (int)n, st));
    MPJ_TRY(lift_inplace(h, Qw, n_pad, (int)n, P<int>(h, S_FLAGS) + 2));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(Q, sizeof(double) * ldq, Qw, sizeof(double) * n_pad, sizeof(double) * n, n,
                                   cudaMemcpyDefault, st));
    int bad[8];
    MPJ_CUDA_TRY(cudaMemcpyAsync(bad, P<int>(h, S_FLAGS), sizeof(bad), cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    return bad[2] ? MPJSVD_ERR_RANK_DEFICIENT : 0;
}

int mpjsvd_apply_q(mpjsvd_handle h, const double* Vr, int64_t m, int64_t k, int64_t ldv, const double* tau, double* C,
                   int64_t ldc, int64_t ncols) {
    if (!h || !Vr || !tau || !C || k > m || ldv < m || ldc < m) return MPJSVD_ERR_INVALID_ARG;
    gemm_set_workspace(nullptr, 0);
    MPJ_TRY(ensure(h, S_WY, sizeof(double) * apply_q_work_elems(m, ncols)));
    MPJ_TRY(apply_q_wy(Vr, m, (int)k, ldv, tau, C, ldc, ncols, P<double>(h, S_WY), h->stream));
    MPJ_CUDA_TRY(cudaStreamSynchronize(h->stream));
    return 0;
}

}  // extern "C"
