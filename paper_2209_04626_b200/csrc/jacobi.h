// jacobi.h -- internal interfaces between the engine (mpjsvd.cu) and the
// kernels of the mpjsvd CUDA path.  Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mpj {

// One block pair (I, J), I < J (block ids), of a Jacobi round: base pointers
// of the two column slabs of X (rows m_pad, ld ldx) and V (rows nv_pad, ld
// ldv) and their widths (0 for a bye block).  Pair-local column c is column c
// of slab 0 for c < w0, else column c - w0 of slab 1 (W = [X_I X_J]).  The
// slabs may live anywhere (the matrix itself on one GPU, shard buffers on
// many: DESIGN.md "Multi-GPU").
template <typename T>
struct PairDesc {
    T* x0;
    T* x1;
    T* v0;
    T* v1;
    int w0, w1;
    int b0, b1;         // block ids (schedule identity of the slabs; the bye block has id >= nblk)
};

// Arguments of one block round-robin Jacobi round (k_jacobi.cu).
template <typename T>
struct JacobiRound {
    const PairDesc<T>* pd;   // device: npairs descriptors of this round
    long long ldx;
    long long m_pad;    // multiple of 32
    int n;
    bool has_v;         // V slabs present
    long long ldv;
    long long nv_pad;   // multiple of 32
    int b, npairs;
    int nsplit;
    long long rows_per_split;   // multiple of 32
    T* partial;         // npairs * nsplit * W * W
    T* E;               // npairs * W * W
    int* flag;          // npairs
    T tol, tol_in;
    int max_inner;
    double* sweep_off;  // device scalar, atomic max (this sweep)
    int* sweep_upd;     // device scalar, atomic add (this sweep)
    int* sweep_inner;   // device [2]: max inner sweeps of a pair, summed inner sweeps (this sweep)
    int* sweep_skip;    // device scalar, atomic add: pairs skipped as unchanged (this sweep)
    int use_tc;         // fp32, W = 64: tcgen05 TF32 (hi/lo split) Gram and update (k_tc.cu)
    // completion-ordered publication of solved pairs (overlapped update):
    // dlist[npairs] (-1 = not yet), dctr[0] = publication tail, dctr[1] = update work counter,
    // dctr[2] = error flag (a consumer timed out); reset by the round's Gram kernel
    int* dlist;
    int* dctr;
    int pdl;            // 1: the update is launched as a programmatic dependent of the solve
    // Gram -> solve overlap: the solve is a programmatic dependent of the Gram and waits per pair for
    // gcnt[pair] == nsplit (each Gram CTA adds 1 after its partial is written; the solve zeroes it)
    int* gcnt;
    int gram_pdl;
    // fp32 tcgen05 Gram with TMA loads (k_tc.cu): host pointer to a CUtensorMap over the matrix that holds
    // every local slab (tbase, leading dimension tld), or nullptr (cp.async Gram)
    const void* tmap;
    const T* tbase;
    long long tld;
    const void* umap;   // host pointer to the 2-D CUtensorMap (box 128 x 32) of the update's raw tiles, or nullptr
    const void* smap;   // host pointer to the 2-D SWIZZLE_128B CUtensorMap (box 32 rows x 32 columns) of the Gram, or nullptr
    // exact skip of unchanged pairs: last_mod[blk] = global round index (sweep * R + round) of the last
    // rotation that touched block blk (-1: none); pair_off = this round's per-slot metric of the previous
    // evaluation (written back every evaluation).  A pair whose two blocks were not rotated since its
    // previous evaluation (global round gidx - R) has the same Gram, hence the same metric and no rotation:
    // its Gram and solve are skipped (skip = 0 disables)
    int* last_mod;
    double* pair_off;
    int gidx, R, skip;
    // kernel-variant switches from the handle's options (no environment reads on the launch path)
    int gram_kt;        // rows per TMA Gram stage (32 / 64), resolved on the host
    int gram_variant;   // cp.async tcgen05 Gram variant
    int update_tpc;     // 0: auto
    int update_ts;      // 1: fp32 update with the A operand in tensor memory (k_pair_update_tc_ts)
    int diag;           // mpjsvd_options.diag_timing
    // L2-aware traversal (mpjsvd_options.l2_order, resolved on the host; fp32 tcgen05 stage): consecutive kernels
    // walk the rows of X in opposite directions, all pairs in step, so that the ~100 MB of X the previous kernel
    // touched last are the first the next one reads (a 126 MB LRU-like L2 gives a cyclic 268 MB stream no hits).
    int gram_il;        // 1: the Gram CTA (pair, split) takes the row tiles split, split + nsplit, ... (top -> bottom)
    int upd_order;      // 1: the update's items are claimed tile group major, bottom group first
};

// the pair's blocks are unchanged since its previous evaluation (exactly one sweep ago)
template <typename T>
__device__ __forceinline__ bool pair_unchanged(const JacobiRound<T>& a, const PairDesc<T>& pd) {
    if (!a.skip) return false;
    const int since = a.gidx - a.R;
    return a.last_mod[pd.b0] < since && a.last_mod[pd.b1] < since;
}

// Gram CTA prologue under gram_pdl: the publication reset is visible, then the solve may launch
template <typename T>
__device__ __forceinline__ void gram_pdl_begin(const JacobiRound<T>& a) {
    if (!a.gram_pdl) return;
    __threadfence();
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
// Gram CTA epilogue under gram_pdl: this CTA's partial is written (every thread), count it for its pair
template <typename T>
__device__ __forceinline__ void gram_pdl_end(const JacobiRound<T>& a, int pair) {
    if (!a.gram_pdl) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(a.gcnt + pair, 1);
    }
}

// reset of the publication list by the first CTA of the round's Gram kernel
template <typename T>
__device__ __forceinline__ void reset_publication(const JacobiRound<T>& a) {
    if (a.dlist == nullptr || blockIdx.x != 0 || blockIdx.y != 0) return;
    for (int i = threadIdx.x; i < a.npairs; i += blockDim.x) a.dlist[i] = -1;
    if (threadIdx.x == 0) { a.dctr[0] = 0; a.dctr[1] = 0; }
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Optional per-launch timing hook (bench profiling): begin/end bracket one launch.
struct ProfHook {
    void* ctx;
    void (*begin)(void* ctx, const char* name);
    void (*end)(void* ctx, const char* name);
};

template <typename T>
int launch_jacobi_round(const JacobiRound<T>& a, int W, cudaStream_t st, const ProfHook* hook = nullptr);
template <typename T>
int gram_ctas_per_sm(int W, int use_tc, long long rows_pad, int tma, int kt, int variant);
// tcgen05 fp32 kernels (k_tc.cu)
int launch_gram_tc(const JacobiRound<float>& a, cudaStream_t st);
// MPJSVD_SOLVE_TIMING=1: print k_pair_solve phase clocks (CTA 0) accumulated over a sweep (tools only)
void solve_timing_report(const char* tag, int sweep);
// 4-D TMA view of the column-major fp32 matrix (rows_pad x cols, ld) whose boxes land in the canonical
// K-major SWIZZLE_NONE operand layout of k_pair_gram_tma; out = 128-byte CUtensorMap.  0 on success.
int make_gram_tmap(void* out, const float* base, long long ld, long long rows_pad, long long cols, int kt);
int make_gram_tmap_sw128(void* out, const float* base, long long ld, long long rows_pad, long long cols);
int gram_tma_kt(long long rows_pad, int forced);
int make_update_tmap(void* out, const float* base, long long ld, long long rows_pad, long long cols);
int launch_update_tc(const JacobiRound<float>& a, cudaStream_t st);
// persistent overlapped variant: drains pairs in the order the solve publishes them (a.pdl)
int launch_update_tc_pdl(const JacobiRound<float>& a, cudaStream_t st);
int gram_tc_ctas_per_sm(long long rows_pad, int tma, int kt, int variant);
template <typename T>
int launch_inner_batch(T* G, T* E, int w, T tol_in, int max_inner, int count, int* rot, cudaStream_t st);

// ---- QR (k_qr.cu) --------------------------------------------------------
struct QrWork {
    int* phys_all;      // grid * n
    int* pos_all;       // grid * n
    double* vn1;        // n
    double* vn2;        // n
    double* cand_val;   // 2 * grid
    int* cand_pos;      // 2 * grid
    int* cand_col;      // 2 * grid
    int grid;           // cooperative grid size used
    int* ready = nullptr;  // 1024 per-column release flags (zeroed once) of qr_panel_chain; null: k_qr_coop panels
    cudaStream_t la_stream = nullptr;   // qr_blocked look-ahead: panel p+1 factored here beside p's trailing update
    cudaEvent_t la_ev0 = nullptr, la_ev1 = nullptr;
};
// In-place Householder QR (pivot = 1: Businger-Golub column pivoting) of the
// m x n matrix A (lda).  Columns stay at their physical place; phys[k] (copy
// of CTA 0) gives the column at logical position k.  tau[k] per logical k.
int qr_coop(double* A, long long lda, int m, int n, double* tau, int pivot, QrWork& w,
            int* phys_out, cudaStream_t st);
int qr_coop_grid(int m, int* grid);  // cooperative grid size for this m
// Unpivoted QR of the m x n panel A (n <= 1024) by k_qr_panel (one CTA per column, per-column release flags
// `ready`, no grid barrier); same outputs as qr_coop with pivot = 0 up to rounding order.
int qr_panel_chain(double* A, long long lda, int m, int n, double* tau, int* ready, cudaStream_t st);
// Column-pivoted QR with xLAQPS-style lazy panel updates (k_qrp.cu); same
// outputs as qr_coop(pivot = 1).  work >= qrp_lazy_work_doubles(n, grid).
int qrp_lazy(double* A, long long lda, int m, int n, double* tau, QrWork& w, double* work, int* phys_out,
             cudaStream_t st);
// fp32 instance (pivots of the mixed-precision RRQR, Alg. 4); work as for
// qrp_lazy (sized in doubles), tau n floats
int qrp_lazy_f32(float* A, long long lda, int m, int n, float* tau, QrWork& w, float* work, int* phys_out,
                 cudaStream_t st);
int qrp_lazy_grid(int m, int n, int* grid, int* nown);
size_t qrp_lazy_work_doubles(int n, int grid);
// out[:, k] = A[:, perm[k]] for k < n (rows m_pad)
int gather_cols(const double* A, long long lda, const int* perm, double* out, long long ldo,
                long long rows, int n, cudaStream_t st);

// ---- dense linear algebra (k_linalg.cu) ---------------------------------
// Workspace the GEMM may use for split-K partials (thread-local, set by the engine).
void gemm_set_workspace(double* ws, size_t elems);
int gemm_f64(int ta, int tb, long long M, long long N, long long K, double alpha, const double* A,
             long long lda, const double* B, long long ldb, double beta, double* C, long long ldc,
             cudaStream_t st);
// shape bit 0: compute only the upper triangle of C (tiles below the diagonal are skipped);
// bit 1: op(A) is lower triangular (the K loop of a row tile stops at its last row)
// bit 2: op(A) is upper triangular (the K loop of a row tile starts at its first row)
int gemm_f64_ex(int ta, int tb, long long M, long long N, long long K, double alpha, const double* A,
                long long lda, const double* B, long long ldb, double beta, double* C, long long ldc, int shape,
                cudaStream_t st);
// Cholesky of the n x n SPD matrix G (upper, in place): G = R^T R.  *bad set
// (device int) if a pivot is not positive.
int potrf_upper(double* G, long long ldg, int n, int* bad, cudaStream_t st);
// Q = V R^-1 (R upper n x n), in place on Q (initialised with V), rows nrows.
int trsm_right_upper(const double* R, long long ldr, double* Q, long long ldq, long long nrows, int n,
                     cudaStream_t st);
// C <- Q C, Q = H_0 ... H_{k-1} packed in Vr (rows m, ld ldv), blocked WY.
// tcache (optional): T factors of panels 0 .. ncached-1 as left by qr_blocked (skips their formation)
int apply_q_wy(const double* Vr, long long m, int k, long long ldv, const double* tau, double* C,
               long long ldc, long long ncols, double* work, cudaStream_t st, const double* tcache = nullptr,
               int ncached = 0);
size_t apply_q_work_elems(long long m, long long ncols);
// Q = H_0 ... H_{k-1} formed in place on C (m x m, the identity on entry), trailing blocks only.
int form_q_wy(const double* Vr, long long m, int k, long long ldv, const double* tau, double* C, long long ldc,
              double* work, cudaStream_t st, const double* tcache = nullptr, int ncached = 0);
// T factors of all WY panels of a k-reflector factorisation into tcache (wy_tcache_elems(k))
int wy_tfactors(const double* Vr, long long m, int k, long long ldv, const double* tau, double* tcache, double* work,
                cudaStream_t st);
// number of WY panels of a k-reflector factorisation whose T qr_blocked leaves in its cache (all but the last)
#ifndef MPJ_WY_PANEL
#define MPJ_WY_PANEL 256
#endif
constexpr int WY_PANEL = MPJ_WY_PANEL;   // reflectors per compact-WY panel (blocked QR, WY application)
inline int wy_cached_panels(int k) { return (k + WY_PANEL - 1) / WY_PANEL - 1; }
inline size_t wy_tcache_elems(int k) { return (size_t)((k + WY_PANEL - 1) / WY_PANEL) * WY_PANEL * WY_PANEL; }
// Blocked Householder QR (no pivoting) in place; work >= apply_q_work_elems(m, n).
// tcache (optional, wy_tcache_elems(n)): receives the T factor of every panel with a trailing update
int qr_blocked(double* A, long long lda, int m, int n, double* tau, QrWork& w, double* work, cudaStream_t st,
               double* tcache = nullptr);

// ---- fp32 QR SVD of the AUTO branch (k_qrsvd.cu, reading c-24) ----
// X32 (n x n, ldx; destroyed: holds the bidiagonalisation) -> U (n x n fp64, ldu; columns in descending
// singular value order).  UB: n x n fp64 scratch (ldu); P: packed fp64 reflectors (ldp >= n); work:
// qrsvd32_work_bytes(n); wy_work: apply_q_work_elems(ldp, n) doubles.  *bad set on an exact zero singular value.
size_t qrsvd32_work_bytes(int n);
int qrsvd32(float* X32, long long ldx, int n, double* U, long long ldu, double* UB, double* P, long long ldp,
            void* work, double* wy_work, int* bad, cudaStream_t st, float* S_out = nullptr);
// ---- misc (k_misc.cu) ----------------------------------------------------
int check_finite(const double* A, long long lda, long long m, long long n, int* bad, cudaStream_t st);
int copy_matrix(const double* src, long long lds, double* dst, long long ldd, long long rows, long long cols,
                cudaStream_t st);
template <typename T>
int set_identity(T* A, long long lda, long long rows_pad, long long n, cudaStream_t st);
// AUTO cond gate (DESIGN.md c-15): out2[0] = ||R_s||_1, out2[1] = ||R_s^-1||_1 for R_s = R diag(1/c),
// c_k = a1n[perm[k]] (written to c); Z (rows_pad x n, ldz) is workspace.
int gate_cond_scaled(const double* R, long long ldr, const double* a1n, const int* perm, int n, double* c,
                     double* Z, long long ldz, long long rows_pad, double* out2, cudaStream_t st);
int transpose_upper(const double* R, long long ldr, double* Rt, long long ldt, int n, long long rows_pad,
                    cudaStream_t st);
int lower_from_rt(const double* Rt, long long ldt, double* X, long long ldx, int n, long long rows_pad,
                  cudaStream_t st);
int upper_of(const double* A, long long lda, double* R, long long ldr, int n, long long rows_pad,
             cudaStream_t st);
int maxabs(const double* A, long long lda, long long rows, long long cols, double* out, cudaStream_t st);
int downcast_scaled(const double* X, long long ldx, float* X32, long long ld32, long long rows_pad, int n,
                    const double* maxabs_dev, cudaStream_t st);
template <typename T>
int col_norms(const T* X, long long ldx, long long rows, int n, double* out, int safe, cudaStream_t st);
int rank_desc(const double* key, int n, int* rank, cudaStream_t st);
// UX(:, j) = Y(:, j) / sig[j]; *bad |= 1 if some sig[j] <= 0
int scale_cols(const double* Y, long long ldy, const double* sig, double* UX, long long ldu, long long rows_pad,
               int n, int* bad, cudaStream_t st);
int sort_upcast_v(const float* V32, long long ld32, const int* rank, double* V, long long ldv,
                  long long rows_pad, int n, cudaStream_t st);
int sort_upcast_scale(const float* X32, long long ld32, const int* rank, const double* sig, double* U,
                      long long ldu, long long rows_pad, int n, int* bad, cudaStream_t st);
int finalize(const double* Y, long long ldy, const double* Q, long long ldq, const double* sig,
             const int* rank, double* UX, long long ldu, double* VX, long long ldvx, double* S,
             long long rows_pad, int n, cudaStream_t st);
int scatter_rows_perm(const double* M, long long ldm, const int* perm, double* V, long long ldv, int n,
                      cudaStream_t st);
int diag_stats(const double* R, long long ldr, int n, double* out2, int* bad, cudaStream_t st);
int gates_orth(const double* X, long long ldx, long long rows_pad, int n, float* Xt, long long ldt,
               double* out, cudaStream_t st);

}  // namespace mpj
