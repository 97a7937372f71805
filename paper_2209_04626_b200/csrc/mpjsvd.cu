// mpjsvd.cu -- the C-ABI (include/mpjsvd.h) and the single-GPU engine that
// drives the kernels of the mixed-precision Jacobi SVD (PAPER.md:405-458,
// Alg. 3) in the order of DESIGN.md "Path".  No exception crosses the ABI;
// every step returns an int code.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/mpjsvd.h"
#include "common.cuh"
#include "comm.h"
#include "jacobi.h"
#include "shard.h"

thread_local int64_t g_mpj_launches = 0;
thread_local int g_mpj_diag = 0;
thread_local int g_mpj_qrp_pe = -1;   // options.qrp_panel_stages of the calling handle
static thread_local char g_last_cuda_err[512] = "no error";

cudaError_t mpj_set_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{fn, dev}];
    if (have >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

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
    S_PART, S_E, S_JFLAG, S_SWEEP, S_QR_PHYS, S_QR_POS, S_QR_VN1, S_QR_VN2, S_QR_CV, S_QR_CP, S_QR_CC, S_QR_RDY,
    S_IOTA, S_TMP1, S_TMP2, S_TAU_U, S_LMOD, S_POFF, S_WY2, S_GEMMWS2, S_TC_TALL, S_TC_P, S_TC_T, S_TC_Z, S_XNORM, S_A1N, S_U32, S_S32, S_SVDWS, S_SOUT, S_GEMMWS, S_QRPW, S_PTAB, S_SHX, S_SHV, S_HDR, S_STAGE, S_PUB, S_GATEC, S_COUNT
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
    void* pinned_tab = nullptr;    // staging of the per-sweep pair-descriptor table
    size_t pinned_cap = 0;
    cudaEvent_t ev[10] = {};
    cudaStream_t aux = nullptr;    // second stream: independent assembly chains (fork/join by events)
    cudaEvent_t fork = nullptr, join = nullptr, tpdone = nullptr;
    cudaStream_t qaux = nullptr;   // look-ahead panel factorisations of qr_blocked
    cudaEvent_t qev0 = nullptr, qev1 = nullptr;
    Comm comm;                     // NCCL (multi-process sharding), inactive by default
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

int ensure_pinned(mpjsvd_handle h, size_t bytes) {
    if (h->pinned_cap >= bytes) return 0;
    if (h->pinned_tab) cudaFreeHost(h->pinned_tab);
    h->pinned_tab = nullptr;
    h->pinned_cap = 0;
    cudaError_t e = cudaMallocHost(&h->pinned_tab, bytes);
    if (e != cudaSuccess) {
        mpj_record_cuda_error(e, "cudaMallocHost", __FILE__, __LINE__);
        cudaGetLastError();
        return MPJSVD_ERR_OUT_OF_MEMORY;
    }
    h->pinned_cap = bytes;
    return 0;
}

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
    int inner_max[64] = {};      // max inner sweeps of a pair, per outer sweep
    int inner_sum[64] = {};      // summed inner sweeps over the updated pairs, per outer sweep
    int skipped[64] = {};        // pairs skipped as unchanged, per outer sweep
};

// Where the X / V column slabs of one Jacobi stage live (shard.h): the
// matrix itself (one GPU: buffer j = block j, nothing moves), or per-rank
// shard buffers of nbuf slabs (m_pad x b, ld m_pad), all ranks in this
// process (virtual shards on one GPU) or only `me` (NCCL, one process/GPU).
template <typename T>
struct JStore {
    ShardPlan plan;
    int me = -1;                       // NCCL rank of this process; -1: every rank is local
    std::vector<T*> xs, vs;            // per rank: base of buffer 0 (nullptr if not local)
    long long slab_x = 0, slab_v = 0;  // elements between consecutive buffers
    bool local(int g) const { return me < 0 || g == me; }
    T* bx(int g, int j) const { return xs[g] + (long long)j * slab_x; }
    T* bv(int g, int j) const { return vs[g] ? vs[g] + (long long)j * slab_v : nullptr; }
};

// One sweep's schedule for the local ranks: descriptor table per round and
// the inter-rank moves after each round (plan advanced M-1 times).
template <typename T>
void build_sweep(JStore<T>& S, int b, int n, std::vector<PairDesc<T>>& table,
                 std::vector<std::vector<ShardPlan::Move>>& moves) {
    ShardPlan& pl = S.plan;
    const int R = pl.M - 1;
    table.clear();
    moves.assign(R, {});
    for (int r = 0; r < R; ++r) {
        for (int g = 0; g < pl.G; ++g) {
            if (!S.local(g)) continue;
            for (int t = 0; t < pl.k; ++t) {
                const ShardPlan::Pair p = pl.pair(g, t);
                PairDesc<T> d;
                d.x0 = S.bx(g, p.buf0);
                d.x1 = S.bx(g, p.buf1);
                d.v0 = S.bv(g, p.buf0);
                d.v1 = S.bv(g, p.buf1);
                d.w0 = pl.width(p.blk0, b, n);
                d.w1 = pl.width(p.blk1, b, n);
                d.b0 = p.blk0;
                d.b1 = p.blk1;
                table.push_back(d);
            }
        }
        pl.advance(&moves[r]);
    }
}

// Transfers of one round's inter-rank moves (bye blocks carry no data).
// lmod (NCCL ranks with the exact skip on): each moved block's last-rotation round travels with it
// (4 bytes in the same group), so the receiving rank can skip the block's pairs exactly like one process.
template <typename T>
int exchange(mpjsvd_handle h, JStore<T>& S, const std::vector<ShardPlan::Move>& mv, size_t bytes_x,
             size_t bytes_v, cudaStream_t st, int* lmod = nullptr) {
    if (mv.empty()) return 0;
    const bool nccl = h->comm.active();
    if (nccl) MPJ_TRY(h->comm.group_start());
    int rc = 0;
    for (const auto& m : mv) {
        if (m.blk >= S.plan.nblk) continue;
        const bool sl = S.local(m.src_rank), dl = S.local(m.dst_rank);
        if (sl && dl) {
            MPJ_CUDA_TRY(cudaMemcpyAsync(S.bx(m.dst_rank, m.dst_buf), S.bx(m.src_rank, m.src_buf), bytes_x,
                                         cudaMemcpyDeviceToDevice, st));
            if (bytes_v)
                MPJ_CUDA_TRY(cudaMemcpyAsync(S.bv(m.dst_rank, m.dst_buf), S.bv(m.src_rank, m.src_buf), bytes_v,
                                             cudaMemcpyDeviceToDevice, st));
        } else if (sl) {
            if (!rc) rc = h->comm.send(S.bx(m.src_rank, m.src_buf), bytes_x, m.dst_rank, st);
            if (!rc && bytes_v) rc = h->comm.send(S.bv(m.src_rank, m.src_buf), bytes_v, m.dst_rank, st);
            if (!rc && lmod) rc = h->comm.send(lmod + m.blk, sizeof(int), m.dst_rank, st);
        } else if (dl) {
            if (!rc) rc = h->comm.recv(S.bx(m.dst_rank, m.dst_buf), bytes_x, m.src_rank, st);
            if (!rc && bytes_v) rc = h->comm.recv(S.bv(m.dst_rank, m.dst_buf), bytes_v, m.src_rank, st);
            if (!rc && lmod) rc = h->comm.recv(lmod + m.blk, sizeof(int), m.src_rank, st);
        }
    }
    if (nccl) {
        const int rc2 = h->comm.group_end();
        if (!rc) rc = rc2;
    }
    return rc;
}

// Block round-robin Jacobi stage (fp32 or fp64) over the slabs of S.
template <typename T>
int run_block_jacobi(mpjsvd_handle h, JStore<T>& S, long long ldx, long long m_pad, int n, bool has_v,
                     long long ldv, long long nv_pad, int b, T tol, T tol_in, int max_sweeps, int max_inner,
                     bool stagnation, JacobiResult& res) {
    cudaStream_t st = h->stream;
    const int W = 2 * b;
    if (W != 16 && W != 32 && W != 64) return MPJSVD_ERR_NOT_SUPPORTED;
    int nlocal = 0;
    for (int g = 0; g < S.plan.G; ++g) nlocal += S.local(g) ? 1 : 0;
    const int npairs = nlocal * S.plan.k;
    const int R = S.plan.M - 1;
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, h->device);
    const int use_tc = (sizeof(T) == 4 && W == 64 && h->opts.fp32_tensor_cores) ? 1 : 0;
    // Gram kernel variant: gram_tma = 2 (default) -> the 128-byte-swizzled TMA Gram, warp-specialised, with the A
    // operand [H ; L] in tensor memory (k_pair_gram_sw_ta: 8 stages of raw columns at 3 CTAs/SM; variant 18).
    // Measured: C5 Gram 179.8 -> 172.8 ms per step against the shared-memory-A kernel
    // (k_pair_gram_sw_ws, variant 16; bitwise equal), which had replaced the CTA-barrier kernel (variants 11 / 10)
    int gram_v = h->opts.gram_variant;
    if (h->opts.gram_tma == 2 && (gram_v < 10 || gram_v > 26)) gram_v = 18;
    long long nsplit = 1;
    if (h->opts.split_rows > 0) {
        nsplit = ceil_div(m_pad, round_up(h->opts.split_rows, 32));
    } else {
        // Row splits of the Gram: minimise waves(npairs * nsplit) / nsplit (wave quantisation of
        // the resident CTA slots), preferring fewer splits (smaller partial reduction) on ties.
        const long long slots = (long long)dev_sms * gram_ctas_per_sm<T>(W, use_tc, m_pad, h->opts.gram_tma,
                                                                           h->opts.gram_kt, gram_v);
        const long long maxsplit = std::max(1LL, std::min(m_pad / 32, 64LL));
        double best = 1e30;
        for (long long ns = 1; ns <= maxsplit; ++ns) {
            const long long rps_ = round_up(ceil_div(m_pad, ns), 32);
            const long long ns_eff = ceil_div(m_pad, rps_);
            const double cost = (double)ceil_div(npairs * ns_eff, slots) * (rps_ + 96) + 16.0 * ns_eff;
            if (cost < best - 1e-9) { best = cost; nsplit = ns_eff; }
        }
    }
    long long rps = round_up(ceil_div(m_pad, nsplit), 32);
    nsplit = ceil_div(m_pad, rps);
    MPJ_TRY(ensure(h, S_PART, sizeof(T) * (size_t)npairs * nsplit * W * W));
    MPJ_TRY(ensure(h, S_E, sizeof(T) * (size_t)npairs * W * W));
    MPJ_TRY(ensure(h, S_JFLAG, sizeof(int) * (size_t)npairs));
    MPJ_TRY(ensure(h, S_SWEEP, 64 * (sizeof(double) + 4 * sizeof(int))));
    MPJ_TRY(ensure(h, S_PTAB, sizeof(PairDesc<T>) * (size_t)R * npairs));
    MPJ_TRY(ensure_pinned(h, sizeof(PairDesc<T>) * (size_t)R * npairs));
    MPJ_TRY(ensure(h, S_PUB, sizeof(int) * (2 * (size_t)npairs + 4)));
    double* d_off = P<double>(h, S_SWEEP);
    int* d_upd = reinterpret_cast<int*>(d_off + 64);
    int* d_inner = d_upd + 64;     // [64][2]
    int* d_skip = d_inner + 128;   // [64]
    MPJ_CUDA_TRY(cudaMemsetAsync(d_off, 0, 64 * (sizeof(double) + 4 * sizeof(int)), st));
    PairDesc<T>* d_tab = P<PairDesc<T>>(h, S_PTAB);
    const size_t bytes_x = sizeof(T) * (size_t)S.slab_x, bytes_v = has_v ? sizeof(T) * (size_t)S.slab_v : 0;

    JacobiRound<T> a;
    a.ldx = ldx; a.m_pad = m_pad; a.n = n;
    a.has_v = has_v; a.ldv = ldv; a.nv_pad = has_v ? nv_pad : 0;
    a.b = b; a.npairs = npairs;
    a.nsplit = (int)nsplit; a.rows_per_split = rps;
    a.partial = P<T>(h, S_PART); a.E = P<T>(h, S_E); a.flag = P<int>(h, S_JFLAG);
    a.tol = tol; a.tol_in = tol_in; a.max_inner = max_inner;
    a.use_tc = use_tc;
    a.gram_kt = gram_tma_kt(m_pad, h->opts.gram_kt);
    a.gram_variant = gram_v;
    a.update_tpc = h->opts.update_tpc;
    a.update_ts = h->opts.update_variant == 1 ? 1 : 0;
    a.diag = h->opts.diag_timing;
    a.dctr = P<int>(h, S_PUB);
    a.dlist = a.dctr + 4;
    a.gcnt = a.dlist + npairs;
    a.gram_pdl = h->opts.gram_pdl;
    MPJ_CUDA_TRY(cudaMemsetAsync(a.gcnt, 0, sizeof(int) * (size_t)npairs, st));
    a.pdl = h->opts.pdl_overlap && (sizeof(T) == 8 || use_tc) ? 1 : 0;
    // TMA-fed fp32 Gram: one tensor map over the matrix holding every local slab (the matrix itself on
    // one GPU, the shard buffers otherwise); falls back to the cp.async Gram if the map cannot be made
    alignas(64) static thread_local unsigned char tmap_buf[128];
    alignas(64) static thread_local unsigned char umap_buf[128];
    alignas(64) static thread_local unsigned char smap_buf[128];
    a.tmap = nullptr;
    a.umap = nullptr;
    a.smap = nullptr;
    a.tbase = nullptr;
    a.tld = 0;
    if constexpr (sizeof(T) == 4) {
        if (use_tc && h->opts.gram_tma) {
            T* base = nullptr;
            long long cols = 0;
            for (int g = 0; g < S.plan.G; ++g)
                if (S.local(g)) { base = S.xs[g]; break; }
            int nlocal_ = 0;
            for (int g = 0; g < S.plan.G; ++g) nlocal_ += S.local(g) ? 1 : 0;
            // contiguous store: the n columns of X; shard store: nlocal * nbuf slabs of b columns
            cols = S.plan.G == 1 && S.me < 0 && S.slab_x == (long long)b * ldx ? n : (long long)nlocal_ * S.plan.nbuf * b;
            if (base) {
                a.tbase = base;
                a.tld = ldx;
            }
            if (base && !has_v && make_update_tmap(umap_buf, base, ldx, m_pad, cols) == 0) a.umap = umap_buf;
            if (base && gram_v >= 10 && gram_v <= 26 &&
                make_gram_tmap_sw128(smap_buf, base, ldx, m_pad, cols) == 0)
                a.smap = smap_buf;
            if (base && make_gram_tmap(tmap_buf, base, ldx, m_pad, cols, a.gram_kt) == 0) {
                a.tmap = tmap_buf;
                // a TMA box covers 64 rows and only zero-fills past the matrix: row slabs must be whole boxes
                a.rows_per_split = round_up(a.rows_per_split, 64LL);
                a.nsplit = (int)ceil_div(m_pad, a.rows_per_split);
            }
        }
    }
    // L2-aware traversal (options.l2_order): the warp-specialised swizzled Gram takes interleaved
    // row tiles top -> bottom and the TMEM-A update claims its tile groups bottom group first.  Off by default
    // (measured on B200: no change at C5, the round kernels are not DRAM-bandwidth bound).
    // -1: on when the fp32 X does not fit in L2 (> 96 MB) and the row slabs are the automatic ones
    a.gram_il = 0;
    a.upd_order = 0;
    if constexpr (sizeof(T) == 4) {
        const bool capable = use_tc && a.smap && gram_v >= 16 && gram_v <= 26;
        const bool big = (double)m_pad * (double)n * sizeof(T) > 96.0 * 1024 * 1024;
        const int lo = h->opts.l2_order;
        if (capable && (lo == 1 || (lo < 0 && big && h->opts.split_rows == 0))) {
            a.gram_il = 1;
            a.upd_order = a.update_ts ? 1 : 0;
        }
    }
    MPJ_CUDA_TRY(cudaMemsetAsync(a.dctr, 0, sizeof(int) * 4, st));
    // exact skip of unchanged pairs (every block's last-rotation round: one array per process; across NCCL
    // ranks the entry travels with the block in the per-round exchange)
    MPJ_TRY(ensure(h, S_LMOD, sizeof(int) * (size_t)(S.plan.M + 8)));
    MPJ_TRY(ensure(h, S_POFF, sizeof(double) * (size_t)R * npairs));
    a.last_mod = P<int>(h, S_LMOD);
    a.R = R;
    a.skip = h->opts.skip_unchanged ? 1 : 0;
    int* lmod_ship = (S.me >= 0 && a.skip) ? a.last_mod : nullptr;
    MPJ_CUDA_TRY(cudaMemsetAsync(a.last_mod, 0xff, sizeof(int) * (size_t)(S.plan.M + 8), st));   // -1

    double* hp = reinterpret_cast<double*>(h->host_pinned);
    double prev = -1.0;
    res = JacobiResult();
    std::vector<PairDesc<T>> table;
    std::vector<std::vector<ShardPlan::Move>> moves;
    for (int sw = 1; sw <= max_sweeps && sw <= 64; ++sw) {
        build_sweep<T>(S, b, n, table, moves);
        memcpy(h->pinned_tab, table.data(), sizeof(PairDesc<T>) * table.size());
        MPJ_CUDA_TRY(cudaMemcpyAsync(d_tab, h->pinned_tab, sizeof(PairDesc<T>) * table.size(),
                                     cudaMemcpyHostToDevice, st));
        a.sweep_off = d_off + (sw - 1);
        a.sweep_upd = d_upd + (sw - 1);
        a.sweep_inner = d_inner + 2 * (sw - 1);
        a.sweep_skip = d_skip + (sw - 1);
        ProfHook hook{&h->prof, &Profiler::hb, &Profiler::he};
        for (int r = 0; r < R; ++r) {
            a.pd = d_tab + (size_t)r * npairs;
            a.pair_off = P<double>(h, S_POFF) + (size_t)r * npairs;
            a.gidx = (sw - 1) * R + r;
            MPJ_TRY(launch_jacobi_round<T>(a, W, st, h->prof.on ? &hook : nullptr));
            if (!moves[r].empty()) {
                if (h->prof.on) h->prof.begin("exchange");
                MPJ_TRY(exchange<T>(h, S, moves[r], bytes_x, bytes_v, st, lmod_ship));
                if (h->prof.on) h->prof.end("exchange");
            }
        }
        if (h->comm.active()) {
            MPJ_TRY(h->comm.allreduce_max_f64(d_off + (sw - 1), 1, st));
            MPJ_TRY(h->comm.allreduce_sum_i32(d_upd + (sw - 1), 1, st));
            MPJ_TRY(h->comm.allreduce_sum_i32(d_skip + (sw - 1), 1, st));
        }
        MPJ_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<int*>(hp + 2), d_inner + 2 * (sw - 1), 2 * sizeof(int),
                                     cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<int*>(hp + 3), a.dctr + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(hp, d_off + (sw - 1), sizeof(double), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(hp + 1, d_upd + (sw - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<int*>(hp + 4), d_skip + (sw - 1), sizeof(int),
                                     cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
        if (h->comm.active()) {
            const int rc = h->comm.async_error();
            if (rc) {
                snprintf(g_last_cuda_err, sizeof(g_last_cuda_err), "%s", nccl_last_error());
                return rc;
            }
        }
        if (h->prof.on) h->prof.resolve();
        solve_timing_report(sizeof(T) == 4 ? "f32" : "f64", sw);
        const double off = hp[0];
        int upd = 0;
        memcpy(&upd, hp + 1, sizeof(int));
        res.sweeps = sw;
        res.off[sw - 1] = off;
        res.upd[sw - 1] = upd;
        memcpy(&res.inner_max[sw - 1], reinterpret_cast<int*>(hp + 2), sizeof(int));
        memcpy(&res.inner_sum[sw - 1], reinterpret_cast<int*>(hp + 2) + 1, sizeof(int));
        memcpy(&res.skipped[sw - 1], reinterpret_cast<int*>(hp + 4), sizeof(int));
        int pub_err = 0;
        memcpy(&pub_err, reinterpret_cast<int*>(hp + 3), sizeof(int));
        if (pub_err) {
            snprintf(g_last_cuda_err, sizeof(g_last_cuda_err), "overlapped update: a consumer timed out waiting for a solved pair");
            return MPJSVD_ERR_CUDA;
        }
        if (upd == 0) { res.converged = true; break; }
        // fp32 near-convergence exit (reading c-10): every pair of this sweep was within 2 eps_tol
        if (stagnation && off <= 2.0 * (double)tol) { res.converged = true; break; }
        // fp32 stagnation exit (reading c-10)
        if (stagnation && sw >= 3 && off <= 1e-4 && prev >= 0 && off > 0.25 * prev) { res.converged = true; break; }
        prev = off;
    }
    return 0;
}

// Contiguous store over the matrix itself (one GPU, one rank).
template <typename T>
int contiguous_store(JStore<T>& S, T* X, long long ldx, T* V, long long ldv, int n, int b) {
    if (S.plan.init((int)ceil_div(n, b), 1, true)) return MPJSVD_ERR_INVALID_ARG;
    S.me = -1;
    S.xs = {X};
    S.vs = {V};
    S.slab_x = (long long)b * ldx;
    S.slab_v = (long long)b * ldv;
    return 0;
}

// Sharded store over G ranks: shard buffers for the local ranks, filled from
// the full matrices Xf (m_pad x n, ld m_pad) / Vf (nv_pad x n) -- which must
// hold the data on every rank that has local shards.
template <typename T>
int sharded_store_in(mpjsvd_handle h, JStore<T>& S, int G, const T* Xf, long long m_pad, const T* Vf,
                     long long nv_pad, int n, int b) {
    cudaStream_t st = h->stream;
    if (S.plan.init((int)ceil_div(n, b), G, false)) return MPJSVD_ERR_INVALID_ARG;
    S.me = h->comm.active() ? h->comm.rank : -1;
    const int nlocal = S.me < 0 ? G : 1;
    S.slab_x = m_pad * b;
    S.slab_v = Vf ? nv_pad * b : 0;
    MPJ_TRY(ensure(h, S_SHX, sizeof(T) * (size_t)nlocal * S.plan.nbuf * S.slab_x));
    if (Vf) MPJ_TRY(ensure(h, S_SHV, sizeof(T) * (size_t)nlocal * S.plan.nbuf * S.slab_v));
    S.xs.assign(G, nullptr);
    S.vs.assign(G, nullptr);
    int li = 0;
    for (int g = 0; g < G; ++g) {
        if (!S.local(g)) continue;
        S.xs[g] = P<T>(h, S_SHX) + (size_t)li * S.plan.nbuf * S.slab_x;
        if (Vf) S.vs[g] = P<T>(h, S_SHV) + (size_t)li * S.plan.nbuf * S.slab_v;
        ++li;
        for (int l = 0; l < 2 * S.plan.k; ++l) {
            const int buf = S.plan.buf_at(g, l), blk = S.plan.blk_of(g, buf);
            const int w = S.plan.width(blk, b, n);
            if (w == 0) continue;
            MPJ_CUDA_TRY(cudaMemcpyAsync(S.bx(g, buf), Xf + (size_t)blk * b * m_pad, sizeof(T) * (size_t)w * m_pad,
                                         cudaMemcpyDeviceToDevice, st));
            if (Vf)
                MPJ_CUDA_TRY(cudaMemcpyAsync(S.bv(g, buf), Vf + (size_t)blk * b * nv_pad,
                                             sizeof(T) * (size_t)w * nv_pad, cudaMemcpyDeviceToDevice, st));
        }
    }
    return 0;
}

// Gather every block back into the full matrices on rank 0.  Virtual shards:
// device copies.  NCCL: each rank sends its whole shard storage (nbuf
// consecutive slabs, one message for X and one for V) to rank 0, which
// receives into a staging area and copies every block to its columns.
template <typename T>
int sharded_store_out(mpjsvd_handle h, JStore<T>& S, T* Xf, long long m_pad, T* Vf, long long nv_pad, int n,
                      int b) {
    cudaStream_t st = h->stream;
    const bool nccl = h->comm.active();
    const int me = nccl ? h->comm.rank : 0;
    const int G = S.plan.G;
    const size_t shard_x = (size_t)S.plan.nbuf * S.slab_x, shard_v = (size_t)S.plan.nbuf * S.slab_v;
    std::vector<T*> srcx(G, nullptr), srcv(G, nullptr);    // where rank g's buffer 0 is readable
    for (int g = 0; g < G; ++g)
        if (S.local(g)) { srcx[g] = S.xs[g]; srcv[g] = S.vs[g]; }
    if (nccl) {
        if (me != 0) {
            MPJ_TRY(h->comm.group_start());
            int rc = h->comm.send(S.xs[me], sizeof(T) * shard_x, 0, st);
            if (!rc && Vf) rc = h->comm.send(S.vs[me], sizeof(T) * shard_v, 0, st);
            const int rc2 = h->comm.group_end();
            return rc ? rc : rc2;
        }
        MPJ_TRY(ensure(h, S_STAGE, sizeof(T) * (size_t)G * (shard_x + shard_v)));
        T* stage = P<T>(h, S_STAGE);
        MPJ_TRY(h->comm.group_start());
        int rc = 0;
        for (int g = 1; g < G; ++g) {
            srcx[g] = stage + (size_t)g * (shard_x + shard_v);
            srcv[g] = Vf ? srcx[g] + shard_x : nullptr;
            if (!rc) rc = h->comm.recv(srcx[g], sizeof(T) * shard_x, g, st);
            if (!rc && Vf) rc = h->comm.recv(srcv[g], sizeof(T) * shard_v, g, st);
        }
        const int rc2 = h->comm.group_end();
        if (rc || rc2) return rc ? rc : rc2;
    }
    for (int blk = 0; blk < S.plan.nblk; ++blk) {
        int g = 0, buf = 0;
        if (!S.plan.locate(blk, g, buf)) return MPJSVD_ERR_INVALID_ARG;
        const int w = S.plan.width(blk, b, n);
        MPJ_CUDA_TRY(cudaMemcpyAsync(Xf + (size_t)blk * b * m_pad, srcx[g] + (size_t)buf * S.slab_x,
                                     sizeof(T) * (size_t)w * m_pad, cudaMemcpyDeviceToDevice, st));
        if (Vf)
            MPJ_CUDA_TRY(cudaMemcpyAsync(Vf + (size_t)blk * b * nv_pad, srcv[g] + (size_t)buf * S.slab_v,
                                         sizeof(T) * (size_t)w * nv_pad, cudaMemcpyDeviceToDevice, st));
    }
    return 0;
}

// One Jacobi stage on full matrices X (m_pad x n, ld ldx) / V: contiguous on
// one rank, else scattered to shards, run, and gathered back to rank 0.
template <typename T>
int jacobi_stage(mpjsvd_handle h, T* X, long long ldx, long long m_pad, int n, T* V, long long ldv,
                 long long nv_pad, int b, T tol, T tol_in, int max_sweeps, int max_inner, bool stagnation,
                 JacobiResult& res) {
    const int G = h->comm.active() ? h->comm.world : std::max(1, (int)h->opts.virtual_shards);
    JStore<T> S;
    if (G == 1) {
        MPJ_TRY(contiguous_store<T>(S, X, ldx, V, ldv, n, b));
        return run_block_jacobi<T>(h, S, ldx, m_pad, n, V != nullptr, ldv, nv_pad, b, tol, tol_in, max_sweeps,
                                   max_inner, stagnation, res);
    }
    if (ldx != m_pad || (V && ldv != nv_pad)) return MPJSVD_ERR_INVALID_ARG;
    MPJ_TRY(sharded_store_in<T>(h, S, G, X, m_pad, V, nv_pad, n, b));
    MPJ_TRY(run_block_jacobi<T>(h, S, m_pad, m_pad, n, V != nullptr, nv_pad, nv_pad, b, tol, tol_in, max_sweeps,
                                max_inner, stagnation, res));
    return sharded_store_out<T>(h, S, X, m_pad, V, nv_pad, n, b);
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
    if (h->cap[S_QR_RDY] < sizeof(int) * 1024) {
        MPJ_TRY(ensure(h, S_QR_RDY, sizeof(int) * 1024));
        MPJ_CUDA_TRY(cudaMemsetAsync(h->buf[S_QR_RDY], 0, sizeof(int) * 1024, h->stream));
    }
    w.ready = h->opts.qr_panel_mode == 1 ? nullptr : P<int>(h, S_QR_RDY);
    const bool lookahead = w.ready && h->opts.qr_panel_mode == 0;
    w.la_stream = lookahead ? h->qaux : nullptr;
    w.la_ev0 = h->qev0;
    w.la_ev1 = h->qev1;
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
    MPJ_TRY(gemm_f64_ex(1, 0, n, n, n, 1.0, Q, ldq, Q, ldq, 0.0, G, n_pad, 1, st));   // upper triangle of Q^T Q
    MPJ_TRY(potrf_upper(G, n_pad, n, bad, st));
    MPJ_TRY(trsm_right_upper(G, n_pad, Q, ldq, n, n, st));
    return 0;
}

// U-route precision switch (Alg. 3 l.446-447): Z = X^T U_low (fp64; X lower
// triangular when lower_x, so op(A) = X^T is upper), Householder QR Z = Q R2 (diag(R2) >= 0),
// Q = H_0 ... H_{n-1} I.  Z is overwritten by the reflectors; Q (n_pad x n, zero padding rows).
int switch_u_inplace(mpjsvd_handle h, const double* X, const double* Ulow, double* Z, double* Q, long long ld,
                     int n, bool lower_x, QrWork& qw, cudaStream_t st) {
    double* tau = P<double>(h, S_TAU_U);
    MPJ_TRY(gemm_f64_ex(1, 0, n, n, n, 1.0, X, ld, Ulow, ld, 0.0, Z, ld, lower_x ? 4 : 0, st));
    MPJ_TRY(ensure(h, S_TC_Z, sizeof(double) * wy_tcache_elems(n)));
    MPJ_TRY(qr_blocked(Z, ld, n, n, tau, qw, P<double>(h, S_WY), st, P<double>(h, S_TC_Z)));
    MPJ_TRY(set_identity<double>(Q, ld, ld, n, st));
    MPJ_TRY(form_q_wy(Z, n, n, ld, tau, Q, ld, P<double>(h, S_WY), st, P<double>(h, S_TC_Z), wy_cached_panels(n)));
    return 0;
}

// NVTX range per stage of factor (nsys / ncu --nvtx), closed on every exit path
struct NvtxStages {
    bool open = false;
    void mark(const char* name) {
        if (open) nvtxRangePop();
        nvtxRangePushA(name);
        open = true;
    }
    void close() {
        if (open) nvtxRangePop();
        open = false;
    }
    ~NvtxStages() { close(); }
};
static const char* const kStageNames[10] = {"mpjsvd:qr_tall", "mpjsvd:qrp", "mpjsvd:lq", "mpjsvd:gates",
                                            "mpjsvd:fp32_stage", "mpjsvd:switch", "mpjsvd:fp64_stage",
                                            "mpjsvd:assemble", "mpjsvd:outputs", nullptr};

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
    NvtxStages nvtx;
    const long long m_pad = round_up(m, 32), n_pad = round_up(n, 32);
    const bool a_dev = A && is_device_ptr(A), u_dev = U && is_device_ptr(U), s_dev = S && is_device_ptr(S),
               v_dev = V && is_device_ptr(V);
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
    MPJ_TRY(ensure(h, S_TAU_U, sizeof(double) * n));
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

    const bool dist = h->comm.active();
    const bool root = !dist || h->comm.rank == 0;
    MPJ_TRY(ensure(h, S_HDR, sizeof(long long) * 8));
    long long* d_hdr = P<long long>(h, S_HDR);
    long long* h_hdr = reinterpret_cast<long long*>(h->host_pinned);
    if (dist) {
        // every rank must factor the same (m, n): max-allreduce of (m, n, -m, -n)
        h_hdr[0] = m; h_hdr[1] = n; h_hdr[2] = -m; h_hdr[3] = -n;
        MPJ_CUDA_TRY(cudaMemcpyAsync(d_hdr, h_hdr, 4 * sizeof(long long), cudaMemcpyHostToDevice, st));
        MPJ_TRY(h->comm.allreduce_max_i64(d_hdr, 4, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(h_hdr, d_hdr, 4 * sizeof(long long), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
        if (h_hdr[0] != -h_hdr[2] || h_hdr[1] != -h_hdr[3]) return MPJSVD_ERR_INVALID_ARG;
    }
    // root's error flags -> every rank (NCCL), so that all ranks leave together
    auto agree_status = [&](int code_if_flag0, int code_if_flag12) -> int {
        if (!dist) return 0;
        int hf[8] = {0};
        if (root) {
            MPJ_CUDA_TRY(cudaMemcpyAsync(h_hdr + 4, flags, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
            MPJ_CUDA_TRY(cudaStreamSynchronize(st));
            memcpy(hf, h_hdr + 4, sizeof(hf));
        }
        h_hdr[0] = hf[0] ? code_if_flag0 : ((hf[1] || hf[2]) ? code_if_flag12 : (hf[3] ? MPJSVD_ERR_BREAKDOWN : 0));
        MPJ_CUDA_TRY(cudaMemcpyAsync(d_hdr, h_hdr, sizeof(long long), cudaMemcpyHostToDevice, st));
        MPJ_TRY(h->comm.bcast(d_hdr, sizeof(long long), 0, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(h_hdr, d_hdr, sizeof(long long), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
        return (int)h_hdr[0];
    };
    MPJ_CUDA_TRY(cudaEventRecord(ev[0], st)); nvtx.mark(kStageNames[0]);
    MPJ_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int) * 8, st));
    QrWork qw;
    std::vector<double> xnorms;
    bool gates_read = false;   // X column norms to read back with the stats
    bool tcp_all = false;      // T factors of every Q_p panel precomputed on the auxiliary stream
    const bool autop = o.path == MPJSVD_PATH_AUTO;
    int taken = o.path == MPJSVD_PATH_FORCE_FP64 ? MPJSVD_TAKEN_FP64 : MPJSVD_TAKEN_JACOBI;
    double cond_scaled = NAN, cond_d = NAN;
    bool input_ok = true;
    if (root) {
    // ---- input -> padded device copy (host memory is staged here: e2e path)
    MPJ_CUDA_TRY(cudaMemsetAsync(dA, 0, sizeof(double) * (size_t)m_pad * n, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(dA, sizeof(double) * m_pad, A, sizeof(double) * lda, sizeof(double) * m, n,
                                   a_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    MPJ_TRY(check_finite(dA, m_pad, m, n, flags + 0, st));
    // a non-finite input must not reach the QRP (its argmax has no finite candidate): read the flag now
    MPJ_CUDA_TRY(cudaMemcpyAsync(h_hdr + 7, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    {
        int bad = 0;
        memcpy(&bad, h_hdr + 7, sizeof(int));
        input_ok = bad == 0;
    }
    if (!input_ok && !dist) return MPJSVD_ERR_NONFINITE;
    }  // root
    if (root && input_ok) {

    // ---- stage 0: tall QR  A = Q_tall R1
    if (m > n) {
        MPJ_TRY(ensure_qr_work(h, (int)m, (int)n, qw));
        PROF_B("qr_coop_tall");
        MPJ_TRY(ensure(h, S_TC_TALL, sizeof(double) * wy_tcache_elems((int)n)));
        MPJ_TRY(qr_blocked(dA, m_pad, (int)m, (int)n, P<double>(h, S_TAU_T0), qw, P<double>(h, S_WY), st,
                           P<double>(h, S_TC_TALL)));
        PROF_E("qr_coop_tall");
        MPJ_TRY(upper_of(dA, m_pad, dA1, n_pad, (int)n, n_pad, st));
    } else {
        MPJ_TRY(copy_matrix(dA, m_pad, dA1, n_pad, n_pad, n, st));
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[1], st)); nvtx.mark(kStageNames[1]);
    if (autop) {
        // column norms of A1 = D of A = B D (cond gate; reading c-15)
        MPJ_TRY(ensure(h, S_A1N, sizeof(double) * n));
        MPJ_TRY(col_norms<double>(dA1, n_pad, n_pad, (int)n, P<double>(h, S_A1N), 1, st));
    }
    // ---- stage 1: column-pivoted QR  A1 P = Q_p R
    MPJ_TRY(ensure_qr_work(h, (int)n, (int)n, qw));
    if (o.mp_rrqr) {
        // mixed-precision RRQR (Alg. 4): the permutation from an fp32 QRP of
        // fl32(A1 2^-e) (exact power-of-two scale, reading c-9), then the fp64 QR of A1 P
        PROF_B("qrp_coop");
        int g = 0, no = 0;
        MPJ_TRY(qrp_lazy_grid((int)n, (int)n, &g, &no));
        MPJ_TRY(ensure(h, S_QRPW, sizeof(double) * qrp_lazy_work_doubles((int)n, g)));
        MPJ_TRY(maxabs(dA1, n_pad, n_pad, n, scal + 4, st));
        MPJ_TRY(downcast_scaled(dA1, n_pad, dX32, n_pad, n_pad, (int)n, scal + 4, st));
        MPJ_TRY(qrp_lazy_f32(dX32, n_pad, (int)n, (int)n, reinterpret_cast<float*>(P<double>(h, S_TAU_T)), qw,
                             reinterpret_cast<float*>(P<double>(h, S_QRPW)), P<int>(h, S_PERM), st));
        PROF_E("qrp_coop");
        MPJ_TRY(gather_cols(dA1, n_pad, P<int>(h, S_PERM), dA1L, n_pad, n_pad, (int)n, st));
        PROF_B("qr_ap");
        MPJ_TRY(ensure(h, S_TC_P, sizeof(double) * wy_tcache_elems((int)n)));
        MPJ_TRY(qr_blocked(dA1L, n_pad, (int)n, (int)n, P<double>(h, S_TAU_P), qw, P<double>(h, S_WY), st,
                           P<double>(h, S_TC_P)));
        PROF_E("qr_ap");
    } else {
    PROF_B("qrp_coop");
    {
        int g = 0, no = 0;
        MPJ_TRY(qrp_lazy_grid((int)n, (int)n, &g, &no));
        MPJ_TRY(ensure(h, S_QRPW, sizeof(double) * qrp_lazy_work_doubles((int)n, g)));
        MPJ_TRY(qrp_lazy(dA1, n_pad, (int)n, (int)n, P<double>(h, S_TAU_P), qw, P<double>(h, S_QRPW), P<int>(h, S_PERM), st));
    }
    PROF_E("qrp_coop");
    MPJ_TRY(gather_cols(dA1, n_pad, P<int>(h, S_PERM), dA1L, n_pad, n_pad, (int)n, st));
    // T factors of Q_p for the assembly, on the auxiliary stream while the later stages run (own WY and
    // split-K workspaces; each launch captures the workspace pointer set when it is issued)
    MPJ_TRY(ensure(h, S_TC_P, sizeof(double) * wy_tcache_elems((int)n)));
    MPJ_TRY(ensure(h, S_WY2, sizeof(double) * apply_q_work_elems(m_pad, n)));
    MPJ_TRY(ensure(h, S_GEMMWS2, sizeof(double) * (size_t)8 * 64 * n_pad + sizeof(double) * 64 * 64 * 64));
    MPJ_CUDA_TRY(cudaEventRecord(h->fork, st));
    MPJ_CUDA_TRY(cudaStreamWaitEvent(h->aux, h->fork, 0));
    gemm_set_workspace(P<double>(h, S_GEMMWS2), h->cap[S_GEMMWS2] / sizeof(double));
    MPJ_TRY(wy_tfactors(dA1L, n, (int)n, n_pad, P<double>(h, S_TAU_P), P<double>(h, S_TC_P), P<double>(h, S_WY2), h->aux));
    MPJ_CUDA_TRY(cudaEventRecord(h->tpdone, h->aux));
    gemm_set_workspace(P<double>(h, S_GEMMWS), h->cap[S_GEMMWS] / sizeof(double));
    tcp_all = true;
    }
    MPJ_TRY(diag_stats(dA1L, n_pad, (int)n, scal + 1, flags + 1, st));
    MPJ_CUDA_TRY(cudaEventRecord(ev[2], st)); nvtx.mark(kStageNames[2]);
    // ---- stage 2: R = L Q_2 via QR of R^T; X = L
    if (o.x_from_lq) {
        MPJ_TRY(transpose_upper(dA1L, n_pad, dRt, n_pad, (int)n, n_pad, st));
        PROF_B("lq_coop");
        MPJ_TRY(ensure(h, S_TC_T, sizeof(double) * wy_tcache_elems((int)n)));
        MPJ_TRY(qr_blocked(dRt, n_pad, (int)n, (int)n, P<double>(h, S_TAU_T), qw, P<double>(h, S_WY), st,
                           P<double>(h, S_TC_T)));
        PROF_E("lq_coop");
        MPJ_TRY(lower_from_rt(dRt, n_pad, dX, n_pad, (int)n, n_pad, st));
    } else {
        MPJ_TRY(upper_of(dA1L, n_pad, dX, n_pad, (int)n, n_pad, st));
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[3], st)); nvtx.mark(kStageNames[3]);
    // ---- stage 3: gate measures, report only
    if (o.compute_gates || autop) {
        PROF_B("gates_orth");
        MPJ_TRY(ensure(h, S_XNORM, sizeof(double) * n));
        MPJ_TRY(gates_orth(dX, n_pad, n_pad, (int)n, dX32, n_pad, scal + 3, st));
        PROF_E("gates_orth");
        MPJ_TRY(col_norms<double>(dX, n_pad, n_pad, (int)n, P<double>(h, S_XNORM), 1, st));
        gates_read = true;
    }
    if (autop) {
        // Alg. 3 gates in order (reading c-15): cond, tail (654-663), orth
        // (428-433, 636-650), then Jacobi if orth <= tol_alg else the fp32 QR SVD (435-445)
        // cond_R = kappa_1(R diag(1/c)), c_k = ||A1(:, perm_k)||: Z = diag(c) R^-1 by the triangular solve
        // (dY is free until Y = X Q), the two 1-norms by column reductions
        MPJ_TRY(ensure(h, S_GATEC, sizeof(double) * (size_t)n + 2 * sizeof(double)));
        double* d_gc = P<double>(h, S_GATEC);
        MPJ_TRY(gate_cond_scaled(dA1L, n_pad, P<double>(h, S_A1N), P<int>(h, S_PERM), (int)n, d_gc, dY, n_pad, n_pad,
                                 d_gc + n, st));
        std::vector<double> a1n(n), xn(n);
        double horth = 0.0, norms2[2] = {0.0, 0.0};
        MPJ_CUDA_TRY(cudaMemcpyAsync(a1n.data(), P<double>(h, S_A1N), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(xn.data(), P<double>(h, S_XNORM), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(&horth, scal + 3, sizeof(double), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(norms2, d_gc + n, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
        double dmx = 0.0, dmn = INFINITY, xmx = 0.0;
        for (int64_t k = 0; k < n; ++k) {
            dmx = a1n[k] > dmx ? a1n[k] : dmx;
            dmn = a1n[k] < dmn ? a1n[k] : dmn;
            xmx = xn[k] > xmx ? xn[k] : xmx;
        }
        cond_scaled = norms2[0] * norms2[1];
        if (!(cond_scaled == cond_scaled)) cond_scaled = INFINITY;
        cond_d = dmn > 0.0 ? dmx / dmn : INFINITY;
        long long small = 0;
        for (int64_t j = 0; j < n; ++j) small += xn[j] < ldexp(xmx, o.tail_cut_log2) ? 1 : 0;
        const double tol_cond = o.tol_cond_mult * pow((double)n, 0.25);
        if (cond_scaled <= tol_cond && cond_d > o.cond_d_min) taken = MPJSVD_TAKEN_SKIP_COND;
        else if ((double)small >= ceil(o.tail_frac * (double)n)) taken = MPJSVD_TAKEN_SKIP_TAIL;
        else if (horth <= o.tol_orth) taken = MPJSVD_TAKEN_SKIP_ORTH;
        else if (horth <= o.tol_alg) taken = MPJSVD_TAKEN_JACOBI;
        else taken = MPJSVD_TAKEN_QRSVD;
    }
    }  // root
    if (autop && dist) {
        // every rank takes root's branch
        h_hdr[0] = taken;
        MPJ_CUDA_TRY(cudaMemcpyAsync(d_hdr, h_hdr, sizeof(long long), cudaMemcpyHostToDevice, st));
        MPJ_TRY(h->comm.bcast(d_hdr, sizeof(long long), 0, st));
        MPJ_CUDA_TRY(cudaMemcpyAsync(h_hdr, d_hdr, sizeof(long long), cudaMemcpyDeviceToHost, st));
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
        taken = (int)h_hdr[0];
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[4], st)); nvtx.mark(kStageNames[4]);
    {
        const int rc = agree_status(MPJSVD_ERR_NONFINITE, MPJSVD_ERR_RANK_DEFICIENT);
        if (rc) return rc;
    }
    // ---- stage 4: fp32 block Jacobi
    JacobiResult r32, r64;
    if (taken == MPJSVD_TAKEN_QRSVD) {
        // fp32 QR SVD of lower(X), U only (k_qrsvd.cu, reading c-24), then the
        // U-route switch Q R2 = X^T working(U_low) (446-447) and Y = X Q; non-root ranks wait for Y and Q
        if (root) {
            MPJ_TRY(maxabs(dX, n_pad, n_pad, n, scal + 0, st));
            MPJ_TRY(downcast_scaled(dX, n_pad, dX32, n_pad, n_pad, (int)n, scal + 0, st));
            MPJ_TRY(ensure(h, S_SVDWS, qrsvd32_work_bytes((int)n)));
            PROF_B("qrsvd32");
            // U_B in dY, packed fp64 reflectors in dVX (both free until the switch), U_low -> dUX
            MPJ_TRY(qrsvd32(dX32, n_pad, (int)n, dUX, n_pad, dY, dVX, n_pad, P<void>(h, S_SVDWS), P<double>(h, S_WY),
                            flags + 1, st));
            PROF_E("qrsvd32");
            MPJ_CUDA_TRY(cudaEventRecord(ev[5], st)); nvtx.mark(kStageNames[5]);
            PROF_B("switch_u");
            MPJ_TRY(switch_u_inplace(h, dX, dUX, dVX, dQ, n_pad, (int)n, o.x_from_lq != 0, qw, st));
            PROF_E("switch_u");
            PROF_B("rv_gemm");
            MPJ_TRY(gemm_f64_ex(0, 0, n_pad, n, n, 1.0, dX, n_pad, dQ, n_pad, 0.0, dY, n_pad, o.x_from_lq ? 2 : 0, st));
            PROF_E("rv_gemm");
        } else {
            MPJ_CUDA_TRY(cudaEventRecord(ev[5], st)); nvtx.mark(kStageNames[5]);
        }
        s.path_taken = MPJSVD_TAKEN_QRSVD;
    } else if (taken == MPJSVD_TAKEN_JACOBI) {
        if (root) {
            MPJ_TRY(maxabs(dX, n_pad, n_pad, n, scal + 0, st));
            MPJ_TRY(downcast_scaled(dX, n_pad, dX32, n_pad, n_pad, (int)n, scal + 0, st));
        }
        const bool uroute = o.switch_u != 0;       // U-route: the fp32 stage computes U_low only
        if (!uroute) MPJ_TRY(set_identity<float>(dV32, n_pad, n_pad, n, st));
        if (dist) {
            PROF_B("bcast");
            MPJ_TRY(h->comm.bcast(dX32, sizeof(float) * nn, 0, st));
            PROF_E("bcast");
        }
        const float tol32 = (float)(o.tol_mult32 * sqrt((double)n) * U32);
        const float tol32_in = tol32 / (float)o.inner_tol_div;
        MPJ_TRY(jacobi_stage<float>(h, dX32, n_pad, n_pad, (int)n, uroute ? nullptr : dV32, n_pad, n_pad, o.block_cols, tol32,
                                    tol32_in, o.max_sweeps32, o.max_inner32, true, r32));
        if (root) {
        // sort by sigma32 (descending, stable) and upcast V32 -> Q
        MPJ_TRY(col_norms<float>(dX32, n_pad, n_pad, (int)n, P<double>(h, S_KEYS), 0, st));
        MPJ_TRY(check_finite(P<double>(h, S_KEYS), n, n, 1, flags + 3, st));     // fp32 stage breakdown
        MPJ_TRY(rank_desc(P<double>(h, S_KEYS), (int)n, P<int>(h, S_RANK), st));
        if (uroute) {
            // U_low = working(X32 Sigma32^-1), sigma32-descending
            MPJ_TRY(sort_upcast_scale(dX32, n_pad, P<int>(h, S_RANK), P<double>(h, S_KEYS), dUX, n_pad, n_pad,
                                      (int)n, flags + 1, st));
        } else {
            MPJ_TRY(sort_upcast_v(dV32, n_pad, P<int>(h, S_RANK), dQ, n_pad, n_pad, (int)n, st));
        }
        MPJ_CUDA_TRY(cudaEventRecord(ev[5], st)); nvtx.mark(kStageNames[5]);
        // ---- stage 5: switch precisions, Y = X Q
        if (uroute) {
            // Q = qr(X^T U_low) (U-route); dVX is free until the finalise step
            PROF_B("switch_u");
            MPJ_TRY(switch_u_inplace(h, dX, dUX, dVX, dQ, n_pad, (int)n, o.x_from_lq != 0, qw, st));
            PROF_E("switch_u");
        } else {
            // Q = qr(fl64(V32)) by CholeskyQR (V-route, reading c-11)
            PROF_B("lift_cholqr");
            MPJ_TRY(lift_inplace(h, dQ, n_pad, (int)n, flags + 2));
            PROF_E("lift_cholqr");
        }
        PROF_B("rv_gemm");
        // X lower triangular (X = L, reading c-7): K range of a row tile ends at its last row
        MPJ_TRY(gemm_f64_ex(0, 0, n_pad, n, n, 1.0, dX, n_pad, dQ, n_pad, 0.0, dY, n_pad, o.x_from_lq ? 2 : 0, st));
        PROF_E("rv_gemm");
        MPJ_TRY(check_finite(dY, n_pad, n, n, flags + 3, st));                   // switch / lift breakdown
        } else {
            MPJ_CUDA_TRY(cudaEventRecord(ev[5], st)); nvtx.mark(kStageNames[5]);
        }
        s.path_taken = MPJSVD_TAKEN_JACOBI;
    } else {
        // fp64 only: forced, or an AUTO gate fired (Q = I, Y = X)
        MPJ_CUDA_TRY(cudaEventRecord(ev[5], st)); nvtx.mark(kStageNames[5]);
        if (root) {
            MPJ_TRY(set_identity<double>(dQ, n_pad, n_pad, n, st));
            MPJ_TRY(copy_matrix(dX, n_pad, dY, n_pad, n_pad, n, st));
        }
        s.path_taken = taken;
    }
    {
        const int rc = agree_status(MPJSVD_ERR_NONFINITE, MPJSVD_ERR_RANK_DEFICIENT);
        if (rc) return rc;
    }
    if (dist) {
        PROF_B("bcast");
        MPJ_TRY(h->comm.bcast(dY, sizeof(double) * nn, 0, st));
        MPJ_TRY(h->comm.bcast(dQ, sizeof(double) * nn, 0, st));
        PROF_E("bcast");
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[6], st)); nvtx.mark(kStageNames[6]);
    // ---- stage 6: fp64 refinement with V := Q
    int v_sweeps64 = 0;
    if (!o.refine_v) {
        const double tol64 = o.tol_mult64 * sqrt((double)n) * U64;
        MPJ_TRY(jacobi_stage<double>(h, dY, n_pad, n_pad, (int)n, dQ, n_pad, n_pad, o.block_cols, tol64,
                                     tol64 / o.inner_tol_div, o.max_sweeps64, o.max_inner, false, r64));
        v_sweeps64 = r64.sweeps;
    } else {
        // sec. 3.4 (reading c-23): refine Y without V; U_X = Y diag(1/||y_j||);
        // V_X = qr(X^T U_X) (the U-route construction in fp64); Y = X V_X; one accumulating refinement
        // from (Y, V := V_X), which "always converges in one sweep"
        const double tol64 = o.tol_mult64 * sqrt((double)n) * U64;
        JacobiResult ra, rb;
        MPJ_TRY(jacobi_stage<double>(h, dY, n_pad, n_pad, (int)n, nullptr, n_pad, n_pad, o.block_cols, tol64,
                                     tol64 / o.inner_tol_div, o.max_sweeps64, o.max_inner, false, ra));
        if (root) {
            PROF_B("refine_v_qr");
            MPJ_TRY(col_norms<double>(dY, n_pad, n_pad, (int)n, P<double>(h, S_SOUT), 1, st));
            MPJ_TRY(scale_cols(dY, n_pad, P<double>(h, S_SOUT), dUX, n_pad, n_pad, (int)n, flags + 1, st));
            MPJ_TRY(switch_u_inplace(h, dX, dUX, dVX, dQ, n_pad, (int)n, o.x_from_lq != 0, qw, st));
            MPJ_TRY(gemm_f64_ex(0, 0, n_pad, n, n, 1.0, dX, n_pad, dQ, n_pad, 0.0, dY, n_pad, o.x_from_lq ? 2 : 0, st));
            PROF_E("refine_v_qr");
        }
        {
            const int rc = agree_status(MPJSVD_ERR_NONFINITE, MPJSVD_ERR_RANK_DEFICIENT);
            if (rc) return rc;
        }
        if (dist) {
            MPJ_TRY(h->comm.bcast(dY, sizeof(double) * nn, 0, st));
            MPJ_TRY(h->comm.bcast(dQ, sizeof(double) * nn, 0, st));
        }
        MPJ_TRY(jacobi_stage<double>(h, dY, n_pad, n_pad, (int)n, dQ, n_pad, n_pad, o.block_cols, tol64,
                                     tol64 / o.inner_tol_div, o.max_sweeps64, o.max_inner, false, rb));
        r64 = ra;
        for (int i = 0; i < rb.sweeps && ra.sweeps + i < 64; ++i) {
            const int k = ra.sweeps + i;
            r64.off[k] = rb.off[i];
            r64.upd[k] = rb.upd[i];
            r64.inner_max[k] = rb.inner_max[i];
            r64.inner_sum[k] = rb.inner_sum[i];
            r64.skipped[k] = rb.skipped[i];
        }
        r64.sweeps = ra.sweeps + rb.sweeps;
        r64.converged = ra.converged && rb.converged;
        v_sweeps64 = rb.sweeps;
    }
    MPJ_CUDA_TRY(cudaEventRecord(ev[7], st)); nvtx.mark(kStageNames[7]);
    auto fill_sweep_stats = [&]() {
        s.sweeps32 = r32.sweeps;
        s.sweeps64 = r64.sweeps;
        s.converged = r64.converged ? 1 : 0;
        for (int i = 0; i < 32; ++i) {
            s.off_trace32[i] = r32.off[i]; s.upd_trace32[i] = r32.upd[i];
            s.off_trace64[i] = r64.off[i]; s.upd_trace64[i] = r64.upd[i];
            s.inner_max_trace32[i] = r32.inner_max[i]; s.inner_sum_trace32[i] = r32.inner_sum[i];
            s.inner_max_trace64[i] = r64.inner_max[i]; s.inner_sum_trace64[i] = r64.inner_sum[i];
            s.skip_trace32[i] = r32.skipped[i]; s.skip_trace64[i] = r64.skipped[i];
        }
        s.v_sweeps64 = v_sweeps64;
        s.final_off32 = r32.sweeps ? r32.off[r32.sweeps - 1] : 0.0;
        s.final_off64 = r64.sweeps ? r64.off[r64.sweeps - 1] : 0.0;
    };
    if (!root) {
        // non-root ranks end after the sharded refinement (outputs live on rank 0)
        MPJ_CUDA_TRY(cudaEventRecord(ev[9], st)); nvtx.close();
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
        if (h->prof.on) h->prof.resolve();
        fill_sweep_stats();
        s.stage_ms[4] = elapsed(ev[4], ev[5]);
        s.stage_ms[5] = elapsed(ev[5], ev[6]);
        s.stage_ms[6] = elapsed(ev[6], ev[7]);
        s.total_ms = elapsed(ev[0], ev[9]);
        s.kernel_launches = g_mpj_launches;
        return r64.converged ? MPJSVD_OK : MPJSVD_WARN_NOT_CONVERGED;
    }
    // ---- stage 7: sigma, U_X, sort; U = Q_tall Q_p U_X; V = P Q_t V_X
    MPJ_TRY(col_norms<double>(dY, n_pad, n_pad, (int)n, P<double>(h, S_SOUT), 1, st));
    MPJ_TRY(rank_desc(P<double>(h, S_SOUT), (int)n, P<int>(h, S_RANK), st));
    MPJ_TRY(finalize(dY, n_pad, dQ, n_pad, P<double>(h, S_SOUT), P<int>(h, S_RANK), dUX, n_pad, dVX, n_pad,
                     P<double>(h, S_KEYS) /* sorted sigma */, n_pad, (int)n, st));
    PROF_B("assemble_wy");
    // V = P Q_t V_X on the auxiliary stream (own WY and split-K workspaces; each launch captures the
    // workspace pointer set when it is issued), U = Q_tall Q_p U_X on the main stream, joined below
    const bool v_chain = o.x_from_lq != 0;
    if (v_chain) {
        MPJ_TRY(ensure(h, S_WY2, sizeof(double) * apply_q_work_elems(m_pad, n)));
        MPJ_TRY(ensure(h, S_GEMMWS2, sizeof(double) * (size_t)8 * 64 * n_pad + sizeof(double) * 64 * 64 * 64));
        MPJ_CUDA_TRY(cudaEventRecord(h->fork, st));
        MPJ_CUDA_TRY(cudaStreamWaitEvent(h->aux, h->fork, 0));
        gemm_set_workspace(P<double>(h, S_GEMMWS2), h->cap[S_GEMMWS2] / sizeof(double));
        MPJ_TRY(apply_q_wy(dRt, n, (int)n, n_pad, P<double>(h, S_TAU_T), dVX, n_pad, n, P<double>(h, S_WY2), h->aux,
                           P<double>(h, S_TC_T), wy_cached_panels((int)n)));
        MPJ_TRY(scatter_rows_perm(dVX, n_pad, P<int>(h, S_PERM), dVout, n_pad, (int)n, h->aux));
        // V's output copy (device, or host on the e2e path) on the auxiliary stream: it overlaps U's chain
        MPJ_CUDA_TRY(cudaMemcpy2DAsync(V, sizeof(double) * ldv, dVout, sizeof(double) * n_pad, sizeof(double) * n, n,
                                       v_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->aux));
        MPJ_CUDA_TRY(cudaEventRecord(h->join, h->aux));
        gemm_set_workspace(P<double>(h, S_GEMMWS), h->cap[S_GEMMWS] / sizeof(double));
    }
    if (tcp_all) MPJ_CUDA_TRY(cudaStreamWaitEvent(st, h->tpdone, 0));   // Q_p's T factors (aux stream)
    MPJ_TRY(apply_q_wy(dA1L, n, (int)n, n_pad, P<double>(h, S_TAU_P), dUX, n_pad, n, P<double>(h, S_WY), st,
                       (o.mp_rrqr || tcp_all) ? P<double>(h, S_TC_P) : nullptr,
                       tcp_all ? (int)ceil_div(n, WY_PANEL) : (o.mp_rrqr ? wy_cached_panels((int)n) : 0)));
    double* Ufin = dUX;
    long long ldUf = n_pad;
    if (m > n) {
        double* dUB = P<double>(h, S_UBIG);
        MPJ_CUDA_TRY(cudaMemsetAsync(dUB, 0, sizeof(double) * (size_t)m_pad * n, st));
        MPJ_TRY(copy_matrix(dUX, n_pad, dUB, m_pad, n, n, st));
        MPJ_TRY(apply_q_wy(dA, m, (int)n, m_pad, P<double>(h, S_TAU_T0), dUB, m_pad, n, P<double>(h, S_WY), st,
                           P<double>(h, S_TC_TALL), wy_cached_panels((int)n)));
        Ufin = dUB;
        ldUf = m_pad;
    }
    if (v_chain) MPJ_CUDA_TRY(cudaStreamWaitEvent(st, h->join, 0));
    else MPJ_TRY(scatter_rows_perm(dVX, n_pad, P<int>(h, S_PERM), dVout, n_pad, (int)n, st));
    PROF_E("assemble_wy");
    MPJ_CUDA_TRY(cudaEventRecord(ev[8], st)); nvtx.mark(kStageNames[8]);
    // ---- outputs (device -> device, or device -> host on the e2e path)
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(U, sizeof(double) * ldu, Ufin, sizeof(double) * ldUf, sizeof(double) * m, n,
                                   u_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (!v_chain)
        MPJ_CUDA_TRY(cudaMemcpy2DAsync(V, sizeof(double) * ldv, dVout, sizeof(double) * n_pad, sizeof(double) * n, n,
                                       v_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaMemcpyAsync(S, P<double>(h, S_KEYS), sizeof(double) * n,
                                 s_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaEventRecord(ev[9], st)); nvtx.close();
    // ---- small read-backs for stats and error flags
    int hflags[8];
    double hscal[8];
    if (gates_read) {
        xnorms.resize(n);
        MPJ_CUDA_TRY(cudaMemcpyAsync(xnorms.data(), P<double>(h, S_XNORM), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    }
    MPJ_CUDA_TRY(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaMemcpyAsync(hscal, scal, sizeof(hscal), cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    if (h->prof.on) h->prof.resolve();
    if (hflags[0]) return MPJSVD_ERR_NONFINITE;
    if (hflags[1] || hflags[2]) return MPJSVD_ERR_RANK_DEFICIENT;
    if (hflags[3]) return MPJSVD_ERR_BREAKDOWN;

    fill_sweep_stats();
    s.cond_estimate = hscal[2] > 0 ? hscal[1] / hscal[2] : INFINITY;
    s.orth_measure = (o.compute_gates || autop) ? hscal[3] : NAN;
    s.cond_scaled = cond_scaled;
    s.cond_d = cond_d;
    s.tail_fraction = NAN;
    if (o.compute_gates || autop) {
        // fraction of "small" columns of X: ||x_j|| < 2^tail_cut_log2 max_j ||x_j|| (reading c-15)
        double mx = 0.0;
        for (double v : xnorms) mx = v > mx ? v : mx;
        long long small = 0;
        for (double v : xnorms) small += v < ldexp(mx, o.tail_cut_log2) ? 1 : 0;
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
    g_mpj_diag = h->opts.diag_timing;
    g_mpj_qrp_pe = h->opts.qrp_panel_stages;
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
    MPJ_TRY(jacobi_stage<T>(h, Xw, m_pad, m_pad, (int)n, Vw, nv_pad, nv_pad, h->opts.block_cols, tol, tol_in,
                            max_sweeps, h->opts.max_inner, stagnation, r));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(X, sizeof(T) * ldx, Xw, sizeof(T) * m_pad, sizeof(T) * m, n, cudaMemcpyDefault, st));
    if (V)
        MPJ_CUDA_TRY(cudaMemcpy2DAsync(V, sizeof(T) * ldv, Vw, sizeof(T) * nv_pad, sizeof(T) * nv, n, cudaMemcpyDefault, st));
    MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    if (sweeps) *sweeps = r.converged ? r.sweeps : -r.sweeps;
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        for (int i = 0; i < 32; ++i) {
            if (is64) {
                stats->off_trace64[i] = r.off[i]; stats->upd_trace64[i] = r.upd[i];
                stats->inner_max_trace64[i] = r.inner_max[i]; stats->inner_sum_trace64[i] = r.inner_sum[i];
                stats->skip_trace64[i] = r.skipped[i];
            } else {
                stats->skip_trace32[i] = r.skipped[i];
                stats->off_trace32[i] = r.off[i]; stats->upd_trace32[i] = r.upd[i];
                stats->inner_max_trace32[i] = r.inner_max[i]; stats->inner_sum_trace32[i] = r.inner_sum[i];
            }
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
    o->virtual_shards = 1;
    o->split_rows = 0;
    o->fp32_tensor_cores = 1;
    o->pdl_overlap = 1;
    o->mp_rrqr = 0;
    o->max_inner32 = 1;
    o->switch_u = 1;
    o->tol_orth = 1e-5;
    o->tol_alg = INFINITY;
    o->tol_cond_mult = 1.0;
    o->cond_d_min = 1e15;
    o->tail_frac = 1.0 / 3.0;
    o->tail_cut_log2 = -60;
    o->gram_tma = 2;
    o->gram_kt = 0;
    o->gram_variant = 0;
    o->update_tpc = 0;
    o->skip_unchanged = 1;
    o->qr_panel_mode = 0;
    o->diag_timing = 0;
    o->refine_v = 0;
    o->update_variant = 1;
    o->qrp_panel_stages = -1;
    o->gram_pdl = 1;
    o->l2_order = 0;
}

int mpjsvd_create(mpjsvd_handle* out, const mpjsvd_options* opts) {
    if (!out) return MPJSVD_ERR_INVALID_ARG;
    *out = nullptr;
    mpjsvd_options o;
    if (opts) o = *opts; else mpjsvd_default_options(&o);
    if (o.num_gpus != 1) return MPJSVD_ERR_NOT_SUPPORTED;   // multi-GPU: one handle per process + mpjsvd_comm_init
    if (o.virtual_shards < 1 || o.virtual_shards > 64 || o.split_rows < 0) return MPJSVD_ERR_INVALID_ARG;
    if (o.block_cols != 8 && o.block_cols != 16 && o.block_cols != 32) return MPJSVD_ERR_NOT_SUPPORTED;
    if (!(o.tol_mult32 > 0) || !(o.tol_mult64 > 0) || o.inner_tol_div < 1 || o.max_sweeps32 < 1 ||
        o.max_sweeps64 < 1 || o.max_inner < 1 || o.max_inner32 < 1 || (o.path != 0 && o.path != 1 && o.path != 2))
        return MPJSVD_ERR_INVALID_ARG;
    if ((o.gram_kt != 0 && o.gram_kt != 32 && o.gram_kt != 64) || o.gram_tma < 0 || o.gram_tma > 2 || o.gram_variant < 0 || o.gram_variant > 26 ||
        o.update_tpc < 0 || o.qr_panel_mode < 0 || o.qr_panel_mode > 2 || o.refine_v < 0 || o.refine_v > 1 || o.update_variant < 0 || o.update_variant > 1 ||
        o.qrp_panel_stages < -1 || o.qrp_panel_stages == 1 || o.qrp_panel_stages > 4 ||
        o.gram_pdl < 0 || o.gram_pdl > 1 || o.l2_order < -1 || o.l2_order > 1)
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
    if (cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->tpdone, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->qaux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->qev0, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->qev1, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        mpjsvd_destroy(h);
        return MPJSVD_ERR_CUDA;
    }
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
    if (h->pinned_tab) cudaFreeHost(h->pinned_tab);
    h->comm.destroy();
    if (h->aux) { cudaStreamSynchronize(h->aux); cudaStreamDestroy(h->aux); }
    if (h->fork) cudaEventDestroy(h->fork);
    if (h->join) cudaEventDestroy(h->join);
    if (h->tpdone) cudaEventDestroy(h->tpdone);
    if (h->qaux) { cudaStreamSynchronize(h->qaux); cudaStreamDestroy(h->qaux); }
    if (h->qev0) cudaEventDestroy(h->qev0);
    if (h->qev1) cudaEventDestroy(h->qev1);
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
        case MPJSVD_ERR_NCCL: return "NCCL error (see mpjsvd_last_cuda_error)";
        case MPJSVD_ERR_OUT_OF_MEMORY: return "out of device memory";
        case MPJSVD_ERR_NOT_SUPPORTED: return "not supported in this build";
        case MPJSVD_ERR_BREAKDOWN: return "non-finite intermediate from a finite input (fp32 stage or precision switch)";
        default: return "unknown error code";
    }
}

const char* mpjsvd_last_cuda_error(void) { return g_last_cuda_err; }

int mpjsvd_comm_unique_id(uint8_t* id) {
    if (!id) return MPJSVD_ERR_INVALID_ARG;
    const int rc = nccl_unique_id(id);
    if (rc) snprintf(g_last_cuda_err, sizeof(g_last_cuda_err), "%s", nccl_last_error());
    return rc;
}

int mpjsvd_comm_init(mpjsvd_handle h, int32_t rank, int32_t world, const uint8_t* id) {
    if (!h || !id || world < 1 || rank < 0 || rank >= world) return MPJSVD_ERR_INVALID_ARG;
    if (h->opts.virtual_shards > 1) return MPJSVD_ERR_INVALID_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) { cudaGetLastError(); return MPJSVD_ERR_CUDA; }
    const int rc = h->comm.init(rank, world, id);
    if (rc) snprintf(g_last_cuda_err, sizeof(g_last_cuda_err), "%s", nccl_last_error());
    return rc;
}

int mpjsvd_comm_info(mpjsvd_handle h, int32_t* rank, int32_t* world) {
    if (!h) return MPJSVD_ERR_INVALID_ARG;
    if (rank) *rank = h->comm.active() ? h->comm.rank : 0;
    if (world) *world = h->comm.active() ? h->comm.world : 1;
    return 0;
}

// ---- shard plan (host only; shard.h) ----
struct mpjsvd_plan_s {
    ShardPlan p;
};

int mpjsvd_plan_create(mpjsvd_plan* out, int32_t nblk, int32_t world) {
    if (!out) return MPJSVD_ERR_INVALID_ARG;
    *out = nullptr;
    mpjsvd_plan pl = new (std::nothrow) mpjsvd_plan_s();
    if (!pl) return MPJSVD_ERR_OUT_OF_MEMORY;
    if (pl->p.init(nblk, world, world == 1)) { delete pl; return MPJSVD_ERR_INVALID_ARG; }
    *out = pl;
    return 0;
}

int mpjsvd_plan_info(mpjsvd_plan pl, int32_t* M, int32_t* k, int32_t* nbuf) {
    if (!pl) return MPJSVD_ERR_INVALID_ARG;
    if (M) *M = pl->p.M;
    if (k) *k = pl->p.k;
    if (nbuf) *nbuf = pl->p.nbuf;
    return 0;
}

int mpjsvd_plan_pairs(mpjsvd_plan pl, int32_t rank, int32_t* out) {
    if (!pl || !out || rank < 0 || rank >= pl->p.G) return MPJSVD_ERR_INVALID_ARG;
    for (int t = 0; t < pl->p.k; ++t) {
        const ShardPlan::Pair q = pl->p.pair(rank, t);
        out[4 * t + 0] = q.buf0; out[4 * t + 1] = q.buf1;
        out[4 * t + 2] = q.blk0; out[4 * t + 3] = q.blk1;
    }
    return pl->p.k;
}

int mpjsvd_plan_advance(mpjsvd_plan pl, int32_t* moves, int32_t cap) {
    if (!pl || (cap > 0 && !moves)) return MPJSVD_ERR_INVALID_ARG;
    std::vector<ShardPlan::Move> mv;
    pl->p.advance(&mv);
    const int cnt = (int)mv.size();
    for (int i = 0; i < cnt && i < cap; ++i) {
        moves[5 * i + 0] = mv[i].blk; moves[5 * i + 1] = mv[i].src_rank; moves[5 * i + 2] = mv[i].src_buf;
        moves[5 * i + 3] = mv[i].dst_rank; moves[5 * i + 4] = mv[i].dst_buf;
    }
    return cnt;
}

int mpjsvd_plan_locate(mpjsvd_plan pl, int32_t blk, int32_t* rank, int32_t* buf) {
    if (!pl) return MPJSVD_ERR_INVALID_ARG;
    int g = 0, b = 0;
    if (!pl->p.locate(blk, g, b)) return MPJSVD_ERR_INVALID_ARG;
    if (rank) *rank = g;
    if (buf) *buf = b;
    return 0;
}

int mpjsvd_plan_destroy(mpjsvd_plan pl) {
    delete pl;
    return 0;
}

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
    if (!h) return MPJSVD_ERR_INVALID_ARG;
    g_mpj_diag = h->opts.diag_timing;
    g_mpj_qrp_pe = h->opts.qrp_panel_stages;
    const bool root = !h->comm.active() || h->comm.rank == 0;
    if (root && (!A || !U || !S || !V)) return MPJSVD_ERR_INVALID_ARG;
    if (n < 2 || m < n || (root && (lda < m || ldu < m || ldv < n))) return MPJSVD_ERR_INVALID_ARG;
    if (m > 16384 || n > 8192) return MPJSVD_ERR_NOT_SUPPORTED;   // QRP: n <= 16 rows x 512 threads
    if (cudaSetDevice(h->device) != cudaSuccess) { cudaGetLastError(); return MPJSVD_ERR_CUDA; }
    int rc = factor_impl(h, A, m, n, lda, U, ldu, S, V, ldv, stats);
    if (rc == MPJSVD_ERR_CUDA || rc == MPJSVD_ERR_OUT_OF_MEMORY) cudaGetLastError();
    return rc;
}

int mpjsvd_gemm_f64(mpjsvd_handle h, int32_t transa, int32_t transb, int64_t M, int64_t N, int64_t K, double alpha,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
    if (!h || !A || !B || !C) return MPJSVD_ERR_INVALID_ARG;
    g_mpj_diag = h->opts.diag_timing;
    g_mpj_qrp_pe = h->opts.qrp_panel_stages;
    MPJ_TRY(ensure(h, S_GEMMWS, sizeof(double) * (size_t)(M > 0 ? M : 1) * (N > 0 ? N : 1) * 16));
    gemm_set_workspace(P<double>(h, S_GEMMWS), h->cap[S_GEMMWS] / sizeof(double));
    int rc = gemm_f64(transa, transb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, h->stream);
    if (rc) return rc;
    return cudaStreamSynchronize(h->stream) == cudaSuccess ? 0 : MPJSVD_ERR_CUDA;
}

int mpjsvd_inner_solve(mpjsvd_handle h, int32_t is_f64, void* G, void* E, int32_t w, int32_t count, double tol_in,
                       int32_t max_inner, int32_t* rotations) {
    if (!h || !G || !E || w < 1 || w > 64 || count < 1) return MPJSVD_ERR_INVALID_ARG;
    g_mpj_diag = h->opts.diag_timing;
    g_mpj_qrp_pe = h->opts.qrp_panel_stages;
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
    g_mpj_diag = h->opts.diag_timing;
    g_mpj_qrp_pe = h->opts.qrp_panel_stages;
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
    if (pivot == 3) {                 // mixed-precision RRQR (Alg. 4): fp32 pivots, fp64 QR of A P
        int g = 0, no = 0;
        MPJ_TRY(qrp_lazy_grid((int)m, (int)n, &g, &no));
        MPJ_TRY(ensure(h, S_QRPW, sizeof(double) * qrp_lazy_work_doubles((int)n, g)));
        MPJ_TRY(ensure(h, S_X32, sizeof(float) * (size_t)m_pad * n));
        MPJ_TRY(ensure(h, S_TAU_T, sizeof(double) * (size_t)n));
        MPJ_TRY(ensure(h, S_SCAL, sizeof(double) * 8));
        MPJ_TRY(ensure(h, S_WY, sizeof(double) * apply_q_work_elems(m_pad, n)));
        double* sc = P<double>(h, S_SCAL);
        MPJ_TRY(maxabs(Aw, m_pad, m_pad, n, sc + 4, st));
        MPJ_TRY(downcast_scaled(Aw, m_pad, P<float>(h, S_X32), m_pad, m_pad, (int)n, sc + 4, st));
        MPJ_TRY(qrp_lazy_f32(P<float>(h, S_X32), m_pad, (int)m, (int)n, reinterpret_cast<float*>(P<double>(h, S_TAU_T)),
                             qw, reinterpret_cast<float*>(P<double>(h, S_QRPW)), phys, st));
        MPJ_TRY(gather_cols(Aw, m_pad, phys, P<double>(h, S_TMP2), m_pad, m_pad, (int)n, st));
        MPJ_TRY(qr_blocked(P<double>(h, S_TMP2), m_pad, (int)m, (int)n, tau, qw, P<double>(h, S_WY), st));
        MPJ_CUDA_TRY(cudaMemcpy2DAsync(A, sizeof(double) * lda, P<double>(h, S_TMP2), sizeof(double) * m_pad,
                                       sizeof(double) * m, n, cudaMemcpyDefault, st));
        if (perm) MPJ_CUDA_TRY(cudaMemcpyAsync(perm, phys, sizeof(int) * n, cudaMemcpyDefault, st));
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
        return 0;
    } else if (pivot == 2) {          // unblocked reference kernel (tests)
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
    g_mpj_diag = h->opts.diag_timing;
    g_mpj_qrp_pe = h->opts.qrp_panel_stages;
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

int mpjsvd_switch_u(mpjsvd_handle h, const double* X, int64_t n, int64_t ldx, const double* Ulow, int64_t ldu,
                    double* Q, int64_t ldq, int32_t x_lower) {
    if (!h || !X || !Ulow || !Q || n < 1 || ldx < n || ldu < n || ldq < n) return MPJSVD_ERR_INVALID_ARG;
    g_mpj_diag = h->opts.diag_timing;
    g_mpj_qrp_pe = h->opts.qrp_panel_stages;
    gemm_set_workspace(nullptr, 0);
    cudaStream_t st = h->stream;
    const long long n_pad = round_up(n, 32);
    const size_t nn = (size_t)n_pad * n;
    MPJ_TRY(ensure(h, S_TMP1, sizeof(double) * 3 * nn));
    MPJ_TRY(ensure(h, S_TMP2, sizeof(double) * nn));
    MPJ_TRY(ensure(h, S_TAU_U, sizeof(double) * n));
    MPJ_TRY(ensure(h, S_WY, sizeof(double) * apply_q_work_elems(n_pad, n)));
    QrWork qw;
    MPJ_TRY(ensure_qr_work(h, (int)n, (int)n, qw));
    double* Xw = P<double>(h, S_TMP1);
    double* Uw = Xw + nn;
    double* Zw = Uw + nn;
    double* Qw = P<double>(h, S_TMP2);
    MPJ_CUDA_TRY(cudaMemsetAsync(Xw, 0, sizeof(double) * 2 * nn, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(Xw, sizeof(double) * n_pad, X, sizeof(double) * ldx, sizeof(double) * n, n,
                                   cudaMemcpyDefault, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(Uw, sizeof(double) * n_pad, Ulow, sizeof(double) * ldu, sizeof(double) * n, n,
                                   cudaMemcpyDefault, st));
    MPJ_TRY(switch_u_inplace(h, Xw, Uw, Zw, Qw, n_pad, (int)n, x_lower != 0, qw, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(Q, sizeof(double) * ldq, Qw, sizeof(double) * n_pad, sizeof(double) * n, n,
                                   cudaMemcpyDefault, st));
    MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    return 0;
}

int mpjsvd_qrsvd32(mpjsvd_handle h, const float* X32, int64_t n, int64_t ldx, double* U, int64_t ldu, float* S) {
    if (!h || !X32 || !U || n < 1 || ldx < n || ldu < n) return MPJSVD_ERR_INVALID_ARG;
    if (n > 16384) return MPJSVD_ERR_NOT_SUPPORTED;
    g_mpj_diag = h->opts.diag_timing;
    g_mpj_qrp_pe = h->opts.qrp_panel_stages;
    if (cudaSetDevice(h->device) != cudaSuccess) { cudaGetLastError(); return MPJSVD_ERR_CUDA; }
    gemm_set_workspace(nullptr, 0);
    cudaStream_t st = h->stream;
    const long long n_pad = round_up(n, 32);
    const size_t nn = (size_t)n_pad * n;
    MPJ_TRY(ensure(h, S_TMP1, sizeof(double) * 3 * nn));
    MPJ_TRY(ensure(h, S_TMP2, sizeof(float) * nn));
    MPJ_TRY(ensure(h, S_WY, sizeof(double) * apply_q_work_elems(n_pad, n)));
    MPJ_TRY(ensure(h, S_SVDWS, qrsvd32_work_bytes((int)n)));
    MPJ_TRY(ensure(h, S_FLAGS, sizeof(int) * 8));
    MPJ_TRY(ensure(h, S_SCAL, sizeof(double) * 8 + sizeof(float) * (size_t)n));
    double* Uw = P<double>(h, S_TMP1);
    double* UBw = Uw + nn;
    double* Pw = UBw + nn;
    float* Xw = P<float>(h, S_TMP2);
    int* flags = P<int>(h, S_FLAGS);
    MPJ_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int) * 8, st));
    MPJ_CUDA_TRY(cudaMemsetAsync(Xw, 0, sizeof(float) * nn, st));
    MPJ_CUDA_TRY(cudaMemsetAsync(Uw, 0, sizeof(double) * nn, st));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(Xw, sizeof(float) * n_pad, X32, sizeof(float) * ldx, sizeof(float) * n, n,
                                   cudaMemcpyDefault, st));
    MPJ_TRY(qrsvd32(Xw, n_pad, (int)n, Uw, n_pad, UBw, Pw, n_pad, P<void>(h, S_SVDWS), P<double>(h, S_WY),
                    flags + 1, st, reinterpret_cast<float*>(P<double>(h, S_SCAL) + 8)));
    MPJ_CUDA_TRY(cudaMemcpy2DAsync(U, sizeof(double) * ldu, Uw, sizeof(double) * n_pad, sizeof(double) * n, n,
                                   cudaMemcpyDefault, st));
    int hf = 0;
    MPJ_CUDA_TRY(cudaMemcpyAsync(&hf, flags + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    if (hf) return MPJSVD_ERR_RANK_DEFICIENT;
    if (S) {
        MPJ_CUDA_TRY(cudaMemcpyAsync(S, reinterpret_cast<float*>(P<double>(h, S_SCAL) + 8), sizeof(float) * n,
                                     cudaMemcpyDefault, st));
        MPJ_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return 0;
}

int mpjsvd_apply_q(mpjsvd_handle h, const double* Vr, int64_t m, int64_t k, int64_t ldv, const double* tau, double* C,
                   int64_t ldc, int64_t ncols) {
    if (!h || !Vr || !tau || !C || k > m || ldv < m || ldc < m) return MPJSVD_ERR_INVALID_ARG;
    g_mpj_diag = h->opts.diag_timing;
    g_mpj_qrp_pe = h->opts.qrp_panel_stages;
    gemm_set_workspace(nullptr, 0);
    MPJ_TRY(ensure(h, S_WY, sizeof(double) * apply_q_work_elems(m, ncols)));
    MPJ_TRY(apply_q_wy(Vr, m, (int)k, ldv, tau, C, ldc, ncols, P<double>(h, S_WY), h->stream));
    MPJ_CUDA_TRY(cudaStreamSynchronize(h->stream));
    return 0;
}

}  // extern "C"
