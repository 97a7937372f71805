// shard.h -- host-side plan of the block round-robin Jacobi schedule over G
// shards (GPUs), SURVEY.md 8(e) / DESIGN.md "Multi-GPU".  Pure host C++ (no
// CUDA): the engine (mpjsvd.cu) drives its kernels and transfers from it, and
// the C-ABI exports it (mpjsvd_plan_*) so the CPU tests can run the same
// exchange logic over torch.distributed/gloo.
//
// Schedule (reading c-4, PAPER.md:262-274 replaced by the circle method): M
// positions; round r pairs position i with M-1-i; after a round the content
// of position p moves to next(p) = p+1 (1 <= p <= M-2), M-1 -> 1, 0 stays.
// Position j holds block j at the start of every sweep (the shift has period
// M-1), so the block pair of round r is (rr_slot(r,i), rr_slot(r,M-1-i)).
//
// Sharding: rank g owns the k = M/(2G) pairs i in [g k, (g+1) k): local
// position l < k is global position g k + l (top), local l >= k is global
// M-1-(g k + l-k) (bottom); local pair t is (t, k+t).  Each rank stores its
// 2k blocks in 2k+2 buffers (two spares receive the <= 2 blocks that arrive
// from neighbours each round, the sent buffers become the spares).  A move
// to another rank is a transfer; a move inside a rank is a rename.  With one
// rank and `contiguous`, buffer j is block j of the matrix itself (nothing
// ever moves).  M is padded to a multiple of 2G with empty (bye) blocks.
#pragma once
#include <vector>

namespace mpj {

class ShardPlan {
public:
    int nblk = 0, G = 1, M = 2, k = 1, nbuf = 2;
    bool contiguous = true;

    struct Pair { int buf0, buf1, blk0, blk1; };      // blk0 < blk1
    struct Move { int blk, src_rank, src_buf, dst_rank, dst_buf; };

    // returns 0, or -1 on bad arguments
    int init(int nblk_, int G_, bool contiguous_) {
        if (nblk_ < 1 || G_ < 1 || (contiguous_ && G_ != 1)) return -1;
        nblk = nblk_;
        G = G_;
        contiguous = contiguous_;
        M = nblk + (nblk & 1);
        if (M < 2) M = 2;
        if (G > 1) M = ((nblk + 2 * G - 1) / (2 * G)) * (2 * G);
        k = M / (2 * G);
        nbuf = contiguous ? M : 2 * k + 2;
        loc2buf.assign((size_t)G * 2 * k, -1);
        buf2blk.assign((size_t)G * nbuf, -1);
        freebuf.assign(G, std::vector<int>());
        for (int g = 0; g < G; ++g)
            for (int l = 0; l < 2 * k; ++l) {
                const int p = gpos(g, l);
                const int buf = contiguous ? p : l;
                loc2buf[(size_t)g * 2 * k + l] = buf;
                buf2blk[(size_t)g * nbuf + buf] = p;       // block p sits at position p
            }
        if (!contiguous)
            for (int g = 0; g < G; ++g) freebuf[g] = {2 * k + 1, 2 * k};
        return 0;
    }

    int gpos(int g, int l) const { return l < k ? g * k + l : M - 1 - (g * k + (l - k)); }
    void owner(int p, int& g, int& l) const {
        if (p < M / 2) { g = p / k; l = p % k; }
        else { const int q = M - 1 - p; g = q / k; l = k + q % k; }
    }
    static int next_pos(int p, int M_) { return p == 0 ? 0 : (p == M_ - 1 ? 1 : p + 1); }

    int buf_at(int g, int l) const { return loc2buf[(size_t)g * 2 * k + l]; }
    int blk_of(int g, int buf) const { return buf2blk[(size_t)g * nbuf + buf]; }
    int width(int blk, int b, int n) const {
        if (blk < 0 || blk >= nblk) return 0;
        const int w = n - blk * b;
        return w < b ? w : b;
    }

    // local pair t of rank g, oriented by block id
    Pair pair(int g, int t) const {
        const int bt = buf_at(g, t), bb = buf_at(g, k + t);
        const int kt = blk_of(g, bt), kb = blk_of(g, bb);
        if (kt < kb) return {bt, bb, kt, kb};
        return {bb, bt, kb, kt};
    }

    // one shift; appends the inter-rank moves in canonical order (source rank,
    // then source local position, ascending): every rank posts its sends and
    // receives in this order, so per-peer message order matches on both sides.
    void advance(std::vector<Move>* remote) {
        std::vector<int> nl((size_t)G * 2 * k, -1);
        std::vector<std::vector<int>> freed(G);
        for (int g = 0; g < G; ++g)
            for (int l = 0; l < 2 * k; ++l) {
                const int p = gpos(g, l), p2 = next_pos(p, M);
                int g2, l2;
                owner(p2, g2, l2);
                const int buf = buf_at(g, l);
                if (g2 == g) {
                    nl[(size_t)g2 * 2 * k + l2] = buf;
                } else {
                    const int blk = blk_of(g, buf);
                    const int dst = freebuf[g2].back();
                    freebuf[g2].pop_back();
                    nl[(size_t)g2 * 2 * k + l2] = dst;
                    buf2blk[(size_t)g2 * nbuf + dst] = blk;
                    freed[g].push_back(buf);
                    if (remote) remote->push_back({blk, g, buf, g2, dst});
                }
            }
        for (int g = 0; g < G; ++g)
            for (int buf : freed[g]) {
                buf2blk[(size_t)g * nbuf + buf] = -1;
                freebuf[g].push_back(buf);
            }
        loc2buf.swap(nl);
    }

    // where block blk is now (rank, buffer); false if absent
    bool locate(int blk, int& g, int& buf) const {
        for (int gg = 0; gg < G; ++gg)
            for (int l = 0; l < 2 * k; ++l) {
                const int bf = buf_at(gg, l);
                if (blk_of(gg, bf) == blk) { g = gg; buf = bf; return true; }
            }
        return false;
    }

private:
    std::vector<int> loc2buf;                 // [G][2k] position -> buffer
    std::vector<int> buf2blk;                 // [G][nbuf] buffer -> block (-1 free)
    std::vector<std::vector<int>> freebuf;    // spare buffers per rank
};

}  // namespace mpj
