"""The multi-GPU shard plan on CPU.

The sharded engine of libmpjsvd.so drives its kernels and NCCL transfers from
the host-side plan exported as mpjsvd_plan_* (include/mpjsvd.h).  These tests
need no GPU:
  * the plan reproduces the circle-method schedule of reading c-4 (the pair
    set of every round, every block pair exactly once per sweep, blocks back
    home after a sweep) for several (N_b, G), including odd N_b and padding;
  * buffer bookkeeping: a rank never holds one buffer twice, receives at most
    two blocks per round into free buffers, and sends what it owns;
  * the exchange logic with real message passing: world-size 2 and 4
    torch.distributed/gloo processes each hold their shard of a matrix, run a
    block one-sided Jacobi pair operation (numpy) on the plan's pairs, move
    blocks with isend/irecv exactly as the plan says, and the gathered result
    is bitwise identical to the one-process run over the same schedule.
"""
import os
import socket

import numpy as np
import pytest

import paper_2209_04626_b200 as mp


def rr_slot(r, j, M):
    """Closed form of the circle method (reading c-4)."""
    return 0 if j == 0 else 1 + ((j - 1 - r) % (M - 1))


CASES = [(8, 1), (7, 1), (1, 1), (256, 8), (256, 4), (64, 2), (10, 2), (5, 2), (6, 3), (3, 4), (33, 8)]


@pytest.mark.parametrize("nblk,G", CASES)
def test_plan_matches_circle_schedule(nblk, G):
    p = mp.ShardPlan(nblk, G)
    M, k = p.M, p.k
    assert M % (2 * G) == 0 and M >= nblk and M == 2 * G * k
    if G == 1:
        assert M == max(2, nblk + (nblk & 1))
    for sweep in range(2):
        seen = set()
        for r in range(M - 1):
            got = []
            for g in range(G):
                bufs = set()
                for (b0, b1, k0, k1) in p.pairs(g):
                    assert k0 < k1
                    assert b0 != b1 and b0 not in bufs and b1 not in bufs
                    bufs |= {b0, b1}
                    got.append((k0, k1))
            want = sorted(tuple(sorted((rr_slot(r, i, M), rr_slot(r, M - 1 - i, M)))) for i in range(M // 2))
            assert sorted(got) == want, (sweep, r)
            seen |= set(got)
            moves = p.advance()
            nin = [0] * G
            nout = [0] * G
            for (blk, sg, sb, dg, db) in moves:
                assert sg != dg
                nout[sg] += 1
                nin[dg] += 1
            assert all(x <= 2 for x in nin) and nin == nout
            if G == 1:
                assert moves == []
        # every unordered pair of the M positions' blocks exactly once per sweep
        assert len(seen) == M * (M - 1) // 2
        # after a sweep every block is back on the rank that owns its home position
        for blk in range(nblk):
            g, _ = p.locate(blk)
            home = blk if blk < M // 2 else M - 1 - blk
            assert g == home // k


def _pair_op(x0, x1):
    """A one-sided Jacobi step on W = [x0 x1] (numpy, fp64): W <- W Q with Q the
    eigenvectors of W^T W (deterministic on fixed inputs)."""
    W = np.concatenate([x0, x1], axis=1)
    if W.shape[1] == 0:
        return x0, x1
    _, Q = np.linalg.eigh(W.T @ W)
    Wn = W @ Q
    return Wn[:, :x0.shape[1]].copy(), Wn[:, x0.shape[1]:].copy()


def _run_sharded(rank, world, nblk, b, rows, sweeps, port, out_path):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        X = np.random.default_rng(5).standard_normal((rows, nblk * b - 3))    # ragged last block
        n = X.shape[1]
        p = mp.ShardPlan(nblk, world)
        width = lambda blk: 0 if blk >= nblk else min(b, n - blk * b)
        # initial buffers: local position l holds the block at its home position, buffer l
        bufs = {}
        for l in range(2 * p.k):
            pos = rank * p.k + l if l < p.k else p.M - 1 - (rank * p.k + l - p.k)
            w = width(pos)
            bufs[l] = X[:, pos * b:pos * b + w].copy() if w else np.zeros((rows, 0))
        for _ in range(sweeps):
            for _ in range(p.M - 1):
                for (b0, b1, k0, k1) in p.pairs(rank):
                    bufs[b0], bufs[b1] = _pair_op(bufs[b0], bufs[b1])
                moves = p.advance()
                reqs, recvd = [], []
                for (blk, sg, sb, dg, db) in moves:       # canonical order, as the engine posts them
                    w = width(blk)
                    if sg == rank:
                        t = torch.from_numpy(np.ascontiguousarray(bufs.pop(sb)))
                        reqs.append(dist.isend(t, dg))
                    elif dg == rank:
                        t = torch.empty((rows, w), dtype=torch.float64)
                        reqs.append(dist.irecv(t, sg))
                        recvd.append((db, t))
                for q in reqs:
                    q.wait()
                for db, t in recvd:
                    bufs[db] = t.numpy()
        # gather to rank 0
        res = np.zeros_like(X)
        for blk in range(nblk):
            g, bf = p.locate(blk)
            w = width(blk)
            if g == rank and rank == 0:
                res[:, blk * b:blk * b + w] = bufs[bf]
            elif g == rank:
                dist.send(torch.from_numpy(np.ascontiguousarray(bufs[bf])), 0)
            elif rank == 0:
                t = torch.empty((rows, w), dtype=torch.float64)
                dist.recv(t, g)
                res[:, blk * b:blk * b + w] = t.numpy()
        if rank == 0:
            np.save(out_path, res)
    finally:
        dist.destroy_process_group()


def _single(nblk, b, rows, sweeps):
    X = np.random.default_rng(5).standard_normal((rows, nblk * b - 3))
    n = X.shape[1]
    p = mp.ShardPlan(nblk, 1)                       # buffer j = block j
    blocks = {j: X[:, j * b:min(n, j * b + b)].copy() for j in range(nblk)}
    for j in range(nblk, p.M):
        blocks[j] = np.zeros((rows, 0))
    for _ in range(sweeps):
        for _ in range(p.M - 1):
            for (b0, b1, k0, k1) in p.pairs(0):
                blocks[b0], blocks[b1] = _pair_op(blocks[b0], blocks[b1])
            assert p.advance() == []
    return np.concatenate([blocks[j] for j in range(nblk)], axis=1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,nblk", [(2, 8), (4, 8), (2, 7), (4, 10)])
def test_gloo_sharded_exchange_bitwise_equals_single(tmp_path, world, nblk):
    import torch.multiprocessing as tmp
    b, rows, sweeps = 4, 24, 2
    out = str(tmp_path / "res.npy")
    tmp.spawn(_run_sharded, args=(world, nblk, b, rows, sweeps, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    want = _single(nblk, b, rows, sweeps)
    if (nblk + (nblk & 1)) % (2 * world) == 0:
        assert np.array_equal(got, want)            # same schedule: bitwise
    else:
        # padded schedule (M rounded up to a multiple of 2G): a different but
        # equally valid ordering -- the column space and norms agree
        assert np.isclose(np.linalg.norm(got), np.linalg.norm(want))
    # the pair operations really ran (columns mutually closer to orthogonal)
    X = np.random.default_rng(5).standard_normal((rows, nblk * b - 3))
    assert not np.allclose(got, X)
