"""World-size-2 CPU test of the sharded path's host logic (gloo).

Each rank takes its contiguous share of a segment's combination space
(cfp_shard_range, adversarial cut points included), computes its local
(A, I) with the oracle on that range only, packs (cost, index) keys with the
library's cfp_pack_keys and all-reduces the keys with MIN.  The merged
tables must equal the single-process oracle tables bit for bit -- the
property the NCCL merge inside libcfp relies on (lexicographic min is
associative and commutative, so any partition and any world size agree).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

INF64 = (1 << 64) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, seeds, align, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2504_00598_b200 import cfp
        from synth import generators as G
        bad = []
        for seed in seeds:
            p = G.tiny_random(seed, mode=("ties", "random")[seed % 2], max_plans=None, max_k=4,
                              max_d=4)
            for tr in range(len(p.transitions)):
                S = p.num_combinations(p.transitions[tr].type)
                lo, hi = cfp.shard_range(S, align, world, rank)
                A, I = O.segment_table_range(p, tr, lo, hi, nthreads=1)
                bits = max(1, int(S).bit_length())
                keys = cfp.pack_keys(A.ravel(), I.ravel(), bits)
                # gloo has no unsigned 64-bit MIN: flip the sign bit (order-preserving)
                t = torch.from_numpy((keys ^ np.uint64(1 << 63)).view(np.int64).copy())
                dist.all_reduce(t, op=dist.ReduceOp.MIN)
                merged = t.numpy().view(np.uint64) ^ np.uint64(1 << 63)
                A2, I2 = cfp.unpack_keys(merged, bits)
                A0, I0 = O.segment_table(p, tr, nthreads=1)
                if not (np.array_equal(A2, A0.ravel()) and np.array_equal(I2, I0.ravel())):
                    bad.append((seed, tr))
        q.put((rank, bad))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("align", [1, 3])
def test_two_rank_merge_equals_single(align):
    from oracle import oracle as O
    O.build()
    from paper_2504_00598_b200 import build as B
    B.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    seeds = list(range(300, 340))
    procs = [ctx.Process(target=_worker, args=(r, world, port, seeds, align, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, bad in res:
        assert not bad, (rank, bad)


def _worker_two_round(rank, world, port, seeds, q):
    """The product's merge (cfp_host.cu execute / merge_ranks): round 1 MIN
    all-reduce of the rank-local bucket minima A; round 2 each rank masks its
    least index to INF where its local A differs from the global A (mask_idx
    kernel), MIN all-reduce of the masked indices.  A, I must equal the
    single-process oracle for every world size and cut."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2504_00598_b200 import cfp
        from synth import generators as G
        flip = np.uint64(1 << 63)

        def umin(a):
            t = torch.from_numpy((a ^ flip).view(np.int64).copy())
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            return t.numpy().view(np.uint64) ^ flip

        bad = []
        for seed in seeds:
            p = G.tiny_random(seed, mode=("ties", "random", "nearmax")[seed % 3], max_plans=None, max_k=4, max_d=4)
            for tr in range(len(p.transitions)):
                S = p.num_combinations(p.transitions[tr].type)
                lo, hi = cfp.shard_range(S, 1, world, rank)
                A, I = O.segment_table_range(p, tr, lo, hi, nthreads=1)
                A, I = A.ravel(), I.ravel()
                Ag = umin(A)                                         # round 1
                Im = np.where(A == Ag, I, np.uint64(INF64))          # mask_idx_kernel
                Ig = umin(Im)                                        # round 2
                Ig = np.where(Ag == np.uint64(INF64), np.uint64(INF64), Ig)
                A0, I0 = O.segment_table(p, tr, nthreads=1)
                if not (np.array_equal(Ag, A0.ravel()) and np.array_equal(Ig, I0.ravel())):
                    bad.append((seed, tr))
        q.put((rank, bad))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_two_round_merge_equals_single(world):
    """The exact two-round (cost, then least index) merge libcfp runs with
    NCCL, on gloo with 2 and 3 ranks."""
    from oracle import oracle as O
    O.build()
    from paper_2504_00598_b200 import build as B
    B.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    seeds = list(range(400, 430))
    procs = [ctx.Process(target=_worker_two_round, args=(r, world, port, seeds, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, bad in res:
        assert not bad, (rank, bad)
