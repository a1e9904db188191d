"""The N > 1 path on CPU: world-size-2 gloo ranks, each evaluating the shard
the library's host-side shard map gives it (block-cyclic chunks of 65536
indices) with the CPU oracle, then one allreduce(MIN) of the packed
(makespan << bits | index) key — the same reduction the GPU path performs
over NCCL. The result must equal the single-process exhaustive search."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2509_23722_b200 import adaptis as A
from paper_2509_23722_b200 import workloads as W


def _medium_problem():
    """~195K candidates (3 shard chunks), each a tiny simulation."""
    rng = W.SplitMix64(4242)
    pr = W.random_problem(rng, 60, 2, 2, tmax=30, cmax=6, bytes_max=9, cap=700)
    sp = W.Space([W.Group(1, W.FULL, combo_mask=0xF), W.Group(2, W.FULL, combo_mask=0x3F)])
    return pr, sp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_map_partitions_the_space():
    pr, sp = _medium_problem()
    N = A.space_size(pr, sp)
    assert N > 2 * 65536
    for world in (1, 2, 3, 4, 8):
        parts = [A.shard_indices(pr, sp, r, world) for r in range(world)]
        allidx = np.concatenate(parts)
        assert allidx.size == N
        assert np.array_equal(np.sort(allidx), np.arange(N, dtype=np.uint64))
        for r, part in enumerate(parts):  # block-cyclic: chunk k belongs to rank k mod world
            assert np.all((part >> np.uint64(16)) % np.uint64(world) == np.uint64(r))


def _rank_main(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        pr, sp = _medium_problem()
        N = A.space_size(pr, sp)
        idx = A.shard_indices(pr, sp, rank, world)
        ev = O.eval_indices(pr, sp, idx, nthreads=2)
        ok = ev["status"] == 0
        key = (1 << 63) - 1
        if ok.any():
            ms = ev["makespan"][ok].astype(object)
            ii = idx[ok].astype(object)
            key = min(A.pack_key(int(m), int(i), N) for m, i in zip(ms, ii))
        t = torch.tensor([key], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)  # the one collective of the search
        q.put((rank, int(t.item()), int(idx.size)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_search_matches_single_process():
    pr, sp = _medium_problem()
    N = A.space_size(pr, sp)
    want = O.search(pr, sp, prune=False, nthreads=4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    keys = {k for _, k, _ in res}
    assert len(keys) == 1  # every rank returns the same winner
    key = keys.pop()
    bits = max(1, (N - 1).bit_length())
    assert (key & ((1 << bits) - 1), key >> bits) == (want["index"], want["makespan"])
    assert sum(n for _, _, n in res) == N
