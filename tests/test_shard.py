"""CPU tests of the N>1 path with a world-size-2 gloo group: contiguous
query shards (the C ABI's split) searched independently and gathered by
plain copy reproduce the full-batch search exactly; the control-plane
collectives (operating-point broadcast, max-over-ranks time) behave."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2603_06660_b200.shard import shard_bounds


def test_shard_bounds_cover_and_match_c_abi():
    for n in (0, 1, 7, 10000, 10001):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, index_path, queries, out_q):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2603_06660_b200.shard import broadcast_int, max_over_ranks

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q0, q1 = shard_bounds(len(queries), world, rank)
    ix = O.OracleIndex(index_path)
    ids, sq, n_out, st = ix.search(queries[q0:q1], 10, 50)
    gathered = [None] * world
    dist.all_gather_object(gathered, (q0, ids, sq, n_out, st))
    efs = broadcast_int(70 if rank == 0 else -1, dist)
    t = max_over_ranks(1.0 + rank, dist)
    if rank == 0:
        out_q.put((gathered, efs, t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_search_equals_full_batch(built):
    fx = built("euc48")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fx["index"], fx["queries"], q))
             for r in range(world)]
    for p in procs:
        p.start()
    gathered, efs, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert efs == 70 and t == 2.0
    gathered.sort(key=lambda g: g[0])
    ids = np.concatenate([g[1] for g in gathered])
    sq = np.concatenate([g[2] for g in gathered])
    st = np.concatenate([g[4] for g in gathered])
    from oracle import oracle as O
    want = O.OracleIndex(fx["index"]).search(fx["queries"], 10, 50)
    assert np.array_equal(ids, want[0]) and np.array_equal(sq, want[1]) and np.array_equal(st, want[3])
