"""Multi-rank path on CPU (gloo, world_size 2): shard ownership, seeded input
generation per global codeword index, and the max-over-ranks timing reduce."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_1404_3458_b200.dist import env_rank, max_over_ranks, shard_range

    r, w, _ = env_rank()
    lo, hi = shard_range(r, w, 3)
    msgs = O.gen_symbols(1404345803, 8, lo, hi - lo, 128)
    orc = O.Oracle(8)
    par = orc.encode_batch(128, msgs, 1)
    # the slowest rank defines the step time
    t = max_over_ranks([0.5 + r, 10.0 - r])
    gathered = [None] * w
    dist.all_gather_object(gathered, (lo, hi, msgs.tolist(), par.tolist(), t))
    if r == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (lo0, hi0, m0, p0, t0), (lo1, hi1, m1, p1, t1) = res
    assert (lo0, hi0, lo1, hi1) == (0, 3, 3, 6)  # disjoint, contiguous, weak scaling
    assert t0 == t1 == [1.5, 10.0]
    from oracle import oracle as O
    full = O.gen_symbols(1404345803, 8, 0, 6, 128)
    np.testing.assert_array_equal(np.asarray(m0 + m1, np.uint16), full)
    orc = O.Oracle(8)
    np.testing.assert_array_equal(np.asarray(p0 + p1, np.uint16), orc.encode_batch(128, full, 2))


def test_split_range_covers_total():
    from paper_1404_3458_b200.dist import split_range
    for total in (4096, 4097, 5):
        for world in (1, 2, 3, 8):
            spans = [split_range(r, world, total) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(ValueError):
        from paper_1404_3458_b200.dist import shard_range
        shard_range(2, 2, 4)
