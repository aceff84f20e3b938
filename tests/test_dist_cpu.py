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


def _bench_worker(rank, world, port, out):
    """bench.py's own rank plumbing (the functions run_codec / run_stripe use):
    shard ownership, seeded per-shard inputs, a per-rank step time reduced
    with max_over_ranks, per-rank values gathered to rank 0."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import oracle as O

    r, w, _ = bench.env_rank()
    lo, hi = bench.codeword_shard(r, w, 2)  # 2 codewords per rank (weak scaling)
    glo, ghi = bench.group_shard(r, w, 21)  # 21 stripe groups over the ranks (strong scaling)
    msgs = O.gen_symbols(bench.SEED_MSG, 8, lo, hi - lo, 128)
    par = O.Oracle(8).encode_batch(128, msgs, 1)
    step_ms = 1.0 + 0.25 * r  # the slowest rank defines the job
    mx = bench.max_over_ranks([step_ms])[0]
    per = bench.gather_to_rank0({"rank": r, "cw": (lo, hi), "groups": (glo, ghi), "ms": step_ms,
                                 "msgs": msgs.tolist(), "par": par.tolist(), "max": mx})
    if r == 0:
        out.put(per)
    dist.barrier()
    dist.destroy_process_group()


def test_eight_rank_bench_plumbing_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    W = 8
    procs = [ctx.Process(target=_bench_worker, args=(r, W, port, q)) for r in range(W)]
    for p in procs:
        p.start()
    per = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [d["rank"] for d in per] == list(range(W))
    cws = [d["cw"] for d in per]
    assert cws[0][0] == 0 and all(a[1] == b[0] for a, b in zip(cws, cws[1:])) and cws[-1][1] == 2 * W
    grs = [d["groups"] for d in per]
    assert grs[0][0] == 0 and all(a[1] == b[0] for a, b in zip(grs, grs[1:])) and grs[-1][1] == 21
    assert all(d["max"] == 1.0 + 0.25 * (W - 1) for d in per)  # max over ranks, on every rank
    from oracle import oracle as O
    import bench
    full = O.gen_symbols(bench.SEED_MSG, 8, 0, 2 * W, 128)
    np.testing.assert_array_equal(np.asarray(sum((d["msgs"] for d in per), []), np.uint16), full)
    np.testing.assert_array_equal(np.asarray(sum((d["par"] for d in per), []), np.uint16),
                                  O.Oracle(8).encode_batch(128, full, 4))
