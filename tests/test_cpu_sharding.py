"""The multi-GPU plumbing of the frame loop (paper_2203_02300_b200/sharding.py)
on CPU: world_size 2 over gloo, as bench.py runs it under torchrun with NCCL."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2203_02300_b200.sharding import Group, stream_seeds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, streams, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    g = Group(world, rank, "gloo")
    seeds = stream_seeds(rank, streams)
    g.barrier()
    # each rank reports a different time; the job's is the max over ranks
    mx = g.max_over_ranks([10.0 + rank, 5.0 * (world - rank)])
    gathered = [None] * world
    torch.distributed.all_gather_object(gathered, seeds)
    g.close()
    out.put((rank, mx, gathered))


def test_two_rank_stream_sharding():
    world, streams = 2, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, streams, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, gathered in res:
        assert mx == [11.0, 10.0]  # max over ranks, element-wise
        flat = [s for seeds in gathered for s in seeds]
        assert len(flat) == world * streams and len(set(flat)) == len(flat)  # disjoint streams
        assert gathered[rank] == stream_seeds(rank, streams)


def test_single_rank_is_a_no_op():
    g = Group(1, 0)
    g.barrier()
    assert g.max_over_ranks([1.5, 2.5]) == [1.5, 2.5]
    g.close()


def test_stream_seed_bounds():
    assert stream_seeds(0, 2) == [61, 62] and stream_seeds(1, 2) == [158, 159]
    with pytest.raises(ValueError):
        stream_seeds(0, 97)
