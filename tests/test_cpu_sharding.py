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


def _band_links_worker(rank, world, port, out):
    """DistLinks (rowband.py) over gloo: the carry chain, the stats gather and
    the solver-handle gather, as the row-band frame uses them under NCCL."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    from paper_2203_02300_b200.rowband import DistLinks

    g = Group(world, rank, "gloo")
    links = DistLinks(torch.distributed, world, rank, device="cpu")
    like = torch.empty(6, dtype=torch.float64)
    got = None
    if rank > 0:
        got = links.get_carry((rank, 0), like).tolist()
    if rank + 1 < world:
        links.put_carry((rank, 0), torch.arange(6, dtype=torch.float64) + 10.0 * rank)
    stats = links.gather_stats({rank: [1.0 + rank, 2.0 * rank, 3.0, -24.0 - rank]})
    blobs = links.gather_bytes({rank: bytes([rank]) * 128})
    # bands of different heights (rank + 2 rows of 5): the whole map in band order
    rows = links.gather_rows({rank: torch.full((rank + 2, 5), float(rank), dtype=torch.float32)}).tolist()
    g.close()
    out.put((rank, got, stats, blobs, rows))


def test_band_links_two_and_three_ranks():
    for world in (2, 3):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        ps = [ctx.Process(target=_band_links_worker, args=(r, world, port, q)) for r in range(world)]
        for p in ps:
            p.start()
        res = sorted(q.get(timeout=120) for _ in range(world))
        for p in ps:
            p.join(timeout=60)
            assert p.exitcode == 0
        for rank, got, stats, blobs, rows in res:
            assert rows == [[float(r)] * 5 for r in range(world) for _ in range(r + 2)]
            # band k receives exactly band k-1's carry
            assert got == (None if rank == 0 else [10.0 * (rank - 1) + i for i in range(6)])
            # every rank holds every band's statistics, rank-ordered
            assert stats == [[1.0 + r, 2.0 * r, 3.0, -24.0 - r] for r in range(world)]
            assert blobs == [bytes([r]) * 128 for r in range(world)]
