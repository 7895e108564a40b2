"""Row bands across real GPUs (BASELINE config D's decomposition):
one process per GPU, DistLinks over NCCL for the aggregation carry chain,
the sparse statistics and the solver handles, and the band solve's
reduction and p halo through CUDA-IPC peer memory (dco_band_solver_export /
connect, pcg_band.cuh). Skipped with fewer than two visible GPUs; the same
kernels and exchange protocol run on one GPU in test_gpu_rowband.py and
test_gpu_band_solve.py, and the torch.distributed links over gloo in
tests/test_cpu_sharding.py.

The bar is the reference's (any decomposition equals the
sequential order): sparse depth bit-exact and dense depth within the solver
tolerance of oracle/_ref's pipeline frame, on every rank."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs two GPUs")]

W, H, D = 640, 360, 48


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(ref):
    from tests.inputs import scene

    fs = [scene(ref, W, H, index=i, seed=91) for i in range(4)]
    q = [ref.downsample_half(f["left"]) for f in fs]
    return fs, q


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(rank)
    import torch.distributed as dist

    from oracle import ref
    from paper_2203_02300_b200.config import Config
    from paper_2203_02300_b200.rowband import DistLinks, RowBandFrames

    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    cfg = Config(d_max=D - 1)
    fs, q = _inputs(ref)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    rb = RowBandFrames(W, H, cfg, DistLinks(dist, world, rank, device="cuda"))
    res = []
    for i in (1, 2):
        mid = fs[i]
        rq = ref.downsample_half(mid["right"])
        got = rb.frame(T(q[i - 1]), T(q[i]), T(q[i + 1]), T(mid["left"]), T(rq),
                       T(np.repeat(mid["left"][:, :, None], 3, 2)))
        g = got[rank]
        res.append((g["rows"], g["dense"].cpu().numpy(), g["sparse"].cpu().numpy(), rb.iterations))
    rb.close()
    dist.barrier()
    dist.destroy_process_group()
    out.put((rank, res))


@pytest.mark.parametrize("world", [2])
def test_rowband_frames_across_gpus(ref, world):
    import torch.multiprocessing as mp

    from paper_2203_02300_b200.config import Config
    from tests.test_gpu_densify import MAX_ABS, RMS

    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, qo)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(qo.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = Config(d_max=D - 1)
    fs, q = _inputs(ref)
    prev = None
    for f, i in enumerate((1, 2)):
        mid = fs[i]
        want = ref.pipeline_frame(q[i - 1], q[i], q[i + 1], mid["left"], ref.downsample_half(mid["right"]),
                                  np.repeat(mid["left"][:, :, None], 3, 2), prev, None, None, cfg)
        iters = set()
        for rank in range(world):
            (r0, r1), dense, sparse, it = got[rank][f]
            assert np.array_equal(sparse.view(np.uint32), want["sparse"][r0:r1].view(np.uint32))
            d = np.abs(dense.astype(np.float64) - want["dense"][r0:r1])
            assert d.max() <= MAX_ABS and np.sqrt((d ** 2).mean()) <= RMS
            iters.add(it)
        assert len(iters) == 1 and abs(iters.pop() - want["iterations"]) <= 2  # every rank ran the same CG
        prev = want["dense"]
