"""Multi-GPU plumbing of the frame loop.

Streams shard naturally: every rank owns its own pipeline streams (keyframe
window and d_pre chain), so there is no data-path collective. torch.distributed
is used only for the barrier around the timed region and the max-over-ranks
time. NCCL on GPUs, gloo for the CPU tests of this logic.
"""
import os

import torch


def world_from_env():
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def stream_seeds(rank, streams, base=61, stride=97):
    """Synthetic-video seeds of a rank's streams: disjoint across ranks for any
    streams < stride, so no two streams of the job process the same frames."""
    if streams >= stride:
        raise ValueError("at most %d streams per rank" % (stride - 1))
    return [base + stride * rank + s for s in range(streams)]


class Group:
    """The job's process group (None when world == 1)."""

    def __init__(self, world, local, backend=None):
        self.world = world
        self.dist = None
        if world > 1:
            import torch.distributed as dist

            backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(backend)
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max_over_ranks(self, values, device="cpu"):
        """Element-wise max of a list of floats over all ranks (timing: the job
        is as slow as its slowest rank)."""
        t = torch.tensor(values, dtype=torch.float64, device=device)
        if self.dist:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()
            self.dist = None
