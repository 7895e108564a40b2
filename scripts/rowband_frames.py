"""Times the row-band frame loop (paper_2203_02300_b200/rowband.py) at BASELINE
config D (3840x2160, D=256) -- or any size -- and prints one JSON line.

  python scripts/rowband_frames.py --bands G        # all G bands on this GPU
  torchrun --nproc-per-node G scripts/rowband_frames.py  # one band per GPU

With one GPU the bands run one after another (the solve as one launch over
all bands), so the time is the sum of the bands' work: it measures the cost
of banding (halo recompute, carry chain, band solve), not the multi-GPU
speed-up. Frames are synthetic (paper_2203_02300_b200/synth.py), 8-bit."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.rowband import DistLinks, LocalLinks, RowBandFrames  # noqa: E402
from paper_2203_02300_b200.sharding import Group, world_from_env  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=3840)
    ap.add_argument("--height", type=int, default=2160)
    ap.add_argument("--disparities", type=int, default=256)
    ap.add_argument("--bands", type=int, default=1)
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    world, rank, local = world_from_env()
    torch.cuda.set_device(local)
    group = Group(world, local)
    W, H = args.width, args.height
    cfg = Config(d_max=args.disparities - 1)
    links = DistLinks(group.dist, world, rank, device="cuda") if world > 1 else LocalLinks(args.bands)
    rb = RowBandFrames(W, H, cfg, links)
    vid = StereoVideo(W, H)
    n = args.warmup + args.frames + 2
    frames = [vid.frame(i) for i in range(n)]
    ing = []
    for l8, r8 in frames:
        lf, lq = dco.ingest_gray8(torch.from_numpy(l8).cuda())
        _, rq = dco.ingest_gray8(torch.from_numpy(r8).cuda())
        ing.append((lf, lq, rq, lf.unsqueeze(-1).expand(H, W, 3).contiguous()))
    times = []
    for i in range(1, n - 1):
        group.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rb.frame(ing[i - 1][1], ing[i][1], ing[i + 1][1], ing[i][0], ing[i][2], ing[i][3])
        b.record()
        torch.cuda.synchronize()
        if i > args.warmup:
            times.append(a.elapsed_time(b))
        if i == args.warmup:
            rb.timing = True
    rb.timing = False
    ms = group.max_over_ranks([float(np.mean(times))])[0]
    spans = {k: round(v / len(times), 3) for k, v in rb.spans.items()}
    if rank == 0:
        print(json.dumps({"workload": "row-band DCO frame %dx%d D=%d" % (W, H, args.disparities),
                          "bands": links.bands, "gpus": world, "ms_per_frame": ms, "frames_per_s": 1000.0 / ms,
                          "iterations": rb.iterations, "frames": len(times), "spans_ms": spans,
                          "mode": "one band per GPU (NCCL + peer memory)" if world > 1 else
                          "all bands on one GPU (sequential bands, one solve launch)"}))
    rb.close()
    group.close()


if __name__ == "__main__":
    main()
