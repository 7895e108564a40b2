"""Device-resident stream throughput at any BASELINE size on one GPU (config C:
1920x1080 D=192 frame batches; config B is bench.py's headline): S concurrent
streams, each on its own CUDA stream and context, L2 flushed before every
frame, CUDA events around K steps of S frames. Prints one JSON line.

  python scripts/throughput.py --width 1920 --height 1080 --disparities 192 --streams 4
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--disparities", type=int, default=192)
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    W, H, S = a.width, a.height, a.streams
    cfg = Config(d_max=a.disparities - 1)
    nframes = 8
    vids = [StereoVideo(W, H, seed=61 + s) for s in range(S)]
    dev = [[tuple(torch.from_numpy(x).cuda() for x in v.frame(i)) for i in range(nframes)] for v in vids]
    ts = [torch.cuda.Stream() for _ in range(S)]
    streams = []
    for s in range(S):
        with torch.cuda.stream(ts[s]):
            streams.append(dco.Stream(W, H, cfg, ctx=dco.new_context(ts[s])))
    flush = [torch.empty(160 << 20, dtype=torch.uint8, device="cuda") for _ in range(S)]
    pos = [0] * S

    def push(s, want=False):
        with torch.cuda.stream(ts[s]):
            flush[s].zero_()
            r = streams[s].push_gray8(*dev[s][pos[s] % nframes], want_result=want)
        pos[s] += 1
        return r

    for _ in range(3 + a.warmup):
        for s in range(S):
            push(s)
    torch.cuda.synchronize()
    main_s = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(main_s)
    for x in ts:
        x.wait_event(t0)
    for _ in range(a.steps):
        for s in range(S):
            push(s)
    for x in ts:
        e = torch.cuda.Event()
        e.record(x)
        main_s.wait_event(e)
    t1.record(main_s)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    it = push(0, want=True).densify_iterations
    print(json.dumps({"workload": "DCO frame %dx%d D=%d steady state" % (W, H, a.disparities), "streams": S,
                      "frames": a.steps * S, "frames_per_s": a.steps * S / (ms / 1000.0),
                      "ms_per_step": ms / a.steps, "iterations": it, "l2": "flushed before every frame"}))
    for st in streams:
        st.close()


if __name__ == "__main__":
    main()
