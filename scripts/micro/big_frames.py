"""Times steady-state stream frames at the larger BASELINE configs on one GPU
(1920x1080 D=192, 3840x2160 D=256): per-frame ms and the per-stage split."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402

SIZES = ((1920, 1080, 192), (3840, 2160, 256))
if len(sys.argv) > 1:  # e.g. 3840x2160
    SIZES = [z for z in SIZES if "%dx%d" % z[:2] in sys.argv[1:]]
for W, H, D in SIZES:
    cfg = Config(d_max=D - 1)
    vid = StereoVideo(W, H)
    frames = [vid.frame(i) for i in range(6)]
    dev = [(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) for a, b in frames]
    s = dco.Stream(W, H, cfg)
    t0 = time.time()
    for i in range(4):
        r = s.push_gray8(*dev[i])
    torch.cuda.synchronize()
    s.set_timing(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 2
    for i in range(n):
        r = s.push_gray8(*dev[4 + i], want_result=(i == n - 1))
    b.record()
    torch.cuda.synchronize()
    spans, nt = s.span_times()
    ms = a.elapsed_time(b) / n
    print("%dx%d D=%d: %.2f ms/frame (%.1f frames/s), iterations %d" % (W, H, D, ms, 1000 / ms, r.densify_iterations))
    print("   ", {k: round(v / max(nt, 1), 3) for k, v in spans.items()})
    s.close()
    del s, dev
    torch.cuda.empty_cache()
