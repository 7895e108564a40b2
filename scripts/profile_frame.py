"""Runs a handful of composited 1280x720 D=128 frames (the bench workload) for
ncu captures: python scripts/profile_frame.py [frames]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402

W, H = 1280, 720
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
vid = StereoVideo(W, H)
s = dco.Stream(W, H, Config(d_max=127))
for i in range(n):
    l8, r8 = vid.frame(i)
    res = s.push_gray8(torch.from_numpy(l8).cuda(), torch.from_numpy(r8).cuda())
torch.cuda.synchronize()
print("frames", n, "iterations", res.densify_iterations)
