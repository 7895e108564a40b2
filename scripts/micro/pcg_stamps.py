"""Per-phase cycle breakdown of one PCG solve (block 0 and the last block)."""
import ctypes
import os
import sys

os.environ["DCO_PCG_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_02300_b200 import dco, native  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402

W, H = 1280, 720
cfg = Config(d_max=127)
vid = StereoVideo(W, H)
s = dco.Stream(W, H, cfg)
for i in range(4):
    l8, r8 = vid.frame(i)
    s.push_gray8(torch.from_numpy(l8).cuda(), torch.from_numpy(r8).cuda(), want_result=False)
torch.cuda.synchronize()
lib = native.load()
buf = (ctypes.c_longlong * 1280)()
lib.dco_debug_pcg_stamps(buf, 1280)
a = np.array(buf[:640]).reshape(64, 10)
b = np.array(buf[640:]).reshape(64, 10)
names = ["A work", "A barrier-reduce", "B work", "B barrier-reduce", "C work", "C barrier-reduce"]
for tag, m in (("block0", a), ("last", b)):
    d = np.diff(m[5:40, :7], axis=1).mean(axis=0)
    tot = (m[6:40, 0] - m[5:39, 0]).mean()
    print(tag, "cycles/iter %.0f" % tot)
    for n, v in zip(names, d):
        print("   %-16s %8.0f" % (n, v))
    e = m[5:40]
    print("   B: work-end->arrive %.0f  atomic %.0f  arrive->released %.0f  released->B-end %.0f" % (
        (e[:, 7] - e[:, 3]).mean(), (e[:, 8] - e[:, 7]).mean(), (e[:, 9] - e[:, 8]).mean(), (e[:, 4] - e[:, 9]).mean()))
