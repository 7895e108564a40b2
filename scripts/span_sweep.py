"""Times the stream's stage spans (one stream alone, CUDA events) of the
1280x720 D=128 frame under a list of environment settings:
  python scripts/span_sweep.py 'DCO_REFINE_SEG=32' 'DCO_REFINE_SEG=64' ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402

W, H = 1280, 720
vid = StereoVideo(W, H)
frames = [tuple(torch.from_numpy(x).cuda() for x in vid.frame(i)) for i in range(12)]
for spec in sys.argv[1:] or [""]:
    saved = dict(os.environ)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    s = dco.Stream(W, H, Config(d_max=127))
    for f in frames[:6]:
        s.push_gray8(*f, want_result=False)
    s.set_timing(True)
    for f in frames[6:]:
        s.push_gray8(*f, want_result=False)
    torch.cuda.synchronize()
    spans, n = s.span_times()
    s.close()
    os.environ.clear()
    os.environ.update(saved)
    print("%-28s " % spec + " ".join("%s=%.4f" % (k, v / n) for k, v in spans.items() if v / n > 0.02))
