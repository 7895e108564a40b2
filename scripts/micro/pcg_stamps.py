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
NB = torch.cuda.get_device_properties(0).multi_processor_count
LEN = 1280 + 64 * 1024 * 3 + 1024
buf = (ctypes.c_longlong * LEN)()
lib.dco_debug_pcg_stamps(buf, LEN)
g = np.array(buf[1280:1280 + 64 * 1024 * 3]).reshape(64, 1024, 3)[:, :NB, :].astype(np.float64)
a = np.array(buf[:640]).reshape(64, 10)
b = np.array(buf[640:1280]).reshape(64, 10)
# stamps: 0 loop head, 3 after halo, 4 after P1, 5 after CTA barrier, 1 after P2, 2 after grid barrier
order = [0, 3, 4, 5, 1, 2]
names = ["halo fill", "P1 (update)", "CTA barrier", "P2 (SpMV + sums)", "grid barrier-reduce"]
for tag, m in (("block0", a), ("last", b)):
    mm = m[5:40][:, order]
    d = np.diff(mm, axis=1).mean(axis=0)
    tot = (m[6:40, 0] - m[5:39, 0]).mean()
    print(tag, "cycles/iter %.0f" % tot)
    for n, v in zip(names, d):
        print("   %-24s %8.0f" % (n, v))

# per-block globaltimer (ns): work duration, arrival skew, release latency
it = slice(5, 40)
work = (g[it, :, 1] - g[it, :, 0])
arr = g[it, :, 1] - g[it, :, 1].min(axis=1, keepdims=True)
rel = g[it, :, 2] - g[it, :, 1].max(axis=1, keepdims=True)
per_iter = np.diff(g[4:40, :, 0].min(axis=1))
print("ns/iter %.0f" % per_iter.mean())
print("work ns: mean %.0f min %.0f max %.0f" % (work.mean(), work.mean(0).min(), work.mean(0).max()))
print("arrival skew ns (last - first): %.0f" % (arr.max(axis=1).mean()))
print("release after last arrival ns: mean %.0f max %.0f" % (rel.mean(), rel.max(axis=1).mean()))
wm = work.mean(0)
order = np.argsort(-wm)
print("slowest blocks:", [(int(b), int(wm[b])) for b in order[:8]])
print("fastest blocks:", [(int(b), int(wm[b])) for b in order[-4:]])
smid = np.array(buf[1280 + 64 * 1024 * 3:1280 + 64 * 1024 * 3 + NB])
print("SM ids of the slowest blocks:", [int(smid[b]) for b in order[:12]])
print("SM ids of the fastest blocks:", [int(smid[b]) for b in order[-12:]])
print("SM ids by block:", [int(v) for v in smid])
halo_ns = (g[it, :, 0] - g[4:39, :, 2])  # loop head after the previous release: the scalar math
print("per-block work ns (block order):", [int(v) for v in wm])
# block 0 globaltimer (ns): kernel entry (after the anchor check), after the
# setup barrier, loop exit, after the final objective barrier
e = np.array(buf[6:10], dtype=np.float64)
print("setup ns %.0f  loop ns %.0f  teardown ns %.0f" % (e[1] - e[0], e[2] - e[1], e[3] - e[2]))
print("entry -> setup start ns %.0f" % (e[0] - buf[636]))
# the stream's own solve span (CUDA events on its stream, includes launch and k_keep_dense)
s.set_timing(True)
for i in range(4, 8):
    l8, r8 = vid.frame(i)
    s.push_gray8(torch.from_numpy(l8).cuda(), torch.from_numpy(r8).cuda(), want_result=False)
spans, nfr = s.span_times()
lib.dco_debug_pcg_stamps(buf, LEN)
e = np.array(buf[6:10], dtype=np.float64)
print("stream solve span ms %.4f; kernel entry->end ms %.4f" % (spans["solve"] / nfr, (e[3] - buf[636]) / 1e6))
