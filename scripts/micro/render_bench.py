"""Times render_virtual of the bench's cube at 1280x720 (CUDA events) and
lists its kernels for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from bench import cube_mesh, frame_pose  # noqa: E402
from paper_2203_02300_b200 import dco  # noqa: E402

W, H = 1280, 720
v, t, c = cube_mesh(0.3)
vg, tg, cg = torch.from_numpy(v).cuda(), torch.from_numpy(t).cuda(), torch.from_numpy(c).cuda()
for _ in range(3):
    vp = dco.transform_mesh(vg, frame_pose(7))
    dco.render_virtual(vp, tg, cg, 1000.0, W / 2, H / 2, W, H)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record()
for k in range(20):
    vp = dco.transform_mesh(vg, frame_pose(k))
    dco.render_virtual(vp, tg, cg, 1000.0, W / 2, H / 2, W, H)
b.record()
torch.cuda.synchronize()
print("render_virtual 1280x720 cube: %.1f us" % (1000 * a.elapsed_time(b) / 20))
