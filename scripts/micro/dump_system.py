"""Dumps the densify inputs of a steady-state 1280x720 frame (for offline solver studies)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402

W, H = 1280, 720
cfg = Config(d_max=127)
vid = StereoVideo(W, H)
s = dco.Stream(W, H, cfg)
for i in range(4):
    l8, r8 = vid.frame(i)
    s.push_gray8(torch.from_numpy(l8).cuda(), torch.from_numpy(r8).cuda())
v = s.views()
sparse = dco.view_tensor(v.sparse, (H, W), torch.float32).clone()
edges = dco.view_tensor(v.edges, (H, W), torch.uint8).clone()
mf = dco.view_tensor(v.m_fuse, (H // 2, W // 2), torch.float32).clone()
mi = dco.view_tensor(v.m_i, (H, W), torch.float32).clone()
dense = dco.view_tensor(v.dense, (H, W), torch.float32).clone()
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/system_1280x720.npz", sparse=sparse.cpu().numpy(), edges=edges.cpu().numpy(),
                    m_fuse=mf.cpu().numpy(), m_i=mi.cpu().numpy(), dense=dense.cpu().numpy())
print("saved")
