"""One capped solve for ncu (DCO_PCG_MODE selects experiment knobs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402

W, H = 1280, 720
cfg = Config(d_max=127)
vid = StereoVideo(W, H)
s = dco.Stream(W, H, cfg)
for i in range(3):
    l8, r8 = vid.frame(i)
    s.push_gray8(torch.from_numpy(l8).cuda(), torch.from_numpy(r8).cuda(), want_result=False)
v = s.views()
sysm = dco.assemble_system(dco.view_tensor(v.sparse, (H, W), torch.float32).clone(),
                           dco.view_tensor(v.edges, (H, W), torch.uint8).clone(),
                           dco.view_tensor(v.m_fuse, (H // 2, W // 2), torch.float32).clone(),
                           dco.view_tensor(v.m_i, (H, W), torch.float32).clone(), None, cfg)
out, st = dco.solve_dense_depth(sysm, cfg.copy(solver_max_iter=40, solver_tol=1e-30), history_cap=0)
print("iterations", st.iterations)
