"""Solves the bench frame's system with an iteration cap and saves the dense
map (for comparing solver variants across processes). The system comes from
system_1280x720.npz, written by scripts/micro/dump_system.py (not tracked)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402

W, H = 1280, 720
cap, tag = int(sys.argv[1]), sys.argv[2]
cfg = Config(d_max=127)
d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "system_1280x720.npz"))
sparse, edges, mf, mi, dense = (torch.from_numpy(d[k]).cuda() for k in ("sparse", "edges", "m_fuse", "m_i", "dense"))
sysm = dco.assemble_system(sparse, edges, mf, mi, dense, cfg)
out, st = dco.solve_dense_depth(sysm, cfg.copy(solver_max_iter=cap, solver_tol=1e-30), history_cap=cap + 1)
np.save("gpurun_out/dense_%s_%d.npy" % (tag, cap), out.cpu().numpy())
print(tag, cap, st.iterations, [float(x) for x in st.residual_history[:8]])
