"""Times solve_dense_depth alone on a real 1280x720 system at several
iteration caps: slope = cost per PCG iteration, intercept = setup/teardown."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402

# usage: pcg_bench.py [W H D_MAX]  (default 1280 720 127)
W, H, DMAX = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (1280, 720, 127)
cfg = Config(d_max=DMAX)
vid = StereoVideo(W, H)
s = dco.Stream(W, H, cfg)
for i in range(4):
    l8, r8 = vid.frame(i)
    res = s.push_gray8(torch.from_numpy(l8).cuda(), torch.from_numpy(r8).cuda())
v = s.views()
sparse = dco.view_tensor(v.sparse, (H, W), torch.float32).clone()
edges = dco.view_tensor(v.edges, (H, W), torch.uint8).clone()
mf = dco.view_tensor(v.m_fuse, (H // 2, W // 2), torch.float32).clone()
mi = dco.view_tensor(v.m_i, (H, W), torch.float32).clone()
dense = dco.view_tensor(v.dense, (H, W), torch.float32).clone()
sysm = dco.assemble_system(sparse, edges, mf, mi, dense, cfg)
for cap in (0, 1, 10, 40, 80):
    c = cfg.copy(solver_max_iter=cap, solver_tol=1e-30)
    for _ in range(2):
        out, st = dco.solve_dense_depth(sysm, c, history_cap=0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 5
    for _ in range(n):
        out, st = dco.solve_dense_depth(sysm, c, history_cap=0)
    b.record()
    torch.cuda.synchronize()
    print("cap %3d iters %3d  %.3f ms/solve" % (cap, st.iterations, a.elapsed_time(b) / n))
out, st = dco.solve_dense_depth(sysm, cfg, history_cap=0)
a.record()
for _ in range(5):
    out, st = dco.solve_dense_depth(sysm, cfg, history_cap=0)
b.record()
torch.cuda.synchronize()
print("default tol: iterations %d  %.3f ms/solve" % (st.iterations, a.elapsed_time(b) / 5))
