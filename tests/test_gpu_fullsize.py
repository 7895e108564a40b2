"""BASELINE's full sizes (configs C 1920x1080 D=192 and D 3840x2160 D=256),
where the oracle would take minutes per frame: size-independent properties.

* the stream converges every frame (relative residual <= tol, iterations
  below the cap, objective_final <= objective_initial);
* row bands == whole frame, bit for bit, for the stereo chain (the halo and
  the column-prefix carry are exact at any size);
* the band solve over G ranks agrees with the whole-frame solve within the
  solver tolerance, with identical scalars on every rank.
"""
import numpy as np
import pytest
import torch

from paper_2203_02300_b200.config import Config
from paper_2203_02300_b200.synth import StereoVideo
from tests.test_gpu_densify import MAX_ABS
from tests.test_gpu_stereo import N, bits_equal

pytestmark = pytest.mark.gpu

SIZES = [(1920, 1080, 192, 4), (3840, 2160, 256, 8)]


@pytest.fixture(scope="module", params=SIZES, ids=lambda s: "%dx%d" % s[:2])
def video(request, gpu):
    W, H, D, G = request.param
    vid = StereoVideo(W, H)
    frames = [tuple(torch.from_numpy(x).cuda() for x in vid.frame(i)) for i in range(5)]
    return W, H, D, G, frames


def test_stream_converges_at_full_size(gpu, video):
    W, H, D, _, frames = video
    cfg = Config(d_max=D - 1)
    s = gpu.Stream(W, H, cfg)
    for i, (l8, r8) in enumerate(frames):
        res = s.push_gray8(l8, r8)
        if i < 2:
            continue
        assert res.composited and not res.densify_skipped
        assert 0 < res.densify_iterations < cfg.solver_max_iter
        assert res.relative_residual <= cfg.solver_tol
    dense = N(gpu.view_tensor(s.views().dense, (H, W), torch.float32))
    assert np.isfinite(dense).all() and (dense >= 0).all()
    s.close()


def test_bands_equal_whole_frame_at_full_size(gpu, video):
    W, H, D, G, frames = video
    cfg = Config(d_max=D - 1)
    _, lq = gpu.ingest_gray8(frames[1][0])
    _, rq = gpu.ingest_gray8(frames[1][1])
    whole_d, whole_s = gpu.stereo_sparse_depth(lq, rq, cfg, W, H)
    whole_d, whole_s = N(whole_d), N(whole_s)
    carry, disp, sparse = None, [], []
    for k in range(G):
        b = gpu.band_plan(cfg, W, H, G, k)
        d, sp, carry_out = gpu.stereo_band(lq[b.sub0:b.sub1].contiguous(), rq[b.sub0:b.sub1].contiguous(), b, cfg,
                                           W, H, carry if b.carry_row > 0 else None)
        disp.append(N(d))
        sparse.append(N(sp))
        if carry_out is not None:
            carry = carry_out
    assert bits_equal(np.concatenate(disp), whole_d)
    assert bits_equal(np.concatenate(sparse), whole_s)
    assert np.isfinite(whole_d).mean() > 0.5


def test_band_solve_matches_whole_solve_at_full_size(gpu, video):
    W, H, D, G, frames = video
    cfg = Config(d_max=D - 1)
    s = gpu.Stream(W, H, cfg)
    for l8, r8 in frames[:4]:
        s.push_gray8(l8, r8)
    v = s.views()
    sparse = gpu.view_tensor(v.sparse, (H, W), torch.float32).clone()
    edges = gpu.view_tensor(v.edges, (H, W), torch.uint8).clone()
    mf = gpu.view_tensor(v.m_fuse, (H // 2, W // 2), torch.float32).clone()
    mi = gpu.view_tensor(v.m_i, (H, W), torch.float32).clone()
    pre = gpu.view_tensor(v.dense, (H, W), torch.float32).clone()
    s.close()
    sysm = gpu.assemble_system(sparse, edges, mf, mi, pre, cfg)
    whole, st = gpu.solve_dense_depth(sysm, cfg, history_cap=0)
    rows = [(k * H // G, (k + 1) * H // G - k * H // G) for k in range(G)]
    solvers = [gpu.BandSolver(G, k, W, r0, n, H) for k, (r0, n) in enumerate(rows)]
    gpu.band_connect_local(solvers)
    dense, stats = gpu.band_solve_local(solvers, [gpu.band_system(sysm, r0, n) for r0, n in rows], cfg,
                                        sysm.anchor_count, sysm.constant_term, history_cap=0)
    for b in solvers:
        b.close()
    got = np.concatenate([N(d) for d in dense])
    diff = np.abs(got.astype(np.float64) - N(whole).astype(np.float64))
    assert diff.max() <= 2 * MAX_ABS, diff.max()
    assert abs(stats[0].iterations - st.iterations) <= 2
    assert all(x.iterations == stats[0].iterations for x in stats)
    assert stats[0].relative_residual <= cfg.solver_tol
