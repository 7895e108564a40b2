"""Row-band densify (pcg_band.cuh): one system split into row bands, each band
a rank with its own block group, the per-iteration all-reduce and the p halo
crossing ranks through the exchange tables -- against the oracle's sequential
solve (densify.cpp:141-222) within the solver tolerance of
test_gpu_densify.py. All ranks run on this GPU as ONE cooperative launch (the
multi-GPU code path with local pointers)."""
import numpy as np
import pytest

from paper_2203_02300_b200.config import Config, UnsolvableFrameError
from tests.inputs import scene
from tests.test_gpu_densify import MAX_ABS, RMS, random_inputs
from tests.test_gpu_stereo import N, T, bits_equal

pytestmark = pytest.mark.gpu


def split_rows(h, g, uneven=False):
    cuts = [k * h // g for k in range(g + 1)]
    if uneven and g > 1:
        cuts[1] = max(1, cuts[1] // 3)
    return [(cuts[k], cuts[k + 1] - cuts[k]) for k in range(g)]


def band_solve(gpu, sys, cfg, g, uneven=False, repeat=1):
    rows = split_rows(sys.height, g, uneven)
    solvers = [gpu.BandSolver(g, k, sys.width, r0, n, sys.height) for k, (r0, n) in enumerate(rows)]
    gpu.band_connect_local(solvers)
    views = [gpu.band_system(sys, r0, n) for r0, n in rows]
    outs = []
    for _ in range(repeat):
        dense, stats = gpu.band_solve_local(solvers, views, cfg, sys.anchor_count, sys.constant_term)
        outs.append((np.concatenate([N(d) for d in dense]), stats))
    for s in solvers:
        s.close()
    return outs


def oracle_solve(gpu, ref, inputs, cfg):
    sparse, edges, m_fuse, m_i, pre = inputs
    want_sys = ref.assemble_system(sparse, edges, m_fuse, m_i, pre, cfg)
    want, st = ref.solve_dense_depth(want_sys, cfg)
    sys = gpu.assemble_system(T(sparse), T(edges), T(m_fuse), T(m_i), None if pre is None else T(pre), cfg)
    return sys, want, st


def check(got, stats, want, st):
    d = np.abs(got.astype(np.float64) - want)
    assert d.max() <= MAX_ABS, d.max()
    assert np.sqrt((d ** 2).mean()) <= RMS
    assert abs(stats[0].iterations - st["iterations"]) <= 2, (stats[0].iterations, st["iterations"])
    for s in stats[1:]:  # every rank took the same branches on the same scalars
        assert s.iterations == stats[0].iterations
        assert s.relative_residual == stats[0].relative_residual
        assert s.objective_final == stats[0].objective_final
    assert abs(stats[0].objective_final - st["objective_final"]) <= 1e-9 * abs(st["objective_final"]) + 1e-9


@pytest.mark.parametrize("g,uneven", [(1, False), (2, False), (3, True), (4, False), (8, True)])
@pytest.mark.parametrize("seed,with_pre", [(5150, False), (5151, True)])
def test_band_solve_small(gpu, ref, g, uneven, seed, with_pre):
    cfg = Config(solver_tol=1e-12, solver_max_iter=3000)
    sys, want, st = oracle_solve(gpu, ref, random_inputs(16, 16, seed, with_pre), cfg)
    (got, stats), = band_solve(gpu, sys, cfg, g, uneven)
    check(got, stats, want, st)


@pytest.mark.parametrize("g", [2, 5, 8])
def test_band_solve_scene(gpu, ref, g):
    """A pipeline frame's system (640x360) with d_pre, split in g bands."""
    cfg = Config(d_max=63)
    fs = [scene(ref, 640, 360, index=i, seed=61) for i in range(4)]
    q = [ref.downsample_half(f["left"]) for f in fs]
    out = ref.pipeline_frame(q[0], q[1], q[2], fs[1]["left"], ref.downsample_half(fs[1]["right"]),
                             np.repeat(fs[1]["left"][:, :, None], 3, 2), None, None, None, cfg)
    fp, ff = ref.compute_flow(q[1], q[0], cfg), ref.compute_flow(q[1], q[2], cfg)
    mp = ref.gradient_amplitude(ref.flow_to_polar(*fp)[0])
    mf = ref.gradient_amplitude(ref.flow_to_polar(*ff)[0])
    m_fuse = ref.normalize_amplitude(ref.box_filter(ref.fuse_amplitudes(fp, ff, mp, mf, cfg), cfg.box_radius))
    edges, m_i = ref.extract_depth_contours_prefiltered(ref.gaussian_blur(fs[1]["left"], cfg.gauss_sigma), m_fuse, cfg)
    sys, want, st = oracle_solve(gpu, ref, (out["sparse"], edges, m_fuse, m_i, out["dense"]), cfg)
    (got, stats), (again, _) = band_solve(gpu, sys, cfg, g, repeat=2)
    check(got, stats, want, st)
    assert bits_equal(got, again)  # deterministic, and the exchange generations carry across solves


def test_band_solve_unsolvable(gpu, ref):
    cfg = Config()
    sys, _, _ = oracle_solve(gpu, ref, random_inputs(16, 16, 5150, False), cfg)
    rows = split_rows(sys.height, 2)
    solvers = [gpu.BandSolver(2, k, sys.width, r0, n, sys.height) for k, (r0, n) in enumerate(rows)]
    gpu.band_connect_local(solvers)
    with pytest.raises(UnsolvableFrameError):
        gpu.band_solve_local(solvers, [gpu.band_system(sys, r0, n) for r0, n in rows], cfg, 0, 0.0)
    for s in solvers:
        s.close()


def test_single_rank_through_the_ipc_api(gpu, ref):
    """export / connect / solve of the one-process-per-GPU API, at one rank
    (its own handle: no peer mapping needed)."""
    cfg = Config(solver_tol=1e-12, solver_max_iter=3000)
    sys, want, st = oracle_solve(gpu, ref, random_inputs(16, 16, 5151, True), cfg)
    s = gpu.BandSolver(1, 0, sys.width, 0, sys.height, sys.height)
    s.connect([s.export()])
    dense, stats = s.solve(gpu.band_system(sys, 0, sys.height), cfg, sys.anchor_count, sys.constant_term)
    check(N(dense), [stats], want, st)
    s.close()
