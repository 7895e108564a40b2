"""Densify (assembly bit-exact, PCG+MR within tolerance), composite (exact)
and the device-resident frame stream vs the reference (densify.cpp,
occlude.cpp:171-194, pipeline.cpp:136-258).

Tolerances: dense depth max-abs <= 1e-5 m and RMS <= 1e-6 m
versus the oracle's sequential-order solve; iteration counts within +-2 of
the oracle's; objective values within 1e-9 relative."""
import numpy as np
import pytest
import torch

from paper_2203_02300_b200.config import Config, InputError, UnsolvableFrameError
from tests.inputs import Rng, scene
from tests.test_gpu_stereo import N, T, bits_equal

pytestmark = pytest.mark.gpu

MAX_ABS = 1e-5
RMS = 1e-6


def random_inputs(w, h, seed, with_pre):
    rng = Rng(seed)
    sparse = np.full((h, w), np.nan, np.float32)
    edges = np.zeros((h, w), np.uint8)
    m_i = np.zeros((h, w), np.float32)
    pre = np.full((h, w), np.nan, np.float32)
    for y in range(h):
        for x in range(w):
            if rng.uniform() < 0.25:
                sparse[y, x] = rng.uniform(0.5, 4.0)
            edges[y, x] = 1 if rng.uniform() < 0.08 else 0
            m_i[y, x] = rng.uniform()
            if rng.uniform() < 0.5:
                pre[y, x] = rng.uniform(0.5, 4.0)
    m_fuse = np.array([rng.uniform() for _ in range((w // 2) * (h // 2))], np.float32).reshape(h // 2, w // 2)
    return sparse, edges, m_fuse, m_i, (pre if with_pre else None)


def gpu_sys_arrays(sys):
    return {k: N(getattr(sys, k)) for k in ("diag", "coup_h", "coup_v", "rhs", "initial", "anchored")}


@pytest.mark.parametrize("seed,with_pre", [(5150, False), (5151, True), (9, True)])
def test_assemble_bit_exact_random(gpu, ref, seed, with_pre):
    cfg = Config()
    sparse, edges, m_fuse, m_i, pre = random_inputs(16, 16, seed, with_pre)
    want = ref.assemble_system(sparse, edges, m_fuse, m_i, pre, cfg)
    sys = gpu.assemble_system(T(sparse), T(edges), T(m_fuse), T(m_i), None if pre is None else T(pre), cfg)
    got = gpu_sys_arrays(sys)
    for k in ("diag", "coup_h", "coup_v", "rhs", "initial", "anchored"):
        assert bits_equal(got[k], want[k]), k
    assert sys.anchor_count == want["anchor_count"]
    assert abs(sys.constant_term - want["constant_term"]) <= 1e-12 * max(1.0, abs(want["constant_term"]))


def test_smoothness_weight(gpu, ref):
    sparse, edges, m_fuse, m_i, _ = random_inputs(12, 10, 3, False)
    for (px, py, qx, qy) in [(0, 0, 1, 0), (3, 4, 3, 5), (11, 9, 10, 9), (5, 5, 5, 4)]:
        assert gpu.smoothness_weight(px, py, qx, qy, T(edges), T(m_fuse), T(m_i)) == \
            ref.smoothness_weight(px, py, qx, qy, edges, m_fuse, m_i)
    with pytest.raises(InputError):
        gpu.smoothness_weight(0, 0, 1, 1, T(edges), T(m_fuse), T(m_i))


def _solve_both(gpu, ref, sparse, edges, m_fuse, m_i, pre, cfg):
    want_sys = ref.assemble_system(sparse, edges, m_fuse, m_i, pre, cfg)
    want, st = ref.solve_dense_depth(want_sys, cfg)
    sys = gpu.assemble_system(T(sparse), T(edges), T(m_fuse), T(m_i), None if pre is None else T(pre), cfg)
    got, gst = gpu.solve_dense_depth(sys, cfg)
    return N(got), gst, want, st


VARIANT_ENV = {"tmem": None, "onchip": "DCO_PCG_NO_TMEM", "big": "DCO_PCG_FORCE_BIG",
               "big768": "DCO_PCG_FORCE_BIG,DCO_PCG_BIG768", "share": "DCO_PCG_SHARE", "stream": "DCO_PCG_FORCE_STREAM"}


@pytest.mark.parametrize("variant", sorted(VARIANT_ENV))
@pytest.mark.parametrize("seed,with_pre", [(5150, False), (5151, True), (77, False)])
def test_solve_small_within_tolerance(gpu, ref, seed, with_pre, variant, monkeypatch):
    """Every solver variant: tmem (default), onchip (registers + shared memory,
    DCO_PCG_NO_TMEM), big (x/xs/coefficients in L2, forced on a small system;
    1024 threads, and big768 the 768-thread instances),
    share (the co-residency kernel) and stream (every vector in global memory,
    the any-size path)."""
    for env in filter(None, (VARIANT_ENV[variant] or "").split(",")):
        monkeypatch.setenv(env, "1")
    cfg = Config(solver_tol=1e-12, solver_max_iter=3000)
    got, gst, want, st = _solve_both(gpu, ref, *random_inputs(16, 16, seed, with_pre), cfg)
    d = np.abs(got.astype(np.float64) - want)
    assert d.max() <= MAX_ABS and np.sqrt((d ** 2).mean()) <= RMS
    assert abs(gst.iterations - st["iterations"]) <= 2
    assert gst.objective_final <= gst.objective_initial + 1e-9


@pytest.mark.parametrize("variant", sorted(VARIANT_ENV))
def test_solve_scene_within_tolerance(gpu, ref, variant, monkeypatch):
    """A real frame's system (640x360 full res) with and without d_pre, on each
    solver variant."""
    for env in filter(None, (VARIANT_ENV[variant] or "").split(",")):
        monkeypatch.setenv(env, "1")
    cfg = Config(d_max=63)
    fs = [scene(ref, 640, 360, index=i, seed=61) for i in range(4)]
    q = [ref.downsample_half(f["left"]) for f in fs]
    out = ref.pipeline_frame(q[0], q[1], q[2], fs[1]["left"], ref.downsample_half(fs[1]["right"]),
                             np.repeat(fs[1]["left"][:, :, None], 3, 2), None, None, None, cfg)
    # rebuild the pipeline's system inputs with the oracle
    fp, ff = ref.compute_flow(q[1], q[0], cfg), ref.compute_flow(q[1], q[2], cfg)
    mp = ref.gradient_amplitude(ref.flow_to_polar(*fp)[0])
    mf = ref.gradient_amplitude(ref.flow_to_polar(*ff)[0])
    m_fuse = ref.normalize_amplitude(ref.box_filter(ref.fuse_amplitudes(fp, ff, mp, mf, cfg), cfg.box_radius))
    edges, m_i = ref.extract_depth_contours_prefiltered(ref.gaussian_blur(fs[1]["left"], cfg.gauss_sigma), m_fuse, cfg)
    assert bits_equal(edges, out["edges"])
    for pre in (None, out["dense"]):
        got, gst, want, st = _solve_both(gpu, ref, out["sparse"], edges, m_fuse, m_i, pre, cfg)
        d = np.abs(got.astype(np.float64) - want)
        assert d.max() <= MAX_ABS, d.max()
        assert np.sqrt((d ** 2).mean()) <= RMS
        assert abs(gst.iterations - st["iterations"]) <= 2, (gst.iterations, st["iterations"])
        assert abs(gst.objective_final - st["objective_final"]) <= 1e-9 * abs(st["objective_final"]) + 1e-9


def test_unsolvable(gpu, ref):
    cfg = Config()
    h, w = 8, 8
    sparse = np.full((h, w), np.nan, np.float32)
    edges = np.zeros((h, w), np.uint8)
    m_i = np.zeros((h, w), np.float32)
    m_fuse = np.zeros((4, 4), np.float32)
    sys = gpu.assemble_system(T(sparse), T(edges), T(m_fuse), T(m_i), None, cfg)
    assert sys.anchor_count == 0
    with pytest.raises(UnsolvableFrameError):
        gpu.solve_dense_depth(sys, cfg)


def test_apply_and_objective(gpu, ref):
    cfg = Config()
    sparse, edges, m_fuse, m_i, pre = random_inputs(16, 12, 4, True)
    want = ref.assemble_system(sparse, edges, m_fuse, m_i, pre, cfg)
    sys = gpu.assemble_system(T(sparse), T(edges), T(m_fuse), T(m_i), T(pre), cfg)
    x = np.random.default_rng(1).random((12, 16))
    assert bits_equal(N(gpu.apply_system(sys, T(x))), ref.apply_system(want, x))
    obj = gpu.objective_value(sys, T(x))
    assert np.isfinite(obj)


def test_composite_exact(gpu, ref):
    # criterion_composite_exhaustive (acceptance.cpp:637-669)
    rng = np.random.default_rng(64646)
    h, w = 64, 64
    real = rng.random((h, w, 3), dtype=np.float32)
    dense = np.where(rng.random((h, w)) < 0.9, rng.uniform(0.2, 3.0, (h, w)), np.nan).astype(np.float32)
    vrgb = rng.random((h, w, 3), dtype=np.float32)
    vdepth = np.where(rng.random((h, w)) < 0.7, rng.uniform(0.2, 3.0, (h, w)), np.nan).astype(np.float32)
    vdepth[0, :8] = dense[0, :8]  # ties go to the virtual layer
    want_c, want_m = ref.composite(real, dense, vrgb, vdepth)
    got_c, got_m = gpu.composite(T(real), T(dense), T(vrgb), T(vdepth))
    assert bits_equal(N(got_c), want_c) and bits_equal(N(got_m), want_m)


def test_stream_matches_reference_pipeline(gpu, ref):
    """Five frames through dco_stream (device-resident window, d_pre chain,
    composite against a rendered cube) vs ref_pipeline_frame per window."""
    W, H = 320, 192
    cfg = Config(d_max=47)
    fs = [scene(ref, W, H, index=i, seed=1234) for i in range(5)]
    vrgb, vdepth = ref.render_cube(W, H, cfg.focal_px, cz=1.5, side=0.3)
    s = gpu.Stream(W, H, cfg)
    s.set_virtual(T(vrgb), T(vdepth))
    prev = None
    for i, f in enumerate(fs):
        res = s.push_gray8(T(f["left8"]), T(f["right8"]))
        if i < 2:
            assert res.composited == 0
            continue
        assert res.composited == 1
        q = [ref.downsample_half(fs[j]["left"]) for j in (i - 2, i - 1, i)]
        mid = fs[i - 1]
        want = ref.pipeline_frame(q[0], q[1], q[2], mid["left"], ref.downsample_half(mid["right"]),
                                  np.repeat(mid["left"][:, :, None], 3, 2), prev, vrgb, vdepth, cfg)
        v = s.views()
        dense = N(gpu.view_tensor(v.dense, (H, W), torch.float32))
        edges = N(gpu.view_tensor(v.edges, (H, W), torch.uint8))
        sparse = N(gpu.view_tensor(v.sparse, (H, W), torch.float32))
        mask = N(gpu.view_tensor(v.mask, (H, W), torch.uint8))
        assert bits_equal(sparse, want["sparse"])
        assert bits_equal(edges, want["edges"])
        d = np.abs(dense.astype(np.float64) - want["dense"])
        assert d.max() <= MAX_ABS and np.sqrt((d ** 2).mean()) <= RMS
        assert abs(res.densify_iterations - want["iterations"]) <= 2
        # the mask is a depth test against the dense map: equal wherever the
        # virtual depth is not within the solver tolerance of the real depth
        close = np.abs(vdepth - want["dense"]) <= 2 * MAX_ABS
        assert ((mask == want["mask"]) | close).all()
        prev = want["dense"]
    s.close()


@pytest.mark.parametrize("w,h", [(1, 1), (1, 9), (9, 1), (2, 3)])
def test_densify_edge_shapes(gpu, ref, w, h):
    """assemble (bit-exact) and solve (tolerance) on 1-pixel-wide and tiny
    systems: no right or down couplings, a single anchor."""
    cfg = Config(solver_tol=1e-12, solver_max_iter=500)
    rng = Rng(w * 13 + h)
    sparse = np.full((h, w), np.nan, np.float32)
    sparse[0, 0] = 1.5
    if w * h > 2:
        sparse[h - 1, w - 1] = 2.5
    edges = np.zeros((h, w), np.uint8)
    m_i = np.array([[rng.uniform() for _ in range(w)] for _ in range(h)], np.float32)
    m_fuse = np.array([[rng.uniform() for _ in range(max(w // 2, 1))] for _ in range(max(h // 2, 1))], np.float32)
    want_sys = ref.assemble_system(sparse, edges, m_fuse, m_i, None, cfg)
    sys = gpu.assemble_system(T(sparse), T(edges), T(m_fuse), T(m_i), None, cfg)
    got = gpu_sys_arrays(sys)
    for k in ("diag", "coup_h", "coup_v", "rhs", "initial", "anchored"):
        assert bits_equal(got[k], want_sys[k]), k
    want, st = ref.solve_dense_depth(want_sys, cfg)
    dense, gst = gpu.solve_dense_depth(sys, cfg)
    d = np.abs(N(dense).astype(np.float64) - want)
    assert d.max() <= MAX_ABS
    assert abs(gst.iterations - st["iterations"]) <= 2


def test_run_streams_equals_individual_pushes(gpu, ref):
    """dco_run_streams (the batched entry point) == pushing each stream's frames
    one call at a time: same results, same final maps, bit for bit."""
    from paper_2203_02300_b200.synth import StereoVideo

    W, H, F = 320, 192, 5
    cfg = Config(d_max=31)
    vids = [StereoVideo(W, H, seed=70 + k) for k in range(2)]
    frames = [[v.frame(i) for i in range(F)] for v in vids]
    L = [torch.from_numpy(np.stack([f[0] for f in fr])).cuda() for fr in frames]
    R = [torch.from_numpy(np.stack([f[1] for f in fr])).cuda() for fr in frames]
    batched = [gpu.Stream(W, H, cfg) for _ in range(2)]
    res = gpu.run_streams(batched, L, R, want_results=True)
    single = [gpu.Stream(W, H, cfg) for _ in range(2)]
    for k in range(2):
        for f in range(F):
            r = single[k].push_gray8(L[k][f], R[k][f])
            assert (r.composited, r.densify_iterations) == (res[k][f].composited, res[k][f].densify_iterations)
    for k in range(2):
        a, b = batched[k].views(), single[k].views()
        for name, shape, dt in (("dense", (H, W), torch.float32), ("composite", (H, W, 3), torch.float32),
                                ("edges", (H, W), torch.uint8)):
            assert bits_equal(N(gpu.view_tensor(getattr(a, name), shape, dt)),
                              N(gpu.view_tensor(getattr(b, name), shape, dt))), name
    for s in batched + single:
        s.close()


def test_stream_unsolvable_frames(gpu, ref):
    """pipeline.cpp:236-242: a frame with no sparse anchor and no previous
    dense map (UnsolvableFrameError) composites against an all-nodata dense
    map, counts the failure and leaves the d_pre chain empty; the next
    solvable frame then starts without d_pre. (With a previous dense map every
    pixel carries the stability term, densify.cpp:85-91, so a frame is
    unsolvable only before the first solve.) Flat gray frames give a WTA
    disparity of 0 everywhere, hence no sparse depth."""
    W, H = 320, 192
    cfg = Config(d_max=47)
    flat8 = np.full((H, W), 128, np.uint8)
    flat = {"left8": flat8, "right8": flat8}
    flat["left"] = flat["right"] = ref.quantize8(flat8.astype(np.float32) / np.float32(255.0))[1]
    fs = [flat, flat, flat] + [scene(ref, W, H, index=i, seed=4242) for i in range(3, 6)]
    vrgb, vdepth = ref.render_cube(W, H, cfg.focal_px, cz=1.5, side=0.3)
    s = gpu.Stream(W, H, cfg)
    s.set_virtual(T(vrgb), T(vdepth))
    prev = None
    skipped = []
    for i, f in enumerate(fs):
        res = s.push_gray8(T(f["left8"]), T(f["right8"]))
        if i < 2:
            continue
        q = [ref.downsample_half(fs[j]["left"]) for j in (i - 2, i - 1, i)]
        mid = fs[i - 1]
        want = ref.pipeline_frame(q[0], q[1], q[2], mid["left"], ref.downsample_half(mid["right"]),
                                  np.repeat(mid["left"][:, :, None], 3, 2), prev, vrgb, vdepth, cfg)
        v = s.views()
        dense = N(gpu.view_tensor(v.dense, (H, W), torch.float32))
        assert bool(res.densify_skipped) == want["unsolvable"]
        skipped.append(want["unsolvable"])
        if want["unsolvable"]:
            assert bits_equal(dense, want["dense"])  # the nodata map
        else:
            d = np.abs(dense.astype(np.float64) - want["dense"])
            assert d.max() <= MAX_ABS
            assert abs(res.densify_iterations - want["iterations"]) <= 2
            prev = want["dense"]
        mask = N(gpu.view_tensor(v.mask, (H, W), torch.uint8))
        comp = N(gpu.view_tensor(v.composite, (H, W, 3), torch.float32))
        close = np.abs(vdepth - want["dense"]) <= 2 * MAX_ABS
        assert ((mask == want["mask"]) | close).all()
        assert bits_equal(comp[~close], want["composite"][~close])
    assert skipped == [True, True, False, False]
    s.close()


def test_stream_save_load_state(gpu, ref):
    """dco_stream_save_state / load_state: a fresh stream loaded with another
    stream's state (keyframe window, previous dense map, frame counter)
    produces the same next frame, bit for bit."""
    from paper_2203_02300_b200.synth import StereoVideo

    W, H = 320, 192
    cfg = Config(d_max=31)
    vid = StereoVideo(W, H, seed=555)
    frames = [vid.frame(i) for i in range(6)]
    a = gpu.Stream(W, H, cfg)
    for l8, r8 in frames[:4]:
        a.push_gray8(T(l8), T(r8))
    torch.cuda.synchronize()
    blob = a.state()
    b = gpu.Stream(W, H, cfg)
    b.load_state(blob)
    for l8, r8 in frames[4:]:
        ra = a.push_gray8(T(l8), T(r8))
        rb = b.push_gray8(T(l8), T(r8))
        assert (ra.composited, ra.densify_iterations) == (rb.composited, rb.densify_iterations)
        va, vb = a.views(), b.views()
        for name, shape, dt in (("dense", (H, W), torch.float32), ("composite", (H, W, 3), torch.float32),
                                ("edges", (H, W), torch.uint8), ("sparse", (H, W), torch.float32)):
            assert bits_equal(N(gpu.view_tensor(getattr(va, name), shape, dt)),
                              N(gpu.view_tensor(getattr(vb, name), shape, dt))), name
    with pytest.raises(InputError):
        b.load_state(blob[:-8])  # truncated state
    a.close()
    b.close()
