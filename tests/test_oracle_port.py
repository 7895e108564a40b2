"""Pins the C restatement (oracle/dco_oracle.c) against the compiled reference
(oracle/_ref) bit for bit, stage by stage, on the reference's own synthetic
scenes and KATs. CPU only."""
import numpy as np
import pytest

from paper_2203_02300_b200.config import Config, ConfigError, InputError, UnsolvableFrameError
from tests.inputs import Rng, random_image, scene


@pytest.fixture(scope="module")
def port():
    from oracle import port as p

    p.lib()
    return p


def same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    if a.dtype == np.float32:
        return np.array_equal(a.view(np.uint32), b.view(np.uint32))
    if a.dtype == np.float64:
        return np.array_equal(a.view(np.uint64), b.view(np.uint64))
    return np.array_equal(a, b)


@pytest.fixture(scope="module", params=[(160, 96, 31, 2718, True), (320, 192, 47, 1234, True), (256, 128, 40, 7, False)],
                ids=lambda p: "%dx%d" % p[:2])
def frames(request, ref):
    w, h, dmax, seed, q = request.param
    fs = [scene(ref, w, h, index=i, seed=seed, quantize=q) for i in range(3)]
    return dict(fs=fs, cfg=Config(d_max=dmax), w=w, h=h)


def test_stereo_chain_port_equals_reference(ref, port, frames):
    cfg, f = frames["cfg"], frames["fs"][1]
    lq, rq = ref.downsample_half(f["left"]), ref.downsample_half(f["right"])
    assert same(port.downsample_half(f["left"]), lq)
    arms = ref.build_cross_windows(lq, cfg)
    assert same(port.build_cross_windows(lq, cfg), arms)
    for ww, wh in ((9, 7), (5, 3)):
        assert same(port.census_transform(lq, ww, wh), ref.census_transform(lq, ww, wh))
    vol = ref.compute_cost_volume(lq, rq, arms, cfg)
    assert same(port.compute_cost_volume(lq, rq, arms, cfg), vol)
    agg = ref.aggregate_costs(vol, arms)
    assert same(port.aggregate_costs(vol, arms), agg)
    wta = ref.select_disparity_wta(agg)
    assert same(port.select_disparity_wta(agg), wta)
    for it in (0, 1, 2):
        assert same(port.refine_disparity_histogram(wta, arms, it), ref.refine_disparity_histogram(wta, arms, it))
    d = ref.refine_disparity_histogram(wta, arms, 2)
    assert same(port.disparity_to_sparse_depth(d, cfg, frames["w"], frames["h"]),
                ref.disparity_to_sparse_depth(d, cfg, frames["w"], frames["h"]))


def test_flow_contour_port_equals_reference(ref, port, frames):
    cfg = frames["cfg"]
    q = [ref.downsample_half(f["left"]) for f in frames["fs"]]
    fp = ref.compute_flow(q[1], q[0], cfg)
    ff = ref.compute_flow(q[1], q[2], cfg)
    for want, got in zip(fp + ff, port.compute_flow(q[1], q[0]) + port.compute_flow(q[1], q[2])):
        assert same(got, want)
    rp, tp = ref.flow_to_polar(*fp)
    gr, gt = port.flow_to_polar(*fp)
    assert same(gr, rp) and same(gt, tp)
    mp, mf = ref.gradient_amplitude(rp), ref.gradient_amplitude(ref.flow_to_polar(*ff)[0])
    assert same(port.gradient_amplitude(rp), mp)
    fused = ref.fuse_amplitudes(fp, ff, mp, mf, cfg)
    assert same(port.fuse_amplitudes(fp, ff, mp, mf, cfg), fused)
    boxed = ref.box_filter(fused, cfg.box_radius)
    assert same(port.box_filter(fused, cfg.box_radius), boxed)
    m_fuse = ref.normalize_amplitude(boxed)
    assert same(port.normalize_amplitude(boxed), m_fuse)
    gray = frames["fs"][1]["left"]
    blurred = ref.gaussian_blur(gray, cfg.gauss_sigma)
    assert same(port.gaussian_blur(gray, cfg.gauss_sigma), blurred)
    e, m = ref.extract_depth_contours_prefiltered(blurred, m_fuse, cfg)
    pe, pm = port.extract_depth_contours_prefiltered(blurred, m_fuse, cfg)
    assert same(pe, e) and same(pm, m) and e.sum() > 0


def test_densify_composite_port_equals_reference(ref, port, frames):
    cfg = frames["cfg"]
    fs = frames["fs"]
    q = [ref.downsample_half(f["left"]) for f in fs]
    mid = fs[1]
    rgb = np.repeat(mid["left"][:, :, None], 3, 2)
    vrgb, vdepth = ref.render_cube(frames["w"], frames["h"], cfg.focal_px)
    out = ref.pipeline_frame(q[0], q[1], q[2], mid["left"], ref.downsample_half(mid["right"]), rgb, None, vrgb,
                             vdepth, cfg)
    fp, ff = ref.compute_flow(q[1], q[0], cfg), ref.compute_flow(q[1], q[2], cfg)
    m_fuse = ref.normalize_amplitude(ref.box_filter(ref.fuse_amplitudes(
        fp, ff, ref.gradient_amplitude(ref.flow_to_polar(*fp)[0]), ref.gradient_amplitude(ref.flow_to_polar(*ff)[0]),
        cfg), cfg.box_radius))
    edges, m_i = ref.extract_depth_contours_prefiltered(ref.gaussian_blur(mid["left"], cfg.gauss_sigma), m_fuse, cfg)
    for pre in (None, out["dense"]):
        want = ref.assemble_system(out["sparse"], edges, m_fuse, m_i, pre, cfg)
        got = port.assemble_system(out["sparse"], edges, m_fuse, m_i, pre, cfg)
        for k in ("diag", "coup_h", "coup_v", "rhs", "initial", "anchored"):
            assert same(got[k], want[k]), k
        assert got["constant_term"] == want["constant_term"] and got["anchor_count"] == want["anchor_count"]
        x = np.random.default_rng(0).random(want["diag"].shape)
        assert same(port.apply_system(got, x), ref.apply_system(want, x))
        dr, sr = ref.solve_dense_depth(want, cfg)
        dp, sp = port.solve_dense_depth(got, cfg)
        assert same(dp, dr)
        assert sp["iterations"] == sr["iterations"]
        assert sp["objective_final"] == sr["objective_final"] and sp["objective_initial"] == sr["objective_initial"]
    c_want, m_want = ref.composite(rgb, out["dense"], vrgb, vdepth)
    c_got, m_got = port.composite(rgb, out["dense"], vrgb, vdepth)
    assert same(c_got, c_want) and same(m_got, m_want)
    assert same(c_want, out["composite"]) and same(m_want, out["mask"])


def test_port_edge_cases(ref, port):
    img = random_image(37, 23, 1)
    assert same(port.downsample_half(img), ref.downsample_half(img))
    with pytest.raises(InputError):
        port.downsample_half(random_image(1, 9, 1))
    with pytest.raises(ConfigError):
        port.census_transform(img, 8, 3)
    with pytest.raises(InputError):
        port.box_filter(img, 0)
    with pytest.raises(InputError):
        port.compute_flow(random_image(7, 30, 1), random_image(7, 30, 2))
    cfg = Config(cross_arm_l1=4, cross_arm_l2=2)
    rng = Rng(77)
    for _ in range(10):
        im = np.array([rng.uniform() for _ in range(64)], np.float32).reshape(8, 8)
        d = np.array([np.nan if rng.uniform() < 0.1 else float(rng.uniform_int(0, 6)) for _ in range(64)],
                     np.float32).reshape(8, 8)
        arms = ref.build_cross_windows(im, cfg)
        assert same(port.refine_disparity_histogram(d, arms, 1), ref.refine_disparity_histogram(d, arms, 1))
    h, w = 8, 8
    sys = port.assemble_system(np.full((h, w), np.nan, np.float32), np.zeros((h, w), np.uint8),
                               np.zeros((4, 4), np.float32), np.zeros((h, w), np.float32), None, Config())
    with pytest.raises(UnsolvableFrameError):
        port.solve_dense_depth(sys, Config())


def test_port_stereo_kat(port, ref):
    """criterion_stereo_oracle through the restatement: ratio=0.993448 valid=74781."""
    cfg = Config()
    f = ref.render_synth_frame(960, 320, 0, square_size=160, square_x0=400.0, square_y0=80.0, shift_x=0.0, seed=7)
    lq, rq = port.downsample_half(f["left"]), port.downsample_half(f["right"])
    arms = port.build_cross_windows(lq, cfg)
    d = port.refine_disparity_histogram(
        port.select_disparity_wta(port.aggregate_costs(port.compute_cost_volume(lq, rq, arms, cfg), arms)), arms, 2)
    sp = port.disparity_to_sparse_depth(d, cfg, 960, 320)
    valid = np.isfinite(sp)
    dq = cfg.focal_px * cfg.baseline_m / sp[valid].astype(np.float64) / 2.0
    truth = np.where(f["gt_depth"][valid] == 1.0, 24.0, 12.0)
    assert valid.sum() == 74781
    assert "%.6f" % ((np.abs(dq - truth) <= 1.0).sum() / valid.sum()) == "0.993448"


def test_lr_consistency_restatement():
    """oracle/ref.lr_consistency on a hand-made pair: a fronto-parallel plane at
    d=2 agrees everywhere x - 2 is inside the map; a disagreeing right view, a
    NaN and an out-of-map match drop out; max_diff is inclusive."""
    from oracle import ref

    dl = np.full((2, 6), 2.0, np.float32)
    dr = np.full((2, 6), 2.0, np.float32)
    dl[0, 5] = np.nan
    dr[1, 2] = 3.0   # right view of (1, 4) disagrees by 1
    out = ref.lr_consistency(dl, dr, 0.5)
    want = np.full((2, 6), np.nan, np.float32)
    want[0, 2:5] = 2.0
    want[1, 2:4] = 2.0
    want[1, 5] = 2.0
    assert np.array_equal(np.isnan(out), np.isnan(want)) and np.array_equal(out[~np.isnan(out)], want[~np.isnan(want)])
    assert np.isfinite(ref.lr_consistency(dl, dr, 1.0)[1, 4])  # |2 - 3| <= 1 keeps it
