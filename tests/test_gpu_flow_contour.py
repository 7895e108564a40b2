"""Flow and depth-contour stages on the GPU vs the reference, bit for bit
(flow.cpp, contour.cpp)."""
import numpy as np
import pytest
import torch

from paper_2203_02300_b200.config import Config, InputError
from tests.inputs import Rng, random_image, scene
from tests.test_gpu_stereo import N, T, bits_equal, mismatch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[(320, 192, 1234), (640, 360, 61)], ids=lambda p: "%dx%d" % p[:2])
def frames(request, ref):
    w, h, seed = request.param
    fs = [scene(ref, w, h, index=i, seed=seed) for i in range(3)]
    q = [ref.downsample_half(f["left"]) for f in fs]
    return dict(fs=fs, q=q, w=w, h=h)


def test_flow_bit_exact(gpu, ref, frames):
    cfg = Config()
    past, mid, fut = frames["q"]
    for to in (past, fut):
        u, v = gpu.compute_flow(T(mid), T(to), cfg)
        ur, vr = ref.compute_flow(mid, to, cfg)
        assert mismatch(N(u), ur) == 0
        assert mismatch(N(v), vr) == 0


def test_flow_translation_kat(gpu, ref):
    # criterion_flow (acceptance.cpp:265-322) on a smooth texture: GPU == oracle
    rng = Rng(11)
    h, w = 96, 128
    p1, p2, p3 = rng.uniform(0, 6.28), rng.uniform(0, 6.28), rng.uniform(0, 6.28)
    tau = 6.283185307179586
    yy, xx = np.mgrid[0:h, 0:w]
    u, v = xx / w, yy / h
    val = (0.5 + 0.17 * np.sin(tau * 3 * u + p1) * np.cos(tau * 2 * v + p2) + 0.15 * np.sin(tau * 5 * v + p3)
           + 0.11 * np.sin(tau * (4 * u + 3 * v) + p1) + 0.07 * np.sin(tau * 8 * u + p2) * np.sin(tau * 6 * v + p3))
    base = np.clip(val, 0, 1).astype(np.float32)
    cfg = Config()
    for sx, sy in [(4, 0), (-4, 0), (0, 3), (-3, 2)]:
        moved = np.roll(np.roll(base, -sy, axis=0), -sx, axis=1)
        gu, gv = gpu.compute_flow(T(moved), T(base), cfg)
        ru, rv = ref.compute_flow(moved, base, cfg)
        assert bits_equal(N(gu), ru) and bits_equal(N(gv), rv)
        assert abs(np.median(N(gu)) - sx) <= 0.5 and abs(np.median(N(gv)) - sy) <= 0.5


def test_flow_rejects_small_frames(gpu):
    with pytest.raises(InputError):
        gpu.compute_flow(T(random_image(7, 20, 1)), T(random_image(7, 20, 2)), Config())


def test_polar_amplitude_fusion_box_normalize(gpu, ref, frames):
    cfg = Config()
    past, mid, fut = frames["q"]
    fp = ref.compute_flow(mid, past, cfg)
    ff = ref.compute_flow(mid, fut, cfg)
    rp, tp = ref.flow_to_polar(*fp)
    r_g, t_g = gpu.flow_to_polar(T(fp[0]), T(fp[1]))
    assert bits_equal(N(r_g), rp) and bits_equal(N(t_g), tp)
    mp = ref.gradient_amplitude(rp)
    assert bits_equal(N(gpu.gradient_amplitude(T(rp))), mp)
    mf = ref.gradient_amplitude(ref.flow_to_polar(*ff)[0])
    fused = ref.fuse_amplitudes(fp, ff, mp, mf, cfg)
    got = gpu.fuse_amplitudes((T(fp[0]), T(fp[1])), (T(ff[0]), T(ff[1])), T(mp), T(mf), cfg)
    assert bits_equal(N(got), fused)
    boxed = ref.box_filter(fused, cfg.box_radius)
    assert bits_equal(N(gpu.box_filter(T(fused), cfg.box_radius)), boxed)
    assert bits_equal(N(gpu.normalize_amplitude(T(boxed))), ref.normalize_amplitude(boxed))


def test_fusion_random_oracle(gpu, ref):
    # criterion_fusion_oracle (acceptance.cpp:328-381): random flows with zeros
    rng = Rng(31415)
    cfg = Config()
    for trial in range(20):
        w, h = rng.uniform_int(5, 16), rng.uniform_int(5, 14)
        a = np.array([rng.uniform(-3, 3) for _ in range(4 * w * h)], np.float32).reshape(4, h, w)
        a[0:2, :, ::3] = 0.0
        mp, mf = random_image(w, h, trial), random_image(w, h, trial + 100)
        want = ref.fuse_amplitudes((a[0], a[1]), (a[2], a[3]), mp, mf, cfg)
        got = gpu.fuse_amplitudes((T(a[0]), T(a[1])), (T(a[2]), T(a[3])), T(mp), T(mf), cfg)
        assert bits_equal(N(got), want)


def test_box_filter_radii_and_nan(gpu, ref):
    a = random_image(53, 29, 9)
    for r in (1, 3, 5, 40):
        assert bits_equal(N(gpu.box_filter(T(a), r)), ref.box_filter(a, r))
    with pytest.raises(InputError):
        gpu.box_filter(T(a), 0)
    b = a.copy()
    b[3, 4] = np.nan
    assert bits_equal(N(gpu.normalize_amplitude(T(b))), ref.normalize_amplitude(b))
    z = np.zeros((9, 9), np.float32)
    assert bits_equal(N(gpu.normalize_amplitude(T(z))), ref.normalize_amplitude(z))


def test_gaussian_and_contours_bit_exact(gpu, ref, frames):
    cfg = Config()
    past, mid, fut = frames["q"]
    fp, ff = ref.compute_flow(mid, past, cfg), ref.compute_flow(mid, fut, cfg)
    mp = ref.gradient_amplitude(ref.flow_to_polar(*fp)[0])
    mf = ref.gradient_amplitude(ref.flow_to_polar(*ff)[0])
    m_fuse = ref.normalize_amplitude(ref.box_filter(ref.fuse_amplitudes(fp, ff, mp, mf, cfg), cfg.box_radius))
    gray = frames["fs"][1]["left"]
    blurred = ref.gaussian_blur(gray, cfg.gauss_sigma)
    assert bits_equal(N(gpu.gaussian_blur(T(gray), cfg.gauss_sigma)), blurred)
    edges, m_i = ref.extract_depth_contours_prefiltered(blurred, m_fuse, cfg)
    ge, gm = gpu.extract_depth_contours_prefiltered(T(blurred), T(m_fuse), cfg)
    assert bits_equal(N(gm), m_i)
    assert bits_equal(N(ge), edges)
    assert edges.sum() > 0
    ge2, gm2 = gpu.extract_depth_contours(T(gray), T(m_fuse), cfg)
    assert bits_equal(N(ge2), edges) and bits_equal(N(gm2), m_i)


def test_contours_ungated_and_thresholds(gpu, ref):
    f = scene(ref, 320, 192, seed=1234)
    gray = f["left"]
    blurred = ref.gaussian_blur(gray, 1.4)
    open_gate = np.ones((96, 160), np.float32)
    for cfg in (Config(), Config(t_low=0.01, t_high=0.2), Config(t_depth=0.5)):
        e, m = ref.extract_depth_contours_prefiltered(blurred, open_gate, cfg)
        ge, gm = gpu.extract_depth_contours_prefiltered(T(blurred), T(open_gate), cfg)
        assert bits_equal(N(ge), e) and bits_equal(N(gm), m)


def test_contour_scene_kat(gpu, ref):
    """criterion_contour_scene (acceptance.cpp:386-463) through the GPU stages:
    recall 1.000000, suppression 0.982492, texture_edges 10738."""
    kw = dict(square_size=80, square_x0=96.0, square_y0=56.0, shift_x=4.0, seed=1234)
    fs = [ref.render_synth_frame(320, 192, i, **kw) for i in range(3)]
    cfg = Config()
    q = [gpu.downsample_half(T(f["left"])) for f in fs]
    fp, ff = gpu.compute_flow(q[1], q[0], cfg), gpu.compute_flow(q[1], q[2], cfg)
    mp = gpu.gradient_amplitude(gpu.flow_to_polar(*fp)[0])
    mf = gpu.gradient_amplitude(gpu.flow_to_polar(*ff)[0])
    fused = gpu.normalize_amplitude(gpu.box_filter(gpu.fuse_amplitudes(fp, ff, mp, mf, cfg), cfg.box_radius))
    gated, _ = gpu.extract_depth_contours(T(fs[1]["left"]), fused, cfg)
    ungated, _ = gpu.extract_depth_contours(T(fs[1]["left"]), torch.ones_like(fused), cfg)
    gated, ungated, gt = N(gated), N(ungated), fs[1]["gt_boundary"]
    h, w = gt.shape
    from scipy.ndimage import maximum_filter

    near2 = maximum_filter(gated, size=5, mode="constant")
    recall = near2[gt == 1].astype(bool).mean()
    reach = 2 * (cfg.box_radius + 5)
    near_b = maximum_filter(gt, size=2 * reach + 1, mode="constant").astype(bool)
    tex = ungated.astype(bool) & ~near_b
    suppression = (~gated.astype(bool) & tex).sum() / tex.sum()
    assert "%.6f" % recall == "1.000000"
    assert "%.6f" % suppression == "0.982492"
    assert int(tex.sum()) == 10738


@pytest.mark.parametrize("w,h", [(2, 2), (3, 5), (17, 2), (64, 3), (5, 64)])
def test_contour_stages_edge_shapes(gpu, ref, w, h):
    """Gaussian (5 taps, clamped borders wider than the image), Sobel/NMS on
    1-3 pixel wide maps, the depth gate on a 1-row m_fuse, box filter radii
    beyond the image (contour.cpp:108-285): bit-exact on ragged shapes."""
    cfg = Config(t_high=0.3, t_low=0.1)
    gray = random_image(w, h, 100 + w + 7 * h)
    gray[:, : w // 2] += 0.3  # an edge to find
    m_fuse = random_image(max(w // 2, 1), max(h // 2, 1), 5 + w)
    blurred = ref.gaussian_blur(gray, cfg.gauss_sigma)
    assert bits_equal(N(gpu.gaussian_blur(T(gray), cfg.gauss_sigma)), blurred)
    edges, m_i = ref.extract_depth_contours_prefiltered(blurred, m_fuse, cfg)
    ge, gm = gpu.extract_depth_contours_prefiltered(T(blurred), T(m_fuse), cfg)
    assert bits_equal(N(gm), m_i) and bits_equal(N(ge), edges)
    for r in (1, 5, 40):
        assert bits_equal(N(gpu.box_filter(T(m_fuse), r)), ref.box_filter(m_fuse, r))
    with pytest.raises(InputError):  # contour.cpp:109, as the reference
        gpu.box_filter(T(m_fuse), 0)
    assert bits_equal(N(gpu.normalize_amplitude(T(m_fuse))), ref.normalize_amplitude(m_fuse))


@pytest.mark.parametrize("w,h", [(16, 16), (16, 41), (37, 16), (100, 17), (33, 70)])
def test_flow_ragged_shapes(gpu, ref, w, h):
    """compute_flow (flow.cpp:29-205) on sizes at the level threshold and with
    patch grids whose last patch is pinned to the border: bit-exact."""
    cfg = Config()
    a = random_image(w, h, 3 * w + h)
    b = np.roll(a, (1, 2), axis=(0, 1)).astype(np.float32)
    u, v = ref.compute_flow(a, b, cfg)
    gu, gv = gpu.compute_flow(T(a), T(b), cfg)
    assert bits_equal(N(gu), u) and bits_equal(N(gv), v)


def test_flow_nonfinite_and_pinned(gpu, ref):
    """k_flow_patch_w against the reference: a textured pair with a NaN blob
    in the target (non-finite steps in the merged first chain phase and in
    later iterations: seed restored, zero-weight patches, the nearest-covered
    fill) and a ragged size with pinned last patches."""
    cfg = Config()
    for w, h, blob in ((160, 96, True), (203, 77, False)):
        a = random_image(w, h, 5 * w + h)
        b = np.roll(a, (2, -3), axis=(0, 1)).astype(np.float32)
        if blob:
            b[40:52, 60:75] = np.nan
        u, v = ref.compute_flow(a, b, cfg)
        gu, gv = gpu.compute_flow(T(a), T(b), cfg)
        assert bits_equal(N(gu), u) and bits_equal(N(gv), v), (w, h)


def test_nms_sector_thresholds_exhaustive(gpu):
    """k_nms_gate classifies the gradient direction by comparing the float
    atan2f value with per-branch float thresholds found on the host; for every
    float in [-4, 4] and the NaNs, the sector equals the reference's double
    expression (contour.cpp:217-232: (a < 0 ? a + pi : a) * 180 / pi against
    22.5 / 67.5 / 112.5 / 157.5)."""
    import ctypes

    from paper_2203_02300_b200 import native

    fn = native.load().dco_debug_nms_check
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    bad = ctypes.c_ulonglong(1)
    assert fn(ctypes.byref(bad)) == 0
    assert bad.value == 0
