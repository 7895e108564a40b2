"""Parity at the BASELINE configs' own sizes (BASELINE.json configs A-D).

The smaller parity tests pin every stage at sizes where the oracle is quick;
these pin the instances the bench and the large configs actually dispatch:

* config B (1280x720, D=128): whole composited frames through dco_stream
  against the reference's run_pipeline body (pipeline.cpp:183-258), the first
  composited frame (no d_pre) and a steady one (d_pre chain). The solve is
  k_pcg_tmem<10, 640> (640 threads; x slots 8..9 in registers).
* config A (640x480, D=64): the same, k_pcg_tmem<5, 512>.
* config C (1920x1080, D=192): the stream's own assembled system solved by
  k_pcg_big<14, 1024> against the reference's solve_dense_depth
  (densify.cpp:141-222) on the same inputs.
* config D (3840x2160, D=256): the same for k_pcg_stream<512,2>, steady
  frame (d_pre from the stream's previous frame).
* every k_pcg_tmem slot count (EPT 2..7 at 1024 threads, 9..11 at 640; 1 is
  the small-system tests') against the oracle on one system, reached with
  DCO_PCG_BLOCKS (fewer, fuller blocks).

Bars: sparse, edges, m_fuse, m_i, flow, composite outside the
solver tolerance band: bit-exact; dense max-abs <= 1e-5 m, RMS <= 1e-6 m;
CG iterations within +-2 of the oracle's."""
import numpy as np
import pytest
import torch

from paper_2203_02300_b200.config import Config
from tests.inputs import scene
from tests.test_gpu_stereo import N, T, bits_equal

pytestmark = pytest.mark.gpu

MAX_ABS = 1e-5
RMS = 1e-6


def _dense_ok(got, want):
    d = np.abs(got.astype(np.float64) - want.astype(np.float64))
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin)
    d = d[fin]
    assert d.max() <= MAX_ABS, d.max()
    assert np.sqrt((d ** 2).mean()) <= RMS, np.sqrt((d ** 2).mean())
    return d.max()


def _view(gpu, v, name, shape, dt):
    return N(gpu.view_tensor(getattr(v, name), shape, dt))


def _stream_vs_reference(gpu, ref, W, H, D, solver, frames=4, seed=61):
    cfg = Config(d_max=D - 1)
    fs = [scene(ref, W, H, index=i, seed=seed) for i in range(frames)]
    vrgb, vdepth = ref.render_cube(W, H, cfg.focal_px, cz=1.5, side=0.3)
    s = gpu.Stream(W, H, cfg)
    s.set_virtual(T(vrgb), T(vdepth))
    prev = None
    report = []
    for i, f in enumerate(fs):
        res = s.push_gray8(T(f["left8"]), T(f["right8"]))
        if i < 2:
            assert res.composited == 0
            continue
        assert res.composited == 1 and res.densify_skipped == 0
        assert s.last_solver() == solver
        q = [ref.downsample_half(fs[j]["left"]) for j in (i - 2, i - 1, i)]
        mid = fs[i - 1]
        rq = ref.downsample_half(mid["right"])
        want = ref.pipeline_frame(q[0], q[1], q[2], mid["left"], rq, np.repeat(mid["left"][:, :, None], 3, 2), prev,
                                  vrgb, vdepth, cfg)
        v = s.views()
        qw, qh = W // 2, H // 2
        assert bits_equal(_view(gpu, v, "sparse", (H, W), torch.float32), want["sparse"])
        assert bits_equal(_view(gpu, v, "edges", (H, W), torch.uint8), want["edges"])
        if i == 2:
            # the intermediate maps of the first window, against the oracle chain
            fp, ff = ref.compute_flow(q[1], q[0], cfg), ref.compute_flow(q[1], q[2], cfg)
            for name, arr in (("flow_past_u", fp[0]), ("flow_past_v", fp[1]), ("flow_future_u", ff[0]),
                              ("flow_future_v", ff[1])):
                assert bits_equal(_view(gpu, v, name, (qh, qw), torch.float32), arr), name
            mp = ref.gradient_amplitude(ref.flow_to_polar(*fp)[0])
            mf = ref.gradient_amplitude(ref.flow_to_polar(*ff)[0])
            m_fuse = ref.normalize_amplitude(ref.box_filter(ref.fuse_amplitudes(fp, ff, mp, mf, cfg), cfg.box_radius))
            assert bits_equal(_view(gpu, v, "m_fuse", (qh, qw), torch.float32), m_fuse)
            edges, m_i = ref.extract_depth_contours_prefiltered(ref.gaussian_blur(mid["left"], cfg.gauss_sigma),
                                                                m_fuse, cfg)
            assert bits_equal(_view(gpu, v, "m_i", (H, W), torch.float32), m_i)
            assert bits_equal(edges, want["edges"])
        dense = _view(gpu, v, "dense", (H, W), torch.float32)
        err = _dense_ok(dense, want["dense"])
        assert abs(res.densify_iterations - want["iterations"]) <= 2, (res.densify_iterations, want["iterations"])
        # composite: exact wherever the virtual depth is outside the solver's
        # tolerance band around the real depth
        mask = _view(gpu, v, "mask", (H, W), torch.uint8)
        comp = _view(gpu, v, "composite", (H, W, 3), torch.float32)
        close = np.abs(vdepth.astype(np.float64) - want["dense"]) <= 2 * MAX_ABS
        assert ((mask == want["mask"]) | close).all()
        assert (comp.view(np.uint32) == want["composite"].view(np.uint32))[~close].all()
        report.append((res.densify_iterations, want["iterations"], err))
        prev = want["dense"]
    s.close()
    return report


def test_config_b_stream_frames_vs_reference(gpu, ref):
    """1280x720 D=128 (the bench's frame): first + steady composited frame."""
    rep = _stream_vs_reference(gpu, ref, 1280, 720, 128, "k_pcg_tmem<10, 640>")
    assert len(rep) == 2
    assert rep[0][1] > rep[1][1]  # the first frame has no d_pre: many more iterations


def test_config_a_stream_frames_vs_reference(gpu, ref):
    """640x480 D=64 (BASELINE config A, the reference's CPU-runnable case)."""
    rep = _stream_vs_reference(gpu, ref, 640, 480, 64, "k_pcg_tmem<5, 512>")
    assert len(rep) == 2


def _stream_system(gpu, W, H, D, frames, seed=61):
    """Pushes `frames` synthetic frames through a stream; returns the last
    frame's solver inputs (sparse, edges, m_fuse, m_i) as device tensors, the
    previous composited frame's dense map (or None), and the stream's own
    dense map and iteration count."""
    from paper_2203_02300_b200.synth import StereoVideo

    cfg = Config(d_max=D - 1)
    vid = StereoVideo(W, H, seed=seed)
    s = gpu.Stream(W, H, cfg)
    pre = None
    res = None
    for i in range(frames):
        l8, r8 = vid.frame(i)
        if i == frames - 1 and i >= 3:
            pre = gpu.view_tensor(s.views().dense, (H, W), torch.float32).clone()
        res = s.push_gray8(T(l8), T(r8))
    v = s.views()
    qw, qh = W // 2, H // 2
    out = {k: gpu.view_tensor(getattr(v, k), shp, dt).clone() for k, shp, dt in (
        ("sparse", (H, W), torch.float32), ("edges", (H, W), torch.uint8), ("m_fuse", (qh, qw), torch.float32),
        ("m_i", (H, W), torch.float32), ("dense", (H, W), torch.float32))}
    solver = s.last_solver()
    s.close()
    return cfg, out, pre, res.densify_iterations, solver


@pytest.mark.parametrize("W,H,D,frames,solver", [
    (1920, 1080, 192, 4, "k_pcg_big<14, 1024>"),
    (3840, 2160, 256, 4, "k_pcg_stream<512,2>"),
])
def test_large_frame_solve_vs_reference(gpu, ref, W, H, D, frames, solver):
    """The stream's own steady-frame system at configs C and D: assembly
    bit-exact, the dispatched solver within tolerance of the reference's."""
    cfg, o, pre, iters, used = _stream_system(gpu, W, H, D, frames)
    assert used == solver
    host = {k: N(v) for k, v in o.items()}
    hpre = None if pre is None else N(pre)
    want_sys = ref.assemble_system(host["sparse"], host["edges"], host["m_fuse"], host["m_i"], hpre, cfg)
    sys = gpu.assemble_system(o["sparse"], o["edges"], o["m_fuse"], o["m_i"], pre, cfg)
    for k in ("diag", "coup_h", "coup_v", "rhs", "initial", "anchored"):
        assert bits_equal(N(getattr(sys, k)), want_sys[k]), k
    want, st = ref.solve_dense_depth(want_sys, cfg)
    got, gst = gpu.solve_dense_depth(sys, cfg)
    assert gpu.last_solver() == solver
    _dense_ok(N(got), want)
    assert abs(gst.iterations - st["iterations"]) <= 2, (gst.iterations, st["iterations"])
    # the stream's frame is the same solve
    assert iters == gst.iterations
    assert bits_equal(host["dense"], N(got))


def _ceil(a, b):
    return -(-a // b)


@pytest.mark.parametrize("ept", [2, 3, 4, 5, 6, 7])
def test_every_tmem_slot_count_vs_reference(gpu, ref, ept, monkeypatch):
    monkeypatch.setenv("DCO_PCG_1024", "1")  # the 1024-thread instances (EPT 6, 7 default to 640 threads)
    _tmem_slot_case(gpu, ref, ept, 1024, "k_pcg_tmem<%d>" % ept, monkeypatch)


@pytest.mark.parametrize("ept", [9, 10, 11])
def test_every_tmem640_slot_count_vs_reference(gpu, ref, ept, monkeypatch):
    """k_pcg_tmem<EPT, 640> (20 warps; XT = (96 - 8 EPT) / 2 x slots in TMEM,
    the rest in registers) on the same 640x360 system, reached with
    DCO_PCG_BLOCKS. (EPT 12 needs a chunk > 7040 unknowns: more shared memory
    than a CTA has, never dispatched.)"""
    _tmem_slot_case(gpu, ref, ept, 640, "k_pcg_tmem<%d, 640>" % ept, monkeypatch)


@pytest.mark.parametrize("ept", [5, 6, 7, 8, 9, 10])
def test_every_tmem512_slot_count_vs_reference(gpu, ref, ept, monkeypatch):
    """k_pcg_tmem<EPT, 512> (16 warps, 128 TMEM columns per warp), dispatched
    for systems needing 3..5 slots at 1024 threads (config A), reached with
    DCO_PCG_BLOCKS."""
    _tmem_slot_case(gpu, ref, ept, 512, "k_pcg_tmem<%d, 512>" % ept, monkeypatch)


def _tmem_slot_case(gpu, ref, ept, threads, name, monkeypatch):
    """k_pcg_tmem<EPT(, threads)> on one real 640x360 system: the largest grid
    whose chunk gives each thread EPT slots (and, for 640 threads, needs 6 or
    more at 1024, where the dispatch takes 640), so the register x slots run at
    a size the oracle solves in a second. (EPT 8 at 1024 threads needs a chunk
    > 7168 unknowns, 229 KB of shared memory: never dispatched.)"""
    W, H = 640, 360
    n = W * H
    k1024 = {1024: range(1, 9), 640: range(6, 9), 512: range(3, 6)}[threads]  # the dispatch's tiers
    blocks = max(b for b in range(1, 149) if _ceil(_ceil(n, b), threads) == ept and
                 _ceil(_ceil(n, b), 1024) in k1024)
    assert _ceil(n, blocks) * 32 + 16 * W <= 222 * 1024
    cfg, o, pre, _, _ = _stream_system(gpu, W, H, 64, 4, seed=7)
    host = {k: N(v) for k, v in o.items()}
    want_sys = ref.assemble_system(host["sparse"], host["edges"], host["m_fuse"], host["m_i"], N(pre), cfg)
    want, st = ref.solve_dense_depth(want_sys, cfg)
    monkeypatch.setenv("DCO_PCG_BLOCKS", str(blocks))
    sys = gpu.assemble_system(o["sparse"], o["edges"], o["m_fuse"], o["m_i"], pre, cfg)
    got, gst = gpu.solve_dense_depth(sys, cfg)
    assert gpu.last_solver() == name
    _dense_ok(N(got), want)
    assert abs(gst.iterations - st["iterations"]) <= 2
