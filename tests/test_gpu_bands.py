"""Row bands: the stereo chain run band by band with the
recompute halo and the aggregation column-prefix carry, concatenated, is bit
for bit the whole frame's -- and so the reference's (stereo.cpp:106-315 via
test_gpu_stereo). The bands run one after another on one GPU, each handing its
carry to the next exactly as the ranks of a multi-GPU job do over NCCL; no
kernel waits on another."""
import numpy as np
import pytest
import torch

from paper_2203_02300_b200.config import Config, InputError
from tests.inputs import scene

pytestmark = pytest.mark.gpu


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def N(t):
    return t.cpu().numpy()


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def run_bands(gpu, lq, rq, cfg, fw, fh, bands):
    disp, sparse, carry = [], [], None
    for k in range(bands):
        b = gpu.band_plan(cfg, fw, fh, bands, k)
        d, s, carry_out = gpu.stereo_band(T(lq[b.sub0:b.sub1]), T(rq[b.sub0:b.sub1]), b, cfg, fw, fh,
                                          carry_in=carry if b.carry_row > 0 else None)
        disp.append(N(d))
        sparse.append(N(s))
        if carry_out is not None:
            carry = carry_out
    return np.concatenate(disp), np.concatenate(sparse)


CASES = [
    # (full w, full h, D, bands, config overrides)
    (640, 480, 64, 2, {}),
    (640, 480, 64, 3, {}),
    (1280, 720, 128, 4, {}),
    (960, 542, 48, 5, {}),  # uneven bands
    (642, 363, 32, 2, {}),  # odd full height: the last band carries the extra row
    (640, 480, 64, 3, dict(hist_iterations=0)),
    (640, 480, 64, 3, dict(hist_iterations=3)),
    (640, 480, 64, 4, dict(census_window_w=7, census_window_h=5, cross_arm_l1=9, cross_arm_l2=5)),
    (320, 480, 32, 8, {}),  # bands thinner than the halo: carries cross several bands
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "%dx%d_D%d_G%d%s" % (c[0], c[1], c[2], c[3],
                                                                         "_" + "_".join(c[4]) if c[4] else ""))
def test_bands_equal_whole_frame(gpu, ref, case):
    fw, fh, D, bands, over = case
    cfg = Config(d_max=D - 1, **over)
    f = scene(ref, (fw + 7) // 8 * 8, (fh + 7) // 8 * 8, seed=7 + bands)  # synth needs multiples of 8
    lq, rq = ref.downsample_half(f["left"][:fh, :fw]), ref.downsample_half(f["right"][:fh, :fw])
    want_d, want_s = gpu.stereo_sparse_depth(T(lq), T(rq), cfg, fw, fh)
    got_d, got_s = run_bands(gpu, lq, rq, cfg, fw, fh, bands)
    assert np.isfinite(got_d).sum() > 0.5 * got_d.size
    assert bits_equal(got_d, N(want_d))
    assert bits_equal(got_s, N(want_s))


def test_bands_equal_reference(gpu, ref):
    """The acceptance KAT frame (acceptance.cpp:114-158) in 3 bands against the
    oracle's own chain."""
    fw, fh, bands = 960, 320, 3
    cfg = Config()
    f = ref.render_synth_frame(960, 320, 0, square_size=160, square_x0=400.0, square_y0=80.0, shift_x=0.0, seed=7)
    lq, rq = ref.downsample_half(f["left"]), ref.downsample_half(f["right"])
    got_d, got_s = run_bands(gpu, lq, rq, cfg, fw, fh, bands)
    arms = ref.build_cross_windows(lq, cfg)
    d = ref.refine_disparity_histogram(
        ref.select_disparity_wta(ref.aggregate_costs(ref.compute_cost_volume(lq, rq, arms, cfg), arms)), arms, 2)
    assert bits_equal(got_d, d)
    assert bits_equal(got_s, ref.disparity_to_sparse_depth(d, cfg, fw, fh))
    assert np.isfinite(got_s).sum() == 74781


def test_carry_is_the_exact_column_prefix(gpu, ref):
    """With a wrong prefix (the right one + 1e15: same differences, coarser
    rounding) the owned rows of a lower band differ: the exchange is real."""
    fw, fh, bands = 640, 480, 2
    cfg = Config(d_max=63)
    f = scene(ref, fw, fh, seed=11)
    lq, rq = ref.downsample_half(f["left"]), ref.downsample_half(f["right"])
    b0 = gpu.band_plan(cfg, fw, fh, bands, 0)
    b1 = gpu.band_plan(cfg, fw, fh, bands, 1)
    _, _, carry = gpu.stereo_band(T(lq[b0.sub0:b0.sub1]), T(rq[b0.sub0:b0.sub1]), b0, cfg, fw, fh)
    assert carry is not None and b1.carry_row > 0
    right, _, _ = gpu.stereo_band(T(lq[b1.sub0:b1.sub1]), T(rq[b1.sub0:b1.sub1]), b1, cfg, fw, fh, carry_in=carry)
    wrong, _, _ = gpu.stereo_band(T(lq[b1.sub0:b1.sub1]), T(rq[b1.sub0:b1.sub1]), b1, cfg, fw, fh,
                                  carry_in=carry + 1e15)
    whole, _ = gpu.stereo_sparse_depth(T(lq), T(rq), cfg, fw, fh)
    assert bits_equal(N(right), N(whole)[b1.row0:b1.row1])
    assert not bits_equal(N(wrong), N(whole)[b1.row0:b1.row1])
    with pytest.raises(InputError):
        gpu.stereo_band(T(lq[b1.sub0:b1.sub1]), T(rq[b1.sub0:b1.sub1]), b1, cfg, fw, fh, carry_in=None)
    with pytest.raises(InputError):
        gpu.stereo_band(T(lq[b1.sub0:b1.sub1 - 1]), T(rq[b1.sub0:b1.sub1 - 1]), b1, cfg, fw, fh, carry_in=carry)


@pytest.mark.parametrize("chunk", [32, 64])
def test_phased_chunked_carry_equals_one_call(gpu, ref, chunk):
    """begin / vpass per slice chunk / end, carries per chunk: the same bits as
    the one-call band and the whole frame."""
    fw, fh, bands = 640, 480, 3
    cfg = Config(d_max=95)
    f = scene(ref, fw, fh, seed=13)
    lq, rq = ref.downsample_half(f["left"]), ref.downsample_half(f["right"])
    nd = 96
    chunks = [(d0, min(nd, d0 + chunk)) for d0 in range(0, nd, chunk)]
    carries, disp = {}, []
    for k in range(bands):
        b = gpu.band_plan(cfg, fw, fh, bands, k)
        gpu.stereo_band_begin(T(lq[b.sub0:b.sub1]), T(rq[b.sub0:b.sub1]), b, cfg, fw, fh)
        for d0, d1 in chunks:
            out = gpu.stereo_band_vpass(b, cfg, fw, fh, d0, d1, carries.get((k, d0)) if b.carry_row > 0 else None)
            if out is not None:
                carries[(k + 1, d0)] = out
        d, _ = gpu.stereo_band_end(b, cfg, fw, fh)
        disp.append(N(d))
    whole, _ = gpu.stereo_sparse_depth(T(lq), T(rq), cfg, fw, fh)
    assert bits_equal(np.concatenate(disp), N(whole))
    with pytest.raises(InputError):  # chunks start at multiples of 32
        b = gpu.band_plan(cfg, fw, fh, bands, 0)
        gpu.stereo_band_begin(T(lq[b.sub0:b.sub1]), T(rq[b.sub0:b.sub1]), b, cfg, fw, fh)
        gpu.stereo_band_vpass(b, cfg, fw, fh, 16, 48)
