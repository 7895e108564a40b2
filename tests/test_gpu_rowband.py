"""A whole row-band frame loop (paper_2203_02300_b200/rowband.py) with G bands
on this GPU against the reference pipeline (pipeline.cpp:183-258 via
oracle/_ref) and the whole-frame stream: sparse depth bit-exact, dense depth
within the solver tolerance, composite exact wherever the depth test is not
decided inside that tolerance; the d_pre chain carried band by band."""
import numpy as np
import pytest

from paper_2203_02300_b200.config import Config
from paper_2203_02300_b200.rowband import LocalLinks, RowBandFrames
from tests.inputs import scene
from tests.test_gpu_densify import MAX_ABS, RMS
from tests.test_gpu_stereo import N, T, bits_equal

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bands,chunk,seq_mean", [(1, None, False), (2, None, False), (3, 32, False), (5, 64, False),
                                                  (3, None, True)])
def test_rowband_frames_match_reference(gpu, ref, bands, chunk, seq_mean):
    """chunk: the carry travels in slice chunks (as under torchrun). seq_mean:
    the frame-wide sparse mean through the gathered-map sequential path (the
    one taken outside the exactness guard) instead of the bands' partials."""
    W, H = 640, 360
    cfg = Config(d_max=47)
    fs = [scene(ref, W, H, index=i, seed=91) for i in range(5)]
    q = [ref.downsample_half(f["left"]) for f in fs]
    rb = RowBandFrames(W, H, cfg, LocalLinks(bands), chunk=chunk)
    rb.force_sequential_mean = seq_mean
    prev = None
    for i in range(1, 4):
        mid = fs[i]
        rq = ref.downsample_half(mid["right"])
        rgb = np.repeat(mid["left"][:, :, None], 3, 2)
        vdepth = np.full((H, W), 1.7, np.float32)
        vdepth[: H // 2] = np.nan
        vrgb = np.full((H, W, 3), 0.25, np.float32)
        want = ref.pipeline_frame(q[i - 1], q[i], q[i + 1], mid["left"], rq, rgb, prev, vrgb, vdepth, cfg)
        got = rb.frame(T(q[i - 1]), T(q[i]), T(q[i + 1]), T(mid["left"]), T(rq), T(rgb), T(vrgb), T(vdepth))
        assert sorted(got) == list(range(bands))
        dense = np.concatenate([N(got[k]["dense"]) for k in range(bands)])
        sparse = np.concatenate([N(got[k]["sparse"]) for k in range(bands)])
        comp = np.concatenate([N(got[k]["composite"]) for k in range(bands)])
        mask = np.concatenate([N(got[k]["mask"]) for k in range(bands)])
        assert bits_equal(sparse, want["sparse"])
        d = np.abs(dense.astype(np.float64) - want["dense"])
        assert d.max() <= MAX_ABS and np.sqrt((d ** 2).mean()) <= RMS, d.max()
        assert abs(rb.iterations - want["iterations"]) <= 2
        close = np.abs(vdepth - want["dense"]) <= 2e-5
        assert ((mask == want["mask"]) | close).all()
        assert bits_equal(comp[~close], want["composite"][~close])
        prev = want["dense"]
    rb.close()
