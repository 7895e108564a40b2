"""Device half of ingest / egress (codec.cpp:23-26, image.cpp:7-15): quantize
and to_gray bit-exact with the reference, and dco.write_pgm / write_ppm files
(device quantisation, bytes over PCIe) byte-identical to the reference's."""
import numpy as np
import pytest
import torch

from tests.test_gpu_stereo import N, T, bits_equal

pytestmark = pytest.mark.gpu


def test_quantize_and_files_equal_reference(gpu, ref, tmp_path):
    rng = np.random.default_rng(11)
    img = rng.uniform(-0.3, 1.3, (33, 47)).astype(np.float32)
    img[0, :6] = [np.nan, 0.0, 1.0, 0.5 / 255, 1.5 / 255, 254.5 / 255]  # NaN, ends, half-way points
    ref.write_pgm(img, str(tmp_path / "r.pgm"))
    want = gpu.read_pnm(str(tmp_path / "r.pgm"))
    assert bits_equal(N(gpu.quantize_u8(T(img))), want)
    gpu.write_pgm(str(tmp_path / "o.pgm"), T(img))
    assert open(tmp_path / "o.pgm", "rb").read() == open(tmp_path / "r.pgm", "rb").read()
    rgb = rng.uniform(-0.1, 1.1, (9, 13, 3)).astype(np.float32)
    ref.write_ppm(rgb, str(tmp_path / "r.ppm"))
    gpu.write_ppm(str(tmp_path / "o.ppm"), T(rgb))
    assert open(tmp_path / "o.ppm", "rb").read() == open(tmp_path / "r.ppm", "rb").read()


def test_to_gray_and_gray8_ingest(gpu, ref, tmp_path):
    rng = np.random.default_rng(12)
    rgb = rng.uniform(0.0, 1.0, (31, 65, 3)).astype(np.float32)
    assert bits_equal(N(gpu.to_gray(T(rgb))), ref.to_gray(rgb))
    # read_gray of a PGM = dco_read_pnm bytes -> dco_ingest_gray8 (bytes / 255 on the device)
    ref.write_pgm(rgb[:, :, 0], str(tmp_path / "g.pgm"))
    b = gpu.read_pnm(str(tmp_path / "g.pgm"))
    full, _ = gpu.ingest_gray8(torch.from_numpy(b).cuda())
    assert bits_equal(N(full), ref.read_pnm(str(tmp_path / "g.pgm")))
