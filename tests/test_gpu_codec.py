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


def test_stream_encoded_outputs_equal_reference_files(gpu, ref, tmp_path):
    """dco_stream_push_gray8_host_encoded: the frame's outputs as run_pipeline
    writes them (pipeline.cpp:266-268). Against a twin stream's float outputs
    (dco_stream_push_gray8_host, same frames, mesh and poses): the composite
    bytes equal the reference's write_ppm payload of the float composite, the
    mask bytes are write_mask_pgm's 0/255 (codec.cpp:243-247), the dense map
    is bit-identical."""
    from paper_2203_02300_b200.config import Config
    from paper_2203_02300_b200.synth import StereoVideo

    W, H = 320, 192
    cfg = Config(d_max=47)
    vid = StereoVideo(W, H, seed=5)
    a, b = gpu.Stream(W, H, cfg), gpu.Stream(W, H, cfg)
    cube_v = np.array([[x, y, z] for z in (-0.15, 0.15) for y in (-0.15, 0.15) for x in (-0.15, 0.15)], np.float32)
    faces = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    cube_t = np.array([t for f in faces for t in ((f[0], f[1], f[2]), (f[0], f[2], f[3]))], np.int32)
    cube_c = np.tile(np.array([1.0, 0.55, 0.1], np.float32), (8, 1))
    for s in (a, b):
        s.set_mesh(cube_v, cube_t, cube_c)
    comp = torch.empty((H, W, 3)).pin_memory()
    mask = torch.empty((H, W), dtype=torch.uint8).pin_memory()
    dense = torch.empty((H, W)).pin_memory()
    comp8 = torch.empty((H, W, 3), dtype=torch.uint8).pin_memory()
    mask8 = torch.empty((H, W), dtype=torch.uint8).pin_memory()
    dense2 = torch.empty((H, W)).pin_memory()
    checked = 0
    for i in range(5):
        l8, r8 = (torch.from_numpy(x).pin_memory() for x in vid.frame(i))
        pose = [1.0, 0, 0, 0.02 * i, 0, 1.0, 0, 0, 0, 0, 1.0, 1.5, 0, 0, 0, 1.0]
        for s in (a, b):
            s.set_next_pose(pose)
        ra = a.push_gray8_host(l8, r8, comp, mask, dense)
        rb = b.push_gray8_host_encoded(l8, r8, comp8, mask8, dense2)
        assert ra.composited == rb.composited
        if not ra.composited:
            continue
        ref.write_ppm(comp.numpy(), str(tmp_path / "c.ppm"))
        payload = open(tmp_path / "c.ppm", "rb").read()[-3 * W * H:]
        assert payload == comp8.numpy().tobytes()
        assert np.array_equal(mask8.numpy(), mask.numpy().astype(np.uint8) * 255)
        assert bits_equal(dense2.numpy(), dense.numpy())
        checked += 1
    assert checked == 3
    a.close()
    b.close()
