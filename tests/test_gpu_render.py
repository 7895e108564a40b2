"""render_virtual / transform_mesh on the GPU vs the reference (oracle/_ref),
bit for bit (occlude.cpp:78-169): the cube of the pipeline,
posed cubes, and random triangle soups with overlaps, equal depths, triangles
behind the camera, degenerate and screen-filling triangles."""
import math

import numpy as np
import pytest
import torch

from paper_2203_02300_b200.config import InputError

pytestmark = pytest.mark.gpu


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def N(t):
    return t.detach().cpu().numpy()


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def cube(cx, cy, cz, side, color=(1.0, 0.55, 0.1)):
    """make_cube_mesh, occlude.cpp:89-105."""
    r = np.float32(side) / np.float32(2.0)
    v = []
    for i in range(8):
        v.append([np.float32(cx) + (r if i & 1 else -r), np.float32(cy) + (r if i & 2 else -r),
                  np.float32(cz) + (r if i & 4 else -r)])
    faces = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    tris = []
    for f in faces:
        tris.append((f[0], f[1], f[2]))
        tris.append((f[0], f[2], f[3]))
    return (np.array(v, np.float32), np.array(tris, np.int32),
            np.tile(np.array(color, np.float32), (8, 1)))


def pose_rt(yaw, pitch, tx, ty, tz):
    cy_, sy = math.cos(yaw), math.sin(yaw)
    cp, sp = math.cos(pitch), math.sin(pitch)
    rz = np.array([[cy_, -sy, 0], [sy, cy_, 0], [0, 0, 1]])
    rx = np.array([[1, 0, 0], [0, cp, -sp], [0, sp, cp]])
    r = rz @ rx
    p = np.eye(4)
    p[:3, :3] = r
    p[:3, 3] = [tx, ty, tz]
    return p.reshape(-1)


def render_both(gpu, ref, v, t, c, focal, w, h, pose=None):
    cx, cy = w / 2.0, h / 2.0
    want_rgb, want_d = ref.render_virtual(v, t, c, focal, cx, cy, w, h, pose)
    vg = T(v)
    if pose is not None:
        vg = gpu.transform_mesh(vg, pose)
        assert bits_equal(N(vg), ref.transform_mesh(v, pose))
    rgb, d = gpu.render_virtual(vg, T(t), T(c), focal, cx, cy, w, h)
    return N(rgb), N(d), want_rgb, want_d


def test_cube_matches_reference(gpu, ref):
    w, h = 320, 192
    v, t, c = cube(0.0, 0.0, 1.5, 0.3)
    rgb, d, want_rgb, want_d = render_both(gpu, ref, v, t, c, 200.0, w, h)
    assert np.isfinite(d).sum() > 1000
    assert bits_equal(d, want_d) and bits_equal(rgb, want_rgb)
    # and the oracle's own cube helper agrees with this mesh
    vr, vd = ref.render_cube(w, h, 200.0, cz=1.5, side=0.3)
    assert bits_equal(vd, want_d) and bits_equal(vr, want_rgb)


@pytest.mark.parametrize("k", range(4))
def test_posed_cube_matches_reference(gpu, ref, k):
    w, h = 640, 360
    v, t, c = cube(0.05 * k, -0.03, 0.0, 0.4, color=(0.2 + 0.1 * k, 0.7, 0.3))
    pose = pose_rt(0.4 * k + 0.1, 0.3 - 0.2 * k, 0.02 * k, 0.01, 1.2 + 0.1 * k)
    rgb, d, want_rgb, want_d = render_both(gpu, ref, v, t, c, 420.0, w, h, pose)
    assert np.isfinite(d).sum() > 1000
    assert bits_equal(d, want_d) and bits_equal(rgb, want_rgb)


@pytest.mark.parametrize("seed", [3, 17, 29])
def test_triangle_soup_matches_reference(gpu, ref, seed):
    """Random overlapping triangles (order-dependent winners), some behind the
    camera, some degenerate, a few huge: the whole index-ordered z-buffer."""
    rng = np.random.default_rng(seed)
    w, h = 256, 160
    nt = 600
    v = np.empty((3 * nt, 3), np.float32)
    for i in range(nt):
        cxy = rng.uniform(-0.8, 0.8, 2)
        z = rng.choice([rng.uniform(0.5, 3.0), 1.0])  # many exactly equal depths
        s = rng.choice([0.02, 0.1, 0.6, 4.0], p=[0.4, 0.4, 0.15, 0.05])
        for k in range(3):
            v[3 * i + k, :2] = cxy + rng.uniform(-s, s, 2)
            v[3 * i + k, 2] = z + (rng.uniform(-0.3, 0.3) if rng.random() < 0.5 else 0.0)
    v[::37, 2] = -0.5  # behind the camera
    v[5, :] = v[4, :]  # a degenerate triangle (two equal vertices)
    t = np.arange(3 * nt, dtype=np.int32).reshape(nt, 3)
    c = rng.uniform(0.0, 1.0, (3 * nt, 3)).astype(np.float32)
    rgb, d, want_rgb, want_d = render_both(gpu, ref, v, t, c, 150.0, w, h)
    assert np.isfinite(d).sum() > 100
    assert bits_equal(d, want_d) and bits_equal(rgb, want_rgb)


def test_many_triangles_per_tile_take_the_ordered_fallback(gpu, ref):
    """More triangles on one tile than the shared-memory sort holds (4096):
    those tiles walk the whole mesh in order; still bit-exact."""
    rng = np.random.default_rng(5)
    w, h = 64, 48
    nt = 5000
    v = np.empty((3 * nt, 3), np.float32)
    for i in range(nt):
        base = rng.uniform(-0.05, 0.05, 2)
        for k in range(3):
            v[3 * i + k, :2] = base + rng.uniform(-0.3, 0.3, 2)
            v[3 * i + k, 2] = rng.uniform(1.0, 2.0)
    t = np.arange(3 * nt, dtype=np.int32).reshape(nt, 3)
    c = rng.uniform(0.0, 1.0, (3 * nt, 3)).astype(np.float32)
    rgb, d, want_rgb, want_d = render_both(gpu, ref, v, t, c, 60.0, w, h)
    assert bits_equal(d, want_d) and bits_equal(rgb, want_rgb)


def test_empty_mesh_and_bad_dims(gpu, ref):
    v = np.zeros((3, 3), np.float32)
    t = np.zeros((0, 3), np.int32)
    c = np.zeros((3, 3), np.float32)
    rgb, d = gpu.render_virtual(T(v), T(t), T(c), 100.0, 8.0, 8.0, 16, 16)
    assert np.isnan(N(d)).all() and (N(rgb) == 0).all()
    with pytest.raises(InputError):
        gpu.render_virtual(T(v), T(np.zeros((1, 3), np.int32)), T(c), 100.0, 0.0, 0.0, 0, 16)


def test_stream_renders_posed_mesh_per_frame(gpu, ref):
    """dco_stream with a mesh and per-frame poses: the composite of every frame
    equals the reference's render_virtual(transform_mesh(mesh, pose of the
    middle frame)) composited on the reference pipeline's dense map."""
    from paper_2203_02300_b200.config import Config
    from tests.inputs import scene

    W, H = 320, 192
    cfg = Config(d_max=47)
    fs = [scene(ref, W, H, index=i, seed=777) for i in range(5)]
    v, t, c = cube(0.0, 0.0, 0.0, 0.25)
    poses = [pose_rt(0.3 * i, 0.2, 0.01 * i, -0.02, 1.3) for i in range(5)]
    s = gpu.Stream(W, H, cfg)
    s.set_mesh(v, t, c)
    prev = None
    for i, f in enumerate(fs):
        s.set_next_pose(poses[i])
        res = s.push_gray8(T(f["left8"]), T(f["right8"]))
        if i < 2:
            continue
        vrgb, vdepth = ref.render_virtual(v, t, c, cfg.focal_px, W / 2.0, H / 2.0, W, H, poses[i - 1])
        q = [ref.downsample_half(fs[j]["left"]) for j in (i - 2, i - 1, i)]
        mid = fs[i - 1]
        want = ref.pipeline_frame(q[0], q[1], q[2], mid["left"], ref.downsample_half(mid["right"]),
                                  np.repeat(mid["left"][:, :, None], 3, 2), prev, vrgb, vdepth, cfg)
        vw = s.views()
        dense = N(gpu.view_tensor(vw.dense, (H, W), torch.float32))
        mask = N(gpu.view_tensor(vw.mask, (H, W), torch.uint8))
        comp = N(gpu.view_tensor(vw.composite, (H, W, 3), torch.float32))
        assert np.isfinite(vdepth).sum() > 500
        # composite == the reference's wherever the depth test is decided away
        # from the solver tolerance (the dense map is tolerance-matched)
        close = np.abs(vdepth - want["dense"]) <= 2e-5
        assert ((mask == want["mask"]) | close).all()
        agree = ~close
        assert bits_equal(comp[agree], want["composite"][agree])
        assert np.abs(dense.astype(np.float64) - want["dense"]).max() <= 1e-5
        prev = want["dense"]
    s.close()
