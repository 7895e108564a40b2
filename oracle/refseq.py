"""Writes a sequence the reference's run_pipeline (pipeline.cpp:108-321) reads:
8-bit PGM frames, a manifest with per-frame poses (load_manifest,
pipeline.cpp:24-55), an OBJ mesh (load_obj, occlude.cpp:10-60) and a
key=value config file (load_config, config.cpp:118-142).

TEST INFRASTRUCTURE ONLY (bench.py's reference arm / cpu_baseline, tests):
the way the reference itself is driven, so its own public API and stock code
path are what gets timed."""
import os

import numpy as np


def write_pgm8(path, img8):
    h, w = img8.shape
    with open(path, "wb") as f:
        f.write(b"P5\n%d %d\n255\n" % (w, h))
        f.write(np.ascontiguousarray(img8, np.uint8).tobytes())


def write_obj(path, vertices, triangles, colors):
    with open(path, "w") as f:
        for v, c in zip(vertices, colors):
            f.write("v %.9g %.9g %.9g %.9g %.9g %.9g\n" % (v[0], v[1], v[2], c[0], c[1], c[2]))
        for t in triangles:
            f.write("f %d %d %d\n" % (t[0] + 1, t[1] + 1, t[2] + 1))


def write_config(path, cfg):
    with open(path, "w") as f:
        for k, v in cfg.as_dict().items():
            f.write("%s=%r\n" % (k, v))


def write_sequence(root, frames, poses=None, mesh=None, cfg=None, keep_outputs=()):
    """frames: list of (left u8, right u8). Returns (config, manifest, out_dir,
    mesh) paths. Per-frame outputs run_pipeline writes (composite PPM, mask
    PGM, dense PFM, timings.csv) go to /dev/null through pre-made symlinks,
    except the frame indices in keep_outputs (real files, for parity checks):
    the writes still execute, outside the reference's frame timer."""
    os.makedirs(root, exist_ok=True)
    out = os.path.join(root, "out")
    os.makedirs(out, exist_ok=True)
    lines = []
    for i, (l8, r8) in enumerate(frames):
        lp, rp = "l%04d.pgm" % i, "r%04d.pgm" % i
        write_pgm8(os.path.join(root, lp), l8)
        write_pgm8(os.path.join(root, rp), r8)
        pose = "" if poses is None else " " + " ".join("%.17g" % x for x in poses[i])
        lines.append("%d %s %s%s\n" % (i, lp, rp, pose))
        if i not in keep_outputs:
            for name in ("composite_%04d.ppm", "mask_%04d.pgm", "dense_%04d.pfm"):
                p = os.path.join(out, name % i)
                if not os.path.lexists(p):
                    os.symlink("/dev/null", p)
    tp = os.path.join(out, "timings.csv")
    if not os.path.lexists(tp):
        os.symlink("/dev/null", tp)
    manifest = os.path.join(root, "manifest.txt")
    with open(manifest, "w") as f:
        f.writelines(lines)
    cfg_path = None
    if cfg is not None:
        cfg_path = os.path.join(root, "config.txt")
        write_config(cfg_path, cfg)
    mesh_path = None
    if mesh is not None:
        mesh_path = os.path.join(root, "mesh.obj")
        write_obj(mesh_path, *mesh)
    return cfg_path, manifest, out, mesh_path


def read_pfm(path):
    """A write_pfm file (codec.cpp:293-309): rows bottom-up, nodata as +inf."""
    with open(path, "rb") as f:
        data = f.read()
    parts = data.split(b"\n", 3)
    w, h = (int(x) for x in parts[1].split())
    scale = float(parts[2])
    arr = np.frombuffer(parts[3][: 4 * w * h], dtype="<f4" if scale < 0 else ">f4").reshape(h, w)
    return np.ascontiguousarray(arr[::-1]).astype(np.float32)
