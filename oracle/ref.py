"""numpy front-end of oracle/_ref/libdco_ref.so (the unmodified reference,
see oracle/ref_capi.cpp). TEST INFRASTRUCTURE ONLY: used by tests/,
__graft_entry__.smoke() and bench.py's CPU legs as the checker / CPU baseline.
Function names are the reference's stage names; arrays are numpy."""
import ctypes
import os

import numpy as np

from . import REF_LIB
from paper_2203_02300_b200.config import Config, raise_for

_lib = None
P = ctypes.c_void_p
I, D, U64 = ctypes.c_int, ctypes.c_double, ctypes.c_uint64
CFG = ctypes.POINTER(Config)


def available():
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError("oracle/_ref/libdco_ref.so missing: run `make -C oracle ref` where /root/reference exists")
        L = ctypes.CDLL(REF_LIB)
        sig = {
            "ref_last_error": (ctypes.c_char_p, []),
            "ref_config_default": (None, [CFG]),
            "ref_config_validate": (I, [CFG]),
            "ref_load_config": (I, [ctypes.c_char_p, CFG]),
            "ref_render_synth_frame": (I, [I, I, D, D, D, D, I, D, D, D, D, U64, I, P, P, P, P, P, P]),
            "ref_pgm_roundtrip": (I, [P, I, I, ctypes.c_char_p, P, P]),
            "ref_write_pgm": (I, [P, I, I, ctypes.c_char_p]),
            "ref_write_ppm": (I, [P, I, I, ctypes.c_char_p]),
            "ref_write_pfm": (I, [P, I, I, ctypes.c_char_p]),
            "ref_read_pnm": (I, [ctypes.c_char_p, I, P, ctypes.c_size_t, ctypes.POINTER(I), ctypes.POINTER(I)]),
            "ref_to_gray": (I, [P, I, I, P]),
            "ref_downsample_half": (I, [P, I, I, P]),
            "ref_build_cross_windows": (I, [P, I, I, CFG, P, P, P, P]),
            "ref_census_transform": (I, [P, I, I, I, I, P]),
            "ref_adaptive_alpha": (D, [I, CFG]),
            "ref_compute_cost_volume": (I, [P, P, I, I, P, P, P, P, CFG, P]),
            "ref_aggregate_costs": (I, [P, I, I, I, I, P, P, P, P, P]),
            "ref_select_disparity_wta": (I, [P, I, I, I, I, P]),
            "ref_refine_disparity_histogram": (I, [P, I, I, P, P, P, P, I, P]),
            "ref_disparity_to_sparse_depth": (I, [P, I, I, CFG, I, I, P]),
            "ref_compute_flow": (I, [P, P, I, I, CFG, P, P]),
            "ref_flow_to_polar": (I, [P, P, I, I, P, P]),
            "ref_gradient_amplitude": (I, [P, I, I, P]),
            "ref_fuse_amplitudes": (I, [P, P, P, P, P, P, I, I, CFG, P]),
            "ref_box_filter": (I, [P, I, I, I, P]),
            "ref_normalize_amplitude": (I, [P, I, I, P]),
            "ref_gaussian_blur": (I, [P, I, I, D, P]),
            "ref_extract_depth_contours_prefiltered": (I, [P, I, I, P, I, I, CFG, P, P]),
            "ref_smoothness_weight": (I, [I, I, I, I, P, I, I, P, I, I, P, ctypes.POINTER(D)]),
            "ref_assemble_system": (I, [P, P, P, I, I, P, P, I, I, CFG, P, P, P, P, P, P, ctypes.POINTER(D), ctypes.POINTER(U64)]),
            "ref_apply_system": (I, [I, I, P, P, P, P, P]),
            "ref_solve_dense_depth": (I, [I, I, P, P, P, P, P, P, D, CFG, P, ctypes.POINTER(I), ctypes.POINTER(D),
                                          ctypes.POINTER(D), ctypes.POINTER(D), P, I]),
            "ref_composite": (I, [P, P, P, P, I, I, P, P]),
            "ref_render_cube": (I, [ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float, D, I, I, P, P]),
            "ref_render_virtual": (I, [P, I, P, I, P, P, D, D, D, I, I, P, P]),
            "ref_transform_mesh": (I, [P, I, P, P]),
            "ref_run_pipeline": (I, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, I, P, P, P,
                                     ctypes.POINTER(I)]),
            "ref_format_bench_report": (I, [I, P, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p]),
            "ref_pipeline_frame": (I, [I, I, P, P, P, P, P, P, P, P, P, CFG, P, P, P, P, P, ctypes.POINTER(I),
                                       ctypes.POINTER(D)]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _check(st):
    if st != 0:
        raise_for(st, lib().ref_last_error().decode())


def default_config():
    c = Config()
    lib().ref_config_default(ctypes.byref(c))
    return c


def validate(cfg):
    _check(lib().ref_config_validate(ctypes.byref(cfg)))


def load_config(path):
    c = Config()
    _check(lib().ref_load_config(path.encode(), ctypes.byref(c)))
    return c


def render_synth_frame(width, height, index=0, z_fg=1.0, z_bg=2.0, focal_px=400.0, baseline_m=0.12,
                       square_size=80, square_x0=96.0, square_y0=56.0, shift_x=4.0, shift_y=0.0, seed=1234):
    """render_synth_frame, synth.cpp:68-135 -> dict of numpy arrays."""
    n = width * height
    out = {k: np.empty(n, np.float32) for k in ("left", "right", "gt_depth", "gt_u", "gt_v")}
    out["gt_boundary"] = np.empty(n, np.uint8)
    _check(lib().ref_render_synth_frame(width, height, z_fg, z_bg, focal_px, baseline_m, square_size, square_x0,
                                        square_y0, shift_x, shift_y, seed, index, _p(out["left"]),
                                        _p(out["right"]), _p(out["gt_depth"]), _p(out["gt_boundary"]),
                                        _p(out["gt_u"]), _p(out["gt_v"])))
    return {k: v.reshape(height, width) for k, v in out.items()}


def quantize8(img):
    """write_pgm quantisation (codec.cpp:23-26, 211-229): bytes, and read_gray's bytes/255.0f."""
    import tempfile

    img = _c(img, np.float32)
    h, w = img.shape
    b = np.empty((h, w), np.uint8)
    back = np.empty((h, w), np.float32)
    with tempfile.NamedTemporaryFile(suffix=".pgm") as f:
        _check(lib().ref_pgm_roundtrip(_p(img), w, h, f.name.encode(), _p(b), _p(back)))
    return b, back


def downsample_half(img):
    img = _c(img, np.float32)
    h, w = img.shape
    out = np.empty((h // 2, w // 2), np.float32)
    _check(lib().ref_downsample_half(_p(img), w, h, _p(out)))
    return out


def build_cross_windows(img, cfg):
    img = _c(img, np.float32)
    h, w = img.shape
    arms = np.empty((4, h, w), np.uint8)
    _check(lib().ref_build_cross_windows(_p(img), w, h, ctypes.byref(cfg), *[_p(arms[i]) for i in range(4)]))
    return arms


def census_transform(img, ww, wh):
    img = _c(img, np.float32)
    h, w = img.shape
    out = np.empty((h, w), np.uint64)
    _check(lib().ref_census_transform(_p(img), w, h, ww, wh, _p(out)))
    return out


def adaptive_alpha(l_min, cfg):
    return lib().ref_adaptive_alpha(l_min, ctypes.byref(cfg))


def compute_cost_volume(left, right, arms, cfg):
    left, right, arms = _c(left, np.float32), _c(right, np.float32), _c(arms, np.uint8)
    h, w = left.shape
    out = np.empty((h, w, cfg.d_max - cfg.d_min + 1), np.float32)
    _check(lib().ref_compute_cost_volume(_p(left), _p(right), w, h, *[_p(arms[i]) for i in range(4)],
                                         ctypes.byref(cfg), _p(out)))
    return out


def aggregate_costs(vol, arms, d_min=0):
    vol, arms = _c(vol, np.float32), _c(arms, np.uint8)
    h, w, nd = vol.shape
    out = np.empty_like(vol)
    _check(lib().ref_aggregate_costs(_p(vol), w, h, d_min, d_min + nd - 1, *[_p(arms[i]) for i in range(4)], _p(out)))
    return out


def select_disparity_wta(vol, d_min=0):
    vol = _c(vol, np.float32)
    h, w, nd = vol.shape
    out = np.empty((h, w), np.float32)
    _check(lib().ref_select_disparity_wta(_p(vol), w, h, d_min, d_min + nd - 1, _p(out)))
    return out


def refine_disparity_histogram(disp, arms, iterations):
    disp, arms = _c(disp, np.float32), _c(arms, np.uint8)
    h, w = disp.shape
    out = np.empty_like(disp)
    _check(lib().ref_refine_disparity_histogram(_p(disp), w, h, *[_p(arms[i]) for i in range(4)], iterations, _p(out)))
    return out


def disparity_to_sparse_depth(disp, cfg, fw, fh):
    disp = _c(disp, np.float32)
    h, w = disp.shape
    out = np.empty((fh, fw), np.float32)
    _check(lib().ref_disparity_to_sparse_depth(_p(disp), w, h, ctypes.byref(cfg), fw, fh, _p(out)))
    return out


def compute_flow(frm, to, cfg):
    frm, to = _c(frm, np.float32), _c(to, np.float32)
    h, w = frm.shape
    u, v = np.empty((h, w), np.float32), np.empty((h, w), np.float32)
    _check(lib().ref_compute_flow(_p(frm), _p(to), w, h, ctypes.byref(cfg), _p(u), _p(v)))
    return u, v


def flow_to_polar(u, v):
    u, v = _c(u, np.float32), _c(v, np.float32)
    h, w = u.shape
    r, t = np.empty_like(u), np.empty_like(u)
    _check(lib().ref_flow_to_polar(_p(u), _p(v), w, h, _p(r), _p(t)))
    return r, t


def gradient_amplitude(r):
    r = _c(r, np.float32)
    h, w = r.shape
    out = np.empty_like(r)
    _check(lib().ref_gradient_amplitude(_p(r), w, h, _p(out)))
    return out


def fuse_amplitudes(past, future, mp, mf, cfg):
    pu, pv = _c(past[0], np.float32), _c(past[1], np.float32)
    fu, fv = _c(future[0], np.float32), _c(future[1], np.float32)
    mp, mf = _c(mp, np.float32), _c(mf, np.float32)
    h, w = mp.shape
    out = np.empty_like(mp)
    _check(lib().ref_fuse_amplitudes(_p(pu), _p(pv), _p(fu), _p(fv), _p(mp), _p(mf), w, h, ctypes.byref(cfg), _p(out)))
    return out


def box_filter(a, radius):
    a = _c(a, np.float32)
    h, w = a.shape
    out = np.empty_like(a)
    _check(lib().ref_box_filter(_p(a), w, h, radius, _p(out)))
    return out


def normalize_amplitude(a):
    a = _c(a, np.float32)
    h, w = a.shape
    out = np.empty_like(a)
    _check(lib().ref_normalize_amplitude(_p(a), w, h, _p(out)))
    return out


def gaussian_blur(img, sigma):
    img = _c(img, np.float32)
    h, w = img.shape
    out = np.empty_like(img)
    _check(lib().ref_gaussian_blur(_p(img), w, h, sigma, _p(out)))
    return out


def extract_depth_contours_prefiltered(blurred, m_fuse, cfg):
    blurred, m_fuse = _c(blurred, np.float32), _c(m_fuse, np.float32)
    h, w = blurred.shape
    qh, qw = m_fuse.shape
    edges = np.empty((h, w), np.uint8)
    m_i = np.empty((h, w), np.float32)
    _check(lib().ref_extract_depth_contours_prefiltered(_p(blurred), w, h, _p(m_fuse), qw, qh, ctypes.byref(cfg),
                                                        _p(edges), _p(m_i)))
    return edges, m_i


def smoothness_weight(px, py, qx, qy, edges, m_fuse, m_i):
    edges, m_fuse, m_i = _c(edges, np.uint8), _c(m_fuse, np.float32), _c(m_i, np.float32)
    h, w = edges.shape
    qh, qw = m_fuse.shape
    out = ctypes.c_double()
    _check(lib().ref_smoothness_weight(px, py, qx, qy, _p(edges), w, h, _p(m_fuse), qw, qh, _p(m_i), ctypes.byref(out)))
    return out.value


def assemble_system(sparse, edges, m_fuse, m_i, d_pre, cfg):
    """-> dict(diag, coup_h, coup_v, rhs, initial, anchored, constant_term, anchor_count)."""
    sparse, edges = _c(sparse, np.float32), _c(edges, np.uint8)
    m_fuse, m_i = _c(m_fuse, np.float32), _c(m_i, np.float32)
    pre = None if d_pre is None else _c(d_pre, np.float32)
    h, w = sparse.shape
    qh, qw = m_fuse.shape
    s = {k: np.empty((h, w), np.float64) for k in ("diag", "coup_h", "coup_v", "rhs", "initial")}
    s["anchored"] = np.empty((h, w), np.uint8)
    ct, ac = ctypes.c_double(), ctypes.c_uint64()
    _check(lib().ref_assemble_system(_p(sparse), _p(edges), _p(m_fuse), qw, qh, _p(m_i), _p(pre), w, h,
                                     ctypes.byref(cfg), _p(s["diag"]), _p(s["coup_h"]), _p(s["coup_v"]),
                                     _p(s["rhs"]), _p(s["initial"]), _p(s["anchored"]), ctypes.byref(ct),
                                     ctypes.byref(ac)))
    s["constant_term"] = ct.value
    s["anchor_count"] = ac.value
    return s


def apply_system(sys, x):
    h, w = sys["diag"].shape
    x = _c(x, np.float64)
    out = np.empty_like(x)
    _check(lib().ref_apply_system(w, h, _p(sys["diag"]), _p(sys["coup_h"]), _p(sys["coup_v"]), _p(x), _p(out)))
    return out


def solve_dense_depth(sys, cfg, history_cap=None):
    """-> (dense, stats dict)."""
    h, w = sys["diag"].shape
    dense = np.empty((h, w), np.float32)
    it, rr, o0, o1 = ctypes.c_int(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    cap = cfg.solver_max_iter + 1 if history_cap is None else history_cap
    hist = np.zeros(max(cap, 1), np.float64)
    _check(lib().ref_solve_dense_depth(w, h, _p(sys["diag"]), _p(sys["coup_h"]), _p(sys["coup_v"]), _p(sys["rhs"]),
                                       _p(sys["initial"]), _p(sys["anchored"]), sys["constant_term"],
                                       ctypes.byref(cfg), _p(dense), ctypes.byref(it), ctypes.byref(rr),
                                       ctypes.byref(o0), ctypes.byref(o1), _p(hist), cap))
    return dense, {"iterations": it.value, "relative_residual": rr.value, "objective_initial": o0.value,
                   "objective_final": o1.value, "residual_history": hist[: min(cap, it.value + 1)].copy()}


def composite(real, dense, vrgb, vdepth):
    real, dense = _c(real, np.float32), _c(dense, np.float32)
    vrgb, vdepth = _c(vrgb, np.float32), _c(vdepth, np.float32)
    h, w = dense.shape
    out = np.empty((h, w, 3), np.float32)
    mask = np.empty((h, w), np.uint8)
    _check(lib().ref_composite(_p(real), _p(dense), _p(vrgb), _p(vdepth), w, h, _p(out), _p(mask)))
    return out, mask


def render_cube(w, h, focal_px, cx=0.0, cy=0.0, cz=1.5, side=0.3):
    """make_cube_mesh + render_virtual: the composite's virtual layer."""
    vrgb = np.empty((h, w, 3), np.float32)
    vdepth = np.empty((h, w), np.float32)
    _check(lib().ref_render_cube(cx, cy, cz, side, focal_px, w, h, _p(vrgb), _p(vdepth)))
    return vrgb, vdepth


def render_virtual(verts, tris, colors, focal_px, cx, cy, w, h, pose=None):
    """transform_mesh (when pose is given) + render_virtual, occlude.cpp:78-169."""
    verts, tris, colors = _c(verts, np.float32), _c(tris, np.int32), _c(colors, np.float32)
    pose_p = _p(_c(pose, np.float64)) if pose is not None else None
    vrgb = np.empty((h, w, 3), np.float32)
    vdepth = np.empty((h, w), np.float32)
    _check(lib().ref_render_virtual(_p(verts), len(verts), _p(tris), len(tris), _p(colors), pose_p, focal_px, cx, cy,
                                    w, h, _p(vrgb), _p(vdepth)))
    return vrgb, vdepth


def transform_mesh(verts, pose):
    """transform_mesh, occlude.cpp:78-87."""
    verts = _c(verts, np.float32)
    out = np.empty_like(verts)
    _check(lib().ref_transform_mesh(_p(verts), len(verts), _p(_c(pose, np.float64)), _p(out)))
    return out


def pipeline_frame(past_q, mid_q, future_q, mid_gray, right_q, mid_rgb, d_pre, vrgb, vdepth, cfg):
    """One composited frame of run_pipeline (pipeline.cpp:183-258).
    -> dict(dense, composite, mask, edges, sparse, iterations, objective, unsolvable)."""
    fh, fw = mid_gray.shape
    arrs = [_c(a, np.float32) if a is not None else None
            for a in (past_q, mid_q, future_q, mid_gray, right_q, mid_rgb, d_pre, vrgb, vdepth)]
    dense = np.empty((fh, fw), np.float32)
    comp = np.empty((fh, fw, 3), np.float32)
    mask = np.empty((fh, fw), np.uint8)
    edges = np.empty((fh, fw), np.uint8)
    sparse = np.empty((fh, fw), np.float32)
    it, obj = ctypes.c_int(0), ctypes.c_double(0.0)
    st = lib().ref_pipeline_frame(fw, fh, *[_p(a) for a in arrs], ctypes.byref(cfg), _p(dense), _p(comp), _p(mask),
                                  _p(edges), _p(sparse), ctypes.byref(it), ctypes.byref(obj))
    if st not in (0, 3):
        _check(st)
    return {"dense": dense, "composite": comp, "mask": mask, "edges": edges, "sparse": sparse,
            "iterations": it.value, "objective": obj.value, "unsolvable": st == 3}


STAGES = ["adaptive filter area construction", "initial parallax", "parallax optimisation", "sparse map",
          "bidirectional optical flow", "amplitude", "fusion", "box filter", "normalisation", "Gaussian filtering",
          "depth contour extraction", "densification", "rendering", "other"]


def run_pipeline(config_path, manifest, out_dir, mesh_path=None, cap=4096):
    """run_pipeline (pipeline.cpp:108-321), the reference's own frame loop over
    a manifest. -> list of dicts per composited frame: index, iterations,
    stages (the 14 StageTimings values, StageTimings::stage_names order) and
    total (ms, the reference's own steady_clock timers)."""
    ms = np.zeros((cap, 15), np.float64)
    it = np.zeros(cap, np.int32)
    idx = np.zeros(cap, np.int32)
    n = ctypes.c_int(0)
    _check(lib().ref_run_pipeline(config_path.encode() if config_path else None, manifest.encode(), out_dir.encode(),
                                  mesh_path.encode() if mesh_path else None, cap, _p(ms), _p(it), _p(idx),
                                  ctypes.byref(n)))
    return [{"index": int(idx[k]), "iterations": int(it[k]), "stages": ms[k, :14].tolist(), "total": float(ms[k, 14])}
            for k in range(n.value)]


def format_bench_report(repetitions, mmm, csv_path=None):
    """format_bench_report (+ write_bench_csv when csv_path), pipeline.cpp:366-391,
    of 15 (mean, min, max) rows: the 14 stages then the frame total."""
    a = _c(mmm, np.float64)
    buf = ctypes.create_string_buffer(8192)
    _check(lib().ref_format_bench_report(repetitions, _p(a), buf, 8192, csv_path.encode() if csv_path else None))
    return buf.value.decode()


def lr_consistency(disp_left, disp_right, max_diff=1.0):
    """Left-right consistency restated in numpy (the reference has none:
    SPEC.md "Non-goals: no left-right cross-checking"; this is the north_star's
    opt-in filter). Keeps d_L(x, y) where x_r = x - round(d_L) lies in the map
    and |d_L - d_R(x_r, y)| <= max_diff (float64 compare); NaN elsewhere."""
    dl = np.asarray(disp_left, np.float32)
    dr = np.asarray(disp_right, np.float32)
    h, w = dl.shape
    out = np.full((h, w), np.nan, np.float32)
    ys, xs = np.nonzero(np.isfinite(dl))
    d = dl[ys, xs]
    xr = xs - np.floor(d + np.float32(0.5)).astype(np.int64)
    ok = (xr >= 0) & (xr < w)
    ys, xs, d, xr = ys[ok], xs[ok], d[ok], xr[ok]
    e = dr[ys, xr]
    keep = np.isfinite(e) & (np.abs(d.astype(np.float64) - e.astype(np.float64)) <= max_diff)
    out[ys[keep], xs[keep]] = d[keep]
    return out


def stereo_disparity(left_q, right_q, cfg):
    """The reference's stereo chain (stereo.cpp:106-299) on quarter images."""
    arms = build_cross_windows(left_q, cfg)
    vol = compute_cost_volume(left_q, right_q, arms, cfg)
    return refine_disparity_histogram(select_disparity_wta(aggregate_costs(vol, arms, cfg.d_min), cfg.d_min), arms,
                                      cfg.hist_iterations)


def write_pgm(img, path):
    """write_pgm, codec.cpp:211-219."""
    img = _c(img, np.float32)
    _check(lib().ref_write_pgm(_p(img), img.shape[1], img.shape[0], path.encode()))


def write_ppm(rgb, path):
    """write_ppm, codec.cpp:221-229."""
    rgb = _c(rgb, np.float32)
    _check(lib().ref_write_ppm(_p(rgb), rgb.shape[1], rgb.shape[0], path.encode()))


def write_pfm(fmap, path):
    """write_pfm, codec.cpp:293-309."""
    fmap = _c(fmap, np.float32)
    _check(lib().ref_write_pfm(_p(fmap), fmap.shape[1], fmap.shape[0], path.encode()))


def read_pnm(path, color=False):
    """read_pnm, codec.cpp:59-82: the floats (bytes / 255.0f)."""
    w, h = I(), I()
    _check(lib().ref_read_pnm(path.encode(), int(color), None, 0, ctypes.byref(w), ctypes.byref(h)))
    out = np.empty((h.value, w.value, 3) if color else (h.value, w.value), np.float32)
    _check(lib().ref_read_pnm(path.encode(), int(color), _p(out), out.size, ctypes.byref(w), ctypes.byref(h)))
    return out


def to_gray(rgb):
    """to_gray, image.cpp:7-15."""
    rgb = _c(rgb, np.float32)
    out = np.empty(rgb.shape[:2], np.float32)
    _check(lib().ref_to_gray(_p(rgb), rgb.shape[1], rgb.shape[0], _p(out)))
    return out
