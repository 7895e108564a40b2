"""numpy front-end of oracle/_lib/libdco_oracle.so, the plain-C restatement
of the reference hot path (oracle/dco_oracle.c). TEST INFRASTRUCTURE ONLY.
Same function names and array conventions as oracle/ref.py so tests can run
both checkers through one interface."""
import ctypes
import os

import numpy as np

from . import PORT_LIB
from paper_2203_02300_b200.config import Config, raise_for

_lib = None
P, I, D, U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
CFG = ctypes.POINTER(Config)


def available():
    return os.path.exists(PORT_LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            from . import build

            build()
        L = ctypes.CDLL(PORT_LIB)
        sig = {
            "dco_o_error": (ctypes.c_char_p, []),
            "dco_o_validate": (I, [CFG]),
            "dco_o_downsample_half": (I, [P, I, I, P]),
            "dco_o_cross_windows": (I, [P, I, I, CFG, P, P, P, P]),
            "dco_o_census": (I, [P, I, I, I, I, P]),
            "dco_o_cost_volume": (I, [P, P, I, I, P, P, P, P, CFG, P]),
            "dco_o_aggregate": (I, [P, I, I, I, P, P, P, P, P]),
            "dco_o_wta": (I, [P, I, I, I, I, P]),
            "dco_o_refine": (I, [P, I, I, P, P, P, P, I, P]),
            "dco_o_sparse_depth": (I, [P, I, I, CFG, I, I, P]),
            "dco_o_flow": (I, [P, P, I, I, P, P]),
            "dco_o_polar": (I, [P, P, I, P, P]),
            "dco_o_gradient_amplitude": (I, [P, I, I, P]),
            "dco_o_fuse": (I, [P, P, P, P, P, P, I, I, D, P]),
            "dco_o_box": (I, [P, I, I, I, P]),
            "dco_o_normalize": (I, [P, I, P]),
            "dco_o_gauss": (I, [P, I, I, D, P]),
            "dco_o_contours": (I, [P, I, I, P, I, I, CFG, P, P]),
            "dco_o_assemble": (I, [P, P, P, I, I, P, P, I, I, CFG, P, P, P, P, P, P, ctypes.POINTER(D),
                                   ctypes.POINTER(U64)]),
            "dco_o_apply": (I, [I, I, P, P, P, P, P]),
            "dco_o_solve": (I, [I, I, P, P, P, P, P, U64, D, CFG, P, ctypes.POINTER(I), ctypes.POINTER(D),
                                ctypes.POINTER(D), ctypes.POINTER(D)]),
            "dco_o_composite": (I, [P, P, P, P, I, I, P, P]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _check(st):
    if st:
        raise_for(st, lib().dco_o_error().decode())


def validate(cfg):
    _check(lib().dco_o_validate(ctypes.byref(cfg)))


def downsample_half(img):
    img = _c(img, np.float32)
    h, w = img.shape
    out = np.empty((h // 2, w // 2), np.float32)
    _check(lib().dco_o_downsample_half(_p(img), w, h, _p(out)))
    return out


def build_cross_windows(img, cfg):
    img = _c(img, np.float32)
    h, w = img.shape
    arms = np.empty((4, h, w), np.uint8)
    _check(lib().dco_o_cross_windows(_p(img), w, h, ctypes.byref(cfg), *[_p(arms[i]) for i in range(4)]))
    return arms


def census_transform(img, ww, wh):
    img = _c(img, np.float32)
    h, w = img.shape
    out = np.empty((h, w), np.uint64)
    _check(lib().dco_o_census(_p(img), w, h, ww, wh, _p(out)))
    return out


def compute_cost_volume(left, right, arms, cfg):
    left, right, arms = _c(left, np.float32), _c(right, np.float32), _c(arms, np.uint8)
    h, w = left.shape
    out = np.empty((h, w, cfg.d_max - cfg.d_min + 1), np.float32)
    _check(lib().dco_o_cost_volume(_p(left), _p(right), w, h, *[_p(arms[i]) for i in range(4)], ctypes.byref(cfg),
                                   _p(out)))
    return out


def aggregate_costs(vol, arms, d_min=0):
    vol, arms = _c(vol, np.float32), _c(arms, np.uint8)
    h, w, nd = vol.shape
    out = np.empty_like(vol)
    _check(lib().dco_o_aggregate(_p(vol), w, h, nd, *[_p(arms[i]) for i in range(4)], _p(out)))
    return out


def select_disparity_wta(vol, d_min=0):
    vol = _c(vol, np.float32)
    h, w, nd = vol.shape
    out = np.empty((h, w), np.float32)
    _check(lib().dco_o_wta(_p(vol), w, h, d_min, nd, _p(out)))
    return out


def refine_disparity_histogram(disp, arms, iterations):
    disp, arms = _c(disp, np.float32), _c(arms, np.uint8)
    h, w = disp.shape
    out = np.empty_like(disp)
    _check(lib().dco_o_refine(_p(disp), w, h, *[_p(arms[i]) for i in range(4)], iterations, _p(out)))
    return out


def disparity_to_sparse_depth(disp, cfg, fw, fh):
    disp = _c(disp, np.float32)
    h, w = disp.shape
    out = np.empty((fh, fw), np.float32)
    _check(lib().dco_o_sparse_depth(_p(disp), w, h, ctypes.byref(cfg), fw, fh, _p(out)))
    return out


def compute_flow(frm, to, cfg=None):
    frm, to = _c(frm, np.float32), _c(to, np.float32)
    h, w = frm.shape
    u, v = np.empty((h, w), np.float32), np.empty((h, w), np.float32)
    _check(lib().dco_o_flow(_p(frm), _p(to), w, h, _p(u), _p(v)))
    return u, v


def flow_to_polar(u, v):
    u, v = _c(u, np.float32), _c(v, np.float32)
    r, t = np.empty_like(u), np.empty_like(u)
    _check(lib().dco_o_polar(_p(u), _p(v), u.size, _p(r), _p(t)))
    return r, t


def gradient_amplitude(r):
    r = _c(r, np.float32)
    h, w = r.shape
    out = np.empty_like(r)
    _check(lib().dco_o_gradient_amplitude(_p(r), w, h, _p(out)))
    return out


def fuse_amplitudes(past, future, mp, mf, cfg):
    arrs = [_c(a, np.float32) for a in (past[0], past[1], future[0], future[1], mp, mf)]
    h, w = arrs[4].shape
    out = np.empty((h, w), np.float32)
    _check(lib().dco_o_fuse(*[_p(a) for a in arrs], w, h, cfg.confidence_offset_k, _p(out)))
    return out


def box_filter(a, radius):
    a = _c(a, np.float32)
    h, w = a.shape
    out = np.empty_like(a)
    _check(lib().dco_o_box(_p(a), w, h, radius, _p(out)))
    return out


def normalize_amplitude(a):
    a = _c(a, np.float32)
    out = np.empty_like(a)
    _check(lib().dco_o_normalize(_p(a), a.size, _p(out)))
    return out


def gaussian_blur(img, sigma):
    img = _c(img, np.float32)
    h, w = img.shape
    out = np.empty_like(img)
    _check(lib().dco_o_gauss(_p(img), w, h, sigma, _p(out)))
    return out


def extract_depth_contours_prefiltered(blurred, m_fuse, cfg):
    blurred, m_fuse = _c(blurred, np.float32), _c(m_fuse, np.float32)
    h, w = blurred.shape
    qh, qw = m_fuse.shape
    edges, m_i = np.empty((h, w), np.uint8), np.empty((h, w), np.float32)
    _check(lib().dco_o_contours(_p(blurred), w, h, _p(m_fuse), qw, qh, ctypes.byref(cfg), _p(edges), _p(m_i)))
    return edges, m_i


def assemble_system(sparse, edges, m_fuse, m_i, d_pre, cfg):
    sparse, edges, m_fuse, m_i = _c(sparse, np.float32), _c(edges, np.uint8), _c(m_fuse, np.float32), _c(m_i, np.float32)
    pre = None if d_pre is None else _c(d_pre, np.float32)
    h, w = sparse.shape
    qh, qw = m_fuse.shape
    s = {k: np.empty((h, w), np.float64) for k in ("diag", "coup_h", "coup_v", "rhs", "initial")}
    s["anchored"] = np.empty((h, w), np.uint8)
    ct, ac = ctypes.c_double(), ctypes.c_uint64()
    _check(lib().dco_o_assemble(_p(sparse), _p(edges), _p(m_fuse), qw, qh, _p(m_i), _p(pre), w, h, ctypes.byref(cfg),
                                _p(s["diag"]), _p(s["coup_h"]), _p(s["coup_v"]), _p(s["rhs"]), _p(s["initial"]),
                                _p(s["anchored"]), ctypes.byref(ct), ctypes.byref(ac)))
    s["constant_term"], s["anchor_count"] = ct.value, ac.value
    return s


def apply_system(sys, x):
    h, w = sys["diag"].shape
    x = _c(x, np.float64)
    out = np.empty_like(x)
    _check(lib().dco_o_apply(w, h, _p(sys["diag"]), _p(sys["coup_h"]), _p(sys["coup_v"]), _p(x), _p(out)))
    return out


def solve_dense_depth(sys, cfg):
    h, w = sys["diag"].shape
    dense = np.empty((h, w), np.float32)
    it, rr, o0, o1 = ctypes.c_int(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _check(lib().dco_o_solve(w, h, _p(sys["diag"]), _p(sys["coup_h"]), _p(sys["coup_v"]), _p(sys["rhs"]),
                             _p(sys["initial"]), sys["anchor_count"], sys["constant_term"], ctypes.byref(cfg),
                             _p(dense), ctypes.byref(it), ctypes.byref(rr), ctypes.byref(o0), ctypes.byref(o1)))
    return dense, {"iterations": it.value, "relative_residual": rr.value, "objective_initial": o0.value,
                   "objective_final": o1.value}


def composite(real, dense, vrgb, vdepth):
    real, dense, vrgb, vdepth = (_c(a, np.float32) for a in (real, dense, vrgb, vdepth))
    h, w = dense.shape
    out, mask = np.empty((h, w, 3), np.float32), np.empty((h, w), np.uint8)
    _check(lib().dco_o_composite(_p(real), _p(dense), _p(vrgb), _p(vdepth), w, h, _p(out), _p(mask)))
    return out, mask
