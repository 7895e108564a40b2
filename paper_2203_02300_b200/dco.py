"""Host-side mirror of the reference's L2 stage API (namespace dco,
/root/reference/proj/include/dco/*.hpp) over the C-ABI of libdco_gpu.so.

Same function names, argument meaning and error behaviour as the reference;
arrays are torch CUDA tensors (device memory, the caller's stream) instead
of std::vector-owning structs. Each function cites the reference function it
replaces. Every call goes to the sm_100a kernels — there is no CPU path.
"""
import ctypes
from dataclasses import dataclass

import torch

from . import native
from .config import Config, InputError

_ctx_cache = {}


def context(device=None):
    """The per-device dco_ctx, bound to torch's current CUDA stream."""
    lib = native.load()
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the DCO hot path has no CPU fallback")
    dev = torch.cuda.current_device() if device is None else int(device)
    ctx = _ctx_cache.get(dev)
    if ctx is None:
        h = ctypes.c_void_p()
        st = lib.dco_create(dev, ctypes.byref(h))
        if st != 0:
            raise RuntimeError("dco_create failed (%d)" % st)
        ctx = h.value
        _ctx_cache[dev] = ctx
    lib.dco_set_stream(ctx, ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    return ctx


def new_context(torch_stream, device=None):
    """A dedicated dco_ctx bound to `torch_stream` (own scratch pool), for
    running several pipeline streams concurrently on one GPU."""
    lib = native.load()
    dev = torch.cuda.current_device() if device is None else int(device)
    h = ctypes.c_void_p()
    st = lib.dco_create(dev, ctypes.byref(h))
    if st != 0:
        raise RuntimeError("dco_create failed (%d)" % st)
    lib.dco_set_stream(h.value, ctypes.c_void_p(torch_stream.cuda_stream))
    return h.value


def kernel_launches(device=None):
    return native.load().dco_kernel_launches(context(device))


def last_solver(ctx=None):
    """Kernel instance of the context's last dense solve, e.g. "k_pcg_tmem<7>"."""
    return native.load().dco_last_solver(context() if ctx is None else ctx).decode()


def _p(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise InputError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise InputError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _call(fn, *args):
    ctx = context()
    native.check(ctx, fn(ctx, *args))


def _lib():
    return native.load()


def _f32(shape, fill=None):
    if fill is None:
        return torch.empty(shape, dtype=torch.float32, device="cuda")
    return torch.full(shape, fill, dtype=torch.float32, device="cuda")


def _hw(img):
    if img.dim() != 2:
        raise InputError("expected a 2-D raster")
    return img.shape[1], img.shape[0]


# --------------------------------------------------------------- pyramid ---
def downsample_half(img):
    """downsample_half, pyramid.cpp:5-17."""
    w, h = _hw(img)
    out = _f32((h // 2, w // 2))
    _call(_lib().dco_downsample_half, _p(img), w, h, _p(out))
    return out


def ingest_gray8(gray8):
    """read_pnm bytes/255.0f (codec.cpp:80) + downsample_half: (full, quarter)."""
    w, h = _hw(gray8)
    full = _f32((h, w))
    quarter = _f32((h // 2, w // 2))
    _call(_lib().dco_ingest_gray8, _p(gray8), w, h, _p(full), _p(quarter))
    return full, quarter


# ------------------------------------------------------ ingest / egress ---
def quantize_u8(img):
    """quantize (codec.cpp:23-26) on the device: clamp to [0, 1], lround(v * 255)."""
    out = torch.empty(img.shape, dtype=torch.uint8, device="cuda")
    _call(_lib().dco_quantize_u8, _p(img), img.numel(), _p(out))
    return out


def to_gray(rgb):
    """to_gray (image.cpp:7-15): Rec. 601 luma of an (h, w, 3) float image."""
    if rgb.dim() != 3 or rgb.shape[2] != 3:
        raise InputError("to_gray: expected an (h, w, 3) image")
    h, w = rgb.shape[0], rgb.shape[1]
    out = _f32((h, w))
    _call(_lib().dco_to_gray, _p(rgb), w, h, _p(out))
    return out


def _codec(fn, *args):
    err = ctypes.create_string_buffer(512)
    st = fn(*args, err, 512)
    if st != 0:
        from .config import raise_for

        raise_for(st, err.value.decode() or "codec error %d" % st)


def read_pnm(path, color=False):
    """read_pnm (codec.cpp:59-82): the payload bytes as a host numpy array,
    (h, w) or (h, w, 3). dco_ingest_gray8 turns gray bytes into read_gray's floats."""
    import numpy as np

    w, h = ctypes.c_int(), ctypes.c_int()
    _codec(_lib().dco_read_pnm, path.encode(), int(color), None, 0, ctypes.byref(w), ctypes.byref(h))
    shape = (h.value, w.value, 3) if color else (h.value, w.value)
    buf = np.empty(shape, np.uint8)
    _codec(_lib().dco_read_pnm, path.encode(), int(color), buf.ctypes.data, buf.nbytes, ctypes.byref(w),
           ctypes.byref(h))
    return buf


def write_pgm(path, img):
    """write_pgm (codec.cpp:211-219): quantised on the device, 1 byte per pixel over PCIe."""
    b = quantize_u8(img).cpu().numpy()
    _codec(_lib().dco_write_pnm, path.encode(), b.ctypes.data, b.shape[1], b.shape[0], 1)


def write_ppm(path, rgb):
    """write_ppm (codec.cpp:221-229) of an (h, w, 3) float image."""
    b = quantize_u8(rgb).cpu().numpy()
    _codec(_lib().dco_write_pnm, path.encode(), b.ctypes.data, b.shape[1], b.shape[0], 3)


def write_pfm(path, fmap):
    """write_pfm (codec.cpp:293-309)."""
    import numpy as np

    a = np.ascontiguousarray(fmap.cpu().numpy() if hasattr(fmap, "cpu") else fmap, np.float32)
    _codec(_lib().dco_write_pfm, path.encode(), a.ctypes.data, a.shape[1], a.shape[0])


# ---------------------------------------------------------------- stereo ---
@dataclass
class CrossWindowField:
    """stereo.hpp:13-35: four u8 arm planes."""

    left: torch.Tensor
    right: torch.Tensor
    up: torch.Tensor
    down: torch.Tensor

    @property
    def width(self):
        return self.left.shape[1]

    @property
    def height(self):
        return self.left.shape[0]

    def planes(self):
        return [_p(self.left), _p(self.right), _p(self.up), _p(self.down)]


def build_cross_windows(img, cfg: Config):
    """build_cross_windows, stereo.cpp:52-68."""
    w, h = _hw(img)
    arms = torch.empty((4, h, w), dtype=torch.uint8, device="cuda")
    f = CrossWindowField(arms[0], arms[1], arms[2], arms[3])
    _call(_lib().dco_build_cross_windows, _p(img), w, h, ctypes.byref(cfg), *f.planes())
    return f


def census_transform(img, window_w, window_h):
    """census_transform, stereo.cpp:70-96 (u64 stored as int64)."""
    w, h = _hw(img)
    out = torch.empty((h, w), dtype=torch.int64, device="cuda")
    _call(_lib().dco_census_transform, _p(img), w, h, window_w, window_h, _p(out))
    return out


def compute_cost_volume(left, right, windows: CrossWindowField, cfg: Config):
    """compute_cost_volume, stereo.cpp:106-150: float [h][w][nd]."""
    w, h = _hw(left)
    if right.shape != left.shape:
        raise InputError("compute_cost_volume: left/right dimensions differ")
    if (windows.width, windows.height) != (w, h):
        raise InputError("compute_cost_volume: cross windows built on different dimensions")
    out = _f32((h, w, cfg.num_disparities))
    _call(_lib().dco_compute_cost_volume, _p(left), _p(right), w, h, *windows.planes(), ctypes.byref(cfg), _p(out))
    return out


def aggregate_costs(vol, windows: CrossWindowField, d_min=0):
    """aggregate_costs, stereo.cpp:152-218."""
    h, w, nd = vol.shape
    if (windows.width, windows.height) != (w, h):
        raise InputError("aggregate_costs: cross windows built on different dimensions")
    out = torch.empty_like(vol)
    _call(_lib().dco_aggregate_costs, _p(vol), w, h, d_min, d_min + nd - 1, *windows.planes(), _p(out))
    return out


def select_disparity_wta(vol, d_min=0):
    """select_disparity_wta, stereo.cpp:220-238."""
    h, w, nd = vol.shape
    out = _f32((h, w))
    _call(_lib().dco_select_disparity_wta, _p(vol), w, h, d_min, d_min + nd - 1, _p(out))
    return out


def refine_disparity_histogram(disp, windows: CrossWindowField, iterations):
    """refine_disparity_histogram, stereo.cpp:240-299."""
    w, h = _hw(disp)
    if (windows.width, windows.height) != (w, h):
        raise InputError("refine_disparity_histogram: cross windows built on different dimensions")
    out = _f32((h, w))
    _call(_lib().dco_refine_disparity_histogram, _p(disp), w, h, *windows.planes(), iterations, _p(out))
    return out


def disparity_to_sparse_depth(disp, cfg: Config, full_width, full_height):
    """disparity_to_sparse_depth, stereo.cpp:301-315."""
    w, h = _hw(disp)
    out = _f32((full_height, full_width))
    _call(_lib().dco_disparity_to_sparse_depth, _p(disp), w, h, ctypes.byref(cfg), full_width, full_height, _p(out))
    return out


def stereo_sparse_depth(left_q, right_q, cfg: Config, full_width, full_height):
    """The stereo chain of pipeline.cpp:184-195 in one call: (disparity, sparse)."""
    w, h = _hw(left_q)
    disp = _f32((h, w))
    sparse = _f32((full_height, full_width))
    _call(_lib().dco_stereo_sparse_depth, _p(left_q), _p(right_q), w, h, ctypes.byref(cfg),
          full_width, full_height, _p(disp), _p(sparse))
    return disp, sparse


def flip_horizontal(img):
    """Mirror a float map left-right."""
    w, h = _hw(img)
    out = _f32((h, w))
    _call(_lib().dco_flip_horizontal, _p(img), w, h, _p(out))
    return out


def lr_consistency(disp_left, disp_right, max_diff=1.0):
    """Left-right consistency (opt-in; the reference applies none, SPEC.md
    Non-goals): d_L where the right view agrees within max_diff, else NaN."""
    w, h = _hw(disp_left)
    if tuple(disp_right.shape) != (h, w):
        raise InputError("lr_consistency: disparity maps differ in size")
    out = _f32((h, w))
    _call(_lib().dco_lr_consistency, _p(disp_left), _p(disp_right), w, h, float(max_diff), _p(out))
    return out


def stereo_sparse_depth_lr(left_q, right_q, cfg: Config, full_width, full_height, max_diff=1.0):
    """The stereo chain with the opt-in left-right check before the sparse map:
    (checked disparity, sparse, left disparity, right disparity)."""
    d_left, _ = stereo_sparse_depth(left_q, right_q, cfg, full_width, full_height)
    d_mirror, _ = stereo_sparse_depth(flip_horizontal(right_q), flip_horizontal(left_q), cfg, full_width,
                                      full_height)
    d_right = flip_horizontal(d_mirror)
    checked = lr_consistency(d_left, d_right, max_diff)
    return checked, disparity_to_sparse_depth(checked, cfg, full_width, full_height), d_left, d_right


# ------------------------------------------------------------- row bands ---
def band_plan(cfg: Config, full_width, full_height, bands, index):
    """dco_band_plan: the quarter rows band `index` of `bands` owns, computes
    (halo) and exchanges the aggregation column prefix at. Host only."""
    b = native.Band()
    st = native.load().dco_band_plan(ctypes.byref(cfg), full_width, full_height, bands, index, ctypes.byref(b))
    if st != 0:
        from .config import raise_for

        raise_for(st, "dco_band_plan: invalid band request (%dx%d, %d bands, index %d)"
                  % (full_width, full_height, bands, index))
    return b


def band_carry_elems(cfg: Config, full_width):
    """Doubles in one carry buffer: (full_width // 2) * nd."""
    return native.load().dco_band_carry_bytes(ctypes.byref(cfg), full_width) // 8


def stereo_band(left_sub, right_sub, band, cfg: Config, full_width, full_height, carry_in=None):
    """dco_stereo_band: the stereo chain of one row band. left_sub/right_sub are
    the quarter rows [band.sub0, band.sub1). Returns (disparity rows
    [row0, row1), sparse full rows [frow0, frow1), carry_out or None)."""
    qw = full_width // 2
    if tuple(left_sub.shape) != (band.sub1 - band.sub0, qw) or left_sub.shape != right_sub.shape:
        raise InputError("stereo_band: sub-images must be (sub1 - sub0, full_width // 2)")
    if carry_in is not None and (carry_in.dtype != torch.float64 or carry_in.numel() != band_carry_elems(cfg, full_width)):
        raise InputError("stereo_band: carry_in must hold (full_width // 2) * nd doubles")
    disp = _f32((band.row1 - band.row0, qw))
    sparse = _f32((band.frow1 - band.frow0, full_width))
    carry_out = None
    if band.carry_out_row >= 0:
        carry_out = torch.empty(band_carry_elems(cfg, full_width), dtype=torch.float64, device="cuda")
    _call(_lib().dco_stereo_band, _p(left_sub), _p(right_sub), ctypes.byref(band), ctypes.byref(cfg),
          full_width, full_height, _p(carry_in), _p(carry_out), _p(disp), _p(sparse))
    return disp, sparse, carry_out


def stereo_band_begin(left_sub, right_sub, band, cfg: Config, full_width, full_height):
    """dco_stereo_band_begin: cross windows, cost and horizontal pass of a band
    (state stays in this context until stereo_band_end)."""
    qw = full_width // 2
    if tuple(left_sub.shape) != (band.sub1 - band.sub0, qw) or left_sub.shape != right_sub.shape:
        raise InputError("stereo_band: sub-images must be (sub1 - sub0, full_width // 2)")
    _call(_lib().dco_stereo_band_begin, _p(left_sub), _p(right_sub), ctypes.byref(band), ctypes.byref(cfg),
          full_width, full_height)


def stereo_band_vpass(band, cfg: Config, full_width, full_height, d0, d1, carry_in=None):
    """dco_stereo_band_vpass over slices [d0, d1): returns the chunk's carry for
    the band below (or None). Carries are (d1 - d0) x (full_width // 2) doubles."""
    qw = full_width // 2
    if carry_in is not None and (carry_in.dtype != torch.float64 or carry_in.numel() != (d1 - d0) * qw):
        raise InputError("stereo_band_vpass: carry_in must hold (d1 - d0) * (full_width // 2) doubles")
    carry_out = None
    if band.carry_out_row >= 0:
        carry_out = torch.empty(((d1 - d0), qw), dtype=torch.float64, device="cuda")
    _call(_lib().dco_stereo_band_vpass, ctypes.byref(band), ctypes.byref(cfg), full_width, full_height, d0, d1,
          _p(carry_in), _p(carry_out))
    return carry_out


def stereo_band_end(band, cfg: Config, full_width, full_height):
    """dco_stereo_band_end: (disparity rows [row0, row1), sparse full rows [frow0, frow1))."""
    qw = full_width // 2
    disp = _f32((band.row1 - band.row0, qw))
    sparse = _f32((band.frow1 - band.frow0, full_width))
    _call(_lib().dco_stereo_band_end, ctypes.byref(band), ctypes.byref(cfg), full_width, full_height, _p(disp),
          _p(sparse))
    return disp, sparse


# ------------------------------------------------------------------ flow ---
def compute_flow(frm, to, cfg: Config):
    """compute_flow, flow.cpp:185-205: (u, v)."""
    w, h = _hw(frm)
    if to.shape != frm.shape:
        raise InputError("compute_flow: frame dimensions differ")
    u, v = _f32((h, w)), _f32((h, w))
    _call(_lib().dco_compute_flow, _p(frm), _p(to), w, h, ctypes.byref(cfg), _p(u), _p(v))
    return u, v


class KeyframeBuffer:
    """KeyframeBuffer, flow.cpp:10-18: capacity-3 sliding window (host state)."""

    def __init__(self):
        self.frames = []

    def push_frame(self, frame):
        if self.frames and tuple(frame.shape) != tuple(self.frames[0].shape):
            raise InputError("push_frame: frame dimensions differ from buffered frames")
        self.frames.append(frame)
        if len(self.frames) > 3:
            self.frames.pop(0)
        if len(self.frames) < 3:
            return None
        return tuple(self.frames)

    def size(self):
        return len(self.frames)

    def clear(self):
        self.frames = []


# --------------------------------------------------------------- contour ---
def flow_to_polar(u, v, with_theta=True):
    """flow_to_polar, contour.cpp:10-25: (r, theta)."""
    w, h = _hw(u)
    r = _f32((h, w))
    theta = _f32((h, w)) if with_theta else None
    _call(_lib().dco_flow_to_polar, _p(u), _p(v), w, h, _p(r), _p(theta))
    return r, theta


def gradient_amplitude(r):
    """gradient_amplitude, contour.cpp:27-42."""
    w, h = _hw(r)
    out = _f32((h, w))
    _call(_lib().dco_gradient_amplitude, _p(r), w, h, _p(out))
    return out


def fuse_amplitudes(flow_past, flow_future, m_past, m_future, cfg: Config):
    """fuse_amplitudes, contour.cpp:82-106. flows are (u, v) pairs."""
    w, h = _hw(m_past)
    for t in (*flow_past, *flow_future, m_future):
        if tuple(t.shape) != (h, w):
            raise InputError("fuse_amplitudes: input dimensions differ")
    out = _f32((h, w))
    _call(_lib().dco_fuse_amplitudes, _p(flow_past[0]), _p(flow_past[1]), _p(flow_future[0]),
          _p(flow_future[1]), _p(m_past), _p(m_future), w, h, ctypes.byref(cfg), _p(out))
    return out


def box_filter(amp, radius):
    """box_filter, contour.cpp:108-136."""
    w, h = _hw(amp)
    out = _f32((h, w))
    _call(_lib().dco_box_filter, _p(amp), w, h, radius, _p(out))
    return out


def normalize_amplitude(amp):
    """normalize_amplitude, contour.cpp:138-147."""
    w, h = _hw(amp)
    out = _f32((h, w))
    _call(_lib().dco_normalize_amplitude, _p(amp), w, h, _p(out))
    return out


def gaussian_blur(img, sigma):
    """gaussian_blur, contour.cpp:149-175."""
    w, h = _hw(img)
    out = _f32((h, w))
    _call(_lib().dco_gaussian_blur, _p(img), w, h, float(sigma), _p(out))
    return out


def extract_depth_contours_prefiltered(blurred, m_fuse, cfg: Config):
    """extract_depth_contours_prefiltered, contour.cpp:177-279: (edges u8, m_i)."""
    w, h = _hw(blurred)
    qw, qh = _hw(m_fuse)
    edges = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    m_i = _f32((h, w))
    _call(_lib().dco_extract_depth_contours_prefiltered, _p(blurred), w, h, _p(m_fuse), qw, qh,
          ctypes.byref(cfg), _p(edges), _p(m_i))
    return edges, m_i


def extract_depth_contours(gray, m_fuse, cfg: Config):
    """extract_depth_contours, contour.cpp:281-285."""
    w, h = _hw(gray)
    qw, qh = _hw(m_fuse)
    edges = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    m_i = _f32((h, w))
    _call(_lib().dco_extract_depth_contours, _p(gray), w, h, _p(m_fuse), qw, qh, ctypes.byref(cfg),
          _p(edges), _p(m_i))
    return edges, m_i


# --------------------------------------------------------------- densify ---
class ConstraintSystem:
    """ConstraintSystem, densify.hpp:19-33 (device arrays + host scalars)."""

    def __init__(self, w, h):
        f64 = dict(dtype=torch.float64, device="cuda")
        self.width, self.height = w, h
        self.diag = torch.zeros((h, w), **f64)
        self.coup_h = torch.zeros((h, w), **f64)
        self.coup_v = torch.zeros((h, w), **f64)
        self.rhs = torch.zeros((h, w), **f64)
        self.initial = torch.zeros((h, w), **f64)
        self.anchored = torch.zeros((h, w), dtype=torch.uint8, device="cuda")
        self.constant_term = 0.0
        self.anchor_count = 0

    def c_struct(self):
        s = native.System()
        s.width, s.height = self.width, self.height
        s.diag, s.coup_h, s.coup_v = _p(self.diag), _p(self.coup_h), _p(self.coup_v)
        s.rhs, s.initial, s.anchored = _p(self.rhs), _p(self.initial), _p(self.anchored)
        s.constant_term = self.constant_term
        s.anchor_count = self.anchor_count
        return s


def smoothness_weight(px, py, qx, qy, b_dp, m_fuse, m_i):
    """smoothness_weight, densify.cpp:26-35."""
    w, h = _hw(b_dp)
    qw, qh = _hw(m_fuse)
    out = ctypes.c_double()
    _call(_lib().dco_smoothness_weight, px, py, qx, qy, _p(b_dp), w, h, _p(m_fuse), qw, qh, _p(m_i),
          ctypes.byref(out))
    return out.value


def assemble_system(d_sparse, b_dp, m_fuse, m_i, d_pre, cfg: Config):
    """assemble_system, densify.cpp:37-116. d_pre may be None."""
    w, h = _hw(d_sparse)
    if tuple(b_dp.shape) != (h, w) or tuple(m_i.shape) != (h, w):
        raise InputError("assemble_system: full-resolution inputs disagree on dimensions")
    if d_pre is not None and tuple(d_pre.shape) != (h, w):
        raise InputError("assemble_system: previous dense map has different dimensions")
    qw, qh = _hw(m_fuse)
    sys = ConstraintSystem(w, h)
    cs = sys.c_struct()
    _call(_lib().dco_assemble_system, _p(d_sparse), _p(b_dp), _p(m_fuse), qw, qh, _p(m_i), _p(d_pre), w, h,
          ctypes.byref(cfg), ctypes.byref(cs))
    sys.constant_term = cs.constant_term
    sys.anchor_count = cs.anchor_count
    return sys


def apply_system(sys: ConstraintSystem, x):
    """apply_system, densify.cpp:118-133."""
    out = torch.empty_like(x)
    cs = sys.c_struct()
    _call(_lib().dco_apply_system, ctypes.byref(cs), _p(x), _p(out))
    return out


def objective_value(sys: ConstraintSystem, x):
    """objective_value, densify.cpp:135-139."""
    out = ctypes.c_double()
    cs = sys.c_struct()
    _call(_lib().dco_objective_value, ctypes.byref(cs), _p(x), ctypes.byref(out))
    return out.value


@dataclass
class SolveStats:
    """SolveStats, densify.hpp:50-56."""

    iterations: int = 0
    relative_residual: float = 0.0
    objective_initial: float = 0.0
    objective_final: float = 0.0
    residual_history: list = None


def solve_dense_depth(sys: ConstraintSystem, cfg: Config, history_cap=None):
    """solve_dense_depth, densify.cpp:141-222: (dense, SolveStats)."""
    dense = _f32((sys.height, sys.width))
    cap = cfg.solver_max_iter + 1 if history_cap is None else history_cap
    hist = (ctypes.c_double * max(cap, 1))()
    st = native.SolveStats()
    st.history = ctypes.cast(hist, ctypes.POINTER(ctypes.c_double))
    st.history_cap = cap
    cs = sys.c_struct()
    _call(_lib().dco_solve_dense_depth, ctypes.byref(cs), ctypes.byref(cfg), _p(dense), ctypes.byref(st))
    stats = SolveStats(st.iterations, st.relative_residual, st.objective_initial, st.objective_final,
                       list(hist[: min(cap, st.iterations + 1)]))
    return dense, stats


# ------------------------------------------------------- row-band solve ---
def band_system(sys: ConstraintSystem, row0, rows):
    """The dco_system of full rows [row0, row0 + rows) of a whole-frame system
    (coup_v of the row above stays readable through the same allocation)."""
    if not (0 <= row0 and rows >= 1 and row0 + rows <= sys.height):
        raise InputError("band_system: rows outside the system")
    s = native.System()
    s.width, s.height = sys.width, rows
    off = row0 * sys.width
    s.diag = sys.diag.data_ptr() + 8 * off
    s.coup_h = sys.coup_h.data_ptr() + 8 * off
    s.coup_v = sys.coup_v.data_ptr() + 8 * off
    s.rhs = sys.rhs.data_ptr() + 8 * off
    s.initial = sys.initial.data_ptr() + 8 * off
    s.anchored = sys.anchored.data_ptr() + off
    s.constant_term = sys.constant_term
    s.anchor_count = sys.anchor_count
    return s


def _stats_of(st, hist, cap):
    return SolveStats(st.iterations, st.relative_residual, st.objective_initial, st.objective_final,
                      list(hist[: min(cap, st.iterations + 1)]) if hist is not None else [])


class BandSolver:
    """One rank's share of a row-band densify solve (dco_band_solver)."""

    def __init__(self, ranks, rank, width, row0, rows, full_height):
        self.ranks, self.rank, self.width, self.row0, self.rows = ranks, rank, width, row0, rows
        self.handle = ctypes.c_void_p()
        _call(_lib().dco_band_solver_create, ranks, rank, width, row0, rows, full_height, ctypes.byref(self.handle))

    def export(self):
        buf = ctypes.create_string_buffer(native.BAND_HANDLE_BYTES)
        native.check(context(), _lib().dco_band_solver_export(self.handle, buf))
        return buf.raw

    def connect(self, handles):
        """handles: every rank's export(), rank order (CUDA IPC: one process per GPU)."""
        blob = b"".join(handles)
        if len(handles) != self.ranks or len(blob) != self.ranks * native.BAND_HANDLE_BYTES:
            raise InputError("BandSolver.connect: one handle per rank")
        native.check(context(), _lib().dco_band_solver_connect(self.handle, blob))

    def solve(self, band_sys, cfg: Config, anchors_total, constant_total, history_cap=None):
        dense = _f32((self.rows, self.width))
        cap = cfg.solver_max_iter + 1 if history_cap is None else history_cap
        hist = (ctypes.c_double * max(cap, 1))()
        st = native.SolveStats()
        st.history = ctypes.cast(hist, ctypes.POINTER(ctypes.c_double))
        st.history_cap = cap
        native.check(context(), _lib().dco_band_solve(self.handle, ctypes.byref(band_sys), ctypes.byref(cfg),
                                                      anchors_total, constant_total, _p(dense), ctypes.byref(st)))
        return dense, _stats_of(st, hist, cap)

    def close(self):
        if self.handle:
            _lib().dco_band_solver_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_streams(streams, left8, right8, want_results=False):
    """dco_run_streams: left8[k] / right8[k] are (frames, h, w) u8 CUDA tensors
    for stream k; all streams advance frame by frame. Returns the per-frame
    results [k][f] when asked (synchronising), else None."""
    n = len(streams)
    if n == 0 or len(left8) != n or len(right8) != n:
        raise InputError("run_streams: one left and one right batch per stream")
    frames = left8[0].shape[0]
    for k, st in enumerate(streams):
        if tuple(left8[k].shape) != (frames, st.full_h, st.full_w) or left8[k].shape != right8[k].shape:
            raise InputError("run_streams: batch k must be (frames, h, w) u8 for stream k")
        if left8[k].dtype != torch.uint8 or right8[k].dtype != torch.uint8:
            raise InputError("run_streams: u8 frames expected")
    for st in streams:
        st._bind()
    hs = (ctypes.c_void_p * n)(*[st.handle for st in streams])
    ls = (ctypes.c_void_p * n)(*[_p(t).value for t in left8])
    rs = (ctypes.c_void_p * n)(*[_p(t).value for t in right8])
    res = (native.FrameResult * (n * frames))() if want_results else None
    st = _lib().dco_run_streams(hs, n, ls, rs, frames, res)
    if st != 0:
        native.check(streams[0].ctx, st)
    if not want_results:
        return None
    return [[res[k * frames + f] for f in range(frames)] for k in range(n)]


def band_connect_local(solvers):
    """All ranks in this process, on this GPU (the emulation of a multi-GPU
    band solve with fewer GPUs than ranks)."""
    arr = (ctypes.c_void_p * len(solvers))(*[s.handle.value for s in solvers])
    native.check(context(), _lib().dco_band_solver_connect_local(arr, len(solvers)))


def band_solve_local(solvers, band_systems, cfg: Config, anchors_total, constant_total, history_cap=None):
    """One cooperative launch running every rank as a block group: (dense
    per band, stats per band)."""
    g = len(solvers)
    dense = [_f32((s.rows, s.width)) for s in solvers]
    cap = cfg.solver_max_iter + 1 if history_cap is None else history_cap
    hist = (ctypes.c_double * max(cap, 1))()
    sts = (native.SolveStats * g)()
    sts[0].history = ctypes.cast(hist, ctypes.POINTER(ctypes.c_double))
    sts[0].history_cap = cap
    arr = (ctypes.c_void_p * g)(*[s.handle.value for s in solvers])
    sys_arr = (native.System * g)(*band_systems)
    out = (ctypes.c_void_p * g)(*[_p(d) for d in dense])
    native.check(context(), _lib().dco_band_solve_local(arr, g, sys_arr, ctypes.byref(cfg), anchors_total,
                                                        constant_total, out, sts))
    return dense, [_stats_of(sts[k], hist if k == 0 else None, cap) for k in range(g)]


# ------------------------------------------------------------- composite ---
def composite(real_rgb, dense, virt_rgb, virt_depth):
    """composite, occlude.cpp:171-194: (color, mask)."""
    h, w = dense.shape
    if tuple(real_rgb.shape) != (h, w, 3) or tuple(virt_rgb.shape) != (h, w, 3) or tuple(virt_depth.shape) != (h, w):
        raise InputError("composite: input dimensions differ")
    out = _f32((h, w, 3))
    mask = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    _call(_lib().dco_composite, _p(real_rgb), _p(dense), _p(virt_rgb), _p(virt_depth), w, h, _p(out), _p(mask))
    return out, mask


# --------------------------------------------------------- virtual layer ---
def transform_mesh(vertices, pose):
    """transform_mesh, occlude.cpp:78-87: vertices (n, 3) float CUDA tensor,
    pose 16 row-major doubles (host sequence)."""
    n = vertices.shape[0]
    out = torch.empty_like(vertices)
    pose_h = (ctypes.c_double * 16)(*[float(v) for v in pose])
    _call(_lib().dco_transform_mesh, _p(vertices), n, ctypes.cast(pose_h, ctypes.c_void_p), _p(out))
    return out


def render_virtual(vertices, triangles, colors, focal_px, cx, cy, width, height):
    """render_virtual, occlude.cpp:107-169: (rgb (h, w, 3), depth (h, w))."""
    rgb = _f32((height, width, 3))
    depth = _f32((height, width))
    _call(_lib().dco_render_virtual, _p(vertices), _p(triangles), _p(colors), triangles.shape[0], float(focal_px),
          float(cx), float(cy), width, height, _p(rgb), _p(depth))
    return rgb, depth


# ---------------------------------------------------------------- stream ---
class Stream:
    """One device-resident pipeline stream (pipeline.cpp:131-258 per frame)."""

    def __init__(self, full_w, full_h, cfg: Config, ctx=None):
        self.lib = native.load()
        self.own_ctx = ctx is not None
        self.ctx = ctx if ctx is not None else context()
        h = ctypes.c_void_p()
        native.check(self.ctx, self.lib.dco_stream_create(self.ctx, full_w, full_h, ctypes.byref(cfg), ctypes.byref(h)))
        self.handle = h.value
        self.full_w, self.full_h = full_w, full_h

    def close(self):
        if self.handle:
            self.lib.dco_stream_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _bind(self):
        if not self.own_ctx:
            context()

    def launches(self):
        return self.lib.dco_kernel_launches(self.ctx)

    def last_solver(self):
        return last_solver(self.ctx)

    def set_virtual(self, virt_rgb, virt_depth):
        self._bind()
        native.check(self.ctx, self.lib.dco_stream_set_virtual(self.handle, _p(virt_rgb), _p(virt_depth)))

    def set_mesh(self, vertices, triangles, colors):
        """Virtual mesh rendered per frame (numpy arrays: (n, 3) float32
        vertices / colours, (m, 3) int32 triangles); None clears it."""
        self._bind()
        if vertices is None:
            native.check(self.ctx, self.lib.dco_stream_set_mesh(self.handle, None, 0, None, 0, None))
            return
        import numpy as np

        v = np.ascontiguousarray(vertices, np.float32)
        t = np.ascontiguousarray(triangles, np.int32)
        c = np.ascontiguousarray(colors, np.float32)
        self._mesh_keep = (v, t, c)
        native.check(self.ctx, self.lib.dco_stream_set_mesh(
            self.handle, ctypes.c_void_p(v.ctypes.data), len(v), ctypes.c_void_p(t.ctypes.data), len(t),
            ctypes.c_void_p(c.ctypes.data)))

    def set_next_pose(self, pose):
        """Pose (16 doubles, row-major) of the next pushed frame; None = none."""
        if pose is None:
            native.check(self.ctx, self.lib.dco_stream_set_next_pose(self.handle, None))
            return
        p = (ctypes.c_double * 16)(*[float(x) for x in pose])
        native.check(self.ctx, self.lib.dco_stream_set_next_pose(self.handle, ctypes.cast(p, ctypes.c_void_p)))

    def push_gray8(self, left8, right8, rgb8=None, want_result=True):
        self._bind()
        res = native.FrameResult()
        native.check(self.ctx, self.lib.dco_stream_push_gray8(
            self.handle, _p(left8), _p(right8), _p(rgb8), ctypes.byref(res) if want_result else None))
        return res if want_result else None

    def push_f32(self, left, right, rgb=None, want_result=True):
        self._bind()
        res = native.FrameResult()
        native.check(self.ctx, self.lib.dco_stream_push_f32(
            self.handle, _p(left), _p(right), _p(rgb), ctypes.byref(res) if want_result else None))
        return res if want_result else None

    def push_gray8_host(self, left8, right8, comp_out=None, mask_out=None, dense_out=None):
        """Host numpy/pinned buffers in and out (end-to-end path)."""
        self._bind()
        res = native.FrameResult()

        def hp(a):
            return None if a is None else ctypes.c_void_p(a.ctypes.data if hasattr(a, "ctypes") else a.data_ptr())

        native.check(self.ctx, self.lib.dco_stream_push_gray8_host(
            self.handle, hp(left8), hp(right8), hp(comp_out), hp(mask_out), hp(dense_out), ctypes.byref(res)))
        return res

    def push_gray8_host_encoded(self, left8, right8, comp_rgb8=None, mask8=None, dense_out=None):
        """Host buffers in and out, the outputs encoded as run_pipeline writes
        them (pipeline.cpp:266-268): composite RGB bytes (write_ppm's quantize),
        mask bytes 0/255 (write_mask_pgm), dense floats."""
        self._bind()
        res = native.FrameResult()

        def hp(a):
            return None if a is None else ctypes.c_void_p(a.ctypes.data if hasattr(a, "ctypes") else a.data_ptr())

        native.check(self.ctx, self.lib.dco_stream_push_gray8_host_encoded(
            self.handle, hp(left8), hp(right8), hp(comp_rgb8), hp(mask8), hp(dense_out), ctypes.byref(res)))
        return res

    SPANS = ["ingest", "cross", "cost", "aggregate", "wta", "refine", "sparse", "flow", "fusion", "box",
             "normalize", "blur", "contour", "assemble", "solve", "composite"]

    def set_lr_check(self, enable=True, max_diff=1.0):
        """Opt-in left-right consistency before the sparse map (not in the
        reference; default off)."""
        native.check(self.ctx, _lib().dco_stream_set_lr_check(self.handle, int(enable), float(max_diff)))

    def set_timing(self, enable=True):
        native.check(self.ctx, self.lib.dco_stream_set_timing(self.handle, 1 if enable else 0))

    def span_times(self):
        """-> (dict span -> total ms over timed frames, frame count)."""
        ms = (ctypes.c_double * len(self.SPANS))()
        n = ctypes.c_uint64()
        native.check(self.ctx, self.lib.dco_stream_span_times(self.handle, ms, ctypes.byref(n)))
        return dict(zip(self.SPANS, list(ms))), n.value

    def views(self):
        v = native.FrameViews()
        native.check(self.ctx, self.lib.dco_stream_views(self.handle, ctypes.byref(v)))
        return v

    def state(self):
        n = self.lib.dco_stream_state_size(self.handle)
        buf = (ctypes.c_char * n)()
        native.check(self.ctx, self.lib.dco_stream_save_state(self.handle, buf, n))
        return bytes(buf)

    def load_state(self, blob):
        buf = (ctypes.c_char * len(blob)).from_buffer_copy(blob)
        native.check(self.ctx, self.lib.dco_stream_load_state(self.handle, buf, len(blob)))


class _CudaArray:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


_TYPESTR = {torch.float32: "<f4", torch.float64: "<f8", torch.uint8: "|u1", torch.int32: "<i4"}


def view_tensor(ptr, shape, dtype):
    """Zero-copy torch view of device memory owned by a Stream (valid until the
    next push overwrites it)."""
    return torch.as_tensor(_CudaArray(ptr, shape, _TYPESTR[dtype]), device="cuda")
