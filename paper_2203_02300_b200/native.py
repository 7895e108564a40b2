"""ctypes binding of libdco_gpu.so (include/dco_gpu.h).

The library is built in-tree by paper_2203_02300_b200/build.py. There is no
CPU fallback: if the shared object is missing or no CUDA device is present,
load() raises instead of degrading."""
import ctypes
import os

from .config import Config, raise_for

BAND_HANDLE_BYTES = 128  # DCO_BAND_HANDLE_BYTES
HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdco_gpu.so")

c_int, c_double, c_size_t, c_uint64 = ctypes.c_int, ctypes.c_double, ctypes.c_size_t, ctypes.c_uint64
c_void_p, c_char_p = ctypes.c_void_p, ctypes.c_char_p
P = ctypes.c_void_p  # device pointers travel as void*


class System(ctypes.Structure):
    """dco_system: device-resident ConstraintSystem (densify.hpp:19-33)."""

    _fields_ = [
        ("width", c_int),
        ("height", c_int),
        ("diag", P),
        ("coup_h", P),
        ("coup_v", P),
        ("rhs", P),
        ("initial", P),
        ("anchored", P),
        ("constant_term", c_double),
        ("anchor_count", c_uint64),
    ]


class SolveStats(ctypes.Structure):
    """dco_solve_stats (densify.hpp:50-56)."""

    _fields_ = [
        ("iterations", c_int),
        ("relative_residual", c_double),
        ("objective_initial", c_double),
        ("objective_final", c_double),
        ("history", ctypes.POINTER(c_double)),
        ("history_cap", c_int),
    ]


class FrameResult(ctypes.Structure):
    _fields_ = [
        ("composited", c_int),
        ("densify_skipped", c_int),
        ("densify_iterations", c_int),
        ("densify_objective", c_double),
        ("relative_residual", c_double),
    ]


class FrameViews(ctypes.Structure):
    _fields_ = [
        ("full_w", c_int),
        ("full_h", c_int),
        ("quarter_w", c_int),
        ("quarter_h", c_int),
        ("disparity", P),
        ("sparse", P),
        ("m_fuse", P),
        ("m_i", P),
        ("edges", P),
        ("dense", P),
        ("composite", P),
        ("mask", P),
        ("flow_past_u", P),
        ("flow_past_v", P),
        ("flow_future_u", P),
        ("flow_future_v", P),
        ("cost_volume", P),
        ("aggregated", P),
        ("volume_layout", c_int),
        ("num_disparities", c_int),
    ]


class Band(ctypes.Structure):
    """dco_band: one row band of a frame split over GPUs."""

    _fields_ = [(n, c_int) for n in ("row0", "row1", "sub0", "sub1", "carry_row", "carry_out_row",
                                     "frow0", "frow1", "halo")]


CFG = ctypes.POINTER(Config)

# name -> (restype, argtypes); every function of include/dco_gpu.h
SIGNATURES = {
    "dco_abi_version": (c_int, []),
    "dco_create": (c_int, [c_int, ctypes.POINTER(c_void_p)]),
    "dco_destroy": (None, [c_void_p]),
    "dco_last_error": (c_char_p, [c_void_p]),
    "dco_set_stream": (c_int, [c_void_p, c_void_p]),
    "dco_synchronize": (c_int, [c_void_p]),
    "dco_kernel_launches": (c_uint64, [c_void_p]),
    "dco_last_solver": (c_char_p, [c_void_p]),
    "dco_config_default": (None, [CFG]),
    "dco_config_validate": (c_int, [CFG, c_char_p, c_size_t]),
    "dco_downsample_half": (c_int, [c_void_p, P, c_int, c_int, P]),
    "dco_ingest_gray8": (c_int, [c_void_p, P, c_int, c_int, P, P]),
    "dco_build_cross_windows": (c_int, [c_void_p, P, c_int, c_int, CFG, P, P, P, P]),
    "dco_census_transform": (c_int, [c_void_p, P, c_int, c_int, c_int, c_int, P]),
    "dco_compute_cost_volume": (c_int, [c_void_p, P, P, c_int, c_int, P, P, P, P, CFG, P]),
    "dco_aggregate_costs": (c_int, [c_void_p, P, c_int, c_int, c_int, c_int, P, P, P, P, P]),
    "dco_select_disparity_wta": (c_int, [c_void_p, P, c_int, c_int, c_int, c_int, P]),
    "dco_refine_disparity_histogram": (c_int, [c_void_p, P, c_int, c_int, P, P, P, P, c_int, P]),
    "dco_disparity_to_sparse_depth": (c_int, [c_void_p, P, c_int, c_int, CFG, c_int, c_int, P]),
    "dco_stereo_sparse_depth": (c_int, [c_void_p, P, P, c_int, c_int, CFG, c_int, c_int, P, P]),
    "dco_flip_horizontal": (c_int, [c_void_p, P, c_int, c_int, P]),
    "dco_lr_consistency": (c_int, [c_void_p, P, P, c_int, c_int, c_double, P]),
    "dco_compute_flow": (c_int, [c_void_p, P, P, c_int, c_int, CFG, P, P]),
    "dco_flow_to_polar": (c_int, [c_void_p, P, P, c_int, c_int, P, P]),
    "dco_gradient_amplitude": (c_int, [c_void_p, P, c_int, c_int, P]),
    "dco_fuse_amplitudes": (c_int, [c_void_p, P, P, P, P, P, P, c_int, c_int, CFG, P]),
    "dco_box_filter": (c_int, [c_void_p, P, c_int, c_int, c_int, P]),
    "dco_normalize_amplitude": (c_int, [c_void_p, P, c_int, c_int, P]),
    "dco_gaussian_blur": (c_int, [c_void_p, P, c_int, c_int, c_double, P]),
    "dco_extract_depth_contours_prefiltered": (
        c_int,
        [c_void_p, P, c_int, c_int, P, c_int, c_int, CFG, P, P],
    ),
    "dco_extract_depth_contours": (c_int, [c_void_p, P, c_int, c_int, P, c_int, c_int, CFG, P, P]),
    "dco_smoothness_weight": (
        c_int,
        [c_void_p, c_int, c_int, c_int, c_int, P, c_int, c_int, P, c_int, c_int, P, ctypes.POINTER(c_double)],
    ),
    "dco_assemble_system": (
        c_int,
        [c_void_p, P, P, P, c_int, c_int, P, P, c_int, c_int, CFG, ctypes.POINTER(System)],
    ),
    "dco_apply_system": (c_int, [c_void_p, ctypes.POINTER(System), P, P]),
    "dco_objective_value": (c_int, [c_void_p, ctypes.POINTER(System), P, ctypes.POINTER(c_double)]),
    "dco_solve_dense_depth": (c_int, [c_void_p, ctypes.POINTER(System), CFG, P, ctypes.POINTER(SolveStats)]),
    "dco_composite": (c_int, [c_void_p, P, P, P, P, c_int, c_int, P, P]),
    "dco_transform_mesh": (c_int, [c_void_p, P, c_int, P, P]),
    "dco_render_virtual": (c_int, [c_void_p, P, P, P, c_int, c_double, c_double, c_double, c_int, c_int, P, P]),
    "dco_quantize_u8": (c_int, [c_void_p, P, c_size_t, P]),
    "dco_to_gray": (c_int, [c_void_p, P, c_int, c_int, P]),
    "dco_read_pnm": (c_int, [c_char_p, c_int, c_void_p, c_size_t, ctypes.POINTER(c_int), ctypes.POINTER(c_int),
                             c_char_p, c_size_t]),
    "dco_write_pnm": (c_int, [c_char_p, c_void_p, c_int, c_int, c_int, c_char_p, c_size_t]),
    "dco_write_pfm": (c_int, [c_char_p, c_void_p, c_int, c_int, c_char_p, c_size_t]),
    "dco_band_plan": (c_int, [CFG, c_int, c_int, c_int, c_int, ctypes.POINTER(Band)]),
    "dco_band_carry_bytes": (c_size_t, [CFG, c_int]),
    "dco_stereo_band": (c_int, [c_void_p, P, P, ctypes.POINTER(Band), CFG, c_int, c_int, P, P, P, P]),
    "dco_band_sparse_stats": (c_int, [c_void_p, P, c_size_t, ctypes.POINTER(c_double)]),
    "dco_band_sparse_mean": (c_int, [ctypes.POINTER(c_double), c_int, ctypes.POINTER(c_double), ctypes.POINTER(c_int)]),
    "dco_sparse_mean": (c_int, [c_void_p, P, c_size_t, ctypes.POINTER(c_double)]),
    "dco_band_assemble": (
        c_int,
        [c_void_p, P, P, P, c_int, c_int, P, P, c_int, c_int, c_int, c_int, CFG, c_double, ctypes.POINTER(System),
         ctypes.POINTER(c_uint64), ctypes.POINTER(c_double)],
    ),
    "dco_stereo_band_begin": (c_int, [c_void_p, P, P, ctypes.POINTER(Band), CFG, c_int, c_int]),
    "dco_stereo_band_vpass": (c_int, [c_void_p, ctypes.POINTER(Band), CFG, c_int, c_int, c_int, c_int, P, P]),
    "dco_stereo_band_end": (c_int, [c_void_p, ctypes.POINTER(Band), CFG, c_int, c_int, P, P]),
    "dco_band_solver_create": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(c_void_p)]),
    "dco_band_solver_destroy": (None, [c_void_p]),
    "dco_band_solver_export": (c_int, [c_void_p, c_void_p]),
    "dco_band_solver_connect": (c_int, [c_void_p, c_void_p]),
    "dco_band_solver_connect_local": (c_int, [ctypes.POINTER(c_void_p), c_int]),
    "dco_band_solve": (c_int, [c_void_p, ctypes.POINTER(System), CFG, c_uint64, c_double, P, ctypes.POINTER(SolveStats)]),
    "dco_band_solve_local": (
        c_int,
        [ctypes.POINTER(c_void_p), c_int, ctypes.POINTER(System), CFG, c_uint64, c_double, ctypes.POINTER(c_void_p),
         ctypes.POINTER(SolveStats)],
    ),
    "dco_stream_create": (c_int, [c_void_p, c_int, c_int, CFG, ctypes.POINTER(c_void_p)]),
    "dco_stream_destroy": (None, [c_void_p]),
    "dco_stream_set_virtual": (c_int, [c_void_p, P, P]),
    "dco_stream_set_mesh": (c_int, [c_void_p, P, c_int, P, c_int, P]),
    "dco_stream_set_next_pose": (c_int, [c_void_p, P]),
    "dco_stream_push_gray8": (c_int, [c_void_p, P, P, P, ctypes.POINTER(FrameResult)]),
    "dco_run_streams": (
        c_int,
        [ctypes.POINTER(c_void_p), c_int, ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p), c_int,
         ctypes.POINTER(FrameResult)],
    ),
    "dco_stream_push_f32": (c_int, [c_void_p, P, P, P, ctypes.POINTER(FrameResult)]),
    "dco_stream_push_gray8_host": (c_int, [c_void_p, P, P, P, P, P, ctypes.POINTER(FrameResult)]),
    "dco_stream_push_gray8_host_encoded": (c_int, [c_void_p, P, P, P, P, P, ctypes.POINTER(FrameResult)]),
    "dco_stream_views": (c_int, [c_void_p, ctypes.POINTER(FrameViews)]),
    "dco_stream_set_lr_check": (c_int, [c_void_p, c_int, c_double]),
    "dco_stream_set_timing": (c_int, [c_void_p, c_int]),
    "dco_stream_span_times": (c_int, [c_void_p, ctypes.POINTER(c_double), ctypes.POINTER(c_uint64)]),
    "dco_stream_state_size": (c_size_t, [c_void_p]),
    "dco_stream_save_state": (c_int, [c_void_p, c_void_p, c_size_t]),
    "dco_stream_load_state": (c_int, [c_void_p, c_void_p, c_size_t]),
}

_lib = None


def load(path=LIB_PATH):
    """Loads libdco_gpu.so and declares every C-ABI signature. Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            "libdco_gpu.so is not built (%s); run `python -m paper_2203_02300_b200.build` "
            "— there is no CPU fallback" % path
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.dco_abi_version() != 3:
        raise RuntimeError("libdco_gpu.so ABI mismatch")
    _lib = lib
    return lib


def check(ctx, status):
    if status != 0:
        msg = load().dco_last_error(ctx)
        raise_for(status, msg.decode() if msg else "error %d" % status)
