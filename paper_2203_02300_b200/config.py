"""PipelineConfig mirror (reference include/dco/config.hpp:11-60) as the ctypes
struct `dco_config` of include/dco_gpu.h, plus the reference's error classes
(include/dco/error.hpp:10-32). Pure Python: importable without a GPU."""
import ctypes

# (name, ctype, default) in PipelineConfig declaration order (config.hpp:13-56)
FIELDS = [
    ("lambda_ad", ctypes.c_double, 10.0),
    ("lambda_census", ctypes.c_double, 40.0),
    ("gamma_l", ctypes.c_double, 1.0),
    ("epsilon", ctypes.c_double, 0.8),
    ("t_high", ctypes.c_double, 0.06),
    ("t_low", ctypes.c_double, 0.03),
    ("t_depth", ctypes.c_double, 0.03),
    ("lambda_d", ctypes.c_double, 0.8),
    ("lambda_s", ctypes.c_double, 1.2),
    ("lambda_s2", ctypes.c_double, 0.02),
    ("d_min", ctypes.c_int, 0),
    ("d_max", ctypes.c_int, 64),
    ("focal_px", ctypes.c_double, 400.0),
    ("baseline_m", ctypes.c_double, 0.12),
    ("census_window_w", ctypes.c_int, 9),
    ("census_window_h", ctypes.c_int, 7),
    ("cross_color_tau", ctypes.c_double, 20.0 / 255.0),
    ("cross_color_tau2", ctypes.c_double, 6.0 / 255.0),
    ("cross_arm_l1", ctypes.c_int, 17),
    ("cross_arm_l2", ctypes.c_int, 8),
    ("box_radius", ctypes.c_int, 5),
    ("gauss_sigma", ctypes.c_double, 1.4),
    ("confidence_offset_k", ctypes.c_double, 2.0),
    ("hist_iterations", ctypes.c_int, 2),
    ("solver_tol", ctypes.c_double, 1e-5),
    ("solver_max_iter", ctypes.c_int, 400),
]


class Config(ctypes.Structure):
    """dco_config / dco::PipelineConfig. Keyword arguments override defaults."""

    _fields_ = [(n, t) for n, t, _ in FIELDS]

    def __init__(self, **overrides):
        super().__init__()
        for n, _, d in FIELDS:
            setattr(self, n, d)
        for k, v in overrides.items():
            if k not in dict((n, 0) for n, _, _ in FIELDS):
                raise InputError("config: unknown key '%s'" % k)
            setattr(self, k, v)

    def copy(self, **overrides):
        c = Config()
        for n, _, _ in FIELDS:
            setattr(c, n, getattr(self, n))
        for k, v in overrides.items():
            setattr(c, k, v)
        return c

    def as_dict(self):
        return {n: getattr(self, n) for n, _, _ in FIELDS}

    @property
    def num_disparities(self):
        return self.d_max - self.d_min + 1


class DcoError(RuntimeError):
    """Base of the reference's exception hierarchy as seen through the C-ABI."""


class InputError(DcoError):
    """dco::InputError (CLI exit code 1)."""


class ConfigError(InputError):
    """dco::ConfigError, an InputError (exit code 1)."""


class CodecError(DcoError):
    """dco::CodecError (exit code 2)."""


class UnsolvableFrameError(DcoError):
    """dco::UnsolvableFrameError (exit code 3)."""


class CudaError(DcoError):
    """Device/driver failure (no reference analogue)."""


# dco_status -> exception class (include/dco_gpu.h)
STATUS_ERRORS = {1: InputError, 5: ConfigError, 2: CodecError, 3: UnsolvableFrameError, 4: CudaError}


def raise_for(status, message):
    if status == 0:
        return
    raise STATUS_ERRORS.get(status, DcoError)(message)
