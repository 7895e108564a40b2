"""B200-native depth-contour-occlusion (arXiv 2203.02300) hot path.

The product is libdco_gpu.so (csrc/*.cu, sm_100a) behind the C-ABI of
include/dco_gpu.h; `dco` mirrors the reference's stage API over it."""
from .config import (CodecError, Config, ConfigError, DcoError, InputError,  # noqa: F401
                     UnsolvableFrameError)

__all__ = ["Config", "DcoError", "InputError", "ConfigError", "CodecError", "UnsolvableFrameError"]
