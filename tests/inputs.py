"""Seeded inputs shared by the parity tests: the reference's own
synthetic scene generator (render_synth_frame, synth.cpp:68-135) through the
8-bit PGM round trip the CLI path applies (codec.cpp:23-26, 80), plus the
xorshift64* generator of the reference's tests (tests/test_util.hpp:16-35)."""
import numpy as np


class Rng:
    """xorshift64* of tests/test_util.hpp:16-35 / acceptance.cpp:51-67."""

    M = (1 << 64) - 1

    def __init__(self, seed):
        self.state = seed if seed else 1

    def next(self):
        s = self.state
        s ^= s >> 12
        s ^= (s << 25) & self.M
        s ^= s >> 27
        self.state = s
        return (s * 0x2545F4914F6CDD1D) & self.M

    def uniform(self, lo=0.0, hi=1.0):
        u = (self.next() >> 11) * 2.0 ** -53
        return lo + (hi - lo) * u

    def uniform_int(self, lo, hi):
        return lo + self.next() % (hi - lo + 1)


def random_image(w, h, seed):
    rng = np.random.default_rng(seed)
    return rng.random((h, w), dtype=np.float32)


def scene(ref, w, h, index=0, seed=61, quantize=True, **kw):
    """One frame of the benchmark scene: square of side ~H/3 at
    (W/3, H/3), shift 4 px/frame. Returns dict with float left/right (after the
    8-bit round trip when quantize) and their bytes."""
    side = max(8, (h // 3) // 8 * 8)
    args = dict(square_size=side, square_x0=float(w // 3), square_y0=float(h // 3), shift_x=4.0, seed=seed)
    args.update(kw)
    f = ref.render_synth_frame(w, h, index, **args)
    if quantize:
        f["left8"], f["left"] = ref.quantize8(f["left"])
        f["right8"], f["right"] = ref.quantize8(f["right"])
    return f
