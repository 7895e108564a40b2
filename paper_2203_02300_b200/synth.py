"""Synthetic stereo-video workload for the benchmark (numpy, product side).

Same scene family as the reference's generator (synth.cpp:68-135
describes it): a value-noise textured square at z_fg sliding horizontally over
a textured background plane at z_bg, imaged by a rectified pair
(focal 400 px, baseline 0.12 m -> full-resolution disparities 48 / 24),
quantised to 8 bit. This is an independent implementation (not the oracle),
so the timed path never executes oracle/ code. Motion ping-pongs so an
arbitrarily long stream stays inside the frame."""
import numpy as np


def _value_noise(h, w, cell, rng):
    gh, gw = h // cell + 2, w // cell + 2
    lattice = rng.random((gh, gw), dtype=np.float32)
    ys, xs = np.arange(h) / cell, np.arange(w) / cell
    y0, x0 = ys.astype(int), xs.astype(int)
    fy, fx = (ys - y0).astype(np.float32), (xs - x0).astype(np.float32)
    fy, fx = fy * fy * (3 - 2 * fy), fx * fx * (3 - 2 * fx)
    a = lattice[y0][:, x0]
    b = lattice[y0][:, x0 + 1]
    c = lattice[y0 + 1][:, x0]
    d = lattice[y0 + 1][:, x0 + 1]
    top = a * (1 - fx) + b * fx
    bot = c * (1 - fx) + d * fx
    return top * (1 - fy[:, None]) + bot * fy[:, None] - 0.5


def texture(h, w, base, seed):
    rng = np.random.default_rng(seed)
    t = base + 0.22 * _value_noise(h, w, 8, rng) + 0.12 * _value_noise(h, w, 4, rng) \
        + 0.06 * (rng.random((h, w), dtype=np.float32) - 0.5)
    return np.clip(t, 0.0, 1.0).astype(np.float32)


class StereoVideo:
    """frames(i) -> (left u8 [h,w], right u8 [h,w]) of a moving-square scene."""

    def __init__(self, width, height, seed=61, focal_px=400.0, baseline_m=0.12, z_fg=1.0, z_bg=2.0,
                 shift_x=4, period=16):
        self.w, self.h = width, height
        self.d_fg = int(round(focal_px * baseline_m / z_fg))
        self.d_bg = int(round(focal_px * baseline_m / z_bg))
        self.side = max(8, (height // 3) // 8 * 8)
        self.x0, self.y0 = width // 3, height // 3
        self.shift, self.period = shift_x, period
        pad = self.d_fg + 8
        self.bg = texture(height, width + pad, 0.62, seed ^ 0xB66B)
        self.fg = texture(self.side, self.side, 0.34, seed ^ 0xF00D)

    def square_x(self, i):
        k = i % (2 * self.period)
        k = k if k < self.period else 2 * self.period - k
        return self.x0 + self.shift * k

    def frame(self, i):
        h, w, s = self.h, self.w, self.side
        sx, sy = self.square_x(i), self.y0
        left = self.bg[:, :w].copy()
        left[sy:sy + s, sx:sx + s] = self.fg
        # right view: background shifted by d_bg, square by d_fg
        right = self.bg[:, self.d_bg:self.d_bg + w].copy()
        rx = sx - self.d_fg
        lo, hi = max(rx, 0), min(rx + s, w)
        if hi > lo:
            right[sy:sy + s, lo:hi] = self.fg[:, lo - rx:hi - rx]
        q = lambda a: np.clip(np.rint(a * 255.0), 0, 255).astype(np.uint8)  # noqa: E731
        return q(left), q(right)
