"""Seeded synthetic inputs shared by the tests, the bench and the oracle runs.

This module holds NO arithmetic of the shearlet method: it only draws images
(and random complex cubes for adjoint tests).  It is the one module both the
CUDA path's callers and the oracle's callers use.

The images stand in for the paper's workloads: a "random image"
and "simple geometric structures", with the per-config
recipe of BASELINE.json ``configs`` / SURVEY.md 8(d).  Every draw comes from
``numpy.random.Generator(PCG64(seed))`` in the documented order; images are
generated in float64 and sampled at pixel centres ((c+1/2)/N, (r+1/2)/N),
painter's order, no clipping.  Callers cast to the run dtype and hand the SAME
cast values to the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Config", "CONFIGS", "config", "make_image", "make_batch",
           "uniform_image", "random_cube", "vertical_line_image", "random_spectra"]


@dataclass(frozen=True)
class Config:
    cid: int
    n: int
    batch: int
    dtype: str          # "f64" | "f32"
    generator: str      # "shapes3" | "ellipses_gradient" | "ellipses_polygons"
    sigma: float
    seed0: int
    label: str


# BASELINE.json "configs" (in order) with SURVEY.md 8(d)'s recipe.
CONFIGS = {
    1: Config(1, 64, 1, "f64", "shapes3", 0.05, 1, "64x64 f64 B=1: 3 disks/triangles + N(0,0.05^2)"),
    2: Config(2, 256, 16, "f32", "ellipses_gradient", 0.05, 2000,
              "256x256 f32 B=16: 3-8 ellipses + linear gradient + N(0,0.05^2)"),
    3: Config(3, 512, 64, "f32", "ellipses_polygons", 0.02, 3000,
              "512x512 f32 B=64: ellipses + polygons + N(0,0.02^2)"),
    4: Config(4, 1024, 32, "f32", "ellipses_polygons", 0.02, 4000,
              "1024x1024 f32 B=32: ellipses + polygons + N(0,0.02^2)"),
    5: Config(5, 4096, 1, "f32", "ellipses_polygons", 0.05, 5000,
              "4096x4096 f32 B=1: ellipses + polygons + N(0,0.05^2)"),
}


def config(cid: int) -> Config:
    return CONFIGS[int(cid)]


class _Canvas:
    """Pixel-centre sampler with bounding-box restricted painting."""

    def __init__(self, n: int):
        self.n = n
        self.img = np.zeros((n, n), dtype=np.float64)
        self.centres = (np.arange(n, dtype=np.float64) + 0.5) / n

    def _box(self, x0, x1, y0, y1):
        n = self.n
        c0, c1 = max(int(np.floor(x0 * n)) - 1, 0), min(int(np.ceil(x1 * n)) + 1, n)
        r0, r1 = max(int(np.floor(y0 * n)) - 1, 0), min(int(np.ceil(y1 * n)) + 1, n)
        if c0 >= c1 or r0 >= r1:
            return None
        xs, ys = np.meshgrid(self.centres[c0:c1], self.centres[r0:r1])
        return (slice(r0, r1), slice(c0, c1)), xs, ys

    def paint_mask(self, bbox, inside_fn, value):
        box = self._box(*bbox)
        if box is None:
            return
        sl, xs, ys = box
        mask = inside_fn(xs, ys)
        self.img[sl][mask] = value

    def disk(self, cx, cy, rad, value):
        self.paint_mask((cx - rad, cx + rad, cy - rad, cy + rad),
                        lambda x, y: (x - cx) ** 2 + (y - cy) ** 2 <= rad * rad, value)

    def ellipse(self, cx, cy, a, b, theta, value):
        ct, st = np.cos(theta), np.sin(theta)
        ext = max(a, b)

        def inside(x, y):
            dx, dy = x - cx, y - cy
            u = dx * ct + dy * st
            v = -dx * st + dy * ct
            return (u / a) ** 2 + (v / b) ** 2 <= 1.0
        self.paint_mask((cx - ext, cx + ext, cy - ext, cy + ext), inside, value)

    def convex_polygon(self, vx, vy, value):
        """vertices in counter-clockwise order (sorted angles)."""
        k = len(vx)

        def inside(x, y):
            ok = np.ones(x.shape, dtype=bool)
            for e in range(k):
                x0, y0, x1, y1 = vx[e], vy[e], vx[(e + 1) % k], vy[(e + 1) % k]
                ok &= (x1 - x0) * (y - y0) - (y1 - y0) * (x - x0) >= 0.0
            return ok
        self.paint_mask((min(vx), max(vx), min(vy), max(vy)), inside, value)


def _polygon_vertices(rng, cx, cy, rad, nv):
    ang = np.sort(rng.uniform(0.0, 2.0 * np.pi, size=nv))
    return cx + rad * np.cos(ang), cy + rad * np.sin(ang)


def make_image(cfg: Config, index: int) -> np.ndarray:
    """Image ``index`` of config ``cfg`` (float64, shape (N, N)).  Draw order is
    fixed: shape count, then each shape's parameters in the order written
    below, then (config 2) the gradient, then the noise field."""
    seed = cfg.seed0 + index
    rng = np.random.Generator(np.random.PCG64(seed))
    canvas = _Canvas(cfg.n)
    if cfg.generator == "shapes3":
        for _ in range(3):
            is_disk = rng.uniform() < 0.5
            cx, cy = rng.uniform(0.2, 0.8, size=2)
            if is_disk:
                rad = rng.uniform(0.05, 0.2)
                value = rng.uniform()
                canvas.disk(cx, cy, rad, value)
            else:
                rad = rng.uniform(0.08, 0.25)
                vx, vy = _polygon_vertices(rng, cx, cy, rad, 3)
                value = rng.uniform()
                canvas.convex_polygon(vx, vy, value)
    else:
        n_ell = int(rng.integers(3, 9))
        for _ in range(n_ell):
            cx, cy = rng.uniform(0.15, 0.85, size=2)
            a, b = rng.uniform(0.04, 0.3, size=2)
            theta = rng.uniform(0.0, np.pi)
            value = rng.uniform()
            canvas.ellipse(cx, cy, a, b, theta, value)
        if cfg.generator == "ellipses_polygons":
            n_poly = int(rng.integers(2, 6))
            for _ in range(n_poly):
                nv = int(rng.integers(3, 7))
                cx, cy = rng.uniform(0.2, 0.8, size=2)
                rad = rng.uniform(0.05, 0.25)
                vx, vy = _polygon_vertices(rng, cx, cy, rad, nv)
                value = rng.uniform()
                canvas.convex_polygon(vx, vy, value)
    img = canvas.img
    if cfg.generator == "ellipses_gradient":
        ga, gb = rng.uniform(-0.25, 0.25, size=2)
        xs, ys = np.meshgrid(canvas.centres, canvas.centres)
        img = img + ga * xs + gb * ys
    img = img + rng.normal(0.0, cfg.sigma, size=img.shape)
    return img


def make_batch(cid: int, batch: int | None = None, n: int | None = None) -> np.ndarray:
    """float64 batch (B, N, N) of config ``cid``; ``batch`` / ``n`` override the
    config's size (same generator, same seeds) for reduced parity cases."""
    cfg = config(cid)
    if n is not None or batch is not None:
        cfg = Config(cfg.cid, n or cfg.n, batch or cfg.batch, cfg.dtype, cfg.generator,
                     cfg.sigma, cfg.seed0, cfg.label)
    return np.stack([make_image(cfg, b) for b in range(cfg.batch)])


def uniform_image(n: int, seed: int) -> np.ndarray:
    """The paper's "random image": i.i.d. U[0,1] pixels."""
    return np.random.Generator(np.random.PCG64(seed)).uniform(size=(n, n))


def vertical_line_image(n: int, column: int | None = None) -> np.ndarray:
    """A one-pixel vertical line (constant along rows m2) for the orientation test."""
    img = np.zeros((n, n))
    img[:, n // 2 if column is None else column] = 1.0
    return img


def random_cube(shape, seed: int) -> np.ndarray:
    """Random complex array (real and imaginary parts N(0,1)) for adjoint tests."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def random_spectra(n: int, eta: int, seed: int, parseval: bool = True) -> np.ndarray:
    """A random user spectra set (eta, n, n), centred layout (omega = 0 at (n/2, n/2)), for the
    user-spectra mode.  Input construction only, not the shearlet method:
      * plane 0 is a random positive "low-pass" on every grid point (so every point is covered);
      * planes 1.. are random non-negative bumps on a random band of columns |u1| in [lo, hi]
        (exercises the per-plane column pruning), zero elsewhere;
      * every plane is point-symmetric, g(u) = g(-u), off the Nyquist lines; on the row
        u2 = -n/2 and the column u1 = -n/2 the values at u and -u are drawn independently
        (asymmetric: the anti parts the even-n decomposition handles exactly);
      * parseval=True divides all planes by sqrt(sum_i g_i^2) pointwise, so sum_i psi_i^2 = 1.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    h = n // 2
    u = np.arange(n) - h                                   # centred coordinates
    u1, u2 = np.meshgrid(u, u)                             # columns omega_1, rows omega_2
    neg = (n - np.arange(n)) % n                           # index of -u (with -(-n/2) = -n/2)
    g = np.zeros((eta, n, n))
    for i in range(eta):
        r = rng.uniform(0.05, 1.0, (n, n))
        if i > 0:
            lo = int(rng.integers(0, h + 1))
            hi = int(rng.integers(lo, h + 1))
            r = r * ((np.abs(u1) >= lo) & (np.abs(u1) <= hi))
            r = r * (rng.uniform(0, 1, (n, n)) < 0.7)
        sym = 0.5 * (r + r[neg][:, neg])                   # point-symmetric copy
        nyq = (u1 == -h) | (u2 == -h)
        g[i] = np.where(nyq, r, sym)
    if parseval:
        g = g / np.sqrt(np.sum(g * g, axis=0))
    return g
