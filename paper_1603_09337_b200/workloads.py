"""Seeded synthetic inputs for BASELINE.json's five configs.

The reference ships no benchmark images (the paper's 512x512 frames are not
public), so these generators stand in for them with the shapes, object
counts, radii and noise levels BASELINE.json states.  Per-image seed =
config base seed + image index; everything is drawn from one
numpy.random.default_rng per image.  Ellipses are rasterised inside their
bounding boxes.

Also restated here: the reference's own benchmark / topology inputs
`jagged_disc` and `noisy_disc` (tests/conftest.py:14-32 of the reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    h: int
    w: int
    r_max: int
    fg: int          # 8 -> (8,4), 4 -> (4,8)
    base_seed: int
    kind: str        # "blobs" | "mazes"
    objects: int = 40
    rad_lo: float = 8.0
    rad_hi: float = 60.0
    noise: float = 0.05
    constraints: float = 0.0   # > 0: seeded keep / avoid masks (constraint_masks), SURVEY §8 row f4


CONFIGS = {
    "c0": Config("c0", 1, 512, 512, 3, 8, 0, "blobs", 40, 8, 60, 0.05),
    "c1": Config("c1", 256, 512, 512, 5, 8, 1000, "blobs", 40, 8, 60, 0.05),
    "c2": Config("c2", 32, 2048, 2048, 10, 8, 2000, "blobs", 160, 30, 240, 0.10),
    "c3": Config("c3", 1, 8192, 8192, 8, 8, 3000, "blobs", 2000, 10, 400, 0.05),
    "c4": Config("c4", 1024, 256, 256, 4, 4, 4000, "mazes", 0, 0, 0, 0.02),
    # c1 with control images (reference smoothing.py:197-206): 1% of the object
    # pixels must stay object (keep), 1% of the background must stay background
    "c1k": Config("c1k", 256, 512, 512, 5, 8, 1000, "blobs", 40, 8, 60, 0.05, 0.01),
}


def _ellipse(img, cy, cx, a, b, theta, value):
    """Set pixels inside the rotated ellipse (semi-axes a along theta, b across)."""
    h, w = img.shape
    rad = int(np.ceil(max(a, b))) + 1
    y0, y1 = max(0, int(cy) - rad), min(h, int(cy) + rad + 1)
    x0, x1 = max(0, int(cx) - rad), min(w, int(cx) + rad + 1)
    if y0 >= y1 or x0 >= x1:
        return
    yy = np.arange(y0, y1, dtype=np.float64)[:, None] - cy
    xx = np.arange(x0, x1, dtype=np.float64)[None, :] - cx
    c, s = np.cos(theta), np.sin(theta)
    u = xx * c + yy * s
    v = -xx * s + yy * c
    inside = (u / a) ** 2 + (v / b) ** 2 <= 1.0
    img[y0:y1, x0:x1][inside] = value


def blob_image(h, w, seed, objects=40, rad_lo=8.0, rad_hi=60.0, noise=0.05) -> np.ndarray:
    """Union of `objects` filled discs/ellipses, each with 0-2 elliptical holes,
    then salt-and-pepper noise (XOR with Bernoulli(noise))."""
    rng = np.random.default_rng(seed)
    img = np.zeros((h, w), np.uint8)
    for _ in range(objects):
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        a = rng.uniform(rad_lo, rad_hi)
        b = a if rng.random() < 0.5 else rng.uniform(rad_lo, rad_hi)
        theta = rng.uniform(0, np.pi)
        n_holes = int(rng.integers(0, 3))
        holes = []
        for _ in range(n_holes):
            ha, hb = a * rng.uniform(0.1, 0.4), b * rng.uniform(0.1, 0.4)
            oy, ox = rng.uniform(-0.4, 0.4) * b, rng.uniform(-0.4, 0.4) * a
            holes.append((cy + oy, cx + ox, ha, hb, rng.uniform(0, np.pi)))
        rad = int(np.ceil(max(a, b))) + 1
        y0, y1 = max(0, int(cy) - rad), min(h, int(cy) + rad + 1)
        x0, x1 = max(0, int(cx) - rad), min(w, int(cx) + rad + 1)
        if y0 >= y1 or x0 >= x1:
            continue
        patch = np.zeros((y1 - y0, x1 - x0), np.uint8)
        _ellipse_local(patch, cy - y0, cx - x0, a, b, theta, 1)
        for (hy, hx, ha, hb, ht) in holes:
            _ellipse_local(patch, hy - y0, hx - x0, ha, hb, ht, 0)
        img[y0:y1, x0:x1] |= patch
    if noise > 0:
        img ^= (rng.random((h, w)) < noise).astype(np.uint8)
    return img


def _ellipse_local(patch, cy, cx, a, b, theta, value):
    _ellipse(patch, cy, cx, a, b, theta, value)


def _stamp_segment(img, y0, x0, y1, x1, width):
    h, w = img.shape
    n = int(max(abs(y1 - y0), abs(x1 - x0))) * 2 + 1
    lo = -((width - 1) // 2)
    hi = lo + width
    for t in np.linspace(0.0, 1.0, n):
        y = int(round(y0 + (y1 - y0) * t))
        x = int(round(x0 + (x1 - x0) * t))
        img[max(0, y + lo):min(h, y + hi), max(0, x + lo):min(w, x + hi)] = 1


def maze_image(h, w, seed, noise=0.02) -> np.ndarray:
    """Thin structures: 2-4 random walks of 6-20 steps on an 8x8 coarse grid,
    rasterised as 1-3 px wide polylines between cell centres; with p=0.7 a
    1-3 px wide spiral; then XOR with Bernoulli(noise)."""
    rng = np.random.default_rng(seed)
    img = np.zeros((h, w), np.uint8)
    cell_h, cell_w = h / 8.0, w / 8.0
    steps4 = ((-1, 0), (1, 0), (0, -1), (0, 1))
    for _ in range(int(rng.integers(2, 5))):
        cy, cx = int(rng.integers(0, 8)), int(rng.integers(0, 8))
        width = int(rng.integers(1, 4))
        for _ in range(int(rng.integers(6, 21))):
            dy, dx = steps4[int(rng.integers(0, 4))]
            ny, nx = min(7, max(0, cy + dy)), min(7, max(0, cx + dx))
            _stamp_segment(img, (cy + 0.5) * cell_h, (cx + 0.5) * cell_w,
                           (ny + 0.5) * cell_h, (nx + 0.5) * cell_w, width)
            cy, cx = ny, nx
    if rng.random() < 0.7:
        width = int(rng.integers(1, 4))
        turns = rng.uniform(2.0, 4.0)
        r_max = 0.45 * min(h, w)
        oy, ox = h / 2 + rng.uniform(-0.1, 0.1) * h, w / 2 + rng.uniform(-0.1, 0.1) * w
        phase = rng.uniform(0, 2 * np.pi)
        n = int(turns * 2 * np.pi * r_max)
        th = np.linspace(0.0, turns * 2 * np.pi, n)
        rr = r_max * th / th[-1]
        ys = np.round(oy + rr * np.sin(th + phase)).astype(int)
        xs = np.round(ox + rr * np.cos(th + phase)).astype(int)
        lo = -((width - 1) // 2)
        for dy in range(lo, lo + width):
            for dx in range(lo, lo + width):
                yy, xx = ys + dy, xs + dx
                ok = (yy >= 0) & (yy < h) & (xx >= 0) & (xx < w)
                img[yy[ok], xx[ok]] = 1
    if noise > 0:
        img ^= (rng.random((h, w)) < noise).astype(np.uint8)
    return img


def config_image(cfg: Config | str, i: int) -> np.ndarray:
    cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    seed = cfg.base_seed + i
    if cfg.kind == "mazes":
        return maze_image(cfg.h, cfg.w, seed, cfg.noise)
    return blob_image(cfg.h, cfg.w, seed, cfg.objects, cfg.rad_lo, cfg.rad_hi, cfg.noise)


def config_batch(cfg: Config | str, start: int = 0, count: int | None = None) -> np.ndarray:
    """Images start..start+count-1 of the config as a uint8 [count, h, w] array."""
    cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    count = cfg.n - start if count is None else count
    out = np.empty((count, cfg.h, cfg.w), np.uint8)
    for k in range(count):
        out[k] = config_image(cfg, start + k)
    return out


def constraint_masks(cfg: Config | str, imgs: np.ndarray, start: int = 0):
    """Seeded keep / avoid masks for a batch of config images (image i uses
    seed base_seed + start + i + 500000): keep = each object pixel with
    probability cfg.constraints, avoid = each background pixel likewise.
    Disjoint, keep inside the object, avoid outside it (the reference's
    validity conditions, smoothing.py:199-206)."""
    cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    frac = cfg.constraints or 0.01
    keep = np.empty_like(imgs)
    avoid = np.empty_like(imgs)
    for k in range(len(imgs)):
        rng = np.random.default_rng(cfg.base_seed + start + k + 500000)
        u = rng.random(imgs[k].shape)
        keep[k] = (imgs[k] == 1) & (u < frac)
        avoid[k] = (imgs[k] == 0) & (u < frac)
    return keep, avoid


def jagged_disc(h, w, radius, amplitudes=((9, 12.0, 0.0), (23, 7.0, 1.2), (41, 4.0, 0.3))):
    """Reference tests/conftest.py:23-32 (the acceptance-8 benchmark input)."""
    yy = np.arange(h)[:, None] - h // 2
    xx = np.arange(w)[None, :] - w // 2
    theta = np.arctan2(yy, xx)
    rr = np.full((h, w), float(radius))
    for freq, amp, phase in amplitudes:
        rr += amp * np.sin(freq * theta + phase)
    return ((yy * yy + xx * xx) <= rr * rr).astype(np.uint8)


def noisy_disc(h, w, radius, rng, flip=0.03):
    """Reference tests/conftest.py:14-20."""
    yy = np.arange(h)[:, None] - h // 2
    xx = np.arange(w)[None, :] - w // 2
    disc = (yy * yy + xx * xx <= radius * radius).astype(np.uint8)
    noise = rng.random((h, w)) < flip
    return (disc ^ noise.astype(np.uint8)).astype(np.uint8)


def random_image(rng, h, w, density):
    """Reference tests/conftest.py:10-11."""
    return (rng.random((h, w)) < density).astype(np.uint8)
