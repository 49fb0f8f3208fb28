"""Synthetic workloads of BASELINE.json's five configs (seeded, deterministic).

The paper's datasets (DSEC driving, table tennis) are not
available; these generators stand in for them with the shapes, sizes and
value distributions BASELINE.json specifies.  Parameters BASELINE.json
leaves open are pinned here:

* RNG: numpy PCG64, seed = 1000 * config_index + stream.
* Gaussian blur: scipy.ndimage.gaussian_filter, truncate = 3 sigma, wrap.
* Brightness ramp: multiplicative, frame k scaled by 1.005 ** k.
* Camera motion: per-frame translation T and rotation theta about the image
  centre, cumulative (frame k sees k*T, k*theta); bilinear resampling of a
  toroidal (wrap-around) background, so no border content is invented.
* Objects: drawn in image space after the camera motion, in index order
  (later objects occlude earlier ones), velocities reflect at the borders.
* c5 flicker: 1 + 0.2 * sin(2 pi k / 30); translation along +x, integer.
* Timestamps: round(k * 1e6 / 30) us (30 fps input, scenes.cpp:10-12).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

FPS = 30.0


@dataclasses.dataclass(frozen=True)
class WorkloadConfig:
    name: str
    width: int
    height: int
    n_frames: int
    method: str            # "difference_only" | "dense" | "sparse"
    n_interp: int
    contrast: float        # log-mode C (both polarities)
    streams: int = 1
    n_objects: int = 12
    max_speed: float = 4.0
    camera: bool = False
    cam_translation: float = 8.0
    cam_rotation_deg: float = 1.0
    ramp: float = 0.005
    textured_objects: bool = False
    blur_sigma: float = 3.0
    unblurred: bool = False
    flicker: float = 0.0
    pan_px: int = 0
    index: int = 1

    @property
    def pixels(self) -> int:
        return self.width * self.height


CONFIGS = {
    "c1": WorkloadConfig("c1", 346, 260, 64, "difference_only", 0, 0.2, index=1),
    "c2": WorkloadConfig("c2", 640, 480, 128, "dense", 10, 0.2, camera=True, index=2),
    "c3": WorkloadConfig("c3", 1280, 720, 256, "sparse", 20, 0.15, n_objects=40, ramp=0.0,
                         textured_objects=True, index=3),
    "c4": WorkloadConfig("c4", 1920, 1080, 120, "dense", 16, 0.2, streams=32, camera=True,
                         cam_translation=6.0, cam_rotation_deg=0.5, max_speed=6.0, index=4),
    "c5": WorkloadConfig("c5", 3840, 2160, 60, "dense", 32, 0.1, n_objects=0, ramp=0.0, unblurred=True,
                         flicker=0.2, pan_px=16, index=5),
}

# Table I integer thresholds of the reference (types.hpp:101-120) for linear mode
LINEAR_THRESHOLDS = {"difference_only": (2, -2), "dense": (2, -2), "sparse": (10, -10)}


def timestamps(n: int) -> np.ndarray:
    return np.array([int(round(k * 1e6 / FPS)) for k in range(n)], dtype=np.int64)


def _blurred_noise(rng, h, w, sigma, lo=40.0, hi=215.0):
    from scipy.ndimage import gaussian_filter

    base = rng.uniform(0.0, 255.0, size=(h, w))
    b = gaussian_filter(base, sigma=sigma, mode="wrap", truncate=3.0)
    mn, mx = float(b.min()), float(b.max())
    return lo + (b - mn) * ((hi - lo) / max(mx - mn, 1e-9))


def _objects(rng, cfg: WorkloadConfig):
    objs = []
    for _ in range(cfg.n_objects):
        kind = "disc" if rng.uniform() < 0.5 else "rect"
        size = rng.uniform(10.0, 40.0)
        inten = rng.uniform(0.0, 255.0)
        x = rng.uniform(0, cfg.width)
        y = rng.uniform(0, cfg.height)
        vx = rng.uniform(-cfg.max_speed, cfg.max_speed)
        vy = rng.uniform(-cfg.max_speed, cfg.max_speed)
        tex = None
        if cfg.textured_objects:
            s = int(math.ceil(2 * size)) + 2
            tex = rng.uniform(-40.0, 40.0, size=(s, s))
            from scipy.ndimage import gaussian_filter
            tex = gaussian_filter(tex, sigma=1.5, mode="wrap", truncate=3.0) * 2.0
        objs.append(dict(kind=kind, size=size, inten=inten, x=x, y=y, vx=vx, vy=vy, tex=tex))
    return objs


def _draw_objects(img, objs, k, cfg):
    h, w = img.shape
    for o in objs:
        # position at frame k with reflection at the borders
        def reflect(p0, v, extent):
            p = p0 + v * k
            period = 2.0 * extent
            p = math.fmod(p, period)
            if p < 0:
                p += period
            return p if p < extent else period - p
        cx = reflect(o["x"], o["vx"], w)
        cy = reflect(o["y"], o["vy"], h)
        s = o["size"]
        x0, x1 = max(0, int(math.floor(cx - s)) - 1), min(w, int(math.ceil(cx + s)) + 2)
        y0, y1 = max(0, int(math.floor(cy - s)) - 1), min(h, int(math.ceil(cy + s)) + 2)
        if x0 >= x1 or y0 >= y1:
            continue
        yy, xx = np.mgrid[y0:y1, x0:x1]
        if o["kind"] == "disc":
            m = (xx - cx) ** 2 + (yy - cy) ** 2 <= s * s
        else:
            half = s / 2.0
            m = (np.abs(xx - cx) <= half) & (np.abs(yy - cy) <= half)
        val = np.full(m.shape, o["inten"])
        if o["tex"] is not None:
            t = o["tex"]
            ts = t.shape[0]
            tx = np.clip(np.floor(xx - cx + s).astype(np.int64), 0, ts - 1)
            ty = np.clip(np.floor(yy - cy + s).astype(np.int64), 0, ts - 1)
            val = val + t[ty, tx]
        region = img[y0:y1, x0:x1]
        region[m] = val[m]


def _camera_sample(bg, k, cfg, t_vec, theta_deg):
    from scipy.ndimage import map_coordinates

    h, w = cfg.height, cfg.width
    bh, bw = bg.shape
    th = math.radians(theta_deg * k)
    c, s = math.cos(th), math.sin(th)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    xc, yc = xx - (w - 1) / 2.0, yy - (h - 1) / 2.0
    # inverse map: frame pixel -> world coordinate
    wx = c * xc - s * yc + (w - 1) / 2.0 - t_vec[0] * k
    wy = s * xc + c * yc + (h - 1) / 2.0 - t_vec[1] * k
    return map_coordinates(bg, [np.mod(wy, bh), np.mod(wx, bw)], order=1, mode="grid-wrap")


def generate(cfg: WorkloadConfig | str, n_frames: int | None = None, stream: int = 0,
             width: int | None = None, height: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Frames (n, h, w) uint8 and timestamps (n,) int64 of one stream of `cfg`."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if width is not None or height is not None:
        cfg = dataclasses.replace(cfg, width=width or cfg.width, height=height or cfg.height)
    n = cfg.n_frames if n_frames is None else n_frames
    rng = np.random.Generator(np.random.PCG64(1000 * cfg.index + stream))
    h, w = cfg.height, cfg.width
    frames = np.zeros((n, h, w), np.uint8)
    if cfg.unblurred:
        tex = rng.integers(0, 256, size=(h, w)).astype(np.float64)
        for k in range(n):
            f = np.roll(tex, cfg.pan_px * k, axis=1)
            if cfg.flicker:
                f = f * (1.0 + cfg.flicker * math.sin(2.0 * math.pi * k / 30.0))
            frames[k] = np.clip(np.rint(f), 0, 255).astype(np.uint8)
        return frames, timestamps(n)
    if cfg.camera:
        bg = _blurred_noise(rng, h + 256, w + 256, cfg.blur_sigma)
        t_vec = rng.uniform(-cfg.cam_translation, cfg.cam_translation, size=2)
        theta = rng.uniform(-cfg.cam_rotation_deg, cfg.cam_rotation_deg)
    else:
        bg = _blurred_noise(rng, h, w, cfg.blur_sigma)
        t_vec, theta = None, 0.0
    objs = _objects(rng, cfg)
    for k in range(n):
        img = _camera_sample(bg, k, cfg, t_vec, theta) if cfg.camera else bg.copy()
        _draw_objects(img, objs, k, cfg)
        if cfg.ramp:
            img = img * (1.0 + cfg.ramp) ** k
        frames[k] = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    return frames, timestamps(n)
