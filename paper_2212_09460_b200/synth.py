"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no Sobel, no voting, no peak
logic): only the workload generators of BASELINE.json ``configs`` (DESIGN.md
section 5 states each recipe) and the caller-supplied Q15 trig table, which
``north_star`` makes an INPUT of every library call ("a caller-supplied Q15
int32 cos/sin table").  Both sides receive the very same bytes.

All randomness is numpy ``Generator(PCG64(seed))`` with draws in the fixed
order documented per generator, so a frame is a pure function of its seed.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np


# ----------------------------------------------------------------------------
# Trig table (input).  DESIGN R11: Q15 int32, cos(0) = 32768 does not fit int16.
# ----------------------------------------------------------------------------
def q15_table(n_theta: int) -> tuple[np.ndarray, np.ndarray]:
    """C[t], S[t] = round-half-up(cos/sin(pi t / n_theta) * 2^15) for the first
    half; for t > n_theta/2 the table is symmetry-completed with Eq. 4-5
    (P:128-134): S[t] = S[n_theta - t], C[t] = -C[n_theta - t]."""
    if n_theta < 1:
        raise ValueError("n_theta must be >= 1")
    t = np.arange(n_theta, dtype=np.float64)
    th = np.pi * t / n_theta
    c = np.floor(np.cos(th) * 32768.0 + 0.5).astype(np.int64)
    s = np.floor(np.sin(th) * 32768.0 + 0.5).astype(np.int64)
    for i in range(n_theta // 2 + 1, n_theta):
        c[i] = -c[n_theta - i]
        s[i] = s[n_theta - i]
    return c.astype(np.int32), s.astype(np.int32)


def f64_table(n_theta: int) -> tuple[np.ndarray, np.ndarray]:
    """SPEC's float64 trig table (build_trig_table mode float64):
    cos/sin(pi t / n_theta) for t <= n_theta/2 with the exact values at 0 and
    90 degrees (cos[n/2] = 0, sin[n/2] = 1), and for t > n_theta/2 the
    Eq. 4-5 completion cos[t] = -cos[n-t], sin[t] = sin[n-t], exactly."""
    if n_theta < 1:
        raise ValueError("n_theta must be >= 1")
    t = np.arange(n_theta, dtype=np.float64)
    th = np.pi * t / n_theta
    c, s = np.cos(th), np.sin(th)
    c[0], s[0] = 1.0, 0.0
    if n_theta % 2 == 0:
        c[n_theta // 2], s[n_theta // 2] = 0.0, 1.0
    for i in range(n_theta // 2 + 1, n_theta):
        c[i] = -c[n_theta - i]
        s[i] = s[n_theta - i]
    return c, s


# ----------------------------------------------------------------------------
# Workload configurations (BASELINE.json configs[0..4]).
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    batch: int
    threshold: int
    n_theta: int
    k: int
    half_theta: int  # peak window half-widths: MATLAB houghpeaks rule (DESIGN R13)
    half_rho: int
    min_votes: int = 1
    seeds: tuple = field(default=())
    description: str = ""


CONFIGS = {
    "cfg1": Config("cfg1", 320, 240, 1, 200, 180, 2, 2, 8, seeds=(0,),
                   description="320x240, two fixed lanes to (160,100), T=200, 180 theta"),
    "cfg2": Config("cfg2", 1280, 720, 1, 200, 180, 4, 2, 29, seeds=(1,),
                   description="1280x720 noisy road, 2 solid + 1 dashed lane, T=200"),
    "cfg3": Config("cfg3", 1280, 720, 256, 200, 180, 4, 2, 29,
                   seeds=tuple(1000 + f for f in range(256)),
                   description="256 x 1280x720 road frames with clutter, T=200"),
    "cfg4": Config("cfg4", 1920, 1080, 64, 160, 720, 8, 7, 44,
                   seeds=tuple(2000 + f for f in range(64)),
                   description="64 x 1920x1080 8x8-block texture + 4 lanes, T=160, 720 theta"),
    "cfg5": Config("cfg5", 4096, 4096, 1, 200, 1024, 64, 10, 116, seeds=(3,),
                   description="4096^2, 200 random segments, T=200, 1024 theta"),
}


def frame_seed(cfg: Config, frame: int) -> int:
    """Seed of global frame index ``frame`` (DESIGN R20).  Frames beyond the
    configured batch (weak-scaling ranks) continue the same seed sequence."""
    if frame < len(cfg.seeds):
        return cfg.seeds[frame]
    return cfg.seeds[0] + frame


# ----------------------------------------------------------------------------
# Raster helpers (scene drawing only).
# ----------------------------------------------------------------------------
def _paint_lane(img: np.ndarray, xb: float, vx: float, vy: float, w: int, value: int,
                dashed: bool) -> None:
    """Lane from the bottom row at column xb toward the vanishing point (vx, vy):
    row y in [ceil(vy), H-1]: s = (H-1-y)/(H-1-vy), xc = xb + (vx-xb) s, paint
    columns [floor(xc - w/2 + 1/2), +w-1] clipped; dashed lanes paint rows with
    floor(16 s) even."""
    h, wd = img.shape
    y_top = max(int(math.ceil(vy)), 0)
    ys = np.arange(y_top, h)
    s = (h - 1 - ys) / (h - 1 - vy)
    if dashed:
        keep = (np.floor(16.0 * s).astype(np.int64) % 2) == 0
        ys, s = ys[keep], s[keep]
    xc = xb + (vx - xb) * s
    x0 = np.floor(xc - w / 2.0 + 0.5).astype(np.int64)
    cols = np.arange(wd)[None, :]
    mask = (cols >= x0[:, None]) & (cols < x0[:, None] + w)
    sub = img[ys]
    sub[mask] = value
    img[ys] = sub


def _lanes_cfg2_model(rng: np.random.Generator, img: np.ndarray, n_lanes: int,
                      dashed_index: int | None) -> None:
    h, w = img.shape
    vx = rng.uniform(0.3 * w, 0.7 * w)
    vy = rng.uniform(0.0, h / 3.0)
    for i in range(n_lanes):
        xb = rng.uniform(0.0, w)
        lw = int(rng.integers(3, 7))
        val = int(rng.integers(200, 256))
        _paint_lane(img, xb, vx, vy, lw, val, dashed=(dashed_index == i))


def gen_cfg1(seed: int = 0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    img = rng.integers(40, 81, size=(240, 320)).astype(np.uint8)
    for xb in (60.0, 260.0):
        _paint_lane(img, xb, 160.0, 100.0, 4, 230, dashed=False)
    return img


def _noisy_background(rng, h, w, lo, hi, sigma) -> np.ndarray:
    bg = rng.integers(lo, hi + 1, size=(h, w)).astype(np.int32)
    noise = np.rint(rng.normal(0.0, sigma, size=(h, w))).astype(np.int32)
    return np.clip(bg + noise, 0, 255).astype(np.uint8)


def gen_cfg2(seed: int = 1, width: int = 1280, height: int = 720) -> np.ndarray:
    """Draw order: background ints, noise normals, vanishing point (vx, vy),
    then per lane (xb, width, value); lane index 2 is dashed."""
    rng = np.random.Generator(np.random.PCG64(seed))
    img = _noisy_background(rng, height, width, 30, 90, 10.0)
    _lanes_cfg2_model(rng, img, 3, dashed_index=2)
    return img


def gen_cfg3(seed: int, width: int = 1280, height: int = 720) -> np.ndarray:
    """cfg2's model (DESIGN R18) plus 0-8 clutter rectangles drawn before the lanes.
    Draw order: background, noise, n_rect, per rect (x0, y0, w, h, value),
    vanishing point, per lane (xb, width, value)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    img = _noisy_background(rng, height, width, 30, 90, 10.0)
    n_rect = int(rng.integers(0, 9))
    for _ in range(n_rect):
        x0 = int(rng.integers(0, width))
        y0 = int(rng.integers(0, height))
        rw = int(rng.integers(10, 81))
        rh = int(rng.integers(10, 81))
        val = int(rng.integers(180, 256))
        img[y0:y0 + rh, x0:x0 + rw] = val
    _lanes_cfg2_model(rng, img, 3, dashed_index=2)
    return img


def gen_cfg4(seed: int, width: int = 1920, height: int = 1080) -> np.ndarray:
    """Per-8x8-block uniform [0,255] levels (DESIGN R17) + 4 solid lanes (R19)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    bh, bw = (height + 7) // 8, (width + 7) // 8
    levels = rng.integers(0, 256, size=(bh, bw)).astype(np.uint8)
    img = np.repeat(np.repeat(levels, 8, axis=0), 8, axis=1)[:height, :width].copy()
    _lanes_cfg2_model(rng, img, 4, dashed_index=None)
    return img


def gen_cfg5(seed: int = 3, width: int = 4096, height: int = 4096,
             n_segments: int = 200) -> np.ndarray:
    """Background uniform [40,80]; n_segments 1-px DDA segments of value 220.
    Draw order: background, then per segment (x0, y0, angle, length)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    img = rng.integers(40, 81, size=(height, width)).astype(np.uint8)
    for _ in range(n_segments):
        x0 = rng.uniform(0.0, width)
        y0 = rng.uniform(0.0, height)
        ang = rng.uniform(0.0, np.pi)
        length = rng.uniform(50.0, 4000.0)
        n = int(math.ceil(length))
        i = np.arange(n + 1, dtype=np.float64)
        xs = np.floor(x0 + i * math.cos(ang) + 0.5).astype(np.int64)
        ys = np.floor(y0 + i * math.sin(ang) + 0.5).astype(np.int64)
        ok = (xs >= 0) & (xs < width) & (ys >= 0) & (ys < height)
        img[ys[ok], xs[ok]] = 220
    return img


_GEN = {"cfg1": lambda s: gen_cfg1(s), "cfg2": lambda s: gen_cfg2(s),
        "cfg3": lambda s: gen_cfg3(s), "cfg4": lambda s: gen_cfg4(s),
        "cfg5": lambda s: gen_cfg5(s)}


def gen_frame(cfg_name: str, frame: int = 0) -> np.ndarray:
    cfg = CONFIGS[cfg_name]
    return _GEN[cfg_name](frame_seed(cfg, frame))


def gen_batch(cfg_name: str, first: int = 0, count: int | None = None,
              out: np.ndarray | None = None) -> np.ndarray:
    """Frames [first, first+count) of a config as uint8 [count][H][W]."""
    cfg = CONFIGS[cfg_name]
    if count is None:
        count = cfg.batch
    if out is None:
        out = np.empty((count, cfg.height, cfg.width), np.uint8)
    for i in range(count):
        out[i] = gen_frame(cfg_name, first + i)
    return out


def random_image(seed: int, width: int, height: int, kind: str = "uniform") -> np.ndarray:
    """Fuzz inputs: 'uniform' bytes, 'binary' {0,255}, 'lowcontrast' [100,140]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "uniform":
        return rng.integers(0, 256, size=(height, width)).astype(np.uint8)
    if kind == "binary":
        return (rng.integers(0, 2, size=(height, width)) * 255).astype(np.uint8)
    if kind == "lowcontrast":
        return rng.integers(100, 141, size=(height, width)).astype(np.uint8)
    raise ValueError(kind)


def sha256(*arrays: np.ndarray) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
