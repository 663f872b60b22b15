"""Seeded synthetic inputs for the BASELINE.json configs.

The paper's datasets (Sintel, KITTI, Middlebury) are not available; these
generators stand in for them with the shapes, sizes and value distributions
BASELINE.json describes.  numpy PCG64 + scipy.ndimage, deterministic for a
given seed.

frame1 : sum over sigma in (1, 2, 4, 8) of gaussian_filter(U(0,1)), min-max
         renormalised to [0, 255], float32
flow   : u, v = gaussian_filter(N(0,1), 40) scaled so max |flow| = maxmag,
         plus (configs 1-4) 3..6 axis-aligned rectangles of constant
         translation r*(cos a, sin a), r ~ U(0, rmax)
frame2 : bilinear backward warp of frame1 at (x - u, y - v) (the reference's
         numpy bilinear formula, core.py:154-170, clamped) + N(0, 2), float32
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np
from scipy.ndimage import gaussian_filter


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    batch: int
    patch_size: int
    overlap: float
    iterations: int
    finest_scale: int
    coarsest_scale: int
    maxmag: float
    rects: bool
    rmax: float
    stream: bool = False


# BASELINE.json configs[0..4]; coarsest scales per SURVEY Table S / App. A.4
CONFIGS = {
    "c0": Config("c0", 1024, 436, 1, 8, 0.30, 16, 3, 5, 20.0, False, 0.0),
    "c1": Config("c1", 1024, 436, 64, 8, 0.50, 32, 1, 5, 20.0, True, 30.0),
    "c2": Config("c2", 1024, 436, 16, 12, 0.75, 128, 0, 5, 40.0, True, 40.0),
    "c3": Config("c3", 1920, 1080, 256, 8, 0.50, 32, 1, 5, 20.0, True, 48.0),
    "c4": Config("c4", 3840, 2160, 31, 12, 0.75, 64, 1, 7, 64.0, True, 64.0, stream=True),
}


def dis_params(cfg: Config, outer_fixed: int | None = 1, coarsest: int | None = None):
    """DisParams for a config: refinement 1 outer / 5 inner (BASELINE)."""
    from paper_1603_03590_b200.params import DisParams, VarParams

    return DisParams(
        patch_size=cfg.patch_size, overlap=cfg.overlap, iterations=cfg.iterations,
        finest_scale=cfg.finest_scale,
        coarsest_scale=cfg.coarsest_scale if coarsest is None else coarsest,
        downscale=2, use_mean_normalization=True, residual_norm="l2",
        variational=VarParams(intensity_weight=5.0, gradient_weight=10.0,
                              smoothness_weight=10.0, inner_sor_iters=5,
                              penalizer_eps=1e-3, sor_omega=1.6,
                              outer_iters_fixed=outer_fixed),
    )


def _bilinear_map(img, xs, ys):
    """core.py:154-170 formula (clamped)."""
    h, w = img.shape
    x = np.clip(xs, 0.0, w - 1.0)
    y = np.clip(ys, 0.0, h - 1.0)
    x0 = np.floor(x).astype(np.int64)
    y0 = np.floor(y).astype(np.int64)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    fx = x - x0
    fy = y - y0
    top = img[y0, x0] * (1.0 - fx) + img[y0, x1] * fx
    bot = img[y1, x0] * (1.0 - fx) + img[y1, x1] * fx
    return top * (1.0 - fy) + bot * fy


def texture(rng, h, w):
    acc = np.zeros((h, w))
    for sigma in (1.0, 2.0, 4.0, 8.0):
        acc += gaussian_filter(rng.uniform(0.0, 1.0, (h, w)), sigma)
    lo, hi = acc.min(), acc.max()
    return ((acc - lo) * (255.0 / (hi - lo))).astype(np.float32)


def smooth_flow(rng, h, w, maxmag, sigma=40.0):
    u = gaussian_filter(rng.standard_normal((h, w)), sigma)
    v = gaussian_filter(rng.standard_normal((h, w)), sigma)
    scale = maxmag / np.hypot(u, v).max()
    return u * scale, v * scale


def add_rects(rng, u, v, rmax):
    h, w = u.shape
    for _ in range(int(rng.integers(3, 7))):
        bw = int(rng.integers(min(32, w // 4 - 1), max(w // 4, 33)))
        bh = int(rng.integers(min(32, h // 4 - 1), max(h // 4, 33)))
        bw = min(bw, w - 1)
        bh = min(bh, h - 1)
        x0 = int(rng.integers(0, w - bw))
        y0 = int(rng.integers(0, h - bh))
        r = rng.uniform(0.0, rmax)
        a = rng.uniform(0.0, 2.0 * math.pi)
        u[y0:y0 + bh, x0:x0 + bw] = r * math.cos(a)
        v[y0:y0 + bh, x0:x0 + bw] = r * math.sin(a)
    return u, v


def warp(frame, u, v):
    h, w = frame.shape
    xs, ys = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    return _bilinear_map(frame.astype(np.float64), xs - u, ys - v)


def make_pair(seed: int, h: int, w: int, maxmag: float, rects: bool, rmax: float):
    """One (frame1, frame2, gt_flow) triple; frames float32, flow float64."""
    rng = np.random.default_rng(seed)
    f1 = texture(rng, h, w)
    u, v = smooth_flow(rng, h, w, maxmag)
    if rects:
        u, v = add_rects(rng, u, v, rmax)
    f2 = warp(f1, u, v) + rng.normal(0.0, 2.0, (h, w))
    return f1, f2.astype(np.float32), np.stack([u, v], axis=-1)


def make_stereo_pair(seed: int, h: int, w: int, maxdisp: float, rects: bool = True):
    """A rectified pair for dis_stereo: frame2 = frame1 warped by a smooth
    horizontal displacement (plus fronto-parallel rectangles), v = 0, + N(0, 2).
    Returns (left, right, gt_u) with right(x + u(x)) ~ left(x)."""
    rng = np.random.default_rng(seed)
    f1 = texture(rng, h, w)
    u = gaussian_filter(rng.standard_normal((h, w)), 20.0)
    u *= maxdisp / max(1e-12, np.abs(u).max())
    if rects:
        for _ in range(int(rng.integers(2, 5))):
            bw = int(rng.integers(max(2, w // 8), max(3, w // 3)))
            bh = int(rng.integers(max(2, h // 8), max(3, h // 3)))
            x0 = int(rng.integers(0, w - bw))
            y0 = int(rng.integers(0, h - bh))
            u[y0:y0 + bh, x0:x0 + bw] = rng.uniform(-maxdisp, maxdisp)
    f2 = warp(f1, u, np.zeros_like(u)) + rng.normal(0.0, 2.0, (h, w))
    return f1, f2.astype(np.float32), u


def make_stream(seed: int, h: int, w: int, n_frames: int, maxmag: float, rmax: float):
    """c4: frames k+1 = warp(clean_k, flow_k) + N(0,2); flow_k blends two
    smooth fields (t = k/(n-1)) plus rectangles.  Returns (n, h, w) f32."""
    rng = np.random.default_rng(seed)
    clean = texture(rng, h, w).astype(np.float64)
    ua, va = smooth_flow(rng, h, w, maxmag)
    ub, vb = smooth_flow(rng, h, w, maxmag)
    u_r, v_r = add_rects(rng, np.zeros((h, w)), np.zeros((h, w)), rmax)
    mask = (u_r != 0) | (v_r != 0)
    frames = np.empty((n_frames, h, w), dtype=np.float32)
    frames[0] = (clean + rng.normal(0.0, 2.0, (h, w))).astype(np.float32)
    for k in range(1, n_frames):
        t = (k - 1) / max(1, n_frames - 2)
        u = (1 - t) * ua + t * ub
        v = (1 - t) * va + t * vb
        u = np.where(mask, u_r, u)
        v = np.where(mask, v_r, v)
        clean = warp(clean, u, v)
        frames[k] = (clean + rng.normal(0.0, 2.0, (h, w))).astype(np.float32)
    return frames


def make_batch(cfg: Config, seed: int = 0, count: int | None = None, first: int = 0,
               h: int | None = None, w: int | None = None):
    """Frames (B, H, W) float32 x2 for pairs [first, first+count) of a config
    (pair i uses seed + i)."""
    h = cfg.height if h is None else h
    w = cfg.width if w is None else w
    n = cfg.batch if count is None else count
    if cfg.stream:
        frames = make_stream(seed, h, w, first + n + 1, cfg.maxmag, cfg.rmax)
        return frames[first:first + n].copy(), frames[first + 1:first + n + 1].copy()
    f1 = np.empty((n, h, w), dtype=np.float32)
    f2 = np.empty((n, h, w), dtype=np.float32)
    for i in range(n):
        a, b, _ = make_pair(seed + first + i, h, w, cfg.maxmag, cfg.rects, cfg.rmax)
        f1[i] = a
        f2[i] = b
    return f1, f2
