"""Seeded image generators and the BASELINE.json configuration table.

The constructions follow BASELINE.json `configs` (c1..c5); the parts BASELINE
leaves open are fixed as proposed in SURVEY.md §8(d) "Synthetic inputs" and
listed in DESIGN.md §"Input recipe".  Every image is generated in float64 with
numpy's PCG64 (`default_rng(seed)`) in a fixed draw order and returned as a
C-contiguous float32 array with values in [0, 255].

No bilateral-filter arithmetic lives here (this module is shared by the oracle
tests and the CUDA path, see the task's independence rule).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Config",
    "CONFIGS",
    "rect_ramp",
    "voronoi_texture",
    "checkerboard",
    "gradient",
    "config_image",
]


def rect_ramp(H: int, W: int, seed: int, n_rect: int = 16, noise: float = 10.0) -> np.ndarray:
    """c1/c4 construction (BASELINE.json configs[0], configs[3]).

    Background: left-to-right ramp 255*x/(W-1).  Then `n_rect` axis-aligned
    rectangles are painted in order; for each rectangle the draws are, in this
    order: height ~ U_int[H/16, H/4], width ~ U_int[W/16, W/4], top ~ U_int over
    valid rows, left ~ U_int over valid columns, value ~ U[0, 255].  Finally
    i.i.d. N(0, noise^2) is added and the result is clipped to [0, 255].
    """
    rng = np.random.default_rng(seed)
    x = np.arange(W, dtype=np.float64)
    img = np.empty((H, W), dtype=np.float64)
    img[:] = 255.0 * x / max(W - 1, 1)
    for _ in range(n_rect):
        h = int(rng.integers(max(H // 16, 1), max(H // 4, 1), endpoint=True))
        w = int(rng.integers(max(W // 16, 1), max(W // 4, 1), endpoint=True))
        top = int(rng.integers(0, H - h, endpoint=True))
        left = int(rng.integers(0, W - w, endpoint=True))
        val = float(rng.uniform(0.0, 255.0))
        img[top:top + h, left:left + w] = val
    img += rng.normal(0.0, noise, size=(H, W))
    np.clip(img, 0.0, 255.0, out=img)
    return np.ascontiguousarray(img.astype(np.float32))


VORONOI_CHUNK = 256   # rows per noise chunk (part of the recipe: chunk k's noise has its own stream)


def voronoi_texture(H: int, W: int, seed: int, n_seeds: int, noise: float,
                    amp: float = 20.0, lam: float = 16.0, theta: float = math.pi / 6,
                    rows: tuple | None = None) -> np.ndarray:
    """c2/c3/c5 construction (BASELINE.json configs[1], [2], [4]).

    Draw order: seed x ~ U[0, W) (n_seeds), seed y ~ U[0, H) (n_seeds), cell
    value ~ U[0, 255] (n_seeds), all from default_rng(seed).  Each pixel (x, y) takes the
    value of the seed nearest (Euclidean) to its centre (x+0.5, y+0.5); texture
    amp*sin(2*pi*(x cos(theta) + y sin(theta))/lam) is added (amp=0 disables it), then
    noise N(0, noise^2), then clip to [0, 255].  The noise of row chunk k (rows
    [256k, 256k+256)) is drawn from its own stream default_rng([seed, 1, k]), so any row
    range can be generated on its own (rows=(r0, r1): rows r0..r1-1 of the H x W image,
    identical to the same rows of the whole image) — each rank of the row-band bench
    generates only its band and halos.
    """
    from scipy.spatial import cKDTree

    r0, r1 = (0, H) if rows is None else (max(0, int(rows[0])), min(H, int(rows[1])))
    rng = np.random.default_rng(seed)
    sx = rng.uniform(0.0, W, size=n_seeds)
    sy = rng.uniform(0.0, H, size=n_seeds)
    val = rng.uniform(0.0, 255.0, size=n_seeds)
    tree = cKDTree(np.stack([sx, sy], axis=1))
    out = np.empty((max(0, r1 - r0), W), dtype=np.float32)
    xs = np.arange(W, dtype=np.float64)
    ct, st = math.cos(theta), math.sin(theta)
    C = VORONOI_CHUNK
    for k in range(r0 // C, (r1 + C - 1) // C):
        c0, c1 = k * C, min(H, (k + 1) * C)
        nrng = np.random.default_rng([seed, 1, k])
        nz = nrng.normal(0.0, noise, size=(c1 - c0, W))
        a, b = max(c0, r0), min(c1, r1)             # rows of this chunk that are wanted
        ys = np.arange(a, b, dtype=np.float64)
        X, Y = np.meshgrid(xs, ys)
        pts = np.stack([(X + 0.5).ravel(), (Y + 0.5).ravel()], axis=1)
        _, idx = tree.query(pts, k=1, workers=-1)
        blk = val[idx].reshape(b - a, W)
        if amp != 0.0:
            blk = blk + amp * np.sin(2.0 * math.pi * (X * ct + Y * st) / lam)
        blk = blk + nz[a - c0:b - c0]
        np.clip(blk, 0.0, 255.0, out=blk)
        out[a - r0:b - r0] = blk.astype(np.float32)
    return out


def checkerboard(H: int, W: int, tile: int, lo: float = 0.0, hi: float = 255.0) -> np.ndarray:
    """Two-level checkerboard, top-left tile = lo."""
    y, x = np.mgrid[0:H, 0:W]
    img = np.where(((y // tile) + (x // tile)) % 2 == 0, lo, hi)
    return np.ascontiguousarray(img.astype(np.float32))


def gradient(H: int, W: int, lo: float = 0.0, hi: float = 255.0) -> np.ndarray:
    """Left-to-right linear ramp lo..hi."""
    x = np.arange(W, dtype=np.float64)
    row = lo + (hi - lo) * x / max(W - 1, 1)
    return np.ascontiguousarray(np.broadcast_to(row, (H, W)).astype(np.float32))


@dataclass(frozen=True)
class Config:
    """One BASELINE.json workload.

    sigma_r is the stated value; sigma_r_twin is the parity-gate twin of
    SURVEY.md §8(c)-Q1 (same image, sigma_s and N, so the same hot-path work).
    """
    name: str
    H: int
    W: int
    batch: int
    sigma_s: tuple
    sigma_r: float
    N: int
    sigma_r_twin: float
    kind: str
    gen: dict = field(default_factory=dict)
    seed: int = 0


CONFIGS = {
    "c1": Config("c1", 256, 256, 1, (3.0,), 30.0, 5, 100.0, "rect",
                 dict(n_rect=16, noise=10.0), seed=1),
    "c2": Config("c2", 1024, 1024, 1, (5.0,), 20.0, 8, 70.0, "voronoi",
                 dict(n_seeds=200, noise=15.0, amp=20.0), seed=2),
    "c3": Config("c3", 4096, 4096, 1, (2.0, 5.0, 10.0, 20.0, 40.0), 15.0, 10, 60.0, "voronoi",
                 dict(n_seeds=2000, noise=20.0, amp=20.0), seed=3),
    "c4": Config("c4", 1024, 1024, 256, (4.0,), 25.0, 6, 85.0, "rect",
                 dict(n_rect=16, noise=10.0), seed=1000),
    "c5": Config("c5", 16384, 16384, 1, (16.0,), 10.0, 12, 55.0, "voronoi",
                 dict(n_seeds=20000, noise=10.0, amp=0.0), seed=5),
}


def config_image(cfg: Config | str, index: int = 0, H: int | None = None, W: int | None = None,
                 rows: tuple | None = None) -> np.ndarray:
    """Image `index` of config `cfg` (batch configs use seed cfg.seed + index).

    H/W override the size (same construction, used for reduced-size parity
    cases); the Voronoi seed count is scaled with the area so the cell size
    stays that of the full config.  rows=(r0, r1) returns only those rows of the
    image (Voronoi constructions generate just them; the others slice).
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    H = cfg.H if H is None else H
    W = cfg.W if W is None else W
    seed = cfg.seed + index
    g = dict(cfg.gen)
    if cfg.kind == "rect":
        img = rect_ramp(H, W, seed, **g)
        return img if rows is None else np.ascontiguousarray(img[max(0, rows[0]):rows[1]])
    if cfg.kind == "voronoi":
        if (H, W) != (cfg.H, cfg.W):
            g["n_seeds"] = max(1, int(round(g["n_seeds"] * H * W / (cfg.H * cfg.W))))
        return voronoi_texture(H, W, seed, rows=rows, **g)
    raise ValueError(cfg.kind)
