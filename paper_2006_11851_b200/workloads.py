"""Seeded synthetic inputs of the BASELINE.json configs (numpy only).

The reference measures on exemplar photographs that are not available
(/examples/ is git-ignored upstream, proj/.gitignore:1), and BASELINE.json
specifies synthetic generators instead.  Everything here is deterministic
(numpy PCG64) and shared bit-for-bit by the GPU path, the oracle and bench.

Coordinates: row 0 = bottom (image.hpp:11-12).  "Top row" = row H-1.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["sinusoid_exemplar", "guidance_planes", "rgbs_planes", "init_output", "CONFIGS",
           "StageSpec", "WorkloadConfig", "gaussian_mixture", "splitmix64", "stage_inputs"]


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = (np.asarray(x, np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def sinusoid_exemplar(size: int, n_sin: int, ramp: float, seed: int,
                      lum_gain: bool = False) -> np.ndarray:
    """uint8 RGB (3, size, size): sum of n_sin random-orientation sinusoids,
    frequency 2..12 cycles/image, scaled linearly from 1x at the top row to
    `ramp`x at the bottom row (perspective), plus uniform noise +-16; optional
    per-row luminance gain 0.5 (bottom) .. 1.0 (top) (config 4)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    theta = rng.uniform(0.0, 2.0 * np.pi, n_sin)
    freq = rng.uniform(2.0, 12.0, n_sin)
    phase = rng.uniform(0.0, 2.0 * np.pi, n_sin)
    color = rng.uniform(0.4, 1.0, (n_sin, 3))
    y, x = np.mgrid[0:size, 0:size].astype(np.float64)
    # row 0 = bottom: top row (y = size-1) has scale 1, bottom row has `ramp`
    scale = 1.0 + (ramp - 1.0) * (size - 1 - y) / max(size - 1, 1)
    acc = np.zeros((3, size, size))
    amp = 110.0 / np.sqrt(n_sin)
    for k in range(n_sin):
        u = (x * np.cos(theta[k]) + y * np.sin(theta[k])) / size
        wave = np.cos(2.0 * np.pi * freq[k] * scale * u + phase[k])
        acc += amp * color[k][:, None, None] * wave[None]
    img = 128.0 + acc + rng.uniform(-16.0, 16.0, (3, size, size))
    if lum_gain:
        gain = 0.5 + 0.5 * y / max(size - 1, 1)
        img = 128.0 + (img - 128.0) * gain[None] - 64.0 * (1.0 - gain[None])
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def guidance_planes(W: int, H: int, G: int) -> np.ndarray:
    """G guidance planes (G, H, W) as fp32-then-fp64 ramps: even g = row ramp
    y/(H-1), odd g = column ramp x/(W-1) (matches the driver's ramp_planes)."""
    out = np.zeros((G, H, W))
    ys = (np.arange(H, dtype=np.float32) / np.float32(max(H - 1, 1))).astype(np.float64)
    xs = (np.arange(W, dtype=np.float32) / np.float32(max(W - 1, 1))).astype(np.float64)
    if H == 1:
        ys[:] = 0.5
    if W == 1:
        xs[:] = 0.5
    for g in range(G):
        out[g] = ys[:, None] if g % 2 == 0 else xs[None, :]
    return out


def rgbs_planes(rgb_u8: np.ndarray, G: int) -> np.ndarray:
    """(3+G, H, W) fp64 state: RGB / 255 plus guidance ramps."""
    _, H, W = rgb_u8.shape
    return np.concatenate([rgb_u8.astype(np.float64) / 255.0, guidance_planes(W, H, G)], 0)


def init_output(ex_planes: np.ndarray, W: int, H: int, G: int, seed: int) -> np.ndarray:
    """Scale-matched seeded copy (the driver's rule): output pixel i takes the
    RGB of exemplar pixel (splitmix64(seed ^ i) % ew, round(s_row * (eh-1)))."""
    C, eh, ew = ex_planes.shape
    og = guidance_planes(W, H, G)
    i = np.arange(W * H, dtype=np.uint64)
    ex = (splitmix64(np.uint64(seed) ^ i) % np.uint64(ew)).astype(np.int64)
    s = np.clip(og[0].reshape(-1), 0.0, 1.0)
    ey = np.floor(s * (eh - 1) + 0.5).astype(np.int64)  # lround for non-negative values
    out = np.zeros((3 + G, H, W))
    for c in range(3):
        out[c] = ex_planes[c][ey, ex].reshape(H, W)
    out[3:] = og
    return out


def gaussian_mixture(n: int, D: int, k: int, sigma: float, seed: int,
                     means: np.ndarray | None = None):
    """Config 2: n float32 vectors from k isotropic Gaussians (means U[0,255]^D)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if means is None:
        means = np.random.Generator(np.random.PCG64(1234)).uniform(0.0, 255.0, (k, D))
    comp = rng.integers(0, k, n)
    X = means[comp] + rng.normal(0.0, sigma, (n, D))
    return X.astype(np.float32)


@dataclass
class StageSpec:
    sizes: tuple = (8,)


@dataclass
class WorkloadConfig:
    name: str
    ex_size: int
    n_sin: int
    ramp: float
    G: int
    out: int
    levels: int
    sizes: tuple
    d_fixed: int = 0
    d_cap: int = 0
    branching: int = 4
    depth: int = 3
    iterations: int = 5
    spacing_rule: str = "w/4"
    lum_gain: bool = False
    seed: int = 1
    extra: dict = field(default_factory=dict)


CONFIGS = {
    0: WorkloadConfig("cfg0-pr1-ref", 64, 8, 2.0, 1, 128, 1, (8,), d_fixed=16, branching=4,
                      depth=3, iterations=5, spacing_rule="4"),
    1: WorkloadConfig("cfg1-multires", 128, 16, 2.0, 1, 256, 3, (32, 16, 8), d_cap=32,
                      branching=8, depth=3, iterations=5),
    3: WorkloadConfig("cfg3-1024-perspective", 256, 32, 3.0, 2, 1024, 3, (32, 16, 8),
                      d_fixed=32, branching=8, depth=4, iterations=10),
    4: WorkloadConfig("cfg4-4096-stress", 512, 32, 3.0, 2, 4096, 4, (32, 16, 8), d_fixed=48,
                      branching=16, depth=3, iterations=10, lum_gain=True),
}


def stage_inputs(cfg: WorkloadConfig, level: int, w: int, G: int | None = None):
    """Exemplar level planes, output dims and init for one stage, built the
    way the driver builds them (block-mean pyramid, ramps re-imposed)."""
    G = cfg.G if G is None else G
    rgb = sinusoid_exemplar(cfg.ex_size, cfg.n_sin, cfg.ramp, cfg.seed, cfg.lum_gain)
    f = 1 << (cfg.levels - 1 - level)
    ex = rgb.astype(np.float64) / 255.0
    if f > 1:
        eh, ew = ex.shape[1] // f, ex.shape[2] // f
        ex = ex[:, : eh * f, : ew * f].reshape(3, eh, f, ew, f)
        # block mean in the reference's order is checked separately; here a
        # plain mean is only used to make stage inputs
        ex = ex.mean(axis=(2, 4))
    _, eh, ew = ex.shape
    planes = np.concatenate([ex, guidance_planes(ew, eh, G)], 0)
    W = H = cfg.out >> (cfg.levels - 1 - level)
    init = init_output(planes, W, H, G, cfg.seed)
    sp = 4 if cfg.spacing_rule == "4" else max(1, w // 4)
    return planes, init, W, H, sp
