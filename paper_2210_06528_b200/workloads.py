"""BASELINE.json configurations and their seeded synthetic input fields.

The reference ships its own normalized-sinc generators (field.cpp:39-64); the
BASELINE configs instead name sin(x)/x, radial sin(r)/r and a combustion-
shaped field.  These generators produce ONE host/device buffer
that is fed identically to the GPU path and to the CPU checkers.  The S3D
dataset is not available here: C4 is a seeded synthetic field with S3D's
704x540x550 shape.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

FOUR_PI = 4.0 * math.pi
C4_SEED = 20221012  # recorded in every bench line


@dataclass(frozen=True)
class Config:
    name: str
    grid: Tuple[int, ...]
    blocks: Tuple[int, ...]
    degree: int
    nctrl: Tuple[int, ...]
    overlap: int
    generator: str
    tolerance: float = 1e-10
    max_iters: int = 20

    @property
    def rank(self):
        return len(self.grid)

    @property
    def bounds(self) -> List[Tuple[float, float]]:
        return [(-FOUR_PI, FOUR_PI)] * self.rank if self.generator != "combustion" else \
            [(0.0, float(g - 1)) for g in self.grid]

    @property
    def points(self) -> int:
        return int(np.prod(self.grid))


CONFIGS = {
    "C1": Config("C1", (10000,), (4,), 3, (64,), 3, "sinc1d"),
    "C2": Config("C2", (1024, 1024), (4, 4), 3, (64, 64), 3, "sinc_radial"),
    "C3": Config("C3", (256, 256, 256), (4, 4, 4), 3, (32, 32, 32), 3, "sinc_radial"),
    # overlap for C4 is not stated in BASELINE.json: delta = p assumed (SURVEY §8 note)
    "C4": Config("C4", (704, 540, 550), (8, 8, 8), 4, (24, 24, 24), 4, "combustion"),
    "C5": Config("C5", (8192, 8192), (16, 16), 5, (128, 128), 5, "sinc_radial"),
}


def scaled(cfg: Config, grid, nctrl, name=None) -> Config:
    """Same shape/degree/overlap family at a smaller size (parity tests)."""
    return Config(name or cfg.name + "-small", tuple(grid), cfg.blocks, cfg.degree, tuple(nctrl), cfg.overlap,
                  cfg.generator, cfg.tolerance, cfg.max_iters)


def weak(cfg: Config, n: int) -> Config:
    """Weak scaling over n GPUs: n times the grid and the block rows along
    axis 0 (same per-block shape), so each rank's block slab is one `cfg`."""
    if n == 1:
        return cfg
    return Config(f"{cfg.name}x{n}", (cfg.grid[0] * n,) + tuple(cfg.grid[1:]), (cfg.blocks[0] * n,) + tuple(cfg.blocks[1:]),
                  cfg.degree, cfg.nctrl, cfg.overlap, cfg.generator, cfg.tolerance, cfg.max_iters)


def _axes(cfg: Config, xp):
    return [xp.linspace(a, b, n, dtype=xp.float64) if xp is np else
            xp.linspace(a, b, n, dtype=xp.float64, device="cuda") for (a, b), n in zip(cfg.bounds, cfg.grid)]


def _sinc(r, xp):
    out = xp.sin(r) / xp.where(r == 0, 1.0, r)
    return xp.where(r == 0, 1.0, out)


def combustion_params(cfg: Config, seed: int = C4_SEED):
    """64 anisotropic Gaussian blobs + 8 low-frequency modes."""
    rng = np.random.default_rng(seed)
    g = np.array(cfg.grid, np.float64)
    blobs = dict(center=rng.uniform(0, 1, (64, cfg.rank)) * (g - 1), sigma=rng.uniform(2, 40, (64, cfg.rank)),
                 amp=rng.uniform(0.1, 1.0, 64))
    modes = dict(freq=rng.integers(1, 4, (8, cfg.rank)).astype(np.float64), phase=rng.uniform(0, 2 * math.pi, 8),
                 amp=rng.uniform(0.05, 0.2, 8))
    return blobs, modes


def make_field_numpy(cfg: Config, seed: int = C4_SEED) -> np.ndarray:
    """Host generator (used for small test sizes)."""
    ax = _axes(cfg, np)
    if cfg.generator == "sinc1d":
        return _sinc(ax[0], np)
    if cfg.generator == "sinc_radial":
        mesh = np.meshgrid(*ax, indexing="ij")
        return _sinc(np.sqrt(sum(m * m for m in mesh)), np)
    if cfg.generator == "combustion":
        return _combustion(cfg, seed, np, ax)
    raise ValueError(cfg.generator)


def _combustion(cfg, seed, xp, ax):
    blobs, modes = combustion_params(cfg, seed)
    shape = cfg.grid
    f = xp.zeros(shape, dtype=xp.float64) if xp is np else xp.zeros(shape, dtype=xp.float64, device="cuda")
    for i in range(64):
        fac = None
        for k in range(cfg.rank):
            g1 = xp.exp(-0.5 * ((ax[k] - float(blobs["center"][i, k])) / float(blobs["sigma"][i, k])) ** 2)
            sh = [1] * cfg.rank
            sh[k] = -1
            g1 = g1.reshape(sh)
            fac = g1 if fac is None else fac * g1
        f += float(blobs["amp"][i]) * fac
    for i in range(8):
        arg = None
        for k in range(cfg.rank):
            a1 = (2 * math.pi * float(modes["freq"][i, k]) / (cfg.grid[k] - 1)) * ax[k]
            sh = [1] * cfg.rank
            sh[k] = -1
            a1 = a1.reshape(sh)
            arg = a1 if arg is None else arg + a1
        f += float(modes["amp"][i]) * xp.sin(arg + float(modes["phase"][i]))
    std = float(f.std())
    if xp is np:
        noise = np.random.default_rng(seed + 1).standard_normal(shape)
    else:
        import torch
        gen = torch.Generator(device="cuda").manual_seed(seed + 1)
        noise = torch.randn(shape, generator=gen, dtype=torch.float64, device="cuda")
    f += (0.01 * std) * noise
    return f


def make_field_torch(cfg: Config, seed: int = C4_SEED):
    """Device generator (bench sizes).  Returns a contiguous CUDA float64 tensor."""
    import torch
    ax = _axes(cfg, torch)
    if cfg.generator == "sinc1d":
        return _sinc(ax[0], torch).contiguous()
    if cfg.generator == "sinc_radial":
        r2 = None
        for k, a in enumerate(ax):
            sh = [1] * cfg.rank
            sh[k] = -1
            t = (a * a).reshape(sh)
            r2 = t if r2 is None else r2 + t
        return _sinc(torch.sqrt(r2), torch).contiguous()
    if cfg.generator == "combustion":
        return _combustion(cfg, seed, torch, ax).contiguous()
    raise ValueError(cfg.generator)


def algorithmic_bytes(cfg: Config, dec, epochs_exchanged: int, store_error: bool = True) -> dict:
    """B = 8(sum|Q_loc| + prod M + 2 sum|P_held|) + 16 E sum n_s (+ 8 prod M for the error field)."""
    bd = dec.block_dims_array()
    q_loc = int(sum(np.prod(bd[b, :, 13] - bd[b, :, 12]) for b in range(dec.nblocks)))
    p_held = int(sum(np.prod(bd[b, :, 9] - bd[b, :, 8]) for b in range(dec.nblocks)))
    ns_total = 0
    hr = [dec._holder_ranges(k) for k in range(dec.rank)]
    sizes = [(h[:, 1] - h[:, 0] + 1).astype(np.int64) for h in hr]
    prod = sizes[0]
    for s in sizes[1:]:
        prod = np.multiply.outer(prod, s)
    ns_total = int(prod[prod > 1].sum())
    M = cfg.points
    b = 8 * (q_loc + M + 2 * p_held) + 16 * epochs_exchanged * ns_total + (8 * M if store_error else 0)
    return dict(bytes=b, q_loc=q_loc, p_held=p_held, ns_total=ns_total, points=M)
