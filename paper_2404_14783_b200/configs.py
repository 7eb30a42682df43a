"""Seeded synthetic inputs for the five BASELINE.json configs.

The paper's data (colour map image, CFD / Lorenz snapshots) is not available;
these generators reproduce the configs' SHAPES and value distributions.
Every random draw comes from the reference's counter RNG (rng.hpp) keyed by
data_seed = 1000 + config number, so any process (GPU, oracle) regenerates
identical inputs.  Matrices are built on the GPU (not timed) and returned as
(4, m, n) float64 CUDA tensors; `rows` selects a row shard.

Ambiguities resolved here: Psi is l x m; the C3 Rademacher
embedding uses the reference's +-1 (the BASELINE's 1/sqrt(4) factor is an
exact power-of-two scale that changes neither range(H) nor HX); "N(0, 1e-3)"
and "N(0, 1e-4)" are standard deviations; C5 amplitudes are 1/|k| and phase
speeds uniform in [0, 2*pi/50) per step.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import qlra as Q

MASK = (1 << 64) - 1
GOLDEN, SALT = 0x9E3779B97F4A7C15, 0xD1B54A32D192ED03


def _mix64(z):
    z &= MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def rng_key(seed):
    return _mix64(seed ^ SALT)


def substream_key(seed, idx):
    """CounterRng(seed).substream(idx).key() (rng.hpp:23-30)."""
    return _mix64(rng_key(seed) ^ _mix64(idx + SALT))


def uniforms(key, n, offset=0):
    """uniform_at(offset .. offset+n-1) of stream `key` (rng.hpp:32-39)."""
    c = np.arange(offset, offset + n, dtype=np.uint64)
    z = (np.uint64(key) + np.uint64(GOLDEN) * (c + np.uint64(1)))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    s: int
    l: int
    kind: int
    rangefinders: tuple

    @property
    def data_seed(self):
        return 1000 + int(self.name[1:])

    def flops(self):
        """Algorithmic sketch flops: 32 flop per qMAC (qmatrix.cpp:235-238)."""
        return 32.0 * self.m * self.n * (self.s + self.l)

    def a_bytes(self):
        return 32.0 * self.m * self.n


CONFIGS = {
    "C1": Config("C1", 1000, 800, 60, 120, Q.GAUSSIAN, (Q.PSEUDO_QR, Q.PSEUDO_SVD)),
    "C2": Config("C2", 8000, 6000, 100, 200, Q.GAUSSIAN, (Q.PSEUDO_QR, Q.PSEUDO_SVD)),
    "C3": Config("C3", 20000, 15000, 220, 440, Q.RADEMACHER, (Q.PSEUDO_QR,)),
    "C4": Config("C4", 31365, 27125, 500, 1000, Q.GAUSSIAN, (Q.PSEUDO_QR, Q.PSEUDO_SVD)),
    "C5": Config("C5", 2097152, 300, 40, 80, Q.GAUSSIAN, (Q.PSEUDO_QR, Q.PSEUDO_SVD)),
}


def _gauss(rows, cols, seed, r0=0, r1=None, ctx=None):
    spec = Q.TestMatrixSpec(Q.GAUSSIAN, rows, cols, seed, 1.0)
    return Q.gen_block(spec, r0, rows if r1 is None else r1, 0, cols, ctx)


def build_matrix(cfg: Config, rows: tuple | None = None, ctx=None) -> torch.Tensor:
    """A (or rows [r0, r1) of A) for config `cfg`, on the current CUDA device."""
    r0, r1 = rows if rows is not None else (0, cfg.m)
    ds = cfg.data_seed
    k1, k2, k3 = (substream_key(ds, i) for i in (1, 2, 3))
    if cfg.name in ("C1", "C2", "C3"):
        rank = {"C1": 50, "C2": 400, "C3": 200}[cfg.name]
        g1 = _gauss(cfg.m, rank, k1, r0, r1, ctx)
        g2 = _gauss(rank, cfg.n, k2, ctx=ctx)
        if cfg.name == "C2":
            sig = torch.arange(1, rank + 1, dtype=torch.float64, device=g1.device) ** -2.0
            g1 = g1 * sig[None, None, :]
        a = Q.qmat_mul(g1, g2, ctx=ctx)
        if cfg.name in ("C1", "C3"):
            a += (1e-3 if cfg.name == "C1" else 1e-6) * _gauss(cfg.m, cfg.n, k3, r0, r1, ctx)
        return a
    if cfg.name == "C4":
        return _image(cfg, r0, r1, ds, ctx)
    return _flow(cfg, r0, r1, ds, ctx)


def _image(cfg, r0, r1, ds, ctx):
    """Pure quaternion 'colour image': each of x, y, z is a sum of 64 random
    2-D sinusoids (f ~ U[0, 0.01] cycles/pixel, phase ~ U[0, 2pi)), min-max
    rescaled to [0, 1] over the FULL image, plus N(0, 1e-3) noise."""
    dev = torch.device("cuda", torch.cuda.current_device())
    a = torch.zeros((4, r1 - r0, cfg.n), dtype=torch.float64, device=dev)
    i = torch.arange(cfg.m, dtype=torch.float64, device=dev)
    j = torch.arange(cfg.n, dtype=torch.float64, device=dev)
    for ch in range(3):
        u = uniforms(substream_key(ds, 10 + ch), 3 * 64)
        fr, fc, ph = 0.01 * u[0::3], 0.01 * u[1::3], 2 * math.pi * u[2::3]
        fr, fc, ph = (torch.tensor(v, device=dev) for v in (fr, fc, ph))
        # sin(a_i + b_j) = sin a_i cos b_j + cos a_i sin b_j  -> rank-128 product
        ai = 2 * math.pi * i[:, None] * fr[None, :] + ph[None, :]
        bj = 2 * math.pi * j[:, None] * fc[None, :]
        left = torch.cat([torch.sin(ai), torch.cos(ai)], 1)
        right = torch.cat([torch.cos(bj), torch.sin(bj)], 1)
        # global min / max from the full image, computed blockwise
        lo, hi = math.inf, -math.inf
        for b0 in range(0, cfg.m, 4096):
            blk = left[b0:b0 + 4096] @ right.T
            lo, hi = min(lo, float(blk.min())), max(hi, float(blk.max()))
        plane = (left[r0:r1] @ right.T - lo) / (hi - lo)
        a[ch + 1] = plane
    noise = _gauss(cfg.m, cfg.n, substream_key(ds, 3), r0, r1, ctx)
    a[1:] += 1e-3 * noise[1:]
    return a


def _flow(cfg, r0, r1, ds, ctx):
    """3-D flow snapshots: rows = 128^3 grid (lexicographic), cols = time.
    w = scalar field, x/y/z = velocity; each a sum of 32 travelling Fourier
    modes a cos(2 pi k.p/128 - omega t + phi), k in {1..8}^3, plus N(0, 1e-4)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    g = 128
    idx = torch.arange(r0, r1, dtype=torch.int64, device=dev)
    p = torch.stack([idx // (g * g), (idx // g) % g, idx % g], 1).to(torch.float64)
    t = torch.arange(cfg.n, dtype=torch.float64, device=dev)
    a = torch.empty((4, r1 - r0, cfg.n), dtype=torch.float64, device=dev)
    for ch in range(4):
        u = uniforms(substream_key(ds, 20 + ch), 5 * 32)
        k = torch.tensor(np.floor(1 + 8 * u[:96]).reshape(32, 3), device=dev)
        ph = torch.tensor(2 * math.pi * u[96:128], device=dev)
        om = torch.tensor(2 * math.pi / 50 * u[128:160], device=dev)
        amp = 1.0 / torch.linalg.vector_norm(k, dim=1)
        theta = 2 * math.pi * (p @ k.T) / g + ph[None, :]
        left = torch.cat([torch.cos(theta) * amp, torch.sin(theta) * amp], 1)
        right = torch.cat([torch.cos(om[None, :] * t[:, None]), torch.sin(om[None, :] * t[:, None])], 1)
        a[ch] = left @ right.T
    a += 1e-4 * _gauss(cfg.m, cfg.n, substream_key(ds, 3), r0, r1, ctx)
    return a
