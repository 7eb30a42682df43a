"""CPU side of the benchmark -- TEST / BASELINE INFRASTRUCTURE ONLY.

The BASELINE configs C1-C5 regenerated on the host (numpy + the oracle's
counter-RNG generator) and the two CPU timing legs of bench.py:

* `reference_step`: the reference's CPU path (the oracle restatement,
  oracle/qlra_oracle.cpp) on all host threads -- `bench.py --impl reference`;
* `cpu_baseline`: the same on ONE pinned core (taskset, OPENBLAS_NUM_THREADS=1)
  -- the repo arm's `cpu_baseline` object.

Only bench.py's CPU legs and tests/ import this module; the product package
never does.  Nothing here touches the GPU.

The C4 / C5 generators mirror paper_2404_14783_b200/configs.py (_image,
_flow): the same RNG draws (reference counter RNG keyed by data_seed =
1000 + config number), the same formulas, evaluated with numpy/OpenBLAS
instead of torch/cuBLAS, so values agree to rounding (not bitwise).
"""
from __future__ import annotations

import math
import os
import time

import numpy as np

from oracle import oracle as O

MASK = (1 << 64) - 1
GOLDEN, SALT = 0x9E3779B97F4A7C15, 0xD1B54A32D192ED03


def _mix64(z):
    z &= MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def substream_key(seed, idx):
    """CounterRng(seed).substream(idx).key() (rng.hpp:23-30)."""
    return _mix64(_mix64(seed ^ SALT) ^ _mix64(idx + SALT))


def uniforms(key, n, offset=0):
    """uniform_at(offset .. offset+n-1) of stream `key` (rng.hpp:32-39)."""
    c = np.arange(offset, offset + n, dtype=np.uint64)
    z = (np.uint64(key) + np.uint64(GOLDEN) * (c + np.uint64(1)))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


# (name, m, n, s, l, kind) -- BASELINE.json configs
SHAPES = {
    "C1": (1000, 800, 60, 120, O.GAUSSIAN),
    "C2": (8000, 6000, 100, 200, O.GAUSSIAN),
    "C3": (20000, 15000, 220, 440, O.RADEMACHER),
    "C4": (31365, 27125, 500, 1000, O.GAUSSIAN),
    "C5": (2097152, 300, 40, 80, O.GAUSSIAN),
}


class Workload:
    def __init__(self, name):
        self.name = name
        self.m, self.n, self.s, self.l, self.kind = SHAPES[name]
        self.data_seed = 1000 + int(name[1:])
        self._image_ext = None

    def flops(self):
        return 32.0 * self.m * self.n * (self.s + self.l)

    # -------------------------------------------------------- matrix ---
    def rows(self, r0, r1, nthreads):
        """Rows [r0, r1) of the config's A, (4, r1 - r0, n) float64."""
        ds = self.data_seed
        if self.name in ("C1", "C2", "C3"):
            rank = {"C1": 50, "C2": 400, "C3": 200}[self.name]
            g1 = O.gen_block(O.GAUSSIAN, self.m, rank, substream_key(ds, 1), r0, r1, 0, rank,
                             nthreads=nthreads)
            g2 = O.gen_test_matrix(O.GAUSSIAN, rank, self.n, substream_key(ds, 2), nthreads=nthreads)
            if self.name == "C2":
                g1 = g1 * (np.arange(1, rank + 1, dtype=np.float64) ** -2.0)[None, None, :]
            a = O.qmat_mul(g1, g2)
            if self.name in ("C1", "C3"):
                a += (1e-3 if self.name == "C1" else 1e-6) * O.gen_block(
                    O.GAUSSIAN, self.m, self.n, substream_key(ds, 3), r0, r1, 0, self.n, nthreads=nthreads)
            return a
        if self.name == "C4":
            return self._image_rows(r0, r1, nthreads)
        return self._flow_rows(r0, r1, nthreads)

    def _image_factors(self, ch):
        u = uniforms(substream_key(self.data_seed, 10 + ch), 3 * 64)
        fr, fc, ph = 0.01 * u[0::3], 0.01 * u[1::3], 2 * math.pi * u[2::3]
        i = np.arange(self.m, dtype=np.float64)
        j = np.arange(self.n, dtype=np.float64)
        ai = 2 * math.pi * i[:, None] * fr[None, :] + ph[None, :]
        bj = 2 * math.pi * j[:, None] * fc[None, :]
        left = np.concatenate([np.sin(ai), np.cos(ai)], 1)
        right = np.concatenate([np.cos(bj), np.sin(bj)], 1)
        return left, right

    def _image_rows(self, r0, r1, nthreads):
        """configs._image: x, y, z = sum of 64 random 2-D sinusoids, min-max
        rescaled over the FULL image to [0, 1], + 1e-3 N(0, 1); w = 0."""
        if self._image_ext is None:
            ext = []
            for ch in range(3):
                left, right = self._image_factors(ch)
                lo, hi = math.inf, -math.inf
                for b0 in range(0, self.m, 4096):
                    blk = left[b0:b0 + 4096] @ right.T
                    lo, hi = min(lo, float(blk.min())), max(hi, float(blk.max()))
                ext.append((lo, hi))
            self._image_ext = ext
        a = np.zeros((4, r1 - r0, self.n))
        for ch in range(3):
            left, right = self._image_factors(ch)
            lo, hi = self._image_ext[ch]
            a[ch + 1] = (left[r0:r1] @ right.T - lo) / (hi - lo)
        noise = O.gen_block(O.GAUSSIAN, self.m, self.n, substream_key(self.data_seed, 3), r0, r1, 0, self.n,
                            nthreads=nthreads)
        a[1:] += 1e-3 * noise[1:]
        return a

    def _flow_rows(self, r0, r1, nthreads):
        """configs._flow: rows = 128^3 grid, cols = time; each plane a sum of
        32 travelling Fourier modes + 1e-4 N(0, 1)."""
        g = 128
        idx = np.arange(r0, r1, dtype=np.int64)
        p = np.stack([idx // (g * g), (idx // g) % g, idx % g], 1).astype(np.float64)
        t = np.arange(self.n, dtype=np.float64)
        a = np.empty((4, r1 - r0, self.n))
        for ch in range(4):
            u = uniforms(substream_key(self.data_seed, 20 + ch), 5 * 32)
            k = np.floor(1 + 8 * u[:96]).reshape(32, 3)
            ph = 2 * math.pi * u[96:128]
            om = 2 * math.pi / 50 * u[128:160]
            amp = 1.0 / np.linalg.norm(k, axis=1)
            theta = 2 * math.pi * (p @ k.T) / g + ph[None, :]
            left = np.concatenate([np.cos(theta) * amp, np.sin(theta) * amp], 1)
            right = np.concatenate([np.cos(om[None, :] * t[:, None]), np.sin(om[None, :] * t[:, None])], 1)
            a[ch] = left @ right.T
        a += 1e-4 * O.gen_block(O.GAUSSIAN, self.m, self.n, substream_key(self.data_seed, 3), r0, r1, 0, self.n,
                                nthreads=nthreads)
        return a

    # -------------------------------------------------------- sketch ---
    def blas_sketch(self, nthreads, block=4096):
        """Full-size Y = A Omega, W = Psi A through the oracle's plane GEMMs
        (qmat_mul, qmatrix.cpp:165-197: OpenBLAS dgemm), A generated and
        consumed in row blocks -- the INPUTS of the timed QB stage (the
        reference's own ordered sketch of C4 is ~41 TFLOP of scalar work)."""
        om = O.gen_test_matrix(self.kind, self.n, self.s, 1, nthreads=nthreads)
        y = np.zeros((4, self.m, self.s))
        w = np.zeros((4, self.l, self.n))
        for r0 in range(0, self.m, block):
            r1 = min(self.m, r0 + block)
            a = self.rows(r0, r1, nthreads)
            y[:, r0:r1] = O.qmat_mul(a, om)
            ps = O.gen_block(self.kind, self.l, self.m, 2, 0, self.l, r0, r1, nthreads=nthreads)
            w += O.qmat_mul(ps, a)
        return y, w


def sketch_sample_time(wl: Workload, a_rows, nthreads):
    """The reference's ordered sketch (sketch_update_rows,
    sketching.cpp:125-139 -> qmat_mul_accumulate_ordered) on a leading row
    block, extrapolated linearly to all m rows (the per-row cost of the
    ordered kernel is exactly constant).  Returns (seconds for A, rows)."""
    b = a_rows.shape[1]
    ys = np.zeros((4, wl.m, wl.s))
    ws = np.zeros((4, wl.l, wl.n))
    t0 = time.perf_counter()
    O.sketch_update_rows(ys, ws, 0, a_rows, 1, 2, wl.kind, 1.0, nthreads)
    return (time.perf_counter() - t0) * wl.m / b, b


def sample_rows(wl: Workload, nthreads, seconds):
    """Rows of serial ordered-sketch work taking ~`seconds` on `nthreads`
    threads (~2.5 GFLOP/s per thread for the scalar kernel)."""
    per_row = 32.0 * wl.n * (wl.s + wl.l)
    return int(max(8, min(wl.m, seconds * 2.5e9 * nthreads / per_row)))


def qb_stage_time(wl: Workload, y, w, method, nthreads):
    qb = O.qb_stage(y, w, 2, method, kind=wl.kind, nthreads=nthreads)
    return qb["rangefinder_s"] + qb["solve_s"], qb


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1
