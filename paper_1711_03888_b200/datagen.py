"""Seeded synthetic snapshots standing in for the paper's HACC / AMDF data.

The paper's 1.8 TB HACC and 34 GB AMDF snapshots are not
available, so BASELINE.json's config descriptions are realised by these
generators (DESIGN.md §7 records the parameters and the measured lag-1
autocorrelations).  Everything is generated in float64 and cast to float32
once; identical arrays feed the oracle and the GPU.

HACC-like (configs 0, 2, 3, 4): an ``Lx x Ly x Lz`` lattice with spacing
``s`` in a periodic box ``[0, s*L)``, emitted in lexicographic (x, y, z)
order, each coordinate plus N(0, 0.5) and wrapped; velocities are three
independent AR(1) series (rho 0.92, sigma 300) with a stationary start.

AMDF-like (configs 1, 3): uniform in ``[0, 100)^3`` emitted in spatial
cells of 64 particles (a power-of-two cell grid) visited in random cell
order; velocities i.i.d. N(0, 1).

Random streams are keyed by (seed, field, block) with 2^20-particle blocks,
so any contiguous particle range -- a multi-GPU shard -- is reproducible on
its own.  The AR(1) recursion restarts (stationary) at each block start.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

BLOCK = 1 << 20
RHO = 0.92
VEL_SIGMA = 300.0
DISP_SIGMA = 0.5


@dataclass(frozen=True)
class HaccSpec:
    lattice: Tuple[int, int, int]
    spacing: float
    seed: int = 20260808

    @property
    def n(self) -> int:
        return self.lattice[0] * self.lattice[1] * self.lattice[2]


@dataclass(frozen=True)
class AmdfSpec:
    n: int
    box: float = 100.0
    cell: int = 64
    seed: int = 20260808


CONFIGS = {
    # BASELINE.json configs[0..4]
    "C0": HaccSpec((100, 100, 100), 2.56),
    "C1": AmdfSpec(1 << 22),
    "C2": HaccSpec((640, 640, 640), 2.5),
    "C3-hacc": HaccSpec((512, 512, 256), 2.5),
    "C3-amdf": AmdfSpec(1 << 26),
    "C4": HaccSpec((1024, 1024, 1024), 2.5),
}


def _ar1_block(e: np.ndarray) -> np.ndarray:
    """v_0 = sigma*e_0, v_t = rho*v_{t-1} + sigma*sqrt(1-rho^2)*e_t."""
    from scipy.signal import lfilter
    c = VEL_SIGMA * np.sqrt(1.0 - RHO * RHO)
    zi = np.array([VEL_SIGMA * e[0] - c * e[0]])
    y, _ = lfilter([c], [1.0, -RHO], e, zi=zi)
    return y


def hacc_range(spec: HaccSpec, p0: int, p1: int,
               out: Optional[Sequence[np.ndarray]] = None) -> List[np.ndarray]:
    """Fields of particles [p0, p1) of the HACC-like lattice snapshot."""
    Lx, Ly, Lz = spec.lattice
    box = (spec.spacing * Lx, spec.spacing * Ly, spec.spacing * Lz)
    m = p1 - p0
    if out is None:
        out = [np.empty(m, np.float32) for _ in range(6)]
    b0 = p0 // BLOCK
    b1 = (p1 + BLOCK - 1) // BLOCK
    for b in range(b0, b1):
        lo = max(p0, b * BLOCK)
        hi = min(p1, (b + 1) * BLOCK)
        if hi <= lo:
            continue
        p = np.arange(b * BLOCK, (b + 1) * BLOCK, dtype=np.int64)
        idx = (p // (Ly * Lz), (p // Lz) % Ly, p % Lz)
        sl = slice(lo - b * BLOCK, hi - b * BLOCK)
        dst = slice(lo - p0, hi - p0)
        for t in range(3):
            rng = np.random.default_rng([spec.seed, t, b])
            disp = rng.normal(0.0, DISP_SIGMA, BLOCK)
            v = np.mod(spec.spacing * idx[t].astype(np.float64) + disp, box[t])
            out[t][dst] = v[sl].astype(np.float32)
        for t in range(3, 6):
            rng = np.random.default_rng([spec.seed, t, b])
            v = _ar1_block(rng.standard_normal(BLOCK))
            out[t][dst] = v[sl].astype(np.float32)
    return list(out)


def _cell_grid(ncell: int) -> Tuple[int, int, int]:
    lg = max(0, int(np.ceil(np.log2(max(ncell, 1)))))
    gx = 1 << ((lg + 2) // 3)
    gy = 1 << ((lg + 1) // 3)
    gz = 1 << (lg // 3)
    return gx, gy, gz


def amdf_range(spec: AmdfSpec, p0: int, p1: int,
               out: Optional[Sequence[np.ndarray]] = None) -> List[np.ndarray]:
    """Fields of particles [p0, p1) of the AMDF-like snapshot."""
    m = p1 - p0
    if out is None:
        out = [np.empty(m, np.float32) for _ in range(6)]
    ncell = (spec.n + spec.cell - 1) // spec.cell
    gx, gy, gz = _cell_grid(ncell)
    perm = np.random.default_rng([spec.seed, 99]).permutation(gx * gy * gz)[:ncell]
    csize = (spec.box / gx, spec.box / gy, spec.box / gz)
    b0 = p0 // BLOCK
    b1 = (p1 + BLOCK - 1) // BLOCK
    for b in range(b0, b1):
        lo = max(p0, b * BLOCK)
        hi = min(p1, (b + 1) * BLOCK)
        if hi <= lo:
            continue
        p = np.arange(b * BLOCK, (b + 1) * BLOCK, dtype=np.int64)
        cell = perm[np.minimum(p // spec.cell, ncell - 1)]
        cidx = (cell // (gy * gz), (cell // gz) % gy, cell % gz)
        sl = slice(lo - b * BLOCK, hi - b * BLOCK)
        dst = slice(lo - p0, hi - p0)
        for t in range(3):
            rng = np.random.default_rng([spec.seed, t, b])
            u = rng.random(BLOCK)
            v = np.minimum((cidx[t] + u) * csize[t], np.nextafter(spec.box, 0))
            out[t][dst] = v[sl].astype(np.float32)
        for t in range(3, 6):
            rng = np.random.default_rng([spec.seed, t, b])
            out[t][dst] = rng.standard_normal(BLOCK)[sl].astype(np.float32)
    return list(out)


def generate(spec, p0: int = 0, p1: Optional[int] = None,
             out: Optional[Sequence[np.ndarray]] = None) -> List[np.ndarray]:
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    if p1 is None:
        p1 = spec.n
    if isinstance(spec, HaccSpec):
        return hacc_range(spec, p0, p1, out)
    return amdf_range(spec, p0, p1, out)


def small_hacc(L: int, spacing: float = 2.56, seed: int = 20260808) -> List[np.ndarray]:
    return generate(HaccSpec((L, L, L), spacing, seed))


def small_amdf(n: int, seed: int = 20260808) -> List[np.ndarray]:
    return generate(AmdfSpec(n, seed=seed))


def lag1(x: np.ndarray) -> float:
    a = x[:-1].astype(np.float64)
    b = x[1:].astype(np.float64)
    a = a - a.mean()
    b = b - b.mean()
    return float((a * b).sum() / np.sqrt((a * a).sum() * (b * b).sum()))
