"""Seeded synthetic inputs (BASELINE.json configs) -- no method arithmetic here.

Initial condition recipe (BASELINE.json ``configs[0]``, restated):
  * uniform cell-centred grid on [0,1]^2, ``nx`` x ``ny`` cells, cell centre
    (x_i, y_j) = ((i+1/2)/nx, (j+1/2)/ny);
  * phi_n = 0.3 where y < 0.2 (base layer) or inside the semicircular
    protrusion of radius 0.1 centred at (0.5, 0.2); 1e-3 elsewhere; plus seeded
    uniform noise in [-1e-3, +1e-3];
  * u = v = 0 (the shear forcing enters through the top-wall boundary value),
    p = 0, c = 1 everywhere.

The noise is drawn from numpy's PCG64 stream in row-major order (row j, then
column i).  ``rows=(j0, j1)`` returns the slab j0 <= j < j1 of the very same
global field by advancing the stream, so a slab decomposition sees exactly the
bits a single rank sees (decomposition invisibility of the inputs).

Array convention everywhere in this repo: shape (ny, nx), index [j, i],
x (i) contiguous.  Staggered velocities use the same (ny, nx) shape:
u[j, i] lives on the x-face x = i/nx, y = (j+1/2)/ny;
v[j, i] lives on the y-face x = (i+1/2)/nx, y = j/ny  (v[0, :] is the wall).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class GridSpec:
    nx: int
    ny: int

    @property
    def hx(self) -> float:
        return 1.0 / self.nx

    @property
    def hy(self) -> float:
        return 1.0 / self.ny


# BASELINE.json configs, by index.  (nx, ny, steps, dt)
CONFIGS = {
    0: dict(name="64x64_1step", nx=64, ny=64, steps=1, dt=1e-4),
    1: dict(name="256x256_100steps", nx=256, ny=256, steps=100, dt=1e-4),
    2: dict(name="1024x1024_50steps", nx=1024, ny=1024, steps=50, dt=1e-4),
    3: dict(name="4096x4096_20steps", nx=4096, ny=4096, steps=20, dt=1e-4),
    4: dict(name="16384x16384_10steps", nx=16384, ny=16384, steps=10, dt=1e-4),
}


def _uniform_rows(seed: int, nx: int, j0: int, j1: int, lo: float, hi: float) -> np.ndarray:
    bg = np.random.PCG64(seed)
    if j0:
        bg.advance(j0 * nx)
    gen = np.random.Generator(bg)
    return gen.uniform(lo, hi, size=(j1 - j0, nx))


def initial_fields(nx: int, ny: int, seed: int = 0, *, radius: float = 0.1,
                   base_height: float = 0.2, centre_x: float = 0.5,
                   phi_biofilm: float = 0.3, phi_background: float = 1e-3,
                   noise: float = 1e-3, rows: tuple[int, int] | None = None) -> dict:
    """Return the seeded initial state {phi, c, u, v, p} as float64 (rows, nx) arrays."""
    j0, j1 = (0, ny) if rows is None else rows
    x = (np.arange(nx, dtype=np.float64) + 0.5) / nx
    y = (np.arange(j0, j1, dtype=np.float64) + 0.5) / ny
    X, Y = np.meshgrid(x, y)  # (rows, nx)
    inside = (Y < base_height) | ((X - centre_x) ** 2 + (Y - base_height) ** 2 < radius ** 2)
    phi = np.where(inside, phi_biofilm, phi_background)
    if noise:
        phi = phi + _uniform_rows(seed, nx, j0, j1, -noise, noise)
    shape = (j1 - j0, nx)
    return dict(
        phi=np.ascontiguousarray(phi),
        c=np.ones(shape),
        u=np.zeros(shape),
        v=np.zeros(shape),
        p=np.zeros(shape),
    )


def random_field(nx: int, ny: int, seed: int, lo: float = 0.0, hi: float = 1.0,
                 rows: tuple[int, int] | None = None) -> np.ndarray:
    """Uniform [lo, hi) fp64 field (BASELINE.json configs[4] matvec sweeps)."""
    j0, j1 = (0, ny) if rows is None else rows
    return _uniform_rows(seed, nx, j0, j1, lo, hi)
