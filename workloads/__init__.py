"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no stencil, no update, no
wavelet): only the velocity models and the workload definitions (grid, dt,
source position and Ricker parameters, receiver positions, step counts), as
recipes in DESIGN.md section 6.  Both ``oracle`` (via tests/bench) and the
product path receive the same fp32 arrays and plain numbers from here.

Velocity models (h = 10 m everywhere):
  HOMO    v = 2000 m/s
  LAYERED 8 equal layers along global z, v_l = 1500 + 3000 l / 7
  HET3D   LAYERED(z) * (1 - 0.2 exp(-|x - x_c|^2 / (2 s^2))) * (1 + 0.02 u),
          s = nx/8 cells, x_c the grid centre (cells), u in [-1, 1) from
          splitmix64(231105038 + global linear index) -- index-addressable so
          each rank can build its own slab.
All values are computed in fp64 and rounded once to fp32.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED = 231105038
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Counter-based splitmix64 (one output per input state), uint64 wraparound."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_pm1(lin_index: np.ndarray) -> np.ndarray:
    """u in [-1, 1) from splitmix64(SEED + index), 53-bit mantissa."""
    z = splitmix64(np.uint64(SEED) + lin_index.astype(np.uint64))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def _layered(gz: np.ndarray, nz_global: int) -> np.ndarray:
    layer = np.minimum((gz * 8) // nz_global, 7)
    return 1500.0 + 3000.0 * layer / 7.0


def velocity(kind: str, dims, z0: int = 0, z1: int | None = None,
             nz_global: int | None = None) -> np.ndarray:
    """fp32 velocity of planes [z0, z1) of a grid ``dims`` (slow->fast).

    ``nz_global`` defaults to dims[0]; ``dims[0]`` is the global nz.
    """
    dims = tuple(int(d) for d in dims)
    nz = dims[0] if nz_global is None else int(nz_global)
    z1 = dims[0] if z1 is None else int(z1)
    shape = (z1 - z0,) + dims[1:]
    if kind == "HOMO":
        return np.full(shape, 2000.0, dtype=np.float32)
    gz = np.arange(z0, z1, dtype=np.int64).reshape((-1,) + (1,) * (len(dims) - 1))
    if kind == "LAYERED":
        return np.broadcast_to(_layered(gz, nz), shape).astype(np.float32)
    if kind == "HET3D":
        if len(dims) != 3:
            raise ValueError("HET3D is 3D")
        ny, nx = dims[1], dims[2]
        out = np.empty(shape, dtype=np.float32)
        sig = nx / 8.0
        yy = np.arange(ny, dtype=np.float64).reshape(-1, 1)
        xx = np.arange(nx, dtype=np.float64).reshape(1, -1)
        zc, yc, xc = (nz - 1) / 2.0, (ny - 1) / 2.0, (nx - 1) / 2.0
        rxy2 = (yy - yc) ** 2 + (xx - xc) ** 2
        lin_xy = (np.arange(ny, dtype=np.int64).reshape(-1, 1) * nx
                  + np.arange(nx, dtype=np.int64).reshape(1, -1))
        for i, g in enumerate(range(z0, z1)):
            lay = 1500.0 + 3000.0 * min((g * 8) // nz, 7) / 7.0
            bump = 1.0 - 0.2 * np.exp(-(rxy2 + (g - zc) ** 2) / (2.0 * sig * sig))
            u = uniform_pm1(np.int64(g) * ny * nx + lin_xy)
            out[i] = (lay * bump * (1.0 + 0.02 * u)).astype(np.float32)
        return out
    if kind == "RANDOM":  # small-test model: v in [1800, 2200)
        lin = np.arange(int(np.prod(shape)), dtype=np.int64) + z0 * int(np.prod(dims[1:]))
        return (2000.0 + 200.0 * uniform_pm1(lin)).reshape(shape).astype(np.float32)
    raise ValueError(f"unknown velocity model {kind}")


@dataclass
class Source:
    idx: tuple
    f: float
    t0: float
    amp: float = 1.0


@dataclass
class Workload:
    name: str
    dims: tuple            # slow -> fast
    model: str
    h: float
    dt: float
    steps: int
    order: int
    sources: list = field(default_factory=list)
    receivers: list = field(default_factory=list)   # list of index tuples
    note: str = ""

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def npts(self) -> int:
        return int(np.prod(self.dims))

    def vel(self) -> np.ndarray:
        return velocity(self.model, self.dims)

    def with_order(self, order: int) -> "Workload":
        w = Workload(**{**self.__dict__})
        w.order = order
        return w


def _row_receivers_2d(z, nx):
    return [(z, x) for x in range(nx)]


def _line_receivers_3d(z, y, nx):
    return [(z, y, x) for x in range(nx)]


def config(name: str, order: int | None = None, steps: int | None = None) -> Workload:
    """The BASELINE.json configurations."""
    if name == "C1":
        w = Workload("C1", (256, 256), "HOMO", 10.0, 1.0e-3, 500, 2,
                     [Source((128, 128), 25.0, 0.040)], _row_receivers_2d(160, 256),
                     "2D 256x256 homogeneous, Ricker at centre, 500 steps")
    elif name == "C2":
        w = Workload("C2", (4096, 4096), "LAYERED", 10.0, 1.0e-3, 2000, 2,
                     [Source((32, 2048), 15.0, 1.0 / 15.0)], _row_receivers_2d(40, 4096),
                     "2D 4096x4096 layered, 2000 steps")
    elif name == "C3":
        w = Workload("C3", (512, 512, 512), "HOMO", 10.0, 1.0e-3, 1000, 2,
                     [Source((256, 256, 256), 25.0, 0.040)], _line_receivers_3d(320, 256, 512),
                     "3D 512^3 homogeneous, 1000 steps")
    elif name == "C4":
        w = Workload("C4", (1024, 1024, 1024), "HET3D", 10.0, 0.5e-3, 500, 2,
                     [Source((32, 512, 512), 15.0, 1.0 / 15.0)], _line_receivers_3d(40, 512, 1024),
                     "3D 1024^3 heterogeneous, 500 steps (strong scaling)")
    elif name.startswith("C5"):
        # C5:P -> (512 P) x 1024 x 1024
        P = int(name.split(":")[1]) if ":" in name else 1
        w = Workload(f"C5:{P}", (512 * P, 1024, 1024), "HET3D", 10.0, 0.5e-3, 200, 2,
                     [Source((32, 512, 512), 15.0, 1.0 / 15.0)], _line_receivers_3d(40, 512, 1024),
                     "3D weak scaling 1024^2 x 512 per GPU")
    else:
        raise ValueError(name)
    if order is not None:
        w.order = order
    if steps is not None:
        w.steps = steps
    return w
