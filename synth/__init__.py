"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no element matrices, stencils,
transfers or solvers).  It only defines the synthetic workloads of
BASELINE.json ``configs[0..4]``:

* the structured Kuhn grid indexing (vertex ``v = i + (n+1)(j + (n+1)k)``,
  element ``e = 6*(i + n*(j + n*k)) + t``, ``t`` = Kuhn permutation index),
* the per-element viscosity class by a centroid predicate,
* the per-element forcing class (element-constant forcing, cfg3/cfg5),
* counter-based splitmix64 random numbers for nodal forcing and apply inputs,
* the face boundary types (0 = homogeneous Dirichlet, 1 = traction free,
  2 = free slip) and the eliminated velocity DoFs they define.

The geometry follows PAPER.md P:720 ("4^3 cubes ... each subdivided into six
tetrahedra"); the Kuhn split itself is the reading of DESIGN.md §3 (R2).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# Kuhn permutations, t = 0..5  <->  sigma.
PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))

DIRICHLET, TRACTION, FREESLIP = 0, 1, 2
FACE_NAMES = ("x0", "x1", "y0", "y1", "z0", "z1")

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, stream: int, idx) -> np.ndarray:
    """U(stream, idx) in [0,1): ((splitmix64((seed<<40)^(stream<<36)^idx) >> 11) * 2^-53)."""
    idx = np.asarray(idx, dtype=np.uint64)
    key = np.uint64((seed << 40) & 0xFFFFFFFFFFFFFFFF) ^ np.uint64(stream << 36)
    r = splitmix64(idx ^ key) >> np.uint64(11)
    return r.astype(np.float64) * (2.0 ** -53)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    class_mu: tuple           # viscosity per element class
    faces: tuple              # 6 face types (x0,x1,y0,y1,z0,z1)
    forcing: str              # "nodal" (iid U[-1,1]) or "element"
    force_table: tuple = ((0.0, 0.0, 0.0),)   # per forcing class (element forcing)
    seed: int = 0

    @property
    def vertices(self) -> int:
        return (self.n + 1) ** 3

    @property
    def dofs(self) -> int:
        """Paper's DoF convention 4(n+1)^3 (19,652 at L=2 / n=16)."""
        return 4 * (self.n + 1) ** 3

    def with_n(self, n: int) -> "Config":
        return dataclasses.replace(self, n=n)


ALL_DIRICHLET = (DIRICHLET,) * 6
TOP_TRACTION = (DIRICHLET,) * 5 + (TRACTION,)
ALL_FREESLIP = (FREESLIP,) * 6

CONFIGS = {
    # BASELINE.json configs[0]: plane x=0.5, mu1=10 (x<0.5), mu2=1, u=0 on all faces
    "cfg1": Config("cfg1", 16, (10.0, 1.0), ALL_DIRICHLET, "nodal"),
    # configs[1]: plane x=0.5, mu1/mu2 = 1e3, traction-free top z=1
    "cfg2": Config("cfg2", 128, (1e3, 1.0), TOP_TRACTION, "nodal"),
    # configs[2]: sphere r=0.25 at centre, mu=1 inside, 1e4 outside; f=(0,0,-1) inside
    "cfg3": Config("cfg3", 256, (1e4, 1.0), ALL_DIRICHLET, "element",
                   ((0.0, 0.0, 0.0), (0.0, 0.0, -1.0))),
    # configs[3]: 64 random spheres, mu=1 inside, 100 outside; nodal f
    "cfg4": Config("cfg4", 512, (100.0, 1.0), ALL_DIRICHLET, "nodal"),
    # configs[4]: lid z>0.9 and inclined plate mu=1e3, mu=1 elsewhere; traction top;
    # f_z=-1 in the plate
    "cfg5": Config("cfg5", 1024, (1.0, 1e3), TOP_TRACTION, "element",
                   ((0.0, 0.0, 0.0), (0.0, 0.0, -1.0))),
    # SURVEY NEXT-1, the paper's own timed workload:
    # viscosity columns mu2 = 10 in (0,1/4)^2 x (0,1) u (3/4,1)^2 x (0,1), mu1 = 1
    # elsewhere; free slip on all faces; f = (0, 0, -cos 2pi x cos 2pi y sin pi z)
    # (nodal values); levels L = 5..8 are n = 4 * 2^L = 128..1024 (4^3 base cubes)
    "cols": Config("cols", 128, (1.0, 10.0), ALL_FREESLIP, "nodal"),
}


def get_config(name: str, n: int | None = None, seed: int = 0) -> Config:
    c = CONFIGS[name]
    c = dataclasses.replace(c, seed=seed)
    return c.with_n(n) if n is not None else c


# ----------------------------------------------------------------------------
# geometry: tet centroids (units of h) for all elements of a block of cube layers
# ----------------------------------------------------------------------------
_CENTROID_OFFSETS = np.zeros((6, 3))
for _t, _s in enumerate(PERMS):
    _CENTROID_OFFSETS[_t, _s[0]] += 0.75
    _CENTROID_OFFSETS[_t, _s[1]] += 0.5
    _CENTROID_OFFSETS[_t, _s[2]] += 0.25


def _centroids(n: int, k0: int, k1: int):
    """Centroids (x,y,z arrays, shape [k1-k0, n, n, 6]) of cube layers k0..k1-1."""
    h = 1.0 / n
    k = np.arange(k0, k1, dtype=np.float64)[:, None, None, None]
    j = np.arange(n, dtype=np.float64)[None, :, None, None]
    i = np.arange(n, dtype=np.float64)[None, None, :, None]
    off = _CENTROID_OFFSETS
    x = (i + off[None, None, None, :, 0]) * h
    y = (j + off[None, None, None, :, 1]) * h
    z = (k + off[None, None, None, :, 2]) * h
    return np.broadcast_arrays(x, y, z)


def _spheres(seed: int, count: int = 64):
    j = np.arange(count, dtype=np.uint64)
    c = np.stack([uniform(seed, 3, 4 * j + d) for d in range(3)], axis=1)
    r = 0.03 + 0.05 * uniform(seed, 3, 4 * j + 3)
    return c, r


def _classes_block(cfg: Config, k0: int, k1: int):
    x, y, z = _centroids(cfg.n, k0, k1)
    name = cfg.name
    if name in ("cfg1", "cfg2"):
        mu_cls = np.where(x < 0.5, 0, 1)
        f_cls = np.zeros_like(mu_cls)
    elif name == "cfg3":
        inside = (x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2 < 0.25 ** 2
        mu_cls = np.where(inside, 1, 0)
        f_cls = np.where(inside, 1, 0)
    elif name == "cfg4":
        c, r = _spheres(cfg.seed)
        inside = np.zeros(x.shape, dtype=bool)
        n = cfg.n
        for s in range(len(r)):
            # only cubes whose index box can hold a centroid inside sphere s
            lo = np.floor((c[s] - r[s]) * n).astype(int) - 1
            hi = np.ceil((c[s] + r[s]) * n).astype(int) + 1
            kk0, kk1 = max(lo[2], k0), min(hi[2], k1)
            if kk0 >= kk1:
                continue
            sl = (slice(kk0 - k0, kk1 - k0), slice(max(lo[1], 0), min(hi[1], n)),
                  slice(max(lo[0], 0), min(hi[0], n)))
            xs, ys, zs = x[sl], y[sl], z[sl]
            inside[sl] |= (xs - c[s, 0]) ** 2 + (ys - c[s, 1]) ** 2 + (zs - c[s, 2]) ** 2 < r[s] ** 2
        mu_cls = np.where(inside, 1, 0)
        f_cls = np.zeros_like(mu_cls)
    elif name == "cols":
        col = ((x < 0.25) & (y < 0.25)) | ((x > 0.75) & (y > 0.75))
        mu_cls = np.where(col, 1, 0)
        f_cls = np.zeros_like(mu_cls)
    elif name == "cfg5":
        s = x + z
        plate = (s >= 1.2 - 0.08 * math.sqrt(2.0)) & (s <= 1.2) & (z <= 0.9)
        lid = z > 0.9
        mu_cls = np.where(plate | lid, 1, 0)
        f_cls = np.where(plate, 1, 0)
    else:
        raise ValueError(name)
    return mu_cls.astype(np.uint8), f_cls.astype(np.uint8)


def element_classes(cfg: Config, k0: int = 0, k1: int | None = None):
    """(viscosity class, forcing class) uint8 arrays, layout [k][j][i][t] flattened.

    Cube layers k0..k1-1 (default: all).  Classes by the tet centroid with strict
    '<' tests; processed in chunks to bound memory.
    """
    n = cfg.n
    k1 = n if k1 is None else k1
    mu = np.empty((k1 - k0, n, n, 6), dtype=np.uint8)
    fc = np.empty_like(mu)
    chunk = max(1, (1 << 22) // (6 * n * n))
    for a in range(k0, k1, chunk):
        b = min(k1, a + chunk)
        m, f = _classes_block(cfg, a, b)
        mu[a - k0:b - k0] = m
        fc[a - k0:b - k0] = f
    return mu.reshape(-1), fc.reshape(-1)


def nodal_forcing(cfg: Config, v0: int = 0, v1: int | None = None) -> np.ndarray:
    """f_a(v) = 2 U(1, 3v+a) - 1 for vertices v0..v1-1, shape (3, v1-v0); for the
    "cols" workload the paper's f = (0, 0, -cos 2pi x cos 2pi y sin pi z) at the
    vertices."""
    v1 = cfg.vertices if v1 is None else v1
    if cfg.name == "cols":
        N1 = cfg.n + 1
        v = np.arange(v0, v1, dtype=np.int64)
        x, y, z = (v % N1) / cfg.n, ((v // N1) % N1) / cfg.n, (v // (N1 * N1)) / cfg.n
        f = np.zeros((3, v1 - v0))
        f[2] = -np.cos(2 * np.pi * x) * np.cos(2 * np.pi * y) * np.sin(np.pi * z)
        return f
    v = np.arange(v0, v1, dtype=np.uint64)
    return np.stack([2.0 * uniform(cfg.seed, 1, 3 * v + a) - 1.0 for a in range(3)])


def apply_input(cfg: Config, v0: int = 0, v1: int | None = None) -> np.ndarray:
    """x_f(v) = 2 U(2, 4v+f) - 1 for fields f = (u1,u2,u3,p), shape (4, v1-v0)."""
    v1 = cfg.vertices if v1 is None else v1
    v = np.arange(v0, v1, dtype=np.uint64)
    return np.stack([2.0 * uniform(cfg.seed, 2, 4 * v + f) - 1.0 for f in range(4)])


def dirichlet_vertex_mask(n: int, faces) -> np.ndarray:
    """Boolean (V,) mask: vertex lies on the closure of a Dirichlet face."""
    idx = np.arange(n + 1)
    k, j, i = np.meshgrid(idx, idx, idx, indexing="ij")
    m = np.zeros((n + 1,) * 3, dtype=bool)
    for f, (coord, val) in enumerate(((i, 0), (i, n), (j, 0), (j, n), (k, 0), (k, n))):
        if faces[f] == DIRICHLET:
            m |= coord == val
    return m.reshape(-1)


def eliminated_mask(n: int, faces) -> np.ndarray:
    """Boolean (3, V) mask: velocity component a of vertex v is fixed to 0 -- all three
    on the closure of a Dirichlet face, component a on a free-slip face of normal
    e_a (u.n = 0).  The boundary-condition definition of the workload."""
    idx = np.arange(n + 1)
    k, j, i = np.meshgrid(idx, idx, idx, indexing="ij")
    m = np.zeros((3,) + (n + 1,) * 3, dtype=bool)
    for f, (coord, val) in enumerate(((i, 0), (i, n), (j, 0), (j, n), (k, 0), (k, n))):
        on = coord == val
        if faces[f] == DIRICHLET:
            m[:, on] = True
        elif faces[f] == FREESLIP:
            m[f // 2][on] = True
    return m.reshape(3, -1)
