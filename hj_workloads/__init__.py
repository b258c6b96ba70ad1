"""Seeded synthetic problem generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no operator, no interpolation,
no value iteration, no labelling).  It only turns the BASELINE.json configs
into plain problem data — the things PAPER.md §2/§3 say the user supplies:
the grid (§3 "structured grid", line 229), the discrete control set
(§3 "discrete version of the control space"), the dynamics
coefficients f, the running cost l, the discount lambda, the step h, and the
boundary-node index vectors X_i of the target pieces (RA input, line 314:
"a collection of vectors such that union(X_i)=X_Gamma").

Both `oracle/` and `paper_1405_3521_b200/` consume a `Problem`; neither imports
the other.  Every random draw is from `numpy.random.default_rng(seed)`.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

DYN_AFFINE = 0      # f(x,a) = c(x) * u_a + A x + b           (configs 1,2,3,5)
DYN_DUBINS = 1      # f(x,a) = (v cos th, v sin th, w a)       (config 4)
DYN_VANDERPOL = 2   # f(x,a) = (x2, mu (1-x1^2) x2 - x1 + a)  (paper §4.1 Ex. 4.2)

COST_KRUZKOV = 0     # min-time, Kruzkov transformed: bracket cost = 1 - beta
COST_DISCOUNTED = 1  # discounted infinite horizon: bracket cost = h * l(x,a)


@dataclasses.dataclass
class Grid:
    """Regular node lattice.  Node i on axis d sits at lo[d] + i*dx[d];
    dx = (hi-lo)/(n-1) on ordinary axes, (hi-lo)/n on periodic axes."""
    n: tuple
    lo: tuple
    hi: tuple
    periodic: tuple

    @property
    def dim(self) -> int:
        return len(self.n)

    @property
    def size(self) -> int:
        return int(np.prod(self.n))

    def spacing(self, d: int) -> float:
        span = self.hi[d] - self.lo[d]
        return span / self.n[d] if self.periodic[d] else span / (self.n[d] - 1)

    def axis(self, d: int) -> np.ndarray:
        return self.lo[d] + np.arange(self.n[d], dtype=np.float64) * self.spacing(d)

    def mesh(self):
        """Node coordinates, each of shape n[::-1] (C order: last axis = x)."""
        axes = [self.axis(d) for d in range(self.dim)]
        return np.meshgrid(*axes[::-1], indexing="ij")[::-1]


@dataclasses.dataclass
class Problem:
    grid: Grid
    dynamics: int
    controls: np.ndarray          # (K, 3) float64; meaning depends on dynamics
    cost: int
    lam: float
    h: float
    tol: float
    max_iter: int
    piece: np.ndarray             # int8 node field, -1 = not a target node
    n_pieces: int
    A: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros((3, 3)))
    b: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(3))
    speed: Optional[np.ndarray] = None   # c(x) node field (float64) or None == 1
    g: Optional[np.ndarray] = None       # g(x_i) node field on target nodes, None == 0
    dubins_v: float = 1.0
    dubins_w: float = 1.0
    vdp_mu: float = 1.0
    l0: float = 0.0
    lq: float = 0.0
    ln: float = 0.0
    lr: float = 0.0
    v_out: float = 1.0
    name: str = ""

    @property
    def n_controls(self) -> int:
        return int(self.controls.shape[0])


@dataclasses.dataclass
class Config:
    """A BASELINE.json config: fine grid problem, coarse grid problem
    (same data on the nested coarse lattice), sub-domain count, overlap band."""
    name: str
    fine: Problem
    coarse: Optional[Problem]
    m: int
    band: int
    ratio: tuple
    dtype: str
    n_max_steps: int
    note: str = ""


# ----------------------------------------------------------------------------
# control sets (§3: "discrete version of the control space A")
# ----------------------------------------------------------------------------
def unit_circle_controls(k: int) -> np.ndarray:
    ang = 2.0 * np.pi * np.arange(k) / k
    c = np.zeros((k, 3))
    c[:, 0] = np.cos(ang)
    c[:, 1] = np.sin(ang)
    return c


def interval_controls(k: int, lo=-1.0, hi=1.0, axis=0) -> np.ndarray:
    c = np.zeros((k, 3))
    c[:, axis] = np.linspace(lo, hi, k)
    return c


def axis_controls() -> np.ndarray:
    return np.array([[1.0, 0, 0], [0, 1.0, 0], [-1.0, 0, 0], [0, -1.0, 0]])


# ----------------------------------------------------------------------------
# target pieces: the node vectors X_i (§3 RA input, line 314)
# ----------------------------------------------------------------------------
def ball_pieces(grid: Grid, centres: Sequence, radii: Sequence) -> np.ndarray:
    """Node belongs to piece k if |x - c_k| <= r_k in the (x, y) plane
    (lowest k wins on overlap).  All theta for 3-D grids."""
    xs = grid.mesh()
    piece = np.full(xs[0].shape, -1, dtype=np.int8)
    for k in range(len(centres) - 1, -1, -1):
        cx, cy = centres[k]
        inside = (xs[0] - cx) ** 2 + (xs[1] - cy) ** 2 <= radii[k] ** 2
        piece[inside] = k
    return piece.reshape(-1)


def sector_pieces(grid: Grid, rho: float, m: int) -> np.ndarray:
    """PAPER.md §4.1 (line 585): target ball B(0,rho) divided "in slices of a
    cake": piece k = nodes of the ball with angle in [2 pi k/m, 2 pi (k+1)/m)."""
    xs = grid.mesh()
    r2 = xs[0] ** 2 + xs[1] ** 2
    ang = np.mod(np.arctan2(xs[1], xs[0]), 2 * np.pi)
    k = np.minimum((ang / (2 * np.pi / m)).astype(np.int64), m - 1)
    piece = np.where(r2 <= rho * rho, k, -1).astype(np.int8)
    return piece.reshape(-1)


def box_edge_pieces(grid: Grid, m: int = 4) -> np.ndarray:
    """PAPER.md §4.1: boundary of the square split per edge.  m=4:
    y=lo, x=hi, y=hi, x=lo (corners go to the first edge listed); m=1: all."""
    nx, ny = grid.n
    piece = np.full((ny, nx), -1, dtype=np.int8)
    if m == 1:
        piece[0, :] = piece[-1, :] = piece[:, 0] = piece[:, -1] = 0
    else:
        piece[:, 0] = 3
        piece[-1, :] = 2
        piece[:, -1] = 1
        piece[0, :] = 0
    return piece.reshape(-1)


def courant_h(speed_bounds: Sequence[float], grid: Grid) -> float:
    """Reading R5: h = min_d dx_d / max|f_d| (per-axis Courant number 1)."""
    return min(grid.spacing(d) / speed_bounds[d] for d in range(grid.dim))


def coarse_grid(fine: Grid, ratio: Sequence[int]) -> Grid:
    n = []
    for d in range(fine.dim):
        if fine.periodic[d]:
            assert fine.n[d] % ratio[d] == 0
            n.append(fine.n[d] // ratio[d])
        else:
            assert (fine.n[d] - 1) % ratio[d] == 0
            n.append((fine.n[d] - 1) // ratio[d] + 1)
    return Grid(tuple(n), fine.lo, fine.hi, fine.periodic)


def seeded_centres(seed: int, count: int, half: float) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(-half, half, size=(count, 2))


def speed_field_c2(grid: Grid) -> np.ndarray:
    """Config 2: c(x) = 1 + 0.5 sin(2 pi x) sin(2 pi y)."""
    x, y = grid.mesh()[:2]
    return (1.0 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y)).reshape(-1)


# ----------------------------------------------------------------------------
# the five BASELINE.json configs (scale < 1 shrinks the grids for tests)
# ----------------------------------------------------------------------------
def _scaled(n: int, scale: float, ratio: int) -> int:
    """Node count (n-1)*scale+1 rounded so that (n-1) stays a multiple of ratio."""
    cells = max(ratio, int(round((n - 1) * scale / ratio)) * ratio)
    return cells + 1


def config1(seed: int = 0, scale: float = 1.0, ratio=None) -> Config:
    """2D eikonal minimum time, 32 unit controls, [-1,1]^2, 101^2, 4 balls r=0.05
    at (+-0.5,+-0.5), Kruzkov, h = dx, tol 1e-10, 4 sub-domains."""
    ratio = 5 if ratio is None else int(ratio)
    n = _scaled(101, scale, ratio)
    g = Grid((n, n), (-1.0, -1.0), (1.0, 1.0), (False, False))
    centres = [(-0.5, -0.5), (0.5, -0.5), (-0.5, 0.5), (0.5, 0.5)]
    radii = [0.05] * 4

    def mk(grid):
        return Problem(grid=grid, dynamics=DYN_AFFINE, controls=unit_circle_controls(32),
                       cost=COST_KRUZKOV, lam=1.0, h=grid.spacing(0), tol=1e-10,
                       max_iter=100000, piece=ball_pieces(grid, centres, radii), n_pieces=4,
                       v_out=1.0, name="eikonal4")
    cg = coarse_grid(g, (ratio, ratio))
    return Config("c1_eikonal_101", mk(g), mk(cg), m=4, band=4, ratio=(ratio, ratio),
                  dtype="f64", n_max_steps=4 * n,
                  note="closed form T(x)=min_k |x-c_k|-r_k; Voronoi labels")


def config2(seed: int = 2, scale: float = 1.0, ratio=None) -> Config:
    """2D variable-speed eikonal, c = 1+0.5 sin sin, 64 controls, 1025^2 fp32,
    8 balls r=0.03 seeded in [-0.9,0.9]^2, tol 1e-7, coarse 129^2."""
    ratio = 8 if ratio is None else int(ratio)
    n = _scaled(1025, scale, ratio)
    g = Grid((n, n), (-1.0, -1.0), (1.0, 1.0), (False, False))
    centres = seeded_centres(seed, 8, 0.9)
    radii = [0.03] * 8

    def mk(grid):
        return Problem(grid=grid, dynamics=DYN_AFFINE, controls=unit_circle_controls(64),
                       cost=COST_KRUZKOV, lam=1.0, h=courant_h([1.5, 1.5], grid), tol=1e-7,
                       max_iter=200000, piece=ball_pieces(grid, centres, radii), n_pieces=8,
                       speed=speed_field_c2(grid), v_out=1.0, name="varspeed8")
    cg = coarse_grid(g, (ratio, ratio))
    return Config("c2_varspeed_1025", mk(g), mk(cg), m=8, band=4, ratio=(ratio, ratio),
                  dtype="f32", n_max_steps=8 * cg.n[0])


def config3(seed: int = 3, scale: float = 1.0, ratio=None) -> Config:
    """2D Zermelo: f = a + (0.5 y, 0), 64 controls, [-2,2]^2, 4097^2 fp32,
    16 balls r=0.04 seeded, coarse 257^2, overlap band 4 cells."""
    ratio = 16 if ratio is None else int(ratio)
    n = _scaled(4097, scale, ratio)
    g = Grid((n, n), (-2.0, -2.0), (2.0, 2.0), (False, False))
    centres = seeded_centres(seed, 16, 1.8)
    radii = [0.04] * 16
    A = np.zeros((3, 3))
    A[0, 1] = 0.5

    def mk(grid):
        return Problem(grid=grid, dynamics=DYN_AFFINE, controls=unit_circle_controls(64),
                       cost=COST_KRUZKOV, lam=1.0, h=courant_h([2.0, 1.0], grid), tol=1e-7,
                       max_iter=400000, piece=ball_pieces(grid, centres, radii), n_pieces=16,
                       A=A, v_out=1.0, name="zermelo16")
    cg = coarse_grid(g, (ratio, ratio))
    return Config("c3_zermelo_4097", mk(g), mk(cg), m=16, band=4, ratio=(ratio, ratio),
                  dtype="f32", n_max_steps=8 * cg.n[0])


def config4(seed: int = 4, scale: float = 1.0, ratio=None) -> Config:
    """3D Dubins car: (cos th, sin th, a), a in 11 values in [-1,1], (x,y) in
    [-3,3]^2, th periodic, 257x257x128 fp32, 8 disks r=0.2 seeded."""
    ratio = (4, 4, 4) if ratio is None else (int(ratio),) * 3
    nxy = _scaled(257, scale, ratio[0])
    nth = max(ratio[2] * 2, int(round(128 * scale / ratio[2])) * ratio[2])
    g = Grid((nxy, nxy, nth), (-3.0, -3.0, 0.0), (3.0, 3.0, 2 * np.pi), (False, False, True))
    centres = seeded_centres(seed, 8, 2.7)
    radii = [0.2] * 8

    def mk(grid):
        return Problem(grid=grid, dynamics=DYN_DUBINS, controls=interval_controls(11),
                       cost=COST_KRUZKOV, lam=1.0, h=courant_h([1.0, 1.0, 1.0], grid),
                       tol=1e-7, max_iter=200000, piece=ball_pieces(grid, centres, radii),
                       n_pieces=8, v_out=1.0, name="dubins8")
    cg = coarse_grid(g, ratio)
    return Config("c4_dubins_257", mk(g), mk(cg), m=8, band=4, ratio=ratio, dtype="f32",
                  n_max_steps=8 * cg.n[0])


def config5(seed: int = 5, scale: float = 1.0, ratio=None) -> Config:
    """2D discounted regulator: f = (x2, a - 0.5 x1), 33 controls in [-1,1],
    l = |x|^2 + 0.1 a^2, lambda = 1, [-2,2]^2, 16385^2 fp32, 32 sub-domains from
    a 513^2 coarse feedback, tol 1e-6.  Reading R12: target B(0,0.2) cut in 32
    sectors (paper §4.1 "slices of a cake"); reading R5b: h = dx^(2/3).  Reading R13b: the
    band (unstated) is two coarse cells, 2 x ratio fine cells — the coarse feedback's
    trajectories leave thinner sets (measured at full size, R13b)."""
    ratio = 32 if ratio is None else int(ratio)
    n = _scaled(16385, scale, ratio)
    g = Grid((n, n), (-2.0, -2.0), (2.0, 2.0), (False, False))
    A = np.zeros((3, 3))
    A[0, 1] = 1.0
    A[1, 0] = -0.5
    ctrl = interval_controls(33, axis=1)   # effect u_a = (0, a)
    l_max = 8.0 + 0.1

    def mk(grid):
        h = grid.spacing(0) ** (2.0 / 3.0)
        beta = 1.0 / (1.0 + h)
        return Problem(grid=grid, dynamics=DYN_AFFINE, controls=ctrl, cost=COST_DISCOUNTED,
                       lam=1.0, h=h, tol=1e-6, max_iter=400000,
                       piece=sector_pieces(grid, 0.2, 32), n_pieces=32, A=A,
                       lq=1.0, lr=0.1, v_out=h * l_max / (1.0 - beta), name="regulator32")
    cg = coarse_grid(g, (ratio, ratio))
    return Config("c5_regulator_16385", mk(g), mk(cg), m=32, band=2 * ratio, ratio=(ratio, ratio),
                  dtype="f32", n_max_steps=int(40.0 / mk(cg).h))


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make(idx: int, scale: float = 1.0, seed: Optional[int] = None, ratio=None) -> Config:
    """BASELINE config `idx` (1..5); scale < 1 shrinks the fine grid, `ratio`
    overrides the fine/coarse nesting ratio (small test grids need a finer coarse
    grid to resolve the target balls)."""
    fn = CONFIGS[idx]
    kw = dict(scale=scale, ratio=ratio)
    if seed is not None:
        kw["seed"] = seed
    return fn(**kw)


def random_field(problem: Problem, seed: int, lo=0.0, hi=1.0) -> np.ndarray:
    """Random node field (for operator property tests)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=problem.grid.size)
