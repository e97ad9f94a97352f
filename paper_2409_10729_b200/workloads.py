"""Seeded synthetic workloads (BASELINE.json configs C1-C5 and the branch-coverage
input G-R) -- the ONLY module shared by the oracle side and the CUDA side.

It holds none of the method's arithmetic: no EOS, no reconstruction, no Riemann
solver, no time stepping.  Every generator returns PRIMITIVE fields
v = (α_iρ_i [N], u_k [d], p, α_i [N]) on cell centres as float64 numpy arrays of
shape (E, nz, ny, nx); conversion to conserved variables is done by each side
with its own code (oracle.prim_to_cons / mfc_prim_to_cons).

Recipes (DESIGN.md §4 "Inputs"):
  C1  1D water-air shock tube, 400 cells, interface at 0.7 m, extrapolation BCs.
  C2  2D air-helium shock-bubble, 1024 x 512 on [0,2] x [0,1], Mach 1.22 shock.
  C3  3D two-fluid shock-droplet, 256^3 on [0,1]^3 periodic, Mach 1.46 air slab.
  C4  C3's block per GPU, stacked along z (weak scaling).
  C5  3D three-fluid (air, water droplet, helium bubble), 512^3 total.
  G-R random primitive fields (uniform draws, 3-point smoothed) that exercise every
      HLLC branch (subsonic, supersonic left/right) and varying WENO weights.
Material constants (AMB-20): air γ=1.4, π∞=0; water γ=4.4, π∞=6e8 Pa; helium
γ=1.648, π∞=0 (density ratio 0.182 to air at equal p, T).
Post-shock states are textbook normal-shock (Rankine-Hugoniot) values for an ideal
gas with γ=1.4, hard-coded here and re-derived in tests/test_workloads.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

SEED = 10729

BC_PERIODIC = -1
BC_REFLECTIVE = -2
BC_EXTRAPOLATION = -3

AIR = (1.4, 0.0)
WATER = (4.4, 6.0e8)
HELIUM = (1.648, 0.0)

# Mach 1.46 normal shock into air at rest, γ = 1.4 (p2/p1, ρ2/ρ1, u2/c1)
M146 = (2.3202, 1.79337, 0.64589)
# Mach 1.22 normal shock into air (ρ, u, p) = (1, 0, 1): post-shock state
M122_POST = (1.376364, 0.394729, 1.569800)


@dataclass
class Problem:
    """A grid, materials and boundary conditions (the arguments of mfc_init)."""
    name: str
    n_fluids: int
    ndim: int
    n: tuple                      # (nx, ny, nz); 1 for inactive dims
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    gamma: tuple = ()
    pi_inf: tuple = ()
    bc: tuple = (BC_PERIODIC,) * 6
    dt: float = 0.0               # a stable fixed time step for this workload
    steps: int = 0                # steps the config names (C1: 200)
    weno_eps: float = 1e-16
    weno_order: int = 5           # 5 (default) or 3
    weno_mapped: bool = False     # WENO5-M weights (Henrick et al. 2005)
    notes: dict = field(default_factory=dict)
    # stretched grid: per axis None (uniform) or the n+1 cell
    # boundaries from lo to hi (tanh_boundaries); geometry only, like lo/hi
    x_cb: tuple = (None, None, None)

    @property
    def E(self) -> int:
        return 2 * self.n_fluids + self.ndim + 1

    @property
    def dx(self):
        return tuple((self.hi[k] - self.lo[k]) / self.n[k] for k in range(3))

    @property
    def stretched(self) -> bool:
        return any(x is not None for x in self.x_cb)

    @property
    def cells(self) -> int:
        return int(self.n[0] * self.n[1] * self.n[2])

    @property
    def shape(self):
        return (self.E, self.n[2], self.n[1], self.n[0])

    def boundaries(self, k: int) -> np.ndarray:
        """The n+1 cell boundaries of axis k (uniform unless x_cb[k] is set)."""
        if self.x_cb[k] is not None:
            return np.asarray(self.x_cb[k], dtype=np.float64)
        return self.lo[k] + np.arange(self.n[k] + 1) * self.dx[k]

    def centres(self, z0: int = 0, z1: int | None = None):
        """Cell-centre coordinates (X, Y, Z) broadcastable to (nz, ny, nx); optionally
        only the z-planes z0 .. z1-1 (slab-wise generation of large grids)."""
        if self.stretched:
            xs = [0.5 * (self.boundaries(k)[1:] + self.boundaries(k)[:-1]) for k in range(3)]
        else:
            xs = [self.lo[k] + (np.arange(self.n[k]) + 0.5) * self.dx[k] for k in range(3)]
        xs[2] = xs[2][z0:z1]
        return xs[0][None, None, :], xs[1][None, :, None], xs[2][:, None, None]

    def with_n(self, n):
        return replace(self, n=tuple(n))


def _assemble(pb: Problem, partial, vel, p, alpha, nz=None):
    """Stack primitive components into (E, nz, ny, nx)."""
    shape = (pb.n[2] if nz is None else nz, pb.n[1], pb.n[0])
    comps = [np.broadcast_to(a, shape) for a in partial]
    comps += [np.broadcast_to(u, shape) for u in vel[: pb.ndim]]
    comps += [np.broadcast_to(p, shape)]
    comps += [np.broadcast_to(a, shape) for a in alpha]
    return np.ascontiguousarray(np.stack(comps).astype(np.float64))


def smooth_step(s, width):
    """0 -> 1 across s = 0 with a tanh profile of the given width (geometry only)."""
    return 0.5 * (1.0 + np.tanh(s / width))


# ------------------------------------------------------- stretched grids (F4)

def tanh_boundaries(n: int, lo: float, hi: float, r: float = 0.5, xi_a: float = 0.3,
                    xi_b: float = 0.7, w: float = 0.05) -> np.ndarray:
    """Cell boundaries x_i = x(i/n), i = 0..n, of a hyperbolic-tangent local refinement
    (Vinokur [16]; DESIGN.md AMB-27): in the computational coordinate ξ ∈ [0, 1]
    the spacing is proportional to
        g(ξ) = 1 - (r/2) [tanh((ξ - ξa)/w) - tanh((ξ - ξb)/w)],
    i.e. cells are finer by the factor (1 - r) between ξa and ξb, with tanh transitions
    of width w; x(ξ) = lo + (hi - lo) G(ξ)/G(1) with G the integral of g (closed form
    through ln cosh).  0 <= r < 1; r = 0 gives the uniform grid."""
    xi = np.arange(n + 1, dtype=np.float64) / n

    def lncosh(z):                 # ln cosh z, overflow-free
        z = np.abs(z)
        return z + np.log1p(np.exp(-2.0 * z)) - np.log(2.0)

    def G(x):
        return x - 0.5 * r * w * (lncosh((x - xi_a) / w) - lncosh(xi_a / w)
                                  - lncosh((x - xi_b) / w) + lncosh(xi_b / w))

    x = lo + (hi - lo) * G(xi) / G(1.0)
    x[0], x[-1] = lo, hi
    return x


def stretched(pb: Problem, axes=(0, 1, 2), **kw) -> Problem:
    """The same problem on a tanh-refined grid along the given active axes."""
    xcb = list(pb.x_cb)
    for k in axes:
        if k < pb.ndim:
            xcb[k] = tanh_boundaries(pb.n[k], pb.lo[k], pb.hi[k], **kw)
    return replace(pb, x_cb=tuple(xcb), name=pb.name + " stretched")


# ----------------------------------------------------------------------- C1

def c1_water_air(n: int = 400) -> Problem:
    """1D water-air shock tube on [0,1] m, interface at 0.7 (fluid 1 water, 2 air)."""
    dx = 1.0 / n
    return Problem("C1 1D water-air shock tube", 2, 1, (n, 1, 1), (0.0, 0.0, 0.0),
                   (1.0, 1.0, 1.0), (WATER[0], AIR[0]), (WATER[1], AIR[1]),
                   (BC_EXTRAPOLATION,) * 2 + (BC_PERIODIC,) * 4,
                   dt=0.4 * dx / 2653.30, steps=200,
                   notes={"x_interface": 0.7, "left": (1000.0, 0.0, 1.0e9),
                          "right": (50.0, 0.0, 1.0e5), "alpha_min": 1e-6})


def c1_prims(pb: Problem) -> np.ndarray:
    X, _, _ = pb.centres()
    left = X < pb.notes["x_interface"]
    am = pb.notes["alpha_min"]
    a_w = np.where(left, 1.0 - am, am)
    a_a = 1.0 - a_w
    rho_w = 1000.0
    rho_a = 50.0
    p = np.where(left, 1.0e9, 1.0e5)
    return _assemble(pb, [a_w * rho_w, a_a * rho_a], [np.zeros_like(X)], p, [a_w, a_a])


# ----------------------------------------------------------------------- C2

def c2_shock_bubble(nx: int = 1024, ny: int = 512) -> Problem:
    """2D air-helium shock-bubble on [0,2] x [0,1] (fluid 1 air, 2 helium)."""
    dxy = 1.0 / ny
    return Problem("C2 2D air-helium shock-bubble", 2, 2, (nx, ny, 1), (0.0, 0.0, 0.0),
                   (2.0, 1.0, 1.0), (AIR[0], HELIUM[0]), (AIR[1], HELIUM[1]),
                   (BC_EXTRAPOLATION, BC_EXTRAPOLATION, BC_REFLECTIVE, BC_REFLECTIVE,
                    BC_PERIODIC, BC_PERIODIC),
                   dt=0.3 * dxy / 3.00918, steps=0,
                   notes={"bubble": (1.0, 0.5, 0.25), "shock_x": 0.6, "alpha_min": 1e-6})


def c2_prims(pb: Problem) -> np.ndarray:
    X, Y, _ = pb.centres()
    xc, yc, r = pb.notes["bubble"]
    am = pb.notes["alpha_min"]
    h = pb.dx[0]
    R = np.sqrt((X - xc) ** 2 + (Y - yc) ** 2)
    a_he = am + (1.0 - 2.0 * am) * smooth_step(r - R, h)
    a_air = 1.0 - a_he
    post = smooth_step(pb.notes["shock_x"] - X, h) * np.ones_like(Y)
    rho_air = 1.0 + (M122_POST[0] - 1.0) * post
    u = M122_POST[1] * post
    p = 1.0 + (M122_POST[2] - 1.0) * post
    rho_he = 0.182 * np.ones_like(R)
    return _assemble(pb, [a_air * rho_air, a_he * rho_he], [u, np.zeros_like(u)], p,
                     [a_air, a_he])


# ----------------------------------------------------------------------- C3

P_ATM = 1.01325e5
RHO_AIR = 1.204
C_AIR = math.sqrt(AIR[0] * P_ATM / RHO_AIR)


def c3_droplet(n: int = 256, nz: int | None = None, z_cells_total: int | None = None) -> Problem:
    """3D shock-droplet grind-time case: water droplet r=0.2 in air, Mach 1.46 slab
    for x < 0.2, [0,1]^3 periodic (fluid 1 water, 2 air)."""
    nz = n if nz is None else nz
    return Problem("C3 3D two-fluid shock-droplet", 2, 3, (n, n, nz), (0.0, 0.0, 0.0),
                   (1.0, 1.0, nz / n), (WATER[0], AIR[0]), (WATER[1], AIR[1]),
                   (BC_PERIODIC,) * 6, dt=_c3_dt(1.0 / n), steps=0,
                   notes={"droplet": (0.5, 0.5, 0.5, 0.2), "shock_x": 0.2, "alpha_min": 1e-6})


def _c3_dt(h):
    # max |u|+c: post-shock air c ≈ 1.2566 c1 ... water c ≈ 1625 m/s dominates
    return 0.3 * h / 1700.0


def c3_prims(pb: Problem, z0: int = 0, z1: int | None = None) -> np.ndarray:
    X, Y, Z = pb.centres(z0, z1)
    xc, yc, zc, r = pb.notes["droplet"]
    am = pb.notes["alpha_min"]
    h = pb.dx[0]
    R = np.sqrt((X - xc) ** 2 + (Y - yc) ** 2 + (Z - zc) ** 2)
    a_w = am + (1.0 - 2.0 * am) * smooth_step(r - R, h)
    a_a = 1.0 - a_w
    s = smooth_step(pb.notes["shock_x"] - X, h) * np.ones_like(a_w)
    rho_a = RHO_AIR * (1.0 + (M146[1] - 1.0) * s)
    p = P_ATM * (1.0 + (M146[0] - 1.0) * s)
    u = M146[2] * C_AIR * s
    rho_w = 1000.0 * np.ones_like(a_w)
    z = np.zeros_like(u)
    return _assemble(pb, [a_w * rho_w, a_a * rho_a], [u, z, z], p, [a_w, a_a], nz=Z.shape[0])


# ----------------------------------------------------------------------- C5

def c5_three_fluid(n: int = 512) -> Problem:
    """3D shock-droplet with a helium bubble, 3 fluids (1 water, 2 air, 3 helium)."""
    return Problem("C5 3D three-fluid shock-droplet", 3, 3, (n, n, n), (0.0, 0.0, 0.0),
                   (1.0, 1.0, 1.0), (WATER[0], AIR[0], HELIUM[0]),
                   (WATER[1], AIR[1], HELIUM[1]), (BC_PERIODIC,) * 6, dt=_c3_dt(1.0 / n),
                   notes={"droplet": (0.5, 0.5, 0.5, 0.15), "bubble": (0.75, 0.5, 0.5, 0.08),
                          "shock_x": 0.2, "alpha_min": 1e-6})


def c5_prims(pb: Problem, z0: int = 0, z1: int | None = None) -> np.ndarray:
    X, Y, Z = pb.centres(z0, z1)
    am = pb.notes["alpha_min"]
    h = pb.dx[0]
    xd, yd, zd, rd = pb.notes["droplet"]
    xb, yb, zb, rb = pb.notes["bubble"]
    Rd = np.sqrt((X - xd) ** 2 + (Y - yd) ** 2 + (Z - zd) ** 2)
    Rb = np.sqrt((X - xb) ** 2 + (Y - yb) ** 2 + (Z - zb) ** 2)
    hw = smooth_step(rd - Rd, h)
    hh = smooth_step(rb - Rb, h)
    a_w = am + (1.0 - 3.0 * am) * hw
    a_h = am + (1.0 - 3.0 * am) * hh * (1.0 - hw)
    a_a = 1.0 - a_w - a_h
    s = smooth_step(pb.notes["shock_x"] - X, h) * np.ones_like(a_w)
    rho_a = RHO_AIR * (1.0 + (M146[1] - 1.0) * s)
    rho_h = 0.182 * rho_a
    p = P_ATM * (1.0 + (M146[0] - 1.0) * s)
    u = M146[2] * C_AIR * s
    rho_w = 1000.0 * np.ones_like(a_w)
    z = np.zeros_like(u)
    return _assemble(pb, [a_w * rho_w, a_a * rho_a, a_h * rho_h], [u, z, z], p,
                     [a_w, a_a, a_h], nz=Z.shape[0])


# ----------------------------------------------------------------------- G-R

def random_problem(ndim: int, n, n_fluids: int = 2, materials: str = "gas",
                   bc=BC_PERIODIC) -> Problem:
    n = tuple(list(n) + [1] * (3 - len(n)))
    if materials == "gas":
        mats = [AIR, HELIUM, (1.6, 0.0)][:n_fluids]
    else:  # water-air(-helium)
        mats = [WATER, AIR, HELIUM][:n_fluids]
    bcs = bc if isinstance(bc, tuple) else (bc,) * 6
    return Problem(f"G-R random {ndim}D N={n_fluids} {materials}", n_fluids, ndim, n,
                   (0.0, 0.0, 0.0), tuple(1.0 * n[k] / n[0] for k in range(3)),
                   tuple(m[0] for m in mats), tuple(m[1] for m in mats), bcs,
                   dt=0.0, notes={"materials": materials})


def random_prims(pb: Problem, seed: int = SEED, smooth: int = 1, speed: float = 2.0):
    """Independent uniform draws per cell, `smooth` passes of a
    periodic 3-point average along every active axis."""
    rng = np.random.default_rng(seed)
    shape = (pb.n[2], pb.n[1], pb.n[0])
    N = pb.n_fluids
    water = pb.notes.get("materials") == "water"
    p0 = 1.0e5 if water else 1.0
    rho0 = [1000.0, 1.204, 0.2][:N] if water else [1.0, 0.182, 0.5][:N]
    cref = 340.0 if water else 1.2

    def sm(a):
        for _ in range(smooth):
            for ax in range(pb.ndim):
                axis = 2 - ax
                a = (np.roll(a, 1, axis) + a + np.roll(a, -1, axis)) / 3.0
        return a

    raw_alpha = [rng.uniform(1e-6, 1.0 - 1e-6, shape) for _ in range(N)]
    raw_alpha = [sm(a) for a in raw_alpha]
    tot = sum(raw_alpha)
    alpha = [a / tot for a in raw_alpha]
    alpha[-1] = 1.0 - sum(alpha[:-1])
    rho = [sm(rng.uniform(0.5, 2.0, shape)) * r0 for r0 in rho0]
    p = sm(rng.uniform(0.5, 2.0, shape)) * p0
    vel = [sm(rng.uniform(-speed, speed, shape)) * cref for _ in range(3)]
    return _assemble(pb, [alpha[i] * rho[i] for i in range(N)], vel, p, alpha)


# ------------------------------------------------------------ smooth waves

def entropy_wave_problem(n: int, ndim: int = 1, axis: int = 0) -> Problem:
    """Two-fluid advected entropy/material wave on a periodic unit domain (order tests)."""
    nn = [1, 1, 1]
    for k in range(ndim):
        nn[k] = n if k == axis else 4
    hi = [1.0, 1.0, 1.0]
    for k in range(ndim):
        hi[k] = 1.0 if k == axis else 4.0 / n
    return Problem(f"entropy wave {ndim}D n={n}", 2, ndim, tuple(nn), (0.0, 0.0, 0.0),
                   tuple(hi), (1.4, 1.6), (0.0, 0.0), (BC_PERIODIC,) * 6,
                   notes={"axis": axis, "u": 1.0, "p": 1.0, "rho": (1.0, 0.5),
                          "a0": 0.5, "a1": 0.25})


def entropy_wave_prims(pb: Problem, cell_average: bool = True) -> np.ndarray:
    """α_1 = a0 + a1 sin(2πs) along `axis`, ρ_1 = 1, ρ_2 = 0.5, u = 1, p = 1.
    With cell_average=True, α_1 and the partial densities are exact cell averages
    (AMB-19), which are linear in α."""
    ax = pb.notes["axis"]
    X = pb.centres()[ax]
    h = pb.dx[ax]
    a0, a1 = pb.notes["a0"], pb.notes["a1"]
    if cell_average:
        xl, xr = X - 0.5 * h, X + 0.5 * h
        s = (np.cos(2 * np.pi * xl) - np.cos(2 * np.pi * xr)) / (2 * np.pi * h)
    else:
        s = np.sin(2 * np.pi * X)
    a_1 = a0 + a1 * s
    a_2 = 1.0 - a_1
    r1, r2 = pb.notes["rho"]
    vel = [np.zeros_like(a_1) for _ in range(3)]
    vel[ax] = vel[ax] + pb.notes["u"]
    p = pb.notes["p"] * np.ones_like(a_1)
    return _assemble(pb, [a_1 * r1, a_2 * r2], vel, p, [a_1, a_2])


def prims_for(pb: Problem, seed: int = SEED) -> np.ndarray:
    """Dispatch by config name."""
    name = pb.name
    if name.startswith("C1"):
        return c1_prims(pb)
    if name.startswith("C2"):
        return c2_prims(pb)
    if name.startswith("C3"):
        return c3_prims(pb)
    if name.startswith("C5"):
        return c5_prims(pb)
    if name.startswith("G-R"):
        return random_prims(pb, seed)
    if name.startswith("entropy"):
        return entropy_wave_prims(pb)
    raise KeyError(name)


CONFIGS = {
    "C1": c1_water_air,
    "C2": c2_shock_bubble,
    "C3": c3_droplet,
    "C5": c5_three_fluid,
}
