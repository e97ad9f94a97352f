"""ctypes wrapper of the plain-C oracle (mfc_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Array conventions (oracle-private, independent of the CUDA path's layout):
  interior arrays: float64, shape (E, nz, ny, nx), C-contiguous, x fastest;
  padded arrays:   float64, shape (E, P2, P1, P0) with P_k = n_k + 6 for an active
                   dimension and 1 otherwise (3 ghost layers per side).
Variable order (SURVEY §8 notation): conserved q = (α_iρ_i [N], ρu_k [d], ρE, α_i [N]),
primitive v = (α_iρ_i [N], u_k [d], p, α_i [N]).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "build", "lib", "Problem", "num_eq", "pad", "unpad", "constants", "cons_to_prim",
    "prim_to_cons", "weno5_minus", "nu_cell_coeffs", "weno5nu_minus", "weno5nu_plus",
    "extend_boundaries", "weno5_plus", "weno5m_minus", "weno5m_plus", "weno3_minus", "weno3_plus", "hllc", "fill_ghosts", "rhs",
    "rhs_padded", "rhs_cells", "rk3_combine", "rk3_step", "count_inadmissible",
    "num_threads", "set_num_threads", "max_wave_rate", "BC_EXTERNAL", "BC_PERIODIC", "BC_REFLECTIVE", "BC_EXTRAPOLATION",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mfc_oracle.c")
_HDR = os.path.join(_HERE, "mfc_oracle.h")
_SO = os.path.join(_HERE, "liboracle.so")
G = 3
MAXF = 3

BC_EXTERNAL = 0
BC_PERIODIC = -1
BC_REFLECTIVE = -2
BC_EXTRAPOLATION = -3


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2 -ffp-contract=off, OpenMP)."""
    stale = (not os.path.exists(_SO)) or any(
        os.path.getmtime(s) > os.path.getmtime(_SO) for s in (_SRC, _HDR))
    if force or stale:
        tmp = _SO + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _SO)
    return _SO


class _OrcProblem(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int32),
        ("d", ctypes.c_int32),
        ("n", ctypes.c_int32 * 3),
        ("dx", ctypes.c_double * 3),
        ("bc", ctypes.c_int32 * 6),
        ("gamma", ctypes.c_double * MAXF),
        ("pi_inf", ctypes.c_double * MAXF),
        ("eps", ctypes.c_double),
        ("weno_order", ctypes.c_int32),
        ("weno_mapped", ctypes.c_int32),
        ("xb", ctypes.c_void_p * 3),
    ]


class _NuCell(ctypes.Structure):
    _fields_ = [("M", ctypes.c_double * 27), ("dm", ctypes.c_double * 3),
                ("dp", ctypes.c_double * 3), ("w", ctypes.c_double)]


_lib = None
_lock = threading.Lock()
_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            P = ctypes.POINTER(_OrcProblem)
            sig = {
                "orc_num_eq": (ctypes.c_int32, [ctypes.c_int32, ctypes.c_int32]),
                "orc_padded_cells": (ctypes.c_int64, [P]),
                "orc_constants": (None, [P, _dp, _dp]),
                "orc_cons_to_prim": (None, [P, ctypes.c_int64, _dp, _dp]),
                "orc_prim_to_cons": (None, [P, ctypes.c_int64, _dp, _dp]),
                "orc_weno5_minus": (ctypes.c_double, [ctypes.c_double] * 6 + [_dp]),
                "orc_weno5_plus": (ctypes.c_double, [ctypes.c_double] * 6 + [_dp]),
                "orc_weno5m_minus": (ctypes.c_double, [ctypes.c_double] * 6 + [_dp]),
                "orc_weno5m_plus": (ctypes.c_double, [ctypes.c_double] * 6 + [_dp]),
                "orc_nu_cell_coeffs": (ctypes.c_int32, [_dp, ctypes.POINTER(_NuCell)]),
                "orc_weno5nu_minus": (ctypes.c_double, [ctypes.POINTER(_NuCell)] +
                                      [ctypes.c_double] * 6 + [_dp]),
                "orc_weno5nu_plus": (ctypes.c_double, [ctypes.POINTER(_NuCell)] +
                                     [ctypes.c_double] * 6 + [_dp]),
                "orc_weno3_minus": (ctypes.c_double, [ctypes.c_double] * 4 + [_dp]),
                "orc_weno3_plus": (ctypes.c_double, [ctypes.c_double] * 4 + [_dp]),
                "orc_hllc": (None, [P, _dp, _dp, ctypes.c_int32, _dp, _dp, _dp, _dp]),
                "orc_fill_ghosts": (None, [P, _dp]),
                "orc_rhs": (None, [P, _dp, _dp]),
                "orc_rhs_cells": (None, [P, _dp, ctypes.c_int64, _i64p, _dp]),
                "orc_rk3_combine": (None, [ctypes.c_int32, ctypes.c_int64, _dp, _dp, _dp,
                                           ctypes.c_double, _dp]),
                "orc_rk3_step": (None, [P, _dp, ctypes.c_double]),
                "orc_count_inadmissible": (ctypes.c_int64, [P, _dp]),
                "orc_max_wave_rate": (ctypes.c_double, [P, _dp]),
                "orc_num_threads": (ctypes.c_int32, []),
                "orc_set_num_threads": (None, [ctypes.c_int32]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


@dataclass
class Problem:
    """Oracle problem description: N fluids, d active dims, n = (nx, ny, nz)."""
    N: int
    d: int
    n: tuple
    dx: tuple
    bc: tuple
    gamma: tuple
    pi_inf: tuple
    eps: float = 1e-16
    weno_order: int = 5
    weno_mapped: int = 0
    # non-uniform grid (F4): per axis None (uniform dx) or the cell boundaries, either the
    # n+1 interior boundaries (ghost cells added by extend_boundaries from this
    # problem's BCs) or all n+7 (ghosts included, e.g. for BC_EXTERNAL faces)
    x_cb: tuple = (None, None, None)
    _c: _OrcProblem = field(default=None, repr=False, compare=False)
    _xb: list = field(default=None, repr=False, compare=False)

    @classmethod
    def from_spec(cls, spec, bc=None, eps=None):
        """Duck-typed: any object with n_fluids, ndim, n, dx, bc, gamma, pi_inf, weno_eps
        (and optionally x_cb: per-axis cell boundaries of a stretched grid)."""
        return cls(N=spec.n_fluids, d=spec.ndim, n=tuple(spec.n), dx=tuple(spec.dx),
                   bc=tuple(spec.bc if bc is None else bc), gamma=tuple(spec.gamma),
                   pi_inf=tuple(spec.pi_inf),
                   eps=float(getattr(spec, "weno_eps", 1e-16) if eps is None else eps),
                   weno_order=int(getattr(spec, "weno_order", 5)),
                   weno_mapped=int(bool(getattr(spec, "weno_mapped", False))),
                   x_cb=tuple(getattr(spec, "x_cb", None) or (None, None, None)))

    def __post_init__(self):
        n = list(self.n) + [1] * (3 - len(self.n))
        self.n = tuple(int(x) for x in n)
        dx = list(self.dx) + [1.0] * (3 - len(self.dx))
        self.dx = tuple(float(x) for x in dx)
        c = _OrcProblem()
        c.N, c.d = int(self.N), int(self.d)
        for k in range(3):
            c.n[k] = self.n[k]
            c.dx[k] = self.dx[k]
        for k in range(6):
            c.bc[k] = int(self.bc[k])
        for i in range(MAXF):
            c.gamma[i] = float(self.gamma[i]) if i < self.N else 0.0
            c.pi_inf[i] = float(self.pi_inf[i]) if i < self.N else 0.0
        c.eps = float(self.eps)
        c.weno_order = int(self.weno_order)
        c.weno_mapped = int(self.weno_mapped)
        xcb = list(self.x_cb) + [None] * (3 - len(self.x_cb))
        self.x_cb = tuple(xcb[:3])
        self._xb = [None, None, None]
        for k in range(3):
            if xcb[k] is None or k >= self.d:
                c.xb[k] = None
                continue
            assert self.weno_order == 5 and not self.weno_mapped, \
                "stretched grids: WENO5-JS only (DESIGN.md AMB-27)"
            xb = np.ascontiguousarray(xcb[k], dtype=np.float64)
            if xb.size == self.n[k] + 1:
                xb = extend_boundaries(xb, self.bc[2 * k], self.bc[2 * k + 1])
            assert xb.size == self.n[k] + 7 and np.all(np.diff(xb) > 0)
            self._xb[k] = xb                      # keeps the memory alive
            c.xb[k] = xb.ctypes.data
        self._c = c

    @property
    def E(self) -> int:
        return 2 * self.N + self.d + 1

    @property
    def padded_shape(self):
        p = [self.n[k] + 2 * G if k < self.d else 1 for k in range(3)]
        return (self.E, p[2], p[1], p[0])

    @property
    def interior_shape(self):
        return (self.E, self.n[2], self.n[1], self.n[0])

    def ptr(self):
        return ctypes.byref(self._c)

    def with_bc(self, bc):
        return Problem(self.N, self.d, self.n, self.dx, tuple(bc), self.gamma, self.pi_inf,
                       self.eps, self.weno_order, self.weno_mapped, self.x_cb)


def extend_boundaries(xb: np.ndarray, bc_lo: int, bc_hi: int) -> np.ndarray:
    """S1 for the grid (DESIGN.md AMB-27): the 3 ghost cells on each side of a stretched
    axis get the widths of the interior cells their DATA come from (periodic
    -1-j <- n-1-j, reflective -1-j <- j, extrapolation <- the boundary cell), laid
    out outward from the boundary; n+1 interior boundaries -> n+7."""
    xb = np.asarray(xb, dtype=np.float64)
    n = xb.size - 1
    w = np.diff(xb)

    def src(g):                      # interior cell whose data ghost cell g (< 0 or >= n) holds
        if g < 0:
            j = -1 - g
            return {BC_PERIODIC: n - 1 - j, BC_REFLECTIVE: j}.get(bc_lo, 0)
        j = g - n
        return {BC_PERIODIC: j, BC_REFLECTIVE: n - 1 - j}.get(bc_hi, n - 1)

    lo = [xb[0]]
    for g in range(-1, -4, -1):
        lo.append(lo[-1] - w[src(g)])
    hi = [xb[-1]]
    for g in range(n, n + 3):
        hi.append(hi[-1] + w[src(g)])
    return np.concatenate([lo[:0:-1], xb, hi[1:]])


def num_eq(N: int, d: int) -> int:
    return int(lib().orc_num_eq(N, d))


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def _interior_slices(P: Problem):
    sl = [slice(G, G + P.n[k]) if k < P.d else slice(0, 1) for k in range(3)]
    return (slice(None), sl[2], sl[1], sl[0])


def pad(P: Problem, q: np.ndarray) -> np.ndarray:
    """Interior (E, nz, ny, nx) -> padded array with zero ghosts."""
    out = np.zeros(P.padded_shape, dtype=np.float64)
    out[_interior_slices(P)] = q
    return out


def unpad(P: Problem, qp: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(qp[_interior_slices(P)])


def constants(P: Problem):
    G_ = np.zeros(MAXF)
    Pi = np.zeros(MAXF)
    lib().orc_constants(P.ptr(), _p(G_), _p(Pi))
    return G_[:P.N].copy(), Pi[:P.N].copy()


def cons_to_prim(P: Problem, q: np.ndarray) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.float64)
    assert q.shape[0] == P.E
    v = np.empty_like(q)
    lib().orc_cons_to_prim(P.ptr(), q[0].size, _p(q), _p(v))
    return v


def prim_to_cons(P: Problem, v: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float64)
    assert v.shape[0] == P.E
    q = np.empty_like(v)
    lib().orc_prim_to_cons(P.ptr(), v[0].size, _p(v), _p(q))
    return q


def weno5_minus(a, b, c, d, e, eps=1e-16):
    w = np.zeros(3)
    val = lib().orc_weno5_minus(a, b, c, d, e, eps, _p(w))
    return val, w


def weno5_plus(a, b, c, d, e, eps=1e-16):
    w = np.zeros(3)
    val = lib().orc_weno5_plus(a, b, c, d, e, eps, _p(w))
    return val, w


def weno5m_minus(a, b, c, d, e, eps=1e-16):
    w = np.zeros(3)
    val = lib().orc_weno5m_minus(a, b, c, d, e, eps, _p(w))
    return val, w


def weno5m_plus(a, b, c, d, e, eps=1e-16):
    w = np.zeros(3)
    val = lib().orc_weno5m_plus(a, b, c, d, e, eps, _p(w))
    return val, w


def nu_cell_coeffs(xb6):
    """Non-uniform WENO5 ingredients of one cell from its 6 stencil boundaries:
    (M[3][3][3], dm[3], dp[3], width, status)."""
    xb6 = np.ascontiguousarray(xb6, dtype=np.float64)
    assert xb6.size == 6
    C = _NuCell()
    st = lib().orc_nu_cell_coeffs(_p(xb6), ctypes.byref(C))
    return C, int(st)


def weno5nu_minus(C, a, b, c, d, e, eps=1e-16):
    w = np.zeros(3)
    return lib().orc_weno5nu_minus(ctypes.byref(C), a, b, c, d, e, eps, _p(w)), w


def weno5nu_plus(C, a, b, c, d, e, eps=1e-16):
    w = np.zeros(3)
    return lib().orc_weno5nu_plus(ctypes.byref(C), a, b, c, d, e, eps, _p(w)), w


def weno3_minus(a, b, c, eps=1e-16):
    w = np.zeros(2)
    val = lib().orc_weno3_minus(a, b, c, eps, _p(w))
    return val, w


def weno3_plus(a, b, c, eps=1e-16):
    w = np.zeros(2)
    val = lib().orc_weno3_plus(a, b, c, eps, _p(w))
    return val, w


def hllc(P: Problem, direction: int, vL, vR):
    G_, Pi = constants(P)
    G_ = np.ascontiguousarray(np.pad(G_, (0, MAXF - P.N)))
    Pi = np.ascontiguousarray(np.pad(Pi, (0, MAXF - P.N)))
    vL = np.ascontiguousarray(vL, dtype=np.float64)
    vR = np.ascontiguousarray(vR, dtype=np.float64)
    F = np.zeros(P.E)
    uf = ctypes.c_double(0.0)
    lib().orc_hllc(P.ptr(), _p(G_), _p(Pi), direction, _p(vL), _p(vR), _p(F),
                   ctypes.byref(uf))
    return F, uf.value


def fill_ghosts(P: Problem, qp: np.ndarray) -> None:
    assert qp.shape == P.padded_shape
    lib().orc_fill_ghosts(P.ptr(), _p(qp))


def rhs_padded(P: Problem, qp: np.ndarray) -> np.ndarray:
    """L(q) on a padded array (ghosts filled in place by the BCs; external faces untouched)."""
    assert qp.shape == P.padded_shape
    out = np.empty_like(qp)
    lib().orc_rhs(P.ptr(), _p(qp), _p(out))
    return out


def rhs(P: Problem, q: np.ndarray) -> np.ndarray:
    """L(q) for an interior array (E, nz, ny, nx)."""
    qp = pad(P, np.asarray(q, dtype=np.float64))
    return unpad(P, rhs_padded(P, qp))


def rhs_cells(P: Problem, qp: np.ndarray, cells: np.ndarray) -> np.ndarray:
    """RHS at the given interior cells ((ncells, 3) int64 of i, j, k), ghosts of qp filled."""
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    assert cells.ndim == 2 and cells.shape[1] == 3
    out = np.empty((cells.shape[0], P.E))
    lib().orc_rhs_cells(P.ptr(), _p(qp), cells.shape[0], cells.ctypes.data_as(_i64p), _p(out))
    return out


def rk3_combine(stage: int, qn: np.ndarray, qs: np.ndarray, L: np.ndarray, dt: float):
    qn, qs, L = (np.ascontiguousarray(a, dtype=np.float64) for a in (qn, qs, L))
    out = np.empty_like(qs)
    lib().orc_rk3_combine(stage, qs.size, _p(qn), _p(qs), _p(L), dt, _p(out))
    return out


def rk3_step(P: Problem, q: np.ndarray, dt: float, nsteps: int = 1) -> np.ndarray:
    qp = pad(P, np.asarray(q, dtype=np.float64))
    for _ in range(nsteps):
        lib().orc_rk3_step(P.ptr(), _p(qp), float(dt))
    return unpad(P, qp)


def count_inadmissible(P: Problem, q: np.ndarray) -> int:
    qp = pad(P, np.asarray(q, dtype=np.float64))
    return int(lib().orc_count_inadmissible(P.ptr(), _p(qp)))


def max_wave_rate(P: Problem, q: np.ndarray) -> float:
    """max over interior cells of max_k (|u_k| + c)/dx_k (dt = CFL / rate)."""
    qp = pad(P, np.asarray(q, dtype=np.float64))
    return float(lib().orc_max_wave_rate(P.ptr(), _p(qp)))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))
