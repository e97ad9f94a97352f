"""Pins of the oracle's S1 ghost fill for the physical boundary conditions (SURVEY §8(c)
S1, DESIGN.md AMB-13; the paper describes no BCs) by identities that follow from what
the conditions MEAN, not from their implementation:

* reflective wall = mirror symmetry.  A field on [0, L] with reflective walls at both
  ends is the restriction of its mirror image on the periodic domain [-L, L]: cell
  -1-j of the doubled domain is cell j reflected (normal momentum negated, every other
  conserved variable even).  Every stencil of a cell in [0, L] then sees exactly the
  values the reflective ghosts hold, so the RHS on [0, L] is BITWISE the periodic
  doubled domain's RHS there.  A wrong mirror index (ghost -1-j <- j+1), a wrong
  negated component (tangential instead of normal momentum) or a missing negation
  breaks it.
* extrapolation = zeroth-order extension.  Extrapolated ghosts are copies of the
  adjacent interior cell, so the RHS equals, bitwise, that of the domain extended by 3
  cells that are copies of the boundary cell (interior cells there, so no BC is
  involved in the compared stencils).  Ghost <- the second cell, or a mirrored index,
  breaks it, for arbitrary (non-uniform) data.

Every axis, both sides, N = 1..3.  The same identities are checked on the GPU in
tests/test_gpu_parity.py."""
import numpy as np
import pytest

import oracle as O
from paper_2409_10729_b200 import workloads as W


def _prob(N, n, bc, mats="gas"):
    pb = W.random_problem(3, n, N, mats)
    return O.Problem(N=N, d=3, n=tuple(n), dx=(0.1, 0.1, 0.1), bc=tuple(bc),
                     gamma=pb.gamma, pi_inf=pb.pi_inf), pb


def _cons(N, n, mats, seed):
    P, pb = _prob(N, n, (W.BC_PERIODIC,) * 6, mats)
    return O.prim_to_cons(P, W.random_prims(pb, seed=seed))


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("N,mats", [(1, "gas"), (2, "water"), (3, "gas")])
def test_reflective_wall_is_the_mirrored_periodic_domain(axis, N, mats):
    n = [9, 8, 7]
    q = _cons(N, n, mats, seed=11 + axis)
    ax = 3 - axis                                  # array axis of `axis` in (E, z, y, x)
    mirror = np.flip(q, axis=ax).copy()
    mirror[N + axis] = -mirror[N + axis]           # normal momentum is odd
    full = np.concatenate([mirror, q], axis=ax)    # [-L, 0) mirrored, [0, L) = q
    nf = list(n)
    nf[axis] = 2 * n[axis]
    bc_half = [W.BC_PERIODIC] * 6
    bc_half[2 * axis] = bc_half[2 * axis + 1] = W.BC_REFLECTIVE
    P_half, _ = _prob(N, n, bc_half, mats)
    P_full, _ = _prob(N, nf, (W.BC_PERIODIC,) * 6, mats)
    r_half = O.rhs(P_half, q)
    r_full = O.rhs(P_full, full)
    sl = [slice(None)] * 4
    sl[ax] = slice(n[axis], 2 * n[axis])
    assert np.array_equal(r_full[tuple(sl)], r_half)
    # the identity is not vacuous: the wall matters for this field
    assert not np.array_equal(O.rhs(P_half.with_bc((W.BC_PERIODIC,) * 6), q), r_half)


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("side", [0, 1])
@pytest.mark.parametrize("N,mats", [(1, "gas"), (2, "water"), (3, "water")])
def test_extrapolation_is_the_constant_extension(axis, side, N, mats):
    n = [8, 7, 9]
    q = _cons(N, n, mats, seed=21 + 2 * axis + side)
    ax = 3 - axis
    edge = [slice(None)] * 4
    edge[ax] = slice(0, 1) if side == 0 else slice(n[axis] - 1, n[axis])
    ext = np.repeat(q[tuple(edge)], 3, axis=ax)    # 3 copies of the boundary cell
    full = np.concatenate([ext, q] if side == 0 else [q, ext], axis=ax)
    ne = list(n)
    ne[axis] += 3
    bc = [W.BC_PERIODIC] * 6
    bc[2 * axis] = bc[2 * axis + 1] = W.BC_REFLECTIVE     # the other side: a wall
    bc[2 * axis + side] = W.BC_EXTRAPOLATION
    P, _ = _prob(N, n, bc, mats)
    P_ext, _ = _prob(N, ne, bc, mats)
    r = O.rhs(P, q)
    r_ext = O.rhs(P_ext, full)
    sl = [slice(None)] * 4
    sl[ax] = slice(3, 3 + n[axis]) if side == 0 else slice(0, n[axis])
    assert np.array_equal(r_ext[tuple(sl)], r)
    # not vacuous: a mirrored extension (reflective ghosts) gives another RHS
    bc2 = list(bc)
    bc2[2 * axis + side] = W.BC_REFLECTIVE
    assert not np.array_equal(O.rhs(P.with_bc(bc2), q), r)


def test_ghost_layers_written_by_the_bcs():
    """The ghost values themselves, for one line per axis, against the definitions:
    periodic -1-j <- n-1-j, extrapolation <- cell 0 / n-1, reflective -1-j <- j with
    the normal momentum negated (face ghosts only)."""
    N, n = 2, [6, 5, 4]
    q = _cons(N, n, "gas", seed=5)
    for axis in range(3):
        for bc in (W.BC_PERIODIC, W.BC_EXTRAPOLATION, W.BC_REFLECTIVE):
            bcs = [W.BC_PERIODIC] * 6
            bcs[2 * axis] = bcs[2 * axis + 1] = bc
            P, _ = _prob(N, n, bcs)
            qp = O.pad(P, q)
            O.fill_ghosts(P, qp)
            ax = 3 - axis
            line = np.moveaxis(qp, ax, -1)[:, 3, 3, :]          # (E, n+6) along axis
            inner = line[:, 3:3 + n[axis]]
            m = n[axis]
            for j in range(3):
                lo, hi = line[:, 2 - j], line[:, 3 + m + j]
                if bc == W.BC_PERIODIC:
                    want_lo, want_hi = inner[:, m - 1 - j], inner[:, j]
                elif bc == W.BC_EXTRAPOLATION:
                    want_lo, want_hi = inner[:, 0], inner[:, m - 1]
                else:
                    want_lo, want_hi = inner[:, j].copy(), inner[:, m - 1 - j].copy()
                    want_lo[N + axis] *= -1
                    want_hi[N + axis] *= -1
                assert np.array_equal(lo, want_lo) and np.array_equal(hi, want_hi), (axis, bc, j)
