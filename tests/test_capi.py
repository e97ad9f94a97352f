"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/mfc.h
declares, validates arguments, and its host-side layout / decomposition bookkeeping
is consistent (no GPU needed: contexts touch the device only when launching work)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2409_10729_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mfc():
    from paper_2409_10729_b200 import build
    build.build()
    from paper_2409_10729_b200 import mfc as m
    return m


def _declared():
    src = open(os.path.join(ROOT, "include", "mfc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mfc_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(mfc):
    declared = _declared()
    assert len(declared) >= 18
    lib = ctypes.CDLL(mfc.SO_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(mfc.EXPORTED)
    assert "sm_100a" in mfc.version()


def test_library_is_sm100a_cubin():
    import subprocess
    so = os.path.join(ROOT, "paper_2409_10729_b200", "libmfc.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _init(mfc, pb, procs=(1, 1, 1), rank=0, nranks=1, gamma=None, pinf=None, bc=None,
          transport=1):
    g = mfc._Grid()
    g.ndim = pb.ndim
    for k in range(3):
        g.n_global[k] = pb.n[k]
        g.lo[k], g.hi[k] = pb.lo[k], pb.hi[k]
        g.procs[k] = procs[k]
    N = pb.n_fluids
    gam = (ctypes.c_double * N)(*(gamma or pb.gamma))
    pi = (ctypes.c_double * N)(*(pinf or pb.pi_inf))
    b = (ctypes.c_int32 * 6)(*(bc or pb.bc))
    c = mfc._Comm()
    c.rank, c.nranks, c.loopback = rank, nranks, transport
    h = ctypes.c_void_p()
    rc = mfc.lib.mfc_init(ctypes.byref(h), ctypes.byref(g), N, gam, pi, b, ctypes.byref(c), 0)
    if rc == 0:
        mfc.lib.mfc_finalize(h)
    return rc, mfc.lib.mfc_last_error().decode()


def test_argument_validation(mfc):
    pb = W.random_problem(3, (16, 16, 16), 2, "water")
    assert _init(mfc, pb)[0] == 0
    assert _init(mfc, pb, gamma=(1.0, 1.4))[0] == -1               # gamma <= 1
    assert _init(mfc, pb, pinf=(-1.0, 0.0))[0] == -1               # pi_inf < 0
    assert _init(mfc, pb, bc=(-1, -3, -1, -1, -1, -1))[0] == -1    # periodic on one end
    assert _init(mfc, pb, bc=(-7,) * 6)[0] == -1                   # unknown bc
    assert _init(mfc, pb, procs=(1, 1, 2), nranks=3)[0] == -1      # prod(procs) != nranks
    assert _init(mfc, pb, procs=(1, 1, 8), nranks=8)[0] == -1      # 2 cells per rank < 3
    rc, msg = _init(mfc, W.Problem("bad", 4, 1, (8, 1, 1), gamma=(1.4,) * 4, pi_inf=(0,) * 4))
    assert rc == -1 and "n_fluids" in msg
    assert _init(mfc, pb, transport=4)[0] == -1                    # unknown transport
    rc, msg = _init(mfc, pb, procs=(1, 1, 2), nranks=2, transport=mfc.TRANSPORT_NCCL_SELF)
    assert rc == -1 and "one-rank" in msg                          # NCCL self: 1 rank only


def test_layout_alignment_and_sizes(mfc):
    for pb in (W.c1_water_air(), W.c2_shock_bubble(), W.c3_droplet(256), W.c5_three_fluid(64),
               W.random_problem(3, (37, 5, 9), 3, "gas")):
        L, nb = mfc.describe(pb)
        assert L.E == pb.E and L.n_local == pb.n and nb == (-1,) * 6
        assert L.stride[3] == 1 and L.stride[2] % 4 == 0            # 32-byte rows
        assert (L.offset % L.stride[2]) % 4 == 0                     # interior x 32 B aligned
        assert L.dims[3] >= pb.n[0] + 4 + 3
        for k in range(1, 3):
            assert L.dims[3 - k] == (pb.n[k] + 6 if k < pb.ndim else 1)
        assert L.n_elems == np.prod(L.dims)
        assert L.workspace_bytes >= 3 * 8 * L.n_elems


@pytest.mark.parametrize("procs", [(1, 1, 4), (1, 2, 2), (2, 2, 2), (1, 1, 3), (2, 1, 3)])
@pytest.mark.parametrize("periodic", [True, False])
def test_decomposition_bookkeeping(mfc, procs, periodic):
    """Extents tile the global grid; neighbour relations are symmetric; periodic wrap."""
    bc = W.BC_PERIODIC if periodic else W.BC_EXTRAPOLATION
    pb = W.random_problem(3, (26, 19, 31), 2, "gas", bc=bc)
    P = int(np.prod(procs))
    info = [mfc.describe(pb, procs, r, P) for r in range(P)]
    cover = np.zeros(pb.n[::-1], dtype=int)
    for L, nb in info:
        lo, n = L.lo_global, L.n_local
        cover[lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]] += 1
    assert np.all(cover == 1)
    for r, (L, nb) in enumerate(info):
        for f in range(6):
            k = f // 2
            if procs[k] == 1 or (not periodic and
                                 ((f % 2 == 0 and L.lo_global[k] == 0) or
                                  (f % 2 == 1 and L.lo_global[k] + L.n_local[k] == pb.n[k]))):
                assert nb[f] == -1
            else:
                o = nb[f]
                assert 0 <= o < P and info[o][1][f ^ 1] == r
                # the neighbour's face is adjacent (mod the global extent)
                Lo = info[o][0]
                if f % 2:
                    assert (L.lo_global[k] + L.n_local[k]) % pb.n[k] == Lo.lo_global[k]
                else:
                    assert (Lo.lo_global[k] + Lo.n_local[k]) % pb.n[k] == L.lo_global[k]


def test_new_entry_points_validate_arguments(mfc):
    """mfc_set_weno_order / _mapped / _eps / mfc_cfl_dt / mfc_rk3_steps reject bad
    arguments before touching the GPU."""
    pb = W.random_problem(3, (8, 8, 8), 2, "gas")
    g = mfc._Grid()
    g.ndim = 3
    for k in range(3):
        g.n_global[k], g.lo[k], g.hi[k], g.procs[k] = 8, 0.0, 1.0, 1
    gam = (ctypes.c_double * 2)(1.4, 1.6)
    pi = (ctypes.c_double * 2)(0.0, 0.0)
    b = (ctypes.c_int32 * 6)(*pb.bc)
    c = mfc._Comm()
    c.rank, c.nranks, c.loopback = 0, 1, 0
    h = ctypes.c_void_p()
    assert mfc.lib.mfc_init(ctypes.byref(h), ctypes.byref(g), 2, gam, pi, b, ctypes.byref(c), 0) == 0
    try:
        assert mfc.lib.mfc_set_weno_order(h, 4) == -1
        assert mfc.lib.mfc_set_weno_order(h, 3) == 0
        assert mfc.lib.mfc_set_weno_order(h, 5) == 0
        assert mfc.lib.mfc_set_weno_mapped(h, 2) == -1
        assert mfc.lib.mfc_set_weno_mapped(h, 1) == 0
        assert mfc.lib.mfc_set_weno_mapped(h, 0) == 0
        assert mfc.lib.mfc_set_weno_mapped(None, 1) == -1
        assert mfc.lib.mfc_set_weno_eps(h, 0.5) == -1
        assert mfc.lib.mfc_set_weno_eps(h, 1e-40) == -1   # (4 eps)^8 would be subnormal
        assert mfc.lib.mfc_set_weno_eps(h, 1e-30) == 0
        assert mfc.lib.mfc_set_weno_eps(h, 1e-16) == 0
        dt = ctypes.c_double(0.0)
        assert mfc.lib.mfc_cfl_dt(h, None, 0.4, ctypes.byref(dt), None, None) == -1
        assert mfc.lib.mfc_rk3_steps(h, None, 1e-3, 1, None) != 0
        assert mfc.lib.mfc_rk3_steps(h, None, float("nan"), 1, None) == -1
        assert mfc.lib.mfc_rk3_step(h, None, 1e-3, None) != 0   # no workspace / NULL q
        assert mfc.lib.mfc_comm_status(h) == 0                   # no NCCL communicator
        assert mfc.lib.mfc_comm_status(None) == -1
    finally:
        mfc.lib.mfc_finalize(h)


def test_ndim_needs_three_cells(mfc):
    rc, msg = _init(mfc, W.Problem("tiny", 2, 2, (8, 2, 1), gamma=(1.4, 1.4), pi_inf=(0, 0)))
    assert rc == -1 and "< 3" in msg
    # a split dimension whose subdomains would be thinner than the ghost depth (the
    # message reports the extent, read before the context is released)
    pb = W.random_problem(3, (8, 8, 8), 2, "gas")
    rc, msg = _init(mfc, pb, procs=(1, 1, 4), rank=0, nranks=4)
    assert rc == -1 and "local extent 2 < 3" in msg


def _ctx(mfc, pb, procs, rank, nranks, transport):
    g = mfc._Grid()
    g.ndim = pb.ndim
    for k in range(3):
        g.n_global[k] = pb.n[k]
        g.lo[k], g.hi[k] = pb.lo[k], pb.hi[k]
        g.procs[k] = procs[k]
    N = pb.n_fluids
    gam = (ctypes.c_double * N)(*pb.gamma)
    pi = (ctypes.c_double * N)(*pb.pi_inf)
    b = (ctypes.c_int32 * 6)(*pb.bc)
    c = mfc._Comm()
    c.rank, c.nranks, c.loopback = rank, nranks, transport
    h = ctypes.c_void_p()
    rc = mfc.lib.mfc_init(ctypes.byref(h), ctypes.byref(g), N, gam, pi, b, ctypes.byref(c), 0)
    return rc, h


def test_fused_halo_entry_points_validate_arguments(mfc):
    """mfc_fused_halo_group / mfc_peer_export / mfc_peer_import reject bad use before
    touching the GPU; the group attach itself is host bookkeeping."""
    pb = W.random_problem(3, (12, 12, 12), 2, "gas")
    assert _ctx(mfc, pb, (1, 1, 2), 0, 2, 3)[0] == -1                 # unknown transport
    hs = []
    for r in range(2):
        rc, h = _ctx(mfc, pb, (1, 1, 2), r, 2, mfc.TRANSPORT_LOOPBACK)
        assert rc == 0
        hs.append(h)
    try:
        H = (ctypes.c_void_p * 2)(*[h.value for h in hs])
        Q = (ctypes.c_void_p * 2)(256, 512)
        assert mfc.lib.mfc_fused_halo_group(H, Q, 2) == -5              # no workspace
        lay = mfc._Layout()
        mfc.lib.mfc_get_layout(hs[0], ctypes.byref(lay))
        for h in hs:     # a fake aligned address: binding only records the split
            assert mfc.lib.mfc_bind_workspace(h, ctypes.c_void_p(1 << 20), lay.workspace_bytes) == 0
        Qbad = (ctypes.c_void_p * 2)(256, 0)
        assert mfc.lib.mfc_fused_halo_group(H, Qbad, 2) == -1           # NULL q
        assert mfc.lib.mfc_fused_halo_group(H, Q, 1) == -1              # group lacks rank 1
        assert mfc.lib.mfc_fused_halo_group(H, Q, 2) == 0
        blob = ctypes.create_string_buffer(mfc.PEER_BLOB_BYTES)
        assert mfc.lib.mfc_peer_export(hs[0], ctypes.c_void_p(256), blob) == -1   # loopback
        assert mfc.lib.mfc_peer_import(hs[0], 0, blob) == -1           # x face: no neighbour
    finally:
        for h in hs:
            mfc.lib.mfc_finalize(h)
    rc, h = _ctx(mfc, pb, (1, 1, 2), 0, 2, mfc.TRANSPORT_PEER)           # no NCCL needed
    assert rc == 0
    try:
        blob = ctypes.create_string_buffer(mfc.PEER_BLOB_BYTES)
        assert mfc.lib.mfc_peer_import(h, 4, blob) == -5                # export first
        assert mfc.lib.mfc_peer_import(h, 7, blob) == -1                # bad face
        assert mfc.lib.mfc_peer_export(h, ctypes.c_void_p(256), blob) == -5   # no workspace
    finally:
        mfc.lib.mfc_finalize(h)


def test_face_blobs_routes_each_face_to_its_neighbour(mfc):
    blobs = [b"r0", b"r1", b"r2", b"r3"]
    assert mfc.face_blobs((-1, -1, 2, 2, 1, 3), blobs) == {2: b"r2", 3: b"r2", 4: b"r1", 5: b"r3"}
    assert mfc.face_blobs((-1,) * 6, blobs) == {}
