"""Thin ctypes binding of libmfc.so (include/mfc.h) -- argument marshalling only.

Every step of the RHS / RK3 path runs in the library's CUDA kernels; this module
only allocates device memory with torch (the memory owner), passes pointers,
sizes and the current CUDA stream, and turns status codes into exceptions.
There is NO fallback: if libmfc.so cannot be loaded, importing this module fails.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# MFC_LIB: an alternative in-tree build (same-box A/B timing, tools/build_ab.sh)
SO_PATH = os.environ.get("MFC_LIB") or os.path.join(_HERE, "libmfc.so")

TRANSPORT_NCCL, TRANSPORT_LOOPBACK, TRANSPORT_PEER, TRANSPORT_NCCL_SELF = 0, 1, 2, 3
PEER_BLOB_BYTES = 512

BC_PERIODIC = -1
BC_REFLECTIVE = -2
BC_EXTRAPOLATION = -3

STATUS = {0: "OK", -1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENCCL", -5: "ESTATE",
          -6: "EUNSUPPORTED"}

EXPORTED = [
    "mfc_init", "mfc_get_layout", "mfc_get_neighbors", "mfc_bind_workspace", "mfc_set_weno_eps",
    "mfc_set_weno_order", "mfc_set_weno_mapped", "mfc_set_grid",
    "mfc_prim_to_cons", "mfc_cons_to_prim", "mfc_count_inadmissible", "mfc_halo_exchange", "mfc_rhs", "mfc_rk3_step",
    "mfc_rk3_steps", "mfc_max_wave_rate", "mfc_cfl_dt",
    "mfc_advance_host", "mfc_set_stream_chunks", "mfc_halo_exchange_group", "mfc_rhs_group", "mfc_rk3_step_group",
    "mfc_fused_halo_group", "mfc_peer_export", "mfc_peer_import",
    "mfc_nccl_get_unique_id", "mfc_comm_status", "mfc_last_launch_count", "mfc_profile_enable", "mfc_profile_read", "mfc_finalize", "mfc_last_error",
    "mfc_version",
]


class MfcError(RuntimeError):
    pass


class _Grid(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("n_global", ctypes.c_int64 * 3),
                ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3),
                ("procs", ctypes.c_int32 * 3)]


class _Comm(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("loopback", ctypes.c_int32)]


class _Layout(ctypes.Structure):
    _fields_ = [("E", ctypes.c_int32), ("ghost", ctypes.c_int32), ("n_fluids", ctypes.c_int32),
                ("ndim", ctypes.c_int32), ("n_local", ctypes.c_int64 * 3),
                ("lo_global", ctypes.c_int64 * 3), ("dims", ctypes.c_int64 * 4),
                ("stride", ctypes.c_int64 * 4), ("offset", ctypes.c_int64),
                ("n_elems", ctypes.c_int64), ("workspace_bytes", ctypes.c_size_t)]


def _load():
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} is missing: run __graft_entry__.build() "
                          "(no CPU fallback exists)")
    L = ctypes.CDLL(SO_PATH)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    pp = ctypes.POINTER(vp)
    sig = {
        "mfc_init": [ctypes.POINTER(vp), ctypes.POINTER(_Grid), i32, ctypes.POINTER(dbl),
                     ctypes.POINTER(dbl), ctypes.POINTER(i32), ctypes.POINTER(_Comm), i32],
        "mfc_get_layout": [vp, ctypes.POINTER(_Layout)],
        "mfc_get_neighbors": [vp, ctypes.POINTER(i32)],
        "mfc_bind_workspace": [vp, vp, ctypes.c_size_t],
        "mfc_set_weno_eps": [vp, dbl],
        "mfc_set_weno_order": [vp, i32],
        "mfc_set_weno_mapped": [vp, i32],
        "mfc_set_grid": [vp, i32, ctypes.POINTER(dbl), i64],
        "mfc_prim_to_cons": [vp, vp, vp, vp],
        "mfc_cons_to_prim": [vp, vp, vp, vp],
        "mfc_count_inadmissible": [vp, vp, vp, vp],
        "mfc_halo_exchange": [vp, vp, vp],
        "mfc_rhs": [vp, vp, vp, vp],
        "mfc_rk3_step": [vp, vp, dbl, vp],
        "mfc_rk3_steps": [vp, vp, dbl, i64, vp],
        "mfc_max_wave_rate": [vp, vp, vp, vp],
        "mfc_cfl_dt": [vp, vp, dbl, ctypes.POINTER(dbl), vp, vp],
        "mfc_advance_host": [vp, vp, vp, vp, i64, dbl, vp],
        "mfc_set_stream_chunks": [vp, i32],
        "mfc_halo_exchange_group": [pp, pp, i32, vp],
        "mfc_rhs_group": [pp, pp, pp, i32, vp],
        "mfc_rk3_step_group": [pp, pp, i32, dbl, vp],
        "mfc_fused_halo_group": [pp, pp, i32],
        "mfc_peer_export": [vp, vp, vp],
        "mfc_peer_import": [vp, i32, vp],
        "mfc_nccl_get_unique_id": [vp],
        "mfc_comm_status": [vp],
        "mfc_last_launch_count": [vp],
        "mfc_profile_enable": [vp, i32],
        "mfc_profile_read": [vp, ctypes.POINTER(dbl), ctypes.POINTER(i64), i32],
        "mfc_finalize": [vp],
        "mfc_last_error": [],
        "mfc_version": [],
    }
    for name, args in sig.items():
        if os.environ.get("MFC_LIB") and not hasattr(L, name):
            continue                   # an older A/B build lacks newer entry points
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.mfc_last_launch_count.restype = i64
    L.mfc_last_error.restype = ctypes.c_char_p
    L.mfc_version.restype = ctypes.c_char_p
    return L


lib = _load()


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib.mfc_last_error().decode(errors="replace")
        raise MfcError(f"{what} failed: {STATUS.get(rc, rc)}: {msg}")


def version() -> str:
    return lib.mfc_version().decode()


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.mfc_nccl_get_unique_id(buf), "mfc_nccl_get_unique_id")
    return buf.raw


def broadcast_unique_id(src: int = 0, group=None) -> bytes:
    """Rank `src` generates the NCCL unique id; every rank of the torch.distributed
    group receives the same 128 bytes (plumbing for mfc_init with nranks > 1)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    assert isinstance(obj[0], (bytes, bytearray)) and len(obj[0]) == 128
    return bytes(obj[0])


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t: torch.Tensor):
    """Device pointer of a float64 CUDA tensor (raises, never asserts: python -O)."""
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda:
        raise ValueError("expected a float64 CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


@dataclass
class Layout:
    E: int
    ghost: int
    n_fluids: int
    ndim: int
    n_local: tuple
    lo_global: tuple
    dims: tuple
    stride: tuple
    offset: int
    n_elems: int
    workspace_bytes: int


class Solver:
    """One subdomain (rank) of the 5-equation RHS / SSP-RK3 path on one GPU."""

    def __init__(self, problem, *, procs=(1, 1, 1), rank=0, nranks=1, nccl_id: bytes | None = None,
                 loopback=False, peer=False, nccl_self=False, device=None, weno_eps=None,
                 n_global=None):
        """nccl_self: one rank whose periodic faces go through the NCCL halo path
        (send / recv to itself; MFC_TRANSPORT_NCCL_SELF, a one-GPU check of that code)."""
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        self.problem = problem
        g = _Grid()
        g.ndim = problem.ndim
        ng = problem.n if n_global is None else n_global
        for k in range(3):
            g.n_global[k] = int(ng[k])
            g.lo[k] = float(problem.lo[k])
            g.hi[k] = float(problem.hi[k])
            g.procs[k] = int(procs[k])
        N = problem.n_fluids
        gam = (ctypes.c_double * N)(*problem.gamma[:N])
        pinf = (ctypes.c_double * N)(*problem.pi_inf[:N])
        bc = (ctypes.c_int32 * 6)(*problem.bc)
        comm = _Comm()
        comm.rank, comm.nranks = rank, nranks
        comm.loopback = (TRANSPORT_NCCL_SELF if nccl_self else TRANSPORT_PEER if peer
                         else TRANSPORT_LOOPBACK if loopback else TRANSPORT_NCCL)
        self._id = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        comm.nccl_unique_id = ctypes.cast(self._id, ctypes.c_void_p) if self._id else None
        h = ctypes.c_void_p()
        _check(lib.mfc_init(ctypes.byref(h), ctypes.byref(g), N, gam, pinf, bc,
                            ctypes.byref(comm), device), "mfc_init")
        self._h = h
        lay = _Layout()
        _check(lib.mfc_get_layout(h, ctypes.byref(lay)), "mfc_get_layout")
        self.layout = Layout(lay.E, lay.ghost, lay.n_fluids, lay.ndim, tuple(lay.n_local),
                             tuple(lay.lo_global), tuple(lay.dims), tuple(lay.stride),
                             lay.offset, lay.n_elems, lay.workspace_bytes)
        nb = (ctypes.c_int32 * 6)()
        _check(lib.mfc_get_neighbors(h, nb), "mfc_get_neighbors")
        self.neighbors = tuple(nb)
        eps = weno_eps if weno_eps is not None else getattr(problem, "weno_eps", 1e-16)
        _check(lib.mfc_set_weno_eps(h, float(eps)), "mfc_set_weno_eps")
        _check(lib.mfc_set_weno_order(h, int(getattr(problem, "weno_order", 5))),
               "mfc_set_weno_order")
        _check(lib.mfc_set_weno_mapped(h, int(bool(getattr(problem, "weno_mapped", False)))),
               "mfc_set_weno_mapped")
        # torch owns the workspace (256-byte aligned by the caching allocator)
        nbytes = self.layout.workspace_bytes
        self.workspace = torch.empty((nbytes + 7) // 8, dtype=torch.float64, device=self.device)
        _check(lib.mfc_bind_workspace(h, _ptr(self.workspace), nbytes), "mfc_bind_workspace")
        # stretched axes (F4): the global cell boundaries of each
        for k, xb in enumerate(getattr(problem, "x_cb", None) or ()):
            if xb is not None and k < problem.ndim:
                self.set_grid(k, xb)

    def set_grid(self, dim: int, x_cb=None):
        """Non-uniform cell boundaries of the GLOBAL axis dim (n_global+1 increasing
        values), or None for the uniform spacing (mfc_set_grid)."""
        if x_cb is None:
            _check(lib.mfc_set_grid(self._h, int(dim), None, 0), "mfc_set_grid")
            return
        x = np.ascontiguousarray(x_cb, dtype=np.float64)
        _check(lib.mfc_set_grid(self._h, int(dim), x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                x.size - 1), "mfc_set_grid")

    # ------------------------------------------------------------- buffers
    def empty_state(self) -> torch.Tensor:
        return torch.zeros(self.layout.n_elems, dtype=torch.float64, device=self.device)

    def interior(self, t: torch.Tensor) -> torch.Tensor:
        """(E, nz, ny, nx) strided view of the interior cells of a state buffer."""
        L = self.layout
        nx, ny, nz = L.n_local
        if t.dim() != 1 or not t.is_contiguous() or t.numel() < L.n_elems:
            raise ValueError(f"state buffer needs >= {L.n_elems} contiguous float64 elements")
        # as_strided's offset counts from the start of the STORAGE: a buffer that is itself
        # a view (t.storage_offset() > 0) starts that far in
        return t.as_strided((L.E, nz, ny, nx), (L.stride[0], L.stride[1], L.stride[2], 1),
                            t.storage_offset() + L.offset)

    def state_from_prims(self, prims: np.ndarray | torch.Tensor) -> torch.Tensor:
        """Upload primitive fields (E, nz, ny, nx) and convert them with mfc_prim_to_cons."""
        v = self.empty_state()
        self.interior(v).copy_(torch.as_tensor(prims, dtype=torch.float64))
        q = self.empty_state()
        self.prim_to_cons(v, q)
        return q

    def state_from_cons(self, cons) -> torch.Tensor:
        q = self.empty_state()
        self.interior(q).copy_(torch.as_tensor(cons, dtype=torch.float64))
        return q

    # ------------------------------------------------------------- calls
    def _sp(self, t: torch.Tensor):
        """Pointer of a state buffer: float64, on this solver's device, contiguous and
        holding at least layout.n_elems elements (the kernels index that far)."""
        p = _ptr(t)
        if t.device != self.device:
            raise ValueError(f"state on {t.device}, solver on {self.device}")
        if not t.is_contiguous() or t.numel() < self.layout.n_elems:
            raise ValueError(f"state buffer needs >= {self.layout.n_elems} contiguous float64 "
                             f"elements (got {t.numel()})")
        return p

    def prim_to_cons(self, v, q, stream=None):
        _check(lib.mfc_prim_to_cons(self._h, self._sp(v), self._sp(q), _stream(stream)),
               "mfc_prim_to_cons")

    def cons_to_prim(self, q, v, stream=None):
        _check(lib.mfc_cons_to_prim(self._h, self._sp(q), self._sp(v), _stream(stream)),
               "mfc_cons_to_prim")

    def halo_exchange(self, q, stream=None):
        _check(lib.mfc_halo_exchange(self._h, self._sp(q), _stream(stream)), "mfc_halo_exchange")

    def rhs(self, q, out=None, stream=None) -> torch.Tensor:
        if out is None:
            out = self.empty_state()
        _check(lib.mfc_rhs(self._h, self._sp(q), self._sp(out), _stream(stream)), "mfc_rhs")
        return out

    def rk3_step(self, q, dt: float, stream=None):
        _check(lib.mfc_rk3_step(self._h, self._sp(q), float(dt), _stream(stream)), "mfc_rk3_step")

    def max_wave_rate(self, q, out=None, stream=None) -> torch.Tensor:
        """Device scalar: max over cells (and ranks) of max_k (|u_k|+c)/dx_k."""
        if out is None:
            out = torch.zeros(1, dtype=torch.float64, device=self.device)
        if out.device != self.device or out.numel() < 1:
            raise ValueError("out must be a float64 tensor on the solver's device")
        _check(lib.mfc_max_wave_rate(self._h, self._sp(q), _ptr(out), _stream(stream)),
               "mfc_max_wave_rate")
        return out

    def count_inadmissible(self, q, stream=None) -> torch.Tensor:
        """Device int64: interior cells that are not finite or have rho <= 0 or c^2 <= 0."""
        out = torch.zeros(1, dtype=torch.int64, device=self.device)
        _check(lib.mfc_count_inadmissible(self._h, self._sp(q), ctypes.c_void_p(out.data_ptr()),
                                          _stream(stream)), "mfc_count_inadmissible")
        return out

    def cfl_dt(self, q, cfl: float, stream=None) -> float:
        """dt = cfl / max_wave_rate (synchronises the stream)."""
        scratch = torch.zeros(1, dtype=torch.float64, device=self.device)
        dt = ctypes.c_double(0.0)
        _check(lib.mfc_cfl_dt(self._h, self._sp(q), float(cfl), ctypes.byref(dt), _ptr(scratch),
                              _stream(stream)), "mfc_cfl_dt")
        return dt.value

    def rk3_steps(self, q, dt: float, nsteps: int, stream=None):
        """nsteps RK3 steps replayed from a CUDA graph of one step."""
        _check(lib.mfc_rk3_steps(self._h, self._sp(q), float(dt), int(nsteps), _stream(stream)),
               "mfc_rk3_steps")

    def advance_host(self, q_in: torch.Tensor, q_out: torch.Tensor, q_dev: torch.Tensor,
                     nsteps: int, dt: float, stream=None):
        """End-to-end call with host buffers (dense interior (E, nz, ny, nx) float64);
        q_dev (a state buffer on the device) holds the result afterwards as well."""
        L = self.layout
        need = L.E * L.n_local[0] * L.n_local[1] * L.n_local[2]
        for name, t in (("q_in", q_in), ("q_out", q_out)):
            if not isinstance(t, torch.Tensor) or t.device.type != "cpu":
                raise ValueError(f"{name} must be a host tensor")
            if t.dtype != torch.float64 or not t.is_contiguous() or t.numel() != need:
                raise ValueError(f"{name} must be a contiguous float64 host tensor of "
                                 f"E*nx*ny*nz = {need} elements (got {t.dtype}, {t.numel()})")
        _check(lib.mfc_advance_host(self._h, ctypes.c_void_p(q_in.data_ptr()),
                                    ctypes.c_void_p(q_out.data_ptr()), self._sp(q_dev),
                                    int(nsteps), float(dt), _stream(stream)), "mfc_advance_host")

    def set_stream_chunks(self, chunks: int):
        """Chunk count of the streamed one-step advance_host (0: off, -1: default)."""
        _check(lib.mfc_set_stream_chunks(self._h, int(chunks)), "mfc_set_stream_chunks")

    KINDS = ("sweep_x", "sweep_y", "sweep_z", "bc_fill", "halo", "eos")

    def profile(self, on: bool = True):
        _check(lib.mfc_profile_enable(self._h, int(on)), "mfc_profile_enable")

    def profile_read(self) -> dict:
        n = len(self.KINDS)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        _check(lib.mfc_profile_read(self._h, ms, cnt, n), "mfc_profile_read")
        return {k: (ms[i], cnt[i]) for i, k in enumerate(self.KINDS)}

    # ------------------------------------------------------------- fused halo (F1)
    def peer_export(self, q) -> bytes:
        """CUDA-IPC handles of q, the RK stage buffers and the flags (mfc_peer_export)."""
        buf = ctypes.create_string_buffer(PEER_BLOB_BYTES)
        _check(lib.mfc_peer_export(self._h, self._sp(q), buf), "mfc_peer_export")
        return buf.raw

    def peer_import(self, face: int, blob: bytes):
        buf = ctypes.create_string_buffer(blob, PEER_BLOB_BYTES)
        _check(lib.mfc_peer_import(self._h, int(face), buf), "mfc_peer_import")

    def attach_fused_halo(self, q, group=None):
        """Collective over the torch.distributed group: register q, exchange the IPC
        blobs (all_gather_object) and attach every neighbour face; ends with a barrier.
        Afterwards the RK3 steps write the neighbours' ghost layers directly."""
        import torch.distributed as dist
        blob = self.peer_export(q)
        torch.cuda.synchronize(self.device)
        blobs = [None] * dist.get_world_size(group)
        dist.all_gather_object(blobs, blob, group=group)
        for face, blob_f in face_blobs(self.neighbors, blobs).items():
            self.peer_import(face, blob_f)
        dist.barrier(group=group)

    def last_launch_count(self) -> int:
        return int(lib.mfc_last_launch_count(self._h))

    def comm_status(self):
        """Raise MfcError if the NCCL communicator saw an asynchronous error
        (ncclCommGetAsyncError); a no-op without NCCL."""
        _check(lib.mfc_comm_status(self._h), "mfc_comm_status")

    def close(self):
        if getattr(self, "_h", None):
            lib.mfc_finalize(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def describe(problem, procs=(1, 1, 1), rank=0, nranks=1):
    """Host-only query of a rank's layout and neighbours (no GPU touched): creates a
    context in loopback mode, reads mfc_get_layout / mfc_get_neighbors, finalizes."""
    g = _Grid()
    g.ndim = problem.ndim
    for k in range(3):
        g.n_global[k] = int(problem.n[k])
        g.lo[k] = float(problem.lo[k])
        g.hi[k] = float(problem.hi[k])
        g.procs[k] = int(procs[k])
    N = problem.n_fluids
    gam = (ctypes.c_double * N)(*problem.gamma[:N])
    pinf = (ctypes.c_double * N)(*problem.pi_inf[:N])
    bc = (ctypes.c_int32 * 6)(*problem.bc)
    comm = _Comm()
    comm.rank, comm.nranks, comm.loopback = rank, nranks, 1
    h = ctypes.c_void_p()
    _check(lib.mfc_init(ctypes.byref(h), ctypes.byref(g), N, gam, pinf, bc, ctypes.byref(comm), 0),
           "mfc_init")
    try:
        lay = _Layout()
        _check(lib.mfc_get_layout(h, ctypes.byref(lay)), "mfc_get_layout")
        nb = (ctypes.c_int32 * 6)()
        _check(lib.mfc_get_neighbors(h, nb), "mfc_get_neighbors")
        return (Layout(lay.E, lay.ghost, lay.n_fluids, lay.ndim, tuple(lay.n_local),
                       tuple(lay.lo_global), tuple(lay.dims), tuple(lay.stride), lay.offset,
                       lay.n_elems, lay.workspace_bytes), tuple(nb))
    finally:
        lib.mfc_finalize(h)


def _arr(objs):
    return (ctypes.c_void_p * len(objs))(*[ctypes.c_void_p(o) for o in objs])


def rk3_step_group(solvers, qs, dt, stream=None):
    """Loopback group step: len(solvers) subdomains on one GPU (comm.loopback = 1)."""
    hs = _arr([s._h.value for s in solvers])
    ps = _arr([s._sp(q).value for s, q in zip(solvers, qs)])
    _check(lib.mfc_rk3_step_group(hs, ps, len(solvers), float(dt), _stream(stream)),
           "mfc_rk3_step_group")


def rhs_group(solvers, qs, outs, stream=None):
    hs = _arr([s._h.value for s in solvers])
    ps = _arr([s._sp(q).value for s, q in zip(solvers, qs)])
    os_ = _arr([s._sp(o).value for s, o in zip(solvers, outs)])
    _check(lib.mfc_rhs_group(hs, ps, os_, len(solvers), _stream(stream)), "mfc_rhs_group")


def halo_exchange_group(solvers, qs, stream=None):
    hs = _arr([s._h.value for s in solvers])
    ps = _arr([s._sp(q).value for s, q in zip(solvers, qs)])
    _check(lib.mfc_halo_exchange_group(hs, ps, len(solvers), _stream(stream)),
           "mfc_halo_exchange_group")


def face_blobs(neighbors, blobs) -> dict:
    """{face: the blob of the neighbour rank across that face} (faces without a
    neighbour rank, neighbors[f] == -1, are skipped)."""
    return {f: blobs[r] for f, r in enumerate(neighbors) if r >= 0}


def fused_halo_group(solvers, qs):
    """Loopback group: the stage sweeps write the group members' ghost layers directly
    (mfc_fused_halo_group); qs become the registered state buffers."""
    hs = _arr([s._h.value for s in solvers])
    ps = _arr([s._sp(q).value for s, q in zip(solvers, qs)])
    _check(lib.mfc_fused_halo_group(hs, ps, len(solvers)), "mfc_fused_halo_group")
