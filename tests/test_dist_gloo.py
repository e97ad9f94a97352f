"""Multi-process host logic of the multi-GPU path, world_size 2 and 3 over `gloo` on
CPU (no GPU needed):
  * the NCCL unique-id bootstrap (rank 0 generates, every rank receives the same bytes);
  * libmfc's decomposition bookkeeping seen from every rank (extents tile the domain,
    neighbour relations symmetric, periodic wrap);
  * the halo protocol of P:94 driven by those neighbour ranks, emulated with the
    oracle: each rank exchanges its 3 boundary planes with send/recv and computes its
    slab's RHS; the gathered result equals the single-domain oracle RHS bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2409_10729_b200 import mfc
    from paper_2409_10729_b200 import workloads as W
    res = {}
    # 1. unique-id bootstrap
    uid = mfc.broadcast_unique_id()
    allid = [None] * world
    dist.all_gather_object(allid, uid)
    res["uid_equal"] = all(x == allid[0] for x in allid) and len(uid) == 128
    # 2. decomposition from libmfc (host only)
    pb = W.random_problem(3, (14, 10, 6 * world + 3), 2, "water")
    procs = (1, 1, world)
    L, nb = mfc.describe(pb, procs, rank, world)
    info = [None] * world
    dist.all_gather_object(info, (L.lo_global, L.n_local, nb))
    res["info"] = info
    # 3. halo exchange protocol (z faces) with the oracle, using libmfc's neighbours
    P = O.Problem.from_spec(pb)
    q = O.prim_to_cons(P, W.random_prims(pb, seed=3))
    z0, nz = L.lo_global[2], L.n_local[2]
    sub = W.Problem("sub", 2, 3, (pb.n[0], pb.n[1], nz),
                    hi=(pb.hi[0], pb.hi[1], pb.hi[2] * nz / pb.n[2]), gamma=pb.gamma,
                    pi_inf=pb.pi_inf, bc=pb.bc[:4] + (O.BC_EXTERNAL, O.BC_EXTERNAL))
    Ps = O.Problem.from_spec(sub)
    qs = O.pad(Ps, q[:, z0:z0 + nz])
    g = 3
    lo_nb, hi_nb = nb[4], nb[5]
    inner = (slice(None), slice(None), slice(g, g + pb.n[1]), slice(g, g + pb.n[0]))
    send_lo = torch.from_numpy(np.ascontiguousarray(qs[:, g:2 * g][:, :, inner[2], inner[3]]))
    send_hi = torch.from_numpy(np.ascontiguousarray(qs[:, nz:nz + g][:, :, inner[2], inner[3]]))
    recv_lo = torch.empty_like(send_lo)
    recv_hi = torch.empty_like(send_hi)
    # libmfc's NCCL ordering: sends in ascending DESTINATION face (my hi face lands in
    # the neighbour's lo face, so it goes first), receives in ascending own face
    ops = [dist.P2POp(dist.isend, send_hi, hi_nb), dist.P2POp(dist.isend, send_lo, lo_nb),
           dist.P2POp(dist.irecv, recv_lo, lo_nb), dist.P2POp(dist.irecv, recv_hi, hi_nb)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    qs[:, 0:g, inner[2], inner[3]] = recv_lo.numpy()
    qs[:, nz + g:nz + 2 * g, inner[2], inner[3]] = recv_hi.numpy()
    r = O.unpad(Ps, O.rhs_padded(Ps, qs))
    parts = [None] * world
    dist.all_gather_object(parts, (z0, r))
    if rank == 0:
        full = np.empty_like(q)
        for zz, rr in parts:
            full[:, zz:zz + rr.shape[1]] = rr
        res["bitwise"] = bool(np.array_equal(full, O.rhs(P, q)))
        torch.save(res, os.path.join(out_dir, "res.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_protocol(world, tmp_path):
    import oracle
    oracle.build()
    from paper_2409_10729_b200 import build
    build.build()
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = torch.load(os.path.join(tmp_path, "res.pt"), weights_only=False)
    assert res["uid_equal"]
    assert res["bitwise"]
    info = res["info"]
    for r, (lo, n, nb) in enumerate(info):
        assert nb[4] == (r - 1) % world and nb[5] == (r + 1) % world   # periodic z ring
        assert nb[:4] == (-1, -1, -1, -1)
    assert sum(n[2] for _, n, _ in info) == 6 * world + 3
