"""Dump the RHS and one RK3 step of a few problems to an .npz (same-box bitwise check of
kernel variants selected by environment, e.g. MFC_X_TILE=1 vs the default):
    python tools/xvariant_dump.py out_a.npz;  MFC_X_TILE=1 python tools/xvariant_dump.py out_b.npz
    python tools/xvariant_dump.py --compare out_a.npz out_b.npz
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cases():
    from paper_2409_10729_b200 import workloads as W
    return {
        "c3_96": W.c3_droplet(96),
        "c2": W.c2_shock_bubble(256, 128),
        "gr3_refl": W.random_problem(3, (70, 21, 22), 2, "gas",
                                     bc=(W.BC_REFLECTIVE, W.BC_EXTRAPOLATION) * 3),
        "gr3_n3": W.random_problem(3, (41, 33, 17), 3, "water"),
        "gr2_n1": W.random_problem(2, (200, 9), 1, "gas"),
        "gr3_256": W.random_problem(3, (256, 8, 6), 2, "water"),
        "gr3_250": W.random_problem(3, (250, 5, 4), 2, "water"),
    }


def dump(path):
    import torch
    from paper_2409_10729_b200 import mfc
    from paper_2409_10729_b200 import workloads as W
    out = {}
    for name, pb in cases().items():
        s = mfc.Solver(pb, device=0)
        q = s.state_from_prims(W.prims_for(pb))
        r = s.rhs(q)
        out[name + "_rhs"] = s.interior(r).cpu().numpy()
        s.rk3_step(q, 1e-7 if name.startswith("c") else 1e-5)
        torch.cuda.synchronize()
        out[name + "_step"] = s.interior(q).cpu().numpy()
    np.savez(path, **out)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    bad = 0
    for k in A.files:
        eq = np.array_equal(A[k], B[k], equal_nan=True)
        d = np.abs(A[k] - B[k]).max()
        print(f"{k:16s} bitwise={eq} maxdiff={d:.3e}")
        bad += not eq
    print("ALL BITWISE" if bad == 0 else f"{bad} DIFFER")
    return bad


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        sys.exit(1 if compare(sys.argv[2], sys.argv[3]) else 0)
    dump(sys.argv[1])
