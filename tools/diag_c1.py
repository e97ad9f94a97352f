"""Diagnose C1 RHS parity: print the worst cells per equation (GPU vs oracle)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
from paper_2409_10729_b200 import workloads as W
from parity import oracle_inputs, gpu_rhs, rel_err
np.set_printoptions(precision=17, linewidth=200)
pb = W.c1_water_air()
P, v, q = oracle_inputs(pb)
ref = O.rhs(P, q)
got = gpu_rhs(pb, q)
print("rel_err", rel_err(got, ref))
for e in range(pb.E):
    d = np.abs(got[e] - ref[e])[0, 0]
    i = int(np.argmax(d))
    print(e, "max|ref|", np.abs(ref[e]).max(), "worst cell", i, "ref", ref[e, 0, 0, i], "gpu", got[e, 0, 0, i])
    print("   neighbours ref", ref[e, 0, 0, max(0, i-3):i+4])
    print("   neighbours gpu", got[e, 0, 0, max(0, i-3):i+4])
print("prims near interface", v[:, 0, 0, 276:284].T)
