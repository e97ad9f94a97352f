"""CPU oracle for the MFC 5-equation RHS hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2409_10729_b200``) never imports it and shares no code with it.

Contents
  mfc_oracle.c / .h   plain fp64 C implementation of SURVEY §8(c) S0-S4
  oracle.py           ctypes wrapper (numpy in, numpy out)
  exact_riemann.py    exact Riemann solver for stiffened gases (Toro [14] ch. 4),
                      an independent pin for the full solver
"""
from .oracle import *  # noqa: F401,F403
