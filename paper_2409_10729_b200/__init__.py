"""B200-native (sm_100a) fp64 RHS hot path of MFC's 5-equation multiphase solver
(arXiv 2409.10729).  The compute path lives in the C-ABI library ``libmfc.so``
(``csrc/``, declared in ``include/mfc.h``); ``mfc`` is its thin ctypes binding."""
