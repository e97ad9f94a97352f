// Sweep / EOS kernels for 3 fluid(s).
#include <algorithm>
#define MFC_NF 3
#include "sweep_inst.cuh"
