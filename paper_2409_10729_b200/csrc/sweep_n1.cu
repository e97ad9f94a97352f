// Sweep / EOS kernels for 1 fluid(s).
#include <algorithm>
#define MFC_NF 1
#include "sweep_inst.cuh"
