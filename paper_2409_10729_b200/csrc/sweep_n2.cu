// Sweep / EOS kernels for 2 fluid(s).
#include <algorithm>
#define MFC_NF 2
#include "sweep_inst.cuh"
