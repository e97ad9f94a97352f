// dispatch.h -- host-side entry points of the templated sweep / EOS kernels,
// one translation unit per fluid count (sweep_n1.cu, sweep_n2.cu, sweep_n3.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

#include "sweep.cuh"

namespace mfc {

// Launch the sweep kernel for N fluids, D dims, direction DIR with epilogue `mode`
// (M_SET / M_RKINIT for DIR == 0, M_ACC / M_ACCN for DIR > 0).
template <int N>
cudaError_t launch_sweep(int D, int DIR, int mode, int order, const SweepArgs& a, dim3 grid,
                         dim3 block, cudaStream_t s);

struct EosArgs {
    const double* in;
    double* out;
    int64_t sE, sZ, sY, base;
    int32_t nx, ny, nz;
    Materials mat;
};

// number of inadmissible interior cells (non-finite, rho <= 0 or c^2 <= 0) added to *out
template <int N>
cudaError_t launch_admissible(int D, const EosArgs& a, unsigned long long* out, cudaStream_t s);

// to_cons = true: primitive -> conserved, false: conserved -> primitive
template <int N>
cudaError_t launch_eos(int D, bool to_cons, const EosArgs& a, cudaStream_t s);

// 1/dx of every interior cell of the stretched axes (nullptr: uniform axis, inv_dx)
struct WaveGrid {
    const double* inv[3];
};

// max over interior cells of max_k (|u_k|+c)/dx_k -> *out (device double, must hold
// 0 or a smaller non-negative value before the launch)
template <int N>
cudaError_t launch_wave_rate(int D, const EosArgs& a, double3 inv_dx, const WaveGrid& wg,
                             double* out, cudaStream_t s);

}  // namespace mfc
