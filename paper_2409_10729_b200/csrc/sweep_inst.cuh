// sweep_inst.cuh -- instantiates the sweep and EOS kernels for one fluid count N
// (included by sweep_n{1,2,3}.cu with MFC_NF defined).
#pragma once
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "dispatch.h"

#ifndef MFC_XPAIR_TMA
#define MFC_XPAIR_TMA 0     // persistent TMA x pair (sweep_x_pair_tma); A/B build flag
#endif

namespace mfc {

template <class M>
__global__ void __launch_bounds__(256) eos_kernel(const EosArgs a, bool to_cons) {
    const int64_t n = (int64_t)a.nx * a.ny * a.nz;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % a.nx);
        const int j = (int)((t / a.nx) % a.ny);
        const int k = (int)(t / ((int64_t)a.nx * a.ny));
        const int64_t c = a.base + (int64_t)k * a.sZ + (int64_t)j * a.sY + i;
        double x[M::E], y[M::E];
#pragma unroll
        for (int e = 0; e < M::E; ++e) x[e] = a.in[c + e * a.sE];
        if (to_cons) prim_to_cons<M>(x, y, a.mat);
        else cons_to_prim<M>(x, y, a.mat);
#pragma unroll
        for (int e = 0; e < M::E; ++e) a.out[c + e * a.sE] = y[e];
    }
}

// CFL wave rate: max over interior cells of max_k (|u_k| + c)/dx_k (AMB-25).
// Block max in shared memory, one atomicMax per block on the bit pattern of the
// (non-negative) double, which orders like an unsigned integer.
template <class M>
__global__ void __launch_bounds__(256) wave_rate_kernel(const EosArgs a, double3 inv_dx,
                                                        WaveGrid wg, unsigned long long* out) {
    __shared__ double red[256];
    const int64_t n = (int64_t)a.nx * a.ny * a.nz;
    double m = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % a.nx);
        const int j = (int)((t / a.nx) % a.ny);
        const int k = (int)(t / ((int64_t)a.nx * a.ny));
        const int64_t c = a.base + (int64_t)k * a.sZ + (int64_t)j * a.sY + i;
        double x[M::E], v[M::E];
#pragma unroll
        for (int e = 0; e < M::E; ++e) x[e] = a.in[c + e * a.sE];
        cons_to_prim_fast<M>(x, v, a.mat);
        double rho = v[0], G = v[M::IA] * a.mat.Gam[0], P = v[M::IA] * a.mat.Pi[0];
#pragma unroll
        for (int f = 1; f < M::N; ++f) {
            rho += v[f];
            G = fma(v[M::IA + f], a.mat.Gam[f], G);
            P = fma(v[M::IA + f], a.mat.Pi[f], P);
        }
        const double cs = sqrt(fma(G + 1.0, v[M::IE], P) / (rho * G));
        // 1/dx per axis: uniform, or the cell's own width on a stretched axis (F4)
        const int ijk[3] = {i, j, k};
        const double idx[3] = {inv_dx.x, inv_dx.y, inv_dx.z};
#pragma unroll
        for (int d = 0; d < M::D; ++d) {
            const double id = wg.inv[d] ? __ldg(wg.inv[d] + ijk[d]) : idx[d];
            m = fmax(m, (fabs(v[M::IM + d]) + cs) * id);
        }
    }
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(red[0]));
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-(kernel, device) setting: raise it
// whenever a launch needs more than that kernel has been given on the current device
// (successes are recorded per kernel and device; a failure is returned, never cached)
template <class K>
static int set_smem_attr(K* kernel, size_t smem) {
    if (smem <= 48 * 1024) return 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{(const void*)kernel, dev}];
    if (smem <= have) return 0;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    have = smem;
    return 0;
}

// Admissibility guard (F3): count interior cells whose conserved state is not finite, or
// whose mixture density or squared sound speed c^2 = ((Gamma+1)p + Pi)/(rho Gamma) is not
// positive (the oracle's orc_count_inadmissible, AMB-14: detection, no limiter).
// The primitives come from the bitwise-specified cons_to_prim.
template <class M>
__global__ void __launch_bounds__(256) admissible_kernel(const EosArgs a,
                                                         unsigned long long* out) {
    __shared__ unsigned long long red[256];
    const int64_t n = (int64_t)a.nx * a.ny * a.nz;
    unsigned long long bad = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % a.nx);
        const int j = (int)((t / a.nx) % a.ny);
        const int k = (int)(t / ((int64_t)a.nx * a.ny));
        const int64_t c = a.base + (int64_t)k * a.sZ + (int64_t)j * a.sY + i;
        double x[M::E], v[M::E];
        bool finite = true;
#pragma unroll
        for (int e = 0; e < M::E; ++e) {
            x[e] = a.in[c + e * a.sE];
            finite = finite && isfinite(x[e]);
        }
        if (!finite) {
            ++bad;
            continue;
        }
        cons_to_prim<M>(x, v, a.mat);
        double rho = v[0], G = __dmul_rn(v[M::IA], a.mat.Gam[0]), P = __dmul_rn(v[M::IA], a.mat.Pi[0]);
#pragma unroll
        for (int f = 1; f < M::N; ++f) {
            rho = __dadd_rn(rho, v[f]);
            G = __dadd_rn(G, __dmul_rn(v[M::IA + f], a.mat.Gam[f]));
            P = __dadd_rn(P, __dmul_rn(v[M::IA + f], a.mat.Pi[f]));
        }
        const double c2 = __ddiv_rn(__dadd_rn(__dmul_rn(__dadd_rn(G, 1.0), v[M::IE]), P),
                                    __dmul_rn(rho, G));
        if (!(rho > 0.0) || !(c2 > 0.0) || !isfinite(c2)) ++bad;
    }
    red[threadIdx.x] = bad;
    __syncthreads();
    for (int s2 = 128; s2 > 0; s2 >>= 1) {
        if (threadIdx.x < s2) red[threadIdx.x] += red[threadIdx.x + s2];
        __syncthreads();
    }
    if (threadIdx.x == 0 && red[0]) atomicAdd(out, red[0]);
}

template <class M, int DIR, int MODE, int ORD, bool PEER = false>
static cudaError_t launch_ring(const SweepArgs& a, dim3 g, dim3 b, cudaStream_t s) {
    constexpr int NTH = sweep_nth<M, DIR, MODE>();
    b = dim3(32, NTH / 32);                          // ring kernels: fixed block shape
    const int64_t warp_lines = (int64_t)((a.nA + 31) / 32) * a.nB;
    g = dim3((unsigned)((warp_lines + b.y - 1) / b.y), 1, g.z);
    constexpr bool TMA = march_tma<M, DIR, MODE, ORD>();
    // + the TMA rings' slot barriers (<= 4 per warp)
    const size_t smem = sweep_smem_per_thread<M, DIR, MODE>() * NTH + (TMA ? 32 * (NTH / 32) : 0);
    const int st = set_smem_attr(sweep_kernel<M, DIR, MODE, ORD, PEER>, smem);
    if (st) return (cudaError_t)st;
    MarchMaps mm{};
    if constexpr (TMA) {
        // padded extents and the interior origin from the strides (x unit stride)
        const int64_t X = DIR == 1 ? a.sS : a.sB, XY = DIR == 1 ? a.sB : a.sS;
        const int64_t Y = XY / X, Z = a.sE / XY;
        mm.ox = (int32_t)(a.base % X);
        mm.oy = (int32_t)((a.base / X) % Y);
        mm.oz = (int32_t)(a.base / XY);
        cudaError_t e;
        if ((e = encode_state_map(&mm.q, a.q, X, Y, Z, M::E, 32)) != cudaSuccess ||
            (e = encode_state_map(&mm.acc, a.acc ? a.acc : a.q, X, Y, Z, M::E, 32)) != cudaSuccess ||
            (e = encode_state_map(&mm.qn, a.qn ? a.qn : a.q, X, Y, Z, M::E, 32)) != cudaSuccess)
            return e;
    }
    sweep_kernel<M, DIR, MODE, ORD, PEER><<<g, b, smem, s>>>(a, mm);
    return cudaGetLastError();
}

template <class M, int DIR, int ORD>
static cudaError_t launch_dir(int mode, const SweepArgs& a, dim3 g, dim3 b, cudaStream_t s) {
    if constexpr (DIR == 0 && M::D >= 2) {
        // row-parallel x sweeps (RHS: M_SET, RK stage: M_RKINIT = the stage base cb*q^s
        // (+ ca*q^n when a.qn is set) + w*c_x)
        if (mode != M_SET && mode != M_RKINIT) return cudaErrorInvalidValue;
        if constexpr (ORD == 5) {
            // two cells per thread (sweep_x_pair): W <= 4 warps, 64 W cells per block
            // (128-cell segments: C3 x 2.15 -> 2.28 ms per step, r93)
            const int W = (int)std::min<int64_t>(4, (a.nS + 63) / 64);
            const int nseg = (a.nS + 64 * W - 1) / (64 * W);
            if constexpr (MFC_XPAIR_TMA != 0) {
                // persistent blocks, the next segment's tile loaded by TMA (sweep_x_pair_tma)
                const int64_t X = a.sA, Y = a.sB / a.sA, Z = a.sE / a.sB;
                const int ox = (int)(a.base % X), oy = (int)((a.base / X) % Y),
                          oz = (int)(a.base / (X * Y));
                const int total = nseg * a.nA * a.nB;
                const size_t smem = x_pair_tma_smem_bytes<M>(64 * W);
                int st;
                if ((st = set_smem_attr(sweep_x_pair_tma<M, false>, smem)) ||
                    (st = set_smem_attr(sweep_x_pair_tma<M, true>, smem)))
                    return (cudaError_t)st;
                cudaFuncSetAttribute(sweep_x_pair_tma<M, false>,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 100);
                cudaFuncSetAttribute(sweep_x_pair_tma<M, true>,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 100);
                CUtensorMap tm;
                cudaError_t e = encode_state_map(&tm, a.q, X, Y, Z, M::E, 64 * W);
                if (e != cudaSuccess) return e;
                int dev = 0, nsm = 0, occ = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
                if (mode == M_SET)
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_x_pair_tma<M, false>, 32 * W, smem);
                else
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_x_pair_tma<M, true>, 32 * W, smem);
                // MFC_XPAIR_TMA == 2: one segment per block (not persistent), the tile kept
                // in shared memory for the epilogue's RK base
                const int grid = MFC_XPAIR_TMA == 2 ? total
                                                    : (int)std::min<int64_t>(total, (int64_t)nsm * std::max(occ, 1));
                if (mode == M_SET)
                    sweep_x_pair_tma<M, false><<<grid, 32 * W, smem, s>>>(tm, a, W, nseg, total, ox, oy, oz);
                else
                    sweep_x_pair_tma<M, true><<<grid, 32 * W, smem, s>>>(tm, a, W, nseg, total, ox, oy, oz);
                return cudaGetLastError();
            }
            const size_t smem = sizeof(double) * x_pair_smem_doubles<M>(64 * W);
            int st;
            if ((st = set_smem_attr(sweep_x_pair<M, false>, smem)) ||
                (st = set_smem_attr(sweep_x_pair<M, true>, smem)))
                return (cudaError_t)st;
            const dim3 gr(nseg, a.nA, a.nB);
            if (mode == M_SET) sweep_x_pair<M, false><<<gr, 32 * W, smem, s>>>(a, W);
            else sweep_x_pair<M, true><<<gr, 32 * W, smem, s>>>(a, W);
        } else {
            // one cell per thread (sweep_x_tile): WENO3, WENO5-M; rows longer than 256
            // cells run as several 8-warp segments with boundary cells
            const int W = (int)std::min<int64_t>(8, (a.nS + 31) / 32);
            const int nseg = (a.nS + 32 * W - 1) / (32 * W);
            const size_t smem = sizeof(double) * x_tile_smem_doubles<M>(32 * W);
            int st;
            if ((st = set_smem_attr(sweep_x_tile<M, ORD, false>, smem)) ||
                (st = set_smem_attr(sweep_x_tile<M, ORD, true>, smem)))
                return (cudaError_t)st;
            const dim3 gr(nseg, a.nA, a.nB);
            if (mode == M_SET) sweep_x_tile<M, ORD, false><<<gr, 32 * W, smem, s>>>(a, W);
            else sweep_x_tile<M, ORD, true><<<gr, 32 * W, smem, s>>>(a, W);
        }
    } else if constexpr (DIR == 0) {
        // 1D: the march is the only sweep (RHS: M_SET, RK stage: M_RKINIT)
        if (mode == M_SET) {
            if (a.po.nf) return cudaErrorInvalidValue;
            return launch_ring<M, DIR, M_SET, ORD>(a, g, b, s);
        }
        if (mode != M_RKINIT) return cudaErrorInvalidValue;
        if (a.po.nf) return launch_ring<M, DIR, M_RKINIT, ORD, true>(a, g, b, s);
        return launch_ring<M, DIR, M_RKINIT, ORD>(a, g, b, s);
    } else {
        // y / z marches; only the last sweep of a stage writes a stage result and may
        // carry the fused halo stores (PEER)
        constexpr bool last = DIR == M::D - 1;
        if (mode == M_ACC) {
            if (a.po.nf) {
                if constexpr (last) return launch_ring<M, DIR, M_ACC, ORD, true>(a, g, b, s);
                return cudaErrorInvalidValue;
            }
            return launch_ring<M, DIR, M_ACC, ORD>(a, g, b, s);
        }
        if (mode == M_ACCN) {
            if constexpr (last) {
                if (a.po.nf) return launch_ring<M, DIR, M_ACCN, ORD, true>(a, g, b, s);
                return launch_ring<M, DIR, M_ACCN, ORD>(a, g, b, s);
            }
        }
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int NF, int ND, int ORD>
static cudaError_t launch_model(int DIR, int mode, const SweepArgs& a, dim3 g, dim3 b,
                                cudaStream_t s) {
    using M = Model<NF, ND>;
    switch (DIR) {
        case 0: return launch_dir<M, 0, ORD>(mode, a, g, b, s);
        case 1: if constexpr (ND > 1) return launch_dir<M, 1, ORD>(mode, a, g, b, s); break;
        case 2: if constexpr (ND > 2) return launch_dir<M, 2, ORD>(mode, a, g, b, s); break;
    }
    return cudaErrorInvalidValue;
}

template <int ORD>
static cudaError_t launch_order(int D, int DIR, int mode, const SweepArgs& a, dim3 g, dim3 b,
                                cudaStream_t s) {
    switch (D) {
        case 1: return launch_model<MFC_NF, 1, ORD>(DIR, mode, a, g, b, s);
        case 2: return launch_model<MFC_NF, 2, ORD>(DIR, mode, a, g, b, s);
        case 3: return launch_model<MFC_NF, 3, ORD>(DIR, mode, a, g, b, s);
    }
    return cudaErrorInvalidValue;
}

template <>
cudaError_t launch_sweep<MFC_NF>(int D, int DIR, int mode, int order, const SweepArgs& a, dim3 g,
                                 dim3 b, cudaStream_t s) {
    if (order == 3) return launch_order<3>(D, DIR, mode, a, g, b, s);
    if (order == 7) return launch_order<7>(D, DIR, mode, a, g, b, s);   // WENO5, stretched
    if (order == 6) return launch_order<6>(D, DIR, mode, a, g, b, s);   // WENO5-M
    return launch_order<5>(D, DIR, mode, a, g, b, s);
}

template <>
cudaError_t launch_wave_rate<MFC_NF>(int D, const EosArgs& a, double3 inv_dx, const WaveGrid& wg,
                                     double* out, cudaStream_t s) {
    const int64_t n = (int64_t)a.nx * a.ny * a.nz;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    auto* o = reinterpret_cast<unsigned long long*>(out);
    switch (D) {
        case 1: wave_rate_kernel<Model<MFC_NF, 1>><<<blocks, 256, 0, s>>>(a, inv_dx, wg, o); break;
        case 2: wave_rate_kernel<Model<MFC_NF, 2>><<<blocks, 256, 0, s>>>(a, inv_dx, wg, o); break;
        case 3: wave_rate_kernel<Model<MFC_NF, 3>><<<blocks, 256, 0, s>>>(a, inv_dx, wg, o); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <>
cudaError_t launch_admissible<MFC_NF>(int D, const EosArgs& a, unsigned long long* out,
                                      cudaStream_t s) {
    const int64_t n = (int64_t)a.nx * a.ny * a.nz;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    switch (D) {
        case 1: admissible_kernel<Model<MFC_NF, 1>><<<blocks, 256, 0, s>>>(a, out); break;
        case 2: admissible_kernel<Model<MFC_NF, 2>><<<blocks, 256, 0, s>>>(a, out); break;
        case 3: admissible_kernel<Model<MFC_NF, 3>><<<blocks, 256, 0, s>>>(a, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <>
cudaError_t launch_eos<MFC_NF>(int D, bool to_cons, const EosArgs& a, cudaStream_t s) {
    const int64_t n = (int64_t)a.nx * a.ny * a.nz;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    switch (D) {
        case 1: eos_kernel<Model<MFC_NF, 1>><<<blocks, 256, 0, s>>>(a, to_cons); break;
        case 2: eos_kernel<Model<MFC_NF, 2>><<<blocks, 256, 0, s>>>(a, to_cons); break;
        case 3: eos_kernel<Model<MFC_NF, 3>><<<blocks, 256, 0, s>>>(a, to_cons); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace mfc
