// sweep.cuh -- the fused per-direction sweep kernel (one per direction x, y, z).
//
// One sweep adds direction DIR's part of eq. (1) to every interior
// cell:  c_e = (F_{e,m-1/2} - F_{e,m+1/2})/dx  (+ a_{i,m} (u^f_{m+1/2} - u^f_{m-1/2})/dx
// for the volume-fraction rows, AMB-5/6), with F from WENO5 + HLLC.
//
// Mapping (B200 design): a thread owns one grid line segment of T cells
// along DIR and MARCHES along it.  Consecutive lanes own neighbouring lines along the
// unit-stride x axis for the y/z sweeps (every load/store of a warp is one contiguous
// 256-byte row), along y for the x sweep.  Per step the thread loads the conserved
// state of ONE new cell, converts it to primitives (S2) and shifts it into a 5-cell
// register window; WENO5 of the window's centre cell yields both of that cell's face
// states; the face between the previous and the current cell gets its HLLC flux; the
// previous cell's update is written.  So every face state, face flux and primitive
// is computed exactly once per segment and never leaves the register file -- no face
// states in HBM (MFC wrote them, ~2 GB per sweep at 256^3), no transposes.
//
// Epilogues (compile-time):
//   EPI_ACC:  acc = (READ_ACC ? acc : 0) + c              (x, y sweeps; rhs mode)
//   EPI_RK :  out = ca*qn + cb*(qs + dt*((READ_ACC ? acc : 0) + c))   (last sweep;
//             SSP-RK3 stage of S4 fused into the flux-difference epilogue)
#pragma once
#include "physics.cuh"

namespace mfc {

enum { EPI_ACC = 0, EPI_RK = 1 };

struct SweepArgs {
    const double* __restrict__ q;   // stencil state (padded layout, ghosts filled)
    double* acc;                    // accumulator (state layout)
    double* out;                    // RK destination (state layout)
    const double* qn;               // RK base state q^n (may alias out)
    int64_t sE;                     // equation stride
    int64_t sS, sA, sB;             // strides along the sweep, lane and third axis
    int64_t base;                   // offset of interior cell (0,0,0), equation 0
    int32_t nS, nA, nB;             // interior extents along sweep / lane / third axis
    int32_t T;                      // segment length along the sweep
    double invd;                    // 1/dx along DIR
    double eps;                     // WENO epsilon
    double dt, ca, cb;              // RK stage coefficients
    Materials mat;
};

template <class M, int DIR, bool READ_ACC, int EPI>
__global__ void __launch_bounds__(128)
sweep_kernel(const SweepArgs a) {
    constexpr int E = M::E;
    const int ia = blockIdx.x * blockDim.x + threadIdx.x;
    const int ib = blockIdx.y * blockDim.y + threadIdx.y;
    if (ia >= a.nA || ib >= a.nB) return;
    const int s0 = blockIdx.z * a.T;
    const int s1 = min(s0 + a.T, a.nS);   // cells s0 .. s1-1 are updated
    const int64_t line = a.base + (int64_t)ia * a.sA + (int64_t)ib * a.sB;
    const double* __restrict__ q = a.q;

    auto load_prim = [&](int s, double (&v)[E]) {
        double qc[E];
        const double* p = q + line + (int64_t)s * a.sS;
#pragma unroll
        for (int e = 0; e < E; ++e) qc[e] = __ldg(p + e * a.sE);
        cons_to_prim<M>(qc, v, a.mat);
    };

    double w[5][E];        // primitive window: cells j-2 .. j+2
#pragma unroll
    for (int k = 1; k < 5; ++k) load_prim(s0 - 4 + k, w[k]);   // cells s0-3 .. s0

    double vm_prev[E];     // v-_{j-1/2} (from cell j-1)
    double F_prev[E];      // flux at face j-3/2
    double uf_prev = 0.0;

    for (int j = s0 - 1; j <= s1; ++j) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int e = 0; e < E; ++e) w[k][e] = w[k + 1][e];
        }
        load_prim(j + 2, w[4]);

        double vm[E], vp[E];
#pragma unroll
        for (int e = 0; e < E; ++e)
            weno5(w[0][e], w[1][e], w[2][e], w[3][e], w[4][e], a.eps, vm[e], vp[e]);

        if (j >= s0) {
            double F[E], uf;
            hllc<M, DIR>(vm_prev, vp, a.mat, F, uf);
            if (j > s0) {
                // update cell j-1: faces j-3/2 (F_prev) and j-1/2 (F); alpha_{j-1} = w[1]
                const int64_t c = line + (int64_t)(j - 1) * a.sS;
                const double div = (uf - uf_prev) * a.invd;
                double L[E];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    double r = (F_prev[e] - F[e]) * a.invd;
                    if (e >= M::IA) r = fma(w[1][e], div, r);
                    L[e] = r;
                }
                if (EPI == EPI_ACC) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        double* p = a.acc + c + e * a.sE;
                        *p = READ_ACC ? (*p + L[e]) : L[e];
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int64_t ce = c + e * a.sE;
                        const double Lt = READ_ACC ? (a.acc[ce] + L[e]) : L[e];
                        const double t = fma(a.dt, Lt, q[ce]);
                        a.out[ce] = (a.ca == 0.0) ? t : fma(a.ca, a.qn[ce], a.cb * t);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < E; ++e) F_prev[e] = F[e];
            uf_prev = uf;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) vm_prev[e] = vm[e];
    }
}

}  // namespace mfc
