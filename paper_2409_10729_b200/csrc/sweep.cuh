// sweep.cuh -- the fused per-direction sweep kernel (one per direction x, y, z).
//
// One sweep adds direction DIR's part of eq. (1) to every interior
// cell:  c_e = (F_{e,m-1/2} - F_{e,m+1/2})/dx  (+ a_{i,m} (u^f_{m+1/2} - u^f_{m-1/2})/dx
// for the volume-fraction rows, AMB-5/6), with F from WENO5 + HLLC.
//
// Mapping: a thread owns one grid line segment of T cells along DIR
// and MARCHES along it.  Consecutive lanes own neighbouring lines along the unit-
// stride x axis for the y/z sweeps (every warp load/store is one contiguous 256-byte
// row), along y for the x sweep.  Per step the thread converts ONE new cell to
// primitives (S2) and shifts it into a 5-cell register window; WENO5 of the window's
// centre cell yields both of that cell's face states; the face between the previous
// and the current cell gets its HLLC flux; the previous cell's update is written.
// Every face state, face flux and primitive is computed once per segment and never
// leaves the register file: no face states in HBM, no transposes.
//
// Latency hiding: every streamed operand (the next cell's state, the epilogue operands
// of the cell updated in a step) is copied into a per-thread shared-memory ring with
// cp.async two march steps before it is used, so no registers are held for it and a
// warp never waits on DRAM inside a step.
//
// Epilogues (compile-time MODE; w = cb*dt in RK stages, 1 for a plain RHS):
//   M_SET   : dst = c                                 (1D x sweep of a RHS: write-only)
//   M_RKINIT: dst = ca*q^n + cb*q^s + w*c             (1D: the only sweep, RK stage; the
//                                                      row-parallel x sweeps of 2D/3D)
//   M_ACC   : dst = acc + w*c                         (y sweep, z sweep)
//   M_ACCN  : dst = acc + w*c + ca*q^n                (last sweep of an RK stage when the
//                                                      x sweep wrote cb*q^s + w*c_x only)
// so the SSP-RK3 stage q^(s+1) = ca q^n + cb (q^s + dt (c_x + c_y + c_z)) (S4) is
// assembled across the sweeps.
#pragma once
#include "physics.cuh"
#include "tma.cuh"

#ifndef MFC_MARCH_FEWOP
#define MFC_MARCH_FEWOP false   // weno5_fewop in the ring marches (spills at 168 registers)
#endif
#ifndef MFC_MARCH_SC
#define MFC_MARCH_SC false      // the curvature-term carry for E > 8 too (spills there)
#endif
#ifndef MFC_DW_ALL
#define MFC_DW_ALL false        // experiment: the difference window in every WENO5 march
#endif
#ifndef MFC_FEWOP_EMAX
#define MFC_FEWOP_EMAX 8
#endif
#ifndef MFC_ACC_MINB
#define MFC_ACC_MINB 3   // resident 128-thread blocks per SM for the non-RK sweep modes
#endif

namespace mfc {

enum { M_SET = 0, M_RKINIT = 1, M_ACC = 2, M_ACCN = 4 };

// Reconstruction of one variable of the window's centre cell (ORD = 5: cells w0..w4,
// ORD = 6: the same with WENO5-M weights, ORD = 3: the inner three).
// FEWOP: the WENO5 form with fewer FP64 operations but longer-lived temporaries
// (x tile only, see weno5_fewop).
template <int ORD, bool FEWOP = false>
__device__ __forceinline__ void reconstruct(double w0, double w1, double w2, double w3, double w4,
                                            double eps4, double eps, double& vm, double& vp) {
    if constexpr (ORD == 6) weno5m(w0, w1, w2, w3, w4, eps4, vm, vp);   // WENO5-M
    else if constexpr (ORD == 5 && FEWOP) weno5_fewop(w0, w1, w2, w3, w4, eps4, vm, vp);
    else if constexpr (ORD == 5) weno5(w0, w1, w2, w3, w4, eps4, vm, vp);
    else weno3(w1, w2, w3, eps, vm, vp);
}

constexpr int BC_GHOST = 1;  // ghost cells of this face are valid in memory (halo exchange)

// Ghost cells of a physical boundary are never stored: a sweep reading cell s of its
// line outside [0, n) reads the interior cell the boundary condition maps it to
// (S1 of DESIGN.md §3: periodic -1-j <- n-1-j, extrapolation <- adjacent interior,
// reflective -1-j <- j with the normal momentum negated).  Each map is linear,
// s' = A + B*s, so it is applied branch-free:
//   periodic lo (A, B) = (n, 1),   hi (-n, 1)
//   extrapolation lo (0, 0),        hi (n-1, 0)
//   reflective lo (-1, -1),         hi (2n-1, -1)   (+ normal momentum flip)
//   ghost (halo-exchanged) (0, 1): read the ghost layer itself
struct GhostMap {
    int32_t alo, blo, ahi, bhi;
    int32_t flip_lo, flip_hi;
};

__device__ __forceinline__ int map_cell(int s, int n, const GhostMap& g) {
    const int lo = g.alo + g.blo * s, hi = g.ahi + g.bhi * s;
    return s < 0 ? lo : (s >= n ? hi : s);
}
__device__ __forceinline__ bool map_flip(int s, int n, const GhostMap& g) {
    return (s < 0 && g.flip_lo) || (s >= n && g.flip_hi);
}

// Fused halo: the sweep that writes an RK stage result also stores
// every result cell lying within 3 cells of a face shared with another rank straight
// into that neighbour's ghost layer (peer memory: the same device for loopback groups,
// a CUDA-IPC mapping of the neighbour's buffer otherwise), so no pack / exchange /
// unpack pass follows the stage.  My cell (x, y, z) with lo <= coord[dim] < hi goes to
// the neighbour's element off + e*sE + x + y*sy + z*sz (off folds the neighbour's
// interior offset and the index shift across the face: +n_nbr on my low face, -n on
// my high face; tangential coordinates are shared by construction of the block
// decomposition).
struct PeerFace {
    double* dst;                    // neighbour's buffer (element 0)
    int64_t off, sE, sy, sz;        // neighbour's layout, shift folded into off
    int32_t dim, lo, hi, pad;       // face dimension; my coordinates [lo, hi) are sent
};
struct PeerOut {
    int32_t nf;                     // faces with a neighbour (0: plain sweep)
    PeerFace f[6];
};

// Copy my just-written result cell (src, equation stride sE) to every neighbour whose
// face it lies next to.  Called for the few boundary cells only (the values are read
// back from the store just made -- L2 hits -- instead of being kept live in registers
// through the march).
template <int E>
__device__ __forceinline__ void peer_copy(const PeerOut& po, int x, int y, int z, const double* src,
                                       int64_t sE) {
    for (int i = 0; i < po.nf; ++i) {
        const PeerFace& p = po.f[i];
        const int ck = p.dim == 0 ? x : (p.dim == 1 ? y : z);
        if (ck < p.lo || ck >= p.hi) continue;
        double* d = p.dst + p.off + x + (int64_t)y * p.sy + (int64_t)z * p.sz;
#pragma unroll
        for (int e = 0; e < E; ++e) d[e * p.sE] = src[e * sE];
    }
}

// Non-uniform grid (F4, DESIGN.md AMB-27): per-cell coefficients of the sweep axis,
// structure of arrays over cells -3 .. n+2 (element (c, m) at nu[c * nu_ld + m + 3]):
//   NU_B + 2k, +1 : b_k = Δ q_k'(x_m) on the two first differences of candidate k's stencil
//   NU_C + 2k, +1 : sqrt(13/3) c_k, c_k = Δ² q_k''/2  (beta_k = b_k² + (13/3) c_k²)
//   NU_PM + 2k, +1: q_k(x_{m+1/2}) - v_m,   NU_PP + 2k, +1: q_k(x_{m-1/2}) - v_m
//   NU_DM + k, NU_DP + k: ideal weights of v- and v+;   NU_INV: 1/Δ_m
// (candidate k's differences: k = 0: (D0, D1), 1: (D1, D2), 2: (D2, D3), D_i = v_{m-1+i} -
//  v_{m-2+i})
enum { NU_B = 0, NU_C = 6, NU_PM = 12, NU_PP = 18, NU_DM = 24, NU_DP = 27, NU_INV = 30,
       NU_NCOEF = 31, NU_CM = 32 };
// The same table cell-major (nuc[(m + 3) * NU_CM + c], 256 bytes per cell): the marches
// read one cell's coefficients per step, the same for the whole warp, from two cache lines
// instead of 31 rows.

struct SweepArgs {
    const double* __restrict__ q;   // stencil state (padded layout, ghosts filled)
    const double* acc;              // accumulator input (M_ACC, M_ACCN)
    double* dst;                    // destination (state layout)
    const double* qn;               // RK base state q^n (M_RKINIT/M_ACCN, read iff ca != 0)
    int64_t sE;                     // equation stride
    int64_t sS, sA, sB;             // strides along the sweep, lane and third axis
    int64_t base;                   // offset of interior cell (0,0,0), equation 0
    int32_t nS, nA, nB;             // interior extents along sweep / lane / third axis
    int32_t T;                      // segment length along the sweep
    int32_t s_lo, s_hi;             // cells [s_lo, s_hi) of the sweep axis are updated
                                    // (segments start at s_lo; [0, nS) for a whole sweep)
    GhostMap gm;                    // boundary maps of the sweep axis (see map_cell)
    double invd;                    // 1/dx along DIR
    double eps4;                    // 4 x WENO epsilon (weno5 works with beta' = 4 beta)
    double eps;                     // WENO epsilon (weno3)
    double w, ca, cb;               // epilogue weights
    Materials mat;
    PeerOut po;                     // fused halo stores (last sweep of a stage only)
    const double* nu;               // non-uniform coefficients of the sweep axis (ORD 7)
    const double* nuc;              // the same, cell-major (marches)
    int64_t nu_ld;                  // their cell stride (n + 6)
};

// The 3D y and z marches (M_ACC, M_ACCN; E <= 8) run the fewer-op WENO (weno5_fewop) at
// 2 blocks/SM, where they have the registers for it, with 128-cell segments and ring
// prefetch distance 2 for all operands (mfc.cu launch_sweep_dir keeps the same test):
// C3 y 2.177 -> 2.096, z 2.246 -> 2.189 ms per step (r62-r64, same box).  E = 10 (C5,
// already 2 blocks/SM): the y march gains (20.8 -> 19.9 ms per step), the z march
// loses (22.1 -> 23.2), r68.  The 2D y march (C2) likewise: 0.1053 -> 0.0978 ms per
// step with both (r76).  The lean
// weno5 at 3 blocks/SM (168 registers) is what the other marches run; weno5_fewop
// spills there (+47%).
template <class M, int DIR, int MODE>
__host__ __device__ constexpr bool march_fewop() {
    return MFC_MARCH_FEWOP ||
           (DIR >= 1 && M::D >= 2 && (MODE == M_ACC || MODE == M_ACCN) &&
            (M::E <= MFC_FEWOP_EMAX || DIR == 1));
}

// Per-thread shared-memory rings for the streamed operands (filled by cp.async PD
// march steps ahead of use; element (slot, e) of thread t at [(slot*E + e)*nthreads + t],
// so a warp's copies and reads are contiguous 256-byte rows):
//   state ring : cells j+2 .. j+4 (1D RK march: j-1 .. j+4, the stage operand q^s(j-1)
//                is the state already streamed three steps earlier);
//   acc / q^n rings : cells j-1 .. j+1.
#ifndef MFC_RING_PD
#define MFC_RING_PD 2    // prefetch distance of the rings, in march steps
#endif
template <int MODE, int PD_>
struct Rings {
    static constexpr int PD = PD_;
    static constexpr bool RK = MODE == M_RKINIT;
    // state cell c lives from its fetch (step c-2-PD) to its conversion (step c-2), or
    // to its use as the stage operand q^s (step c+1); operands of cell c from step
    // c+1-PD to step c+1
    static constexpr int QS = RK ? PD + 4 : PD + 1;
    static constexpr int AS = (MODE == M_ACC || MODE == M_ACCN) ? PD + 1 : 0;
    static constexpr int NS = (RK || MODE == M_ACCN) ? PD + 1 : 0;
    static constexpr int OS = PD + 1;   // operand ring length (AS or NS when present)
    static constexpr int SLOTS = QS + AS + NS;
};

// M_ACCN streams three operands: prefetch distance 1 keeps it at 48 KB per block at
// 3 blocks/SM
template <class M, int DIR, int MODE>
__host__ __device__ constexpr int ring_pd() {
    return (MODE == M_ACCN && !march_fewop<M, DIR, MODE>()) ? 1 : MFC_RING_PD;
}
template <class M, int DIR, int MODE>
using RingsOf = Rings<MODE, ring_pd<M, DIR, MODE>()>;

template <class M, int DIR, int MODE>
constexpr size_t sweep_smem_per_thread() { return (size_t)RingsOf<M, DIR, MODE>::SLOTS * M::E * sizeof(double); }

// Threads per block of the ring sweeps (a compile-time constant so that ring offsets
// fold into instruction immediates): 128, or 64 where 12 ring slots of E > 9 doubles
// would not leave room for two blocks per SM.
#ifndef MFC_FEWOP_NTH
#define MFC_FEWOP_NTH 128   // threads per block of the fewer-op y/z marches
#endif
#ifndef MFC_FEWOP_MINB
#define MFC_FEWOP_MINB 2    // and their resident blocks per SM (2 x 128 at <= 255 registers)
#endif
template <class M, int DIR, int MODE>
__host__ __device__ constexpr int sweep_nth() {
    return march_fewop<M, DIR, MODE>() ? MFC_FEWOP_NTH
                                       : ((MODE == M_RKINIT && M::E > 9) ? 64 : 128);
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }

template <class M, int DIR, int MODE, int ORD = 5>
__host__ __device__ constexpr int sweep_min_blocks() {
    if (march_fewop<M, DIR, MODE>() && ORD != 7) return MFC_FEWOP_MINB;
    if (march_fewop<M, DIR, MODE>() || ORD == 7) return 2;   // (ORD 7: 30 coefficients)
    return ((MODE == M_ACC || MODE == M_SET || MODE == M_ACCN) && M::E <= 8) ? MFC_ACC_MINB : 2;
}

// TMA rings (MFC_MARCH_TMA): the 3D y/z accumulate marches fill their per-warp rings
// with cp.async.bulk.tensor boxes of 32 lanes x E equations (one box per operand and
// step, issued by lane 0 of the warp, completion on one mbarrier per ring slot) instead
// of E per-thread cp.async of 8 bytes per operand and step.
#ifndef MFC_MARCH_TMA
#define MFC_MARCH_TMA 0
#endif

template <class M, int DIR, int MODE, int ORD>
__host__ __device__ constexpr bool march_tma() {
    return MFC_MARCH_TMA && M::D == 3 && DIR >= 1 && (MODE == M_ACC || MODE == M_ACCN) && ORD != 7;
}
// tensor maps of the marches' streamed operands (state, accumulator, q^n) and the
// padded coordinates of interior cell (0, 0, 0)
struct MarchMaps {
    CUtensorMap q, acc, qn;
    int32_t ox, oy, oz;
};

template <class M, int DIR, int MODE, int ORD, bool PEER = false>
__global__ void __launch_bounds__(sweep_nth<M, DIR, MODE>(), sweep_min_blocks<M, DIR, MODE, ORD>())
sweep_kernel(const SweepArgs a, const __grid_constant__ MarchMaps mm) {
    constexpr int E = M::E;
    using R = RingsOf<M, DIR, MODE>;
    constexpr bool TMA = march_tma<M, DIR, MODE, ORD>();
    extern __shared__ __align__(128) double smem[];
    constexpr int nth = sweep_nth<M, DIR, MODE>();            // == blockDim.x * blockDim.y
    const int tid = threadIdx.y * 32 + threadIdx.x;      // blockDim.x == 32
    // cp.async rings: element (slot, e) of thread t at [(slot*E + e)*nth + t];
    // TMA rings: per warp w, [slot][E][32] (a box lands contiguously), element at
    // [w*SLOTS*E*32 + (slot*E + e)*32 + lane] for the slot of the respective ring
    constexpr int RS = TMA ? 32 : nth;                      // row stride of a ring
    double* const wbase = TMA ? smem + (size_t)threadIdx.y * R::SLOTS * E * 32 : smem;
    double* const ringQ = wbase + (TMA ? threadIdx.x : tid);   // QS slots
    double* const ringA = ringQ + R::QS * E * RS;           // AS slots
    double* const ringN = ringA + R::AS * E * RS;           // NS slots
    auto at = [&](double* ring, int slot, int e) -> double& { return ring[(slot * E + e) * RS]; };

    // warp-lines (32 consecutive lines along the lane axis A) are numbered A-chunk
    // fastest, and a block's warps take consecutive warp-lines: 2D / 1D grids (nB == 1)
    // fill all warps of a block too
    const int nAw = (a.nA + 31) >> 5;
    const int wl = blockIdx.x * (nth >> 5) + threadIdx.y;
    const int ia = (wl % nAw) * 32 + threadIdx.x;
    const int ib = wl / nAw;
    if (ia >= a.nA || ib >= a.nB) return;                   // no block-level sync below
    // TMA: ring slot barriers of this warp (after the ring rows in the dynamic smem)
    uint64_t* const wbar = reinterpret_cast<uint64_t*>(smem + (size_t)(nth / 32) * R::SLOTS * E * 32) +
                           threadIdx.y * 4;
    if constexpr (TMA) {
        if (threadIdx.x == 0) {
            for (int k = 0; k <= R::PD; ++k) mbar_init(wbar + k, 1);
            mbar_fence_init();
        }
        __syncwarp(__activemask());
    }
    const int ia0 = ia - threadIdx.x;                       // the warp's first lane
    uint32_t tma_par = 0;                                   // phase parity per slot (bit k)
    const int s0 = a.s_lo + blockIdx.z * a.T;
    const int s1 = min(s0 + a.T, a.s_hi);   // cells s0 .. s1-1 are updated
    const int64_t line = a.base + (int64_t)ia * a.sA + (int64_t)ib * a.sB;
    const double* __restrict__ q = a.q;
    // fused halo: does my line touch a shared face (tangential faces: the whole line;
    // faces normal to the sweep: the 3 end cells of the line)?
    bool peer_line = false, peer_ends = false;
    if constexpr (PEER) {
        constexpr int LA = DIR == 0 ? 1 : 0, LB = DIR == 2 ? 1 : 2;
        for (int i = 0; i < a.po.nf; ++i) {
            const PeerFace& p = a.po.f[i];
            if (p.dim == DIR) peer_ends = true;
            else if (p.dim == LA) peer_line |= ia >= p.lo && ia < p.hi;
            else if (p.dim == LB) peer_line |= ib >= p.lo && ib < p.hi;
        }
    }

    auto fetch = [&](double* ring, int slot, const double* src, int cell) {
        const int sc = map_cell(cell, a.nS, a.gm);
        const double* p = src + line + (int64_t)sc * a.sS;
#pragma unroll
        for (int e = 0; e < E; ++e) cp_async8(&at(ring, slot, e), p + e * a.sE);
    };
    // group for step j (issued PD steps earlier): state of cell j+2 -> state slot sq,
    // epilogue operands of cell j-1 -> operand slot sa.  Slots: state cell c at
    // (c+3) % QS, operands at (c+3) % OS.
    // TMA box of cell `cell` along the sweep for this warp's 32 lanes (all E equations)
    auto tma_fetch = [&](const CUtensorMap* map, double* slot_base, uint64_t* bar, int cell) {
        const int sc = map_cell(cell, a.nS, a.gm);
        const int cy = DIR == 1 ? mm.oy + sc : mm.oy + ib;
        const int cz = DIR == 2 ? mm.oz + sc : mm.oz + ib;
        tma_load_4d(slot_base, map, bar, mm.ox + ia0, cy, cz, 0);
    };
    auto issue = [&](int j, int sq, int sa) {
        if constexpr (TMA) {
            // slot sq == sa for these marches (QS == AS == NS == PD + 1); lane 0 of the
            // warp issues after every lane has read the slot's previous contents
            __syncwarp(__activemask());
            if (threadIdx.x == 0) {
                const int c = j - 1;
                const bool st = j <= s1;              // (cells past s1+2 are never read)
                const bool ops = c >= s0 && c < s1;
                const bool qn = R::NS && a.ca != 0.0 && ops;
                const uint32_t bytes = (uint32_t)(E * 32 * sizeof(double)) *
                                       ((st ? 1u : 0u) + (R::AS && ops ? 1u : 0u) + (qn ? 1u : 0u));
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(wbar + sq, bytes);
                double* const wb = wbase;
                if (st) tma_fetch(&mm.q, wb + (size_t)sq * E * 32, wbar + sq, j + 2);
                if (R::AS && ops) tma_fetch(&mm.acc, wb + (size_t)(R::QS + sa) * E * 32, wbar + sq, c);
                if (qn) tma_fetch(&mm.qn, wb + (size_t)(R::QS + R::AS + sa) * E * 32, wbar + sq, c);
            }
        } else {
            if (j + 2 <= s1 + 2) fetch(ringQ, sq, q, j + 2);
            const int c = j - 1;
            if (c >= s0 && c < s1) {
                if (R::AS) fetch(ringA, sa, a.acc, c);
                if (R::NS && a.ca != 0.0) fetch(ringN, sa, a.qn, c);
            }
            cp_async_commit();
        }
    };
    auto inc = [](int k, int n) { return k + 1 == n ? 0 : k + 1; };

    // Primitive window of cells j-2 .. j+2 (a, b, c, d, e).  The DW marches carry it in
    // first differences instead: w[0] = D0 = b-a, w[1] = D1 = c-b, w[2] = c, w[3] = d,
    // w[4] = e (the cell converted this step), so a step forms D2 = d-c, D3 = e-d only
    // (-2 FP64 per variable; bitwise the same differences), and the volume fractions
    // of cell j-1 (the alpha div(u) source) ride along in bA.
    // (the 2D/3D y/z marches, all at 2 blocks/SM: C5 z 22.3 -> 22.0 ms per step with the
    // lean weno5 too, r70; the 1D marches keep 168 registers, where it spills)
    constexpr bool DW = ORD == 5 && (MFC_DW_ALL || (M::D >= 2 && DIR >= 1 &&
                                                    (MODE == M_ACC || MODE == M_ACCN)));
    // SC: the difference marches also carry the curvature terms S = (13/3)s^2 + eps' of
    // the difference pairs (D0,D1) and (D1,D2), formed one and two steps earlier, so a
    // step forms the S of (D2,D3) only (weno5_fewop_s; bitwise the same S values)
    // (E <= 8: C3 y 2.143 -> 2.085, z 2.232 -> 2.217 ms per step, r83; E = 10 spills 8 B)
    constexpr bool SC = DW && (MFC_MARCH_SC || M::E <= 8) && march_fewop<M, DIR, MODE>();
    double w[5][E];
    double bA[M::N];
    double Sc[2][SC ? E : 1];
    {
        double qc[E];
#pragma unroll
        for (int k = 1; k < 5; ++k) {                 // cells s0-3 .. s0 (direct loads)
            const int sc = map_cell(s0 - 4 + k, a.nS, a.gm);
            const double* p = q + line + (int64_t)sc * a.sS;
#pragma unroll
            for (int e = 0; e < E; ++e) qc[e] = __ldg(p + e * a.sE);
            if (map_flip(s0 - 4 + k, a.nS, a.gm)) qc[M::IM + DIR] = -qc[M::IM + DIR];
            if (R::RK) {                              // keep for the q^s epilogue operand
#pragma unroll
                for (int e = 0; e < E; ++e) at(ringQ, (s0 - 4 + k + 3) % R::QS, e) = qc[e];
            }
            cons_to_prim_fast<M>(qc, w[k], a.mat);
        }
        if constexpr (DW) {           // cells s0-3 .. s0 in w[1..4] -> D0, D1, c, d, b_alpha
#pragma unroll
            for (int i = 0; i < M::N; ++i) bA[i] = w[2][M::IA + i];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                w[0][e] = w[2][e] - w[1][e];
                w[1][e] = w[3][e] - w[2][e];
                if constexpr (SC) {       // w[0] carries s0 = D1 - D0 instead of D0
                    const double D2 = w[4][e] - w[3][e];
                    w[0][e] = w[1][e] - w[0][e];
                    Sc[0][e] = weno_S(w[0][e], a.eps4);
                    Sc[1][e] = weno_S(D2 - w[1][e], a.eps4);
                }
                w[2][e] = w[3][e];
                w[3][e] = w[4][e];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < R::PD; ++i) issue(s0 - 1 + i, (s0 + 4 + i) % R::QS, (s0 + 1 + i) % R::OS);
    // rotating slots at step j: conversion (cell j+2), fetch (cell j+2+PD), q^s (cell
    // j-1), operands of cell j-1, operand fetch (cell j-1+PD)
    int kq = (s0 + 4) % R::QS;
    int kqf = (s0 + 4 + R::PD) % R::QS;
    int kqs = (s0 + 1) % R::QS;
    int ka = (s0 + 1) % R::OS;
    int kaf = (s0 + 1 + R::PD) % R::OS;

    double vm_prev[E];     // v-_{j-1/2} (from cell j-1)
    double F_prev[E];      // flux at face j-3/2
    double uf_prev = 0.0;

    for (int j = s0 - 1; j <= s1; ++j) {
        if constexpr (TMA) {                          // the boxes of step j have landed
            mbar_wait(wbar + kq % (R::PD + 1), (tma_par >> (kq % (R::PD + 1))) & 1u);
            tma_par ^= 1u << (kq % (R::PD + 1));
        } else if constexpr (R::PD == 2) {
            cp_async_wait_1();                        // group of step j has landed
        } else {
            cp_async_wait_all();
        }
        issue(j + R::PD, kqf, kaf);
        if constexpr (!DW) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
#pragma unroll
                for (int e = 0; e < E; ++e) w[k][e] = w[k + 1][e];
            }
        }
        {
            double qc[E];
#pragma unroll
            for (int e = 0; e < E; ++e) qc[e] = at(ringQ, kq, e);
            if (map_flip(j + 2, a.nS, a.gm)) qc[M::IM + DIR] = -qc[M::IM + DIR];
            cons_to_prim_fast<M>(qc, w[4], a.mat);
        }

        double vm[E], vp[E];
        double bAn[M::N];      // (DW) volume fractions of cell j, the next step's b_alpha
        // stretched axis: cell j's coefficients, one warp-uniform 256-byte row of the
        // cell-major table read as 16-byte loads (E <= 8; E = 10 has not the registers to
        // hold the row and reads each coefficient where it is used)
        constexpr bool KV = ORD == 7 && M::E <= 8;
        double Kc[KV ? NU_CM : 1];
        if constexpr (KV) {
            const double2* k2 = reinterpret_cast<const double2*>(a.nuc + (int64_t)(j + 3) * NU_CM);
#pragma unroll
            for (int i = 0; i < NU_CM / 2; ++i) {
                const double2 kv = __ldg(k2 + i);
                Kc[2 * i] = kv.x;
                Kc[2 * i + 1] = kv.y;
            }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if constexpr (DW) {
                const double D2 = w[3][e] - w[2][e], D3 = w[4][e] - w[3][e];
                if constexpr (SC) {
                    const double s1 = D2 - w[1][e], s2 = D3 - D2;
                    const double S2 = weno_S(s2, a.eps4);
                    weno5_fewop_s(fma(2.0, w[1][e], w[0][e]), w[1][e], D2, D3, w[2][e], w[0][e],
                                  s1, s2, Sc[0][e], Sc[1][e], S2, vm[e], vp[e]);
                    Sc[0][e] = Sc[1][e];
                    Sc[1][e] = S2;
                    w[0][e] = s1;         // the next step's s0 (its w[1] = D2 below)
                } else if constexpr (march_fewop<M, DIR, MODE>())
                    weno5_fewop_d(w[0][e], w[1][e], D2, D3, w[2][e], a.eps4, vm[e], vp[e]);
                else
                    weno5_d(w[0][e], w[1][e], D2, D3, w[2][e], a.eps4, vm[e], vp[e]);
                if (e >= M::IA) bAn[e - M::IA] = w[2][e];
                if constexpr (!SC) w[0][e] = w[1][e];
                w[1][e] = D2;
                w[2][e] = w[3][e];
                w[3][e] = w[4][e];
            } else if constexpr (ORD == 7) {      // non-uniform grid: cell j's coefficients
                if constexpr (KV)
                    weno5_nu<true>(w[1][e] - w[0][e], w[2][e] - w[1][e], w[3][e] - w[2][e],
                                   w[4][e] - w[3][e], w[2][e], Kc, 1, a.eps, vm[e], vp[e]);
                else
                    weno5_nu(w[1][e] - w[0][e], w[2][e] - w[1][e], w[3][e] - w[2][e],
                             w[4][e] - w[3][e], w[2][e], a.nuc + (int64_t)(j + 3) * NU_CM, 1,
                             a.eps, vm[e], vp[e]);
            } else {
                reconstruct<ORD, march_fewop<M, DIR, MODE>()>(w[0][e], w[1][e], w[2][e], w[3][e],
                                                                w[4][e], a.eps4, a.eps, vm[e], vp[e]);
            }
        }

        if (j >= s0) {
            double F[E], uf;
            hllc<M, DIR>(vm_prev, vp, a.mat, F, uf);
            if (j > s0) {
                // cell j-1: faces j-3/2 (F_prev) and j-1/2 (F); alpha_{j-1} = w[1]
                const int cc = j - 1;
                const int64_t c = line + (int64_t)cc * a.sS;
                const double du = uf - uf_prev;
                // 1/dx of cell j-1: uniform, or its own width on a stretched axis
                const double invd =
                    ORD == 7 ? __ldg(a.nuc + (int64_t)(cc + 3) * NU_CM + NU_INV) : a.invd;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    double r = F_prev[e] - F[e];                 // dx * c_e
                    if (e >= M::IA) r = fma(DW ? bA[e - M::IA] : w[1][e], du, r);
                    double out;
                    if (MODE == M_SET) out = r * invd;
                    else if (MODE == M_ACC) out = fma(a.w * invd, r, at(ringA, ka, e));
                    else if (MODE == M_ACCN)
                        out = fma(a.ca, at(ringN, ka, e), fma(a.w * invd, r, at(ringA, ka, e)));
                    else {
                        const double qs = at(ringQ, kqs, e);
                        const double base = a.ca != 0.0
                                                ? fma(a.ca, at(ringN, ka, e), a.cb * qs)
                                                : a.cb * qs;
                        out = fma(a.w * invd, r, base);
                    }
                    a.dst[c + e * a.sE] = out;
                }
                if constexpr (PEER) {
                    if (peer_line || (peer_ends && (cc < 3 || cc >= a.nS - 3))) {
                        // cell coordinates: sweep axis DIR = cc, lane axis = ia, third = ib
                        constexpr int LA = DIR == 0 ? 1 : 0, LB = DIR == 2 ? 1 : 2;
                        int xyz[3];
                        xyz[DIR] = cc;
                        xyz[LA] = ia;
                        xyz[LB] = ib;
                        peer_copy<E>(a.po, xyz[0], xyz[1], xyz[2], a.dst + c, a.sE);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < E; ++e) F_prev[e] = F[e];
            uf_prev = uf;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) vm_prev[e] = vm[e];
        if constexpr (DW) {
#pragma unroll
            for (int i = 0; i < M::N; ++i) bA[i] = bAn[i];
        }
        kq = inc(kq, R::QS);
        kqf = inc(kqf, R::QS);
        kqs = inc(kqs, R::QS);
        ka = inc(ka, R::OS);
        kaf = inc(kaf, R::OS);
    }
    if constexpr (TMA) {
        // the PD boxes issued for steps past the segment end: wait so that no TMA write
        // is in flight into this block's shared memory when the warp exits
        for (int i = 0; i < R::PD; ++i) {
            mbar_wait(wbar + kq % (R::PD + 1), (tma_par >> (kq % (R::PD + 1))) & 1u);
            tma_par ^= 1u << (kq % (R::PD + 1));
            kq = inc(kq, R::QS);
        }
    } else {
        cp_async_wait_all();
    }
}


}  // namespace mfc

namespace mfc {

// ---------------------------------------------------------------------------
// x sweep, row-parallel tile form (2D/3D, epilogue M_SET or the RK stage base).
//
// A block owns the row segment [x0, x0+32W) of one (y, z) row (W <= 8 warps; one
// block per row up to 256 cells), thread t the cell x0+t: loads and stores are
// contiguous along x, no transpose, no register window, every face computed once.
// Every exchange between cells goes through one shared-memory row per quantity,
// indexed by cell:
//   V  [E][seg+6] : primitives of cells x0-3 .. x0+seg+2 (6 halo cells loaded by
//                   threads 0..5, boundary-mapped like every other cell);
//   VM [E][seg+2] : v-_{m+1/2} of cells x0-1 .. x0+seg;
//   FS [E+1][seg+1]: F and u^f of faces x0-1/2 .. x0+seg-1/2 (aliases V, dead by then).
// WENO reads its four stencil neighbours as four conflict-free row loads per variable
// (no warp borders, no lane-indexed selects: r48's shuffle form spent ~20 extra
// instructions per variable on them); the face x-1/2 takes v-(x-1) from VM, the cell
// update F(x+1/2) from FS.  A whole periodic row wraps by index (face -1/2 = face
// n-1/2); otherwise 2E threads of the last warp reconstruct the two boundary cells
// x0-1 (v-) and x0+seg (v+), one variable each, and one thread the face x0+seg-1/2.
// Nothing but v, v+ and F is live across the three barriers: 80 registers, 3 blocks
// (24 warps) per SM without spills (the shuffle form needed 128 and ran 2 per SM).
// ---------------------------------------------------------------------------
#ifndef MFC_XT_MINB
#define MFC_XT_MINB 3    // resident 256-thread blocks per SM for E <= 8 (80 registers, no
#endif                   // spills)
#ifndef MFC_XT_MINB_BIG
#define MFC_XT_MINB_BIG 3    // E > 8: 3 blocks too (24-48 bytes of spills, still faster: C5 x 29.1 -> 24.1 ms/step, r51)
#endif
template <class M, int ORD = 5>
__host__ __device__ constexpr int x_tile_minb() {
    // the stretched-grid WENO (ORD 7) holds its cell's coefficients: 2 blocks, 128 registers
    return ORD == 7 ? 2 : (M::E <= 8 ? MFC_XT_MINB : MFC_XT_MINB_BIG);
}

// RK stage base of the x sweeps (RKB): cb*q^s, plus ca*q^n when the host hands q^n over
// (MFC_XBASE_N; otherwise the last sweep adds it, M_ACCN)
__device__ __forceinline__ double xbase(const SweepArgs& a, int64_t i) {
    const double b = a.cb * __ldg(a.q + i);
    return (a.qn != nullptr && a.ca != 0.0) ? fma(a.ca, __ldg(a.qn + i), b) : b;
}

template <class M>
__host__ __device__ constexpr size_t x_tile_smem_doubles(int seg) {
    return (size_t)((M::E * (seg + 6) > (M::E + 1) * (seg + 1)) ? M::E * (seg + 6)
                                                                 : (M::E + 1) * (seg + 1)) +
           (size_t)M::E * (seg + 2) + M::E;
}

template <class M, int ORD, bool RKB>
__global__ void __launch_bounds__(256, x_tile_minb<M, ORD>())
sweep_x_tile(const SweepArgs a, int W) {
    constexpr int E = M::E;
    const int t = threadIdx.x;
    const int seg = 32 * W;
    const int x0 = blockIdx.x * seg;
    const int n = a.nS;
    const int x1 = min(x0 + seg, n);                 // cells x0 .. x1-1 are updated
    const bool wrap = (a.gm.blo == 1 && a.gm.alo == n) && x0 == 0 && x1 == n;
    const int x = x0 + t;
    const int64_t row = a.base + (int64_t)blockIdx.y * a.sA + (int64_t)blockIdx.z * a.sB;
    const int LV = seg + 6, LM = seg + 2, LF = seg + 1;
    extern __shared__ double sm[];
    double* const V = sm;                            // [E][LV]; FS [E+1][LF] after phase 2
    double* const FS = sm;
    double* const VM = sm + x_tile_smem_doubles<M>(seg) - (size_t)E * LM - E;   // [E][LM]
    double* const VPX = VM + (size_t)E * LM;         // [E]: v+(x0+seg)

    auto load_prim = [&](int cell, double (&v)[E]) {
        const int sc = map_cell(min(cell, x1 + 2), n, a.gm);   // beyond x1+2: unused
        const double* p = a.q + row + sc;
        double qc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) qc[e] = __ldg(p + e * a.sE);
        if (map_flip(min(cell, x1 + 2), n, a.gm)) qc[M::IM] = -qc[M::IM];
        cons_to_prim_fast<M>(qc, v, a.mat);
    };

    // 1. primitives of my cell (index t+3) and of the six halo cells
    double v[E];
    load_prim(x, v);
#pragma unroll
    for (int e = 0; e < E; ++e) V[e * LV + t + 3] = v[e];
    if (t < 6) {
        double h[E];
        load_prim(t < 3 ? x0 - 3 + t : x0 + seg + t - 3, h);
        const int i = t < 3 ? t : seg + t;
#pragma unroll
        for (int e = 0; e < E; ++e) V[e * LV + i] = h[e];
    }
    __syncthreads();

    // 2. WENO of my cell: stencil cells x-2 .. x+2 at V[e][t+1 .. t+5]
    double vp[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const double* r = V + e * LV + t + 1;
        double vm;
        if constexpr (ORD == 7)            // non-uniform grid: cell x's coefficients
            weno5_nu(r[1] - r[0], v[e] - r[1], r[3] - v[e], r[4] - r[3], v[e],
                     a.nu + (min(x, x1) + 3), a.nu_ld, a.eps, vm, vp[e]);
        else
            reconstruct<ORD, true>(r[0], r[1], v[e], r[3], r[4], a.eps4, a.eps, vm, vp[e]);
        VM[e * LM + t + 1] = vm;
    }
    if (!wrap) {
        const int k = t - (seg - 32);                // lanes 0 .. 2E-1 of the last warp
        if (k >= 0 && k < 2 * E) {
            const bool right = k >= E;
            const int e = right ? k - E : k;
            const double* r = V + e * LV + (right ? seg + 1 : 0);
            double bm, bp;
            if constexpr (ORD == 7)
                weno5_nu(r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[2],
                         a.nu + ((right ? min(x0 + seg, x1) : x0 - 1) + 3), a.nu_ld, a.eps,
                         bm, bp);   // (right and x1 < x0 + seg: unused, index kept in range)
            else
                reconstruct<ORD, true>(r[0], r[1], r[2], r[3], r[4], a.eps4, a.eps, bm, bp);
            if (right) VPX[e] = bp;
            else VM[e * LM] = bm;
        }
    }
    __syncthreads();

    // 3. face x-1/2 from v-(x-1) and my v+  (phase-2 reads of V are complete: FS
    //    overwrites it)
    double F[E], uf;
    {
        const int li = (wrap && t == 0) ? n : t;
        double vL[E];
#pragma unroll
        for (int e = 0; e < E; ++e) vL[e] = VM[e * LM + li];
        hllc<M, 0>(vL, vp, a.mat, F, uf);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) FS[e * LF + t] = F[e];
    FS[E * LF + t] = uf;
    if (!wrap && x1 == x0 + seg && t == 0) {         // face x0+seg-1/2
        double vl[E], vr[E], FB[E], ufB;
#pragma unroll
        for (int e = 0; e < E; ++e) { vl[e] = VM[e * LM + seg]; vr[e] = VPX[e]; }
        hllc<M, 0>(vl, vr, a.mat, FB, ufB);
#pragma unroll
        for (int e = 0; e < E; ++e) FS[e * LF + seg] = FB[e];
        FS[E * LF + seg] = ufB;
    }
    __syncthreads();

    // 4. cell update with F(x+1/2)
    if (x < x1) {
        const int ri = (wrap && t + 1 == n) ? 0 : t + 1;
        const double du = FS[E * LF + ri] - uf;
        const double invd = ORD == 7 ? __ldg(a.nu + NU_INV * a.nu_ld + x + 3) : a.invd;
        const double wi = a.w * invd;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            double r = F[e] - FS[e * LF + ri];
            if (e >= M::IA) r = fma(v[e], du, r);
            if constexpr (RKB)
                a.dst[row + x + e * a.sE] = fma(wi, r, xbase(a, row + x + e * a.sE));
            else
                a.dst[row + x + e * a.sE] = r * invd;
        }
    }
}

// ---------------------------------------------------------------------------
// x sweep, two cells per thread (sweep_x_pair; 2D/3D, WENO5, epilogue M_SET or the RK
// stage base).  Same row-segment structure as sweep_x_tile, but thread t owns the two
// neighbouring cells x0+2t and x0+2t+1: their stencils share four of five first
// differences and three of four curvature terms S = (13/3) s^2 + eps' (weno5_fewop_s),
// the face between them never leaves the registers, and only every other face and v-
// go through shared memory.  Primitives sit in shared memory split by parity of the
// tile index (Ve / Vo), so the stride-2 neighbour reads of a warp stay conflict-free.
//   Ve/Vo [E][seg/2+3]: primitives of tile indices i (cell x0-3+i), i even / odd;
//   VM2   [E][NT+1]   : v- of every thread's second cell (index t+1; index 0: cell x0-1);
//   FS    [E+1][NT+1] : F, u^f of every thread's first face x0+2t-1/2 (aliases Ve/Vo;
//                       index NT: face x0+seg-1/2).
// A whole periodic row of even length wraps by index; otherwise 2E threads of the last
// warp reconstruct the cells x0-1 (v-) and x0+seg (v+) with the same arithmetic
// sequence as the main path, and one thread the face x0+seg-1/2 (AMB-22: bitwise the
// same face whichever segment computes it).
// ---------------------------------------------------------------------------
// resident 128-thread blocks per SM: 5 for E <= 8 (96 registers, 12 B of spills; C3 x
// 2.14 -> 2.05 ms per step against 4, r80), 4 for E = 10 (128 registers, no spills; 5
// spills more and loses: C5 x 21.8 -> 25.1); 3 (168 registers) and 2 are slower.
#ifndef MFC_XP_MINB
#define MFC_XP_MINB 5
#endif
#ifndef MFC_XP_MINB_BIG
#define MFC_XP_MINB_BIG 4
#endif
template <class M>
__host__ __device__ constexpr int x_pair_minb() { return M::E <= 8 ? MFC_XP_MINB : MFC_XP_MINB_BIG; }
template <class M>
__host__ __device__ constexpr size_t x_pair_smem_doubles(int seg) {
    const size_t nt = (size_t)seg / 2;
    const size_t v = (size_t)2 * M::E * (nt + 3);
    const size_t f = (size_t)(M::E + 1) * (nt + 1);
    return (v > f ? v : f) + (size_t)M::E * (nt + 1) + M::E;
}

template <class M, bool RKB>
__global__ void __launch_bounds__(128, x_pair_minb<M>())
sweep_x_pair(const SweepArgs a, int W) {
    constexpr int E = M::E;
    const int t = threadIdx.x;
    const int NT = 32 * W;
    const int seg = 2 * NT;
    const int x0 = blockIdx.x * seg;
    const int n = a.nS;
    const int x1 = min(x0 + seg, n);                 // cells x0 .. x1-1 are updated
    const bool wrap = (a.gm.blo == 1 && a.gm.alo == n) && x0 == 0 && x1 == n && (n & 1) == 0;
    const int tl = n / 2 - 1;                        // (wrap) thread owning the last cell
    const int xa = x0 + 2 * t;                       // my cells xa, xa+1
    const int64_t row = a.base + (int64_t)blockIdx.y * a.sA + (int64_t)blockIdx.z * a.sB;
    const int LH = NT + 3, LP = NT + 1;
    extern __shared__ double sm[];
    double* const Ve = sm;                           // [E][LH]
    double* const Vo = sm + (size_t)E * LH;          // [E][LH]
    double* const FS = sm;                           // [E+1][LP] after phase 2
    double* const VM2 = sm + x_pair_smem_doubles<M>(seg) - (size_t)E * LP - E;   // [E][LP]
    double* const VPX = VM2 + (size_t)E * LP;        // [E]
    auto V = [&](int e, int i) -> double& {
        return (i & 1) ? Vo[e * LH + (i >> 1)] : Ve[e * LH + (i >> 1)];
    };

    auto load_prim = [&](int cell, double (&v)[E]) {
        const int cl = min(cell, x1 + 2);            // beyond x1+2: unused
        const double* p = a.q + row + map_cell(cl, n, a.gm);
        double qc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) qc[e] = __ldg(p + e * a.sE);
        if (map_flip(cl, n, a.gm)) qc[M::IM] = -qc[M::IM];
        cons_to_prim_fast<M>(qc, v, a.mat);
    };

    // 1. primitives of my two cells (tile indices 2t+3, 2t+4) and of the six halo cells
    double v0[E], v1[E];
    load_prim(xa, v0);
    load_prim(xa + 1, v1);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        Vo[e * LH + t + 1] = v0[e];
        Ve[e * LH + t + 2] = v1[e];
    }
    if (t < 6) {
        double h[E];
        load_prim(t < 3 ? x0 - 3 + t : x0 + seg + t - 3, h);
        const int i = t < 3 ? t : seg + t;
#pragma unroll
        for (int e = 0; e < E; ++e) V(e, i) = h[e];
    }
    __syncthreads();

    // 2. WENO of both cells: differences D_i = v_i - v_{i-1}, i = 2t+2 .. 2t+6
    double vm0[E], vp0[E], vp1[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const double a1 = Vo[e * LH + t], a2 = Ve[e * LH + t + 1];
        const double b5 = Vo[e * LH + t + 2], b6 = Ve[e * LH + t + 3];
        const double D2 = a2 - a1, D3 = v0[e] - a2, D4 = v1[e] - v0[e], D5 = b5 - v1[e],
                     D6 = b6 - b5;
        const double s3 = D3 - D2, s4 = D4 - D3, s5 = D5 - D4, s6 = D6 - D5;
        const double S3 = weno_S(s3, a.eps4), S4 = weno_S(s4, a.eps4), S5 = weno_S(s5, a.eps4),
                     S6 = weno_S(s6, a.eps4);
        double vm1;
        weno5_fewop_s(fma(3.0, D3, -D2), D3, D4, D5, v0[e], s3, s4, s5, S3, S4, S5, vm0[e],
                      vp0[e]);
        weno5_fewop_s(fma(3.0, D4, -D3), D4, D5, D6, v1[e], s4, s5, s6, S4, S5, S6, vm1, vp1[e]);
        VM2[e * LP + t + 1] = vm1;
    }
    if (!wrap) {
        const int k = t - (NT - 32);                 // lanes 0 .. 2E-1 of the last warp
        if (k >= 0 && k < 2 * E) {
            const bool right = k >= E;
            const int e = right ? k - E : k;
            const int i0 = right ? seg + 1 : 0;      // stencil tile indices i0 .. i0+4
            double r[5];
#pragma unroll
            for (int j = 0; j < 5; ++j) r[j] = V(e, i0 + j);
            const double D0 = r[1] - r[0], D1 = r[2] - r[1], D2 = r[3] - r[2], D3 = r[4] - r[3];
            const double s0 = D1 - D0, s1 = D2 - D1, s2 = D3 - D2;
            double bm, bp;
            weno5_fewop_s(fma(3.0, D1, -D0), D1, D2, D3, r[2], s0, s1, s2, weno_S(s0, a.eps4),
                          weno_S(s1, a.eps4), weno_S(s2, a.eps4), bm, bp);
            if (right) VPX[e] = bp;
            else VM2[e * LP] = bm;
        }
    }
    __syncthreads();

    // 3. my faces xa-1/2 (v- of the cell before, from VM2) and xa+1/2 (both in registers)
    double FA[E], ufA, FB[E], ufB;
    {
        const int li = (wrap && t == 0) ? tl + 1 : t;
        double vL[E];
#pragma unroll
        for (int e = 0; e < E; ++e) vL[e] = VM2[e * LP + li];
        hllc<M, 0>(vL, vp0, a.mat, FA, ufA);
    }
    hllc<M, 0>(vm0, vp1, a.mat, FB, ufB);
#pragma unroll
    for (int e = 0; e < E; ++e) FS[e * LP + t] = FA[e];
    FS[E * LP + t] = ufA;
    if (!wrap && x1 == x0 + seg && t == 0) {         // face x0+seg-1/2
        double vl[E], vr[E], FE[E], ufE;
#pragma unroll
        for (int e = 0; e < E; ++e) { vl[e] = VM2[e * LP + NT]; vr[e] = VPX[e]; }
        hllc<M, 0>(vl, vr, a.mat, FE, ufE);
#pragma unroll
        for (int e = 0; e < E; ++e) FS[e * LP + NT] = FE[e];
        FS[E * LP + NT] = ufE;
    }
    __syncthreads();

    // 4. updates: cell xa with (FA, FB), cell xa+1 with (FB, the next thread's FA)
    const double wi = a.w * a.invd;
    if (xa < x1) {
        const double du = ufB - ufA;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            double r = FA[e] - FB[e];
            if (e >= M::IA) r = fma(v0[e], du, r);
            if constexpr (RKB)
                a.dst[row + xa + e * a.sE] = fma(wi, r, xbase(a, row + xa + e * a.sE));
            else
                a.dst[row + xa + e * a.sE] = r * a.invd;
        }
    }
    if (xa + 1 < x1) {
        const int ri = (wrap && t == tl) ? 0 : t + 1;
        const double du = FS[E * LP + ri] - ufB;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            double r = FB[e] - FS[e * LP + ri];
            if (e >= M::IA) r = fma(v1[e], du, r);
            if constexpr (RKB)
                a.dst[row + xa + 1 + e * a.sE] = fma(wi, r, xbase(a, row + xa + 1 + e * a.sE));
            else
                a.dst[row + xa + 1 + e * a.sE] = r * a.invd;
        }
    }
}


// ---------------------------------------------------------------------------
// x sweep, two cells per thread, PERSISTENT with TMA tile loads (sweep_x_pair_tma).
//
// The same arithmetic as sweep_x_pair, segment by segment, but a block loops over row
// segments (sid = blockIdx.x, += gridDim.x) and the raw conserved state of a segment
// (E rows of seg cells, one 4D tensor-map box) is loaded by TMA into shared memory while
// the block computes the previous segment: issued by one thread right after the
// block's first barrier of segment k (the raw tile of k is converted by then), it has
// phases 2-4 of segment k to land, and phase 1 of segment k+1 waits on the mbarrier
// instead of on DRAM (sweep_x_pair: long-scoreboard stalls at the first use of the
// loaded state, 16 % of stall samples, r102).  The 6 halo cells come from the tile when
// they lie in the segment (a whole periodic row), else from global memory.  The RK
// base operands q^s, q^n of the epilogue are read from global memory (q^s: L2 hit).
//   raw [E][seg] : the segment's conserved state (TMA destination, 128-byte aligned)
// followed by the shared layout of sweep_x_pair.
// ---------------------------------------------------------------------------
#ifndef MFC_XPAIR_TMA_NBUF
#define MFC_XPAIR_TMA_NBUF 2      // raw tiles per block: 2 = double buffer (the epilogue
#endif                            // reads q^s from its tile; 3 blocks/SM at 57 KB)
template <class M>
__host__ __device__ constexpr size_t x_pair_tma_smem_bytes(int seg) {
    return (size_t)MFC_XPAIR_TMA_NBUF * M::E * seg * sizeof(double) +
           x_pair_smem_doubles<M>(seg) * sizeof(double) + 16 * MFC_XPAIR_TMA_NBUF;
}
template <class M>
__host__ __device__ constexpr int x_pair_tma_minb() { return MFC_XPAIR_TMA_NBUF == 2 ? 3 : x_pair_minb<M>(); }

template <class M, bool RKB>
__global__ void __launch_bounds__(128, x_pair_tma_minb<M>())
sweep_x_pair_tma(const __grid_constant__ CUtensorMap tq, const SweepArgs a, int W, int nsegr,
                 int nseg_total, int ox, int oy, int oz) {
    constexpr int E = M::E;
    const int t = threadIdx.x;
    const int NT = 32 * W;
    const int seg = 2 * NT;
    const int n = a.nS;
    const int LH = NT + 3, LP = NT + 1;
    constexpr int NB = MFC_XPAIR_TMA_NBUF;
    extern __shared__ __align__(128) double smx[];
    double* const raw0 = smx;                                  // [NB][E][seg]
    double* const sm = smx + (size_t)NB * E * seg;
    double* const Ve = sm;                                     // [E][LH]
    double* const Vo = sm + (size_t)E * LH;                    // [E][LH]
    double* const FS = sm;                                     // [E+1][LP] after phase 2
    double* const VM2 = sm + x_pair_smem_doubles<M>(seg) - (size_t)E * LP - E;   // [E][LP]
    double* const VPX = VM2 + (size_t)E * LP;                  // [E]
    uint64_t* const bar0 = reinterpret_cast<uint64_t*>(sm + x_pair_smem_doubles<M>(seg));
    auto V = [&](int e, int i) -> double& {
        return (i & 1) ? Vo[e * LH + (i >> 1)] : Ve[e * LH + (i >> 1)];
    };
    const uint32_t tx_bytes = (uint32_t)(E * seg * sizeof(double));
    // segment sid -> x0 and its row (y, z) = (r % nA, r / nA)
    auto issue = [&](int sid, int b) {
        const int r = sid / nsegr, x0s = (sid % nsegr) * seg;
        mbar_arrive_expect_tx(bar0 + b, tx_bytes);
        tma_load_4d(raw0 + (size_t)b * E * seg, &tq, bar0 + b, ox + x0s, oy + r % a.nA,
                    oz + r / a.nA, 0);
    };
    if (t == 0) {
        tma_prefetch_desc(&tq);
        for (int b = 0; b < NB; ++b) mbar_init(bar0 + b, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (t == 0)
        for (int b = 0; b < NB; ++b)
            if ((int)(blockIdx.x + b * gridDim.x) < nseg_total) issue(blockIdx.x + b * gridDim.x, b);
    uint32_t parity = 0;                  // phase parity of the current buffer's barrier
    const double wi = a.w * a.invd;

    int it = 0;
    for (int sid = blockIdx.x; sid < nseg_total; sid += gridDim.x, ++it) {
        const int buf = NB == 2 ? (it & 1) : 0;
        double* const raw = raw0 + (size_t)buf * E * seg;
        uint64_t* const bar = bar0 + buf;
        const int rr = sid / nsegr;
        const int x0 = (sid % nsegr) * seg;
        const int x1 = min(x0 + seg, n);
        const bool wrap = (a.gm.blo == 1 && a.gm.alo == n) && x0 == 0 && x1 == n && (n & 1) == 0;
        const int tl = n / 2 - 1;
        const int xa = x0 + 2 * t;
        const int64_t row = a.base + (int64_t)(rr % a.nA) * a.sA + (int64_t)(rr / a.nA) * a.sB;

        // RK stage base of my cell x: cb*q^s (+ ca*q^n); q^s from the tile when it is kept
        // to the epilogue (double buffer), else re-read (L2)
        // (single buffer: the tile is kept when the block has no next segment to load)
        const bool kept = NB == 2 || sid + (int)gridDim.x >= nseg_total;
        auto tbase = [&](int x, int e) -> double {
            const double qs = kept ? raw[e * seg + (x - x0)] : __ldg(a.q + row + x + e * a.sE);
            const double b = a.cb * qs;
            return (a.qn != nullptr && a.ca != 0.0) ? fma(a.ca, __ldg(a.qn + row + x + e * a.sE), b) : b;
        };
        // cell of the tile (mapped like every stencil cell) -> primitives
        auto tile_prim = [&](int cell, double (&v)[E]) {
            const int cl = min(cell, x1 + 2);
            const int sc = map_cell(cl, n, a.gm);
            double qc[E];
            if (sc >= x0 && sc < x0 + seg) {
#pragma unroll
                for (int e = 0; e < E; ++e) qc[e] = raw[e * seg + (sc - x0)];
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) qc[e] = __ldg(a.q + row + sc + e * a.sE);
            }
            if (map_flip(cl, n, a.gm)) qc[M::IM] = -qc[M::IM];
            cons_to_prim_fast<M>(qc, v, a.mat);
        };

        // 1. primitives of my two cells and of the six halo cells (tile landed)
        mbar_wait(bar, parity);
        if (NB == 1 || buf == 1) parity ^= 1;     // each buffer's barrier completes once
                                                  // per NB segments
        if constexpr (RKB) {
            // q^n of my cells, read in the epilogue: start it towards L1 now
            if (a.qn != nullptr && a.ca != 0.0 && xa < x1)
#pragma unroll
                for (int e = 0; e < E; ++e)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(a.qn + row + xa + e * a.sE));
        }
        double v0[E], v1[E];
        tile_prim(xa, v0);
        tile_prim(xa + 1, v1);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            Vo[e * LH + t + 1] = v0[e];
            Ve[e * LH + t + 2] = v1[e];
        }
        if (t < 6) {
            double h[E];
            tile_prim(t < 3 ? x0 - 3 + t : x0 + seg + t - 3, h);
            const int i = t < 3 ? t : seg + t;
#pragma unroll
            for (int e = 0; e < E; ++e) V(e, i) = h[e];
        }
        __syncthreads();
        // single buffer: the tile is converted, load the block's next segment into it
        if (NB == 1 && t == 0 && sid + (int)gridDim.x < nseg_total) {
            fence_proxy_async_smem();
            issue(sid + gridDim.x, 0);
        }

        // 2. WENO of both cells
        double vm0[E], vp0[E], vp1[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double a1 = Vo[e * LH + t], a2 = Ve[e * LH + t + 1];
            const double b5 = Vo[e * LH + t + 2], b6 = Ve[e * LH + t + 3];
            const double D2 = a2 - a1, D3 = v0[e] - a2, D4 = v1[e] - v0[e], D5 = b5 - v1[e],
                         D6 = b6 - b5;
            const double s3 = D3 - D2, s4 = D4 - D3, s5 = D5 - D4, s6 = D6 - D5;
            const double S3 = weno_S(s3, a.eps4), S4 = weno_S(s4, a.eps4), S5 = weno_S(s5, a.eps4),
                         S6 = weno_S(s6, a.eps4);
            double vm1;
            weno5_fewop_s(fma(3.0, D3, -D2), D3, D4, D5, v0[e], s3, s4, s5, S3, S4, S5, vm0[e],
                          vp0[e]);
            weno5_fewop_s(fma(3.0, D4, -D3), D4, D5, D6, v1[e], s4, s5, s6, S4, S5, S6, vm1, vp1[e]);
            VM2[e * LP + t + 1] = vm1;
        }
        if (!wrap) {
            const int k = t - (NT - 32);
            if (k >= 0 && k < 2 * E) {
                const bool right = k >= E;
                const int e = right ? k - E : k;
                const int i0 = right ? seg + 1 : 0;
                double r[5];
#pragma unroll
                for (int j = 0; j < 5; ++j) r[j] = V(e, i0 + j);
                const double D0 = r[1] - r[0], D1 = r[2] - r[1], D2 = r[3] - r[2], D3 = r[4] - r[3];
                const double s0 = D1 - D0, s1 = D2 - D1, s2 = D3 - D2;
                double bm, bp;
                weno5_fewop_s(fma(3.0, D1, -D0), D1, D2, D3, r[2], s0, s1, s2, weno_S(s0, a.eps4),
                              weno_S(s1, a.eps4), weno_S(s2, a.eps4), bm, bp);
                if (right) VPX[e] = bp;
                else VM2[e * LP] = bm;
            }
        }
        __syncthreads();

        // 3. my faces xa-1/2 and xa+1/2
        double FA[E], ufA, FB[E], ufB;
        {
            const int li = (wrap && t == 0) ? tl + 1 : t;
            double vL[E];
#pragma unroll
            for (int e = 0; e < E; ++e) vL[e] = VM2[e * LP + li];
            hllc<M, 0>(vL, vp0, a.mat, FA, ufA);
        }
        hllc<M, 0>(vm0, vp1, a.mat, FB, ufB);
#pragma unroll
        for (int e = 0; e < E; ++e) FS[e * LP + t] = FA[e];
        FS[E * LP + t] = ufA;
        if (!wrap && x1 == x0 + seg && t == 0) {
            double vl[E], vr[E], FE[E], ufE;
#pragma unroll
            for (int e = 0; e < E; ++e) { vl[e] = VM2[e * LP + NT]; vr[e] = VPX[e]; }
            hllc<M, 0>(vl, vr, a.mat, FE, ufE);
#pragma unroll
            for (int e = 0; e < E; ++e) FS[e * LP + NT] = FE[e];
            FS[E * LP + NT] = ufE;
        }
        __syncthreads();

        // 4. updates
        if (xa < x1) {
            const double du = ufB - ufA;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                double r = FA[e] - FB[e];
                if (e >= M::IA) r = fma(v0[e], du, r);
                if constexpr (RKB)
                    a.dst[row + xa + e * a.sE] = fma(wi, r, tbase(xa, e));
                else
                    a.dst[row + xa + e * a.sE] = r * a.invd;
            }
        }
        if (xa + 1 < x1) {
            const int ri = (wrap && t == tl) ? 0 : t + 1;
            const double du = FS[E * LP + ri] - ufB;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                double r = FB[e] - FS[e * LP + ri];
                if (e >= M::IA) r = fma(v1[e], du, r);
                if constexpr (RKB)
                    a.dst[row + xa + 1 + e * a.sE] = fma(wi, r, tbase(xa + 1, e));
                else
                    a.dst[row + xa + 1 + e * a.sE] = r * a.invd;
            }
        }
        __syncthreads();      // FS (aliasing Ve/Vo) is read above; the next segment writes Ve/Vo
        // double buffer: this tile is free now (its last reads were the RK bases above)
        if (NB == 2 && t == 0 && sid + 2 * (int)gridDim.x < nseg_total) {
            fence_proxy_async_smem();
            issue(sid + 2 * gridDim.x, buf);
        }
    }
}

}  // namespace mfc
