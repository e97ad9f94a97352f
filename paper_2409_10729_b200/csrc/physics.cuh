// physics.cuh -- per-cell / per-face device functions of the fused sweep kernels.
//
// The arithmetic is DESIGN.md §3 re-derived for the GPU:
//  * cons -> prim (S2) uses the exact operation order of the specification with
//    explicit round-to-nearest intrinsics (no FMA contraction), so the pressure of
//    a water cell -- which loses log10(Pi/(Gamma p)) digits in rhoE - KE - Pi
//    (AMB-18) -- is bitwise the specified value.
//  * WENO5-JS (Shu [15]) is evaluated once per cell for BOTH face
//    states of that cell (v-_{m+1/2} and v+_{m-1/2} share beta_k), with the three
//    alpha_k = d_k/(beta_k+eps)^2 normalised through products of the other two
//    (beta_j+eps)^2, i.e. one reciprocal per side instead of three divisions.
//    Same weights up to rounding.
//  * HLLC (Toro [14] ch.10) in the compact branch form of S3, with
//    the face velocity u^f that also feeds the alpha*div(u) source (AMB-5/6).
#pragma once
#include <cstdint>

#ifndef MFC_WENO_ONE_RCP
#define MFC_WENO_ONE_RCP 1      // r98: C3 x -0.034, y -0.010, z -0.014 ms per step (3 reps)
#endif
#ifndef MFC_WENO5M_ONE_RCP
#define MFC_WENO5M_ONE_RCP 1   // r100: C3 --weno 5m 10.43-10.53 -> 10.32-10.42 ms (3 reps)
#endif
#ifndef MFC_WENO3_ONE_RCP
#define MFC_WENO3_ONE_RCP 1      // r102: C3 --weno 3 5.493-5.512 -> 5.461-5.484 ms (3 reps)
#endif
#ifndef MFC_WENO5M_ALPHA
#define MFC_WENO5M_ALPHA 1      // r101: C3 --weno 5m 10.322 -> 10.304 ms (3 reps; x +0.007, z -0.023)
#endif
#ifndef MFC_HLLC_ONE_RCP
#define MFC_HLLC_ONE_RCP 1   // r96: x -0.015, y -0.01 ms per step (same box, 3 repetitions)
#endif

namespace mfc {

constexpr int kGhost = 3;
constexpr int kMaxFluids = 3;

template <int NF, int ND>
struct Model {
    static constexpr int N = NF;              // fluids
    static constexpr int D = ND;              // active dimensions
    static constexpr int E = 2 * NF + ND + 1; // equations
    static constexpr int IM = NF;             // first momentum / velocity
    static constexpr int IE = NF + ND;        // energy / pressure
    static constexpr int IA = NF + ND + 1;    // first volume fraction
};

struct Materials {
    double Gam[kMaxFluids];   // 1/(gamma_i - 1)
    double Pi[kMaxFluids];    // gamma_i pi_inf_i/(gamma_i - 1)
};

// Fast reciprocal: MUFU.RCP64H seed r0 (~2^-23 relative error d) and one third-order
// correction r = r0 (1 + e + e^2), e = 1 - x r0, leaving O(d^3) ~ 2^-69.  Used only
// where the specification does not fix the rounding (WENO weights, HLLC quotients,
// the sweeps' EOS); the API conversions keep IEEE division.
__device__ __forceinline__ double rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = __fma_rn(-x, r, 1.0);
    e = __fma_rn(e, e, e);
    return __fma_rn(r, e, r);
}

// S2: conserved -> primitive, in the specified order, no contraction:
//   rho = ((a1r1 + a2r2) + ...);  u_k = (rho u_k)/rho;  KE = 0.5 * sum_k (rho u_k) u_k;
//   Gamma = sum a_i Gamma_i;  Pi = sum a_i Pi_i;  p = ((rhoE - KE) - Pi)/Gamma.
template <class M>
__device__ __forceinline__ void cons_to_prim(const double (&q)[M::E], double (&v)[M::E],
                                             const Materials& mat) {
    double rho = q[0];
#pragma unroll
    for (int i = 1; i < M::N; ++i) rho = __dadd_rn(rho, q[i]);
    double ke = 0.0;
#pragma unroll
    for (int k = 0; k < M::D; ++k) {
        const double u = __ddiv_rn(q[M::IM + k], rho);
        v[M::IM + k] = u;
        ke = __dadd_rn(ke, __dmul_rn(q[M::IM + k], u));
    }
    ke = __dmul_rn(0.5, ke);
    double G = __dmul_rn(q[M::IA], mat.Gam[0]);
    double P = __dmul_rn(q[M::IA], mat.Pi[0]);
#pragma unroll
    for (int i = 1; i < M::N; ++i) {
        G = __dadd_rn(G, __dmul_rn(q[M::IA + i], mat.Gam[i]));
        P = __dadd_rn(P, __dmul_rn(q[M::IA + i], mat.Pi[i]));
    }
#pragma unroll
    for (int i = 0; i < M::N; ++i) {
        v[i] = q[i];
        v[M::IA + i] = q[M::IA + i];
    }
    v[M::IE] = __ddiv_rn(__dsub_rn(__dsub_rn(q[M::IE], ke), P), G);
}

// S2 for the sweep kernels: the same formulas with ONE reciprocal per cell,
// r = 1/(rho*Gamma): 1/rho = Gamma*r, 1/Gamma = rho*r (FMA allowed).  Differs from
// the specified order by a few ulp of each term (within the parity metric of
// DESIGN.md AMB-17); the bitwise-specified version above serves mfc_cons_to_prim.
template <class M>
__device__ __forceinline__ void cons_to_prim_fast(const double (&q)[M::E], double (&v)[M::E],
                                                  const Materials& mat) {
    // explicit roundings: a march converts its first cells and the streamed ones at two
    // inline sites, which must not contract differently (bitwise segment independence)
    double rho = q[0];
#pragma unroll
    for (int i = 1; i < M::N; ++i) rho = __dadd_rn(rho, q[i]);
    double G = __dmul_rn(q[M::IA], mat.Gam[0]);
    double P = __dmul_rn(q[M::IA], mat.Pi[0]);
#pragma unroll
    for (int i = 1; i < M::N; ++i) {
        G = __fma_rn(q[M::IA + i], mat.Gam[i], G);
        P = __fma_rn(q[M::IA + i], mat.Pi[i], P);
    }
    const double r = rcp(__dmul_rn(rho, G));
    const double irho = __dmul_rn(G, r), iG = __dmul_rn(rho, r);
    double ke = 0.0;
#pragma unroll
    for (int k = 0; k < M::D; ++k) {
        const double u = __dmul_rn(q[M::IM + k], irho);
        v[M::IM + k] = u;
        ke = __fma_rn(q[M::IM + k], u, ke);
    }
#pragma unroll
    for (int i = 0; i < M::N; ++i) {
        v[i] = q[i];
        v[M::IA + i] = q[M::IA + i];
    }
    v[M::IE] = __dmul_rn(__dsub_rn(__fma_rn(-0.5, ke, q[M::IE]), P), iG);
}

// Fast reciprocal square root: MUFU.RSQ64H seed y0 and one third-order correction
// y = y0 (1 + e/2 + 3e^2/8), e = 1 - x y0^2.
__device__ __forceinline__ double rsqrt_fast(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}

// Inverse EOS: rho u_k = rho*u_k;  KE = 0.5 sum (rho u_k) u_k;  rhoE = (Gamma p + Pi) + KE.
template <class M>
__device__ __forceinline__ void prim_to_cons(const double (&v)[M::E], double (&q)[M::E],
                                             const Materials& mat) {
    double rho = v[0];
#pragma unroll
    for (int i = 1; i < M::N; ++i) rho = __dadd_rn(rho, v[i]);
    double ke = 0.0;
#pragma unroll
    for (int k = 0; k < M::D; ++k) {
        const double m = __dmul_rn(rho, v[M::IM + k]);
        q[M::IM + k] = m;
        ke = __dadd_rn(ke, __dmul_rn(m, v[M::IM + k]));
    }
    ke = __dmul_rn(0.5, ke);
    double G = __dmul_rn(v[M::IA], mat.Gam[0]);
    double P = __dmul_rn(v[M::IA], mat.Pi[0]);
#pragma unroll
    for (int i = 1; i < M::N; ++i) {
        G = __dadd_rn(G, __dmul_rn(v[M::IA + i], mat.Gam[i]));
        P = __dadd_rn(P, __dmul_rn(v[M::IA + i], mat.Pi[i]));
    }
#pragma unroll
    for (int i = 0; i < M::N; ++i) {
        q[i] = v[i];
        q[M::IA + i] = v[M::IA + i];
    }
    q[M::IE] = __dadd_rn(__dadd_rn(__dmul_rn(G, v[M::IE]), P), ke);
}

// WENO5-JS for one variable of cell m from a..e = v_{m-2..m+2}:
//   vm = v-_{m+1/2} (linear weights 0.1, 0.6, 0.3), vp = v+_{m-1/2} (0.3, 0.6, 0.1).
// Same weights and candidates as the specification, evaluated in first differences
// D0..D3 = b-a, c-b, d-c, e-d:
//   beta'_k = 4 beta_k = (13/3) s_k^2 + r_k^2,  s = (D1-D0, D2-D1, D3-D2),
//             r = (3D1-D0, D1+D2, D3-3D2)      (eps' = 4 eps keeps every alpha_k ratio),
//   alpha_k ~ d_k / t_k, t_k = (beta'_k + eps')^2, multiplied through by t0 t1 t2:
//             alpha_k ~ d_k P_k with P_k = product of the other two t_j,
//   candidates as corrections to c: 6(p_k - c) = (5D1-2D0, D1+2D2, 4D2-D3) for v-,
//             (D0-4D1, -2D1-D2, 2D3-5D2) for v+,
//   v = c + (sum_k d_k P_k (p_k - c)) / (sum_k d_k P_k):  one reciprocal per side,
//   with the linear weights scaled to integers (below) so no product is spent on them.
// (weno5_d takes the differences D0..D3 and the centre value c: the marches carry
//  D0, D1 from the previous step, where they were that step's D1, D2 -- the same
//  subtractions of the same operands, so bitwise the same values.)
__device__ __forceinline__ void weno5_d(double D0, double D1, double D2, double D3, double c,
                                        double eps4, double& vm, double& vp) {
    constexpr double k133 = 13.0 / 3.0;
    const double s0 = D1 - D0, s1 = D2 - D1, s2 = D3 - D2;
    const double r0 = fma(3.0, D1, -D0), r1 = D1 + D2, r2 = fma(-3.0, D2, D3);
    double t0 = fma(k133 * s0, s0, fma(r0, r0, eps4)); t0 *= t0;
    double t1 = fma(k133 * s1, s1, fma(r1, r1, eps4)); t1 *= t1;
    double t2 = fma(k133 * s2, s2, fma(r2, r2, eps4)); t2 *= t2;
    const double P0 = t1 * t2, P1 = t0 * t2, P2 = t0 * t1;
    // sum_k d_k P_k scaled by 10 (integer weights), the corrections 6(p_k - c) by 10/6:
    //   v- (10d = 1, 6, 3): Dm = P0 + 6 P1 + 3 P2,
    //       Nm = P0 (5D1-2D0)/6 + P1 (D1+2D2) + P2 (2D2-D3/2),          v- = c + Nm/Dm
    //   v+ (10d = 3, 6, 1): Dp = 3 P0 + 6 P1 + P2,
    //       Np = P0 (D0/2-2D1) + P1 (-2D1-D2) + P2 (D3/3-5D2/6),        v+ = c + Np/Dp
    constexpr double k56 = 5.0 / 6.0, k13 = 1.0 / 3.0;
    const double xm0 = fma(k56, D1, -k13 * D0);
    const double xm1 = fma(2.0, D2, D1);
    const double xm2 = fma(2.0, D2, -0.5 * D3);
    const double Dm = fma(6.0, P1, fma(3.0, P2, P0));
    const double Nm = fma(P2, xm2, fma(P1, xm1, P0 * xm0));
    vm = fma(Nm, rcp(Dm), c);
    const double xp0 = fma(-2.0, D1, 0.5 * D0);
    const double xp1 = fma(-2.0, D1, -D2);
    const double xp2 = fma(k13, D3, -k56 * D2);
    const double Dp = fma(3.0, P0, fma(6.0, P1, P2));
    const double Np = fma(P2, xp2, fma(P1, xp1, P0 * xp0));
    vp = fma(Np, rcp(Dp), c);
}

// WENO5-JS with two FP64 operations fewer per variable than weno5 (same beta'_k, t_k,
// P_k), used by the row-parallel x tile, whose 80 registers leave room for it; in the
// 168-register y/z marches its longer-lived differences spill (r61: y/z +47% per
// launch), so those keep weno5.
//   candidates as corrections to c: A_k = 6(p_k - c) = (5D1-2D0, D1+2D2, 4D2-D3) for v-,
//             (D0-4D1, -2D1-D2, 2D3-5D2) for v+,
//   v = c + (1/6) (sum_k d_k P_k A_k) / (sum_k d_k P_k):  one reciprocal per side.
// The numerator takes X_k = lambda (10 d_k/6) A_k with lambda = 2, which makes every X_k
// ONE operation on the differences already formed (no product spent on a weight):
//   v-: X = (A0/3, 2 A1, A2) = ((2/3) s0 + D1, 3 r1 + s1, D2 - r2),
//       denominator 20 sum d_k P_k = 2 P0 + 12 P1 + 6 P2;
//   v+: X = (A0, 2 A1, A2/3) = -(r0 + D1, 3 r1 - s1, D2 - (2/3) s2),
//       denominator 6 P0 + 12 P1 + 2 P2.
// (51 FP64 operations per variable; weno5 takes 53.)
__device__ __forceinline__ void weno5_fewop_d(double D0, double D1, double D2, double D3, double c,
                                              double eps4, double& vm, double& vp) {
    constexpr double k133 = 13.0 / 3.0, k23 = 2.0 / 3.0;
    const double s0 = D1 - D0, s1 = D2 - D1, s2 = D3 - D2;
    const double r0 = fma(3.0, D1, -D0), r1 = D1 + D2, r2 = fma(-3.0, D2, D3);
    double t0 = fma(k133 * s0, s0, fma(r0, r0, eps4)); t0 *= t0;
    double t1 = fma(k133 * s1, s1, fma(r1, r1, eps4)); t1 *= t1;
    double t2 = fma(k133 * s2, s2, fma(r2, r2, eps4)); t2 *= t2;
    const double P0 = t1 * t2, P1 = t0 * t2, P2 = t0 * t1;
    const double xm0 = fma(k23, s0, D1), xm1 = fma(3.0, r1, s1), xm2 = D2 - r2;
    const double A12 = 12.0 * P1;        // shared by both weight sums (5 operations, not 6)
    const double Dm = fma(2.0, P0, fma(6.0, P2, A12));
    const double Nm = fma(P2, xm2, fma(P1, xm1, P0 * xm0));
    const double yp0 = r0 + D1, yp1 = fma(3.0, r1, -s1), yp2 = fma(-k23, s2, D2);   // = -X
    const double Dp = fma(6.0, P0, fma(2.0, P2, A12));
    const double Np = fma(P2, yp2, fma(P1, yp1, P0 * yp0));
#if MFC_WENO_ONE_RCP
    const double R = rcp(Dm * Dp);           // see weno5_fewop_s
    vm = fma(Nm * Dp, R, c);
    vp = fma(-Np * Dm, R, c);
#else
    vm = fma(Nm, rcp(Dm), c);
    vp = fma(-Np, rcp(Dp), c);
#endif
}

// weno5_fewop with the curvature terms passed in: S_k = (13/3) s_k^2 + eps' formed by the
// caller (fma(k133 s, s, eps')), beta'_k + eps' = r_k^2 + S_k.  A thread reconstructing two
// neighbouring cells shares the s_k and S_k of the difference pairs both stencils
// contain (sweep_x_pair); every cell's arithmetic is the same sequence whichever role
// (first or second of a pair, or a segment-boundary cell) it has.
// The caller also forms r0 = 3D1 - D0: the x pair as fma(3, D1, -D0), a march that
// carries s0 instead of D0 as 2D1 + s0.
__device__ __forceinline__ void weno5_fewop_s(double r0, double D1, double D2, double D3, double c,
                                              double s0, double s1, double s2, double S0,
                                              double S1, double S2, double& vm, double& vp) {
    constexpr double k23 = 2.0 / 3.0;
    const double r1 = D1 + D2, r2 = fma(-3.0, D2, D3);
    double t0 = fma(r0, r0, S0); t0 *= t0;
    double t1 = fma(r1, r1, S1); t1 *= t1;
    double t2 = fma(r2, r2, S2); t2 *= t2;
    const double P0 = t1 * t2, P1 = t0 * t2, P2 = t0 * t1;
    const double xm0 = fma(k23, s0, D1), xm1 = fma(3.0, r1, s1), xm2 = D2 - r2;
    const double A12 = 12.0 * P1;        // shared by both weight sums (5 operations, not 6)
    const double Dm = fma(2.0, P0, fma(6.0, P2, A12));
    const double Nm = fma(P2, xm2, fma(P1, xm1, P0 * xm0));
    const double yp0 = r0 + D1, yp1 = fma(3.0, r1, -s1), yp2 = fma(-k23, s2, D2);   // = -X
    const double Dp = fma(6.0, P0, fma(2.0, P2, A12));
    const double Np = fma(P2, yp2, fma(P1, yp1, P0 * yp0));
#if MFC_WENO_ONE_RCP
    // one reciprocal for both sides: 1/Dm = Dp R, 1/Dp = Dm R, R = 1/(Dm Dp)
    // (Dm Dp <= ~1e170 for |dv| <= 1e10, >= ~1e-123 for eps' = 4e-16)
    const double R = rcp(Dm * Dp);
    vm = fma(Nm * Dp, R, c);
    vp = fma(-Np * Dm, R, c);
#else
    vm = fma(Nm, rcp(Dm), c);
    vp = fma(-Np, rcp(Dp), c);
#endif
}
__device__ __forceinline__ double weno_S(double s, double eps4) {
    return fma((13.0 / 3.0) * s, s, eps4);
}

__device__ __forceinline__ void weno5(double a, double b, double c, double d, double e,
                                      double eps4, double& vm, double& vp) {
    weno5_d(b - a, c - b, d - c, e - d, c, eps4, vm, vp);
}
__device__ __forceinline__ void weno5_fewop(double a, double b, double c, double d, double e,
                                            double eps4, double& vm, double& vp) {
    weno5_fewop_d(b - a, c - b, d - c, e - d, c, eps4, vm, vp);
}

// WENO5-JS on a non-uniform grid (F4, DESIGN.md AMB-27) for one variable of cell m from
// its first differences D0..D3 (D_i = v_{m-1+i} - v_{m-2+i}) and v_m = c, with the cell's
// coefficients K (K[i * ld] = coefficient i of the NU_* layout in sweep.cuh):
//   b_k, s_k = sqrt(13/3) c_k: two products on candidate k's differences each,
//   beta_k = b_k² + s_k²,  t_k = (beta_k + eps)²,  P_k = product of the other two t_j,
//   v- = v_m + (sum_k d-_k P_k A-_k) / (sum_k d-_k P_k),  A-_k = q_k(x_{m+1/2}) - v_m
//   (the same with d+ and A+ for v+), one reciprocal for both sides as in weno5_fewop_s.
// (PLAIN: K is a register array or shared memory, read with plain loads; else read-only
//  global loads)
template <bool PLAIN>
__device__ __forceinline__ double nu_ld(const double* K) {
    if constexpr (PLAIN) return *K;
    else return __ldg(K);
}
template <bool PLAIN = false>
__device__ __forceinline__ void weno5_nu(double D0, double D1, double D2, double D3, double c,
                                         const double* __restrict__ K, int64_t ld, double eps,
                                         double& vm, double& vp) {
    const double Da[3] = {D0, D1, D2}, Db[3] = {D1, D2, D3};
    double t[3], Am[3], Ap[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double b = fma(nu_ld<PLAIN>(K + (2 * k) * ld), Da[k], nu_ld<PLAIN>(K + (2 * k + 1) * ld) * Db[k]);
        const double sc = fma(nu_ld<PLAIN>(K + (6 + 2 * k) * ld), Da[k], nu_ld<PLAIN>(K + (7 + 2 * k) * ld) * Db[k]);
        double tk = fma(b, b, fma(sc, sc, eps));
        t[k] = tk * tk;
        Am[k] = fma(nu_ld<PLAIN>(K + (12 + 2 * k) * ld), Da[k], nu_ld<PLAIN>(K + (13 + 2 * k) * ld) * Db[k]);
        Ap[k] = fma(nu_ld<PLAIN>(K + (18 + 2 * k) * ld), Da[k], nu_ld<PLAIN>(K + (19 + 2 * k) * ld) * Db[k]);
    }
    const double P0 = t[1] * t[2], P1 = t[0] * t[2], P2 = t[0] * t[1];
    const double wm0 = nu_ld<PLAIN>(K + 24 * ld) * P0, wm1 = nu_ld<PLAIN>(K + 25 * ld) * P1,
                 wm2 = nu_ld<PLAIN>(K + 26 * ld) * P2;
    const double wp0 = nu_ld<PLAIN>(K + 27 * ld) * P0, wp1 = nu_ld<PLAIN>(K + 28 * ld) * P1,
                 wp2 = nu_ld<PLAIN>(K + 29 * ld) * P2;
    const double Zm = (wm0 + wm1) + wm2, Zp = (wp0 + wp1) + wp2;
    const double Nm = fma(wm2, Am[2], fma(wm1, Am[1], wm0 * Am[0]));
    const double Np = fma(wp2, Ap[2], fma(wp1, Ap[1], wp0 * Ap[0]));
    const double R = rcp(Zm * Zp);
    vm = fma(Nm * Zp, R, c);
    vp = fma(Np * Zm, R, c);
}

// WENO5-M (Henrick, Aslam & Powers, JCP 207 (2005) 542): the Jiang-Shu
// weights omega_k = d_k P_k / sum_j d_j P_j (P_k as in weno5) mapped by
//   g_k(w) = w (d_k + d_k^2 - 3 d_k w + w^2) / (d_k^2 + w (1 - 2 d_k))
// and renormalised, multiplied through by the three denominators:
//   omega*_k ~ Q_k = num_k den_i den_j,  v = c + (sum_k Q_k A_k/6) / sum_k Q_k,
// A_k = 6 (p_k - c) the candidate corrections (as in weno5): two reciprocals per side.
__device__ __forceinline__ void weno5m_side(const double (&P)[3], const double (&A)[3],
                                            const double (&d)[3], double c, double& v) {
    const double W = rcp(fma(d[2], P[2], fma(d[1], P[1], d[0] * P[0])));
    double num[3], den[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double w = d[k] * P[k] * W;
        num[k] = w * fma(w, w - 3.0 * d[k], fma(d[k], d[k], d[k]));
        den[k] = fma(w, 1.0 - 2.0 * d[k], d[k] * d[k]);
    }
    const double Q0 = num[0] * (den[1] * den[2]);
    const double Q1 = num[1] * (den[0] * den[2]);
    const double Q2 = num[2] * (den[0] * den[1]);
    const double N = fma(Q2, A[2], fma(Q1, A[1], Q0 * A[0]));
    v = fma(N * (1.0 / 6.0), rcp((Q0 + Q1) + Q2), c);
}

// the mapped, un-normalised weights of one side given W = 1/sum_k d_k P_k:
// N = sum_k Q_k A_k, S = sum_k Q_k
__device__ __forceinline__ void weno5m_sums(const double (&P)[3], const double (&A)[3],
                                            const double (&d)[3], double W, double& N,
                                            double& S) {
    double num[3], den[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double w = d[k] * P[k] * W;
        num[k] = w * fma(w, w - 3.0 * d[k], fma(d[k], d[k], d[k]));
        den[k] = fma(w, 1.0 - 2.0 * d[k], d[k] * d[k]);
    }
    const double Q0 = num[0] * (den[1] * den[2]);
    const double Q1 = num[1] * (den[0] * den[2]);
    const double Q2 = num[2] * (den[0] * den[1]);
    N = fma(Q2, A[2], fma(Q1, A[1], Q0 * A[0]));
    S = (Q0 + Q1) + Q2;
}

// weno5m_sums from the unnormalised weights a_k = d_k P_k: w_k = a_k W
__device__ __forceinline__ void weno5m_sums_a(const double (&a)[3], const double (&A)[3],
                                              const double (&d)[3], double W, double& N,
                                              double& S) {
    double num[3], den[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double w = a[k] * W;
        num[k] = w * fma(w, w - 3.0 * d[k], fma(d[k], d[k], d[k]));
        den[k] = fma(w, 1.0 - 2.0 * d[k], d[k] * d[k]);
    }
    const double Q0 = num[0] * (den[1] * den[2]);
    const double Q1 = num[1] * (den[0] * den[2]);
    const double Q2 = num[2] * (den[0] * den[1]);
    N = fma(Q2, A[2], fma(Q1, A[1], Q0 * A[0]));
    S = (Q0 + Q1) + Q2;
}

__device__ __forceinline__ void weno5m(double a, double b, double c, double d, double e,
                                       double eps4, double& vm, double& vp) {
    constexpr double k133 = 13.0 / 3.0;
    const double D0 = b - a, D1 = c - b, D2 = d - c, D3 = e - d;
    const double s0 = D1 - D0, s1 = D2 - D1, s2 = D3 - D2;
    const double r0 = fma(3.0, D1, -D0), r1 = D1 + D2, r2 = fma(-3.0, D2, D3);
    double t0 = fma(k133 * s0, s0, fma(r0, r0, eps4)); t0 *= t0;
    double t1 = fma(k133 * s1, s1, fma(r1, r1, eps4)); t1 *= t1;
    double t2 = fma(k133 * s2, s2, fma(r2, r2, eps4)); t2 *= t2;
    const double P[3] = {t1 * t2, t0 * t2, t0 * t1};
    const double Am[3] = {fma(5.0, D1, -2.0 * D0), fma(2.0, D2, D1), fma(4.0, D2, -D3)};
    const double Ap[3] = {fma(-4.0, D1, D0), fma(-2.0, D1, -D2), fma(2.0, D3, -5.0 * D2)};
    const double dm[3] = {0.1, 0.6, 0.3}, dp[3] = {0.3, 0.6, 0.1};
#if MFC_WENO5M_ONE_RCP
    // both sides at once, one reciprocal for each pair of divisions (as in weno5_fewop_d):
    // 1/Zm = Zp R1, 1/Zp = Zm R1 with R1 = 1/(Zm Zp), and the same for the two
    // renormalisations. Zm Zp ~ P^2 (<= ~1e160 for |dv| <= 1e10, >= ~1e-124 for
    // eps' = 4e-16); the sums of Q are O(1e-3 .. 1).
    double Nm, Sm, Np, Sp;
#if MFC_WENO5M_ALPHA
    // the unnormalised Jiang-Shu weights a_k = d_k P_k formed once (0.6 P1 shared by both
    // sides) and reused for the sums and for w_k = a_k W: 4 FP64 fewer per variable
    const double a1 = 0.6 * P[1];
    const double am[3] = {0.1 * P[0], a1, 0.3 * P[2]}, ap[3] = {0.3 * P[0], a1, 0.1 * P[2]};
    const double Zm = (am[0] + am[1]) + am[2], Zp = (ap[0] + ap[1]) + ap[2];
    const double R1 = rcp(Zm * Zp);
    weno5m_sums_a(am, Am, dm, Zp * R1, Nm, Sm);
    weno5m_sums_a(ap, Ap, dp, Zm * R1, Np, Sp);
#else
    const double Zm = fma(dm[2], P[2], fma(dm[1], P[1], dm[0] * P[0]));
    const double Zp = fma(dp[2], P[2], fma(dp[1], P[1], dp[0] * P[0]));
    const double R1 = rcp(Zm * Zp);
    const double Wm = Zp * R1, Wp = Zm * R1;
    weno5m_sums(P, Am, dm, Wm, Nm, Sm);
    weno5m_sums(P, Ap, dp, Wp, Np, Sp);
#endif
    const double R2 = rcp(Sm * Sp) * (1.0 / 6.0);
    vm = fma(Nm * Sp, R2, c);
    vp = fma(Np * Sm, R2, c);
#else
    weno5m_side(P, Am, dm, c, vm);
    weno5m_side(P, Ap, dp, c, vp);
#endif
}

// WENO3-JS ("third or fifth-order"; F2) for one variable of cell m from
// a..c = v_{m-1..m+1}, in first differences D0 = b-a, D1 = c-b:
//   beta = (D0^2, D1^2), alpha_k ~ d_k/(beta_k+eps)^2 multiplied through by t0 t1,
//   v- = b + (d0 t1 D0/2 + d1 t0 D1/2)/(d0 t1 + d1 t0),  d = (1/3, 2/3)
//   v+ = b - (e0 t1 D0/2 + e1 t0 D1/2)/(e0 t1 + e1 t0),  e = (2/3, 1/3)
__device__ __forceinline__ void weno3(double a, double b, double c, double eps, double& vm,
                                      double& vp) {
    const double D0 = b - a, D1 = c - b;
    double t0 = fma(D0, D0, eps); t0 *= t0;
    double t1 = fma(D1, D1, eps); t1 *= t1;
    const double wm0 = t1 * (1.0 / 3.0), wm1 = t0 * (2.0 / 3.0);
    const double wp0 = t1 * (2.0 / 3.0), wp1 = t0 * (1.0 / 3.0);
#if MFC_WENO3_ONE_RCP
    // one reciprocal for both sides (as in weno5_fewop_d): Zm Zp ~ t^2 with
    // t_k = (D_k^2 + eps)^2, so >= ~1e-120 for eps >= 1e-30, <= ~1e80 for |dv| <= 1e10
    const double Zm = wm0 + wm1, Zp = wp0 + wp1;
    const double R = rcp(Zm * Zp) * 0.5;
    vm = fma(fma(wm1, D1, wm0 * D0) * Zp, R, b);
    vp = fma(-fma(wp1, D1, wp0 * D0) * Zm, R, b);
#else
    vm = fma(0.5 * fma(wm1, D1, wm0 * D0), rcp(wm0 + wm1), b);
    vp = fma(-0.5 * fma(wp1, D1, wp0 * D0), rcp(wp0 + wp1), b);
#endif
}

// HLLC face flux F[E] and face velocity uf for the normal direction DIR
// from the reconstructed primitive states vL (cell m's v-) and vR (cell m+1's v+).
template <class M, int DIR>
__device__ __forceinline__ void hllc(const double (&vL)[M::E], const double (&vR)[M::E],
                                     const Materials& mat, double (&F)[M::E], double& uf) {
    double rL = vL[0], rR = vR[0];
#pragma unroll
    for (int i = 1; i < M::N; ++i) { rL += vL[i]; rR += vR[i]; }
    double GL = vL[M::IA] * mat.Gam[0], GR = vR[M::IA] * mat.Gam[0];
    double PL = vL[M::IA] * mat.Pi[0], PR = vR[M::IA] * mat.Pi[0];
#pragma unroll
    for (int i = 1; i < M::N; ++i) {
        GL = fma(vL[M::IA + i], mat.Gam[i], GL);
        GR = fma(vR[M::IA + i], mat.Gam[i], GR);
        PL = fma(vL[M::IA + i], mat.Pi[i], PL);
        PR = fma(vR[M::IA + i], mat.Pi[i], PR);
    }
    const double uL = vL[M::IM + DIR], uR = vR[M::IM + DIR];
    const double pL = vL[M::IE], pR = vR[M::IE];
    // c = sqrt(A/B) = A * rsqrt(A*B), A = (Gamma+1)p + Pi, B = rho*Gamma (AMB-10)
    const double AL = fma(GL + 1.0, pL, PL), AR = fma(GR + 1.0, pR, PR);
    const double cL = AL * rsqrt_fast(AL * (rL * GL));
    const double cR = AR * rsqrt_fast(AR * (rR * GR));
    const double sL = fmin(uL - cL, uR - cR);
    const double sR = fmax(uL + cL, uR + cR);
    const double aL = rL * (sL - uL), aR = rR * (sR - uR);
    // (every multiply-add is an explicit fma: contraction must not depend on the
    //  inlining site, so a face computed by two code paths is bitwise identical)
#if MFC_HLLC_ONE_RCP
    // s_S = num/den with den = aL - aR < 0 (aL < 0 < aR for positive densities and sound
    // speeds), so s_S >= 0  <=>  num <= 0: the side is chosen before any division, and
    // ONE reciprocal R = 1/(den dK D2), D2 = den dS = sK den - num, serves s_S = num dK D2 R,
    // 1/(dK dS) = den^2 R and p_K/(s_K-u_K) = p_K D2 den R (one MUFU round trip fewer on
    // the face's dependency chain)
    const double num = fma(-aR, uR, fma(aL, uL, pR - pL));
    const double den = aL - aR;
    const bool left = num <= 0.0;
#else
    const double sS = fma(-aR, uR, fma(aL, uL, pR - pL)) * rcp(aL - aR);

    const bool left = sS >= 0.0;
#endif
    const double sK = left ? sL : sR;
    const double sstar = left ? fmin(0.0, sL) : fmax(0.0, sR);
    const double rK = left ? rL : rR;
    const double uK = left ? uL : uR;
    const double pK = left ? pL : pR;
    const double GK = left ? GL : GR;
    const double PK = left ? PL : PR;
    double uu = 0.0;
    double vK[M::E];
#pragma unroll
    for (int e = 0; e < M::E; ++e) vK[e] = left ? vL[e] : vR[e];
#pragma unroll
    for (int k = 0; k < M::D; ++k) uu = fma(vK[M::IM + k], vK[M::IM + k], uu);
    const double EK = fma(0.5, rK * uu, fma(GK, pK, PK));
    const double dK = sK - uK;
#if MFC_HLLC_ONE_RCP
    const double D2 = fma(sK, den, -num);
    const double R = rcp((den * dK) * D2);
    const double sS = num * ((dK * D2) * R);
    const double rr = (den * den) * R;       // 1/(dK dS)
    const double pdK = pK * ((D2 * den) * R);   // p_K/(s_K-u_K)
#else
    const double dS = sK - sS;
    const double rr = rcp(dK * dS);          // one reciprocal for xi and p_K/(s_K-u_K)
    const double pdK = pK * (dS * rr);
#endif
    const double xi = (dK * dK) * rr;
    const double ufv = fma(sstar, xi - 1.0, uK);
#pragma unroll
    for (int i = 0; i < M::N; ++i) {
        F[i] = vK[i] * ufv;
        F[M::IA + i] = vK[M::IA + i] * ufv;
    }
#pragma unroll
    for (int k = 0; k < M::D; ++k) {
        if (k == DIR) {
            F[M::IM + k] = fma(sstar, rK * fma(xi, sS, -uK), fma(rK * uK, uK, pK));
        } else {
            F[M::IM + k] = (rK * vK[M::IM + k]) * ufv;
        }
    }
    const double inner = fma(sS - uK, fma(rK, sS, pdK), EK);
    F[M::IE] = fma(sstar, fma(xi, inner, -EK), uK * (EK + pK));
    uf = ufv;
}

}  // namespace mfc
