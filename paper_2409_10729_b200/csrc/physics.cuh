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

// Fast reciprocal: MUFU.RCP64H seed + two Newton steps (relative error ~1 ulp).
// Used only where the specification does not fix the rounding (WENO weights,
// HLLC quotients); the EOS path keeps IEEE division.
__device__ __forceinline__ double rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = __fma_rn(-x, r, 1.0);
    r = __fma_rn(r, e, r);
    e = __fma_rn(-x, r, 1.0);
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
    double rho = q[0];
#pragma unroll
    for (int i = 1; i < M::N; ++i) rho += q[i];
    double G = q[M::IA] * mat.Gam[0];
    double P = q[M::IA] * mat.Pi[0];
#pragma unroll
    for (int i = 1; i < M::N; ++i) {
        G = fma(q[M::IA + i], mat.Gam[i], G);
        P = fma(q[M::IA + i], mat.Pi[i], P);
    }
    const double r = rcp(rho * G);
    const double irho = G * r, iG = rho * r;
    double ke = 0.0;
#pragma unroll
    for (int k = 0; k < M::D; ++k) {
        const double u = q[M::IM + k] * irho;
        v[M::IM + k] = u;
        ke = fma(q[M::IM + k], u, ke);
    }
#pragma unroll
    for (int i = 0; i < M::N; ++i) {
        v[i] = q[i];
        v[M::IA + i] = q[M::IA + i];
    }
    v[M::IE] = ((q[M::IE] - 0.5 * ke) - P) * iG;
}

// Fast reciprocal square root: MUFU.RSQ64H seed + two Newton steps.
__device__ __forceinline__ double rsqrt_fast(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double h = 0.5 * x;
    double e = fma(-h * y, y, 0.5);
    y = fma(y, e, y);
    e = fma(-h * y, y, 0.5);
    return fma(y, e, y);
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
// alpha_k ~ d_k / t_k with t_k = (beta_k + eps)^2; multiplying every alpha_k by
// t0 t1 t2 gives alpha_k ~ d_k * prod_{j != k} t_j, and the candidate polynomials
// are kept scaled by 6, so each side costs one reciprocal.
__device__ __forceinline__ void weno5(double a, double b, double c, double d, double e,
                                      double eps, double& vm, double& vp) {
    constexpr double k1312 = 13.0 / 12.0;
    const double s0 = fma(-2.0, b, a + c);
    const double r0 = fma(-4.0, b, fma(3.0, c, a));
    const double s1 = fma(-2.0, c, b + d);
    const double r1 = b - d;
    const double s2 = fma(-2.0, d, c + e);
    const double r2 = fma(-4.0, d, fma(3.0, c, e));
    const double b0 = fma(k1312 * s0, s0, 0.25 * (r0 * r0));
    const double b1 = fma(k1312 * s1, s1, 0.25 * (r1 * r1));
    const double b2 = fma(k1312 * s2, s2, 0.25 * (r2 * r2));
    double t0 = b0 + eps; t0 *= t0;
    double t1 = b1 + eps; t1 *= t1;
    double t2 = b2 + eps; t2 *= t2;
    const double P0 = t1 * t2, P1 = t0 * t2, P2 = t0 * t1;
    // 6 x candidate values
    const double m0 = fma(11.0, c, fma(-7.0, b, 2.0 * a));
    const double m1 = fma(2.0, d, fma(5.0, c, -b));
    const double m2 = fma(5.0, d, fma(2.0, c, -e));
    const double p0 = fma(2.0, c, fma(5.0, b, -a));
    const double p1 = fma(5.0, c, fma(2.0, b, -d));
    const double p2 = fma(2.0, e, fma(-7.0, d, 11.0 * c));
    const double wm0 = 0.1 * P0, wm1 = 0.6 * P1, wm2 = 0.3 * P2;
    const double wp0 = 0.3 * P0, wp1 = 0.6 * P1, wp2 = 0.1 * P2;
    const double Dm = 6.0 * ((wm0 + wm1) + wm2);
    const double Dp = 6.0 * ((wp0 + wp1) + wp2);
    const double Nm = fma(wm2, m2, fma(wm1, m1, wm0 * m0));
    const double Np = fma(wp2, p2, fma(wp1, p1, wp0 * p0));
    vm = Nm * rcp(Dm);
    vp = Np * rcp(Dp);
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
    const double sS = (fma(aL, uL, pR - pL) - aR * uR) * rcp(aL - aR);

    const bool left = sS >= 0.0;
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
    const double EK = fma(GK, pK, PK) + 0.5 * (rK * uu);
    const double dK = sK - uK;
    const double dS = sK - sS;
    const double rr = rcp(dK * dS);          // one reciprocal for xi and p_K/(s_K-u_K)
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
    const double inner = fma(sS - uK, fma(rK, sS, pK * (dS * rr)), EK);
    F[M::IE] = fma(sstar, fma(xi, inner, -EK), uK * (EK + pK));
    uf = ufv;
}

}  // namespace mfc
