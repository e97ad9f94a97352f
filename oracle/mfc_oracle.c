/*
 * mfc_oracle.c -- TEST INFRASTRUCTURE ONLY (see mfc_oracle.h).
 *
 * A plain, slow, obviously-correct CPU implementation of one RHS evaluation
 * and one SSP-RK3 step of the Allaire 5-equation model (arXiv 2409.10729,
 * PAPER.md §II, lines 54-84), written step by step in the order of
 * DESIGN.md §3 "Oracle algorithm" (= SURVEY.md §8(c) S0-S4).  Nothing is
 * blocked, fused or reordered beyond what those steps state.  Compiled with
 * -O2 -ffp-contract=off so every a*b+c rounds twice, as written.
 *
 * Pins (tests/test_oracle_*.py): EOS closed forms, WENO5 exactness on
 * quadratics and order of accuracy, HLLC consistency / upwinding / contact
 * and an independent textbook HLLC, exact Riemann solutions (Toro ch. 4;
 * Sod and C1 convergence and plateaus), uniform-state and p-u equilibrium
 * preservation, discrete conservation, RK3 amplification factor, the
 * reflective / extrapolation ghost maps (mirror and constant-extension
 * identities), the non-uniform-grid WENO5 (quadratic / quartic exactness,
 * smoothness-indicator closed forms, fifth order on a tanh grid) and the
 * admissibility count.
 */
#include "mfc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ layout */

int32_t orc_num_eq(int32_t N, int32_t d) { return 2 * N + d + 1; } /* SURVEY §8 notation */

void orc_padded_dims(const orc_problem* P, int64_t out[3]) {
    for (int k = 0; k < 3; ++k) out[k] = (k < P->d) ? (int64_t)P->n[k] + 2 * ORC_G : 1;
}

int64_t orc_padded_cells(const orc_problem* P) {
    int64_t pd[3];
    orc_padded_dims(P, pd);
    return pd[0] * pd[1] * pd[2];
}

/* Linear index of padded cell (i,j,k) (padded coordinates). */
static inline int64_t cell_index(const int64_t pd[3], int64_t i, int64_t j, int64_t k) {
    return (k * pd[1] + j) * pd[0] + i;
}

/* ----------------------------------------------------------------- S0, S2 */

/* S0 (AMB-3): ρE = Γp + Π + ½ρu·u with Γ_i = 1/(γ_i−1),
 * Π_i = γ_i π∞,i/(γ_i−1); the coefficients 1/(γ−1) and γπ∞/(γ−1) of P:66. */
void orc_constants(const orc_problem* P, double* Gam, double* Pi) {
    for (int i = 0; i < P->N; ++i) {
        Gam[i] = 1.0 / (P->gamma[i] - 1.0);
        Pi[i] = (P->gamma[i] * P->pi_inf[i]) / (P->gamma[i] - 1.0);
    }
}

/* S2 cons -> prim, in exactly this order (AMB-18):
 *   ρ = ((α1ρ1 + α2ρ2) + …);  u_k = (ρu_k)/ρ;  KE = ½·Σ_k (ρu_k)·u_k;
 *   Γ = Σ α_iΓ_i;  Π = Σ α_iΠ_i;  p = ((ρE − KE) − Π)/Γ. */
void orc_cons_to_prim_cell(const orc_problem* P, const double* Gam, const double* Pi,
                           const double* q, double* v) {
    const int N = P->N, d = P->d;
    const int im = N, iE = N + d, ia = N + d + 1;
    double rho = q[0];
    for (int i = 1; i < N; ++i) rho = rho + q[i];
    double ke = 0.0;
    for (int k = 0; k < d; ++k) {
        const double u = q[im + k] / rho;
        v[im + k] = u;
        ke = ke + q[im + k] * u;
    }
    ke = 0.5 * ke;
    double G = q[ia] * Gam[0];
    double PI = q[ia] * Pi[0];
    for (int i = 1; i < N; ++i) {
        G = G + q[ia + i] * Gam[i];
        PI = PI + q[ia + i] * Pi[i];
    }
    for (int i = 0; i < N; ++i) {
        v[i] = q[i];
        v[ia + i] = q[ia + i];
    }
    v[iE] = ((q[iE] - ke) - PI) / G;
}

/* Inverse of S2 (used to build inputs and by the EOS pins):
 *   ρ = Σ α_iρ_i;  ρu_k = ρ·u_k;  KE = ½·Σ_k (ρu_k)·u_k;  ρE = (Γ·p + Π) + KE. */
void orc_prim_to_cons_cell(const orc_problem* P, const double* Gam, const double* Pi,
                           const double* v, double* q) {
    const int N = P->N, d = P->d;
    const int im = N, iE = N + d, ia = N + d + 1;
    double rho = v[0];
    for (int i = 1; i < N; ++i) rho = rho + v[i];
    double ke = 0.0;
    for (int k = 0; k < d; ++k) {
        const double m = rho * v[im + k];
        q[im + k] = m;
        ke = ke + m * v[im + k];
    }
    ke = 0.5 * ke;
    double G = v[ia] * Gam[0];
    double PI = v[ia] * Pi[0];
    for (int i = 1; i < N; ++i) {
        G = G + v[ia + i] * Gam[i];
        PI = PI + v[ia + i] * Pi[i];
    }
    for (int i = 0; i < N; ++i) {
        q[i] = v[i];
        q[ia + i] = v[ia + i];
    }
    q[iE] = (G * v[iE] + PI) + ke;
}

void orc_cons_to_prim(const orc_problem* P, int64_t ncells, const double* q, double* v) {
    double Gam[ORC_MAXF], Pi[ORC_MAXF];
    orc_constants(P, Gam, Pi);
    const int E = orc_num_eq(P->N, P->d);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ncells; ++c) {
        double qc[ORC_MAXE], vc[ORC_MAXE];
        for (int e = 0; e < E; ++e) qc[e] = q[e * ncells + c];
        orc_cons_to_prim_cell(P, Gam, Pi, qc, vc);
        for (int e = 0; e < E; ++e) v[e * ncells + c] = vc[e];
    }
}

void orc_prim_to_cons(const orc_problem* P, int64_t ncells, const double* v, double* q) {
    double Gam[ORC_MAXF], Pi[ORC_MAXF];
    orc_constants(P, Gam, Pi);
    const int E = orc_num_eq(P->N, P->d);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ncells; ++c) {
        double qc[ORC_MAXE], vc[ORC_MAXE];
        for (int e = 0; e < E; ++e) vc[e] = v[e * ncells + c];
        orc_prim_to_cons_cell(P, Gam, Pi, vc, qc);
        for (int e = 0; e < E; ++e) q[e * ncells + c] = qc[e];
    }
}

/* --------------------------------------------------------------- S3 WENO5 */

/* Jiang–Shu smoothness indicators of the three 3-cell candidate stencils
 * (P:84 cites Shu [15]):
 *   β0 = 13/12(a−2b+c)² + ¼(a−4b+3c)²
 *   β1 = 13/12(b−2c+d)² + ¼(b−d)²
 *   β2 = 13/12(c−2d+e)² + ¼(3c−4d+e)² */
static void weno5_beta(double a, double b, double c, double d, double e, double beta[3]) {
    double t1, t2;
    t1 = (a - 2.0 * b) + c;
    t2 = (a - 4.0 * b) + 3.0 * c;
    beta[0] = (13.0 / 12.0) * (t1 * t1) + 0.25 * (t2 * t2);
    t1 = (b - 2.0 * c) + d;
    t2 = b - d;
    beta[1] = (13.0 / 12.0) * (t1 * t1) + 0.25 * (t2 * t2);
    t1 = (c - 2.0 * d) + e;
    t2 = (3.0 * c - 4.0 * d) + e;
    beta[2] = (13.0 / 12.0) * (t1 * t1) + 0.25 * (t2 * t2);
}

/* α_k = d_k/(β_k+ε)², ω_k = α_k/Σα, value = Σ ω_k p_k. */
static double weno5_combine(const double beta[3], const double dk[3], const double p[3],
                            double eps, double* weights) {
    double alpha[3];
    for (int k = 0; k < 3; ++k) {
        const double s = beta[k] + eps;
        alpha[k] = dk[k] / (s * s);
    }
    const double sum = (alpha[0] + alpha[1]) + alpha[2];
    double w[3];
    for (int k = 0; k < 3; ++k) w[k] = alpha[k] / sum;
    if (weights) {
        for (int k = 0; k < 3; ++k) weights[k] = w[k];
    }
    return (w[0] * p[0] + w[1] * p[1]) + w[2] * p[2];
}

/* WENO5-M (SURVEY §8(f) F2 "mapped WENO-M"; Henrick, Aslam & Powers 2005, eq. (8)):
 * the Jiang-Shu weights ω_k = α_k/Σα (as above) are mapped by
 *   g_k(ω) = ω (d_k + d_k² − 3 d_k ω + ω²) / (d_k² + ω (1 − 2 d_k))
 * and renormalised, ω*_k = g_k(ω_k) / Σ_j g_j(ω_j); value = Σ ω*_k p_k. */
static double weno5m_combine(const double beta[3], const double dk[3], const double p[3],
                             double eps, double* weights) {
    double alpha[3];
    for (int k = 0; k < 3; ++k) {
        const double s = beta[k] + eps;
        alpha[k] = dk[k] / (s * s);
    }
    const double sum = (alpha[0] + alpha[1]) + alpha[2];
    double g[3];
    for (int k = 0; k < 3; ++k) {
        const double w = alpha[k] / sum;
        const double num = w * (((dk[k] + dk[k] * dk[k]) - 3.0 * dk[k] * w) + w * w);
        const double den = dk[k] * dk[k] + w * (1.0 - 2.0 * dk[k]);
        g[k] = num / den;
    }
    const double gsum = (g[0] + g[1]) + g[2];
    double wm[3];
    for (int k = 0; k < 3; ++k) wm[k] = g[k] / gsum;
    if (weights) {
        for (int k = 0; k < 3; ++k) weights[k] = wm[k];
    }
    return (wm[0] * p[0] + wm[1] * p[1]) + wm[2] * p[2];
}

/* v⁻_{m+½} from cell m's stencil a..e = v_{m−2..m+2}; linear weights
 * (0.1, 0.6, 0.3); p0 = (2a−7b+11c)/6, p1 = (−b+5c+2d)/6, p2 = (2c+5d−e)/6. */
double orc_weno5_minus(double a, double b, double c, double d, double e, double eps,
                       double* weights) {
    double beta[3];
    weno5_beta(a, b, c, d, e, beta);
    const double dk[3] = {0.1, 0.6, 0.3};
    double p[3];
    p[0] = ((2.0 * a - 7.0 * b) + 11.0 * c) / 6.0;
    p[1] = ((-b + 5.0 * c) + 2.0 * d) / 6.0;
    p[2] = ((2.0 * c + 5.0 * d) - e) / 6.0;
    return weno5_combine(beta, dk, p, eps, weights);
}

/* Mirror image: v⁺_{m−½}, same β, p0 = (−a+5b+2c)/6, p1 = (2b+5c−d)/6,
 * p2 = (11c−7d+2e)/6, linear weights (0.3, 0.6, 0.1). */
double orc_weno5_plus(double a, double b, double c, double d, double e, double eps,
                      double* weights) {
    double beta[3];
    weno5_beta(a, b, c, d, e, beta);
    const double dk[3] = {0.3, 0.6, 0.1};
    double p[3];
    p[0] = ((-a + 5.0 * b) + 2.0 * c) / 6.0;
    p[1] = ((2.0 * b + 5.0 * c) - d) / 6.0;
    p[2] = ((11.0 * c - 7.0 * d) + 2.0 * e) / 6.0;
    return weno5_combine(beta, dk, p, eps, weights);
}

/* WENO5-M face states: the same candidates and β as orc_weno5_minus / _plus. */
double orc_weno5m_minus(double a, double b, double c, double d, double e, double eps,
                        double* weights) {
    double beta[3];
    weno5_beta(a, b, c, d, e, beta);
    const double dk[3] = {0.1, 0.6, 0.3};
    double p[3];
    p[0] = ((2.0 * a - 7.0 * b) + 11.0 * c) / 6.0;
    p[1] = ((-b + 5.0 * c) + 2.0 * d) / 6.0;
    p[2] = ((2.0 * c + 5.0 * d) - e) / 6.0;
    return weno5m_combine(beta, dk, p, eps, weights);
}

double orc_weno5m_plus(double a, double b, double c, double d, double e, double eps,
                       double* weights) {
    double beta[3];
    weno5_beta(a, b, c, d, e, beta);
    const double dk[3] = {0.3, 0.6, 0.1};
    double p[3];
    p[0] = ((-a + 5.0 * b) + 2.0 * c) / 6.0;
    p[1] = ((2.0 * b + 5.0 * c) - d) / 6.0;
    p[2] = ((11.0 * c - 7.0 * d) + 2.0 * e) / 6.0;
    return weno5m_combine(beta, dk, p, eps, weights);
}

/* WENO3-JS: candidates from the 2-cell stencils {m-1,m} and {m,m+1},
 *   v^-_{m+1/2}: p0 = (-a+3b)/2, p1 = (b+c)/2, d = (1/3, 2/3)
 *   v^+_{m-1/2}: p0 = (a+b)/2,   p1 = (3b-c)/2, d = (2/3, 1/3)
 *   beta0 = (b-a)^2, beta1 = (c-b)^2, alpha_k = d_k/(beta_k+eps)^2. */
static double weno3_combine(const double beta[2], const double dk[2], const double p[2],
                            double eps, double* weights) {
    double alpha[2];
    for (int k = 0; k < 2; ++k) {
        const double s = beta[k] + eps;
        alpha[k] = dk[k] / (s * s);
    }
    const double sum = alpha[0] + alpha[1];
    const double w0 = alpha[0] / sum, w1 = alpha[1] / sum;
    if (weights) {
        weights[0] = w0;
        weights[1] = w1;
    }
    return w0 * p[0] + w1 * p[1];
}

double orc_weno3_minus(double a, double b, double c, double eps, double* weights) {
    const double beta[2] = {(b - a) * (b - a), (c - b) * (c - b)};
    const double dk[2] = {1.0 / 3.0, 2.0 / 3.0};
    const double p[2] = {(-a + 3.0 * b) / 2.0, (b + c) / 2.0};
    return weno3_combine(beta, dk, p, eps, weights);
}

double orc_weno3_plus(double a, double b, double c, double eps, double* weights) {
    const double beta[2] = {(b - a) * (b - a), (c - b) * (c - b)};
    const double dk[2] = {2.0 / 3.0, 1.0 / 3.0};
    const double p[2] = {(a + b) / 2.0, (3.0 * b - c) / 2.0};
    return weno3_combine(beta, dk, p, eps, weights);
}

/* ------------------------------------------- S3 WENO5, non-uniform grid (F4) */

/* t^k by repeated multiplication. */
static double ipow(double t, int k) {
    double r = 1.0;
    for (int i = 0; i < k; ++i) r = r * t;
    return r;
}

/* Average of t^i over the interval [tl, tr]: (tr^(i+1) - tl^(i+1)) / ((i+1)(tr - tl)). */
static double avg_pow(double tl, double tr, int i) {
    return (ipow(tr, i + 1) - ipow(tl, i + 1)) / ((double)(i + 1) * (tr - tl));
}

/* Solve A X = B in place (A n x n row-major, B n x nrhs row-major) by Gaussian
 * elimination with partial pivoting; X overwrites B. */
static void gauss_solve(int n, double* A, double* B, int nrhs) {
    for (int k = 0; k < n; ++k) {
        int piv = k;
        for (int r = k + 1; r < n; ++r)
            if (fabs(A[r * n + k]) > fabs(A[piv * n + k])) piv = r;
        if (piv != k) {
            for (int c = 0; c < n; ++c) {
                const double t = A[k * n + c];
                A[k * n + c] = A[piv * n + c];
                A[piv * n + c] = t;
            }
            for (int c = 0; c < nrhs; ++c) {
                const double t = B[k * nrhs + c];
                B[k * nrhs + c] = B[piv * nrhs + c];
                B[piv * nrhs + c] = t;
            }
        }
        for (int r = k + 1; r < n; ++r) {
            const double f = A[r * n + k] / A[k * n + k];
            for (int c = k; c < n; ++c) A[r * n + c] = A[r * n + c] - f * A[k * n + c];
            for (int c = 0; c < nrhs; ++c) B[r * nrhs + c] = B[r * nrhs + c] - f * B[k * nrhs + c];
        }
    }
    for (int k = n - 1; k >= 0; --k) {
        for (int c = 0; c < nrhs; ++c) {
            double acc = B[k * nrhs + c];
            for (int j = k + 1; j < n; ++j) acc = acc - A[k * n + j] * B[j * nrhs + c];
            B[k * nrhs + c] = acc / A[k * n + k];
        }
    }
}

/* DESIGN.md AMB-27 ("local mesh refinement ... hyperbolic tangent
 * function"): the WENO5-JS ingredients of cell m on a non-uniform grid, from their
 * definitions in the local coordinate t = (x - x_m)/Δ_m (see mfc_oracle.h). */
int32_t orc_nu_cell_coeffs(const double* xb6, orc_nu_cell* out) {
    const double w = xb6[3] - xb6[2];                 /* Δ_m */
    const double xm = 0.5 * (xb6[2] + xb6[3]);        /* centre of cell m */
    double t[6];                                      /* boundaries in local coordinates */
    for (int j = 0; j < 6; ++j) t[j] = (xb6[j] - xm) / w;
    out->w = w;
    /* candidates: (a, b, c) = M[k] v, M[k] = A_k^{-1}, A_k[j][i] = avg_{cell m-2+k+j} t^i */
    for (int k = 0; k < 3; ++k) {
        double A[9], B[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
        for (int j = 0; j < 3; ++j)
            for (int i = 0; i < 3; ++i) A[j * 3 + i] = avg_pow(t[k + j], t[k + j + 1], i);
        gauss_solve(3, A, B, 3);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) out->M[k][i][j] = B[i * 3 + j];
    }
    /* ideal weights at t_f = +1/2 (v-) and -1/2 (v+): the degree-4 reconstruction
     * weights R (A5^T R = (1, t_f, .., t_f^4)) against the candidates' weights
     * r^(k)_j = sum_i t_f^i M[k][i][j] on their outermost cells */
    for (int side = 0; side < 2; ++side) {
        const double tf = side == 0 ? 0.5 : -0.5;
        double A5t[25], R[5];
        for (int j = 0; j < 5; ++j)
            for (int i = 0; i < 5; ++i) A5t[i * 5 + j] = avg_pow(t[j], t[j + 1], i);
        for (int i = 0; i < 5; ++i) R[i] = ipow(tf, i);
        gauss_solve(5, A5t, R, 1);
        double r0 = 0.0, r2 = 0.0;                    /* r^(0)_{m-2}, r^(2)_{m+2} */
        for (int i = 0; i < 3; ++i) {
            r0 = r0 + ipow(tf, i) * out->M[0][i][0];
            r2 = r2 + ipow(tf, i) * out->M[2][i][2];
        }
        double* d = side == 0 ? out->dm : out->dp;
        d[0] = R[0] / r0;
        d[2] = R[4] / r2;
        d[1] = (1.0 - d[0]) - d[2];
    }
    for (int k = 0; k < 3; ++k)
        if (!(out->dm[k] > 0.0) || !(out->dp[k] > 0.0)) return -1;
    return 0;
}

/* β_k = b² + (13/3)c² and q_k(t_f) of the three candidates of cell m. */
static void weno5nu_parts(const orc_nu_cell* C, const double v[5], double tf, double beta[3],
                          double p[3]) {
    for (int k = 0; k < 3; ++k) {
        double abc[3];
        for (int i = 0; i < 3; ++i)
            abc[i] = (C->M[k][i][0] * v[k] + C->M[k][i][1] * v[k + 1]) + C->M[k][i][2] * v[k + 2];
        beta[k] = abc[1] * abc[1] + (13.0 / 3.0) * (abc[2] * abc[2]);
        p[k] = (abc[0] + abc[1] * tf) + abc[2] * (tf * tf);
    }
}

double orc_weno5nu_minus(const orc_nu_cell* C, double a, double b, double c, double d, double e,
                         double eps, double* weights) {
    const double v[5] = {a, b, c, d, e};
    double beta[3], p[3];
    weno5nu_parts(C, v, 0.5, beta, p);
    return weno5_combine(beta, C->dm, p, eps, weights);
}

double orc_weno5nu_plus(const orc_nu_cell* C, double a, double b, double c, double d, double e,
                        double eps, double* weights) {
    const double v[5] = {a, b, c, d, e};
    double beta[3], p[3];
    weno5nu_parts(C, v, -0.5, beta, p);
    return weno5_combine(beta, C->dp, p, eps, weights);
}

/* Coefficients of cells -1 .. n of axis dir (index m+1), or NULL on a uniform axis. */
static orc_nu_cell* nu_axis(const orc_problem* P, int dir) {
    if (!P->xb[dir]) return NULL;
    const int64_t n = P->n[dir];
    orc_nu_cell* C = (orc_nu_cell*)malloc(sizeof(orc_nu_cell) * (size_t)(n + 2));
    for (int64_t m = -1; m <= n; ++m) orc_nu_cell_coeffs(P->xb[dir] + (m + 1), C + (m + 1));
    return C;
}

/* ---------------------------------------------------------------- S3 HLLC */

typedef struct {
    double rho, G, PI, u, p, rhoE, c;
} side_state;

/* Per side K: ρ_K, Γ_K, Π_K from the reconstructed α and α_iρ_i;
 * ρE_K = (Γ_K p_K + Π_K) + ½ρ_K(u·u);  c_K = sqrt(((Γ_K+1)p_K + Π_K)/(ρ_KΓ_K))
 * (AMB-10: the sound speed of the single mixture EOS of P:66). */
static side_state hllc_side(const orc_problem* P, const double* Gam, const double* Pi,
                            int dir, const double* v) {
    const int N = P->N, d = P->d;
    const int im = N, iE = N + d, ia = N + d + 1;
    side_state s;
    s.rho = v[0];
    for (int i = 1; i < N; ++i) s.rho = s.rho + v[i];
    s.G = v[ia] * Gam[0];
    s.PI = v[ia] * Pi[0];
    for (int i = 1; i < N; ++i) {
        s.G = s.G + v[ia + i] * Gam[i];
        s.PI = s.PI + v[ia + i] * Pi[i];
    }
    double uu = 0.0;
    for (int k = 0; k < d; ++k) uu = uu + v[im + k] * v[im + k];
    s.u = v[im + dir];
    s.p = v[iE];
    s.rhoE = (s.G * s.p + s.PI) + 0.5 * (s.rho * uu);
    s.c = sqrt(((s.G + 1.0) * s.p + s.PI) / (s.rho * s.G));
    return s;
}

/* HLLC (Toro [14] ch. 10) in compact branch form (DESIGN.md §3 S3):
 *   s_L = min(u_L−c_L, u_R−c_R);  s_R = max(u_L+c_L, u_R+c_R)   (AMB-9)
 *   s_S = (p_R − p_L + ρ_Lu_L(s_L−u_L) − ρ_Ru_R(s_R−u_R)) / (ρ_L(s_L−u_L) − ρ_R(s_R−u_R))
 *   s_S ≥ 0: K = L, s* = min(0, s_L);  else K = R, s* = max(0, s_R)
 *   ξ = (s_K−u_K)/(s_K−s_S);  u^f = u_K + s*(ξ−1)
 *   F[α_iρ_i] = (α_iρ_i)_K u^f
 *   F[ρu_n]   = ρ_Ku_K² + p_K + s*(ρ_Kξs_S − ρ_Ku_K)
 *   F[ρu_t]   = ρ_Ku_{t,K} u^f
 *   F[ρE]     = u_K(ρE_K+p_K) + s*(ξ(ρE_K + (s_S−u_K)(ρ_Ks_S + p_K/(s_K−u_K))) − ρE_K)
 *   F[α_i]    = α_{i,K} u^f */
void orc_hllc(const orc_problem* P, const double* Gam, const double* Pi, int32_t dir,
              const double* vL, const double* vR, double* F, double* uf) {
    const int N = P->N, d = P->d;
    const int im = N, iE = N + d, ia = N + d + 1;
    const side_state L = hllc_side(P, Gam, Pi, dir, vL);
    const side_state R = hllc_side(P, Gam, Pi, dir, vR);
    const double sL = fmin(L.u - L.c, R.u - R.c);
    const double sR = fmax(L.u + L.c, R.u + R.c);
    const double num = ((R.p - L.p) + (L.rho * L.u) * (sL - L.u)) - (R.rho * R.u) * (sR - R.u);
    const double den = L.rho * (sL - L.u) - R.rho * (sR - R.u);
    const double sS = num / den;

    const double* vK;
    side_state K;
    double sK, sstar;
    if (sS >= 0.0) {
        vK = vL;
        K = L;
        sK = sL;
        sstar = fmin(0.0, sL);
    } else {
        vK = vR;
        K = R;
        sK = sR;
        sstar = fmax(0.0, sR);
    }
    const double xi = (sK - K.u) / (sK - sS);
    const double ufv = K.u + sstar * (xi - 1.0);

    for (int i = 0; i < N; ++i) F[i] = vK[i] * ufv;
    for (int k = 0; k < d; ++k) {
        if (k == dir) {
            F[im + k] = ((K.rho * K.u) * K.u + K.p) + sstar * ((K.rho * xi) * sS - K.rho * K.u);
        } else {
            F[im + k] = (K.rho * vK[im + k]) * ufv;
        }
    }
    const double inner = K.rhoE + (sS - K.u) * (K.rho * sS + K.p / (sK - K.u));
    F[iE] = K.u * (K.rhoE + K.p) + sstar * (xi * inner - K.rhoE);
    for (int i = 0; i < N; ++i) F[ia + i] = vK[ia + i] * ufv;
    *uf = ufv;
}

/* Face m+½ from the primitive window w = cells m−2..m+3 ([6][E], AoS):
 * v_L = v⁻ from cell m (cells m−2..m+2), v_R = v⁺ from cell m+1 (m−1..m+3);
 * WENO3 uses the inner cells m−1..m+1 and m..m+2.  Cm: NULL on a uniform axis, else
 * the non-uniform coefficients of cells m, m+1. */
static void face_flux(const orc_problem* P, const double* Gam, const double* Pi, int dir,
                      const double* w, const orc_nu_cell* Cm, double* F, double* uf) {
    const int E = orc_num_eq(P->N, P->d);
    double vL[ORC_MAXE], vR[ORC_MAXE];
    for (int e = 0; e < E; ++e) {
        if (Cm) {   /* non-uniform axis: cell m's v-, cell m+1's v+ (Cm[0], Cm[1]) */
            vL[e] = orc_weno5nu_minus(Cm, w[0 * E + e], w[1 * E + e], w[2 * E + e], w[3 * E + e],
                                      w[4 * E + e], P->eps, NULL);
            vR[e] = orc_weno5nu_plus(Cm + 1, w[1 * E + e], w[2 * E + e], w[3 * E + e],
                                     w[4 * E + e], w[5 * E + e], P->eps, NULL);
        } else if (P->weno_order == 3) {
            vL[e] = orc_weno3_minus(w[1 * E + e], w[2 * E + e], w[3 * E + e], P->eps, NULL);
            vR[e] = orc_weno3_plus(w[2 * E + e], w[3 * E + e], w[4 * E + e], P->eps, NULL);
        } else if (P->weno_mapped) {
            vL[e] = orc_weno5m_minus(w[0 * E + e], w[1 * E + e], w[2 * E + e], w[3 * E + e],
                                     w[4 * E + e], P->eps, NULL);
            vR[e] = orc_weno5m_plus(w[1 * E + e], w[2 * E + e], w[3 * E + e], w[4 * E + e],
                                    w[5 * E + e], P->eps, NULL);
        } else {
            vL[e] = orc_weno5_minus(w[0 * E + e], w[1 * E + e], w[2 * E + e], w[3 * E + e],
                                    w[4 * E + e], P->eps, NULL);
            vR[e] = orc_weno5_plus(w[1 * E + e], w[2 * E + e], w[3 * E + e], w[4 * E + e],
                                   w[5 * E + e], P->eps, NULL);
        }
    }
    orc_hllc(P, Gam, Pi, dir, vL, vR, F, uf);
}

/* ------------------------------------------------------------ S1 ghosts */

/* Ghost layer j (0..2) next to a face:
 *   periodic:      ghost −1−j ← interior n−1−j;   ghost n+j ← interior j
 *   extrapolation: every ghost ← adjacent interior cell
 *   reflective:    ghost −1−j ← interior j; ghost n+j ← interior n−1−j; normal momentum negated
 *   external (0):  untouched (filled by the caller, "neighbour rank"). */
void orc_fill_ghosts(const orc_problem* P, double* q) {
    const int N = P->N, d = P->d, E = orc_num_eq(N, d);
    int64_t pd[3];
    orc_padded_dims(P, pd);
    const int64_t ncell = pd[0] * pd[1] * pd[2];
    const int64_t o[3] = {ORC_G, d >= 2 ? ORC_G : 0, d >= 3 ? ORC_G : 0};
    for (int dir = 0; dir < d; ++dir) {
        const int64_t n = P->n[dir];
        const int t1 = (dir + 1) % 3, t2 = (dir + 2) % 3;
        for (int side = 0; side < 2; ++side) {
            const int bc = P->bc[2 * dir + side];
            if (bc == ORC_BC_EXTERNAL) continue;
            for (int64_t b = 0; b < P->n[t2]; ++b) {
                for (int64_t a = 0; a < P->n[t1]; ++a) {
                    for (int j = 0; j < ORC_G; ++j) {
                        int64_t ghost, src;
                        if (side == 0) {
                            ghost = -1 - j;
                            if (bc == ORC_BC_PERIODIC) src = n - 1 - j;
                            else if (bc == ORC_BC_REFLECTIVE) src = j;
                            else src = 0;
                        } else {
                            ghost = n + j;
                            if (bc == ORC_BC_PERIODIC) src = j;
                            else if (bc == ORC_BC_REFLECTIVE) src = n - 1 - j;
                            else src = n - 1;
                        }
                        int64_t gi[3], si[3];
                        gi[dir] = o[dir] + ghost;
                        si[dir] = o[dir] + src;
                        gi[t1] = si[t1] = o[t1] + a;
                        gi[t2] = si[t2] = o[t2] + b;
                        const int64_t gc = cell_index(pd, gi[0], gi[1], gi[2]);
                        const int64_t sc = cell_index(pd, si[0], si[1], si[2]);
                        for (int e = 0; e < E; ++e) {
                            double val = q[e * ncell + sc];
                            if (bc == ORC_BC_REFLECTIVE && e == N + dir) val = -val;
                            q[e * ncell + gc] = val;
                        }
                    }
                }
            }
        }
    }
}

/* --------------------------------------------------------- S3 full RHS */

/* One RHS evaluation (eq. (1) integrated over cell m):
 *   rhs_e += (F_{e,m−½} − F_{e,m+½})·(1/Δ)                 for every e
 *   rhs_{α_i} += α_{i,m}·((u^f_{m+½} − u^f_{m−½})·(1/Δ))   (AMB-5/6)
 * for the active directions x, y, z in that order. */
void orc_rhs(const orc_problem* P, double* q, double* rhs) {
    const int N = P->N, d = P->d, E = orc_num_eq(N, d);
    const int ia = N + d + 1;
    double Gam[ORC_MAXF], Pi[ORC_MAXF];
    orc_constants(P, Gam, Pi);
    int64_t pd[3];
    orc_padded_dims(P, pd);
    const int64_t ncell = pd[0] * pd[1] * pd[2];
    const int64_t o[3] = {ORC_G, d >= 2 ? ORC_G : 0, d >= 3 ? ORC_G : 0};

    orc_fill_ghosts(P, q);
    memset(rhs, 0, sizeof(double) * (size_t)(E * ncell));

    for (int dir = 0; dir < d; ++dir) {
        const int64_t n = P->n[dir];
        const int t1 = (dir + 1) % 3, t2 = (dir + 2) % 3;
        const int64_t n1 = P->n[t1], n2 = P->n[t2];
        const double invd = 1.0 / P->dx[dir];
        orc_nu_cell* NU = nu_axis(P, dir);        /* cells -1 .. n at NU[m+1] */
#pragma omp parallel
        {
            double* v = (double*)malloc(sizeof(double) * (size_t)((n + 2 * ORC_G) * E));
            double* F = (double*)malloc(sizeof(double) * (size_t)((n + 1) * E));
            double* uf = (double*)malloc(sizeof(double) * (size_t)(n + 1));
            int64_t* cidx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 2 * ORC_G));
#pragma omp for collapse(2) schedule(static)
            for (int64_t b = 0; b < n2; ++b) {
                for (int64_t a = 0; a < n1; ++a) {
                    /* gather the line's cells (with ghosts) and convert to primitives */
                    for (int64_t m = 0; m < n + 2 * ORC_G; ++m) {
                        int64_t ii[3];
                        ii[dir] = m;
                        ii[t1] = o[t1] + a;
                        ii[t2] = o[t2] + b;
                        cidx[m] = cell_index(pd, ii[0], ii[1], ii[2]);
                        double qc[ORC_MAXE];
                        for (int e = 0; e < E; ++e) qc[e] = q[e * ncell + cidx[m]];
                        orc_cons_to_prim_cell(P, Gam, Pi, qc, v + m * E);
                    }
                    /* faces m+½ for m = −1..n−1 -> F[m+1]; window starts at cell m−2 */
                    for (int64_t m = -1; m < n; ++m) {
                        const double* w = v + (m - 2 + ORC_G) * E;
                        face_flux(P, Gam, Pi, dir, w, NU ? NU + (m + 1) : NULL, F + (m + 1) * E,
                                  uf + (m + 1));
                    }
                    for (int64_t m = 0; m < n; ++m) {
                        const int64_t c = cidx[m + ORC_G];
                        /* 1/Δ_m: uniform spacing, or the width of cell m */
                        const double id = NU ? 1.0 / NU[m + 1].w : invd;
                        for (int e = 0; e < E; ++e)
                            rhs[e * ncell + c] =
                                rhs[e * ncell + c] + (F[m * E + e] - F[(m + 1) * E + e]) * id;
                        for (int i = 0; i < N; ++i)
                            rhs[(ia + i) * ncell + c] =
                                rhs[(ia + i) * ncell + c] +
                                q[(ia + i) * ncell + c] * ((uf[m + 1] - uf[m]) * id);
                    }
                }
            }
            free(v);
            free(F);
            free(uf);
            free(cidx);
        }
        free(NU);
    }
}

void orc_rhs_cells(const orc_problem* P, const double* q, int64_t ncells, const int64_t* cells,
                   double* out) {
    const int N = P->N, d = P->d, E = orc_num_eq(N, d);
    const int ia = N + d + 1;
    double Gam[ORC_MAXF], Pi[ORC_MAXF];
    orc_constants(P, Gam, Pi);
    int64_t pd[3];
    orc_padded_dims(P, pd);
    const int64_t ncell = pd[0] * pd[1] * pd[2];
    const int64_t o[3] = {ORC_G, d >= 2 ? ORC_G : 0, d >= 3 ? ORC_G : 0};
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ncells; ++c) {
        double acc[ORC_MAXE];
        for (int e = 0; e < E; ++e) acc[e] = 0.0;
        const int64_t ci = cell_index(pd, o[0] + cells[3 * c], o[1] + cells[3 * c + 1],
                                      o[2] + cells[3 * c + 2]);
        for (int dir = 0; dir < d; ++dir) {
            const int64_t mc = cells[3 * c + dir];      /* the cell's index along dir */
            /* non-uniform axis: coefficients of cells m-1, m, m+1 from the boundaries */
            orc_nu_cell NU3[3];
            if (P->xb[dir])
                for (int s = 0; s < 3; ++s) orc_nu_cell_coeffs(P->xb[dir] + (mc + s), NU3 + s);
            const double invd = P->xb[dir] ? 1.0 / NU3[1].w : 1.0 / P->dx[dir];
            /* primitive window: cells m−3..m+3 along dir */
            double w[7 * ORC_MAXE];
            for (int s = -3; s <= 3; ++s) {
                int64_t ii[3] = {o[0] + cells[3 * c], o[1] + cells[3 * c + 1],
                                 o[2] + cells[3 * c + 2]};
                ii[dir] += s;
                const int64_t cc = cell_index(pd, ii[0], ii[1], ii[2]);
                double qc[ORC_MAXE];
                for (int e = 0; e < E; ++e) qc[e] = q[e * ncell + cc];
                orc_cons_to_prim_cell(P, Gam, Pi, qc, w + (s + 3) * E);
            }
            double Fm[ORC_MAXE], Fp[ORC_MAXE], ufm, ufp;
            const orc_nu_cell* nu = P->xb[dir] ? NU3 : NULL;
            face_flux(P, Gam, Pi, dir, w, nu, Fm, &ufm);                      /* face m−½ */
            face_flux(P, Gam, Pi, dir, w + E, nu ? nu + 1 : NULL, Fp, &ufp);  /* face m+½ */
            for (int e = 0; e < E; ++e) acc[e] = acc[e] + (Fm[e] - Fp[e]) * invd;
            for (int i = 0; i < N; ++i)
                acc[ia + i] = acc[ia + i] + q[(ia + i) * ncell + ci] * ((ufp - ufm) * invd);
        }
        for (int e = 0; e < E; ++e) out[c * E + e] = acc[e];
    }
}

/* ------------------------------------------------------------- S4 RK3 */

/* SSP-RK3, Shu–Osher form (BASELINE.json north_star; AMB-11):
 *   q(1) = q^n + dt·L(q^n)
 *   q(2) = 0.75·q^n + 0.25·(q(1) + dt·L(q(1)))
 *   q^{n+1} = (1/3)·q^n + (2/3)·(q(2) + dt·L(q(2))) */
void orc_rk3_combine(int32_t stage, int64_t n, const double* qn, const double* qs,
                     const double* L, double dt, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double t = qs[i] + dt * L[i];
        if (stage == 1) out[i] = t;
        else if (stage == 2) out[i] = 0.75 * qn[i] + 0.25 * t;
        else out[i] = (1.0 / 3.0) * qn[i] + (2.0 / 3.0) * t;
    }
}

void orc_rk3_step(const orc_problem* P, double* q, double dt) {
    const int E = orc_num_eq(P->N, P->d);
    const int64_t n = orc_padded_cells(P) * E;
    double* qn = (double*)malloc(sizeof(double) * (size_t)n);
    double* qs = (double*)malloc(sizeof(double) * (size_t)n);
    double* L = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(qn, q, sizeof(double) * (size_t)n);
    orc_rhs(P, q, L);                       /* L(q^n)   (fills q's ghosts) */
    orc_rk3_combine(1, n, qn, q, L, dt, qs);
    orc_rhs(P, qs, L);                      /* L(q(1)) */
    orc_rk3_combine(2, n, qn, qs, L, dt, qs);
    orc_rhs(P, qs, L);                      /* L(q(2)) */
    orc_rk3_combine(3, n, qn, qs, L, dt, q);
    free(qn);
    free(qs);
    free(L);
}

/* --------------------------------------------------------- diagnostics */

int64_t orc_count_inadmissible(const orc_problem* P, const double* q) {
    const int N = P->N, d = P->d, E = orc_num_eq(N, d);
    const int ia = N + d + 1;
    double Gam[ORC_MAXF], Pi[ORC_MAXF];
    orc_constants(P, Gam, Pi);
    int64_t pd[3];
    orc_padded_dims(P, pd);
    const int64_t ncell = pd[0] * pd[1] * pd[2];
    const int64_t o[3] = {ORC_G, d >= 2 ? ORC_G : 0, d >= 3 ? ORC_G : 0};
    int64_t bad = 0;
#pragma omp parallel for collapse(2) reduction(+ : bad) schedule(static)
    for (int64_t k = 0; k < P->n[2]; ++k) {
        for (int64_t j = 0; j < P->n[1]; ++j) {
            for (int64_t i = 0; i < P->n[0]; ++i) {
                const int64_t c = cell_index(pd, o[0] + i, o[1] + j, o[2] + k);
                double qc[ORC_MAXE], v[ORC_MAXE];
                int finite = 1;
                for (int e = 0; e < E; ++e) {
                    qc[e] = q[e * ncell + c];
                    if (!isfinite(qc[e])) finite = 0;
                }
                if (!finite) {
                    ++bad;
                    continue;
                }
                orc_cons_to_prim_cell(P, Gam, Pi, qc, v);
                double rho = v[0];
                for (int i2 = 1; i2 < N; ++i2) rho = rho + v[i2];
                double G = v[ia] * Gam[0], PI = v[ia] * Pi[0];
                for (int i2 = 1; i2 < N; ++i2) {
                    G = G + v[ia + i2] * Gam[i2];
                    PI = PI + v[ia + i2] * Pi[i2];
                }
                const double c2 = ((G + 1.0) * v[N + d] + PI) / (rho * G);
                if (!(rho > 0.0) || !(c2 > 0.0) || !isfinite(c2)) ++bad;
            }
        }
    }
    return bad;
}

double orc_max_wave_rate(const orc_problem* P, const double* q) {
    const int N = P->N, d = P->d, E = orc_num_eq(N, d);
    const int ia = N + d + 1;
    double Gam[ORC_MAXF], Pi[ORC_MAXF];
    orc_constants(P, Gam, Pi);
    int64_t pd[3];
    orc_padded_dims(P, pd);
    const int64_t ncell = pd[0] * pd[1] * pd[2];
    const int64_t o[3] = {ORC_G, d >= 2 ? ORC_G : 0, d >= 3 ? ORC_G : 0};
    double rate = 0.0;
    for (int64_t k = 0; k < P->n[2]; ++k) {
        for (int64_t j = 0; j < P->n[1]; ++j) {
            for (int64_t i = 0; i < P->n[0]; ++i) {
                const int64_t cc = cell_index(pd, o[0] + i, o[1] + j, o[2] + k);
                double qc[ORC_MAXE], v[ORC_MAXE];
                for (int e = 0; e < E; ++e) qc[e] = q[e * ncell + cc];
                orc_cons_to_prim_cell(P, Gam, Pi, qc, v);
                double rho = v[0];
                for (int i2 = 1; i2 < N; ++i2) rho = rho + v[i2];
                double G = v[ia] * Gam[0], PI = v[ia] * Pi[0];
                for (int i2 = 1; i2 < N; ++i2) {
                    G = G + v[ia + i2] * Gam[i2];
                    PI = PI + v[ia + i2] * Pi[i2];
                }
                const double c = sqrt(((G + 1.0) * v[N + d] + PI) / (rho * G));
                const int64_t ijk[3] = {i, j, k};
                for (int dir = 0; dir < d; ++dir) {
                    /* Δ of this cell: uniform spacing or its own width (F4) */
                    const double h = P->xb[dir] ? P->xb[dir][ijk[dir] + 4] - P->xb[dir][ijk[dir] + 3]
                                                : P->dx[dir];
                    const double r = (fabs(v[N + dir]) + c) / h;
                    if (r > rate) rate = r;
                }
            }
        }
    }
    return rate;
}

void orc_set_num_threads(int32_t n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int32_t orc_num_threads(void) {
#ifdef _OPENMP
    return (int32_t)omp_get_max_threads();
#else
    return 1;
#endif
}
