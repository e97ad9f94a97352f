/*
 * mfc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the right-hand side of the
 * Allaire 5-equation model as described in arXiv 2409.10729 (PAPER.md
 * §II-A, §II-B, lines 54-84) with the readings of DESIGN.md §3 (SURVEY.md
 * §8(c) S0-S4, AMB-1..22).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * constant or helper with the CUDA path (paper_2409_10729_b200/csrc) and
 * never includes include/mfc.h.
 *
 * Arithmetic: IEEE fp64, compiled with -O2 -ffp-contract=off (no FMA), every
 * expression in the order written in DESIGN.md §3.
 *
 * Layout (oracle-private): q[E][P2][P1][P0], x fastest, where
 * P_k = n_k + 6 for an active dimension (3 ghost layers per side) and 1 for an
 * inactive one.  Interior cell (i,j,k) lives at (i+3, j+3, k+3) for active
 * dims, index 0 for inactive dims.
 */
#ifndef MFC_ORACLE_H
#define MFC_ORACLE_H
#include <stdint.h>

#define ORC_G 3                 /* ghost depth: WENO5 needs cells m-3..m+2 (AMB-12) */
#define ORC_MAXF 3              /* maximum number of fluids */
#define ORC_MAXE (2 * ORC_MAXF + 3 + 1)

/* Boundary codes (MFC-style, AMB-13).  0 = ghosts supplied by the caller
 * (used to emulate a neighbouring subdomain, S1 "neighbour rank"). */
#define ORC_BC_EXTERNAL 0
#define ORC_BC_PERIODIC (-1)
#define ORC_BC_REFLECTIVE (-2)
#define ORC_BC_EXTRAPOLATION (-3)

typedef struct {
    int32_t N;                  /* number of fluids, 1..3 (AMB-4) */
    int32_t d;                  /* active dimensions, 1..3 */
    int32_t n[3];               /* interior cells per dim (1 if inactive) */
    double dx[3];               /* uniform spacing per dim (AMB-7) */
    int32_t bc[6];              /* x_lo, x_hi, y_lo, y_hi, z_lo, z_hi */
    double gamma[ORC_MAXF];     /* stiffened-gas gamma_i > 1 */
    double pi_inf[ORC_MAXF];    /* stiffened-gas pi_inf_i >= 0 */
    double eps;                 /* WENO epsilon (AMB-8), default 1e-16 */
    int32_t weno_order;         /* 5 (WENO5-JS, default) or 3 (WENO3-JS) */
    int32_t weno_mapped;        /* 1: WENO5-M weights (Henrick et al. 2005) */
    /* Non-uniform (stretched) grid, SURVEY §8(f) F4 / P:92: NULL = uniform spacing dx[k];
     * else n[k]+7 cell boundaries of axis k, x_{-7/2} .. x_{n+5/2} (interior cell i spans
     * [xb[i+3], xb[i+4]]; the 3 ghost cells per side are part of the input, see
     * oracle.py extend_boundaries).  WENO5-JS only (weno_order 5, not mapped). */
    const double* xb[3];
} orc_problem;

/* WENO5-JS on a non-uniform grid (DESIGN.md AMB-27), per cell m, from the definitions
 * in the local coordinate t = (x - x_m)/Δ_m of cell m (x_m its centre):
 *   candidate k = 0, 1, 2 (stencil cells m-2+k .. m+k): the quadratic q_k(t) = a + b t + c t²
 *     whose AVERAGES over the three stencil cells are the cell values;
 *   v-_{m+1/2} = Σ ω_k q_k(+1/2),  v+_{m-1/2} = Σ ω_k q_k(-1/2);
 *   β_k = Σ_{l=1,2} Δ_m^{2l-1} ∫_cell (d^l q_k/dx^l)² dx = b² + (13/3) c²  (Jiang-Shu);
 *   ideal weights: Σ_k d_k q_k(t_face) = the degree-4 reconstruction from the 5 cell
 *     averages at the same face, read off the coefficients of cells m-2 (only in k=0)
 *     and m+2 (only in k=2), d_1 = 1 - d_0 - d_2;
 *   α_k = d_k/(β_k+ε)², ω_k = α_k/Σα (as in the uniform case). */
typedef struct {
    double M[3][3][3];          /* candidate k: (a, b, c) = M[k] (v_{m-2+k}, v_{m-1+k}, v_{m+k}) */
    double dm[3], dp[3];        /* ideal weights of v-_{m+1/2} and v+_{m-1/2} */
    double w;                   /* Δ_m */
} orc_nu_cell;

#ifdef __cplusplus
extern "C" {
#endif

int32_t orc_num_eq(int32_t N, int32_t d);
int64_t orc_padded_cells(const orc_problem* P);
void orc_padded_dims(const orc_problem* P, int64_t out[3]);

/* S0: Gamma_i = 1/(gamma_i-1), Pi_i = gamma_i*pi_inf_i/(gamma_i-1). */
void orc_constants(const orc_problem* P, double* Gam, double* Pi);

/* S2 per cell: q[E] -> v[E]; v = (a_i r_i, u_k, p, a_i). */
void orc_cons_to_prim_cell(const orc_problem* P, const double* Gam, const double* Pi,
                           const double* q, double* v);
/* Inverse EOS (P:66 with AMB-3): rhoE = (Gamma*p + Pi) + 0.5*rho*(u.u). */
void orc_prim_to_cons_cell(const orc_problem* P, const double* Gam, const double* Pi,
                           const double* v, double* q);
/* Field versions over SoA arrays [E][ncells]. */
void orc_cons_to_prim(const orc_problem* P, int64_t ncells, const double* q, double* v);
void orc_prim_to_cons(const orc_problem* P, int64_t ncells, const double* v, double* q);

/* S3 WENO5-JS (Jiang-Shu, [15] of the paper): from cell values
 * a..e = v_{m-2..m+2}: minus -> v^-_{m+1/2}, plus -> v^+_{m-1/2}.
 * weights[3] (may be NULL) receives the normalised omega_k. */
double orc_weno5_minus(double a, double b, double c, double d, double e, double eps,
                       double* weights);
double orc_weno5_plus(double a, double b, double c, double d, double e, double eps,
                      double* weights);

/* WENO3-JS ("third or fifth-order accurate WENO", Shu [15]) from a..c =
 * v_{m-1..m+1}: minus -> v^-_{m+1/2} (linear weights 1/3 on stencil {m-1,m},
 * 2/3 on {m,m+1}), plus -> v^+_{m-1/2} (2/3, 1/3); beta = squared differences. */
/* WENO5-M (mapped weights, Henrick, Aslam & Powers, JCP 207 (2005) 542, eq. (8)):
 * the Jiang-Shu omega_k mapped by g_k(w) = w (d_k + d_k^2 - 3 d_k w + w^2) /
 * (d_k^2 + w (1 - 2 d_k)) and renormalised.  weights (optional) gets the mapped ones. */
double orc_weno5m_minus(double a, double b, double c, double d, double e, double eps,
                        double* weights);
double orc_weno5m_plus(double a, double b, double c, double d, double e, double eps,
                       double* weights);
/* Coefficients of cell m from the 6 boundaries xb6 = x_{m-5/2} .. x_{m+5/2}; returns 0,
 * or -1 if an ideal weight is not positive (grid too strongly stretched for WENO5). */
int32_t orc_nu_cell_coeffs(const double* xb6, orc_nu_cell* out);
double orc_weno5nu_minus(const orc_nu_cell* C, double a, double b, double c, double d, double e,
                         double eps, double* weights);
double orc_weno5nu_plus(const orc_nu_cell* C, double a, double b, double c, double d, double e,
                        double eps, double* weights);
double orc_weno3_minus(double a, double b, double c, double eps, double* weights);
double orc_weno3_plus(double a, double b, double c, double eps, double* weights);

/* S3 HLLC (Toro [14] ch. 10) in the compact branch form of DESIGN.md §3.
 * dir = 0,1,2 selects the normal velocity.  F[E] gets the flux, *uf the face
 * velocity used by the alpha*div(u) source (AMB-6). */
void orc_hllc(const orc_problem* P, const double* Gam, const double* Pi, int32_t dir,
              const double* vL, const double* vR, double* F, double* uf);

/* S1 ghost fill for every active dimension (face ghosts only). */
void orc_fill_ghosts(const orc_problem* P, double* q);

/* One RHS evaluation L(q) (eq. (1) integrated): fills ghosts (S1)
 * then accumulates x, y, z contributions (S3) into rhs (interior cells of a
 * padded array; ghost entries of rhs are set to 0). */
void orc_rhs(const orc_problem* P, double* q, double* rhs);

/* The same RHS, computed independently at a list of interior cells
 * (cells[3*c+0..2] = i, j, k), q's ghosts already filled.  out[c*E + e]. */
void orc_rhs_cells(const orc_problem* P, const double* q, int64_t ncells,
                   const int64_t* cells, double* out);

/* S4 SSP-RK3 stage combination (AMB-11), pointwise over n values:
 * stage 1: out = qs + dt*L
 * stage 2: out = 0.75*qn + 0.25*(qs + dt*L)
 * stage 3: out = (1/3)*qn + (2/3)*(qs + dt*L) */
void orc_rk3_combine(int32_t stage, int64_t n, const double* qn, const double* qs,
                     const double* L, double dt, double* out);

/* One SSP-RK3 step on the padded state q (in place), ghost fill before each L. */
void orc_rk3_step(const orc_problem* P, double* q, double dt);

/* CFL wave rate (DESIGN.md AMB-25): max over interior cells of
 * max_k (|u_k| + c)/dx_k with c^2 = ((Gamma+1)p + Pi)/(rho Gamma) (AMB-10).
 * dt = CFL / rate. */
double orc_max_wave_rate(const orc_problem* P, const double* q);

/* Admissibility check (AMB-14): returns number of interior cells with
 * non-finite values, rho <= 0 or c^2 <= 0. */
int64_t orc_count_inadmissible(const orc_problem* P, const double* q);

/* Threads the OpenMP runtime will use (for the cpu_baseline report), and a setter
 * (the single-thread grind of bench.py's cpu_baseline). */
int32_t orc_num_threads(void);
void orc_set_num_threads(int32_t n);

#ifdef __cplusplus
}
#endif
#endif
