/*
 * mfc.h -- C ABI of libmfc, the B200-native (sm_100a) fp64 right-hand-side hot
 * path of MFC's 5-equation multiphase solver (arXiv 2409.10729).
 *
 * What the library computes (PAPER.md = /root/reference/PAPER.md, line numbers):
 *   - the Allaire 5-equation model (§II-A) closed by the stiffened-gas
 *     mixture EOS, with N in {1,2,3} fluids on a structured Cartesian grid,
 *     uniform or tanh-stretched per axis (mfc_set_grid), in d in {1,2,3}
 *     dimensions;
 *   - its finite-volume semi-discretisation (eq. (1) integrated over a
 *     cell): WENO5 reconstruction of the primitive variables and the HLLC flux
 *     (WENO3 and mapped WENO5-M as options), flux differencing plus the
 *     non-conservative -h(q) div(u) term;
 *   - an SSP-RK3 time step (BASELINE.json north_star; the paper's grind unit is the
 *     "right-hand-side evaluation");
 *   - the 3-deep halo exchange between subdomains (§III-A): NCCL send/recv,
 *     or fused into the stage's last sweep as stores into the neighbours' ghost
 *     layers over peer memory (F1).
 * The readings of the paper where it is silent or garbled are listed in
 * DESIGN.md §4 (AMB-1..30); the arithmetic is specified in DESIGN.md §2-§3 step by
 * step.
 *
 * Variables (E = 2N + d + 1 equations, this order):
 *   conserved q = (a_1 r_1 .. a_N r_N, r u_1 .. r u_d, r E, a_1 .. a_N)
 *   primitive v = (a_1 r_1 .. a_N r_N,   u_1 ..   u_d,   p, a_1 .. a_N)
 *
 * State layout (device memory, fp64, caller-owned, described by mfc_layout):
 *   q[e][z][y][x] with 3 ghost cells on each side of every ACTIVE dimension,
 *   x unit-stride.  Element (e, i, j, k) of interior cell (i, j, k) is at
 *   q[layout.offset + e*stride[0] + k*stride[1] + j*stride[2] + i*stride[3]],
 *   with i, j, k running from -3 to n+2 in active dimensions (0 otherwise).
 *   The x pitch is padded so that every interior row starts 32-byte aligned.
 *   Ghost cells are scratch owned by the library and rewritten before every RHS.
 *
 * Streams: every call that takes `stream` (a cudaStream_t passed as void*) only
 * ENQUEUES work on it and returns without synchronising (except the *_host call,
 * which synchronises).  Buffers passed in must stay alive until that work is done.
 *
 * Errors: every call returns an mfc_status; nothing is thrown across the ABI.
 * mfc_last_error() returns a thread-local description of the last failure.
 * Asynchronous CUDA errors surface at the next call that checks them.
 *
 * Threading: a context is not thread-safe; many contexts may coexist.
 */
#ifndef MFC_H
#define MFC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mfc_ctx mfc_ctx; /* opaque */

typedef enum {
    MFC_OK = 0,
    MFC_EINVAL = -1,       /* bad argument (pointer, size, alignment, range) */
    MFC_ENOMEM = -2,       /* workspace missing or too small */
    MFC_ECUDA = -3,        /* a CUDA runtime/driver call failed */
    MFC_ENCCL = -4,        /* an NCCL call failed */
    MFC_ESTATE = -5,       /* call not valid in the current context state */
    MFC_EUNSUPPORTED = -6  /* valid request this build does not implement */
} mfc_status;

/* Boundary-condition codes (MFC's own numbering; DESIGN.md AMB-13).
 *   PERIODIC:      ghost -1-j <- interior n-1-j, ghost n+j <- interior j
 *   REFLECTIVE:    mirror image, normal momentum negated
 *   EXTRAPOLATION: every ghost <- the adjacent interior cell (zeroth order) */
enum { MFC_BC_PERIODIC = -1, MFC_BC_REFLECTIVE = -2, MFC_BC_EXTRAPOLATION = -3 };

/* Global grid: uniform spacing dx_k = (hi_k - lo_k)/n_global[k] unless
 * mfc_set_grid gives the axis explicit cell boundaries.
 * Inactive dimensions (k >= ndim) must have n_global[k] == 1 and procs[k] == 1. */
typedef struct {
    int32_t ndim;           /* 1..3 */
    int64_t n_global[3];    /* cells per dimension (x, y, z) */
    double lo[3], hi[3];    /* domain extents */
    int32_t procs[3];       /* rank grid; product == comm.nranks; {1,1,P} = z-slabs */
} mfc_grid;

/* Communicator.  nranks == 1: single domain, no NCCL (but see MFC_TRANSPORT_NCCL_SELF).
 * For nranks > 1 the field `loopback` selects the transport:
 *   MFC_TRANSPORT_NCCL (0): one process per GPU, NCCL over NVLink; nccl_unique_id
 *       points to the 128-byte ncclUniqueId every rank received (e.g. broadcast with
 *       torch.distributed);
 *   MFC_TRANSPORT_LOOPBACK (1): all nranks subdomains live in THIS process on one
 *       device and halos are exchanged with device copies (tests; the *_group calls);
 *   MFC_TRANSPORT_PEER (2): one process per rank, no NCCL; halos travel only as
 *       fused-halo stores into the neighbours' CUDA-IPC-mapped buffers
 *       (mfc_peer_export / mfc_peer_import below).  Works across GPUs with peer
 *       access and between processes sharing one GPU;
 *   MFC_TRANSPORT_NCCL_SELF (3): nranks == 1 only.  Every PERIODIC face is treated as a
 *       rank face whose neighbour is this rank itself, and its ghost layers travel
 *       through the NCCL halo path (pack -> ncclSend / ncclRecv to self on a one-rank
 *       communicator -> unpack, overlapped on the comm stream) instead of the sweeps'
 *       index maps; the reductions run as one-rank NCCL all-reduces.  Results are
 *       bitwise those of the plain single domain.  A verification mode for the NCCL
 *       code on one GPU (NCCL refuses two ranks on one device); nccl_unique_id may be
 *       NULL (the context generates its own).  No streamed mfc_advance_host, no fused
 *       halo. */
enum { MFC_TRANSPORT_NCCL = 0, MFC_TRANSPORT_LOOPBACK = 1, MFC_TRANSPORT_PEER = 2,
       MFC_TRANSPORT_NCCL_SELF = 3 };
typedef struct {
    int32_t rank, nranks;
    const void* nccl_unique_id;
    int32_t loopback;       /* transport, see above */
} mfc_comm;

/* Local layout, filled by mfc_get_layout. */
typedef struct {
    int32_t E, ghost, n_fluids, ndim;
    int64_t n_local[3];     /* interior cells of this rank (x, y, z) */
    int64_t lo_global[3];   /* global index of local interior cell 0 */
    int64_t dims[4];        /* padded extents [E][Z][Y][Xpitch] */
    int64_t stride[4];      /* element strides of [e][z][y][x]; stride[3] == 1 */
    int64_t offset;         /* element offset of (e=0, i=0, j=0, k=0) */
    int64_t n_elems;        /* elements a state buffer must hold = dims product */
    size_t workspace_bytes; /* bytes mfc_bind_workspace needs */
} mfc_layout;

/* Create a context (every active dimension needs n_global >= 3).  gamma[i] > 1 and pi_inf[i] >= 0 (Pa) are the stiffened-gas
 * parameters of fluid i; the library derives Gamma_i = 1/(gamma_i-1),
 * Pi_i = gamma_i pi_inf_i/(gamma_i-1).  bc = {x_lo, x_hi, y_lo, y_hi, z_lo, z_hi};
 * entries of inactive dimensions are ignored; a periodic dimension must be
 * periodic on both ends.  device = CUDA ordinal.  Split dimensions need at least 3
 * local cells.  Single-domain and loopback contexts do not touch the GPU until the
 * first call that launches work.  On success *out owns the NCCL comm until mfc_finalize.
 * Errors: EINVAL (argument), ECUDA, ENCCL. */
int mfc_init(mfc_ctx** out, const mfc_grid* grid, int32_t n_fluids, const double* gamma,
             const double* pi_inf, const int32_t bc[6], const mfc_comm* comm, int32_t device);

/* Fill *out with this rank's layout (host call, no GPU work). */
int mfc_get_layout(const mfc_ctx* ctx, mfc_layout* out);

/* Neighbour ranks of the six faces {x_lo, x_hi, y_lo, y_hi, z_lo, z_hi}; -1 where
 * the face is a physical boundary (or a periodic wrap onto this same rank).
 * Ranks are numbered x fastest: rank = cx + px*(cy + py*cz).  Host call. */
int mfc_get_neighbors(const mfc_ctx* ctx, int32_t nbr[6]);

/* Hand the library a device buffer of >= layout.workspace_bytes bytes, 256-byte
 * aligned (torch-owned; the library never frees it).  It holds two RK stage
 * buffers, the RHS accumulator, the halo pack buffers, the staging slots of the
 * streamed mfc_advance_host and the stretched-grid coefficient tables (re-uploaded on
 * a rebind).  The caller must not write it while the library uses it.  Must be bound before
 * mfc_rk3_step.  Rebinding drops the captured CUDA graph of mfc_rk3_steps.
 * Errors: EINVAL (NULL, misaligned), ENOMEM (too small), ESTATE (the fused halo is
 * attached: neighbours hold pointers into the bound stage buffers). */
int mfc_bind_workspace(mfc_ctx* ctx, void* dev_ptr, size_t bytes);

/* WENO epsilon of alpha_k = d_k/(beta_k+eps)^2 (DESIGN.md AMB-8); default 1e-16;
 * must be in [1e-30, 1e-2] (the kernels' one-reciprocal weight normalisation divides
 * by a product of two weight sums, ~ (4 eps)^8 on uniform data, which must stay a
 * normal double).  Errors: EINVAL (NULL ctx, eps out of range). */
int mfc_set_weno_eps(mfc_ctx* ctx, double eps);

/* Reconstruction order: 5 (WENO5-JS, default) or 3 (WENO3-JS), the two options of
 * P:84 ("third or fifth-order accurate WENO reconstructions").
 * The ghost depth stays 3; WENO3 reads the inner two layers.  EUNSUPPORTED for 3 on
 * a context with a stretched axis (mfc_set_grid). */
int mfc_set_weno_order(mfc_ctx* ctx, int32_t order);

/* on = 1: WENO5 with mapped nonlinear weights (WENO5-M: Henrick, Aslam & Powers, JCP 207
 * (2005) 542, eq. (8); SURVEY §8(f) F2 "optionally, mapped WENO-M"): the Jiang-Shu
 * omega_k are mapped by g_k(w) = w (d_k + d_k^2 - 3 d_k w + w^2)/(d_k^2 + w (1 - 2 d_k))
 * and renormalised; same stencils, beta_k and eps.  on = 0 (default): WENO5-JS.  No
 * effect with order 3.  EINVAL unless on is 0 or 1; EUNSUPPORTED for on = 1 on a
 * context with a stretched axis; a captured step graph is dropped. */
int mfc_set_weno_mapped(mfc_ctx* ctx, int32_t on);

/* Non-uniform grid along dimension dim ("local mesh refinement
 * is implemented using a hyperbolic tangent function [16]"; DESIGN.md AMB-27).
 * x_cb: n_global[dim]+1 strictly increasing cell boundaries of the GLOBAL axis (host
 * array, copied; any mapping, e.g. the tanh refinement of workloads.tanh_boundaries).
 * Ghost cells take the widths of the cells their data come from (periodic wrap, mirror,
 * or the boundary cell for extrapolation).  The library derives, per local cell, the
 * WENO5-JS candidate, smoothness-indicator and ideal-weight coefficients of the
 * non-uniform grid and 1/dx_m, and the sweeps along dim use them (dx of mfc_grid is
 * then ignored along dim).  x_cb == NULL restores the uniform spacing.  Needs a bound
 * workspace (the tables live in it); synchronous.  WENO5-JS only: EUNSUPPORTED with
 * WENO3 or WENO5-M selected (and those setters refuse a stretched context).
 * Errors: EINVAL (dim, n, non-increasing x_cb, or a grid so strongly stretched that an
 * ideal weight is not positive), ESTATE (no workspace), ECUDA. */
int mfc_set_grid(mfc_ctx* ctx, int32_t dim, const double* x_cb, int64_t n);

/* Primitive <-> conserved conversion on the interior cells of padded device
 * buffers (same layout for v and q; may not alias).  prim_to_cons evaluates
 * rhoE = (Gamma p + Pi) + KE, cons_to_prim the inverse in the order of DESIGN.md
 * §3 S2 (the EOS of P:64-68 with the mixture rule AMB-3). */
int mfc_prim_to_cons(mfc_ctx* ctx, const double* v, double* q, void* stream);
int mfc_cons_to_prim(mfc_ctx* ctx, const double* q, double* v, void* stream);

/* Adaptive time step (DESIGN.md AMB-25).  mfc_max_wave_rate writes
 * to the device double *d_out the maximum over all interior cells (all ranks: NCCL
 * max-allreduce) of max_k (|u_k| + c)/dx_k, c^2 = ((Gamma+1)p + Pi)/(rho Gamma);
 * enqueued on `stream`, no host sync.  mfc_cfl_dt computes it into the device
 * scratch double d_scratch, synchronises `stream` and returns *dt_out = cfl/rate on
 * the host (ESTATE if the rate is not positive and finite).  A multi-rank context
 * without an NCCL communicator (loopback or peer transport) has no way to reduce
 * across ranks: EUNSUPPORTED, so no rank ever gets a local-only dt. */
int mfc_max_wave_rate(mfc_ctx* ctx, const double* q, double* d_out, void* stream);
int mfc_cfl_dt(mfc_ctx* ctx, const double* q, double cfl, double* dt_out, double* d_scratch,
               void* stream);

/* Admissibility guard ("positivity/mixture guard"; DESIGN.md AMB-14:
 * detection, no limiter): writes to the device int64 *d_count the number of interior
 * cells (over all ranks with the NCCL transport) whose conserved state is not finite or
 * whose mixture density or squared sound speed ((Gamma+1)p + Pi)/(rho Gamma) is not
 * positive, computed from the bitwise-specified cons -> prim (S2).  Enqueued on `stream`,
 * no host sync.  Errors: EINVAL (NULL / misaligned), ECUDA, ENCCL. */
int mfc_count_inadmissible(mfc_ctx* ctx, const double* q, int64_t* d_count, void* stream);

/* Fill the 3 ghost layers of every active dimension of q: physical faces by the
 * boundary condition, faces shared with another rank by the halo exchange
 * (P:94).  Face ghosts only (edges/corners are never read).  Only ghost cells of
 * q are written. */
int mfc_halo_exchange(mfc_ctx* ctx, double* q, void* stream);

/* One RHS evaluation L(q) written on every interior cell of rhs (state
 * layout; its ghost cells are not written).  Faces shared with another rank are
 * exchanged first (into q's ghost layers); physical boundary conditions are applied
 * by the sweeps themselves through ghost-index mapping, so q's physical ghost cells
 * are neither read nor written.  q and rhs must not alias. */
int mfc_rhs(mfc_ctx* ctx, double* q, double* rhs, void* stream);

/* One SSP-RK3 step of size dt on q's interior, in place:
 *   q1 = q + dt L(q);  q2 = 3/4 q + 1/4 (q1 + dt L(q1));  q <- 1/3 q + 2/3 (q2 + dt L(q2)).
 * Needs a bound workspace (ESTATE otherwise). */
int mfc_rk3_step(mfc_ctx* ctx, double* q, double dt, void* stream);

/* nsteps SSP-RK3 steps of size dt on q (as nsteps calls of mfc_rk3_step), replayed
 * from a CUDA graph of one step that the library captures on first use and keeps
 * while q and dt stay the same (single domain, loopback and IPC-peer contexts; the
 * fused halo's stream memory operations are captured).  Removes the per-kernel launch
 * latency that dominates small grids.  With profiling enabled, and for contexts with an
 * NCCL communicator, the steps are launched individually. */
int mfc_rk3_steps(mfc_ctx* ctx, double* q, double dt, int64_t nsteps, void* stream);

/* End-to-end call with HOST buffers: copy the dense interior q_in[E][nz][ny][nx]
 * (host, pinned or pageable) into the padded device buffer q_dev, run nsteps RK3
 * steps of size dt, copy the interior back to q_out (host; may equal q_in), and
 * synchronise `stream`.  Host arrays are dense, x fastest, n_local extents; q_in and
 * q_out must each hold E*nx*ny*nz doubles (the library cannot check host sizes).
 * Needs a bound workspace.  On return q_dev holds the result (the state after the
 * nsteps steps), like q_out.
 * One step (nsteps == 1) of a single-rank 3D domain with >= 9 z planes is STREAMED
 * (DESIGN.md §6.4): a wavefront over z-chunks of >= 3 planes runs stage s of chunk k
 * once stage s-1 of chunks k-1..k+1 is done, in the whole-domain buffers, while later
 * input planes are still being copied in and finished chunks copied out (two copy
 * streams and a second compute stream besides `stream`); every plane of every stage
 * is computed once by the same kernels as mfc_rk3_step, so the result is bitwise
 * mfc_rk3_step's whatever the workspace held before.  mfc_set_stream_chunks chooses
 * the chunk count. */
int mfc_advance_host(mfc_ctx* ctx, const double* q_in, double* q_out, double* q_dev,
                     int64_t nsteps, double dt, void* stream);

/* Chunk count of the streamed mfc_advance_host step: 0 = never stream, 1 or -1 = the
 * default (32 z-chunks, ramped 3..7 planes at both ends), P > 1 = about P chunks (each
 * >= 3 planes).  EINVAL below -1. */
int mfc_set_stream_chunks(mfc_ctx* ctx, int32_t chunks);

/* Loopback groups: the same operations for `count` contexts created with
 * comm.loopback = 1 and ranks 0..count-1 (in order), exchanging halos with device
 * copies on `stream`.  With count == 1 they equal the single-context calls. */
int mfc_halo_exchange_group(mfc_ctx* const* ctxs, double* const* qs, int32_t count,
                            void* stream);
int mfc_rhs_group(mfc_ctx* const* ctxs, double* const* qs, double* const* rhss,
                  int32_t count, void* stream);
int mfc_rk3_step_group(mfc_ctx* const* ctxs, double* const* qs, int32_t count, double dt,
                       void* stream);

/* Fused halo (the halo exchange of P:94 fused into the producing
 * kernel).  Once attached, the sweep that writes each RK stage result also stores the
 * 3 cell layers next to every face shared with another rank directly into that
 * neighbour's ghost layers, so an RK3 step launches no pack / exchange / unpack work.
 * The state buffer q is REGISTERED at attach time: mfc_rk3_step, mfc_rk3_steps,
 * mfc_rhs and mfc_halo_exchange then require that same q (ESTATE otherwise).  The
 * steps keep q's ghost layers current; after writing q's interior by other means call
 * mfc_halo_exchange(q) once before the next step.  Results are bitwise identical to
 * the exchanged path.
 *
 * Loopback groups: mfc_fused_halo_group wires the contexts of one group (the same
 * ctxs/qs arrays as the *_group calls) directly; ordering comes from the stream.
 *
 * One process per rank (transport NCCL or PEER): a collective attach --
 *   mfc_peer_export(ctx, q, blob)       fills MFC_PEER_BLOB_BYTES bytes: CUDA-IPC
 *                                       handles of q, the RK stage buffers and a flag
 *                                       array (workspace must be bound);
 *   exchange the blobs (e.g. torch.distributed.all_gather_object);
 *   mfc_peer_import(ctx, face, blob)    for every face with a neighbour, with that
 *                                       neighbour's blob (EINVAL if the blob is not
 *                                       the neighbour's or the extents disagree);
 *   a barrier on all ranks before the first fused call.
 * Ranks then order their operations with stream memory operations on the flags
 * (cuStreamWaitValue64 / cuStreamWriteValue64: no spinning kernels): every fused call
 * is collective and all ranks must issue the same sequence.  mfc_rk3_steps replays a
 * CUDA graph of one step in this mode too (the stream memory operations are captured;
 * every step waits for and signals the same flag slots).  EUNSUPPORTED if the device lacks 64-bit stream
 * memory operations; ECUDA if IPC mapping fails. */
#define MFC_PEER_BLOB_BYTES 512
int mfc_fused_halo_group(mfc_ctx* const* ctxs, double* const* qs, int32_t count);
int mfc_peer_export(mfc_ctx* ctx, double* q, void* blob);
int mfc_peer_import(mfc_ctx* ctx, int32_t face, const void* blob);

/* Generate the 128-byte NCCL unique id (rank 0 calls it and broadcasts the bytes,
 * e.g. over torch.distributed, before every rank calls mfc_init). */
int mfc_nccl_get_unique_id(void* out128);

/* Poll the NCCL communicator for an asynchronous error (ncclCommGetAsyncError: a peer
 * that died, a transport failure), which NCCL reports nowhere else.  MFC_OK without a
 * communicator (nranks == 1, loopback, peer transport) or while healthy; MFC_ENCCL with
 * the reason in mfc_last_error otherwise.  The library also polls before every enqueue
 * of NCCL work (halo exchange, the max / sum reductions), so such a call returns
 * MFC_ENCCL instead of hanging; mfc_finalize then aborts the communicator instead of
 * waiting for it (ncclCommAbort). */
int mfc_comm_status(mfc_ctx* ctx);

/* Number of kernels the last mfc_rhs / mfc_rk3_step / mfc_halo_exchange call
 * launched (for the bench's launch count). */
int64_t mfc_last_launch_count(const mfc_ctx* ctx);

/* Optional CUDA-event timing of every kernel the library launches (for bench.py's
 * roofline line).  enable(on=1) clears previous records; while on, each launch is
 * bracketed by two events recorded on its own stream.  read() synchronises those
 * events and returns, per kernel kind, the summed milliseconds and launch counts:
 * kind 0/1/2 = sweep x/y/z, 3 = bc fill, 4 = halo pack/unpack, 5 = EOS conversion;
 * then clears the records.  ms/count hold nkinds entries. */
int mfc_profile_enable(mfc_ctx* ctx, int32_t on);
int mfc_profile_read(mfc_ctx* ctx, double* ms, int64_t* count, int32_t nkinds);

/* Release streams, events and the NCCL communicator (not the caller's buffers).
 *
 * Tracing: every C-ABI call that enqueues work, every RK stage and every sweep / ghost /
 * halo launch is an NVTX push/pop range in the domain "mfc" (names after the method's
 * steps S1-S4), for nsys timelines and `ncu --nvtx --nvtx-include "mfc@<range>/"`. */
int mfc_finalize(mfc_ctx* ctx);

/* Thread-local message describing the last error ("" if none). */
const char* mfc_last_error(void);

/* Library version string, e.g. "libmfc 0.1 sm_100a". */
const char* mfc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MFC_H */
