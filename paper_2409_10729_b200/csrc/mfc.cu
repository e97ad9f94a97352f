// mfc.cu -- libmfc context, layout, ghost/halo kernels, the streamed host-to-host step
// and the C ABI of include/mfc.h.
//
// Call graph of one SSP-RK3 step:
//   for stage s = 1..3:
//     halo exchange of the stage state with neighbour ranks only (pack -> NCCL
//       send/recv or loopback copies -> unpack, on a comm stream; or none with the
//       fused halo); physical boundaries are applied inside the sweeps by index mapping
//     sweep x (acc = cb*q^s + w*c_x), sweep y (acc += w*c_y), sweep z (stage result =
//       acc + w*c_z + ca*q^n), the sweeps along split dimensions waiting for the halo
//   stage 1: q -> S1,  stage 2: S1 -> S2,  stage 3: S2 -> q (in place, pointwise)
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mfc.h"
#include "dispatch.h"

using namespace mfc;

// ------------------------------------------------------------ TMA tensor maps

namespace mfc {
cudaError_t encode_state_map(CUtensorMap* out, const double* base, int64_t X, int64_t Y,
                             int64_t Z, int E, int box_x) {
    using Fn = CUresult(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                        CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                        CUtensorMapFloatOOBfill);
    static Fn* fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        void* p = nullptr;
        const cudaError_t e = cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000,
                                                               cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) return cudaErrorNotSupported;
        fn = (Fn*)p;
    }
    const cuuint64_t dims[4] = {(cuuint64_t)X, (cuuint64_t)Y, (cuuint64_t)Z, (cuuint64_t)E};
    const cuuint64_t strides[3] = {(cuuint64_t)X * 8, (cuuint64_t)(X * Y) * 8,
                                   (cuuint64_t)(X * Y * Z) * 8};
    const cuuint32_t box[4] = {(cuuint32_t)box_x, 1, 1, (cuuint32_t)E};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
}  // namespace mfc


namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU_TRY(expr)                                                                  \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess)                                                        \
            return fail(MFC_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e),   \
                        __FILE__, __LINE__);                                          \
    } while (0)

#define NCCL_TRY(expr)                                                                \
    do {                                                                              \
        ncclResult_t _r = (expr);                                                     \
        if (_r != ncclSuccess)                                                        \
            return fail(MFC_ENCCL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(_r),   \
                        __FILE__, __LINE__);                                          \
    } while (0)

constexpr int kXOff = 4;  // interior x starts at pitch index 4: 1 pad + 3 ghosts (32 B aligned)
constexpr int kStreamChunks = 32;   // z-chunks of a streamed advance_host step
constexpr int kStageCzMin = 3;      // a chunk spans at least the 3-cell stencil reach
constexpr int kStageSlots = 4;      // dense staging slots per direction
constexpr int BC_NEIGHBOR = 1;

}  // namespace

struct mfc_ctx {
    int device = 0;
    int N = 0, D = 0, E = 0;
    int64_t nl[3] = {1, 1, 1};     // local interior cells
    int64_t lo_g[3] = {0, 0, 0};   // global index of local cell 0
    int64_t dims[4] = {0, 0, 0, 0};
    int64_t stride[4] = {0, 0, 0, 1};
    int64_t off[3] = {0, 0, 0};    // interior offset per axis (x, y, z) in padded coords
    int64_t offset = 0, n_elems = 0;
    double dx[3] = {1, 1, 1};
    int bc[6] = {0, 0, 0, 0, 0, 0};  // physical bc code, or BC_NEIGHBOR
    int bc_phys[6] = {0, 0, 0, 0, 0, 0};  // the global domain's boundary conditions
    int64_t n_global[3] = {1, 1, 1};
    int nbr[6] = {-1, -1, -1, -1, -1, -1};
    Materials mat{};
    double eps = 1e-16;
    int weno_order = 5;
    int weno_mapped = 0;           // WENO5-M weights (mfc_set_weno_mapped)
    int rank = 0, nranks = 1, procs[3] = {1, 1, 1}, coords[3] = {0, 0, 0};
    bool loopback = false;
    ncclComm_t comm = nullptr;
    bool comm_failed = false;   // an asynchronous NCCL error was seen: abort, not destroy
    // workspace
    char* ws = nullptr;
    size_t ws_bytes = 0, ws_need = 0;
    double* S1 = nullptr;
    double* S2 = nullptr;
    double* acc = nullptr;
    double* sendb[6] = {};
    double* recvb[6] = {};
    int64_t face_elems[3] = {0, 0, 0};  // E * 3 * area of a face normal to dim k
    int64_t launches = 0;
    int stream_chunks = -1;       // streamed advance_host: z-chunks (-1 default, 0 off)
    // non-uniform grid (F4): global cell boundaries per stretched axis (host copy) and
    // the per-cell coefficient tables in the workspace (NU_NCOEF x (n_local + 6))
    std::vector<double> xcb[3];
    double* nu[3] = {nullptr, nullptr, nullptr};
    // optional per-launch CUDA-event timing (mfc_profile_*)
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    struct Rec { int kind; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    size_t ev_used = 0;
    // halo exchange overlapped with the sweeps that do not read the exchanged ghosts
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    // CUDA graph of one RK3 step (mfc_rk3_steps), keyed on the state pointer and dt
    cudaGraphExec_t graph = nullptr;
    cudaStream_t cap_stream = nullptr;
    const double* graph_q = nullptr;
    double graph_dt = 0.0;
    int64_t graph_launches = 0;
    // fused halo (F1): the last sweep of every RK stage stores the cells next to a
    // shared face into the neighbour's ghost layers; pf[f][b] = destination in the
    // neighbour across face f of its buffer b (0 = registered state q, 1 = S1, 2 = S2)
    int transport = 0;             // MFC_TRANSPORT_NCCL / _LOOPBACK / _PEER
    bool fused = false;            // every neighbour face attached
    bool peer_sync = false;        // IPC peers: stream memory operations order the ops
    double* fused_q = nullptr;     // the registered state buffer
    PeerFace pf[6][3] = {};
    bool pf_set[6] = {};
    uint64_t* flags = nullptr;     // device [8]: flags[f] written by the neighbour across f
    CUdeviceptr peer_flag[6] = {}; // the neighbour's 3 flag slots for its face f^1
    uint64_t epoch = 0;            // fused-halo operations completed by this rank
    uint64_t waited = 0;           // neighbour operations awaited (and slots reset) so far
    uint64_t graph_phase = 0;      // (epoch % 3, epoch - waited) the graph was captured at
    std::vector<void*> ipc_maps;   // IPC mappings this context opened
    // streamed mfc_advance_host (one step, host buffers): the sweeps of one RK stage
    // restricted to z planes [zr0, zr1) (zr1 < 0: whole domain), copy streams, events
    int64_t zr0 = 0, zr1 = -1;
    int64_t stage_cz = 0;          // planes per staging slot (0: no staging rings)
    double* stage_in = nullptr;    // kStageSlots dense input pieces [E][cz][ny][nx]
    double* stage_out = nullptr;   // kStageSlots dense result chunks
    std::vector<cudaEvent_t> ev_scat;
    cudaStream_t st_in = nullptr, st_out = nullptr, st_s1 = nullptr;
    std::vector<cudaEvent_t> ev_piece, ev_comp, ev_out, ev_s1;
    cudaEvent_t ev_start = nullptr;
};

namespace {

// bytes of one dense staging slot of the streamed step (E x stage_cz planes)
size_t stage_slot_bytes(const mfc_ctx* c) {
    return ((size_t)c->E * c->stage_cz * c->nl[0] * c->nl[1] * sizeof(double) + 255) / 256 * 256;
}

// ---------------------------------------------------------------- kernels

struct FaceGeom {
    int64_t sE, s[3];     // strides for e and axes x, y, z (s[0] == 1)
    int64_t base;         // offset of interior (0,0,0)
    int32_t n[3];         // interior extents
    int32_t E;
};

// Element t of the 3 layers next to a face of dimension dir (E x 3 x area elements):
// consecutive t walk along x wherever x is a transverse axis, so the warps' loads and
// stores are coalesced rows:  dir z: (x, y, j, e), dir y: (x, z, j, e);  across an x
// face, where a row holds only the 3 layer cells, the layer index runs fastest:
// (j, y, z, e).  Returns e; off = the element's offset from g.base + e g.sE with the
// coordinate along dir at 0, j = its layer, sd = the stride along dir.  (Scalars and
// selects only: a coordinate array indexed by the runtime dir lives in local memory.)
__device__ __forceinline__ int face_elem(int64_t t, const FaceGeom& g, int dir, int64_t& off,
                                         int& j, int64_t& sd) {
    int64_t r = t;
    if (dir == 0) {
        j = (int)(r % kGhost); r /= kGhost;
        const int64_t y = r % g.n[1]; r /= g.n[1];
        const int64_t z = r % g.n[2]; r /= g.n[2];
        off = y * g.s[1] + z * g.s[2];
        sd = 1;
    } else {
        const int64_t x = r % g.n[0]; r /= g.n[0];
        const int no = dir == 1 ? g.n[2] : g.n[1];
        const int64_t o = r % no; r /= no;
        j = (int)(r % kGhost); r /= kGhost;
        off = x + o * (dir == 1 ? g.s[2] : g.s[1]);
        sd = dir == 1 ? g.s[1] : g.s[2];
    }
    return (int)r;
}

// Physical-boundary ghost fill along dimension `dir`, both sides (S1 of DESIGN.md §3):
// periodic: ghost -1-j <- n-1-j, ghost n+j <- j; extrapolation: <- adjacent interior;
// reflective: mirror with the normal momentum (equation mom) negated.
__global__ void bc_fill_kernel(double* q, const __grid_constant__ FaceGeom g, int dir, int bc_lo, int bc_hi, int mom) {
    const int t1 = (dir + 1) % 3, t2 = (dir + 2) % 3;
    const int64_t face = (int64_t)g.n[t1] * g.n[t2] * kGhost;
    const int64_t total = face * 2 * g.E;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t es = t / face;           // (side, e) = (es % 2, es / 2)
        const int side = (int)(es % 2);
        const int e = (int)(es / 2);
        int64_t off, sd;
        int j;
        face_elem(t - es * face, g, dir, off, j, sd);
        const int bc = side ? bc_hi : bc_lo;
        if (bc == BC_NEIGHBOR) continue;
        const int n = g.n[dir];
        int ghost, src;
        if (side == 0) {
            ghost = -1 - j;
            src = bc == MFC_BC_PERIODIC ? n - 1 - j : (bc == MFC_BC_REFLECTIVE ? j : 0);
        } else {
            ghost = n + j;
            src = bc == MFC_BC_PERIODIC ? j : (bc == MFC_BC_REFLECTIVE ? n - 1 - j : n - 1);
        }
        const int64_t c0 = g.base + e * g.sE + off;
        double v = q[c0 + (int64_t)src * sd];
        if (bc == MFC_BC_REFLECTIVE && e == mom) v = -v;
        q[c0 + (int64_t)ghost * sd] = v;
    }
}

// Halo pack/unpack of every rank face of a subdomain in ONE launch.  Buffer element t
// of a face is face_elem's element t (x fastest where x is transverse, the layer index
// across an x face), viewed as rows of length L: z and y faces rows of n_x cells (one
// per (other transverse coordinate, layer, e)), x faces rows of 3 n_y (layer, y) pairs
// (one per (z, e)).  Block (row, face): the row's coordinates are formed once per
// block, in 32-bit arithmetic; its threads stride along the row (coalesced).  Pack
// reads the 3 interior layers next to the face (layer j = interior index j on the low
// side, n-3+j on the high side); unpack writes the 3 ghost layers (-3+j low, n+j high),
// so a buffer packed on one rank's high face unpacks verbatim into the neighbour's low
// ghosts.
struct FaceSet {
    int nf;
    int dir[6], side[6];
    double* buf[6];
};

__device__ __forceinline__ int face_rows(const int32_t n[3], int E, int dir) {
    return dir == 0 ? n[2] * E : (dir == 1 ? n[2] : n[1]) * kGhost * E;
}

// (__grid_constant__: fs stays in the parameter bank and is indexed by blockIdx.y there;
//  a by-value copy indexed dynamically went through every thread's local memory: 23x
//  the L2 write traffic of the packed data, r221)
__global__ void halo_pack_kernel(double* q, const __grid_constant__ FaceGeom g,
                                 const __grid_constant__ FaceSet fs,
                                 bool unpack) {
    const int f = blockIdx.y;
    const int dir = fs.dir[f], side = fs.side[f];
    const int rows = face_rows(g.n, g.E, dir);
    const int n = g.n[dir];
    const int L = dir == 0 ? kGhost * g.n[1] : g.n[0];
    const int64_t sd = dir == 0 ? 1 : (dir == 1 ? g.s[1] : g.s[2]);     // stride along dir
    double* const buf = fs.buf[f];
    auto layer = [&](int j) {             // the index along dir that layer j reads / writes
        return !unpack ? (side == 0 ? j : n - kGhost + j) : (side == 0 ? j - kGhost : n + j);
    };
    for (int row = blockIdx.x; row < rows; row += gridDim.x) {
        double* const b = buf + (int64_t)row * L;
        if (dir == 0) {                       // row = z + n_z e; element i = j + 3 y
            const int z = row % g.n[2], e = row / g.n[2];
            const int64_t r0 = g.base + e * g.sE + z * g.s[2];
            for (int i = threadIdx.x; i < L; i += blockDim.x) {
                const int j = i % kGhost, y = i / kGhost;
                const int64_t a = r0 + y * g.s[1] + layer(j);
                if (!unpack) b[i] = q[a];
                else q[a] = b[i];
            }
        } else {                              // row = o + n_o (j + 3 e); element i = x
            const int no = dir == 1 ? g.n[2] : g.n[1];
            const int64_t so = dir == 1 ? g.s[2] : g.s[1];
            const int o = row % no, je = row / no;
            const int j = je % kGhost, e = je / kGhost;
            const int64_t r0 = g.base + e * g.sE + o * so + layer(j) * sd;
            for (int i = threadIdx.x; i < L; i += blockDim.x) {
                if (!unpack) b[i] = q[r0 + i];
                else q[r0 + i] = b[i];
            }
        }
    }
}

// Dense <-> padded planes: dense[e][z][y][x] (nz planes) <-> padded interior planes
// z0 .. z0+nz of a state with strides sE, sZ, sY (x unit stride), base = interior offset.
__global__ void dense_planes_kernel(double* dense, double* padded, int64_t base, int64_t sE,
                                    int64_t sZ, int64_t sY, int nx, int ny, int64_t z0, int nz,
                                    int E, bool to_dense) {
    const int64_t plane = (int64_t)nx * ny, tot = plane * nz * E;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ez = t / plane, r = t - ez * plane;
        const int64_t e = ez / nz, z = ez - e * nz;
        const int64_t y = r / nx, x = r - y * nx;
        double* p = padded + base + e * sE + (z0 + z) * sZ + y * sY + x;
        if (to_dense) dense[t] = *p;
        else *p = dense[t];
    }
}

int grid_for(int64_t n, int threads) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 32));
}

FaceGeom geom(const mfc_ctx* c) {
    FaceGeom g;
    g.sE = c->stride[0];
    g.s[0] = 1;
    g.s[1] = c->stride[2];
    g.s[2] = c->stride[1];
    g.base = c->offset;
    for (int k = 0; k < 3; ++k) g.n[k] = (int32_t)c->nl[k];
    g.E = c->E;
    return g;
}

// Padded layout of a subdomain with interior extents nl (the same formula for every
// rank, so a neighbour's layout follows from its extents).
struct Lay {
    int64_t dims[4], stride[4], offset, n_elems;
};
Lay layout_for(int D, int E, const int64_t nl[3]) {
    Lay L;
    const int64_t X = ((kXOff + nl[0] + kGhost) + 3) / 4 * 4;
    const int64_t Y = D >= 2 ? nl[1] + 2 * kGhost : 1;
    const int64_t Z = D >= 3 ? nl[2] + 2 * kGhost : 1;
    L.dims[0] = E; L.dims[1] = Z; L.dims[2] = Y; L.dims[3] = X;
    L.stride[3] = 1; L.stride[2] = X; L.stride[1] = X * Y; L.stride[0] = X * Y * Z;
    L.offset = (D >= 3 ? kGhost : 0) * L.stride[1] + (D >= 2 ? kGhost : 0) * L.stride[2] + kXOff;
    L.n_elems = E * X * Y * Z;
    return L;
}

// Destination of my face f in a neighbour with interior extents nn and layout L
// (buffer nbuf): my cells with coordinate in [lo, hi) along the face dimension land in
// its ghost layer, at index + nn[k] across my low face, - n[k] across my high face.
PeerFace make_peer_face(const mfc_ctx* c, int f, double* nbuf, const Lay& L, const int64_t nn[3]) {
    const int k = f / 2, side = f % 2;
    PeerFace p{};
    p.dst = nbuf;
    p.sE = L.stride[0];
    p.sy = L.stride[2];
    p.sz = L.stride[1];
    const int64_t sk = k == 0 ? 1 : (k == 1 ? p.sy : p.sz);
    const int64_t shift = side == 0 ? nn[k] : -c->nl[k];
    p.off = L.offset + shift * sk;
    p.dim = k;
    p.lo = side == 0 ? 0 : (int32_t)c->nl[k] - kGhost;
    p.hi = side == 0 ? kGhost : (int32_t)c->nl[k];
    return p;
}

// Fused-halo exchange of a state (mfc_halo_exchange / mfc_rhs in fused mode): my 3
// interior layers next to face p go straight into the neighbour's ghost layers.
__global__ void peer_exchange_kernel(const double* q, const __grid_constant__ FaceGeom g,
                                     PeerFace p) {
    const int k = p.dim, t1 = (k + 1) % 3, t2 = (k + 2) % 3;
    const int64_t total = (int64_t)g.n[t1] * g.n[t2] * kGhost * g.E;
    // the neighbour's strides along the transverse axes and along k
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t off, sd;
        int j;
        const int64_t e = face_elem(t, g, k, off, j, sd);
        // my element (x, y, z) -> the neighbour's (x, y, z) + p.off: recompute its offset
        // from my coordinates (the layouts differ in padding)
        int64_t x, y, z;
        if (k == 0) {
            x = p.lo + j;
            y = (t / kGhost) % g.n[1];
            z = (t / kGhost / g.n[1]) % g.n[2];
        } else if (k == 1) {
            x = t % g.n[0];
            z = (t / g.n[0]) % g.n[2];
            y = p.lo + j;
        } else {
            x = t % g.n[0];
            y = (t / g.n[0]) % g.n[1];
            z = p.lo + j;
        }
        const double v = q[g.base + e * g.sE + off + (int64_t)(p.lo + j) * sd];
        p.dst[p.off + e * p.sE + x + y * p.sy + z * p.sz] = v;
    }
}

// ------------------------------------------------------- non-uniform grids (F4)
//
// DESIGN.md AMB-27.  WENO5 on a stretched axis reconstructs from cell averages on cells of
// unequal width.  The coefficients of cell m come from the primitive function
// V(x) = integral of v from the left end of a stencil: at the stencil's cell boundaries
// y_0 < .. < y_K it is known exactly (partial sums of v_j h_j), its interpolating
// polynomial of degree K has derivative q = V' = the reconstruction polynomial of the
// K cells (Shu, NASA CR-97-206253, 1997, §2.2), so
//   q^(r)(x) = sum_i V(y_i) L_i^(r+1)(x),  weight of v_j: h_j sum_{i > j} L_i^(r+1)(x)
// with L_i the Lagrange basis on the y's.  Everything is evaluated in the local coordinate
// t = (x - x_m)/dx_m of cell m (widths and positions scaled by dx_m), so b = q'(0) and
// c = q''(0)/2 are the t-polynomial's coefficients and beta = b^2 + (13/3) c^2.

// the coefficient-major table (NU_NCOEF rows of n + 6 cells; the x tile reads a row per
// coefficient across its lanes), then a cell-major copy (NU_CM doubles per cell, 256-byte
// aligned; a march step reads the 31 coefficients of one cell, warp-uniform)
size_t nu_cm_offset(const mfc_ctx* c, int k) {       // in doubles
    return ((size_t)NU_NCOEF * (c->nl[k] + 2 * kGhost) + NU_CM - 1) / NU_CM * NU_CM;
}
size_t nu_table_bytes(const mfc_ctx* c, int k) {
    return ((nu_cm_offset(c, k) + (size_t)NU_CM * (c->nl[k] + 2 * kGhost)) * sizeof(double) + 255) /
           256 * 256;
}

bool any_stretched(const mfc_ctx* c) {
    for (int k = 0; k < 3; ++k)
        if (!c->xcb[k].empty()) return true;
    return false;
}

// r-th derivative at x of the Lagrange basis polynomial L_i on nodes y[0..K]
double lagrange_deriv(const double* y, int K, int i, int r, double x) {
    // coefficients of prod_{l != i} (x - y_l) / (y_i - y_l), lowest degree first
    double cf[8] = {1.0, 0, 0, 0, 0, 0, 0, 0};
    int deg = 0;
    for (int l = 0; l <= K; ++l) {
        if (l == i) continue;
        const double inv = 1.0 / (y[i] - y[l]);
        for (int d = deg + 1; d >= 0; --d) {
            const double lo = d > 0 ? cf[d - 1] : 0.0;
            cf[d] = (lo - y[l] * cf[d]) * inv;
        }
        ++deg;
    }
    double v = 0.0;
    for (int d = deg; d >= r; --d) {      // Horner on the r-th derivative
        double f = 1.0;
        for (int q = 0; q < r; ++q) f *= (double)(d - q);
        v = v * x + f * cf[d];
    }
    return v;
}

// weights w[0..K-1] on the K cell values of the r-th derivative, at x, of the
// reconstruction polynomial of the cells between nodes y[0..K]
void recon_weights(const double* y, int K, int r, double x, double* w) {
    double Lp[8];
    for (int i = 0; i <= K; ++i) Lp[i] = lagrange_deriv(y, K, i, r + 1, x);
    for (int j = 0; j < K; ++j) {
        double sum = 0.0;
        for (int i = j + 1; i <= K; ++i) sum += Lp[i];
        w[j] = (y[j + 1] - y[j]) * sum;
    }
}

// Widths of the global cells -3 .. n+2 of axis k (index g + 3): a ghost cell has the
// width of the cell its data come from (periodic wrap, mirror, or the boundary cell).
std::vector<double> extended_widths(const std::vector<double>& x, int bc_lo, int bc_hi) {
    const int64_t n = (int64_t)x.size() - 1;
    auto src = [&](int64_t g) -> int64_t {           // data source of cell g
        if (g >= 0 && g < n) return g;
        if (g < 0) {
            const int64_t j = -1 - g;
            return bc_lo == MFC_BC_PERIODIC ? n - 1 - j : (bc_lo == MFC_BC_REFLECTIVE ? j : 0);
        }
        const int64_t j = g - n;
        return bc_hi == MFC_BC_PERIODIC ? j : (bc_hi == MFC_BC_REFLECTIVE ? n - 1 - j : n - 1);
    };
    std::vector<double> w(n + 6);
    for (int64_t g = -3; g < n + 3; ++g) {
        const int64_t i = src(g);
        w[g + 3] = x[i + 1] - x[i];
    }
    return w;
}

// Coefficient table of local axis k (host) -> the workspace.
int upload_nu_table(mfc_ctx* c, int k) {
    const int64_t n = c->nl[k], ld = n + 2 * kGhost;
    const std::vector<double> we = extended_widths(c->xcb[k], c->bc_phys[2 * k],
                                                   c->bc_phys[2 * k + 1]);
    std::vector<double> tab((size_t)NU_NCOEF * ld, 0.0);
    auto T = [&](int coef, int64_t m) -> double& { return tab[(size_t)coef * ld + m + kGhost]; };
    for (int64_t m = -1; m <= n; ++m) {
        const int64_t g = c->lo_g[k] + m;                 // global cell
        const double* hw = &we[g + 3 - 2];               // widths of cells g-2 .. g+2
        const double h = hw[2];
        // boundaries in units of h from the centre of cell m, built from the WIDTHS only,
        // so a cell's coefficients do not depend on where it sits (a periodic ghost
        // cell -1 and cell n-1, or the same cell seen by two subdomains, agree bitwise)
        double t[6];
        t[2] = -0.5;
        t[3] = 0.5;
        t[1] = t[2] - hw[1] / h;
        t[0] = t[1] - hw[0] / h;
        t[4] = t[3] + hw[3] / h;
        t[5] = t[4] + hw[4] / h;
        double wm[3][3], wp[3][3];                        // candidate weights at t = +-1/2
        for (int kk = 0; kk < 3; ++kk) {
            double wb[3], wc[3];
            recon_weights(t + kk, 3, 0, 0.5, wm[kk]);
            recon_weights(t + kk, 3, 0, -0.5, wp[kk]);
            recon_weights(t + kk, 3, 1, 0.0, wb);        // q'(0)
            recon_weights(t + kk, 3, 2, 0.0, wc);        // q''(0)
            const double sc = 0.5 * std::sqrt(13.0 / 3.0);
            // difference form (the weights of q' and q'' sum to 0, those of q to 1):
            //   k = 0: cells m-2, m-1, m   -> (-w0) D0 + (-w0 - w1) D1
            //   k = 1: cells m-1, m, m+1   -> (-w0) D1 + (w2) D2
            //   k = 2: cells m, m+1, m+2   -> (w1 + w2) D2 + (w2) D3
            auto diff = [&](const double* w, double& ca, double& cb) {
                if (kk == 0) { ca = -w[0]; cb = -w[0] - w[1]; }
                else if (kk == 1) { ca = -w[0]; cb = w[2]; }
                else { ca = w[1] + w[2]; cb = w[2]; }
            };
            diff(wb, T(NU_B + 2 * kk, m), T(NU_B + 2 * kk + 1, m));
            double s0, s1;
            diff(wc, s0, s1);
            T(NU_C + 2 * kk, m) = sc * s0;
            T(NU_C + 2 * kk + 1, m) = sc * s1;
            diff(wm[kk], T(NU_PM + 2 * kk, m), T(NU_PM + 2 * kk + 1, m));
            diff(wp[kk], T(NU_PP + 2 * kk, m), T(NU_PP + 2 * kk + 1, m));
        }
        // ideal weights: the 5-cell reconstruction against the outer cells' candidates
        for (int side = 0; side < 2; ++side) {
            double W5[5];
            recon_weights(t, 5, 0, side == 0 ? 0.5 : -0.5, W5);
            const double(&w)[3][3] = side == 0 ? wm : wp;
            const double d0 = W5[0] / w[0][0], d2 = W5[4] / w[2][2], d1 = 1.0 - d0 - d2;
            if (!(d0 > 0.0 && d1 > 0.0 && d2 > 0.0))
                return fail(MFC_EINVAL, "axis %d cell %lld: ideal WENO5 weight <= 0 (grid too "
                                        "strongly stretched)", k, (long long)m);
            const int base = side == 0 ? NU_DM : NU_DP;
            T(base, m) = d0;
            T(base + 1, m) = d1;
            T(base + 2, m) = d2;
        }
        T(NU_INV, m) = 1.0 / h;
    }
    CU_TRY(cudaMemcpy(c->nu[k], tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
    std::vector<double> cm((size_t)NU_CM * ld, 0.0);
    for (int64_t m = 0; m < ld; ++m)
        for (int cf = 0; cf < NU_NCOEF; ++cf) cm[(size_t)m * NU_CM + cf] = tab[(size_t)cf * ld + m];
    CU_TRY(cudaMemcpy(c->nu[k] + nu_cm_offset(c, k), cm.data(), cm.size() * sizeof(double),
                      cudaMemcpyHostToDevice));
    return MFC_OK;
}

// ------------------------------------------------------------ profiling

enum { K_SWEEP_X = 0, K_SWEEP_Y = 1, K_SWEEP_Z = 2, K_BC = 3, K_HALO = 4, K_EOS = 5, K_NKIND = 6 };

cudaEvent_t prof_event(mfc_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}

// NVTX ranges (SURVEY §5 tracing) in the domain "mfc": one per C-ABI call, RK stage,
// sweep and ghost/halo launch, named after the steps of the method, so an nsys
// timeline or `ncu --nvtx --nvtx-include "mfc@..."` selects them.  They mark the host
// side's enqueue; without an attached tool each push/pop is a test of a function pointer.
nvtxDomainHandle_t nvtx_domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("mfc");
    return d;
}

struct NvtxRange {
    explicit NvtxRange(const char* name) {
        nvtxEventAttributes_t at = {};
        at.version = NVTX_VERSION;
        at.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        at.messageType = NVTX_MESSAGE_TYPE_ASCII;
        at.message.ascii = name;
        nvtxDomainRangePushEx(nvtx_domain(), &at);
    }
    ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// sweep d = S2-S3 along d (cons->prim, WENO, HLLC, differencing, the RK stage epilogue);
// ghost fill = S1 physical faces; halo = S1 neighbour faces (pack / unpack / peer stores)
const char* const kKindName[K_NKIND] = {"sweep x", "sweep y", "sweep z", "ghost fill", "halo",
                                        "EOS"};

// Brackets one kernel launch with events on its stream when profiling is on, and with
// an NVTX range always.
struct ProfScope {
    mfc_ctx* c;
    cudaStream_t s;
    int kind;
    cudaEvent_t a = nullptr;
    NvtxRange nv;
    ProfScope(mfc_ctx* c_, cudaStream_t s_, int k) : c(c_), s(s_), kind(k), nv(kKindName[k]) {
        if (c->prof && (a = prof_event(c))) cudaEventRecord(a, s);
    }
    ~ProfScope() {
        if (!a) return;
        cudaEvent_t b = prof_event(c);
        if (!b) return;
        cudaEventRecord(b, s);
        c->recs.push_back({kind, a, b});
    }
};

int set_device(const mfc_ctx* c) {
    CU_TRY(cudaSetDevice(c->device));
    return MFC_OK;
}

// ------------------------------------------------------------ ghost filling

int bc_fill(mfc_ctx* c, double* q, cudaStream_t s) {
    const FaceGeom g = geom(c);
    for (int dir = 0; dir < c->D; ++dir) {
        if (c->bc[2 * dir] == BC_NEIGHBOR && c->bc[2 * dir + 1] == BC_NEIGHBOR) continue;
        const int t1 = (dir + 1) % 3, t2 = (dir + 2) % 3;
        const int64_t total = c->nl[t1] * c->nl[t2] * kGhost * 2 * c->E;
        ProfScope ps(c, s, K_BC);
        bc_fill_kernel<<<grid_for(total, 256), 256, 0, s>>>(q, g, dir, c->bc[2 * dir],
                                                              c->bc[2 * dir + 1], c->N + dir);
        CU_TRY(cudaGetLastError());
        ++c->launches;
    }
    return MFC_OK;
}

// one launch packs (or unpacks) every rank face of c
int halo_faces(mfc_ctx* c, double* q, bool unpack, cudaStream_t s) {
    const FaceGeom g = geom(c);
    FaceSet fs{};
    int rows = 0;
    for (int f = 0; f < 2 * c->D; ++f) {
        if (c->bc[f] != BC_NEIGHBOR) continue;
        const int dir = f / 2;
        fs.dir[fs.nf] = dir;
        fs.side[fs.nf] = f % 2;
        fs.buf[fs.nf] = unpack ? c->recvb[f] : c->sendb[f];
        ++fs.nf;
        const int64_t r = dir == 0 ? c->nl[2] * c->E : (dir == 1 ? c->nl[2] : c->nl[1]) * kGhost * c->E;
        rows = (int)std::max<int64_t>(rows, r);
    }
    if (fs.nf == 0) return MFC_OK;
    ProfScope ps(c, s, K_HALO);
    const dim3 grid((unsigned)std::min(rows, 148 * 64), (unsigned)fs.nf);
    halo_pack_kernel<<<grid, 256, 0, s>>>(q, g, fs, unpack);
    CU_TRY(cudaGetLastError());
    ++c->launches;
    return MFC_OK;
}

int halo_pack(mfc_ctx* c, const double* q, cudaStream_t s) {
    return halo_faces(c, const_cast<double*>(q), false, s);
}

int halo_unpack(mfc_ctx* c, double* q, cudaStream_t s) { return halo_faces(c, q, true, s); }

bool has_neighbors(const mfc_ctx* c) {
    for (int f = 0; f < 2 * c->D; ++f)
        if (c->bc[f] == BC_NEIGHBOR) return true;
    return false;
}

int need_ws(const mfc_ctx* c, bool stages) {
    if (!c->ws && (stages || has_neighbors(c)))
        return fail(MFC_ESTATE, "workspace not bound (mfc_bind_workspace)");
    return MFC_OK;
}

// Ghost fill for a set of contexts (count == 1: NCCL or single domain; > 1: loopback).
// physical == false: only faces shared with another rank (the sweeps apply physical
// boundary conditions themselves by index mapping, so the RHS path skips bc_fill).
int exchange_fused(mfc_ctx* const* cs, double* const* qs, int count, cudaStream_t s,
                   bool physical);
bool group_fused(mfc_ctx* const* cs, int count, int* err);

// An asynchronous NCCL failure (a peer that died, a network error) is reported by
// ncclCommGetAsyncError only; it is polled before every enqueue of NCCL work and by
// mfc_comm_status, and turns into MFC_ENCCL instead of a hang at the next collective.
int comm_async_error(mfc_ctx* c) {
    if (!c->comm) return MFC_OK;
    ncclResult_t ar = ncclSuccess;
    const ncclResult_t r = ncclCommGetAsyncError(c->comm, &ar);
    if (r != ncclSuccess) return fail(MFC_ENCCL, "ncclCommGetAsyncError: %s", ncclGetErrorString(r));
    if (ar != ncclSuccess && ar != ncclInProgress) {
        c->comm_failed = true;
        return fail(MFC_ENCCL, "NCCL asynchronous error: %s", ncclGetErrorString(ar));
    }
    return MFC_OK;
}

int exchange(mfc_ctx* const* cs, double* const* qs, int count, cudaStream_t s,
             bool physical = true) {
    {
        int err = MFC_OK;
        if (group_fused(cs, count, &err)) return exchange_fused(cs, qs, count, s, physical);
        if (err) return err;
    }
    if (cs[0]->transport == MFC_TRANSPORT_PEER)
        return fail(MFC_ESTATE, "peer transport: attach every neighbour (mfc_peer_import) first");
    for (int r = 0; r < count; ++r) {
        int st = need_ws(cs[r], false);
        if (st) return st;
        if (physical && (st = bc_fill(cs[r], qs[r], s))) return st;
        if ((st = halo_pack(cs[r], qs[r], s))) return st;
    }
    if (count == 1 && (cs[0]->nranks > 1 || cs[0]->transport == MFC_TRANSPORT_NCCL_SELF) &&
        !cs[0]->loopback) {
        mfc_ctx* c = cs[0];
        if (has_neighbors(c)) {
            int st = comm_async_error(c);
            if (st) return st;
            // NCCL pairs the k-th send A->B with the k-th receive on B from A.  The
            // message of my face f lands in the neighbour's face f^1, and every rank
            // posts its receives in ascending face order, so sends are posted in
            // ascending order of the DESTINATION face f^1 (1,0,3,2,5,4).  This matters
            // when both faces of an axis have the same peer (2 ranks, periodic).
            NCCL_TRY(ncclGroupStart());
            for (int g = 0; g < 2 * c->D; ++g) {
                const int f = g ^ 1;
                if (c->bc[f] != BC_NEIGHBOR) continue;
                NCCL_TRY(ncclSend(c->sendb[f], (size_t)c->face_elems[f / 2], ncclFloat64,
                                  c->nbr[f], c->comm, s));
            }
            for (int f = 0; f < 2 * c->D; ++f) {
                if (c->bc[f] != BC_NEIGHBOR) continue;
                NCCL_TRY(ncclRecv(c->recvb[f], (size_t)c->face_elems[f / 2], ncclFloat64,
                                  c->nbr[f], c->comm, s));
            }
            NCCL_TRY(ncclGroupEnd());
        }
    } else if (count > 1 || cs[0]->loopback) {
        // loopback: my send buffer of face f goes to the receive buffer of the
        // opposite face of neighbour nbr[f]
        for (int r = 0; r < count; ++r) {
            mfc_ctx* c = cs[r];
            for (int f = 0; f < 2 * c->D; ++f) {
                if (c->bc[f] != BC_NEIGHBOR) continue;
                const int o = c->nbr[f];
                if (o < 0 || o >= count)
                    return fail(MFC_EINVAL, "loopback group lacks rank %d", o);
                const int fo = f ^ 1;
                CU_TRY(cudaMemcpyAsync(cs[o]->recvb[fo], c->sendb[f],
                                       sizeof(double) * c->face_elems[f / 2],
                                       cudaMemcpyDeviceToDevice, s));
            }
        }
    }
    for (int r = 0; r < count; ++r) {
        int st = halo_unpack(cs[r], qs[r], s);
        if (st) return st;
    }
    return MFC_OK;
}

// ------------------------------------------------------------ fused halo (F1)
//
// Every rank performs the same sequence of fused-halo operations (collective calls).
// Operation number e (1, 2, ...) of a rank: wait until every neighbour has completed
// operation e-1, read my ghost layers, write the neighbours' ghost layers, then signal
// e to each neighbour.  Ghosts read in operation e were written in the neighbours'
// operation e-1; ghosts I write in operation e are read by the neighbour in its
// operation e+1, and the neighbour read the previous contents of that buffer (written
// 3 operations earlier, buffers rotate q -> S1 -> S2 -> q) in its operation e-2, which
// the wait on e-1 covers.  Waits and signals are stream memory operations (no
// spinning kernel); loopback groups on one stream need neither.
//
// Flags: 3 slots per face, slot e % 3 is "the neighbour completed operation e"
// (values 0 / 1).  The neighbour sets it; I wait for 1 and reset it to 0 (every slot is
// consumed once, in order).  Neighbours are at most one operation apart (operation e+1
// waits for the other's e), so when a neighbour next sets slot e % 3 -- at its
// operation e+3 -- I have long reset it.  The values are the same in every step, so a
// step captured in a CUDA graph replays correctly (mfc_rk3_steps); an epoch counter
// compared with >= would bake one step's values into the graph.

using FnStreamValue64 = CUresult(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
extern FnStreamValue64* p_wait_value;
extern FnStreamValue64* p_write_value;

// wait until every neighbour has completed operation `value` (consuming the slots of
// every operation not awaited yet, in order)
int peer_wait(mfc_ctx* c, cudaStream_t s, uint64_t value) {
    for (uint64_t v = c->waited + 1; v <= value; ++v) {
        if (v == 0) continue;
        for (int f = 0; f < 2 * c->D; ++f) {
            if (c->bc[f] != BC_NEIGHBOR) continue;
            const CUdeviceptr slot = (CUdeviceptr)(c->flags + 3 * f + v % 3);
            CUresult r = p_wait_value((CUstream)s, slot, 1, CU_STREAM_WAIT_VALUE_EQ);
            if (r == CUDA_SUCCESS)
                r = p_write_value((CUstream)s, slot, 0, CU_STREAM_WRITE_VALUE_DEFAULT);
            if (r != CUDA_SUCCESS) return fail(MFC_ECUDA, "stream memory operation failed (%d)", (int)r);
        }
        c->waited = v;
    }
    return MFC_OK;
}

int peer_signal(mfc_ctx* c, cudaStream_t s) {
    ++c->epoch;
    for (int f = 0; f < 2 * c->D; ++f) {
        if (c->bc[f] != BC_NEIGHBOR) continue;
        // default flags: the write is ordered after (and flushes) all prior work
        const CUresult r = p_write_value((CUstream)s, c->peer_flag[f] + 8 * (c->epoch % 3), 1,
                                         CU_STREAM_WRITE_VALUE_DEFAULT);
        if (r != CUDA_SUCCESS) return fail(MFC_ECUDA, "cuStreamWriteValue64 failed (%d)", (int)r);
    }
    return MFC_OK;
}

// Fused exchange of the registered states: (wait) -> physical ghosts, my boundary
// layers into the neighbours' ghosts -> (signal, then wait until the neighbours'
// layers have arrived in mine).
int exchange_fused(mfc_ctx* const* cs, double* const* qs, int count, cudaStream_t s,
                   bool physical) {
    for (int r = 0; r < count; ++r) {
        mfc_ctx* c = cs[r];
        if (qs[r] != c->fused_q)
            return fail(MFC_ESTATE, "fused halo: q is not the registered state buffer");
        int st;
        if (c->peer_sync && (st = peer_wait(c, s, c->epoch))) return st;
        if (physical && (st = bc_fill(c, qs[r], s))) return st;
        const FaceGeom g = geom(c);
        for (int f = 0; f < 2 * c->D; ++f) {
            if (c->bc[f] != BC_NEIGHBOR) continue;
            ProfScope ps(c, s, K_HALO);
            peer_exchange_kernel<<<grid_for(c->face_elems[f / 2], 256), 256, 0, s>>>(
                qs[r], g, c->pf[f][0]);
            CU_TRY(cudaGetLastError());
            ++c->launches;
        }
        if (c->peer_sync && (st = peer_signal(c, s))) return st;
    }
    for (int r = 0; r < count; ++r) {
        int st;
        if (cs[r]->peer_sync && (st = peer_wait(cs[r], s, cs[r]->epoch))) return st;
    }
    return MFC_OK;
}

bool group_fused(mfc_ctx* const* cs, int count, int* err) {
    int nf = 0;
    for (int r = 0; r < count; ++r) nf += cs[r]->fused ? 1 : 0;
    *err = (nf != 0 && nf != count)
               ? fail(MFC_ESTATE, "fused halo attached on some contexts of the group only")
               : MFC_OK;
    return nf == count;
}

// ------------------------------------------------------------------ sweeps

// Segment length T of the marches.  Longer segments waste less on the (T+2)/T halo
// recomputation; shorter ones give more warps.  Measured on C3 256^3 (profiles, T sweep
// r25b): the best is the largest T <= 128 that still gives >= 3 waves of resident
// warps (x, y: 128; z, with 3 resident blocks/SM, 64).
int seg_len(const mfc_ctx* c, int dir, int resident_warps_per_sm) {
    const int t1 = dir == 0 ? 1 : 0;          // lane axis
    const int t2 = dir == 2 ? 1 : 2;          // third axis
    const int64_t warp_lines = (c->nl[t1] + 31) / 32 * c->nl[t2];
    const int64_t n = c->nl[dir];
    const double resident = 148.0 * resident_warps_per_sm;
    int T = 128;
    while (T > 16 && (double)warp_lines * ((n + T - 1) / T) < 3.0 * resident) T /= 2;
    if (c->D == 1) T = (int)std::max<int64_t>(8, std::min<int64_t>(32, n / 8 + 1));
    return (int)std::min<int64_t>(T, n);
}

int launch_sweep_dir(mfc_ctx* c, int dir, int mode, const double* q, const double* acc,
                     double* dst, const double* qn, double w, double ca, double cb,
                     cudaStream_t s, const PeerOut* po = nullptr) {
    SweepArgs a;
    a.po.nf = 0;
    if (po) a.po = *po;
    a.q = q;
    a.acc = acc;
    a.dst = dst;
    a.qn = qn;
    a.sE = c->stride[0];
    const int64_t sax[3] = {1, c->stride[2], c->stride[1]};  // x, y, z
    int la, lb;
    if (dir == 0) { la = 1; lb = 2; }
    else if (dir == 1) { la = 0; lb = 2; }
    else { la = 0; lb = 1; }
    a.sS = sax[dir];
    a.sA = sax[la];
    a.sB = sax[lb];
    a.base = c->offset;
    a.nS = (int32_t)c->nl[dir];
    a.nA = (int32_t)c->nl[la];
    a.nB = (int32_t)c->nl[lb];
    // resident warps per SM: 12 for the non-RK ring sweeps with E <= 8 (3 blocks), else 8
    // (8 for the 3D y/z marches, which run at 2 blocks/SM: sweep.cuh march_fewop; T = 128
    // there at 256^3, C3 y 2.114 -> 2.096 ms per step against T = 64, r63)
    const bool fewop = dir >= 1 && c->D >= 2 && (mode == M_ACC || mode == M_ACCN) && c->E <= 8;
    const bool three = c->E <= 8 && dir > 0 && (mode == M_ACC || mode == M_ACCN) && !fewop;
    a.T = seg_len(c, dir, three ? 12 : 8);
    a.s_lo = 0;
    a.s_hi = a.nS;
    // a z-plane range (streamed step, c->zr1 >= 0): the z sweep updates cells
    // [zr0, zr1) of its lines, the x and y sweeps only the planes of that range
    if (c->zr1 >= 0 && c->D == 3) {
        if (dir == 2) {
            a.s_lo = (int32_t)c->zr0;
            a.s_hi = (int32_t)c->zr1;
        } else {
            a.base += c->zr0 * a.sB;
            a.nB = (int32_t)(c->zr1 - c->zr0);
        }
    }
    // physical faces are applied by index mapping inside the sweep; faces shared with
    // another rank read the ghost layers the halo exchange wrote
    {
        const int n = a.nS, lo = c->bc[2 * dir], hi = c->bc[2 * dir + 1];
        GhostMap& g = a.gm;
        g.alo = 0; g.blo = 1; g.ahi = 0; g.bhi = 1; g.flip_lo = g.flip_hi = 0;
        if (lo == MFC_BC_PERIODIC) { g.alo = n; g.blo = 1; }
        else if (lo == MFC_BC_EXTRAPOLATION) { g.alo = 0; g.blo = 0; }
        else if (lo == MFC_BC_REFLECTIVE) { g.alo = -1; g.blo = -1; g.flip_lo = 1; }
        if (hi == MFC_BC_PERIODIC) { g.ahi = -n; g.bhi = 1; }
        else if (hi == MFC_BC_EXTRAPOLATION) { g.ahi = n - 1; g.bhi = 0; }
        else if (hi == MFC_BC_REFLECTIVE) { g.ahi = 2 * n - 1; g.bhi = -1; g.flip_hi = 1; }
    }
    a.invd = 1.0 / c->dx[dir];
    a.eps4 = 4.0 * c->eps;
    a.eps = c->eps;
    a.w = w;
    a.ca = ca;
    a.cb = cb;
    a.mat = c->mat;
    // (the ring marches fix their own block shape, 32 x NTH/32, and the x-row kernels
    // their own grid; only the segment count along the sweep is passed on)
    const dim3 block(32, 1);
    const dim3 grid(1, 1, (a.s_hi - a.s_lo + a.T - 1) / a.T);
    cudaError_t e;
    ProfScope ps(c, s, K_SWEEP_X + dir);
    // kernel template order: 3, 5, 6 = WENO5 with mapped weights, 7 = WENO5 on a
    // stretched axis (per-cell coefficient tables, F4)
    const bool nu = !c->xcb[dir].empty();
    const int ord = nu ? 7 : ((c->weno_order == 5 && c->weno_mapped) ? 6 : c->weno_order);
    a.nu = nu ? c->nu[dir] : nullptr;
    a.nuc = nu ? c->nu[dir] + nu_cm_offset(c, dir) : nullptr;
    a.nu_ld = c->nl[dir] + 2 * kGhost;
    switch (c->N) {
        case 1: e = launch_sweep<1>(c->D, dir, mode, ord, a, grid, block, s); break;
        case 2: e = launch_sweep<2>(c->D, dir, mode, ord, a, grid, block, s); break;
        case 3: e = launch_sweep<3>(c->D, dir, mode, ord, a, grid, block, s); break;
        default: return fail(MFC_EINVAL, "bad N");
    }
    if (e != cudaSuccess) return fail(MFC_ECUDA, "sweep launch: %s", cudaGetErrorString(e));
    ++c->launches;
    return MFC_OK;
}

// One RHS evaluation of the stencil state q, assembled across the sweeps:
//   rk == false: dst = c_x + c_y + c_z                    (acc == dst, the rhs buffer)
//   rk == true : dst = ca*qn + cb*(q + dt*(c_x + c_y + c_z)), accumulating in acc:
//     1D: x = M_RKINIT -> dst;
//     2D/3D: x = M_RKINIT -> acc (cb*q + w*c_x, plus ca*qn in 3D with E <= 8), the middle
//     sweep M_ACC, the last sweep M_ACCN (adds ca*qn) or M_ACC.
int sweeps(mfc_ctx* c, const double* q, double* acc, double* dst, bool rk, const double* qn,
           double dt, double ca, double cb, cudaStream_t s, cudaEvent_t halo = nullptr,
           int peer_buf = -1) {
    const double w = rk ? cb * dt : 1.0;
    bool waited = false;
    for (int dir = 0; dir < c->D; ++dir) {
        // only a sweep along a split dimension reads exchanged ghost layers: it (and
        // everything after it on the stream) waits for the comm stream's halo event,
        // or, with IPC peers, for every neighbour's flag to reach the last operation
        if (!waited && (c->bc[2 * dir] == BC_NEIGHBOR || c->bc[2 * dir + 1] == BC_NEIGHBOR)) {
            if (halo) CU_TRY(cudaStreamWaitEvent(s, halo, 0));
            if (c->peer_sync && peer_buf >= 0) {
                const int st = peer_wait(c, s, c->epoch);
                if (st) return st;
            }
            waited = true;
        }
        const bool last = dir == c->D - 1;
        double* out = last ? dst : acc;
        // RK stage assembly (2D/3D): the row-parallel x sweep writes cb*q^s + w*c_x (its
        // own cells, coalesced), the middle sweep adds w*c_y and the last one
        // w*c + ca*q^n (M_ACCN, stages 2-3)
        const bool xb = rk && c->D >= 2;
        // 3D, E <= 8: the x sweep also adds ca*q^n, and the z sweep is a plain accumulate
        // (M_ACC) in every stage: C3 x +0.10, z -0.15 ms per step (r89, three same-box
        // repetitions); E = 10 loses (C5 x +1.37, z -0.84)
        const bool xbn = xb && c->D == 3 && c->E <= 8;
        int mode;
        if (dir == 0) mode = rk ? M_RKINIT : M_SET;
        else mode = (rk && last && ca != 0.0 && !xbn) ? M_ACCN : M_ACC;
        const double wd = w;
        PeerOut po;
        po.nf = 0;
        if (last && peer_buf >= 0)
            for (int f = 0; f < 2 * c->D; ++f)
                if (c->bc[f] == BC_NEIGHBOR) po.f[po.nf++] = c->pf[f][peer_buf];
        // the x sweep gets q^n only when it adds ca*q^n (its kernels test qn != nullptr)
        const double* qn_d = (dir == 0 && xb && !xbn) ? nullptr : qn;
        int st = launch_sweep_dir(c, dir, mode, q, acc, out, qn_d, wd, ca, cb, s, &po);
        if (st) return st;
    }
    return MFC_OK;
}

int check_ptr(const void* p, const char* name) {
    if (!p) return fail(MFC_EINVAL, "%s is NULL", name);
    if (((uintptr_t)p) % 32 != 0) return fail(MFC_EINVAL, "%s is not 32-byte aligned", name);
    return MFC_OK;
}

// Start the halo exchange of the stage states `in` on the comm stream of cs[0], forked
// from stream s; returns the event the sweeps along split dimensions wait on (nullptr
// when no rank has a neighbour).  With z-slabs the x and y sweeps run meanwhile.
int halo_async(mfc_ctx* const* cs, double* const* in, int count, cudaStream_t s,
               cudaEvent_t* out) {
    *out = nullptr;
    bool any = false;
    for (int r = 0; r < count; ++r) any = any || has_neighbors(cs[r]);
    if (!any) return MFC_OK;
    mfc_ctx* c0 = cs[0];
    if (!c0->comm_stream) CU_TRY(cudaStreamCreateWithFlags(&c0->comm_stream, cudaStreamNonBlocking));
    if (!c0->ev_ready) CU_TRY(cudaEventCreateWithFlags(&c0->ev_ready, cudaEventDisableTiming));
    if (!c0->ev_halo) CU_TRY(cudaEventCreateWithFlags(&c0->ev_halo, cudaEventDisableTiming));
    CU_TRY(cudaEventRecord(c0->ev_ready, s));
    CU_TRY(cudaStreamWaitEvent(c0->comm_stream, c0->ev_ready, 0));
    int st = exchange(cs, in, count, c0->comm_stream, false);
    if (st) return st;
    CU_TRY(cudaEventRecord(c0->ev_halo, c0->comm_stream));
    *out = c0->ev_halo;
    return MFC_OK;
}

int rk3_group(mfc_ctx* const* cs, double* const* qs, int count, double dt, cudaStream_t s) {
    static const double CA[3] = {0.0, 0.75, 1.0 / 3.0};
    static const double CB[3] = {1.0, 0.25, 2.0 / 3.0};
    for (int r = 0; r < count; ++r) {
        int st = need_ws(cs[r], true);
        if (st) return st;
        if ((st = check_ptr(qs[r], "q"))) return st;
        cs[r]->launches = 0;
    }
    int err = MFC_OK;
    const bool fused = group_fused(cs, count, &err);
    if (err) return err;
    for (int r = 0; fused && r < count; ++r)
        if (qs[r] != cs[r]->fused_q)
            return fail(MFC_ESTATE, "fused halo: q is not the registered state buffer");
    std::vector<double*> in(count);
    // S4: stage 1 q1 = qn + dt L(qn), 2: q2 = 3/4 qn + 1/4 (q1 + dt L(q1)),
    // 3: qn+1 = 1/3 qn + 2/3 (q2 + dt L(q2))
    static const char* const kStage[3] = {"RK3 stage 1", "RK3 stage 2", "RK3 stage 3"};
    for (int stage = 0; stage < 3; ++stage) {
        NvtxRange nv(kStage[stage]);
        for (int r = 0; r < count; ++r)
            in[r] = stage == 0 ? qs[r] : (stage == 1 ? cs[r]->S1 : cs[r]->S2);
        cudaEvent_t halo = nullptr;
        int st;
        // fused: the previous stage's last sweep already wrote the ghost layers
        if (!fused && (st = halo_async(cs, in.data(), count, s, &halo))) return st;
        for (int r = 0; r < count; ++r) {
            mfc_ctx* c = cs[r];
            double* out = stage == 0 ? c->S1 : (stage == 1 ? c->S2 : qs[r]);
            const int pb = fused ? (stage == 0 ? 1 : (stage == 1 ? 2 : 0)) : -1;
            if ((st = sweeps(c, in[r], c->acc, out, true, qs[r], dt, CA[stage], CB[stage], s,
                             halo, pb)))
                return st;
            if (fused && c->peer_sync && (st = peer_signal(c, s))) return st;
        }
    }
    return MFC_OK;
}

// ------------------------------------------------------- streamed advance_host
//
// One RK3 step of a host-resident state with the PCIe transfers overlapped by a
// wavefront over z-chunks of cz >= 3 planes.  A stage's sweeps restricted to the planes
// of chunk k read the stage input within 3 planes of it (the WENO5/HLLC reach), i.e.
// only chunks k-1, k, k+1, so stage s of chunk k can run as soon as stage s-1 of its
// two neighbours is done:
//   step j: stage 1 of chunk j, stage 2 of chunk j-1, stage 3 of chunk j-2.
// The buffers are the whole-domain ones of an ordinary step (q_dev, S1, S2, acc); every
// plane of every stage is computed exactly once, by the same code as the whole-domain
// step (the z sweep's line segments merely start at chunk boundaries: AMB-22), so the
// result is bitwise mfc_rk3_step's and it is left in q_dev.  Stage 3 writes q_dev in
// place, which is safe because stage 1 of chunk k+1 (the last reader of chunk k's input
// planes) runs before stage 3 of chunk k.  A periodic z axis closes the ring at chunk
// 0: stage 2 of chunk 0 reads stage 1 of chunk P-1, so it waits for the end, and so do
// the three stage-3 chunks that read it (P-1, 0 and 1); chunk 0's input planes stay
// intact until then (r2 fix: stage 3 of chunk 1 used to run inside the wavefront and
// read chunk 0's stage-2 planes before they were computed).
//   st_in : H2D of input piece j (= chunk j's planes) into q_dev; periodic: the piece
//           holding the last 3 planes first                             -> ev_piece[j]
//   s     : the stage sweeps in wavefront order; stage 1 of chunk k waits for the
//           pieces within 3 planes of it                                 -> ev_comp[k]
//   st_out: D2H of chunk k's result planes into q_out                    -> ev_out[k]
//   st_s1 : stage 1 of every chunk (and the scatters of the input pieces) -> ev_s1[k];
//           s then runs stages 2 and 3 only, stage 2 of chunk k after ev_s1 of chunks
//           k-1..k+1.  Stage 1 of chunk j+1 depends on input pieces alone, so it runs
//           concurrently with stages 2/3 of the chunks behind it: the small chunk
//           kernels fill each other's tails.
//           Every buffer plane is still written by one kernel and read after it:
//           stage s of chunk k touches acc / its output only on chunk k's planes, and
//           stage 3's in-place write of chunk k follows stage 2 of chunk k+1, which
//           follows stage 1 of chunk k+2 (the last reader of chunk k's input).
constexpr int kStageReach = 3;

int copy_planes_h(const mfc_ctx* c, bool h2d, const double* host_in, double* host_out,
                  double* dev, int64_t z0, int64_t nz, cudaStream_t st) {
    // planes [z0, z0+nz) of the dense host array <-> the same interior planes of dev
    const size_t row = (size_t)c->nl[0] * sizeof(double);
    const size_t pitch = (size_t)c->stride[2] * sizeof(double);
    const size_t plane_h = (size_t)c->nl[0] * c->nl[1];
    for (int e = 0; e < c->E; ++e) {
        cudaMemcpy3DParms p = {};
        double* d = dev + c->offset + e * c->stride[0] + z0 * c->stride[1];
        const size_t ho = (size_t)e * plane_h * c->nl[2] + (size_t)z0 * plane_h;
        double* h = h2d ? const_cast<double*>(host_in) + ho : host_out + ho;
        cudaPitchedPtr hp = make_cudaPitchedPtr(h, row, c->nl[0], c->nl[1]);
        cudaPitchedPtr dp = make_cudaPitchedPtr(d, pitch, c->nl[0], c->dims[2]);
        p.srcPtr = h2d ? hp : dp;
        p.dstPtr = h2d ? dp : hp;
        p.extent = make_cudaExtent(row, c->nl[1], nz);
        p.kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
        CU_TRY(cudaMemcpy3DAsync(&p, st));
    }
    return MFC_OK;
}

// Chunk depth of the streamed step, 0 when the step is not streamed.
int64_t stream_cz(const mfc_ctx* c) {
    const int chunks = c->stream_chunks;
    if (chunks == 0 || c->D != 3 || c->nranks != 1 || c->fused || !c->ws || has_neighbors(c))
        return 0;
    const int64_t nz = c->nl[2];
    const int64_t want = chunks > 1 ? chunks : kStreamChunks;
    const int64_t cz = std::max<int64_t>(kStageReach, (nz + want - 1) / want);
    return nz / kStageReach >= 3 ? cz : 0;
}

// stage (0, 1, 2) of the RK3 step of q, restricted to z planes [za, zb)
int rk3_stage_planes(mfc_ctx* c, double* q, int stage, double dt, int64_t za, int64_t zb,
                     cudaStream_t s) {
    static const double CA[3] = {0.0, 0.75, 1.0 / 3.0};
    static const double CB[3] = {1.0, 0.25, 2.0 / 3.0};
    double* in = stage == 0 ? q : (stage == 1 ? c->S1 : c->S2);
    double* out = stage == 0 ? c->S1 : (stage == 1 ? c->S2 : q);
    c->zr0 = za;
    c->zr1 = zb;
    const int st = sweeps(c, in, c->acc, out, true, q, dt, CA[stage], CB[stage], s);
    c->zr0 = 0;
    c->zr1 = -1;
    return st;
}

int advance_streamed(mfc_ctx* c, const double* q_in, double* q_out, double* q_dev, double dt,
                     int64_t cz, cudaStream_t s) {
    const int64_t nz = c->nl[2];
    // chunks of >= 3 planes (every chunk spans the stencil reach, so stage s of chunk k
    // reads stage s-1 of chunks k-1, k, k+1 only): balanced floor/ceil(nz/P) planes, or
    // (default, when nz allows) ramped -- 3, 4, 5, 6, 7 planes at both ends, cz in the
    // middle -- so the first result leaves after a few thin pieces instead of six full
    // ones and the last stages after the final piece are short (the D2H stream, busy
    // from the first result to the end, is the critical path: r75 trace)
    std::vector<int64_t> zb;   // chunk k = planes [zb[k], zb[k+1])
    {
        std::vector<int64_t> head;
        for (int64_t w = kStageReach; w < cz && head.size() < 5; ++w) head.push_back(w);
        int64_t hsum = 0;
        for (int64_t w : head) hsum += w;
        const bool ramp = !head.empty() && nz - 2 * hsum >= 2 * cz;
        zb.push_back(0);
        if (ramp) {
            for (int64_t w : head) zb.push_back(zb.back() + w);
            const int64_t mid = nz - 2 * hsum, m = (mid + cz - 1) / cz;
            const int64_t m0 = zb.back();
            for (int64_t i = 1; i <= m; ++i) zb.push_back(m0 + i * mid / m);
            for (auto it = head.rbegin(); it != head.rend(); ++it) zb.push_back(zb.back() + *it);
        } else {
            const int64_t Pu = std::min<int64_t>((nz + cz - 1) / cz, nz / kStageReach);
            for (int64_t k = 1; k <= Pu; ++k) zb.push_back(k * nz / Pu);
        }
    }
    const int P = (int)zb.size() - 1;
    int64_t max_cz = 0;
    for (int k = 0; k < P; ++k) max_cz = std::max<int64_t>(max_cz, zb[k + 1] - zb[k]);
    const bool per = c->bc[4] == MFC_BC_PERIODIC;
    auto mk = [](std::vector<cudaEvent_t>& v, int n) -> cudaError_t {
        while ((int)v.size() < n) {
            cudaEvent_t e;
            cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            if (r != cudaSuccess) return r;
            v.push_back(e);
        }
        return cudaSuccess;
    };
    CU_TRY(mk(c->ev_piece, P));
    CU_TRY(mk(c->ev_comp, P));
    CU_TRY(mk(c->ev_out, P));
    CU_TRY(mk(c->ev_s1, P));
    if (!c->st_s1) CU_TRY(cudaStreamCreateWithFlags(&c->st_s1, cudaStreamNonBlocking));
    cudaStream_t sa = c->st_s1;                    // stage 1 + input scatters
    if (!c->ev_start) CU_TRY(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
    if (!c->st_in) CU_TRY(cudaStreamCreateWithFlags(&c->st_in, cudaStreamNonBlocking));
    if (!c->st_out) CU_TRY(cudaStreamCreateWithFlags(&c->st_out, cudaStreamNonBlocking));
    auto z0 = [&](int k) { return zb[k]; };
    auto z1 = [&](int k) { return zb[k + 1]; };
    int st;
#ifdef MFC_STREAM_TRACE
    constexpr bool tr = true;      // debug build: per-piece timeline on stderr
#else
    constexpr bool tr = false;
#endif
    std::vector<std::pair<std::string, cudaEvent_t>> tr_ev;
    auto mark = [&](const std::string& name, cudaStream_t on) {
        if (!tr) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, on);
        tr_ev.emplace_back(name, e);
    };
    CU_TRY(cudaEventRecord(c->ev_start, s));
    mark("start", s);
    CU_TRY(cudaStreamWaitEvent(c->st_in, c->ev_start, 0));
    if (sa != s) CU_TRY(cudaStreamWaitEvent(sa, c->ev_start, 0));
    CU_TRY(cudaStreamWaitEvent(c->st_out, c->ev_start, 0));
    // Dense staging (c->stage_in / stage_out rings of kStageSlots pieces): the PCIe
    // copies are plain contiguous runs (E per piece) instead of 2 KB-row pitched
    // copies, which lost a quarter of the bidirectional bandwidth (r57 trace); a small
    // kernel scatters / gathers the padded planes on the compute stream.
    const bool staged = c->stage_in && max_cz <= c->stage_cz;
    CU_TRY(mk(c->ev_scat, P));
    const int64_t plane_d = c->nl[0] * c->nl[1];
    const size_t slot = stage_slot_bytes(c) / sizeof(double);
    // one 2D copy per piece: E rows of n planes (host row pitch nz planes)
    auto dense_copy = [&](bool h2d, double* dense, int64_t za, int64_t n, cudaStream_t on) -> int {
        double* h = (h2d ? const_cast<double*>(q_in) : q_out) + (size_t)za * plane_d;
        const size_t w = (size_t)n * plane_d * sizeof(double);
        const size_t hp = (size_t)nz * plane_d * sizeof(double);
        if (h2d) CU_TRY(cudaMemcpy2DAsync(dense, w, h, hp, w, c->E, cudaMemcpyHostToDevice, on));
        else CU_TRY(cudaMemcpy2DAsync(h, hp, dense, w, w, c->E, cudaMemcpyDeviceToHost, on));
        return MFC_OK;
    };
    auto planes_kernel = [&](double* dense, int64_t za, int64_t n, bool to_dense,
                             cudaStream_t on) -> int {
        dense_planes_kernel<<<grid_for(n * plane_d * c->E, 256), 256, 0, on>>>(
            dense, q_dev, c->offset, c->stride[0], c->stride[1], c->stride[2], (int)c->nl[0],
            (int)c->nl[1], za, (int)n, c->E, to_dense);
        CU_TRY(cudaGetLastError());
        ++c->launches;
        return MFC_OK;
    };
    // 1. input pieces (upload order: periodic, the piece holding the last 3 planes first)
    const int first = per ? P - 1 : 0;
    std::vector<int> order(P), rank_of(P);
    for (int i = 0; i < P; ++i) {
        order[i] = (first + i) % P;
        rank_of[order[i]] = i;
    }
    auto enqueue_h2d = [&](int i) -> int {   // input piece of upload rank i
        const int j = order[i];
        int r;
        if (staged) {
            // slot i % R is free once piece order[i - R] has been scattered (that scatter
            // is enqueued on s before this call: see need_piece)
            if (i >= kStageSlots)
                CU_TRY(cudaStreamWaitEvent(c->st_in, c->ev_scat[order[i - kStageSlots]], 0));
            if ((r = dense_copy(true, c->stage_in + (i % kStageSlots) * slot, z0(j), z1(j) - z0(j),
                                c->st_in)))
                return r;
        } else if ((r = copy_planes_h(c, true, q_in, nullptr, q_dev, z0(j), z1(j) - z0(j), c->st_in))) {
            return r;
        }
        CU_TRY(cudaEventRecord(c->ev_piece[j], c->st_in));
        mark("in" + std::to_string(j), c->st_in);
        return MFC_OK;
    };
    for (int i = 0; i < (staged ? std::min(P, kStageSlots) : P); ++i)
        if ((st = enqueue_h2d(i))) return st;
    // 2. the wavefront
    int scattered = 0;   // pieces scattered into q_dev, in upload order
    auto need_piece = [&](int j) -> int {
        if (!staged) return cudaStreamWaitEvent(sa, c->ev_piece[j], 0) == cudaSuccess
                                ? MFC_OK : fail(MFC_ECUDA, "stream wait");
        while (scattered <= rank_of[j]) {
            const int jj = order[scattered];
            CU_TRY(cudaStreamWaitEvent(sa, c->ev_piece[jj], 0));
            int r = planes_kernel(c->stage_in + (scattered % kStageSlots) * slot, z0(jj),
                                  z1(jj) - z0(jj), false, sa);
            if (r) return r;
            CU_TRY(cudaEventRecord(c->ev_scat[jj], sa));
            if (scattered + kStageSlots < P && (r = enqueue_h2d(scattered + kStageSlots))) return r;
            ++scattered;
        }
        return MFC_OK;
    };
    std::vector<int> gathered;   // chunks gathered for D2H, in order
    int last_out = 0;            // chunk whose D2H was enqueued last
    auto stage = [&](int sg, int k) -> int {
        int r;
        if (sg == 0) {   // the input pieces within reach of chunk k
            for (int m = k - 1; m <= k + 1; ++m) {
                if (!per && (m < 0 || m >= P)) continue;
                if ((r = need_piece((m + P) % P))) return r;
            }
        }
        if (sg == 1 && sa != s) {   // stage 1 of the chunks within reach, on sa
            for (int m = k - 1; m <= k + 1; ++m) {
                if (!per && (m < 0 || m >= P)) continue;
                CU_TRY(cudaStreamWaitEvent(s, c->ev_s1[(m + P) % P], 0));
            }
        }
        cudaStream_t on = sg == 0 ? sa : s;
        if ((r = rk3_stage_planes(c, q_dev, sg, dt, z0(k), z1(k), on))) return r;
        if (sg == 0) CU_TRY(cudaEventRecord(c->ev_s1[k], sa));
        mark("s" + std::to_string(sg + 1) + "c" + std::to_string(k), on);
        if (sg == 2) {
            double* dense = nullptr;
            if (staged) {
                const int o = (int)gathered.size();
                dense = c->stage_out + (o % kStageSlots) * slot;
                // slot o % R is free once the D2H of the chunk gathered R earlier is done
                if (o >= kStageSlots) CU_TRY(cudaStreamWaitEvent(s, c->ev_out[gathered[o - kStageSlots]], 0));
                gathered.push_back(k);
                if ((r = planes_kernel(dense, z0(k), z1(k) - z0(k), true, s))) return r;
            }
            CU_TRY(cudaEventRecord(c->ev_comp[k], s));
            CU_TRY(cudaStreamWaitEvent(c->st_out, c->ev_comp[k], 0));
            if (staged) {
                if ((r = dense_copy(false, dense, z0(k), z1(k) - z0(k), c->st_out))) return r;
            } else if ((r = copy_planes_h(c, false, nullptr, q_out, q_dev, z0(k), z1(k) - z0(k),
                                          c->st_out))) {
                return r;
            }
            CU_TRY(cudaEventRecord(c->ev_out[k], c->st_out));
            last_out = k;              // st_out is in order: its last event covers all
            mark("out" + std::to_string(k), c->st_out);
        }
        return MFC_OK;
    };
    c->launches = 0;
    // periodic z: stage 2 of chunk 0 needs stage 1 of chunk P-1, so it runs after the
    // loop, and so does every stage 3 that reads it: chunks P-1, 0 and 1
    const int k2 = per ? 1 : 0;                     // first chunk whose stage 2 is in the loop
    const int k3 = per ? 2 : 0;                     // first chunk whose stage 3 is in the loop
    const int e3 = per ? P - 1 : P;                 // end of the loop's stage-3 chunks
    for (int j = 0; j <= P + 1; ++j) {
        if (j < P && (st = stage(0, j))) return st;
        if (j - 1 >= k2 && j - 1 < P && (st = stage(1, j - 1))) return st;
        if (j - 2 >= k3 && j - 2 < e3 && (st = stage(2, j - 2))) return st;
    }
    if (per) {
        if ((st = stage(1, 0)) || (st = stage(2, P - 1)) || (st = stage(2, 0))) return st;
        if (P - 1 != 1 && (st = stage(2, 1))) return st;
    }
    CU_TRY(cudaStreamWaitEvent(s, c->ev_out[last_out], 0));
    CU_TRY(cudaStreamSynchronize(s));
    if (tr) {   // MFC_STREAM_TRACE: ms after the start at which each piece / chunk finished
        std::string line = "mfc stream trace (ms): ";
        for (size_t i = 0; i < tr_ev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tr_ev[0].second, tr_ev[i].second);
            char b[64];
            snprintf(b, sizeof b, "%s %.2f; ", tr_ev[i].first.c_str(), ms);
            line += b;
        }
        fprintf(stderr, "%s\n", line.c_str());
        for (auto& e : tr_ev) cudaEventDestroy(e.second);
    }
    return MFC_OK;
}

int rhs_group(mfc_ctx* const* cs, double* const* qs, double* const* rhss, int count,
              cudaStream_t s) {
    for (int r = 0; r < count; ++r) {
        int st;
        if ((st = check_ptr(qs[r], "q")) || (st = check_ptr(rhss[r], "rhs"))) return st;
        if (qs[r] == rhss[r]) return fail(MFC_EINVAL, "q and rhs alias");
        cs[r]->launches = 0;
    }
    int err = MFC_OK;
    const bool fused = group_fused(cs, count, &err);
    if (err) return err;
    if (fused) {
        // exchange (operation e), then read the ghosts and signal e+1 when done
        int st = exchange_fused(cs, qs, count, s, false);
        if (st) return st;
        for (int r = 0; r < count; ++r) {
            if ((st = sweeps(cs[r], qs[r], rhss[r], rhss[r], false, nullptr, 0, 0, 0, s)))
                return st;
            if (cs[r]->peer_sync && (st = peer_signal(cs[r], s))) return st;
        }
        return MFC_OK;
    }
    cudaEvent_t halo = nullptr;
    int st = halo_async(cs, qs, count, s, &halo);
    if (st) return st;
    for (int r = 0; r < count; ++r)
        if ((st = sweeps(cs[r], qs[r], rhss[r], rhss[r], false, nullptr, 0, 0, 0, s, halo)))
            return st;
    return MFC_OK;
}

// ---------------------------------------------------------- driver entry points
// The few driver-API calls (stream memory operations, address ranges) are resolved
// through the runtime at first use, so libmfc.so does not link libcuda and still
// loads on a machine without a GPU driver.

template <class F>
int drv(const char* name, F** fn) {
    if (*fn) return MFC_OK;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    void* p = nullptr;
    const cudaError_t e = cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
        return fail(MFC_ECUDA, "driver entry point %s unavailable", name);
    *fn = (F*)p;
    return MFC_OK;
}

using FnMemGetAddressRange = CUresult(CUdeviceptr*, size_t*, CUdeviceptr);
using FnDeviceGetAttribute = CUresult(int*, CUdevice_attribute, CUdevice);
using FnDeviceGet = CUresult(CUdevice*, int);
FnStreamValue64* p_wait_value = nullptr;
FnStreamValue64* p_write_value = nullptr;
FnMemGetAddressRange* p_addr_range = nullptr;
FnDeviceGetAttribute* p_dev_attr = nullptr;
FnDeviceGet* p_dev_get = nullptr;

// ---------------------------------------------------------- CUDA IPC plumbing

constexpr uint64_t kPeerMagic = 0x3152454550434d46ull;   // "FMCPEER1"

struct PeerBlob {                 // what mfc_peer_export hands to the neighbours
    uint64_t magic;
    int32_t rank, E, D, pad;
    int64_t nl[3];
    cudaIpcMemHandle_t h[4];      // allocations holding q, S1, S2, flags
    int64_t off[4];               // byte offsets of those buffers inside them
};
static_assert(sizeof(PeerBlob) <= MFC_PEER_BLOB_BYTES, "peer blob size");

// A process maps each exported allocation once (cudaIpcOpenMemHandle refuses a second
// mapping of the same handle); contexts share the mapping with a reference count.
std::mutex g_ipc_mu;
std::map<std::string, std::pair<void*, int>> g_ipc;

int ipc_open(const cudaIpcMemHandle_t& h, void** out) {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    const std::string key((const char*)&h, sizeof h);
    auto it = g_ipc.find(key);
    if (it != g_ipc.end()) {
        ++it->second.second;
        *out = it->second.first;
        return MFC_OK;
    }
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(MFC_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    g_ipc[key] = {p, 1};
    *out = p;
    return MFC_OK;
}

void ipc_release(void* p) {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    for (auto it = g_ipc.begin(); it != g_ipc.end(); ++it) {
        if (it->second.first != p) continue;
        if (--it->second.second == 0) {
            cudaIpcCloseMemHandle(p);
            g_ipc.erase(it);
        }
        return;
    }
}

}  // namespace

// =================================================================== C ABI

extern "C" {

const char* mfc_last_error(void) { return g_err.c_str(); }

const char* mfc_version(void) { return "libmfc 0.1 sm_100a fp64"; }

int mfc_init(mfc_ctx** out, const mfc_grid* grid, int32_t n_fluids, const double* gamma,
             const double* pi_inf, const int32_t bc[6], const mfc_comm* comm, int32_t device) {
    g_err.clear();
    if (!out || !grid || !gamma || !pi_inf || !bc) return fail(MFC_EINVAL, "NULL argument");
    *out = nullptr;
    if (grid->ndim < 1 || grid->ndim > 3) return fail(MFC_EINVAL, "ndim must be 1..3");
    if (n_fluids < 1 || n_fluids > kMaxFluids) return fail(MFC_EINVAL, "n_fluids must be 1..3");
    for (int i = 0; i < n_fluids; ++i) {
        if (!(gamma[i] > 1.0) || !std::isfinite(gamma[i]))
            return fail(MFC_EINVAL, "gamma[%d] must be > 1", i);
        if (!(pi_inf[i] >= 0.0) || !std::isfinite(pi_inf[i]))
            return fail(MFC_EINVAL, "pi_inf[%d] must be >= 0", i);
    }
    const int D = grid->ndim;
    int nranks = comm ? comm->nranks : 1;
    int rank = comm ? comm->rank : 0;
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(MFC_EINVAL, "bad rank/nranks");
    int64_t prod = 1;
    for (int k = 0; k < 3; ++k) {
        const int p = grid->procs[k] > 0 ? grid->procs[k] : 1;
        prod *= p;
        if (k >= D && (grid->n_global[k] != 1 || p != 1))
            return fail(MFC_EINVAL, "inactive dim %d must have n=1, procs=1", k);
        if (k < D) {
            if (grid->n_global[k] < kGhost)
                return fail(MFC_EINVAL, "n_global[%d] = %lld < 3 (WENO5 stencil)", k,
                            (long long)grid->n_global[k]);
            if (!(grid->hi[k] > grid->lo[k])) return fail(MFC_EINVAL, "hi[%d] <= lo[%d]", k, k);
            const bool per_lo = bc[2 * k] == MFC_BC_PERIODIC, per_hi = bc[2 * k + 1] == MFC_BC_PERIODIC;
            if (per_lo != per_hi) return fail(MFC_EINVAL, "dim %d periodic on one end only", k);
            for (int sd = 0; sd < 2; ++sd) {
                const int b = bc[2 * k + sd];
                if (b != MFC_BC_PERIODIC && b != MFC_BC_REFLECTIVE && b != MFC_BC_EXTRAPOLATION)
                    return fail(MFC_EINVAL, "bc[%d] = %d unknown", 2 * k + sd, b);
            }
        }
    }
    if (prod != nranks) return fail(MFC_EINVAL, "prod(procs) = %lld != nranks = %d",
                                    (long long)prod, nranks);

    mfc_ctx* c = new mfc_ctx();
    c->device = device;
    c->N = n_fluids;
    c->D = D;
    c->E = 2 * n_fluids + D + 1;
    c->rank = rank;
    c->nranks = nranks;
    c->transport = comm ? comm->loopback : MFC_TRANSPORT_NCCL;
    if (c->transport < MFC_TRANSPORT_NCCL || c->transport > MFC_TRANSPORT_NCCL_SELF) {
        delete c;
        return fail(MFC_EINVAL, "comm.loopback (transport) must be 0, 1, 2 or 3");
    }
    if (c->transport == MFC_TRANSPORT_NCCL_SELF && nranks != 1) {
        delete c;
        return fail(MFC_EINVAL, "MFC_TRANSPORT_NCCL_SELF is a one-rank mode (nranks = %d)", nranks);
    }
    c->loopback = c->transport == MFC_TRANSPORT_LOOPBACK;
    for (int k = 0; k < 3; ++k) c->procs[k] = grid->procs[k] > 0 ? grid->procs[k] : 1;
    c->coords[0] = rank % c->procs[0];
    c->coords[1] = (rank / c->procs[0]) % c->procs[1];
    c->coords[2] = rank / (c->procs[0] * c->procs[1]);
    for (int k = 0; k < 3; ++k) {
        const int64_t n = grid->n_global[k], p = c->procs[k], ci = c->coords[k];
        const int64_t base = n / p, rem = n % p;
        c->nl[k] = base + (ci < rem ? 1 : 0);
        c->lo_g[k] = ci * base + std::min<int64_t>(ci, rem);
        c->dx[k] = k < D ? (grid->hi[k] - grid->lo[k]) / (double)n : 1.0;
        if (k < D && p > 1 && c->nl[k] < kGhost) {
            const long long nl = (long long)c->nl[k];
            delete c;
            return fail(MFC_EINVAL, "dim %d: local extent %lld < 3", k, nl);
        }
        if (k < D && bc[2 * k] == MFC_BC_PERIODIC && n < kGhost) {
            delete c;
            return fail(MFC_EINVAL, "periodic dim %d needs >= 3 cells", k);
        }
    }
    // neighbours (rank = cx + px*(cy + py*cz))
    for (int k = 0; k < 3; ++k) c->n_global[k] = grid->n_global[k];
    for (int k = 0; k < D; ++k) {
        for (int sd = 0; sd < 2; ++sd) {
            const int f = 2 * k + sd;
            c->bc[f] = bc[f];
            c->bc_phys[f] = bc[f];
            if (c->transport == MFC_TRANSPORT_NCCL_SELF && bc[f] == MFC_BC_PERIODIC) {
                c->bc[f] = BC_NEIGHBOR;      // a periodic face is a rank face with myself
                c->nbr[f] = rank;
                continue;
            }
            if (c->procs[k] == 1) continue;
            int cc[3] = {c->coords[0], c->coords[1], c->coords[2]};
            cc[k] += sd ? 1 : -1;
            if (cc[k] < 0 || cc[k] >= c->procs[k]) {
                if (bc[f] != MFC_BC_PERIODIC) continue;
                cc[k] = (cc[k] + c->procs[k]) % c->procs[k];
            }
            c->bc[f] = BC_NEIGHBOR;
            c->nbr[f] = cc[0] + c->procs[0] * (cc[1] + c->procs[1] * cc[2]);
        }
    }
    for (int i = 0; i < n_fluids; ++i) {
        c->mat.Gam[i] = 1.0 / (gamma[i] - 1.0);
        c->mat.Pi[i] = (gamma[i] * pi_inf[i]) / (gamma[i] - 1.0);
    }
    // layout
    const Lay L = layout_for(D, c->E, c->nl);
    for (int k = 0; k < 4; ++k) {
        c->dims[k] = L.dims[k];
        c->stride[k] = L.stride[k];
    }
    c->off[0] = kXOff;
    c->off[1] = D >= 2 ? kGhost : 0;
    c->off[2] = D >= 3 ? kGhost : 0;
    c->offset = L.offset;
    c->n_elems = L.n_elems;
    size_t need = 3 * (size_t)c->n_elems * sizeof(double);
    for (int k = 0; k < D; ++k) {
        const int t1 = (k + 1) % 3, t2 = (k + 2) % 3;
        c->face_elems[k] = (int64_t)c->E * kGhost * c->nl[t1] * c->nl[t2];
        for (int sd = 0; sd < 2; ++sd)
            if (c->bc[2 * k + sd] == BC_NEIGHBOR)
                need += 2 * (((size_t)c->face_elems[k] * sizeof(double) + 255) / 256 * 256);
    }
    // non-uniform grid coefficient tables, one per active axis (F4)
    for (int k = 0; k < D; ++k) need += nu_table_bytes(c, k);
    // streamed advance_host (single-rank 3D): dense staging rings for the PCIe copies
    if (D == 3 && nranks == 1 && c->transport != MFC_TRANSPORT_NCCL_SELF &&
        c->nl[2] >= 3 * kStageCzMin) {
        c->stage_cz = std::max<int64_t>(kStageCzMin, (c->nl[2] + kStreamChunks - 1) / kStreamChunks);
        need += 2 * kStageSlots * stage_slot_bytes(c);
    }
    c->ws_need = need;

    // The device is only touched here when NCCL needs it; single-domain and loopback
    // contexts are pure host bookkeeping until the first GPU call (so layouts can be
    // queried on a machine without a GPU).
    const bool self = c->transport == MFC_TRANSPORT_NCCL_SELF;
    if ((nranks > 1 && c->transport == MFC_TRANSPORT_NCCL) || self) {
        if (cudaSetDevice(device) != cudaSuccess) {
            delete c;
            return fail(MFC_ECUDA, "cudaSetDevice(%d) failed", device);
        }
        ncclUniqueId id;
        if (comm->nccl_unique_id) {
            memcpy(&id, comm->nccl_unique_id, sizeof id);
        } else if (self) {           // a one-rank communicator: its own id
            const ncclResult_t r = ncclGetUniqueId(&id);
            if (r != ncclSuccess) {
                delete c;
                return fail(MFC_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
            }
        } else {
            delete c;
            return fail(MFC_EINVAL, "nccl_unique_id is NULL with nranks > 1");
        }
        ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            delete c;
            return fail(MFC_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
        }
    }
    *out = c;
    return MFC_OK;
}

int mfc_get_layout(const mfc_ctx* c, mfc_layout* o) {
    if (!c || !o) return fail(MFC_EINVAL, "NULL argument");
    o->E = c->E;
    o->ghost = kGhost;
    o->n_fluids = c->N;
    o->ndim = c->D;
    for (int k = 0; k < 3; ++k) {
        o->n_local[k] = c->nl[k];
        o->lo_global[k] = c->lo_g[k];
    }
    for (int k = 0; k < 4; ++k) {
        o->dims[k] = c->dims[k];
        o->stride[k] = c->stride[k];
    }
    o->offset = c->offset;
    o->n_elems = c->n_elems;
    o->workspace_bytes = c->ws_need;
    return MFC_OK;
}

int mfc_get_neighbors(const mfc_ctx* c, int32_t nbr[6]) {
    if (!c || !nbr) return fail(MFC_EINVAL, "NULL argument");
    for (int f = 0; f < 6; ++f) nbr[f] = c->bc[f] == BC_NEIGHBOR ? c->nbr[f] : -1;
    return MFC_OK;
}

int mfc_bind_workspace(mfc_ctx* c, void* p, size_t bytes) {
    if (!c || !p) return fail(MFC_EINVAL, "NULL argument");
    if ((uintptr_t)p % 256) return fail(MFC_EINVAL, "workspace not 256-byte aligned");
    if (bytes < c->ws_need)
        return fail(MFC_ENOMEM, "workspace %zu < %zu bytes", bytes, c->ws_need);
    if (c->fused)
        return fail(MFC_ESTATE, "fused halo attached: the neighbours hold pointers into the "
                                "bound stage buffers; rebinding is not allowed");
    if (c->graph) {                  // the captured step reads and writes the old buffers
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    c->ws = (char*)p;
    c->ws_bytes = bytes;
    char* w = c->ws;
    const size_t sb = (size_t)c->n_elems * sizeof(double);
    c->S1 = (double*)w; w += sb;
    c->S2 = (double*)w; w += sb;
    c->acc = (double*)w; w += sb;
    if (c->stage_cz) {
        c->stage_in = (double*)w; w += kStageSlots * stage_slot_bytes(c);
        c->stage_out = (double*)w; w += kStageSlots * stage_slot_bytes(c);
    }
    for (int k = 0; k < c->D; ++k) {
        c->nu[k] = (double*)w;
        w += nu_table_bytes(c, k);
    }
    for (int f = 0; f < 6; ++f) {
        c->sendb[f] = c->recvb[f] = nullptr;
        if (f / 2 < c->D && c->bc[f] == BC_NEIGHBOR) {
            const size_t fb = ((size_t)c->face_elems[f / 2] * sizeof(double) + 255) / 256 * 256;
            c->sendb[f] = (double*)w; w += fb;
            c->recvb[f] = (double*)w; w += fb;
        }
    }
    // a rebind keeps the stretched grids: their tables move into the new workspace
    for (int k = 0; k < c->D; ++k) {
        if (c->xcb[k].empty()) continue;
        const int st = upload_nu_table(c, k);
        if (st) return st;
    }
    return MFC_OK;
}

int mfc_set_grid(mfc_ctx* c, int32_t dim, const double* x_cb, int64_t n) {
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    if (dim < 0 || dim >= c->D) return fail(MFC_EINVAL, "dim %d is not active", dim);
    int st;
    if ((st = need_ws(c, true))) return st;
    if ((st = set_device(c))) return st;
    if (c->graph) {                  // captured kernels depend on the grid
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    if (!x_cb) {
        c->xcb[dim].clear();
        return MFC_OK;
    }
    if (n != c->n_global[dim]) return fail(MFC_EINVAL, "n = %lld != n_global[%d] = %lld",
                                           (long long)n, dim, (long long)c->n_global[dim]);
    if (c->weno_order != 5 || c->weno_mapped)
        return fail(MFC_EUNSUPPORTED, "stretched grids run WENO5-JS only (DESIGN.md AMB-27)");
    std::vector<double> x(x_cb, x_cb + n + 1);
    for (int64_t i = 0; i < n; ++i)
        if (!(x[i + 1] > x[i]) || !std::isfinite(x[i]) || !std::isfinite(x[i + 1]))
            return fail(MFC_EINVAL, "x_cb must be finite and strictly increasing (index %lld)",
                        (long long)i);
    std::vector<double> keep = std::move(c->xcb[dim]);
    c->xcb[dim] = std::move(x);
    if ((st = upload_nu_table(c, dim))) {
        c->xcb[dim] = std::move(keep);
        return st;
    }
    return MFC_OK;
}

int mfc_set_stream_chunks(mfc_ctx* c, int32_t chunks) {
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    if (chunks < -1) return fail(MFC_EINVAL, "chunks must be >= -1");
    c->stream_chunks = chunks;
    return MFC_OK;
}

int mfc_set_weno_mapped(mfc_ctx* c, int32_t on) {
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    if (on != 0 && on != 1) return fail(MFC_EINVAL, "mapped must be 0 or 1");
    if (on && any_stretched(c))
        return fail(MFC_EUNSUPPORTED, "stretched grids run WENO5-JS only (DESIGN.md AMB-27)");
    c->weno_mapped = on;
    if (c->graph) {                  // captured kernels depend on the weights
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return MFC_OK;
}

int mfc_set_weno_order(mfc_ctx* c, int32_t order) {
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    if (order != 3 && order != 5) return fail(MFC_EINVAL, "WENO order must be 3 or 5");
    if (order != 5 && any_stretched(c))
        return fail(MFC_EUNSUPPORTED, "stretched grids run WENO5-JS only (DESIGN.md AMB-27)");
    c->weno_order = order;
    if (c->graph) {                  // captured kernels depend on the order
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return MFC_OK;
}

int mfc_set_weno_eps(mfc_ctx* c, double eps) {
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    // >= 1e-30: the one-reciprocal WENO forms divide by products of two weight sums,
    // ~ (4 eps)^8 on uniform data, which must stay a normal double (rcp.approx.ftz)
    if (!(eps >= 1e-30 && eps <= 1e-2)) return fail(MFC_EINVAL, "eps out of [1e-30, 1e-2]");
    c->eps = eps;
    if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    return MFC_OK;
}

static int eos(mfc_ctx* c, const double* in, double* out, bool to_cons, void* stream) {
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    int st;
    if ((st = check_ptr(in, "input")) || (st = check_ptr(out, "output"))) return st;
    if (in == out) return fail(MFC_EINVAL, "input and output alias");
    if ((st = set_device(c))) return st;
    EosArgs a;
    a.in = in;
    a.out = out;
    a.sE = c->stride[0];
    a.sZ = c->stride[1];
    a.sY = c->stride[2];
    a.base = c->offset;
    a.nx = (int32_t)c->nl[0];
    a.ny = (int32_t)c->nl[1];
    a.nz = (int32_t)c->nl[2];
    a.mat = c->mat;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    switch (c->N) {
        case 1: e = launch_eos<1>(c->D, to_cons, a, s); break;
        case 2: e = launch_eos<2>(c->D, to_cons, a, s); break;
        default: e = launch_eos<3>(c->D, to_cons, a, s); break;
    }
    if (e != cudaSuccess) return fail(MFC_ECUDA, "eos launch: %s", cudaGetErrorString(e));
    return MFC_OK;
}

int mfc_max_wave_rate(mfc_ctx* c, const double* q, double* d_out, void* stream) {
    NvtxRange nv("mfc_max_wave_rate");
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    if (c->nranks > 1 && c->transport != MFC_TRANSPORT_NCCL)
        return fail(MFC_EUNSUPPORTED, "max wave rate over %d ranks needs the NCCL transport "
                                      "(loopback / peer contexts cannot reduce across ranks)",
                    c->nranks);
    int st;
    if ((st = check_ptr(q, "q")) || (st = set_device(c))) return st;
    if (!d_out || ((uintptr_t)d_out) % 8) return fail(MFC_EINVAL, "d_out NULL or misaligned");
    cudaStream_t s = (cudaStream_t)stream;
    EosArgs a;
    a.in = q;
    a.out = nullptr;
    a.sE = c->stride[0];
    a.sZ = c->stride[1];
    a.sY = c->stride[2];
    a.base = c->offset;
    a.nx = (int32_t)c->nl[0];
    a.ny = (int32_t)c->nl[1];
    a.nz = (int32_t)c->nl[2];
    a.mat = c->mat;
    const double3 inv = make_double3(1.0 / c->dx[0], 1.0 / c->dx[1], 1.0 / c->dx[2]);
    WaveGrid wg;
    for (int k = 0; k < 3; ++k)   // stretched axes: the 1/dx row of the table, from cell 0
        wg.inv[k] = (k < c->D && !c->xcb[k].empty())
                        ? c->nu[k] + NU_INV * (c->nl[k] + 2 * kGhost) + kGhost : nullptr;
    CU_TRY(cudaMemsetAsync(d_out, 0, sizeof(double), s));
    cudaError_t e;
    switch (c->N) {
        case 1: e = launch_wave_rate<1>(c->D, a, inv, wg, d_out, s); break;
        case 2: e = launch_wave_rate<2>(c->D, a, inv, wg, d_out, s); break;
        default: e = launch_wave_rate<3>(c->D, a, inv, wg, d_out, s); break;
    }
    if (e != cudaSuccess) return fail(MFC_ECUDA, "wave rate launch: %s", cudaGetErrorString(e));
    if (c->comm) {
        if ((st = comm_async_error(c))) return st;
        NCCL_TRY(ncclAllReduce(d_out, d_out, 1, ncclFloat64, ncclMax, c->comm, s));
    }
    return MFC_OK;
}

int mfc_count_inadmissible(mfc_ctx* c, const double* q, int64_t* d_count, void* stream) {
    NvtxRange nv("mfc_count_inadmissible");
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    int st;
    if ((st = check_ptr(q, "q")) || (st = set_device(c))) return st;
    if (!d_count || ((uintptr_t)d_count) % 8) return fail(MFC_EINVAL, "d_count NULL or misaligned");
    cudaStream_t s = (cudaStream_t)stream;
    EosArgs a;
    a.in = q;
    a.out = nullptr;
    a.sE = c->stride[0];
    a.sZ = c->stride[1];
    a.sY = c->stride[2];
    a.base = c->offset;
    a.nx = (int32_t)c->nl[0];
    a.ny = (int32_t)c->nl[1];
    a.nz = (int32_t)c->nl[2];
    a.mat = c->mat;
    CU_TRY(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
    auto* o = reinterpret_cast<unsigned long long*>(d_count);
    cudaError_t e;
    switch (c->N) {
        case 1: e = launch_admissible<1>(c->D, a, o, s); break;
        case 2: e = launch_admissible<2>(c->D, a, o, s); break;
        default: e = launch_admissible<3>(c->D, a, o, s); break;
    }
    if (e != cudaSuccess) return fail(MFC_ECUDA, "admissibility launch: %s", cudaGetErrorString(e));
    if (c->comm) {
        if ((st = comm_async_error(c))) return st;
        NCCL_TRY(ncclAllReduce(d_count, d_count, 1, ncclInt64, ncclSum, c->comm, s));
    }
    return MFC_OK;
}

int mfc_cfl_dt(mfc_ctx* c, const double* q, double cfl, double* dt_out, double* d_scratch,
               void* stream) {
    NvtxRange nv("mfc_cfl_dt");
    if (!c || !dt_out || !d_scratch) return fail(MFC_EINVAL, "NULL argument");
    if (!(cfl > 0.0) || !std::isfinite(cfl)) return fail(MFC_EINVAL, "cfl must be > 0");
    int st = mfc_max_wave_rate(c, q, d_scratch, stream);
    if (st) return st;
    double rate = 0.0;
    CU_TRY(cudaMemcpyAsync(&rate, d_scratch, sizeof(double), cudaMemcpyDeviceToHost,
                           (cudaStream_t)stream));
    CU_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    if (!(rate > 0.0) || !std::isfinite(rate))
        return fail(MFC_ESTATE, "wave rate %g is not positive and finite", rate);
    *dt_out = cfl / rate;
    return MFC_OK;
}

int mfc_prim_to_cons(mfc_ctx* c, const double* v, double* q, void* stream) {
    return eos(c, v, q, true, stream);
}

int mfc_cons_to_prim(mfc_ctx* c, const double* q, double* v, void* stream) {
    return eos(c, q, v, false, stream);
}

int mfc_halo_exchange(mfc_ctx* c, double* q, void* stream) {
    NvtxRange nv("mfc_halo_exchange");
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    int st;
    if ((st = check_ptr(q, "q")) || (st = set_device(c))) return st;
    c->launches = 0;
    return exchange(&c, &q, 1, (cudaStream_t)stream);
}

int mfc_rhs(mfc_ctx* c, double* q, double* rhs, void* stream) {
    NvtxRange nv("mfc_rhs");
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    int st = set_device(c);
    if (st) return st;
    return rhs_group(&c, &q, &rhs, 1, (cudaStream_t)stream);
}

int mfc_rk3_step(mfc_ctx* c, double* q, double dt, void* stream) {
    NvtxRange nv("mfc_rk3_step");
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    if (!std::isfinite(dt)) return fail(MFC_EINVAL, "dt not finite");
    int st = set_device(c);
    if (st) return st;
    return rk3_group(&c, &q, 1, dt, (cudaStream_t)stream);
}

int mfc_rk3_steps(mfc_ctx* c, double* q, double dt, int64_t nsteps, void* stream) {
    NvtxRange nv("mfc_rk3_steps");
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    if (!std::isfinite(dt)) return fail(MFC_EINVAL, "dt not finite");
    if (nsteps < 0) return fail(MFC_EINVAL, "nsteps < 0");
    int st = set_device(c);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (c->prof || c->comm) {
        // per-launch event timing needs the plain launches; NCCL contexts launch every
        // step plainly too (capturing NCCL send/recv in a graph has never run on more than
        // one GPU with this build)
        for (int64_t i = 0; i < nsteps; ++i)
            if ((st = rk3_group(&c, &q, 1, dt, s))) return st;
        return MFC_OK;
    }
    if (nsteps == 0) return MFC_OK;
    // IPC peers: the captured flag slots depend on the operation phase (peer_wait).  A
    // step that starts one awaited operation behind (epoch - waited == 1, the state
    // every step leaves) advances both counters by 3, so one graph serves all of them;
    // from any other state (after an exchange or an RHS call) one plain step first
    if (c->peer_sync && c->epoch - c->waited != 1) {
        if ((st = rk3_group(&c, &q, 1, dt, s))) return st;
        if (--nsteps == 0) return MFC_OK;
    }
    const uint64_t phase = c->peer_sync ? ((c->epoch % 3) | ((c->epoch - c->waited) << 2)) : 0;
    if (!c->graph || c->graph_q != q || c->graph_dt != dt || c->graph_phase != phase) {
        if (c->graph) {
            cudaGraphExecDestroy(c->graph);
            c->graph = nullptr;
        }
        if (!c->cap_stream) CU_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
        CU_TRY(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
        st = rk3_group(&c, &q, 1, dt, c->cap_stream);
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
        if (st) {
            if (g) cudaGraphDestroy(g);
            return st;
        }
        if (e != cudaSuccess) return fail(MFC_ECUDA, "graph capture: %s", cudaGetErrorString(e));
        const cudaError_t ei = cudaGraphInstantiate(&c->graph, g, 0);
        cudaGraphDestroy(g);
        if (ei != cudaSuccess) return fail(MFC_ECUDA, "graph instantiate: %s", cudaGetErrorString(ei));
        c->graph_q = q;
        c->graph_dt = dt;
        c->graph_phase = phase;
        c->graph_launches = c->launches;
        // the capture advanced the host-side operation counters by one step; undo it,
        // every launch below accounts for its own step
        if (c->peer_sync) {
            c->epoch -= 3;
            c->waited -= 3;
        }
    }
    for (int64_t i = 0; i < nsteps; ++i) {
        CU_TRY(cudaGraphLaunch(c->graph, s));
        if (c->peer_sync) {          // the replayed step's three operations
            c->epoch += 3;
            c->waited += 3;
        }
    }
    c->launches = c->graph_launches * nsteps;
    return MFC_OK;
}

int mfc_advance_host(mfc_ctx* c, const double* q_in, double* q_out, double* q_dev,
                     int64_t nsteps, double dt, void* stream) {
    NvtxRange nv("mfc_advance_host");
    if (!c || !q_in || !q_out) return fail(MFC_EINVAL, "NULL argument");
    if (nsteps < 0) return fail(MFC_EINVAL, "nsteps < 0");
    int st;
    if ((st = check_ptr(q_dev, "q_dev")) || (st = set_device(c))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (nsteps == 1) {
        const int64_t cz = stream_cz(c);
        if (cz > 0) {
            c->launches = 0;
            return advance_streamed(c, q_in, q_out, q_dev, dt, cz, s);
        }
    }
    const size_t row = (size_t)c->nl[0] * sizeof(double);
    const size_t pitch = (size_t)c->stride[2] * sizeof(double);
    auto copy = [&](bool h2d) -> int {
        for (int e = 0; e < c->E; ++e) {
            cudaMemcpy3DParms p = {};
            double* dev = q_dev + c->offset + e * c->stride[0];
            double* host = (double*)(h2d ? q_in : q_out) + (size_t)e * c->nl[0] * c->nl[1] * c->nl[2];
            cudaPitchedPtr hp = make_cudaPitchedPtr(host, row, c->nl[0], c->nl[1]);
            cudaPitchedPtr dp = make_cudaPitchedPtr(dev, pitch, c->nl[0], c->dims[2]);
            p.srcPtr = h2d ? hp : dp;
            p.dstPtr = h2d ? dp : hp;
            p.extent = make_cudaExtent(row, c->nl[1], c->nl[2]);
            p.kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
            CU_TRY(cudaMemcpy3DAsync(&p, s));
        }
        return MFC_OK;
    };
    if ((st = copy(true))) return st;
    // fused halo: the ghost layers of a freshly written state come from one exchange
    if (c->fused && (st = exchange(&c, &q_dev, 1, s))) return st;
    if ((st = mfc_rk3_steps(c, q_dev, dt, nsteps, stream))) return st;
    if ((st = copy(false))) return st;
    CU_TRY(cudaStreamSynchronize(s));
    return MFC_OK;
}

int mfc_halo_exchange_group(mfc_ctx* const* cs, double* const* qs, int32_t count, void* stream) {
    NvtxRange nv("mfc_halo_exchange_group");
    if (!cs || !qs || count < 1) return fail(MFC_EINVAL, "bad group");
    int st = set_device(cs[0]);
    if (st) return st;
    for (int r = 0; r < count; ++r) cs[r]->launches = 0;
    return exchange(cs, qs, count, (cudaStream_t)stream);
}

int mfc_rhs_group(mfc_ctx* const* cs, double* const* qs, double* const* rhss, int32_t count,
                  void* stream) {
    NvtxRange nv("mfc_rhs_group");
    if (!cs || !qs || !rhss || count < 1) return fail(MFC_EINVAL, "bad group");
    int st = set_device(cs[0]);
    if (st) return st;
    return rhs_group(cs, qs, rhss, count, (cudaStream_t)stream);
}

int mfc_rk3_step_group(mfc_ctx* const* cs, double* const* qs, int32_t count, double dt,
                       void* stream) {
    NvtxRange nv("mfc_rk3_step_group");
    if (!cs || !qs || count < 1) return fail(MFC_EINVAL, "bad group");
    int st = set_device(cs[0]);
    if (st) return st;
    return rk3_group(cs, qs, count, dt, (cudaStream_t)stream);
}

int mfc_fused_halo_group(mfc_ctx* const* cs, double* const* qs, int32_t count) {
    if (!cs || !qs || count < 1) return fail(MFC_EINVAL, "bad group");
    for (int r = 0; r < count; ++r) {
        int st;
        if (!cs[r]) return fail(MFC_EINVAL, "NULL ctx");
        if ((st = need_ws(cs[r], true)) || (st = check_ptr(qs[r], "q"))) return st;
        if ((cs[r]->transport != MFC_TRANSPORT_LOOPBACK && count > 1) ||
            cs[r]->transport == MFC_TRANSPORT_NCCL_SELF)
            return fail(MFC_EINVAL, "fused group needs loopback contexts");
    }
    for (int r = 0; r < count; ++r) {
        mfc_ctx* c = cs[r];
        for (int f = 0; f < 2 * c->D; ++f) {
            if (c->bc[f] != BC_NEIGHBOR) continue;
            const int o = c->nbr[f];
            if (o < 0 || o >= count) return fail(MFC_EINVAL, "group lacks rank %d", o);
            const mfc_ctx* n = cs[o];
            for (int k = 0; k < 3; ++k)
                if (k != f / 2 && n->nl[k] != c->nl[k])
                    return fail(MFC_EINVAL, "neighbour extents do not match across face %d", f);
            const Lay L = layout_for(n->D, n->E, n->nl);
            c->pf[f][0] = make_peer_face(c, f, qs[o], L, n->nl);
            c->pf[f][1] = make_peer_face(c, f, n->S1, L, n->nl);
            c->pf[f][2] = make_peer_face(c, f, n->S2, L, n->nl);
            c->pf_set[f] = true;
        }
        c->fused_q = qs[r];
        c->fused = true;
        c->peer_sync = false;
    }
    return MFC_OK;
}

int mfc_peer_export(mfc_ctx* c, double* q, void* blob) {
    if (!c || !blob) return fail(MFC_EINVAL, "NULL argument");
    if (c->transport == MFC_TRANSPORT_LOOPBACK)
        return fail(MFC_EINVAL, "loopback contexts attach with mfc_fused_halo_group");
    if (c->nranks < 2) return fail(MFC_EINVAL, "a single-rank context has no peers");
    int st;
    if ((st = need_ws(c, true)) || (st = check_ptr(q, "q")) || (st = set_device(c))) return st;
    if ((st = drv("cuDeviceGet", &p_dev_get)) || (st = drv("cuDeviceGetAttribute", &p_dev_attr)) ||
        (st = drv("cuMemGetAddressRange", &p_addr_range)) ||
        (st = drv("cuStreamWaitValue64", &p_wait_value)) ||
        (st = drv("cuStreamWriteValue64", &p_write_value)))
        return st;
    CUdevice dev;
    int memops = 0;
    if (p_dev_get(&dev, c->device) != CUDA_SUCCESS ||
        p_dev_attr(&memops, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, dev) != CUDA_SUCCESS)
        return fail(MFC_ECUDA, "cuDeviceGetAttribute failed");
    if (!memops) return fail(MFC_EUNSUPPORTED, "device lacks 64-bit stream memory operations");
    if (!c->flags) {                 // 6 faces x 3 slots (see peer_wait)
        CU_TRY(cudaMalloc(&c->flags, 18 * sizeof(uint64_t)));
        CU_TRY(cudaMemset(c->flags, 0, 18 * sizeof(uint64_t)));
    }
    PeerBlob b{};
    b.magic = kPeerMagic;
    b.rank = c->rank;
    b.E = c->E;
    b.D = c->D;
    for (int k = 0; k < 3; ++k) b.nl[k] = c->nl[k];
    const void* ptrs[4] = {q, c->S1, c->S2, c->flags};
    for (int i = 0; i < 4; ++i) {
        CUdeviceptr base = 0;
        size_t size = 0;
        if (p_addr_range(&base, &size, (CUdeviceptr)ptrs[i]) != CUDA_SUCCESS)
            return fail(MFC_ECUDA, "cuMemGetAddressRange failed for buffer %d", i);
        CU_TRY(cudaIpcGetMemHandle(&b.h[i], (void*)base));
        b.off[i] = (int64_t)((CUdeviceptr)ptrs[i] - base);
    }
    memcpy(blob, &b, sizeof b);
    c->fused_q = q;
    CU_TRY(cudaDeviceSynchronize());   // flags are zero before any neighbour signals
    return MFC_OK;
}

int mfc_peer_import(mfc_ctx* c, int32_t face, const void* blob) {
    if (!c || !blob) return fail(MFC_EINVAL, "NULL argument");
    if (face < 0 || face >= 2 * c->D || c->bc[face] != BC_NEIGHBOR)
        return fail(MFC_EINVAL, "face %d has no neighbour rank", face);
    if (!c->fused_q || !c->flags) return fail(MFC_ESTATE, "call mfc_peer_export first");
    int st;
    if ((st = set_device(c))) return st;
    PeerBlob b;
    memcpy(&b, blob, sizeof b);
    if (b.magic != kPeerMagic) return fail(MFC_EINVAL, "not an mfc_peer_export blob");
    if (b.rank != c->nbr[face])
        return fail(MFC_EINVAL, "blob of rank %d, face %d needs rank %d", b.rank, face, c->nbr[face]);
    if (b.E != c->E || b.D != c->D) return fail(MFC_EINVAL, "neighbour has another model");
    for (int k = 0; k < 3; ++k)
        if (k != face / 2 && b.nl[k] != c->nl[k])
            return fail(MFC_EINVAL, "neighbour extents do not match across face %d", face);
    char* base[4];
    for (int i = 0; i < 4; ++i) {
        void* p = nullptr;
        if ((st = ipc_open(b.h[i], &p))) return st;
        c->ipc_maps.push_back(p);
        base[i] = (char*)p + b.off[i];
    }
    const Lay L = layout_for(b.D, b.E, b.nl);
    for (int i = 0; i < 3; ++i) c->pf[face][i] = make_peer_face(c, face, (double*)base[i], L, b.nl);
    c->peer_flag[face] = (CUdeviceptr)((uint64_t*)base[3] + 3 * (face ^ 1));
    c->pf_set[face] = true;
    bool all = true;
    for (int f = 0; f < 2 * c->D; ++f)
        if (c->bc[f] == BC_NEIGHBOR && !c->pf_set[f]) all = false;
    if (all) {
        c->fused = true;
        c->peer_sync = true;
        c->epoch = 0;
        c->waited = 0;
    }
    return MFC_OK;
}

int64_t mfc_last_launch_count(const mfc_ctx* c) { return c ? c->launches : -1; }

int mfc_nccl_get_unique_id(void* out128) {
    if (!out128) return fail(MFC_EINVAL, "NULL argument");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out128, &id, sizeof id);
    return MFC_OK;
}

int mfc_profile_enable(mfc_ctx* c, int32_t on) {
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    c->prof = on != 0;
    c->recs.clear();
    c->ev_used = 0;
    return MFC_OK;
}

int mfc_profile_read(mfc_ctx* c, double* ms, int64_t* count, int32_t nkinds) {
    if (!c || !ms || !count || nkinds < 1) return fail(MFC_EINVAL, "bad argument");
    for (int k = 0; k < nkinds; ++k) { ms[k] = 0.0; count[k] = 0; }
    for (const auto& r : c->recs) {
        CU_TRY(cudaEventSynchronize(r.b));
        float t = 0.f;
        CU_TRY(cudaEventElapsedTime(&t, r.a, r.b));
        if (r.kind < nkinds) { ms[r.kind] += t; count[r.kind] += 1; }
    }
    c->recs.clear();
    c->ev_used = 0;
    return MFC_OK;
}

int mfc_comm_status(mfc_ctx* c) {
    if (!c) return fail(MFC_EINVAL, "NULL ctx");
    return comm_async_error(c);
}

int mfc_finalize(mfc_ctx* c) {
    if (!c) return MFC_OK;
    for (void* p : c->ipc_maps) ipc_release(p);
    if (c->flags) cudaFree(c->flags);
    if (c->graph) cudaGraphExecDestroy(c->graph);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->ev_ready) cudaEventDestroy(c->ev_ready);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->comm) {
        // a communicator with an asynchronous error may never finish its pending work:
        // abort it instead of waiting in ncclCommDestroy
        ncclResult_t ar = ncclSuccess;
        if (!c->comm_failed && ncclCommGetAsyncError(c->comm, &ar) == ncclSuccess &&
            (ar == ncclSuccess || ar == ncclInProgress))
            ncclCommDestroy(c->comm);
        else
            ncclCommAbort(c->comm);
    }
    for (auto e : c->ev_piece) cudaEventDestroy(e);
    for (auto e : c->ev_comp) cudaEventDestroy(e);
    for (auto e : c->ev_out) cudaEventDestroy(e);
    for (auto e : c->ev_scat) cudaEventDestroy(e);
    if (c->ev_start) cudaEventDestroy(c->ev_start);
    for (auto e : c->ev_s1) cudaEventDestroy(e);
    if (c->st_in) cudaStreamDestroy(c->st_in);
    if (c->st_out) cudaStreamDestroy(c->st_out);
    if (c->st_s1) cudaStreamDestroy(c->st_s1);
    delete c;
    return MFC_OK;
}

}  // extern "C"
