// efem_internal.cuh -- shared internals of libefem.so (product path only).
// Nothing here is shared with oracle/; the two implementations are
// independent.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/efem.h"

namespace efem {

// ---- flags written by kernels (workspace header) ---------------------------
enum : int {
    F_INVALID_NODE = 0,  // element references a node id outside [0, n_nodes)
    F_CAPACITY = 1,      // a per-thread list overflowed
    F_ROW_MISMATCH = 2,  // numeric row length != symbolic row length (internal error)
    F_DEGENERATE = 3,    // det B_K == 0 or non-finite
    F_FAN_OVER = 4,      // (internal, not an error) a node fan overflowed the fixed-capacity fill (fan2d.cu)
    F_NFLAGS = 8
};

struct WsHeader {
    int flags[F_NFLAGS];
    unsigned long long bad_element;  // atomicMin of the first degenerate element
    long long totals[2];             // n_dofs, nnz (read back with the flags in one copy)
    long long pad;
    // row window of a bound partition (efem_part_*_async), written on the
    // device: first local row, rows, local CSR offset of the first row,
    // entries, global id of the first row
    long long win[6];
    int fan_big;      // the last fan pass saw a node fan of > FAN_SMALL triangles (fan2d.cu)
};

// Instance words e << 3 | k (element e < 2^27, local entity k); the two top
// bits of bucket words carry run / boundary flags (dofs.cu).
constexpr int INST_MASK = 0x3fffffff;

// ---- element kinds ------------------------------------------------------------
// Local numbering follows PAPER.md Fig. 1 (lines 54-157), 0-based:
//   2D edges (start->end): e0 = 1->2, e1 = 2->0, e2 = 0->1  (edge k opposite vertex k)
//   3D edges: e0 = 0->1, e1 = 0->2, e2 = 0->3, e3 = 1->2, e4 = 2->3, e5 = 3->1
//   3D faces: f_k = all vertices but vertex 3-k  ({0,1,2},{0,1,3},{0,2,3},{1,2,3})
template <int DIM, int ELEM>
struct Kind {
    static constexpr int D = DIM;
    static constexpr int NV = DIM + 1;
    static constexpr bool FACES = (DIM == 3 && ELEM == EFEM_RT0);
    static constexpr int M = DIM == 2 ? 3 : (ELEM == EFEM_RT0 ? 4 : 6);
    static constexpr int EK = FACES ? 3 : 2;  // nodes per entity
    static constexpr int ELEMENT = ELEM;
};

__host__ __device__ constexpr int edge_start(int dim, int k) {
    return dim == 2 ? (k == 0 ? 1 : k == 1 ? 2 : 0)
                    : (k == 0 ? 0 : k == 1 ? 0 : k == 2 ? 0 : k == 3 ? 1 : k == 4 ? 2 : 3);
}
__host__ __device__ constexpr int edge_end(int dim, int k) {
    return dim == 2 ? (k == 0 ? 2 : k == 1 ? 0 : 1)
                    : (k == 0 ? 1 : k == 1 ? 2 : k == 2 ? 3 : k == 3 ? 2 : k == 4 ? 3 : 1);
}

// ---- host-side plan -------------------------------------------------------------
struct Plan {
    int dim = 0, element = 0, m = 0, nv = 0, ek = 0;
    int64_t n_nodes = 0, n_elems = 0;
    const double* coords = nullptr;
    const int32_t* elems = nullptr;
    int64_t r_max = 0;  // upper bound of n_dofs (n_elems * m)

    // workspace
    char* ws = nullptr;
    size_t ws_bytes = 0, ws_need = 0;
    WsHeader* hdr = nullptr;
    int32_t* cnt = nullptr;         // N+1 instances per minimum node (counting sort; zero between calls)
    int32_t* ent_cnt = nullptr;     // N+1 entities per node
    int32_t* bucket_ptr = nullptr;  // N+1
    int32_t* bucket = nullptr;      // T*m instances (e << 3 | k); after enumeration sorted by
                                    // (entity, element): the entity -> element incidence
    uint64_t* bkey = nullptr;       // T*m bucket sort keys (filled by k_bucket<fill>)
    int32_t* binst = nullptr;       // T*m instance words (3D faces only)
    int32_t* bx = nullptr;          // T*m xor of the tet's vertices (3D edges only)
    int32_t* nbr = nullptr;         // r_max larger endpoint of each edge (3D edges only)
    int32_t* e2d = nullptr;         // T*m elems2dofs
    int32_t* inc_ptr = nullptr;     // r_max+1 entity -> first incidence in bucket
    int32_t* row_ptr = nullptr;     // r_max+1 CSR row offsets (3D edges only; others: closed form)
    int2* rec = nullptr;            // r_max row records {first, last instance} (2D edges, 3D faces)
    int32_t* d2n = nullptr;         // r_max*ek (written only when want_d2n)
    int32_t* ent_ptr = nullptr;     // N+1 first DOF id of each node's entities
    int32_t* nnz_cnt = nullptr;     // N+1 CSR entries of each node's rows
    int32_t *ent_bsum = nullptr, *ent_bpre = nullptr, *nnz_bsum = nullptr, *nnz_bpre = nullptr;  // per node tile
    int64_t* d_totals = nullptr;    // == hdr->totals
    // 2D node-fan pipeline (fan2d.cu): fans of the triangles by smallest /
    // middle vertex; it writes rec / inc_ptr / e2d above for k_rows_tri
    int32_t* fan_ptr = nullptr;      // N+1
    int32_t* fan = nullptr;          // 2T triangle ids
    unsigned long long* fan_tiles = nullptr;  // look-back tile states
    int32_t* fan_fix = nullptr;      // N * FAN_FIXC: fixed-capacity fans (one-pass fill)
    int32_t* fan_csum = nullptr;     // tile sums of the fallback scan of the fan counts
    int32_t* ne3_fan = nullptr;      // NE0 3D: N * 24 fixed-capacity tet fans (dofs.cu k_fill_fan3)
    int32_t* ne3_fcnt = nullptr;     // their counts
    // owned node range of a distributed plan (dist2d.cu): the fan pipeline
    // builds rows only for nodes [own_lo, own_lo + own_n); own_n < 0: all
    int64_t own_lo = 0, own_n = -1;
    int32_t* node_ent = nullptr;     // optional: first row of each owned node (dist2d.cu)
    bool fan_valid = false;          // rec / inc_ptr / e2d are current from the fan pipeline
    bool fan_small = false;          // the last read-back saw no fan above FAN_SMALL (fan2d.cu kernel choice)
    bool want_d2n = false;
    bool exact_ne3 = false;  // NE0 3D: exact link counts (non-manifold meshes), efem_plan_set_exact
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;

    // host pinned readback
    int64_t* h_scalars = nullptr;  // [0] n_dofs [1] nnz
    WsHeader* h_hdr = nullptr;

    // CUDA graph of the enumeration sequence (captured once on an internal
    // stream; replayed with event handshakes against the caller's stream)
    cudaStream_t gstream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaGraphExec_t g_enum = nullptr;
    bool graph_failed = false;
    int64_t graph_launches = 0;
    // efem_assemble_async as one graph (enumeration + row kernel), keyed by
    // the output arrays / capacities / forms it was captured for
    cudaGraphExec_t g_async = nullptr;
    int64_t async_launches = 0;
    efem_csr async_key{};
    unsigned async_forms = 0;

    // bound partition (efem_part_bind): the rank's node range [part_lo,
    // part_hi) and its local node range [part_l0, part_l1) in this sub-mesh
    bool part_bound = false;
    int64_t part_lo = 0, part_hi = 0, part_l0 = 0, part_l1 = 0;
    const int32_t* part_sub2global = nullptr;
    cudaGraphExec_t g_part = nullptr;  // enumeration + owned counts + window
    int64_t part_launches = 0;
    int32_t* part_key = nullptr;

    // state: enumerated = the bucket-pipeline arrays (dofs.cu: incidence,
    // elems2dofs, ...) are current; symbolic = n_dofs / nnz are known
    bool enumerated = false, symbolic = false;
    bool async_pending = false;  // efem_assemble_async ran; sizes arrive with efem_plan_check
    bool async_fan = false;      // ... through the 2D node-fan pipeline (else the bucket pipeline)
    int64_t n_dofs = 0, nnz = 0;
};

// Ghost triangles of a distributed 2D assembly (dist2d.cu, assemble.cu
// GhostDeepPolicy): local triangle index e >= base is a ghost, its row values
// at vals[(e - base) * 12 + 4 k ..]; columns are elems2dofs + col_base (with
// a device row window: col_base = the window's global first row).
struct GhostArgs {
    const double* vals = nullptr;
    int base = 0x7fffffff;
    int col_base = 0;
};

// Rows [row0, row0 + n_rows) of a plan, written to a CSR whose entry 0 is the
// plan's entry row_ptr[row0] = out_base; own DOF of local row i is
// own_base + i; column ids from e2d (local or globalised).
struct RowWindow {
    int64_t row0 = 0, n_rows = 0;
    int own_base = 0, out_base = 0;
    const int32_t* e2d = nullptr;
    // asynchronous assembly: n_rows / nnz are read on the device from the
    // header totals; n_rows, cap_nnz above are then the output capacities
    bool dyn = false;
    int64_t cap_nnz = 0;
    // bound partition, asynchronous: row0 / n_rows / out_base / own_base come
    // from this device window (WsHeader::win); n_rows, cap_nnz are capacities
    const long long* win = nullptr;
    // distributed 2D assembly: ghost triangles (GhostDeepPolicy)
    bool ghost = false;
    GhostArgs gh;
};

// ---- error plumbing --------------------------------------------------------------
void set_error(const std::string& msg);
void set_bad_element(int64_t e);
void count_launch(int n = 1);

#define EFEM_CUDA_TRY(expr)                                                          \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess) {                                                     \
            ::efem::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));   \
            return EFEM_ECUDA;                                                       \
        }                                                                            \
    } while (0)

// EFEM_DEBUG_SYNC=1 in the environment: synchronise after every launch and
// report the failing launch site (debugging aid; off by default, graphs off).
bool debug_sync();

#define EFEM_LAUNCH_CHECK()                                                          \
    do {                                                                             \
        ::efem::count_launch();                                                      \
        cudaError_t _e = cudaGetLastError();                                         \
        if (_e == cudaSuccess && ::efem::debug_sync()) _e = cudaDeviceSynchronize();  \
        if (_e != cudaSuccess) {                                                     \
            ::efem::set_error(std::string("kernel launch (") + __FILE__ + ":" +       \
                              std::to_string(__LINE__) + "): " + cudaGetErrorString(_e)); \
            return EFEM_ECUDA;                                                       \
        }                                                                            \
    } while (0)

// kernel-launch entry points (defined in the .cu files)
efem_status launch_build_mesh(int dim, int n, double alpha, uint64_t seed, double* coords, int32_t* elems,
                              cudaStream_t s);
efem_status run_enumerate(Plan& p, cudaStream_t s);
efem_status run_symbolic(Plan& p, cudaStream_t s);
efem_status run_numeric(Plan& p, unsigned forms, efem_csr* out, cudaStream_t s);
efem_status run_signs(Plan& p, cudaStream_t s);
// the bucket-pipeline arrays for the consumers that need them (DOF tables,
// loads, field errors, partitions): enumerates if they are not current
efem_status ensure_enumerated(Plan& p, cudaStream_t s);
// 2D node-fan pipeline (fan2d.cu)
inline bool uses_fan(const Plan& p) { return p.dim == 2; }
efem_status launch_fan_symbolic(Plan& p, cudaStream_t s, bool reset = true);
efem_status launch_hdr_reset(Plan& p, cudaStream_t s);
size_t fan_tiles_bytes(int64_t n_nodes);
constexpr int FAN_FIXC = 8;  // largest fixed fan capacity (fan2d.cu)
// row_ptr helpers (api.cu): 2D edges / 3D faces keep no row_ptr array, row r
// starts at r + (m-1) inc_ptr[r]; 3D edges store it (plan row_ptr).
bool row_ptr_stored(const Plan& p);
efem_status write_row_ptr(Plan& p, int64_t r0, int64_t n, int32_t* out, cudaStream_t s);
efem_status row_start_host(Plan& p, int64_t r, int64_t* start, cudaStream_t s);

inline unsigned grid_for(int64_t n, int tpb) { return (unsigned)((n + tpb - 1) / tpb); }

}  // namespace efem
