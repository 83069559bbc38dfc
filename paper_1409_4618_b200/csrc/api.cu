// api.cu -- the C-ABI of include/efem.h: plans, workspace layout, the
// enumerate -> symbolic -> numeric pipeline, status plumbing.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "efem_internal.cuh"

namespace efem {

// launchers defined in dofs.cu / assemble.cu
efem_status launch_enumerate(Plan& p, cudaStream_t s);
efem_status launch_signs(Plan& p, int8_t* out, cudaStream_t s);
efem_status launch_rows_any(Plan& p, unsigned forms, efem_csr* out, const RowWindow& w, cudaStream_t s);
efem_status launch_build_lshape(int m, double alpha, uint64_t seed, double* coords, int32_t* elems, cudaStream_t s);
// integrate.cu (f1 / f2)
int quad6_size(int dim);
efem_status launch_quad_points(int dim, const double* coords, const int32_t* elems, int64_t n_elems, double* pts,
                               cudaStream_t s);
efem_status launch_load(Plan& p, int pairing, const double* fq, double* b, cudaStream_t s);
size_t reduce_ws_bytes();
efem_status launch_norm_l2(int dim, const double* coords, const int32_t* elems, int64_t n_elems, const double* fq,
                           int nf, double* per_elem, double* total, double* part, cudaStream_t s);
efem_status launch_field_error(Plan& p, const double* coeffs, const double* Eq, const double* Dq, double* err2,
                               double* scratch, cudaStream_t s);
efem_status launch_spmv(const efem_csr* A, double alpha, double beta, const double* x, double* y, cudaStream_t s);
size_t cg_ws_bytes(int64_t n);
efem_status run_cg(const efem_csr* A, double alpha, double beta, const double* b, double* x, double rtol, int maxit,
                   int* iters, double* relres, void* ws, cudaStream_t s);

namespace {
thread_local std::string g_last_error;
thread_local int64_t g_bad_element = -1;
std::atomic<int64_t> g_launches{0};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
    size_t hdr, cnt, ent_cnt, bucket_ptr, bucket, bkey, binst, bx, nbr, e2d, inc_ptr, row_ptr, rec, d2n, ent_ptr, nnz_cnt, tiles, totals, cub, total;
    size_t fan_ptr, fan, fan_tiles, fan_fix, fan_csum, ne3_fan, ne3_fcnt;
};

Layout layout(const Plan& p, size_t cub_bytes) {
    Layout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += align256(bytes);
        return o;
    };
    const size_t N1 = (size_t)p.n_nodes + 1;
    const size_t Tm = (size_t)p.n_elems * p.m;
    L.hdr = take(sizeof(WsHeader));
    L.cnt = take(N1 * 4);
    L.ent_cnt = take(N1 * 4);
    L.bucket_ptr = take(N1 * 4);
    L.bucket = take(Tm * 4);
    const bool faces = p.dim == 3 && p.element == EFEM_RT0;
    L.bkey = take(Tm * (p.dim == 3 ? 16 : 8));  // 3D: 16-byte {key, aux} records
    L.binst = take(4);
    L.bx = take(p.dim == 3 && !faces ? Tm * 4 : 4);
    L.nbr = take(p.dim == 3 && !faces ? (size_t)p.r_max * 4 : 4);
    L.e2d = take(Tm * 4);
    L.inc_ptr = take(((size_t)p.r_max + 1) * 4);
    const bool ne3 = p.dim == 3 && p.element == EFEM_NED0;
    L.row_ptr = take(ne3 ? ((size_t)p.r_max + 1) * 4 : 4);
    L.rec = take(ne3 ? 8 : (size_t)p.r_max * 8);
    L.d2n = take((size_t)p.r_max * p.ek * 4);
    L.ent_ptr = take(N1 * 4);
    L.nnz_cnt = take(N1 * 4);
    L.tiles = take(4 * ((size_t)p.n_nodes / 64 + 4) * 4);  // ent / nnz tile sums and prefixes
    L.totals = take(16);
    L.cub = take(cub_bytes);
    const bool fan = uses_fan(p);
    L.fan_ptr = take(fan ? N1 * 4 : 4);
    L.fan = take(fan ? (size_t)p.n_elems * 2 * 4 : 4);
    L.fan_tiles = take(fan ? fan_tiles_bytes(p.n_nodes) : 8);
    L.fan_fix = take(fan ? (size_t)p.n_nodes * FAN_FIXC * 4 : 4);
    L.fan_csum = take(fan ? ((size_t)p.n_nodes / 2048 + 2) * 4 : 4);
    L.ne3_fan = take(ne3 ? (size_t)p.n_nodes * 24 * 4 : 4);  // (NE3_FAN_C, dofs.cu)
    L.ne3_fcnt = take(ne3 ? (size_t)p.n_nodes * 4 : 4);
    L.total = off;
    return L;
}

efem_status flags_status(const Plan& p) {
    const WsHeader& h = *p.h_hdr;
    if (h.flags[F_INVALID_NODE]) {
        set_error("an element references a node id outside [0, n_nodes)");
        return EFEM_EINVAL;
    }
    if (h.flags[F_DEGENERATE]) {
        set_bad_element((int64_t)h.bad_element);
        set_error("degenerate element (det B_K == 0 or non-finite): " + std::to_string(h.bad_element));
        return EFEM_EDEGENERATE;
    }
    if (h.flags[F_CAPACITY]) {
        set_error("capacity exceeded: an output smaller than the assembled pattern (efem_assemble_async / "
                  "efem_part_numeric_async), or a node too irregular for the per-thread limits");
        return EFEM_ECAPACITY;
    }
    if (h.flags[F_ROW_MISMATCH]) {
        set_error("row structure differs from the closed-form row length: the mesh is not conforming "
                  "(duplicate elements, or an entity shared by more elements than a conforming mesh allows), "
                  "or (NE0 3D) an edge whose tets do not form one fan -- efem_plan_set_exact(plan, 1) "
                  "sizes such rows exactly");
        return EFEM_EINVAL;
    }
    return EFEM_OK;
}

efem_status read_flags(Plan& p, cudaStream_t s) {
    EFEM_CUDA_TRY(cudaMemcpyAsync(p.h_hdr, p.hdr, sizeof(WsHeader), cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    if (uses_fan(p)) p.fan_small = p.h_hdr->fan_big == 0;  // (a performance hint only)
    return flags_status(p);
}

// Enumeration = ~10 dependent launches + one D2H of the header; replayed as a
// CUDA graph (captured once on the plan's internal stream, handshaking with
// the caller's stream through events) to cut the launch gaps.
efem_status enumerate_graph(Plan& p, cudaStream_t s, bool* used, bool sync = true) {
    *used = false;
    if (p.graph_failed || p.want_d2n || debug_sync()) return EFEM_OK;
    if (!p.g_enum) {
        if (!p.gstream) {
            if (cudaStreamCreateWithFlags(&p.gstream, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&p.ev_in, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&p.ev_out, cudaEventDisableTiming) != cudaSuccess) {
                p.graph_failed = true;
                cudaGetLastError();
                return EFEM_OK;
            }
        }
        cudaGraph_t graph = nullptr;
        if (cudaStreamBeginCapture(p.gstream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            p.graph_failed = true;
            cudaGetLastError();
            return EFEM_OK;
        }
        const int64_t l0 = g_launches.load();
        efem_status st = launch_enumerate(p, p.gstream);
        const cudaError_t ce = cudaMemcpyAsync(p.h_hdr, p.hdr, sizeof(WsHeader), cudaMemcpyDeviceToHost, p.gstream);
        const cudaError_t ee = cudaStreamEndCapture(p.gstream, &graph);
        p.graph_launches = g_launches.load() - l0;
        g_launches.fetch_sub(p.graph_launches);  // counted when the graph replays
        if (st != EFEM_OK || ce != cudaSuccess || ee != cudaSuccess ||
            cudaGraphInstantiate(&p.g_enum, graph, 0) != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            p.g_enum = nullptr;
            p.graph_failed = true;
            cudaGetLastError();
            return EFEM_OK;
        }
        cudaGraphDestroy(graph);
    }
    EFEM_CUDA_TRY(cudaEventRecord(p.ev_in, s));
    EFEM_CUDA_TRY(cudaStreamWaitEvent(p.gstream, p.ev_in, 0));
    EFEM_CUDA_TRY(cudaGraphLaunch(p.g_enum, p.gstream));
    count_launch((int)p.graph_launches);
    EFEM_CUDA_TRY(cudaEventRecord(p.ev_out, p.gstream));
    EFEM_CUDA_TRY(cudaStreamWaitEvent(s, p.ev_out, 0));
    if (sync) EFEM_CUDA_TRY(cudaStreamSynchronize(p.gstream));
    *used = true;
    return EFEM_OK;
}

// row_ptr of rows [r0, r0 + n] (n + 1 entries), relative to row r0's start.
// 2D edges / 3D faces: closed form r + (m-1) inc_ptr[r]; 3D edges: stored.
__global__ void k_row_ptr(const int32_t* __restrict__ inc_ptr, const int32_t* __restrict__ row_ptr, int64_t r0,
                          int64_t n, int c, int32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    const int64_t r = r0 + i;
    const int64_t v = row_ptr ? (int64_t)row_ptr[r] - row_ptr[r0]
                              : (r + (int64_t)c * inc_ptr[r]) - (r0 + (int64_t)c * inc_ptr[r0]);
    out[i] = (int32_t)v;
}

}  // namespace

bool row_ptr_stored(const Plan& p) { return p.dim == 3 && p.element == EFEM_NED0; }

efem_status write_row_ptr(Plan& p, int64_t r0, int64_t n, int32_t* out, cudaStream_t s) {
    k_row_ptr<<<grid_for(n + 1, 256), 256, 0, s>>>(p.inc_ptr, row_ptr_stored(p) ? p.row_ptr : nullptr, r0, n, p.m - 1,
                                                   out);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status row_start_host(Plan& p, int64_t r, int64_t* start, cudaStream_t s) {
    int32_t v = 0;
    EFEM_CUDA_TRY(cudaMemcpyAsync(&v, (row_ptr_stored(p) ? p.row_ptr : p.inc_ptr) + r, 4, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    *start = row_ptr_stored(p) ? (int64_t)v : r + (int64_t)(p.m - 1) * v;
    return EFEM_OK;
}

void set_error(const std::string& msg) { g_last_error = msg; }
bool debug_sync() {
    static const bool on = [] {
        const char* v = std::getenv("EFEM_DEBUG_SYNC");
        return v && v[0] && v[0] != '0';
    }();
    return on;
}
void set_bad_element(int64_t e) { g_bad_element = e; }
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ------------------------------------------------------------------------------------
efem_status run_enumerate(Plan& p, cudaStream_t s) {
    efem_status st;
    bool used = false;
    if ((st = enumerate_graph(p, s, &used)) != EFEM_OK) return st;
    if (used) {
        st = flags_status(p);
    } else {
        if ((st = launch_enumerate(p, s)) != EFEM_OK) return st;  // resets the header itself
        st = read_flags(p, s);                                     // one D2H of flags + totals, synchronises
    }
    if (st != EFEM_OK) return st;
    p.n_dofs = p.h_hdr->totals[0];
    p.nnz = p.h_hdr->totals[1];
    p.enumerated = true;
    return EFEM_OK;
}

efem_status ensure_enumerated(Plan& p, cudaStream_t s) {
    return p.enumerated ? EFEM_OK : run_enumerate(p, s);
}

// 2D: the node-fan pipeline's symbolic half (fan2d.cu) and one read-back of
// the flags and sizes.  3D: the enumeration already yields the exact row
// lengths (closed-form counts, dofs.cu).
efem_status run_symbolic(Plan& p, cudaStream_t s) {
    efem_status st;
    if (uses_fan(p)) {
        if ((st = launch_fan_symbolic(p, s)) != EFEM_OK) return st;
        if ((st = read_flags(p, s)) != EFEM_OK) return st;
        p.n_dofs = p.h_hdr->totals[0];
        p.nnz = p.h_hdr->totals[1];
        p.fan_valid = true;
    } else if (!p.enumerated) {
        if ((st = run_enumerate(p, s)) != EFEM_OK) return st;
    }
    p.symbolic = true;
    return EFEM_OK;
}

// The numeric row kernels write row_ptr themselves (EFEM_PATTERN).
efem_status run_numeric(Plan& p, unsigned forms, efem_csr* out, cudaStream_t s) {
    efem_status st;
    if (p.n_dofs == 0) {
        if (forms & EFEM_PATTERN) EFEM_CUDA_TRY(cudaMemsetAsync(out->row_ptr, 0, 4, s));
        return EFEM_OK;
    }
    if (uses_fan(p) && !p.fan_valid && !p.enumerated) {  // (either pipeline writes rec / inc_ptr / e2d)
        if ((st = launch_fan_symbolic(p, s)) != EFEM_OK) return st;
        p.fan_valid = true;
    }
    RowWindow w;
    w.row0 = 0;
    w.n_rows = p.n_dofs;
    w.own_base = 0;
    w.out_base = 0;
    w.e2d = p.e2d;
    if ((st = launch_rows_any(p, forms, out, w, s)) != EFEM_OK) return st;
    return EFEM_OK;
}

}  // namespace efem

using namespace efem;

extern "C" {

const char* efem_status_string(efem_status st) {
    switch (st) {
        case EFEM_OK: return "EFEM_OK";
        case EFEM_EINVAL: return "EFEM_EINVAL";
        case EFEM_EDEGENERATE: return "EFEM_EDEGENERATE";
        case EFEM_ENOMEM: return "EFEM_ENOMEM";
        case EFEM_EWORKSPACE: return "EFEM_EWORKSPACE";
        case EFEM_EOVERFLOW: return "EFEM_EOVERFLOW";
        case EFEM_ECUDA: return "EFEM_ECUDA";
        case EFEM_ENCCL: return "EFEM_ENCCL";
        case EFEM_ECAPACITY: return "EFEM_ECAPACITY";
        case EFEM_ESTATE: return "EFEM_ESTATE";
    }
    return "unknown efem_status";
}

const char* efem_last_error(void) { return g_last_error.c_str(); }
int64_t efem_last_bad_element(void) { return g_bad_element; }
int64_t efem_launch_count(void) { return g_launches.load(); }

efem_status efem_mesh_sizes(int dim, int n, int64_t* n_nodes, int64_t* n_elems) {
    if ((dim != 2 && dim != 3) || n < 1 || !n_nodes || !n_elems) {
        set_error("efem_mesh_sizes: dim must be 2 or 3, n >= 1, outputs non-NULL");
        return EFEM_EINVAL;
    }
    const int64_t n1 = (int64_t)n + 1;
    *n_nodes = dim == 2 ? n1 * n1 : n1 * n1 * n1;
    *n_elems = dim == 2 ? 2ll * n * n : 6ll * n * n * n;
    if (*n_elems * (dim + 1) >= (1ll << 31) || *n_nodes >= (1ll << 31)) {
        set_error("efem_mesh_sizes: mesh does not fit int32 indices");
        return EFEM_EOVERFLOW;
    }
    return EFEM_OK;
}

efem_status efem_build_mesh(int dim, int n, double jitter_frac, uint64_t seed, double* coords, int32_t* elems,
                            efem_stream_t stream) {
    int64_t N, T;
    efem_status st = efem_mesh_sizes(dim, n, &N, &T);
    if (st != EFEM_OK) return st;
    // interior jitter must keep every element valid: 2 alpha sqrt(d) < 1/sqrt(2)
    const double lim = 1.0 / (2.0 * std::sqrt(2.0 * dim));
    if (!coords || !elems || !(jitter_frac >= 0.0) || !(jitter_frac < lim)) {
        set_error("efem_build_mesh: NULL array or jitter_frac outside [0, 1/(2 sqrt(2 dim)))");
        return EFEM_EINVAL;
    }
    return launch_build_mesh(dim, n, jitter_frac, seed, coords, elems, (cudaStream_t)stream);
}

efem_status efem_lshape_sizes(int m, int64_t* n_nodes, int64_t* n_elems) {
    if (m < 2 || (m & 1) || !n_nodes || !n_elems) {
        set_error("efem_lshape_sizes: m must be even and >= 2, outputs non-NULL");
        return EFEM_EINVAL;
    }
    const int64_t h = m / 2;
    *n_nodes = (h + 1) * (m + 1) + (m - h) * (h + 1);
    *n_elems = 2 * (h * m + (m - h) * h);
    if (*n_elems * 3 >= (1ll << 31)) {
        set_error("efem_lshape_sizes: mesh does not fit int32 indices");
        return EFEM_EOVERFLOW;
    }
    return EFEM_OK;
}

efem_status efem_build_mesh_lshape(int m, double jitter_frac, uint64_t seed, double* coords, int32_t* elems,
                                   efem_stream_t stream) {
    int64_t N, T;
    efem_status st = efem_lshape_sizes(m, &N, &T);
    if (st != EFEM_OK) return st;
    const double lim = 1.0 / (2.0 * std::sqrt(2.0 * 2));
    if (!coords || !elems || !(jitter_frac >= 0.0) || !(jitter_frac < lim)) {
        set_error("efem_build_mesh_lshape: NULL array or jitter_frac outside [0, 1/(4 sqrt(2)))");
        return EFEM_EINVAL;
    }
    return launch_build_lshape(m, jitter_frac, seed, coords, elems, (cudaStream_t)stream);
}

efem_status efem_plan_create(efem_plan* plan, const efem_mesh* mesh, efem_element element, size_t* ws_bytes) {
    if (!plan || !mesh || !ws_bytes) {
        set_error("efem_plan_create: NULL argument");
        return EFEM_EINVAL;
    }
    if ((mesh->dim != 2 && mesh->dim != 3) || (element != EFEM_RT0 && element != EFEM_NED0) ||
        mesh->n_nodes < 0 || mesh->n_elems < 0 || (mesh->n_elems > 0 && (!mesh->coords || !mesh->elems))) {
        set_error("efem_plan_create: bad mesh (dim 2|3, element RT0|NED0, non-negative sizes, device arrays)");
        return EFEM_EINVAL;
    }
    if ((reinterpret_cast<uintptr_t>(mesh->elems) & 15) != 0 && mesh->dim == 3) {
        set_error("efem_plan_create: 3D elems must be 16-byte aligned (int4 loads)");
        return EFEM_EINVAL;
    }
    Plan* p = new (std::nothrow) Plan;
    if (!p) return EFEM_ENOMEM;
    p->dim = mesh->dim;
    p->element = element;
    p->nv = mesh->dim + 1;
    p->m = mesh->dim == 2 ? 3 : (element == EFEM_RT0 ? 4 : 6);
    p->ek = (mesh->dim == 3 && element == EFEM_RT0) ? 3 : 2;
    p->n_nodes = mesh->n_nodes;
    p->n_elems = mesh->n_elems;
    p->coords = mesh->coords;
    p->elems = mesh->elems;
    p->r_max = p->n_elems * p->m;
    const int64_t nnz_c = (p->dim == 3 && element == EFEM_NED0) ? 5 : p->m - 1;
    if (p->n_elems >= (1ll << 27) || p->n_nodes >= (1ll << 31) - 1 || p->r_max * p->ek >= (1ll << 31) ||
        p->r_max + nnz_c * p->n_elems * p->m >= (1ll << 31)) {
        delete p;
        set_error("efem_plan_create: mesh too large for int32 indexing (n_elems < 2^27)");
        return EFEM_EOVERFLOW;
    }
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (int)(p->n_nodes + 1));
    p->cub_bytes = cub_bytes;
    p->ws_need = layout(*p, cub_bytes).total;
    if (cudaMallocHost(&p->h_scalars, 64) != cudaSuccess || cudaMallocHost(&p->h_hdr, sizeof(WsHeader)) != cudaSuccess) {
        delete p;
        set_error("efem_plan_create: cudaMallocHost failed");
        return EFEM_ECUDA;
    }
    *ws_bytes = p->ws_need;
    *plan = reinterpret_cast<efem_plan>(p);
    return EFEM_OK;
}

efem_status efem_plan_set_workspace(efem_plan plan, void* ws, size_t ws_bytes) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p) return EFEM_EINVAL;
    if (!ws || ws_bytes < p->ws_need || (reinterpret_cast<uintptr_t>(ws) & 255)) {
        set_error("efem_plan_set_workspace: workspace NULL, too small or not 256-byte aligned");
        return EFEM_EWORKSPACE;
    }
    const Layout L = layout(*p, p->cub_bytes);
    char* b = static_cast<char*>(ws);
    p->ws = b;
    p->ws_bytes = ws_bytes;
    p->hdr = reinterpret_cast<WsHeader*>(b + L.hdr);
    p->cnt = reinterpret_cast<int32_t*>(b + L.cnt);
    p->ent_cnt = reinterpret_cast<int32_t*>(b + L.ent_cnt);
    p->bucket_ptr = reinterpret_cast<int32_t*>(b + L.bucket_ptr);
    p->bucket = reinterpret_cast<int32_t*>(b + L.bucket);
    p->bkey = reinterpret_cast<uint64_t*>(b + L.bkey);
    p->binst = reinterpret_cast<int32_t*>(b + L.binst);
    p->bx = reinterpret_cast<int32_t*>(b + L.bx);
    p->nbr = reinterpret_cast<int32_t*>(b + L.nbr);
    p->e2d = reinterpret_cast<int32_t*>(b + L.e2d);
    p->inc_ptr = reinterpret_cast<int32_t*>(b + L.inc_ptr);
    p->row_ptr = reinterpret_cast<int32_t*>(b + L.row_ptr);
    p->rec = reinterpret_cast<int2*>(b + L.rec);
    p->d2n = reinterpret_cast<int32_t*>(b + L.d2n);
    p->ent_ptr = reinterpret_cast<int32_t*>(b + L.ent_ptr);
    p->nnz_cnt = reinterpret_cast<int32_t*>(b + L.nnz_cnt);
    {
        const size_t nt = (size_t)p->n_nodes / 64 + 4;
        int32_t* tl = reinterpret_cast<int32_t*>(b + L.tiles);
        p->ent_bsum = tl;
        p->ent_bpre = tl + nt;
        p->nnz_bsum = tl + 2 * nt;
        p->nnz_bpre = tl + 3 * nt;
    }
    p->d_totals = reinterpret_cast<int64_t*>(&p->hdr->totals[0]);
    p->cub_tmp = b + L.cub;
    p->fan_ptr = reinterpret_cast<int32_t*>(b + L.fan_ptr);
    p->fan = reinterpret_cast<int32_t*>(b + L.fan);
    p->fan_tiles = reinterpret_cast<unsigned long long*>(b + L.fan_tiles);
    p->fan_fix = reinterpret_cast<int32_t*>(b + L.fan_fix);
    p->fan_csum = reinterpret_cast<int32_t*>(b + L.fan_csum);
    p->ne3_fan = reinterpret_cast<int32_t*>(b + L.ne3_fan);
    p->ne3_fcnt = reinterpret_cast<int32_t*>(b + L.ne3_fcnt);
    p->fan_valid = false;
    p->enumerated = p->symbolic = false;
    // counters that must start at zero (the fill pass restores cnt to zero;
    // entry N of the count arrays is never written)
    EFEM_CUDA_TRY(cudaMemset(p->cnt, 0, ((size_t)p->n_nodes + 1) * 4));
    EFEM_CUDA_TRY(cudaMemset(p->ent_cnt, 0, ((size_t)p->n_nodes + 1) * 4));
    EFEM_CUDA_TRY(cudaMemset(p->nnz_cnt, 0, ((size_t)p->n_nodes + 1) * 4));
    if (p->g_enum) {
        cudaGraphExecDestroy(p->g_enum);
        p->g_enum = nullptr;
    }
    if (p->g_async) {
        cudaGraphExecDestroy(p->g_async);
        p->g_async = nullptr;
    }
    if (p->g_part) {
        cudaGraphExecDestroy(p->g_part);
        p->g_part = nullptr;
    }
    return EFEM_OK;
}

efem_status efem_plan_set_exact(efem_plan plan, int exact) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p) {
        set_error("efem_plan_set_exact: NULL plan");
        return EFEM_EINVAL;
    }
    if (p->exact_ne3 != (exact != 0)) {
        p->exact_ne3 = exact != 0;
        p->enumerated = p->symbolic = false;
        if (p->g_enum) {  // the captured enumeration bakes the mode in
            cudaGraphExecDestroy(p->g_enum);
            p->g_enum = nullptr;
        }
        if (p->g_async) {
            cudaGraphExecDestroy(p->g_async);
            p->g_async = nullptr;
        }
    }
    return EFEM_OK;
}

efem_status efem_plan_destroy(efem_plan plan) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p) return EFEM_OK;
    if (p->h_scalars) cudaFreeHost(p->h_scalars);
    if (p->h_hdr) cudaFreeHost(p->h_hdr);
    if (p->g_enum) cudaGraphExecDestroy(p->g_enum);
    if (p->g_async) cudaGraphExecDestroy(p->g_async);
    if (p->g_part) cudaGraphExecDestroy(p->g_part);
    if (p->ev_in) cudaEventDestroy(p->ev_in);
    if (p->ev_out) cudaEventDestroy(p->ev_out);
    if (p->gstream) cudaStreamDestroy(p->gstream);
    delete p;
    return EFEM_OK;
}

static efem_status need_ws(Plan* p) {
    if (!p) {
        set_error("NULL plan");
        return EFEM_EINVAL;
    }
    if (!p->ws) {
        set_error("plan has no workspace (efem_plan_set_workspace)");
        return EFEM_EWORKSPACE;
    }
    return EFEM_OK;
}

efem_status efem_enumerate_dofs(efem_plan plan, efem_dofs* out, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    efem_status st = need_ws(p);
    if (st != EFEM_OK) return st;
    if (!out) {
        set_error("efem_enumerate_dofs: NULL out");
        return EFEM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    p->symbolic = false;
    p->enumerated = false;
    p->want_d2n = true;
    st = run_enumerate(*p, s);
    p->want_d2n = false;
    if (st != EFEM_OK) return st;
    out->n_dofs = p->n_dofs;
    if (out->dofs2nodes && p->n_dofs)
        EFEM_CUDA_TRY(cudaMemcpyAsync(out->dofs2nodes, p->d2n, p->n_dofs * p->ek * 4, cudaMemcpyDeviceToDevice, s));
    if (out->elems2dofs && p->n_elems)
        EFEM_CUDA_TRY(cudaMemcpyAsync(out->elems2dofs, p->e2d, p->n_elems * p->m * 4, cudaMemcpyDeviceToDevice, s));
    if (out->signs && (st = launch_signs(*p, out->signs, s)) != EFEM_OK) return st;
    return EFEM_OK;
}

efem_status efem_assemble_symbolic(efem_plan plan, int64_t* n_rows, int64_t* nnz, int32_t* row_ptr,
                                   efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    efem_status st = need_ws(p);
    if (st != EFEM_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    p->enumerated = false;  // the end-to-end path always re-enumerates
    p->symbolic = false;
    if ((st = run_symbolic(*p, s)) != EFEM_OK) return st;
    if (n_rows) *n_rows = p->n_dofs;
    if (nnz) *nnz = p->nnz;
    if (row_ptr) {
        if ((st = ensure_enumerated(*p, s)) != EFEM_OK) return st;
        return write_row_ptr(*p, 0, p->n_dofs, row_ptr, s);
    }
    return EFEM_OK;
}

efem_status efem_assemble_numeric(efem_plan plan, unsigned forms, efem_csr* out, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    efem_status st = need_ws(p);
    if (st != EFEM_OK) return st;
    if (!p->symbolic) {
        set_error("efem_assemble_numeric before efem_assemble_symbolic");
        return EFEM_ESTATE;
    }
    const bool has_nz = p->nnz > 0;
    if (!out || out->n_rows != p->n_dofs || out->nnz != p->nnz || (has_nz && !out->col_idx) ||
        ((forms & EFEM_PATTERN) && !out->row_ptr) || (has_nz && (forms & EFEM_MASS) && !out->vals_mass) ||
        (has_nz && (forms & EFEM_STIFF) && !out->vals_stiff) || (forms & ~7u)) {
        set_error("efem_assemble_numeric: out sizes must equal symbolic n_rows/nnz; arrays for every form bit; "
                  "col_idx always required");
        return EFEM_EINVAL;
    }
    return run_numeric(*p, forms, out, (cudaStream_t)stream);
}

efem_status efem_plan_check(efem_plan plan, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    efem_status st = need_ws(p);
    if (st != EFEM_OK) return st;
    st = read_flags(*p, (cudaStream_t)stream);
    if (p->async_pending) {  // sizes of the last efem_assemble_async
        p->async_pending = false;
        p->n_dofs = p->h_hdr->totals[0];
        p->nnz = p->h_hdr->totals[1];
        p->symbolic = st == EFEM_OK;
        if (p->async_fan) p->fan_valid = st == EFEM_OK;
        else p->enumerated = st == EFEM_OK;
    }
    return st;
}

// the header read-back as one warp's stores into the pinned (UVA-mapped)
// host buffer: a posted PCIe write instead of a copy-engine transfer
__global__ void k_mirror_hdr(const WsHeader* __restrict__ hdr, WsHeader* h_hdr) {
    constexpr int W = sizeof(WsHeader) / 4;
    const int* src = reinterpret_cast<const int*>(hdr);
    volatile int* dst = reinterpret_cast<volatile int*>(h_hdr);
    for (int i = threadIdx.x; i < W; i += 32) dst[i] = src[i];
    __threadfence_system();
}

efem_status efem_plan_check_async(efem_plan plan, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    efem_status st = need_ws(p);
    if (st != EFEM_OK) return st;
    WsHeader* dptr = nullptr;
    if (cudaHostGetDevicePointer((void**)&dptr, p->h_hdr, 0) == cudaSuccess && dptr) {
        k_mirror_hdr<<<1, 32, 0, (cudaStream_t)stream>>>(p->hdr, dptr);
        EFEM_LAUNCH_CHECK();
    } else {
        cudaGetLastError();
        EFEM_CUDA_TRY(cudaMemcpyAsync(p->h_hdr, p->hdr, sizeof(WsHeader), cudaMemcpyDeviceToHost,
                                      (cudaStream_t)stream));
    }
    return EFEM_OK;
}

efem_status efem_assemble_async(efem_plan plan, unsigned forms, efem_csr* out, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    efem_status st = need_ws(p);
    if (st != EFEM_OK) return st;
    if (!out || out->n_rows < 0 || out->nnz < 0 || (forms & ~7u) || !out->row_ptr ||
        (out->nnz > 0 && (!out->col_idx || ((forms & EFEM_MASS) && !out->vals_mass) ||
                          ((forms & EFEM_STIFF) && !out->vals_stiff)))) {
        set_error("efem_assemble_async: out capacities / arrays (row_ptr always, col_idx, a vals array per form bit)");
        return EFEM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    p->enumerated = p->symbolic = false;
    p->fan_valid = false;
    p->async_pending = true;
    p->async_fan = uses_fan(*p);
    auto enqueue = [&](cudaStream_t q) -> efem_status {
        efem_status e = uses_fan(*p) ? launch_fan_symbolic(*p, q) : launch_enumerate(*p, q);
        if (e != EFEM_OK) return e;
        RowWindow w;
        w.row0 = 0;
        w.n_rows = out->n_rows;  // capacity; the kernels read the real count on the device
        w.own_base = 0;
        w.out_base = 0;
        w.e2d = p->e2d;
        w.dyn = true;
        w.cap_nnz = out->nnz;
        if (out->n_rows == 0) {
            if (forms & EFEM_PATTERN) EFEM_CUDA_TRY(cudaMemsetAsync(out->row_ptr, 0, 4, q));
            return EFEM_OK;
        }
        return launch_rows_any(*p, forms, out, w, q);
    };
    // one CUDA graph for the whole call (captured on the plan's stream,
    // replayed with event handshakes); re-captured when the outputs change
    const bool same = p->g_async && p->async_forms == forms && !std::memcmp(&p->async_key, out, sizeof(efem_csr));
    if (!same && p->g_async) {
        cudaGraphExecDestroy(p->g_async);
        p->g_async = nullptr;
    }
    if (!p->g_async && !p->graph_failed && !p->want_d2n && !debug_sync()) {
        bool ok = p->gstream != nullptr;
        if (!ok) {
            ok = cudaStreamCreateWithFlags(&p->gstream, cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming) == cudaSuccess;
        }
        cudaGraph_t graph = nullptr;
        if (ok && cudaStreamBeginCapture(p->gstream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            const int64_t l0 = g_launches.load();
            const efem_status e = enqueue(p->gstream);
            const cudaError_t ee = cudaStreamEndCapture(p->gstream, &graph);
            p->async_launches = g_launches.load() - l0;
            g_launches.fetch_sub(p->async_launches);  // counted at replay
            if (e == EFEM_OK && ee == cudaSuccess && cudaGraphInstantiate(&p->g_async, graph, 0) == cudaSuccess) {
                p->async_key = *out;
                p->async_forms = forms;
            } else {
                p->g_async = nullptr;
            }
            if (graph) cudaGraphDestroy(graph);
        }
        cudaGetLastError();
    }
    if (p->g_async) {
        // (a graph captured on the plan's stream replays on the caller's)
        EFEM_CUDA_TRY(cudaGraphLaunch(p->g_async, s));
        count_launch((int)p->async_launches);
        return EFEM_OK;
    }
    return enqueue(s);
}

efem_status efem_assemble_host(efem_plan plan, const double* h_coords, const int32_t* h_elems, efem_csr* d_out,
                               efem_csr* h_out, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    efem_status st = need_ws(p);
    if (st != EFEM_OK) return st;
    if (!h_coords || !h_elems || !d_out || !h_out) {
        set_error("efem_assemble_host: NULL argument");
        return EFEM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    EFEM_CUDA_TRY(cudaMemcpyAsync(const_cast<double*>(p->coords), h_coords, p->n_nodes * p->dim * 8,
                                  cudaMemcpyHostToDevice, s));
    EFEM_CUDA_TRY(cudaMemcpyAsync(const_cast<int32_t*>(p->elems), h_elems, p->n_elems * p->nv * 4,
                                  cudaMemcpyHostToDevice, s));
    int64_t R, nnz;
    if ((st = efem_assemble_symbolic(plan, &R, &nnz, nullptr, stream)) != EFEM_OK) return st;
    if (d_out->nnz < nnz || d_out->n_rows < R || h_out->nnz < nnz || h_out->n_rows < R) {
        set_error("efem_assemble_host: output capacity smaller than the pattern");
        return EFEM_EINVAL;
    }
    efem_csr d = *d_out;
    d.n_rows = R;
    d.nnz = nnz;
    if ((st = efem_assemble_numeric(plan, EFEM_ALL, &d, stream)) != EFEM_OK) return st;
    EFEM_CUDA_TRY(cudaMemcpyAsync(h_out->row_ptr, d.row_ptr, (R + 1) * 4, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaMemcpyAsync(h_out->col_idx, d.col_idx, nnz * 4, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaMemcpyAsync(h_out->vals_mass, d.vals_mass, nnz * 8, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaMemcpyAsync(h_out->vals_stiff, d.vals_stiff, nnz * 8, cudaMemcpyDeviceToHost, s));
    if ((st = read_flags(*p, s)) != EFEM_OK) return st;
    h_out->n_rows = R;
    h_out->nnz = nnz;
    return EFEM_OK;
}

// ---- f1 / f2 -------------------------------------------------------------------------
int efem_quad_size(int dim) { return (dim == 2 || dim == 3) ? quad6_size(dim) : 0; }

efem_status efem_quad_points(const efem_mesh* mesh, double* pts, efem_stream_t stream) {
    if (!mesh || (mesh->dim != 2 && mesh->dim != 3) || mesh->n_elems < 0 ||
        (mesh->n_elems > 0 && (!pts || !mesh->coords || !mesh->elems))) {
        set_error("efem_quad_points: bad mesh or NULL output");
        return EFEM_EINVAL;
    }
    return launch_quad_points(mesh->dim, mesh->coords, mesh->elems, mesh->n_elems, pts, (cudaStream_t)stream);
}

efem_status efem_assemble_load(efem_plan plan, int pairing, const double* fq, double* b, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    efem_status st = need_ws(p);
    if (st != EFEM_OK) return st;
    if (!p->symbolic) {
        set_error("efem_assemble_load before efem_assemble_symbolic");
        return EFEM_ESTATE;
    }
    if ((pairing != EFEM_PAIR_VALUE && pairing != EFEM_PAIR_DERIV) || (p->n_dofs > 0 && (!fq || !b))) {
        set_error("efem_assemble_load: pairing must be EFEM_PAIR_VALUE or EFEM_PAIR_DERIV, arrays non-NULL");
        return EFEM_EINVAL;
    }
    if ((st = ensure_enumerated(*p, (cudaStream_t)stream)) != EFEM_OK) return st;
    return launch_load(*p, pairing, fq, b, (cudaStream_t)stream);
}

efem_status efem_norm_l2(const efem_mesh* mesh, const double* fq, int nf, double* per_elem, double* total, void* ws,
                         size_t* ws_bytes, efem_stream_t stream) {
    if (!ws_bytes) {
        set_error("efem_norm_l2: NULL ws_bytes");
        return EFEM_EINVAL;
    }
    if (!ws) {
        *ws_bytes = reduce_ws_bytes();
        return EFEM_OK;
    }
    if (!mesh || (mesh->dim != 2 && mesh->dim != 3) || nf < 1 || !total || *ws_bytes < reduce_ws_bytes() ||
        (mesh->n_elems > 0 && (!fq || !per_elem))) {
        set_error("efem_norm_l2: bad arguments or workspace too small");
        return EFEM_EINVAL;
    }
    return launch_norm_l2(mesh->dim, mesh->coords, mesh->elems, mesh->n_elems, fq, nf, per_elem, total,
                          static_cast<double*>(ws), (cudaStream_t)stream);
}

efem_status efem_field_error(efem_plan plan, const double* coeffs, const double* Eq, const double* Dq, double* err2,
                             void* ws, size_t* ws_bytes, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    efem_status st = need_ws(p);
    if (st != EFEM_OK) return st;
    if (!ws_bytes) {
        set_error("efem_field_error: NULL ws_bytes");
        return EFEM_EINVAL;
    }
    const size_t need = (size_t)(2 * p->n_elems) * sizeof(double) + reduce_ws_bytes();
    if (!ws) {
        *ws_bytes = need;
        return EFEM_OK;
    }
    if (!p->symbolic) {
        set_error("efem_field_error before efem_assemble_symbolic");
        return EFEM_ESTATE;
    }
    if (*ws_bytes < need || !err2 || (p->n_elems > 0 && (!coeffs || !Eq || !Dq))) {
        set_error("efem_field_error: bad arguments or workspace too small");
        return EFEM_EINVAL;
    }
    if ((st = ensure_enumerated(*p, (cudaStream_t)stream)) != EFEM_OK) return st;
    return launch_field_error(*p, coeffs, Eq, Dq, err2, static_cast<double*>(ws), (cudaStream_t)stream);
}

efem_status efem_spmv(const efem_csr* A, double alpha, double beta, const double* x, double* y,
                      efem_stream_t stream) {
    if (!A || A->n_rows < 0 || (A->n_rows > 0 && (!A->row_ptr || !A->col_idx || !A->vals_mass || !A->vals_stiff ||
                                                  !x || !y))) {
        set_error("efem_spmv: NULL array");
        return EFEM_EINVAL;
    }
    return launch_spmv(A, alpha, beta, x, y, (cudaStream_t)stream);
}

efem_status efem_cg(const efem_csr* A, double alpha, double beta, const double* b, double* x, double rtol, int maxit,
                    int* iters, double* relres, void* ws, size_t* ws_bytes, efem_stream_t stream) {
    if (!A || !ws_bytes) {
        set_error("efem_cg: NULL argument");
        return EFEM_EINVAL;
    }
    if (!ws) {
        *ws_bytes = cg_ws_bytes(A->n_rows);
        return EFEM_OK;
    }
    if (*ws_bytes < cg_ws_bytes(A->n_rows) || !iters || !relres || maxit < 0 || !(rtol >= 0.0) ||
        (A->n_rows > 0 && (!b || !x || !A->row_ptr || !A->col_idx || !A->vals_mass || !A->vals_stiff))) {
        set_error("efem_cg: bad arguments or workspace too small");
        return EFEM_EINVAL;
    }
    return run_cg(A, alpha, beta, b, x, rtol, maxit, iters, relres, ws, (cudaStream_t)stream);
}

}  // extern "C"
