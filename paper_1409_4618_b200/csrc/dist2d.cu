// dist2d.cu -- multi-GPU assembly of the 2D matrices (SURVEY.md §8(e),
// BASELINE north_star: "the elements are partitioned into contiguous slabs
// per GPU; each GPU assembles its slab, and off-rank rows are exchanged with
// NCCL all-to-all over NVLink into row-owned CSR slices").
//
// Ownership.  Rank r holds the element slab [elem_lo, elem_hi) and owns the
// nodes [lo_r, lo_{r+1}) (lo_r = the smallest vertex of its slab, made
// monotone; lo_0 = 0, lo_P = N).  DOF ids are lexicographic in the sorted
// node pair (reading C10), so the edges whose smaller node it
// owns are a contiguous block of global rows: its CSR slice.
//
// A row (a, b) receives the local matrices of the <= 2 triangles holding it
// (PAPER.md:335-342, 696); such a triangle has a as its smallest or middle
// vertex.  The contributions of a rank's slab to rows it does not own are
// the off-rank rows:
//   A  the slab rank computes the local matrices (the 2D closed form of
//      PAPER.md:344-363, element.cuh tri_vals, the same code as the 1-GPU
//      kernel) of its triangles whose smallest or middle vertex another rank
//      owns and sends them, with the triangle's vertex ids, to that owner
//      (grouped ncclSend / ncclRecv: an all-to-all-v in which only slab
//      neighbours are non-empty);
//   -  every rank enumerates its owned rows from the fans of its owned nodes
//      over its held triangles (own slab + received ghosts; fan2d.cu) and the
//      ranks all-gather their row / entry totals (-> global offsets);
//   B  the ids of the columns owned elsewhere (edges of held triangles whose
//      smaller node another rank owns) are answered by their owners
//      (grouped send / receive of int32 ids for requests fixed at setup);
//   -  the numeric row kernel (assemble.cu k_rows_tri, GhostTriPolicy) sums
//      each owned row from local triangles (computed) and ghosts (received)
//      in ascending element order, as the 1-GPU kernel does.
// The ranks' slices concatenate to the 1-GPU matrices.  Per step the bytes
// exchanged are O(interface): 112 B per ghost triangle, 4 B per requested
// id, 16 B per rank of totals.
//
// Setup (untimed, once per partition; synchronising) fixes the
// communication pattern from the topology: node ranges, which triangles go
// where, which column ids are requested from whom.
//
// Transport: NCCL, called from this library (efem_comm wraps an
// ncclComm_t), or -- for tests of several ranks inside one process on one
// device -- a local group whose exchanges are device-to-device copies.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "element.cuh"

namespace efem {
efem_status launch_rows_any(Plan& p, unsigned forms, efem_csr* out, const RowWindow& w, cudaStream_t s);
}

struct efem_comm_s {
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1;
};

namespace efem {
namespace {

constexpr int REC_D = 14;  // doubles per ghost record: {g0, g1}, {g2, e} as int pairs, 12 row values

#define EFEM_NCCL_TRY(expr)                                                          \
    do {                                                                             \
        ncclResult_t _r = (expr);                                                    \
        if (_r != ncclSuccess) {                                                     \
            ::efem::set_error(std::string(#expr) + ": " + ncclGetErrorString(_r));   \
            return EFEM_ENCCL;                                                       \
        }                                                                            \
    } while (0)

__global__ void k_gather_kept(const int32_t* __restrict__ elems, const int32_t* __restrict__ keep, int64_t n,
                              int32_t* __restrict__ held) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t e = __ldg(keep + i);
    held[3 * i] = __ldg(elems + 3 * e);
    held[3 * i + 1] = __ldg(elems + 3 * e + 1);
    held[3 * i + 2] = __ldg(elems + 3 * e + 2);
}

// A: the local matrix rows of the triangles to send, in the three rotated
// frames the row kernel uses (row k: vertex k first)
__global__ void k_ghost_pack(const double* __restrict__ coords, const int32_t* __restrict__ elems,
                             const int32_t* __restrict__ tris, int64_t n, double* __restrict__ out, WsHeader* hdr) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int e = __ldg(tris + i);
    const int g[3] = {__ldg(elems + 3 * (int64_t)e), __ldg(elems + 3 * (int64_t)e + 1),
                      __ldg(elems + 3 * (int64_t)e + 2)};
    const double2* c2 = reinterpret_cast<const double2*>(coords);
    const double2 x[3] = {__ldg(c2 + g[0]), __ldg(c2 + g[1]), __ldg(c2 + g[2])};
    double* r = out + i * REC_D;
    reinterpret_cast<int2*>(r)[0] = make_int2(g[0], g[1]);
    reinterpret_cast<int2*>(r)[1] = make_int2(g[2], e);
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const TriVals V = tri_vals(x[k], x[(k + 1) % 3], x[(k + 2) % 3]);
        bad |= !(fabs(V.det) > 0.0 && fabs(V.det) < INFINITY);
        r[2 + 4 * k] = V.m0;
        r[3 + 4 * k] = V.v1;
        r[4 + 4 * k] = V.v2;
        r[5 + 4 * k] = V.ck;
    }
    if (bad) {
        atomicOr(&hdr->flags[F_DEGENERATE], 1);
        atomicMin(&hdr->bad_element, (unsigned long long)e);
    }
}

__global__ void k_unpack(const double* __restrict__ rec, int64_t n, int32_t* __restrict__ held,
                         double* __restrict__ gvals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* r = rec + i * REC_D;
    const int2 a = reinterpret_cast<const int2*>(r)[0], b = reinterpret_cast<const int2*>(r)[1];
    held[3 * i] = a.x;
    held[3 * i + 1] = a.y;
    held[3 * i + 2] = b.x;
#pragma unroll
    for (int q = 0; q < 12; ++q) gvals[12 * i + q] = r[2 + q];
}

// global offsets of this rank's rows and entries from the gathered totals;
// the row window the numeric kernel reads: {first local row 0, rows, CSR
// offset 0, entries, global id of row 0, global entry offset}
__global__ void k_offsets(const long long* __restrict__ totals, int nranks, int rank, long long* __restrict__ win) {
    if (threadIdx.x != 0) return;
    long long r0 = 0, z0 = 0;
    for (int s = 0; s < rank; ++s) {
        r0 += totals[2 * s];
        z0 += totals[2 * s + 1];
    }
    win[0] = 0;
    win[1] = totals[2 * rank];
    win[2] = 0;
    win[3] = totals[2 * rank + 1];
    win[4] = r0;
    win[5] = z0;
}

// B (owner side): global id of the requested edge (u, v), u owned: scan the
// rows of u (ascending v); the larger endpoint of row i is read off its first
// incidence (rec[i].x = e << 3 | k: local edge k of held triangle e)
__global__ void k_respond(const int2* __restrict__ keys, int64_t n, const int32_t* __restrict__ node_ent, int64_t lo,
                          const int2* __restrict__ rec, const int32_t* __restrict__ held,
                          const long long* __restrict__ win, int32_t* __restrict__ ids, WsHeader* hdr) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int2 kv = __ldg(keys + i);
    const int64_t lu = kv.x - lo;
    int id = -1;
    for (int r = __ldg(node_ent + lu), re = __ldg(node_ent + lu + 1); r < re; ++r) {
        const int inst = __ldg(&rec[r].x);
        const int e = inst >> 3, k = inst & 7;
        const int s0 = __ldg(held + 3 * (int64_t)e + (k + 1) % 3), s1 = __ldg(held + 3 * (int64_t)e + (k + 2) % 3);
        if (max(s0, s1) == kv.y) {
            id = r + (int)win[4];
            break;
        }
    }
    if (id < 0) atomicOr(&hdr->flags[F_ROW_MISMATCH], 1);
    ids[i] = id;
}

// elems2dofs of the held triangles relative to the rank's first row (the
// row kernel adds it back): the owned entries are the fan pass's local ids,
// the requested ones the owners' answers (global ids) shifted down
__global__ void k_fill(int32_t* __restrict__ e2d, const int32_t* __restrict__ slots, const int32_t* __restrict__ ids,
                       int64_t n, const long long* __restrict__ win) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) e2d[__ldg(slots + i)] = __ldg(ids + i) - (int)win[4];
}

template <class T>
T* dalloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) return nullptr;
    return static_cast<T*>(p);
}

}  // namespace

struct DistPlan {
    int rank = 0, P = 1;
    efem_comm comm = nullptr;  // NULL: a local group (efem_dist_group_create)
    int element = 0;
    int64_t N = 0, T = 0, e_lo = 0, e_hi = 0;
    const double* coords = nullptr;
    const int32_t* elems = nullptr;
    std::vector<int64_t> lo;  // P + 1 node range bounds
    int64_t n_keep = 0, n_ghost = 0, n_held = 0;
    std::vector<int64_t> send_off, recv_off, req_off, resp_off;  // P + 1 each (element counts)
    // device
    int32_t* keep = nullptr;       // n_keep global triangle ids
    int32_t* send_tris = nullptr;  // ghost triangles to send, by destination rank
    double* sendA = nullptr;       // REC_D per sent triangle
    double* recvA = nullptr;       // REC_D per received triangle, by source rank
    int32_t* held = nullptr;       // 3 per held triangle: kept, then ghosts
    double* gvals = nullptr;       // 12 per ghost
    int32_t* req_slots = nullptr;  // e2d slots whose ids other ranks own, by owner
    int32_t* req_ids = nullptr;    // their answers
    int2* resp_keys = nullptr;     // edges other ranks ask this rank for, by asking rank
    int32_t* resp_ids = nullptr;
    long long* totals = nullptr;   // 2 P gathered {rows, entries}
    int32_t* node_ent = nullptr;
    void* ws = nullptr;
    efem_plan plan = nullptr;
    efem_csr cap{};  // capacities of the last step's slice
    bool stepped = false;
    // the step as one CUDA graph (kernels and NCCL calls), captured on the
    // plan's own stream and replayed with event handshakes; keyed by the slice
    cudaStream_t gs = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaGraphExec_t graph = nullptr;
    efem_csr gkey{};
    unsigned gforms = 0;
    bool gfan_small = false;  // the fan-pass register path the graph was captured with
    bool graph_failed = false;
    int64_t graph_launches = 0;

    Plan& p() { return *reinterpret_cast<Plan*>(plan); }
    int owner(int64_t v) const {
        return (int)(std::upper_bound(lo.begin(), lo.end(), v) - lo.begin()) - 1;
    }
    ~DistPlan() {
        if (graph) cudaGraphExecDestroy(graph);
        if (ev_in) cudaEventDestroy(ev_in);
        if (ev_out) cudaEventDestroy(ev_out);
        if (gs) cudaStreamDestroy(gs);
        if (plan) efem_plan_destroy(plan);
        for (void* q : {(void*)keep, (void*)send_tris, (void*)sendA, (void*)recvA, (void*)held, (void*)gvals,
                        (void*)req_slots, (void*)req_ids, (void*)resp_keys, (void*)resp_ids, (void*)totals,
                        (void*)node_ent, ws})
            if (q) cudaFree(q);
    }
};

namespace {

// ---- setup, host side ---------------------------------------------------------------
// one rank's slab on the host: vertex ids, validated
efem_status slab_host(const DistPlan& D, std::vector<int32_t>& h, cudaStream_t s) {
    h.resize((size_t)(D.e_hi - D.e_lo) * 3);
    if (!h.empty())
        EFEM_CUDA_TRY(cudaMemcpyAsync(h.data(), D.elems + D.e_lo * 3, h.size() * 4, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    for (int32_t v : h)
        if (v < 0 || v >= D.N) {
            set_error("efem_dist: an element references a node id outside [0, n_nodes)");
            return EFEM_EINVAL;
        }
    return EFEM_OK;
}

// node ranges from the slabs' smallest vertices (monotone; lo_0 = 0, lo_P = N)
void node_ranges(DistPlan& D, const std::vector<int64_t>& mins) {
    D.lo.assign(D.P + 1, 0);
    for (int r = 1; r < D.P; ++r) D.lo[r] = std::max(D.lo[r - 1], std::min(mins[r], D.N));
    D.lo[D.P] = D.N;
}

// which slab triangles stay (smallest or middle vertex owned here) and which
// go where (the owners of the smallest / middle vertex)
void classify(const DistPlan& D, const std::vector<int32_t>& h, std::vector<int32_t>& keep,
              std::vector<std::vector<int32_t>>& send) {
    send.assign(D.P, {});
    for (int64_t i = 0; i < D.e_hi - D.e_lo; ++i) {
        int v[3] = {h[3 * i], h[3 * i + 1], h[3 * i + 2]};
        std::sort(v, v + 3);
        const int op = D.owner(v[0]), oq = D.owner(v[1]);
        const int e = (int)(D.e_lo + i);
        if (op == D.rank || oq == D.rank) keep.push_back(e);
        if (op != D.rank) send[op].push_back(e);
        if (oq != D.rank && oq != op) send[oq].push_back(e);
    }
}

// the e2d slots of the held triangles whose edge's smaller node another rank
// owns: (slot, u, v) requests grouped by owner
void requests(const DistPlan& D, const std::vector<int32_t>& held, std::vector<std::vector<int32_t>>& slots,
              std::vector<std::vector<int2>>& keys) {
    slots.assign(D.P, {});
    keys.assign(D.P, {});
    const int64_t nh = (int64_t)held.size() / 3;
    for (int64_t i = 0; i < nh; ++i)
        for (int k = 0; k < 3; ++k) {  // local edge k: vertices k+1, k+2 (Fig. 1, reading C4)
            const int a = held[3 * i + (k + 1) % 3], b = held[3 * i + (k + 2) % 3];
            const int u = std::min(a, b), v = std::max(a, b);
            const int o = D.owner(u);
            if (o == D.rank) continue;
            slots[o].push_back((int32_t)(3 * i + k));
            keys[o].push_back(make_int2(u, v));
        }
}

// ---- transport ------------------------------------------------------------------------
// all-to-all-v of fixed per-peer counts: NCCL grouped send / receive
efem_status nccl_alltoallv(DistPlan& D, const void* send, const std::vector<int64_t>& soff, void* recv,
                           const std::vector<int64_t>& roff, size_t elem_bytes, cudaStream_t s) {
    EFEM_NCCL_TRY(ncclGroupStart());
    for (int d = 0; d < D.P; ++d) {
        if (d == D.rank) continue;
        const size_t ns = (size_t)(soff[d + 1] - soff[d]) * elem_bytes, nr = (size_t)(roff[d + 1] - roff[d]) * elem_bytes;
        if (ns) EFEM_NCCL_TRY(ncclSend((const char*)send + soff[d] * elem_bytes, ns, ncclChar, d, D.comm->nccl, s));
        if (nr) EFEM_NCCL_TRY(ncclRecv((char*)recv + roff[d] * elem_bytes, nr, ncclChar, d, D.comm->nccl, s));
    }
    EFEM_NCCL_TRY(ncclGroupEnd());
    return EFEM_OK;
}

// the same between the plans of a local group (device-to-device copies)
template <class GetSend, class GetRecv>
efem_status group_alltoallv(std::vector<DistPlan*>& G, GetSend snd, GetRecv rcv, size_t elem_bytes, cudaStream_t s) {
    for (DistPlan* src : G)
        for (DistPlan* dst : G) {
            if (src == dst) continue;
            const std::vector<int64_t>& so = snd(src).second;
            const std::vector<int64_t>& ro = rcv(dst).second;
            const size_t n = (size_t)(so[dst->rank + 1] - so[dst->rank]) * elem_bytes;
            if (n != (size_t)(ro[src->rank + 1] - ro[src->rank]) * elem_bytes) {
                set_error("efem_dist: local group exchange sizes disagree");
                return EFEM_ESTATE;
            }
            if (n)
                EFEM_CUDA_TRY(cudaMemcpyAsync((char*)rcv(dst).first + ro[src->rank] * elem_bytes,
                                              (const char*)snd(src).first + so[dst->rank] * elem_bytes, n,
                                              cudaMemcpyDeviceToDevice, s));
        }
    return EFEM_OK;
}

std::vector<int64_t> offsets(const std::vector<size_t>& counts) {
    std::vector<int64_t> o(counts.size() + 1, 0);
    for (size_t i = 0; i < counts.size(); ++i) o[i + 1] = o[i] + (int64_t)counts[i];
    return o;
}

// NCCL setup exchange: every rank sends out_by_dst[d] (host vectors of POD T)
// to rank d; returns in_by_src.  Counts first (all-gather of the P x P count
// matrix), then the payloads through device staging.
template <class T>
efem_status nccl_setup_exchange(DistPlan& D, const std::vector<std::vector<T>>& out, std::vector<std::vector<T>>& in,
                                cudaStream_t s) {
    const int P = D.P;
    std::vector<long long> mine(P), all((size_t)P * P);
    for (int d = 0; d < P; ++d) mine[d] = (long long)out[d].size();
    long long* dbuf = dalloc<long long>((size_t)P * P + P);
    if (!dbuf) return EFEM_ECUDA;
    EFEM_CUDA_TRY(cudaMemcpyAsync(dbuf, mine.data(), P * 8, cudaMemcpyHostToDevice, s));
    EFEM_NCCL_TRY(ncclAllGather(dbuf, dbuf + P, P, ncclInt64, D.comm->nccl, s));
    EFEM_CUDA_TRY(cudaMemcpyAsync(all.data(), dbuf + P, (size_t)P * P * 8, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(dbuf);
    std::vector<size_t> sc(P), rc(P);
    for (int d = 0; d < P; ++d) {
        sc[d] = out[d].size();
        rc[d] = (size_t)all[(size_t)d * P + D.rank];
    }
    std::vector<int64_t> so = offsets(sc), ro = offsets(rc);
    std::vector<T> hs((size_t)so[P]), hr((size_t)ro[P]);
    for (int d = 0; d < P; ++d) std::copy(out[d].begin(), out[d].end(), hs.begin() + so[d]);
    T* ds = dalloc<T>(hs.size());
    T* dr = dalloc<T>(hr.size());
    if (!ds || !dr) return EFEM_ECUDA;
    if (!hs.empty()) EFEM_CUDA_TRY(cudaMemcpyAsync(ds, hs.data(), hs.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    efem_status st = nccl_alltoallv(D, ds, so, dr, ro, sizeof(T), s);
    if (st != EFEM_OK) return st;
    if (!hr.empty()) EFEM_CUDA_TRY(cudaMemcpyAsync(hr.data(), dr, hr.size() * sizeof(T), cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(ds);
    cudaFree(dr);
    in.assign(P, {});
    for (int r = 0; r < P; ++r) in[r].assign(hr.begin() + ro[r], hr.begin() + ro[r + 1]);
    return EFEM_OK;
}

// ---- setup, device side ---------------------------------------------------------------
efem_status finish_setup(DistPlan& D, const std::vector<int32_t>& keep, const std::vector<std::vector<int32_t>>& send,
                         const std::vector<std::vector<int32_t>>& ghost_topo /* by source rank, 3 per triangle */,
                         const std::vector<std::vector<int32_t>>& req_slots,
                         const std::vector<std::vector<int2>>& resp_keys, cudaStream_t s) {
    const int P = D.P;
    std::vector<size_t> c(P);
    for (int d = 0; d < P; ++d) c[d] = send[d].size();
    D.send_off = offsets(c);
    for (int d = 0; d < P; ++d) c[d] = ghost_topo[d].size() / 3;
    D.recv_off = offsets(c);
    for (int d = 0; d < P; ++d) c[d] = req_slots[d].size();
    D.req_off = offsets(c);
    for (int d = 0; d < P; ++d) c[d] = resp_keys[d].size();
    D.resp_off = offsets(c);
    D.n_keep = (int64_t)keep.size();
    D.n_ghost = D.recv_off[P];
    D.n_held = D.n_keep + D.n_ghost;
    auto up = [&](auto* dst, const auto& v) -> efem_status {
        if (!v.empty()) EFEM_CUDA_TRY(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, s));
        return EFEM_OK;
    };
    std::vector<int32_t> flat_send, flat_slots;
    std::vector<int2> flat_keys;
    for (int d = 0; d < P; ++d) {
        flat_send.insert(flat_send.end(), send[d].begin(), send[d].end());
        flat_slots.insert(flat_slots.end(), req_slots[d].begin(), req_slots[d].end());
        flat_keys.insert(flat_keys.end(), resp_keys[d].begin(), resp_keys[d].end());
    }
    if (!(D.keep = dalloc<int32_t>(keep.size())) || !(D.send_tris = dalloc<int32_t>(flat_send.size())) ||
        !(D.sendA = dalloc<double>(flat_send.size() * REC_D)) || !(D.recvA = dalloc<double>((size_t)D.n_ghost * REC_D)) ||
        !(D.held = dalloc<int32_t>((size_t)D.n_held * 3)) || !(D.gvals = dalloc<double>((size_t)D.n_ghost * 12)) ||
        !(D.req_slots = dalloc<int32_t>(flat_slots.size())) || !(D.req_ids = dalloc<int32_t>(flat_slots.size())) ||
        !(D.resp_keys = dalloc<int2>(flat_keys.size())) || !(D.resp_ids = dalloc<int32_t>(flat_keys.size())) ||
        !(D.totals = dalloc<long long>(2 * (size_t)P)) ||
        !(D.node_ent = dalloc<int32_t>((size_t)(D.lo[D.rank + 1] - D.lo[D.rank]) + 1))) {
        set_error("efem_dist: cudaMalloc failed");
        return EFEM_ECUDA;
    }
    efem_status st;
    if ((st = up(D.keep, keep)) != EFEM_OK || (st = up(D.send_tris, flat_send)) != EFEM_OK ||
        (st = up(D.req_slots, flat_slots)) != EFEM_OK || (st = up(D.resp_keys, flat_keys)) != EFEM_OK)
        return st;
    // the plan over the held triangles (global node ids, rows of the owned nodes only)
    efem_mesh hm{2, D.N, D.n_held, D.coords, D.held};
    size_t ws_bytes = 0;
    if ((st = efem_plan_create(&D.plan, &hm, (efem_element)D.element, &ws_bytes)) != EFEM_OK) return st;
    if (cudaMalloc(&D.ws, ws_bytes) != cudaSuccess) {
        set_error("efem_dist: workspace cudaMalloc failed");
        return EFEM_ECUDA;
    }
    if ((st = efem_plan_set_workspace(D.plan, D.ws, ws_bytes)) != EFEM_OK) return st;
    Plan& p = D.p();
    p.own_lo = D.lo[D.rank];
    p.own_n = D.lo[D.rank + 1] - D.lo[D.rank];
    p.node_ent = D.node_ent;
    // the slab's kept triangles into the held array, once: the connectivity
    // (and with it this setup's classification) is fixed for the plan's life;
    // coordinates are read every step
    if (D.n_keep > 0) {
        k_gather_kept<<<grid_for(D.n_keep, 256), 256, 0, s>>>(D.elems, D.keep, D.n_keep, D.held);
        EFEM_LAUNCH_CHECK();
    }
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    return EFEM_OK;
}

// ---- the step, phase by phase -----------------------------------------------------------
efem_status ph_pack(DistPlan& D, cudaStream_t s) {
    Plan& p = D.p();
    // the step's header reset happens here (the fan pass below keeps it), so
    // a degenerate ghost flagged by the pack survives to the check
    efem_status st = launch_hdr_reset(p, s);
    if (st != EFEM_OK) return st;
    const int64_t ns = D.send_off[D.P];
    if (ns > 0) {
        k_ghost_pack<<<grid_for(ns, 256), 256, 0, s>>>(D.coords, D.elems, D.send_tris, ns, D.sendA, p.hdr);
        EFEM_LAUNCH_CHECK();
    }
    return EFEM_OK;
}

efem_status ph_symbolic(DistPlan& D, cudaStream_t s) {
    Plan& p = D.p();
    if (D.n_ghost > 0) {
        k_unpack<<<grid_for(D.n_ghost, 256), 256, 0, s>>>(D.recvA, D.n_ghost, D.held + 3 * D.n_keep, D.gvals);
        EFEM_LAUNCH_CHECK();
    }
    efem_status st = launch_fan_symbolic(p, s, false);
    if (st != EFEM_OK) return st;
    // this rank's {rows, entries} into its slot of the gathered totals
    EFEM_CUDA_TRY(cudaMemcpyAsync(D.totals + 2 * D.rank, &p.hdr->totals[0], 16, cudaMemcpyDeviceToDevice, s));
    return EFEM_OK;
}

efem_status ph_respond(DistPlan& D, cudaStream_t s) {
    Plan& p = D.p();
    k_offsets<<<1, 32, 0, s>>>(D.totals, D.P, D.rank, p.hdr->win);
    EFEM_LAUNCH_CHECK();
    const int64_t n = D.resp_off[D.P];
    if (n > 0) {
        k_respond<<<grid_for(n, 256), 256, 0, s>>>(D.resp_keys, n, D.node_ent, D.lo[D.rank], p.rec, D.held,
                                                    p.hdr->win, D.resp_ids, p.hdr);
        EFEM_LAUNCH_CHECK();
    }
    return EFEM_OK;
}

efem_status ph_numeric(DistPlan& D, unsigned forms, efem_csr* slice, cudaStream_t s) {
    Plan& p = D.p();
    const int64_t nr = D.req_off[D.P];
    if (nr > 0) {
        k_fill<<<grid_for(nr, 256), 256, 0, s>>>(p.e2d, D.req_slots, D.req_ids, nr, p.hdr->win);
        EFEM_LAUNCH_CHECK();
    }
    D.cap = *slice;
    if (slice->n_rows == 0) {  // (a size query, or an empty slice: the row kernel does not run)
        if ((forms & EFEM_PATTERN) && slice->row_ptr) EFEM_CUDA_TRY(cudaMemsetAsync(slice->row_ptr, 0, 4, s));
        return EFEM_OK;
    }
    RowWindow w;
    w.row0 = 0;
    w.n_rows = slice->n_rows;  // capacity: the window's sizes are read on the device
    w.cap_nnz = slice->nnz;
    w.e2d = p.e2d;
    w.win = p.hdr->win;
    w.ghost = true;
    w.gh.vals = D.gvals;
    w.gh.base = (int)D.n_keep;
    w.gh.col_base = 0;  // (set from the device window in the kernel)
    return launch_rows_any(p, forms, slice, w, s);
}

efem_status check_one(DistPlan& D, int64_t* window, cudaStream_t s) {
    Plan& p = D.p();
    WsHeader h;
    EFEM_CUDA_TRY(cudaMemcpyAsync(&h, p.hdr, sizeof(WsHeader), cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    p.fan_small = h.fan_big == 0;  // (the fan pass's register path for the next step)
    if (window) {
        window[0] = h.win[4];  // global id of the first row
        window[1] = h.win[1];  // rows
        window[2] = h.win[5];  // global offset of the first entry
        window[3] = h.win[3];  // entries
    }
    if (h.flags[F_INVALID_NODE]) {
        set_error("an element references a node id outside [0, n_nodes)");
        return EFEM_EINVAL;
    }
    if (h.flags[F_DEGENERATE]) {
        set_bad_element((int64_t)h.bad_element);
        set_error("degenerate element: " + std::to_string(h.bad_element));
        return EFEM_EDEGENERATE;
    }
    if (h.win[1] > D.cap.n_rows || h.win[3] > D.cap.nnz || h.flags[F_CAPACITY]) {
        set_error("efem_dist: slice capacity smaller than the owned rows (see the window for the sizes)");
        return EFEM_ECAPACITY;
    }
    if (h.flags[F_ROW_MISMATCH]) {
        set_error("non-conforming mesh (an edge in more than two triangles) or an unanswered column id");
        return EFEM_EINVAL;
    }
    return EFEM_OK;
}

efem_status validate_mesh(const efem_mesh* mesh, efem_element element) {
    if (!mesh || mesh->dim != 2 || (element != EFEM_RT0 && element != EFEM_NED0) || mesh->n_nodes < 0 ||
        mesh->n_elems < 0 || (mesh->n_elems > 0 && (!mesh->coords || !mesh->elems))) {
        set_error("efem_dist: a 2D mesh (triangles) and RT0 | NED0 (3D meshes: efem_part_*)");
        return EFEM_EINVAL;
    }
    return EFEM_OK;
}

}  // namespace
}  // namespace efem

using namespace efem;

extern "C" {

efem_status efem_comm_unique_id(unsigned char* id) {
    if (!id) return EFEM_EINVAL;
    ncclUniqueId u;
    EFEM_NCCL_TRY(ncclGetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, sizeof(u));
    return EFEM_OK;
}

efem_status efem_comm_init(efem_comm* comm, const unsigned char* id, int nranks, int rank) {
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("efem_comm_init: bad arguments");
        return EFEM_EINVAL;
    }
    efem_comm c = new (std::nothrow) efem_comm_s;
    if (!c) return EFEM_ENOMEM;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    const ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        return EFEM_ENCCL;
    }
    c->rank = rank;
    c->nranks = nranks;
    *comm = c;
    return EFEM_OK;
}

efem_status efem_comm_destroy(efem_comm comm) {
    if (!comm) return EFEM_OK;
    if (comm->nccl) ncclCommDestroy(comm->nccl);
    delete comm;
    return EFEM_OK;
}

efem_status efem_dist_plan_create(efem_dist_plan* plan, const efem_mesh* mesh, efem_element element, int64_t elem_lo,
                                  int64_t elem_hi, efem_comm comm, efem_stream_t stream) {
    efem_status st = validate_mesh(mesh, element);
    if (st != EFEM_OK) return st;
    if (!plan || !comm || elem_lo < 0 || elem_hi < elem_lo || elem_hi > mesh->n_elems) {
        set_error("efem_dist_plan_create: NULL plan / comm or a slab outside [0, n_elems)");
        return EFEM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    DistPlan* D = new (std::nothrow) DistPlan;
    if (!D) return EFEM_ENOMEM;
    D->rank = comm->rank;
    D->P = comm->nranks;
    D->comm = comm;
    D->element = element;
    D->N = mesh->n_nodes;
    D->T = mesh->n_elems;
    D->coords = mesh->coords;
    D->elems = mesh->elems;
    D->e_lo = elem_lo;
    D->e_hi = elem_hi;
    auto fail = [&](efem_status e) {
        delete D;
        return e;
    };
    std::vector<int32_t> h;
    if ((st = slab_host(*D, h, s)) != EFEM_OK) return fail(st);
    // node ranges: all-gather of the slabs' smallest vertices
    long long mn = D->N;
    for (int32_t v : h) mn = std::min<long long>(mn, v);
    long long* dm = dalloc<long long>(D->P + 1);
    if (!dm) return fail(EFEM_ECUDA);
    EFEM_CUDA_TRY(cudaMemcpyAsync(dm, &mn, 8, cudaMemcpyHostToDevice, s));
    {
        const ncclResult_t r = ncclAllGather(dm, dm + 1, 1, ncclInt64, comm->nccl, s);
        if (r != ncclSuccess) {
            cudaFree(dm);
            set_error(std::string("ncclAllGather: ") + ncclGetErrorString(r));
            return fail(EFEM_ENCCL);
        }
    }
    std::vector<long long> mins_ll(D->P);
    EFEM_CUDA_TRY(cudaMemcpyAsync(mins_ll.data(), dm + 1, D->P * 8, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(dm);
    node_ranges(*D, std::vector<int64_t>(mins_ll.begin(), mins_ll.end()));
    std::vector<int32_t> keep;
    std::vector<std::vector<int32_t>> send;
    classify(*D, h, keep, send);
    // setup exchange 1: the ghost triangles' vertex ids (their owners build requests)
    std::vector<std::vector<int32_t>> topo_out(D->P), topo_in;
    for (int d = 0; d < D->P; ++d)
        for (int32_t e : send[d])
            for (int c = 0; c < 3; ++c) topo_out[d].push_back(h[3 * (e - D->e_lo) + c]);
    if ((st = nccl_setup_exchange(*D, topo_out, topo_in, s)) != EFEM_OK) return fail(st);
    std::vector<int32_t> held;
    for (int32_t e : keep)
        for (int c = 0; c < 3; ++c) held.push_back(h[3 * (e - D->e_lo) + c]);
    for (int r = 0; r < D->P; ++r) held.insert(held.end(), topo_in[r].begin(), topo_in[r].end());
    std::vector<std::vector<int32_t>> slots;
    std::vector<std::vector<int2>> keys, keys_in;
    requests(*D, held, slots, keys);
    // setup exchange 2: the requested edges to their owners
    if ((st = nccl_setup_exchange(*D, keys, keys_in, s)) != EFEM_OK) return fail(st);
    if ((st = finish_setup(*D, keep, send, topo_in, slots, keys_in, s)) != EFEM_OK) return fail(st);
    *plan = reinterpret_cast<efem_dist_plan>(D);
    return EFEM_OK;
}

efem_status efem_dist_group_create(efem_dist_plan* plans, int nranks, const efem_mesh* mesh, efem_element element,
                                   const int64_t* elem_bounds, efem_stream_t stream) {
    efem_status st = validate_mesh(mesh, element);
    if (st != EFEM_OK) return st;
    if (!plans || nranks < 1 || !elem_bounds || elem_bounds[0] != 0 || elem_bounds[nranks] != mesh->n_elems) {
        set_error("efem_dist_group_create: NULL arrays or slab bounds not covering [0, n_elems)");
        return EFEM_EINVAL;
    }
    for (int r = 0; r < nranks; ++r)
        if (elem_bounds[r + 1] < elem_bounds[r]) {
            set_error("efem_dist_group_create: slab bounds must be non-decreasing");
            return EFEM_EINVAL;
        }
    cudaStream_t s = (cudaStream_t)stream;
    const int P = nranks;
    std::vector<DistPlan*> G(P, nullptr);
    auto fail = [&](efem_status e) {
        for (DistPlan* d : G) delete d;
        return e;
    };
    std::vector<std::vector<int32_t>> h(P);
    std::vector<int64_t> mins(P);
    for (int r = 0; r < P; ++r) {
        G[r] = new (std::nothrow) DistPlan;
        if (!G[r]) return fail(EFEM_ENOMEM);
        DistPlan& D = *G[r];
        D.rank = r;
        D.P = P;
        D.element = element;
        D.N = mesh->n_nodes;
        D.T = mesh->n_elems;
        D.coords = mesh->coords;
        D.elems = mesh->elems;
        D.e_lo = elem_bounds[r];
        D.e_hi = elem_bounds[r + 1];
        if ((st = slab_host(D, h[r], s)) != EFEM_OK) return fail(st);
        int64_t mn = D.N;
        for (int32_t v : h[r]) mn = std::min<int64_t>(mn, v);
        mins[r] = mn;
    }
    std::vector<std::vector<int32_t>> keep(P);
    std::vector<std::vector<std::vector<int32_t>>> send(P), topo_out(P);
    for (int r = 0; r < P; ++r) {
        node_ranges(*G[r], mins);
        classify(*G[r], h[r], keep[r], send[r]);
        topo_out[r].assign(P, {});
        for (int d = 0; d < P; ++d)
            for (int32_t e : send[r][d])
                for (int c = 0; c < 3; ++c) topo_out[r][d].push_back(h[r][3 * (e - G[r]->e_lo) + c]);
    }
    std::vector<std::vector<std::vector<int32_t>>> topo_in(P, std::vector<std::vector<int32_t>>(P)), slots(P);
    std::vector<std::vector<std::vector<int2>>> keys(P), keys_in(P, std::vector<std::vector<int2>>(P));
    for (int r = 0; r < P; ++r)
        for (int d = 0; d < P; ++d) topo_in[d][r] = topo_out[r][d];
    for (int r = 0; r < P; ++r) {
        std::vector<int32_t> held;
        for (int32_t e : keep[r])
            for (int c = 0; c < 3; ++c) held.push_back(h[r][3 * (e - G[r]->e_lo) + c]);
        for (int q = 0; q < P; ++q) held.insert(held.end(), topo_in[r][q].begin(), topo_in[r][q].end());
        requests(*G[r], held, slots[r], keys[r]);
    }
    for (int r = 0; r < P; ++r)
        for (int d = 0; d < P; ++d) keys_in[d][r] = keys[r][d];
    for (int r = 0; r < P; ++r)
        if ((st = finish_setup(*G[r], keep[r], send[r], topo_in[r], slots[r], keys_in[r], s)) != EFEM_OK)
            return fail(st);
    for (int r = 0; r < P; ++r) plans[r] = reinterpret_cast<efem_dist_plan>(G[r]);
    return EFEM_OK;
}

efem_status efem_dist_layout(const int32_t* h_elems, int64_t n_nodes, int64_t n_elems, const int64_t* elem_bounds,
                             int nranks, int rank, int64_t* out) {
    if (!h_elems || !elem_bounds || !out || nranks < 1 || rank < 0 || rank >= nranks || n_nodes < 0 || n_elems < 0 ||
        elem_bounds[0] != 0 || elem_bounds[nranks] != n_elems) {
        set_error("efem_dist_layout: bad arguments");
        return EFEM_EINVAL;
    }
    std::vector<int64_t> mins(nranks);
    for (int r = 0; r < nranks; ++r) {
        if (elem_bounds[r + 1] < elem_bounds[r]) return EFEM_EINVAL;
        int64_t mn = n_nodes;
        for (int64_t i = elem_bounds[r] * 3; i < elem_bounds[r + 1] * 3; ++i) {
            if (h_elems[i] < 0 || h_elems[i] >= n_nodes) return EFEM_EINVAL;
            mn = std::min<int64_t>(mn, h_elems[i]);
        }
        mins[r] = mn;
    }
    DistPlan D;
    D.rank = rank;
    D.P = nranks;
    D.N = n_nodes;
    D.e_lo = elem_bounds[rank];
    D.e_hi = elem_bounds[rank + 1];
    node_ranges(D, mins);
    std::vector<int32_t> h(h_elems + D.e_lo * 3, h_elems + D.e_hi * 3), keep;
    std::vector<std::vector<int32_t>> send;
    classify(D, h, keep, send);
    out[0] = D.lo[rank];
    out[1] = D.lo[rank + 1];
    out[2] = (int64_t)keep.size();
    for (int d = 0; d < nranks; ++d) out[3 + d] = (int64_t)send[d].size();
    return EFEM_OK;
}

efem_status efem_dist_info(efem_dist_plan plan, int64_t* info) {
    DistPlan* D = reinterpret_cast<DistPlan*>(plan);
    if (!D || !info) return EFEM_EINVAL;
    info[0] = D->lo[D->rank];
    info[1] = D->lo[D->rank + 1];
    info[2] = D->n_keep;
    info[3] = D->n_ghost;
    info[4] = D->send_off[D->P];
    info[5] = D->req_off[D->P];
    info[6] = D->resp_off[D->P];
    // bytes this rank sends per step: ghost records, answered ids, its totals
    info[7] = D->send_off[D->P] * REC_D * 8 + D->resp_off[D->P] * 4 + 16;
    return EFEM_OK;
}

efem_status efem_dist_assemble(efem_dist_plan plan, unsigned forms, efem_csr* slice, efem_stream_t stream) {
    DistPlan* D = reinterpret_cast<DistPlan*>(plan);
    if (!D || !D->comm || !slice || (forms & ~7u) || !slice->row_ptr ||
        (slice->nnz > 0 && (!slice->col_idx || ((forms & EFEM_MASS) && !slice->vals_mass) ||
                            ((forms & EFEM_STIFF) && !slice->vals_stiff)))) {
        set_error("efem_dist_assemble: NULL plan (or a local-group plan), or slice arrays missing");
        return EFEM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    auto enqueue = [&](cudaStream_t q) -> efem_status {
        efem_status st;
        // A: ghost local matrices to the row owners
        if ((st = ph_pack(*D, q)) != EFEM_OK) return st;
        if ((st = nccl_alltoallv(*D, D->sendA, D->send_off, D->recvA, D->recv_off, REC_D * 8, q)) != EFEM_OK)
            return st;
        if ((st = ph_symbolic(*D, q)) != EFEM_OK) return st;
        // totals: {rows, entries} of every rank
        EFEM_NCCL_TRY(ncclAllGather(D->totals + 2 * D->rank, D->totals, 2, ncclInt64, D->comm->nccl, q));
        if ((st = ph_respond(*D, q)) != EFEM_OK) return st;
        // B: column ids answered by their owners
        if ((st = nccl_alltoallv(*D, D->resp_ids, D->resp_off, D->req_ids, D->req_off, 4, q)) != EFEM_OK) return st;
        return ph_numeric(*D, forms, slice, q);
    };
    const bool same = D->graph && D->gforms == forms && !std::memcmp(&D->gkey, slice, sizeof(efem_csr)) &&
                      D->gfan_small == D->p().fan_small;
    if (!same && D->graph) {
        cudaGraphExecDestroy(D->graph);
        D->graph = nullptr;
    }
    if (!D->graph && !D->graph_failed && !debug_sync()) {
        bool ok = D->gs != nullptr;
        if (!ok)
            ok = cudaStreamCreateWithFlags(&D->gs, cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&D->ev_in, cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&D->ev_out, cudaEventDisableTiming) == cudaSuccess;
        cudaGraph_t g = nullptr;
        if (ok && cudaStreamBeginCapture(D->gs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            const int64_t l0 = efem_launch_count();
            const efem_status e = enqueue(D->gs);
            const cudaError_t ee = cudaStreamEndCapture(D->gs, &g);
            D->graph_launches = efem_launch_count() - l0;
            count_launch(-(int)D->graph_launches);  // counted at replay
            if (e == EFEM_OK && ee == cudaSuccess && cudaGraphInstantiate(&D->graph, g, 0) == cudaSuccess) {
                D->gkey = *slice;
                D->gforms = forms;
                D->gfan_small = D->p().fan_small;
            } else {
                D->graph = nullptr;
                D->graph_failed = true;  // (enqueue directly from now on)
            }
            if (g) cudaGraphDestroy(g);
        }
        cudaGetLastError();
    }
    if (D->graph) {
        D->cap = *slice;
        EFEM_CUDA_TRY(cudaEventRecord(D->ev_in, s));
        EFEM_CUDA_TRY(cudaStreamWaitEvent(D->gs, D->ev_in, 0));
        EFEM_CUDA_TRY(cudaGraphLaunch(D->graph, D->gs));
        count_launch((int)D->graph_launches);
        EFEM_CUDA_TRY(cudaEventRecord(D->ev_out, D->gs));
        EFEM_CUDA_TRY(cudaStreamWaitEvent(s, D->ev_out, 0));
        return EFEM_OK;
    }
    return enqueue(s);
}

efem_status efem_dist_assemble_group(efem_dist_plan* plans, int nranks, unsigned forms, efem_csr* slices,
                                     efem_stream_t stream) {
    if (!plans || nranks < 1 || !slices || (forms & ~7u)) {
        set_error("efem_dist_assemble_group: NULL arrays");
        return EFEM_EINVAL;
    }
    std::vector<DistPlan*> G(nranks);
    for (int r = 0; r < nranks; ++r) {
        G[r] = reinterpret_cast<DistPlan*>(plans[r]);
        if (!G[r] || G[r]->comm || G[r]->rank != r || G[r]->P != nranks || !slices[r].row_ptr) {
            set_error("efem_dist_assemble_group: plans of one local group, in rank order, and their slices");
            return EFEM_EINVAL;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    efem_status st;
    for (DistPlan* D : G)
        if ((st = ph_pack(*D, s)) != EFEM_OK) return st;
    auto sendA = [](DistPlan* d) { return std::make_pair((void*)d->sendA, std::cref(d->send_off)); };
    auto recvA = [](DistPlan* d) { return std::make_pair((void*)d->recvA, std::cref(d->recv_off)); };
    if ((st = group_alltoallv(G, sendA, recvA, REC_D * 8, s)) != EFEM_OK) return st;
    for (DistPlan* D : G)
        if ((st = ph_symbolic(*D, s)) != EFEM_OK) return st;
    for (DistPlan* src : G)  // all-gather of the totals
        for (DistPlan* dst : G)
            if (src != dst)
                EFEM_CUDA_TRY(cudaMemcpyAsync(dst->totals + 2 * src->rank, src->totals + 2 * src->rank, 16,
                                              cudaMemcpyDeviceToDevice, s));
    for (DistPlan* D : G)
        if ((st = ph_respond(*D, s)) != EFEM_OK) return st;
    auto resp = [](DistPlan* d) { return std::make_pair((void*)d->resp_ids, std::cref(d->resp_off)); };
    auto req = [](DistPlan* d) { return std::make_pair((void*)d->req_ids, std::cref(d->req_off)); };
    if ((st = group_alltoallv(G, resp, req, 4, s)) != EFEM_OK) return st;
    for (int r = 0; r < nranks; ++r)
        if ((st = ph_numeric(*G[r], forms, &slices[r], s)) != EFEM_OK) return st;
    return EFEM_OK;
}

efem_status efem_dist_check(efem_dist_plan plan, int64_t* window, efem_stream_t stream) {
    DistPlan* D = reinterpret_cast<DistPlan*>(plan);
    if (!D) return EFEM_EINVAL;
    return check_one(*D, window, (cudaStream_t)stream);
}

efem_status efem_dist_plan_destroy(efem_dist_plan plan) {
    delete reinterpret_cast<DistPlan*>(plan);
    return EFEM_OK;
}

}  // extern "C"
