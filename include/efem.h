/*
 * efem.h -- C-ABI of libefem.so: B200 (sm_100a) assembly of the global mass
 * and stiffness matrices of lowest-order Raviart-Thomas (RT0, H(div)) and
 * Nedelec (NE0, H(curl)) edge elements on affine triangle / tetrahedron
 * meshes into CSR.
 *
 * Paper: I. Anjam, J. Valdman, "Fast MATLAB assembly of FEM matrices in 2D and
 * 3D: Edge elements", arXiv:1409.4618.  "PAPER.md:N" cites line N of its LaTeX
 * source.  The four matrices are (Sec. 2.4)
 *     M_ij = int_Omega eta_i . eta_j,
 *     K_ij = int_Omega div eta_i div eta_j      (RT0)
 *     K_ij = int_Omega curl eta_i . curl eta_j  (NE0),
 * over the global, sign-corrected Piola-mapped basis (PAPER.md:240-245,
 * 291-331).  The readings of the paper this library takes (3D RT
 * normalisation, 3D sign rules, DOF order ...) are listed in DESIGN.md.
 *
 * Conventions shared by every call
 *   - All arrays are DEVICE memory owned by the caller (PyTorch tensors in
 *     the Python binding) unless a parameter name starts with h_.  The
 *     library never frees caller memory.
 *   - Every call that takes a cudaStream_t only enqueues work on that stream
 *     unless documented as "synchronising".
 *   - Indices are 0-based int32; meshes with > 2^31-1 entries are rejected
 *     with EFEM_EOVERFLOW.
 *   - Every call returns an efem_status; on error no output is guaranteed and
 *     efem_last_error() returns a thread-local message.
 */
#ifndef EFEM_H
#define EFEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* efem_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    EFEM_OK = 0,
    EFEM_EINVAL = -1,      /* bad argument: dim not in {2,3}, n < 1, NULL pointer, node id out of range,
                              jitter outside [0, 1/(2 sqrt(2 d))) ...; or a non-conforming mesh: an
                              edge (2D) / face (3D RT0) in more than two elements, or (3D NE0) an edge
                              whose tets do not form one fan (see efem_assemble_numeric) */
    EFEM_EDEGENERATE = -2, /* an element has det B_K == 0 (or non-finite); efem_last_bad_element() names it */
    EFEM_ENOMEM = -3,      /* host allocation failed */
    EFEM_EWORKSPACE = -4,  /* workspace NULL or smaller than efem_plan_create reported */
    EFEM_EOVERFLOW = -5,   /* a count does not fit int32 (nnz >= 2^31, T*(d+1) >= 2^31 ...) or
                              n_elems >= 2^27 (instance words e << 3 | k carry two flag bits) */
    EFEM_ECUDA = -6,       /* CUDA runtime error; message in efem_last_error() */
    EFEM_ENCCL = -7,       /* NCCL error (distributed entry points) */
    EFEM_ECAPACITY = -8,   /* a node touches more elements / owns more entities than the
                              per-thread capacity (EFEM_MAX_NODE_ELEMS etc.); mesh too irregular */
    EFEM_ESTATE = -9       /* calls made out of order (e.g. numeric before symbolic) */
} efem_status;

typedef enum {
    EFEM_RT0 = 0, /* Raviart-Thomas: 2D -> one DOF per edge (normal flux), 3D -> one per face */
    EFEM_NED0 = 1 /* Nedelec (first kind): one DOF per edge (tangential moment), 2D and 3D */
} efem_element;

/* forms bitmask for efem_assemble_numeric */
enum { EFEM_MASS = 1, EFEM_STIFF = 2, EFEM_PATTERN = 4, EFEM_ALL = 7 };

/* capacities of the per-thread register / local-memory lists */
enum { EFEM_MAX_NODE_ENTITIES = 64, EFEM_MAX_ROW_ELEMS = 32, EFEM_MAX_ROW_NNZ = 128 };

/* A mesh (nodes2coord, elems2nodes).
 *   coords : n_nodes x dim fp64, row-major (node i at coords[i*dim .. i*dim+dim-1])
 *   elems  : n_elems x (dim+1) int32, row-major; any vertex order (the sign
 *            data absorbs orientation). */
typedef struct {
    int32_t dim;
    int64_t n_nodes;
    int64_t n_elems;
    const double* coords;
    const int32_t* elems;
} efem_mesh;

/* Global DOF tables.
 *   dofs2nodes : n_dofs x 2 (edges) or x 3 (3D RT faces) int32, each row the
 *                ascending node ids of the entity; rows in lexicographic order
 *                (DOF id = rank; reading C10)
 *   elems2dofs : n_elems x m int32 (m = 3 / 4 / 6 local DOFs, Fig. 1 order)
 *   signs      : n_elems x m int8, +1 / -1 */
typedef struct {
    int64_t n_dofs;
    int32_t* dofs2nodes;
    int32_t* elems2dofs;
    int8_t* signs;
} efem_dofs;

/* CSR output; M and K share one pattern (all structural entries kept,
 * columns ascending within a row).  row_ptr: n_rows+1, col_idx/vals: nnz. */
typedef struct {
    int64_t n_rows;
    int64_t nnz;
    int32_t* row_ptr;
    int32_t* col_idx;
    double* vals_mass;
    double* vals_stiff;
} efem_csr;

typedef struct efem_plan_s* efem_plan;

/* ---- meshes (input generator, untimed) -------------------------------------- */

/* Sizes of the structured unit-square / unit-cube mesh with n cells per axis:
 * 2D -> (n+1)^2 nodes, 2 n^2 triangles; 3D -> (n+1)^3 nodes, 6 n^3 Kuhn tets. */
efem_status efem_mesh_sizes(int dim, int n, int64_t* n_nodes, int64_t* n_elems);

/* Seeded structured mesh (SPEC.md:49-58 for the split):
 * node id = i + (n+1) j (+ (n+1)^2 k); interior nodes jittered uniformly by
 * +-jitter_frac/n per axis from a SplitMix64 counter hash of (seed, node*dim+axis);
 * 2D cells split along the lower-left/upper-right diagonal, 3D cubes into the
 * 6 Kuhn tets around the (0,0,0)-(1,1,1) diagonal.  m->coords / m->elems must
 * point to caller-allocated device arrays of the sizes above; m->dim,
 * n_nodes, n_elems are filled in.  Bit-identical to the CPU oracle's
 * generator. */
efem_status efem_build_mesh(int dim, int n, double jitter_frac, uint64_t seed, double* coords, int32_t* elems,
                            efem_stream_t stream);

/* ---- plans ------------------------------------------------------------------- */

/* Create a host-side plan for assembling `element` on `mesh` (device arrays,
 * which must stay alive and unchanged while the plan is used).  Returns in
 * *ws_bytes the device workspace the plan needs (an upper bound derived from
 * n_nodes, n_elems).  No device work.  Errors: EFEM_EINVAL, EFEM_EOVERFLOW,
 * EFEM_ENOMEM. */
/* the paper's 2D timing domain, the L-shape
 * (0,1)^2 \ (1/2,1)^2 (Table 1), as the m x m unit-square grid
 * (m even) with the cells of the removed quadrant dropped; level L of
 * Table 1 is m = 2^(L+1) (#E = 9/4 m^2 + 2 m).  Nodes / cells row-major over
 * what remains, 2 triangles per cell as efem_build_mesh; jitter on interior
 * nodes only (the re-entrant edges are boundary).  Untimed input generator. */
efem_status efem_lshape_sizes(int m, int64_t* n_nodes, int64_t* n_elems);
efem_status efem_build_mesh_lshape(int m, double jitter_frac, uint64_t seed, double* coords, int32_t* elems,
                                   efem_stream_t stream);

efem_status efem_plan_create(efem_plan* plan, const efem_mesh* mesh, efem_element element, size_t* ws_bytes);

/* Attach the caller-allocated device workspace (>= *ws_bytes, 256-byte
 * aligned).  Contents are the plan's state between the calls below; the
 * caller must not touch it. */
efem_status efem_plan_set_workspace(efem_plan plan, void* ws, size_t ws_bytes);

efem_status efem_plan_destroy(efem_plan plan);

/* NE0 3D only (no-op otherwise): size every edge row from the exact number of
 * distinct link vertices (slower symbolic pass) instead of the manifold
 * closed form 1 + 3t + 2[boundary] (reading M1), for meshes with
 * non-manifold edges.  Takes effect at the next symbolic call. */
efem_status efem_plan_set_exact(efem_plan plan, int exact);

/* ---- the hot path ------------------------------------------------------------ */

/* DOF enumeration + orientation (Sec. 3 get_edges /
 * get_faces / signs_edges / signs_faces).  Synchronising (reads n_dofs back).
 * out->n_dofs is always set.  If out->dofs2nodes / elems2dofs / signs are
 * non-NULL they are filled (each may be NULL independently).  Idempotent:
 * a second call on the same plan only copies the tables out. */
efem_status efem_enumerate_dofs(efem_plan plan, efem_dofs* out, efem_stream_t stream);

/* Symbolic assembly: DOF enumeration + CSR sparsity pattern sizes, always
 * recomputed from the mesh arrays (the mesh may have changed since the last
 * call; 2D: the node-fan pipeline, 3D: the bucket pipeline): the structural
 * pattern is the union over elements of dofs(K) x dofs(K) (PAPER.md:696,
 * reading C9).  Synchronising (reads n_rows / nnz back).  If row_ptr != NULL
 * it receives the n_rows+1 row offsets.  Returns EFEM_EOVERFLOW when
 * nnz >= 2^31. */
efem_status efem_assemble_symbolic(efem_plan plan, int64_t* n_rows, int64_t* nnz, int32_t* row_ptr,
                                   efem_stream_t stream);

/* Numeric assembly into caller-allocated CSR arrays (sizes from symbolic):
 * local matrices computed in fp64 registers and summed
 * per row in ascending element order.  Every row's column set is re-derived
 * here and compared with the symbolic row length; a mismatch (a mesh the
 * closed-form row lengths do not describe: 3D NE0 rows are sized
 * 1 + 3t + 2[edge on the boundary], valid when the tets around every edge
 * form one fan, a cycle or a path) is reported by efem_plan_check as
 * EFEM_EINVAL, never as wrong values.  forms: EFEM_PATTERN writes row_ptr and
 * col_idx, EFEM_MASS vals_mass, EFEM_STIFF vals_stiff (NULL allowed for
 * arrays whose bit is clear).  Asynchronous: degenerate elements are
 * reported by efem_plan_check. */
efem_status efem_assemble_numeric(efem_plan plan, unsigned forms, efem_csr* out, efem_stream_t stream);

/* The whole hot path in one asynchronous call, for repeated assembly into an
 * output allocated from an earlier efem_assemble_symbolic of the same (or a
 * topologically identical) mesh: enumeration, pattern and values are all
 * recomputed on the device, the row and entry counts stay on the device
 * (no host round trip); out->n_rows / out->nnz are the CAPACITIES.  A
 * pattern that does not fit is flagged (EFEM_ECAPACITY) and nothing is
 * written.  Follow with efem_plan_check, which also makes the new sizes the
 * plan's (efem_assemble_numeric may then be called).  Never synchronises. */
efem_status efem_assemble_async(efem_plan plan, unsigned forms, efem_csr* out, efem_stream_t stream);

/* Synchronising: returns EFEM_EDEGENERATE / EFEM_ECAPACITY if a kernel since
 * the last check flagged one, else EFEM_OK (or EFEM_ECUDA). */
efem_status efem_plan_check(efem_plan plan, efem_stream_t stream);

/* The device half of efem_plan_check: enqueues the read-back of the flags
 * and sizes (one small D2H copy into the plan's pinned buffer) without
 * waiting, so a timing event recorded after it brackets all device work of
 * a step; efem_plan_check then waits and decodes (it copies again, so the
 * result is never stale).  Never synchronises. */
efem_status efem_plan_check_async(efem_plan plan, efem_stream_t stream);

/* End-to-end convenience used for the "e2e" number: HOST mesh in, HOST CSR
 * out.  Copies h_coords / h_elems into the plan's device mesh arrays (the
 * plan must have been created on device arrays of the same sizes), runs
 * symbolic + numeric, checks, and copies row_ptr / col_idx / vals back into
 * h_out (host arrays with capacity h_out->nnz, h_out->n_rows+1 set by the
 * caller from a previous symbolic call).  d_out are device CSR arrays of the
 * same capacity.  Synchronising. */
efem_status efem_assemble_host(efem_plan plan, const double* h_coords, const int32_t* h_elems, efem_csr* d_out,
                               efem_csr* h_out, efem_stream_t stream);

/* ---- partitioned (multi-GPU) assembly, SURVEY.md §8(e) / DESIGN.md §9 ---------------
 * Rank r owns the rows of the entities whose minimum node lies in [node_lo,
 * node_hi); with contiguous node ranges these are contiguous global rows, so
 * the ranks' CSR slices concatenate to the 1-GPU matrix byte for byte.  Each
 * rank assembles from a two-hop sub-mesh (elements touching the nodes of the
 * elements touching its range); the exchange is an allgather of per-node
 * entity counts (done by the caller, e.g. torch.distributed / NCCL). */

/* Sub-mesh of `full` for the node range.  Call with ws == NULL to get
 * *ws_bytes; then with ws and sub_coords == NULL (synchronising) for the
 * sizes; then with caller-allocated sub_coords (n_sub_nodes x dim),
 * sub_elems (n_sub_elems x (dim+1), local node ids) and sub2global
 * (n_sub_nodes, ascending global node ids), same ws untouched in between. */
efem_status efem_partition(const efem_mesh* full, int64_t node_lo, int64_t node_hi, void* ws, size_t* ws_bytes,
                           int64_t* n_sub_nodes, int64_t* n_sub_elems, double* sub_coords, int32_t* sub_elems,
                           int32_t* sub2global, efem_stream_t stream);

/* After efem_assemble_symbolic on the sub-mesh plan: owned_cnt[g - node_lo] =
 * number of entities whose minimum node is global node g (device, node_hi -
 * node_lo ints, the rank's contribution to the allgather); info (host, 4) =
 * {first owned local row, owned rows, local CSR offset of that row, owned CSR
 * entries}.  Synchronising. */
efem_status efem_part_counts(efem_plan plan, const int32_t* sub2global, int64_t node_lo, int64_t node_hi,
                             int32_t* owned_cnt, int64_t* info, efem_stream_t stream);

/* Exclusive scan of the allgathered per-node counts (n = global node count)
 * into global_ent_ptr (n+1): the global id of node g's first entity.  ws ==
 * NULL returns *ws_bytes. */
efem_status efem_part_scan(const int32_t* global_cnt, int64_t n, int32_t* global_ent_ptr, void* ws, size_t* ws_bytes,
                           efem_stream_t stream);

/* elems2dofs of the sub-mesh in global DOF ids (n_sub_elems x m, device). */
efem_status efem_part_globalize(efem_plan plan, const int32_t* sub2global, const int32_t* global_ent_ptr,
                                int32_t* e2d_global, efem_stream_t stream);

/* The owned rows as a CSR slice with global column ids: slice->row_ptr
 * starts at 0 (add the rank's global entry offset to place it); n_rows / nnz
 * must equal info[1] / info[3]; global_first_row = global_ent_ptr[node_lo]. */
efem_status efem_part_numeric(efem_plan plan, unsigned forms, const int64_t* info, int64_t global_first_row,
                              const int32_t* e2d_global, efem_csr* slice, efem_stream_t stream);

/* ---- partitioned assembly, asynchronous form ---------------------------------------
 * The same computation as efem_part_counts / _scan / _globalize / _numeric,
 * with every size kept on the device, so a rank's step needs no host round
 * trip before efem_plan_check (which reports capacity overflow and the mesh
 * flags).  Per step, all enqueued on one stream:
 *   efem_part_enumerate_async(plan, owned_cnt)   enumeration of the sub-mesh,
 *        owned_cnt as for efem_part_counts, and the row window on the device
 *   [caller: allgather of owned_cnt -> global_cnt]
 *   efem_part_scan(global_cnt, ...)  ->  global_ent_ptr
 *   efem_part_globalize(plan, sub2global, global_ent_ptr, e2d_global)
 *        (also records the window's global first row global_ent_ptr[node_lo])
 *   efem_part_numeric_async(plan, forms, e2d_global, slice)
 *   efem_plan_check(plan)
 * DESIGN.md §9. */

/* Binds the sub-mesh plan (workspace set) to the rank's node range: finds
 * the local node range of [node_lo, node_hi) in sub2global (ascending;
 * device, kept by pointer until the next bind).  Synchronising; once per
 * partition.  EFEM_EINVAL on NULL / bad range. */
efem_status efem_part_bind(efem_plan plan, const int32_t* sub2global, int64_t node_lo, int64_t node_hi,
                           efem_stream_t stream);

/* Enumeration of a bound plan plus the owned counts: owned_cnt (device,
 * node_hi - node_lo ints) as efem_part_counts writes them; the row window
 * {first owned local row, owned rows, local CSR offset of that row, owned
 * entries} stays on the device.  Asynchronous (one CUDA graph per owned_cnt
 * array).  EFEM_ESTATE if the plan is not bound. */
efem_status efem_part_enumerate_async(efem_plan plan, int32_t* owned_cnt, efem_stream_t stream);

/* The owned rows into `slice` (device; slice->n_rows / nnz are CAPACITIES,
 * the window's sizes are read on the device): row_ptr from 0, global column
 * ids.  A window larger than the capacities writes nothing and makes
 * efem_plan_check return EFEM_ECAPACITY.  Needs efem_part_enumerate_async
 * and efem_part_globalize before it on the stream. */
efem_status efem_part_numeric_async(efem_plan plan, unsigned forms, const int32_t* e2d_global, efem_csr* slice,
                                    efem_stream_t stream);

/* Copies the device window {first owned local row, owned rows, local CSR
 * offset, owned entries, global first row} (5 int64) into window_dev
 * (device), e.g. for an allgather of the owned entry counts. */
efem_status efem_part_window(efem_plan plan, int64_t* window_dev, efem_stream_t stream);

/* ---- O(interface) exchange for the owner-computes partition ------------
 * Instead of all-gathering every node's entity count (O(N) per rank), each
 * rank scans its owned counts (efem_part_scan over its width), the ranks
 * all-gather their totals (one int each), efem_part_add_offset turns the
 * local prefix into global first DOF ids, and every rank answers only the
 * first ids of its nodes that other ranks' sub-meshes hold (ghost nodes):
 * efem_index_gather (dst[j] = src[idx[j] + bias]) builds the answers and the
 * owned part of the sub-mesh's first ids, efem_index_scatter (dst[idx[j]] =
 * src[j]) places the received ones.  efem_part_globalize_sub then maps
 * elems2dofs to global ids from those per-SUB-MESH-node first ids (sub_first,
 * device, n_sub_nodes) and records the window's global first row
 * (sub_first[l0]; [l0, l1) = the owned sub-mesh nodes). */
efem_status efem_part_add_offset(int32_t* first, int64_t n, const int32_t* totals, int rank, efem_stream_t stream);
efem_status efem_index_gather(int32_t* dst, const int32_t* src, const int32_t* idx, int64_t n, int32_t bias,
                              efem_stream_t stream);
efem_status efem_index_scatter(int32_t* dst, const int32_t* idx, const int32_t* src, int64_t n, efem_stream_t stream);
efem_status efem_part_globalize_sub(efem_plan plan, const int32_t* sub_first, int64_t l0, int64_t l1,
                                    int32_t* e2d_global, efem_stream_t stream);

/* ---- distributed 2D assembly over NCCL (BASELINE north_star) -----------
 * The elements are split into contiguous slabs, one per rank (one process
 * per GPU).  Rank r owns the nodes [lo_r, lo_{r+1}), lo_r = the smallest
 * vertex of its slab (made non-decreasing; lo_0 = 0, lo_P = n_nodes), hence
 * the edges whose smaller node it owns: the contiguous block of global rows
 * [first_row, first_row + rows) of M and K (DOF ids are lexicographic in the
 * sorted node pair; the global matrices PAPER.md:335-342).
 * Per step a rank computes the local matrices of its own
 * slab only and sends those of the triangles holding another rank's rows to
 * that rank (grouped ncclSend / ncclRecv), the ranks all-gather their row /
 * entry totals, and the owners answer the ids of the columns they own; each
 * rank then writes its CSR slice: row_ptr from 0, global column ids, values
 * summed in ascending element order.  The slices concatenated in rank order
 * are the 1-GPU matrices (pattern byte for byte).  NCCL is called by this
 * library; the caller only moves the 128-byte unique id between processes.
 * Triangles (dim 2) only; 3D meshes use efem_part_* (owner computes). */
typedef struct efem_comm_s* efem_comm;
typedef struct efem_dist_plan_s* efem_dist_plan;

/* A fresh ncclUniqueId (128 bytes) into id (host), on one rank. */
efem_status efem_comm_unique_id(unsigned char* id);
/* ncclCommInitRank over the given id; collective over the nranks processes
 * (blocking).  The CUDA device current at the call is the rank's device. */
efem_status efem_comm_init(efem_comm* comm, const unsigned char* id, int nranks, int rank);
efem_status efem_comm_destroy(efem_comm comm);

/* Setup of one rank (collective, synchronising, untimed): mesh = the whole
 * mesh in this rank's device memory (dim 2; kept by pointer: coordinates are
 * read at every step, the connectivity at this setup -- it fixes the plan's
 * communication pattern, so it must not change afterwards), the rank's
 * slab [elem_lo, elem_hi) of it, comm from efem_comm_init.  Computes the node
 * ranges and the communication pattern (which triangles go to which rank,
 * which column ids each rank answers) and allocates the plan's own device
 * buffers (freed by efem_dist_plan_destroy).  EFEM_EINVAL: not a 2D mesh,
 * bad slab, node id out of range; EFEM_ENCCL / EFEM_ECUDA. */
efem_status efem_dist_plan_create(efem_dist_plan* plan, const efem_mesh* mesh, efem_element element, int64_t elem_lo,
                                  int64_t elem_hi, efem_comm comm, efem_stream_t stream);

/* The same for all nranks ranks of a LOCAL GROUP inside one process on one
 * device (elem_bounds: nranks + 1 non-decreasing slab bounds, 0 ..
 * n_elems): every exchange becomes a device-to-device copy.  For testing
 * the multi-rank logic where only one GPU exists; plans[r] is rank r. */
efem_status efem_dist_group_create(efem_dist_plan* plans, int nranks, const efem_mesh* mesh, efem_element element,
                                   const int64_t* elem_bounds, efem_stream_t stream);

/* Host-only: the partition this library computes at setup, for rank `rank`
 * of nranks over the HOST copy h_elems of a 2D mesh split at elem_bounds
 * (nranks + 1): out (host, 3 + nranks) = {owned nodes lo, hi, kept slab
 * triangles, triangles sent to rank 0 .. nranks-1}.  No device work (used
 * by the CPU tests of the multi-rank logic). */
efem_status efem_dist_layout(const int32_t* h_elems, int64_t n_nodes, int64_t n_elems, const int64_t* elem_bounds,
                             int nranks, int rank, int64_t* out);

/* info (host, 8): owned nodes lo, hi; kept slab triangles; ghost triangles
 * received; triangles sent; column ids requested; ids answered; bytes this
 * rank sends per step. */
efem_status efem_dist_info(efem_dist_plan plan, int64_t* info);

/* One step on this rank (collective; asynchronous on the stream): the slice
 * (device) has CAPACITIES slice->n_rows / nnz; a window larger than them is
 * not written and makes efem_dist_check return EFEM_ECAPACITY (a first call
 * with zero capacities is the size query).  forms as efem_assemble_numeric. */
efem_status efem_dist_assemble(efem_dist_plan plan, unsigned forms, efem_csr* slice, efem_stream_t stream);

/* One step of every rank of a local group (slices[r] for rank r). */
efem_status efem_dist_assemble_group(efem_dist_plan* plans, int nranks, unsigned forms, efem_csr* slices,
                                     efem_stream_t stream);

/* Synchronising: window (host, 4) = {global first row, rows, global offset of
 * the first entry, entries} of the last step; the step's status
 * (EFEM_EDEGENERATE / EFEM_ECAPACITY / EFEM_EINVAL for a non-conforming mesh). */
efem_status efem_dist_check(efem_dist_plan plan, int64_t* window, efem_stream_t stream);
efem_status efem_dist_plan_destroy(efem_dist_plan plan);

/* ---- vectorized integration (Sec. 3.1)
 * The paper's recipe: map the quadrature points of the reference element to
 * every element at once, evaluate the user's function there (the caller does
 * this, vectorized, on the device), then reduce per element.  Degree-6 rules
 * (PAPER.md:637, 648): 12 points per triangle (Dunavant), 24 per
 * tetrahedron (Keast).  Point order within an element (fq rows follow it):
 * each symmetry orbit in turn -- 2D: (a,b,b) orbits as (l0,l1,l2) = (a,b,b),
 * (b,a,b), (b,b,a), then the 6-point orbit in lexicographic permutation
 * order; 3D: the four (a,a,a,b) orbits as (b,a,a,a)..(a,a,a,b) with l0 first,
 * then the 12-point orbit with a at slots i0 < i1, b at i2, c at i3 in
 * lexicographic (i0, i1, i2) order; the point is (l1, l2[, l3]). */
enum { EFEM_PAIR_VALUE = 0, EFEM_PAIR_DERIV = 1 };

/* points per element of the degree-6 rule: 12 (dim 2), 24 (dim 3); 0 otherwise */
int efem_quad_size(int dim);

/* pts (device, n_elems x nq x dim): F_K(xh_q) = B_K xh_q + b_K. */
efem_status efem_quad_points(const efem_mesh* mesh, double* pts, efem_stream_t stream);

/* Load vector b (device, n_dofs) after efem_assemble_symbolic:
 *   b_i = sum_K sum_q w_q |det B_K| f(x_q) . phi_i(x_q)          pairing EFEM_PAIR_VALUE, fq: T x nq x dim
 *   b_i = sum_K sum_q w_q |det B_K| f(x_q) . (D phi_i)(x_q)      pairing EFEM_PAIR_DERIV, fq: T x nq x nd
 * phi_i the global, sign-corrected Piola-mapped basis (PAPER.md:240-245,
 * 291-331), D = div (RT, nd = 1), curl (Ned 2D nd = 1, 3D nd = 3).  Summed
 * per DOF over its elements in ascending element order (deterministic). */
efem_status efem_assemble_load(efem_plan plan, int pairing, const double* fq, double* b, efem_stream_t stream);

/* ||f||^2 = sum_K sum_q w_q |det B_K| |f(x_q)|^2 (the norm_L2 listing,
 * PAPER.md:633-645).  fq: T x nq x nf (device); per_elem (device, T) gets
 * ||f||^2_K, total (device, 1 double) their fixed-order sum.  ws == NULL
 * returns *ws_bytes. */
efem_status efem_norm_l2(const efem_mesh* mesh, const double* fq, int nf, double* per_elem, double* total, void* ws,
                         size_t* ws_bytes, efem_stream_t stream);

/* Error of v = sum_i coeffs_i phi_i (after symbolic): err2 (device, 2) =
 * { ||E - v||^2, ||D E - D v||^2 } from exact values Eq (T x nq x dim) and
 * Dq (T x nq x nd) at the quadrature points.  ws == NULL returns *ws_bytes. */
efem_status efem_field_error(efem_plan plan, const double* coeffs, const double* Eq, const double* Dq, double* err2,
                             void* ws, size_t* ws_bytes, efem_stream_t stream);

/* y = alpha K x + beta M x on an assembled CSR (vals_stiff = K, vals_mass = M). */
efem_status efem_spmv(const efem_csr* A, double alpha, double beta, const double* x, double* y,
                      efem_stream_t stream);

/* Jacobi-preconditioned conjugate gradients for (alpha K + beta M) x = b
 * (SPD for alpha, beta > 0): x (device) is the initial guess on entry, the
 * iterate on return; stops when ||r|| <= rtol ||b|| (checked every 20
 * iterations) or after maxit.  Synchronising.  ws == NULL returns *ws_bytes. */
efem_status efem_cg(const efem_csr* A, double alpha, double beta, const double* b, double* x, double rtol, int maxit,
                    int* iters, double* relres, void* ws, size_t* ws_bytes, efem_stream_t stream);

/* ---- SURVEY.md §8(f) f3 support: linear nodal (P1) elements ------------------
 * The majorant example's approximation v.  Rows = nodes; the
 * pattern of row a is a and every node sharing an element with it (sorted);
 * vals_stiff = int grad l_a . grad l_b, vals_mass = int l_a l_b, summed per row
 * in ascending element order.  Same two-phase protocol as efem_plan. */
typedef struct efem_p1_plan_s* efem_p1_plan;

efem_status efem_p1_plan_create(efem_p1_plan* plan, const efem_mesh* mesh, size_t* ws_bytes);
efem_status efem_p1_plan_set_workspace(efem_p1_plan plan, void* ws, size_t ws_bytes);
efem_status efem_p1_plan_destroy(efem_p1_plan plan);
/* node -> element incidence, row lengths; synchronising (returns n_rows = n_nodes, nnz);
 * EFEM_ECAPACITY if a node touches more than 64 elements or 63 neighbours */
efem_status efem_p1_symbolic(efem_p1_plan plan, int64_t* n_rows, int64_t* nnz, efem_stream_t stream);
/* row_ptr, col_idx, vals_mass (may be NULL), vals_stiff (may be NULL); synchronising (degenerate check) */
efem_status efem_p1_numeric(efem_p1_plan plan, efem_csr* out, efem_stream_t stream);
/* b_a = sum_K sum_q w_q |det B_K| f(x_q) l_a(x_q); fq: T x nq (degree-6 points, efem_quad_points order) */
efem_status efem_p1_load(efem_p1_plan plan, const double* fq, double* b, efem_stream_t stream);
/* grad v (piecewise constant) written at every quadrature point: grad_q T x nq x dim */
efem_status efem_p1_gradient(const efem_mesh* mesh, const double* v, double* grad_q, efem_stream_t stream);
/* Symmetric Dirichlet elimination on a CSR in place: entries in masked rows or
 * columns set to 0 (vals_stiff diagonal of masked rows to 1, vals_mass 0);
 * b[masked] = 0 (b may be NULL).  For homogeneous boundary values. */
efem_status efem_dirichlet(efem_csr* A, const uint8_t* mask, double* b, efem_stream_t stream);

/* ---- diagnostics ------------------------------------------------------------- */
const char* efem_status_string(efem_status status);
const char* efem_last_error(void);
int64_t efem_last_bad_element(void);
/* number of kernel launches issued by the library since process start */
int64_t efem_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* EFEM_H */
