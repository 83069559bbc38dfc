/* Plain-C use of the boundary (include/efem.h, libefem.so): build config 2's
 * mesh recipe at a small size on the device, assemble NE0 M and K into CSR,
 * check the sizes against the closed forms and both
 * matrices for symmetry on the host.  No Python, no torch.
 *
 *   gcc -std=c11 -O2 examples/c_abi_example.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1409_4618_b200 -lefem -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1409_4618_b200 -o /tmp/efem_c && /tmp/efem_c 64
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "efem.h"

#define CK(x)                                                                              \
    do {                                                                                   \
        efem_status s_ = (x);                                                              \
        if (s_ != EFEM_OK) {                                                               \
            fprintf(stderr, "%s: %s (%s)\n", #x, efem_status_string(s_), efem_last_error()); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)
#define CU(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
            return 1;                                                           \
        }                                                                       \
    } while (0)

/* value of entry (i, j) of a CSR matrix (columns ascending), NAN if absent */
static double at(const int32_t* rp, const int32_t* ci, const double* v, int i, int j) {
    int lo = rp[i], hi = rp[i + 1];
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (ci[mid] < j) lo = mid + 1; else hi = mid;
    }
    return lo < rp[i + 1] && ci[lo] == j ? v[lo] : NAN;
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 64;
    int64_t N = 0, T = 0;
    CK(efem_mesh_sizes(2, n, &N, &T));
    double* coords;
    int32_t* elems;
    CU(cudaMalloc((void**)&coords, (size_t)N * 2 * sizeof(double)));
    CU(cudaMalloc((void**)&elems, (size_t)T * 3 * sizeof(int32_t)));
    CK(efem_build_mesh(2, n, 0.2, 1, coords, elems, NULL));  /* config 2's jitter and seed */

    efem_mesh mesh = {2, N, T, coords, elems};
    efem_plan plan;
    size_t ws_bytes = 0;
    void* ws;
    CK(efem_plan_create(&plan, &mesh, EFEM_NED0, &ws_bytes));
    CU(cudaMalloc(&ws, ws_bytes));
    CK(efem_plan_set_workspace(plan, ws, ws_bytes));

    int64_t R = 0, nnz = 0;
    CK(efem_assemble_symbolic(plan, &R, &nnz, NULL, NULL));
    efem_csr A = {R, nnz, NULL, NULL, NULL, NULL};
    CU(cudaMalloc((void**)&A.row_ptr, (size_t)(R + 1) * 4));
    CU(cudaMalloc((void**)&A.col_idx, (size_t)nnz * 4));
    CU(cudaMalloc((void**)&A.vals_mass, (size_t)nnz * 8));
    CU(cudaMalloc((void**)&A.vals_stiff, (size_t)nnz * 8));
    CK(efem_assemble_numeric(plan, EFEM_ALL, &A, NULL));
    CK(efem_plan_check(plan, NULL));

    int ok = R == 3LL * n * n + 2LL * n && nnz == 15LL * n * n + 2LL * n;  /* closed forms */
    int32_t* rp = malloc((size_t)(R + 1) * 4);
    int32_t* ci = malloc((size_t)nnz * 4);
    double* vm = malloc((size_t)nnz * 8);
    double* vk = malloc((size_t)nnz * 8);
    CU(cudaMemcpy(rp, A.row_ptr, (size_t)(R + 1) * 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(ci, A.col_idx, (size_t)nnz * 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(vm, A.vals_mass, (size_t)nnz * 8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(vk, A.vals_stiff, (size_t)nnz * 8, cudaMemcpyDeviceToHost));
    double asym = 0.0, trace_m = 0.0;  /* max |A_ij - A_ji| / max_j |A_ij| over M and K */
    for (int i = 0; i < R; ++i) {
        double sm = 0.0, sk = 0.0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            sm = fmax(sm, fabs(vm[p]));
            sk = fmax(sk, fabs(vk[p]));
        }
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const int j = ci[p];
            const double mt = at(rp, ci, vm, j, i), kt = at(rp, ci, vk, j, i);
            /* (a missing transposed entry is NAN and fails the test below) */
            asym = fmax(asym, fmax(fabs(vm[p] - mt) / sm, fabs(vk[p] - kt) / sk));
            if (j == i) {
                trace_m += vm[p];
                ok &= vm[p] > 0.0;  /* SPD mass matrix: positive diagonal */
            }
        }
    }
    ok &= asym <= 1e-12;  /* symmetric pattern, values to rounding (north_star's tolerance) */
    printf("n=%d  elements=%lld  dofs=%lld  nnz=%lld  max|A-A^T|/rowmax=%g  tr(M)=%.12g  %s\n", n, (long long)T,
           (long long)R, (long long)nnz, asym, trace_m, ok ? "OK" : "FAILED");
    free(rp), free(ci), free(vm), free(vk);
    cudaFree(A.row_ptr), cudaFree(A.col_idx), cudaFree(A.vals_mass), cudaFree(A.vals_stiff);
    efem_plan_destroy(plan);
    cudaFree(ws), cudaFree(coords), cudaFree(elems);
    return ok ? 0 : 2;
}
