"""Measurement of the SURVEY §8(f) NEXT-row kernels (f1 loads / norms /
field errors, f2 SpMV and a CG iteration) on config 2's mesh: device time
per call (CUDA events, L2 flushed before each call, median of reps) and the
achieved fraction of the measured HBM copy peak, counting ALGORITHMIC bytes
(stated per kernel below).  Prints a table; `python tools/f_rows_bench.py`.

Algorithmic bytes per call (2D, T elements, N nodes, R DOFs, nq = 12 points):
  quad_points   mesh in (N*16 + T*12) + points out T*nq*2*8
  load (value)  mesh + elems2dofs T*12 + f at points T*nq*2*8 in + b R*8 out
  norm_l2 (nf=2) mesh + f T*nq*2*8 in + per-element T*8 out
  field_error   mesh + elems2dofs + coefficients R*8 + E T*nq*2*8 + curl E T*nq*8 in
  spmv          CSR (R+1)*4 + nnz*(4+8+8) + x R*8 in + y R*8 out
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from workloads import CONFIGS, counts  # noqa: E402

C = CONFIGS[2]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.0)
coords, elems = api.build_mesh(2, C["n"], C["alpha"], C["seed"], device="cuda:0")
asm = api.Assembler(coords, elems, C["element"])
A = asm.assemble()
N, T, R, nnz = counts(2, C["element"], C["n"])
nq = api.quad_size(2)
X = api.quad_points(coords, elems)
F = torch.randn((T, nq, 2), dtype=torch.float64, device="cuda")
D = torch.randn((T, nq, 1), dtype=torch.float64, device="cuda")
u = torch.randn(R, dtype=torch.float64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
mesh_b = N * 16 + T * 12


def timed(fn, reps=15):
    ts = []
    for r in range(reps):
        flush.fill_(r & 0xff)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


rows = [
    ("quad_points", lambda: api.quad_points(coords, elems), mesh_b + T * nq * 2 * 8),
    ("load (value pairing)", lambda: asm.load(F, api.VALUE), mesh_b + T * 12 + T * nq * 2 * 8 + R * 8),
    ("norm_l2 (nf = 2)", lambda: api.norm_l2(coords, elems, F), mesh_b + T * nq * 2 * 8 + T * 8),
    ("field_error", lambda: asm.field_error(u, F, D), mesh_b + T * 12 + R * 8 + T * nq * 3 * 8),
    ("spmv (K + M)", lambda: api.spmv(A, u, 1.0, 1.0), (R + 1) * 4 + nnz * 20 + R * 16),
]
print(f"config 2 mesh: T = {T}, R = {R}, nnz = {nnz}; HBM peak {peak:.0f} GB/s (MEASURED_PEAKS.json)")
print(f"{'kernel':24s} {'ms':>8s} {'alg. MB':>9s} {'GB/s':>8s} {'frac':>6s}")
for name, fn, b in rows:
    ms = timed(fn)
    print(f"{name:24s} {ms:8.4f} {b / 1e6:9.1f} {b / (ms * 1e-3) / 1e9:8.0f} {b / (ms * 1e-3) / 1e9 / peak:6.3f}")
# a CG iteration: run a fixed number of iterations and divide
b = asm.load(F, api.VALUE)
for it_n in (1, 101):
    t = timed(lambda: api.cg(A, b, 1.0, 1.0, rtol=1e-300, maxit=it_n), reps=5)
    if it_n == 1:
        t1 = t
    else:
        per = (t - t1) / 100
print(f"{'CG iteration (K + M)':24s} {per:8.4f}   (spmv + 2 dot + 3 axpy + Jacobi; Python-free loop in efem_cg)")
