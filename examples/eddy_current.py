"""The paper's 2D eddy-current experiment (Table 5) on the
CUDA path: NE0 mass + curl-curl stiffness (the hot path), the load F against
the global basis and the H(curl) error by the degree-6 vectorized integration
(SURVEY §8(f) f1), a Jacobi-CG solve of (K + M) v = b (f2).

    python examples/eddy_current.py [--sizes 128 256 ... 4096] [--rtol 1e-12]

Prints one row per mesh next to the paper's printed error (the paper's
timings are for MATLAB on a 2014 CPU; this compares results, not speed).
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import problems as P  # noqa: E402
from paper_1409_4618_b200 import api  # noqa: E402
from workloads import NED0  # noqa: E402


def run(n, rtol):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    c, e = api.build_mesh(2, n, 0.0, 0, device="cuda:0")
    torch.cuda.synchronize()
    ev[0].record()
    asm = api.Assembler(c, e, NED0)
    A = asm.assemble()
    ev[1].record()
    X = api.quad_points(c, e)
    x1, x2 = X[..., 0], X[..., 1]
    b = asm.load(torch.stack(P.eddy_F(x1, x2, torch), dim=-1), api.VALUE)
    ev[2].record()
    t0 = time.perf_counter()
    u, it, rr = api.cg(A, b, 1.0, 1.0, rtol=rtol)
    cg_s = time.perf_counter() - t0
    ev[3].record()
    err = asm.field_error(u, torch.stack(P.eddy_E(x1, x2, torch), dim=-1), P.eddy_curlE(x1, x2, torch).unsqueeze(-1))
    ev[4].record()
    torch.cuda.synchronize()
    err = err.cpu().numpy()
    return {"n": n, "T": int(e.shape[0]), "E": asm.n_rows, "error": math.sqrt(err[0] + err[1]), "cg_iters": it,
            "cg_relres": rr, "assemble_ms": ev[0].elapsed_time(ev[1]), "load_ms": ev[1].elapsed_time(ev[2]),
            "cg_s": cg_s, "error_ms": ev[3].elapsed_time(ev[4])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="*", default=[128, 256, 512, 1024, 2048])
    ap.add_argument("--rtol", type=float, default=1e-12)
    a = ap.parse_args()
    paper = {r["n"]: r for r in json.load(open(os.path.join(ROOT, "tests", "golden", "paper_table5_eddy.json")))["rows"]}
    print(f"{'#T':>10} {'#E':>10} {'error (CUDA)':>14} {'paper':>12} {'rel.diff':>9} {'CG it':>7} "
          f"{'assemble ms':>11} {'load ms':>8} {'CG s':>7} {'error ms':>8}")
    for n in a.sizes:
        r = run(n, a.rtol)
        p = paper.get(n, {}).get("error")
        rel = abs(r["error"] - p) / p if p else float("nan")
        print(f"{r['T']:>10} {r['E']:>10} {r['error']:>14.7e} {p if p else float('nan'):>12.6e} {rel:>9.1e} "
              f"{r['cg_iters']:>7} {r['assemble_ms']:>11.3f} {r['load_ms']:>8.3f} {r['cg_s']:>7.2f} "
              f"{r['error_ms']:>8.3f}", flush=True)


if __name__ == "__main__":
    main()
