"""The paper's functional-majorant example (Algorithm 1,
Tables 3-4) on the CUDA path:

  v   = P1 solution of -lap u = f, u = 0 on the boundary (bubble u);
  (a) RT0: ((1+beta) C_F^2 K + (1+1/beta) M) y = -(1+beta) C_F^2 (f, div phi) + (1+1/beta) (grad v, phi)
  (b) beta = ||grad v - y|| / (C_F ||div y + f||)
  stop when the majorant changes by less than 1e-4 (relative).

    python examples/majorant.py [--dim 2] [--sizes 16 256 1024 4096]

Prints (iteration, beta, sqrt(majorant), I_eff) per mesh, with the paper's
printed values (reading F1 in DESIGN.md: the printed M is the square root of
the Young-split majorant, beta / I_eff are truncated to the shown digits).
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
from workloads import RT0  # noqa: E402


def run(dim, n, max_iter=8, stop=1e-4, rtol=1e-12):
    """Algorithm 1 on the GPU; returns ([(beta, sqrt M, I_eff)], ||grad(u - v)||^2, timings)."""
    t = {}
    t0 = time.perf_counter()
    c, e = api.build_mesh(dim, n, 0.0, 0, device="cuda:0")
    X = api.quad_points(c, e)
    F = P.bubble_f(X, torch)
    # v: P1 Poisson solve, homogeneous Dirichlet on the boundary of (0,1)^d
    p1 = api.P1Assembler(c, e)
    K1 = p1.assemble()
    b1 = p1.load(F)
    bnd = ((c.abs() < 1e-14) | ((c - 1.0).abs() < 1e-14)).any(dim=1)
    api.dirichlet(K1, bnd, b1)
    v, it_v, _ = api.cg(K1, b1, 1.0, 0.0, rtol=rtol)
    GV = api.p1_gradient(c, e, v)
    err2 = api.norm_l2(c, e, P.bubble_grad(X, torch) - GV)[0].item()
    torch.cuda.synchronize()
    t["p1_s"] = time.perf_counter() - t0
    # RT0 matrices once, the two loads once
    t0 = time.perf_counter()
    asm = api.Assembler(c, e, RT0)
    A = asm.assemble()
    b_div = asm.load(F.unsqueeze(-1), api.DERIVATIVE)
    b_val = asm.load(GV, api.VALUE)
    torch.cuda.synchronize()
    t["rt_assemble_s"] = time.perf_counter() - t0
    CF = P.friedrichs_unit(dim)
    beta, prev, hist, y = 1.0, None, [], None
    t0 = time.perf_counter()
    for _ in range(max_iter):
        a1, a2 = (1.0 + beta) * CF ** 2, 1.0 + 1.0 / beta
        y, _, _ = api.cg(A, -a1 * b_div + a2 * b_val, a1, a2, x0=y, rtol=rtol)
        d = asm.field_error(y, GV, -F.unsqueeze(-1)).cpu()
        d1, d2 = float(d[0]), float(d[1])
        Mcal = a2 * d1 + a1 * d2
        hist.append((beta, math.sqrt(Mcal), math.sqrt(Mcal / err2)))
        if prev is not None and abs(prev - Mcal) / prev < stop:
            break
        prev = Mcal
        beta = math.sqrt(d1) / (CF * math.sqrt(d2))
    t["algorithm_s"] = time.perf_counter() - t0
    return hist, err2, t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--sizes", type=int, nargs="*", default=None)
    a = ap.parse_args()
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_table3_4_majorant.json")))
    tab = g["table3_2d"] if a.dim == 2 else g["table4_3d"]
    sizes = a.sizes or (tab["n"] if a.dim == 2 else [12, 24, 48, 96])
    for n in sizes:
        hist, err2, t = run(a.dim, n)
        T = (2 if a.dim == 2 else 6) * n ** a.dim
        paper = None
        if T in tab["T"]:
            paper = tab["rows"][tab["T"].index(T)]
        print(f"#T = {T}  ||grad(u-v)|| = {math.sqrt(err2):.6e}  P1 {t['p1_s']:.2f}s  RT0 {t['rt_assemble_s']:.2f}s  "
              f"Alg.1 {t['algorithm_s']:.2f}s", flush=True)
        for i, (beta, sm, ieff) in enumerate(hist):
            pp = paper[i] if paper and i < len(paper) else None
            ps = f"   paper: {pp[1]:.3f} {pp[2]:.6f} {pp[3]:.2f}" if pp else ""
            print(f"  iter {i + 1}: beta {beta:.4f}  M {sm:.7f}  I_eff {ieff:.4f}{ps}", flush=True)


if __name__ == "__main__":
    main()
