"""Benchmark: end-to-end RT0 / NE0 assembly (symbolic + numeric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl efem|reference]

One JSON line on rank 0.  A "step" is one pass of the whole hot path over the
device-resident mesh of the chosen BASELINE config: DOF enumeration + signs,
sparsity pattern, local matrices and CSR values (efem_assemble_async, i.e.
enumeration + pattern + numeric with the counts kept on the device, then the
read-back of the flags and sizes, efem_plan_check_async).  Each step's CUDA
events bracket that device work; the host half of the check (wait, decode
the flags) runs after the end event, every step.  L2 is flushed between
timed steps (a 512 MiB write, untimed).  value = elements / second over all
ranks.
See DESIGN.md "Measurement" for the roofline bytes and the oracle baseline.
"""
from __future__ import annotations

import argparse
import math
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIGS, ELEMENT_NAMES, counts  # noqa: E402

METRIC = "elements assembled/sec (local matrices + CSR)"
UNIT = "elem/s"


def algorithmic_bytes(cfg):
    """north_star: mesh in (coords fp64 + int32 connectivity) + CSR out
    (int32 row_ptr / col_idx, fp64 vals for M and K on one pattern)."""
    N, T, R, nnz = counts(cfg["dim"], cfg["element"], cfg["n"])
    mesh_in = N * cfg["dim"] * 8 + T * (cfg["dim"] + 1) * 4
    csr_out = (R + 1) * 4 + nnz * 4 + 2 * nnz * 8
    return mesh_in + csr_out, T


def traffic_capture(cfg):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one whole
    step, summed over its kernels, and per kernel, from the committed ncu
    capture of tools/profile_step.py (profiles/traffic.json, written by
    tools/traffic_json.py).  A static capture, not measured in this run."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t[cfg["name"]]
    except Exception:
        return None


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a moment before its first sample: wait for it,
            # then keep only samples taken from here on (the timed region)
            t_end = time.time() + 3.0
            while not self.lines and time.time() < t_end:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


_ORACLE_MESH = {}


# FP64 flops of the NE0-3D row kernel per (row, tet) pair of the fast path
# (k_rows_ne3, assemble.cu: tet edge vectors 9, three area normals 27, det 5,
# fourth normal 6, seven Gram dot products 35, 1/|det| and the two scales 5,
# six mass and six curl-curl values 50, the twelve accumulations 12), and the
# measured B200 FP64 FMA peak (tools/fp64_peak.cu, profiles/r2/fp64_peak.txt).
NE3_FLOPS_PER_ROW_TET = 149
FP64_PEAK_TFLOPS = 34.2


def fp64_line(cfg, T, num_ms):
    """The NE0-3D numeric kernel against the FP64 ALU (it is instruction /
    ALU bound, not HBM bound): flops = 149 per (row, tet) x 6 T pairs."""
    if not (cfg["dim"] == 3 and cfg["element"] == 1):
        return None
    fl = NE3_FLOPS_PER_ROW_TET * 6 * T
    tf = fl / (num_ms * 1e-3) / 1e12
    return {"bound": "alu", "kernel": "k_rows_ne3", "flops": fl, "achieved": tf, "peak": FP64_PEAK_TFLOPS,
            "unit": "TFLOP/s", "frac": tf / FP64_PEAK_TFLOPS, "peak_source": "measured, tools/fp64_peak.cu"}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, budget_elems=None, threads=None):
    """The oracle as it stands on a bounded sample of the same workload (the
    first T_s elements of the config's mesh: all their DOFs and rows), mesh
    already in host RAM.  threads = None: the row-range form
    (ora_assemble_blocked, bitwise the serial oracle) on every host core;
    threads = 0: the serial ora_assemble (one core)."""
    import numpy as np

    from oracle import oracle as ora

    key = (cfg["dim"], cfg["n"], cfg["alpha"], cfg["seed"])
    if key not in _ORACLE_MESH:  # (built once per run: the reference arm calls this every step)
        _ORACLE_MESH.clear()
        _ORACLE_MESH[key] = ora.build_mesh(*key)
    coords, elems = _ORACLE_MESH[key]
    if threads is None:
        threads = host_cores()
    if budget_elems is None:
        budget_elems = (1 << 23) if cfg["dim"] == 2 else (1 << 21)
    ts = min(elems.shape[0], budget_elems)
    sub = np.ascontiguousarray(elems[:ts])
    t0 = time.perf_counter()
    ora.assemble(cfg["dim"], cfg["element"], coords, sub, threads=threads)
    dt = time.perf_counter() - t0
    how = (f"{threads} threads, row-range blocks" if threads else "1 thread")
    return {"value": ts / dt, "unit": UNIT, "cores": max(threads, 1), "kind": "oracle",
            "sample": f"first {ts} of {elems.shape[0]} elements of {cfg['name']} ({dt:.1f} s, {how}, "
                      f"g++ -O2 -ffp-contract=off, std::map accumulator)"}


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    # the whole run stays within about a minute of oracle work on all host
    # cores, whatever K is: ~2^26 (2D) / 2^23 (3D) elements in total, split
    # over the K steps
    total = (1 << 26) if cfg["dim"] == 2 else (1 << 23)
    budget = int(min(max(total // max(args.steps, 1), 1 << 12), (1 << 23) if cfg["dim"] == 2 else (1 << 21)))
    for _ in range(args.warmup):
        cpu_baseline(cfg, budget_elems=1 << 12)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(cfg, budget_elems=budget))
    total = time.perf_counter() - t0
    ts = min(budget, counts(cfg["dim"], cfg["element"], cfg["n"])[1])
    value = ts * args.steps / sum(ts / v["value"] for v in vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg["name"], "element": ELEMENT_NAMES[cfg["element"]],
                                            "dim": cfg["dim"], "n": cfg["n"], "jitter": cfg["alpha"],
                                            "seed": cfg["seed"], "sample_elems": ts},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": vals[-1]["cores"], "kind": "oracle",
                             "sample": vals[-1]["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_efem(args, cfg):
    import torch

    from paper_1409_4618_b200 import api

    ws, rank, local = dist_env()
    if ws > 1 or args.dist:
        return run_efem_dist(args, cfg)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    coords, elems = api.build_mesh(cfg["dim"], cfg["n"], cfg["alpha"], cfg["seed"], device=dev)
    asm = api.Assembler(coords, elems, cfg["element"])
    asm.symbolic()
    out = asm.alloc_csr()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        # the whole hot path (enumeration, pattern, values) in one asynchronous
        # call into the CSR sized by the first symbolic call, then the
        # read-back of the flags and sizes (the device half of the check)
        asm.assemble_async(out, api.ALL)
        asm.check_async()

    for _ in range(max(args.warmup, 3)):
        step()
        asm.check()
    torch.cuda.synchronize()

    # timed region: K steps, each bracketed by its own events, L2 flushed in between (untimed)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = api.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.fill_(k & 0xff)
            starts[k].record(stream)
            step()
            ends[k].record(stream)
            asm.check()  # host half of the check (wait + decode), every step, after the device window
        torch.cuda.synchronize()
    launches = api.launch_count() - l0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    T = elems.shape[0]
    value = T * args.steps / (total_ms * 1e-3)

    # dominant kernel (the numeric call: one row-kernel launch), timed alone the same way
    nk = max(args.steps, 5)
    ks = [torch.cuda.Event(enable_timing=True) for _ in range(nk)]
    ke = [torch.cuda.Event(enable_timing=True) for _ in range(nk)]
    for k in range(nk):
        flush.fill_(k & 0xff)
        ks[k].record(stream)
        asm.numeric(out, api.ALL)
        ke[k].record(stream)
    torch.cuda.synchronize()
    asm.check()
    num_ms = sum(s.elapsed_time(e) for s, e in zip(ks, ke)) / nk
    sym_ms = total_ms / args.steps - num_ms

    alg_bytes, _ = algorithmic_bytes(cfg)
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)" if peak else "fallback (B200_PROFILING.md)"
    peak = peak or 6650.0
    step_s = total_ms / args.steps * 1e-3
    step_gbs = alg_bytes / step_s / 1e9
    num_gbs = alg_bytes / (num_ms * 1e-3) / 1e9
    cap = traffic_capture(cfg)

    # end to end through the public API with HOST buffers (copies inside the timed region)
    h_c = coords.cpu().pin_memory()
    h_e = elems.cpu().pin_memory()
    h_out = api.CSR(*(torch.empty_like(t, device="cpu").pin_memory() for t in
                      (out.row_ptr, out.col_idx, out.vals_M, out.vals_K)))
    d_out = asm.alloc_csr()
    asm.assemble_host(h_c, h_e, d_out, h_out)  # warm
    e2e_steps = max(3, min(args.steps, 10))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        asm.assemble_host(h_c, h_e, d_out, h_out)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    h2d = h_c.numel() * 8 + h_e.numel() * 4
    d2h = (h_out.row_ptr.numel() + h_out.col_idx.numel()) * 4 + 2 * h_out.vals_M.numel() * 8

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "element": ELEMENT_NAMES[cfg["element"]], "dim": cfg["dim"],
                   "n": cfg["n"], "jitter": cfg["alpha"], "seed": cfg["seed"], "n_elems": T,
                   "n_rows": asm.n_rows, "nnz": asm.nnz, "l2": "flushed between timed steps (512 MiB write)"},
        "phase_ms": {"symbolic": sym_ms, "numeric": num_ms},
        # the whole step (enumeration + pattern + values, every kernel of one
        # efem_assemble_async) against the HBM roofline of north_star's
        # algorithmic bytes (mesh in + CSR out), DESIGN.md §8
        "roofline": {"bound": "hbm", "achieved": step_gbs, "peak": peak, "unit": "GB/s",
                     "frac": step_gbs / peak,
                     "traffic": (cap or {}).get("step_dram_bytes"),
                     "kernel": "whole step (all kernels of efem_assemble_async, one CUDA graph)",
                     "algorithmic_bytes": alg_bytes, "peak_source": peak_src,
                     "traffic_read": (cap or {}).get("step_dram_read"),
                     "traffic_write": (cap or {}).get("step_dram_write"),
                     "traffic_source": (cap or {}).get("source", "none"),
                     "numeric_kernel": {"kernel": ("k_rows_ne3" if (cfg["dim"] == 3 and cfg["element"] == 1)
                                                   else "k_rows_tri") + " (the numeric call alone)",
                                        "ms": num_ms, "achieved": num_gbs, "frac": num_gbs / peak}},
        "fp64": fp64_line(cfg, T, num_ms),
        "e2e": {"value": T / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_efem_dist(args, cfg):
    """N > 1: one process per GPU over NCCL.  2D (configs 1, 2, 5; config 5 is
    BASELINE's 1/2/4/8-GPU sweep): efem_dist_* -- element slab per rank,
    row-owned CSR slice, the off-rank contributions (ghost triangles' local
    matrices) and column ids exchanged by NCCL inside libefem (dist2d.cu);
    the mesh is fixed, so the scaling is strong.  Each rank builds the full
    mesh and the partition's communication pattern (untimed setup).  A timed
    step is one efem_dist_assemble into the rank's slice; its CUDA events
    bracket the device work, the flag check follows.  Time = max over ranks
    of the summed per-step device time.  3D configs: the owner-computes
    partition (efem_part_*, dist.AsyncStep)."""
    import torch
    import torch.distributed as dist

    from paper_1409_4618_b200 import api
    from paper_1409_4618_b200 import dist as pdist

    ws, rank, local = dist_env()
    if "MASTER_ADDR" not in os.environ:  # (--dist at N = 1 without torchrun)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]), RANK="0",
                              WORLD_SIZE="1")
    n_dev = torch.cuda.device_count()
    torch.cuda.set_device(local % n_dev)
    dev = torch.device("cuda", local % n_dev)
    dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    coords, elems = api.build_mesh(cfg["dim"], cfg["n"], cfg["alpha"], cfg["seed"], device=dev)
    T = elems.shape[0]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    exch = None
    if cfg["dim"] == 2:
        comm = pdist.nccl_comm(rank, ws)
        bounds = pdist.slab_bounds(T, ws)
        part = pdist.DistAssembler(coords, elems, cfg["element"], bounds[rank], bounds[rank + 1], comm)
        part.assemble()  # sizes the slice (untimed)
        exch = part.info()[7]

        def step():
            part.step()

        def check():
            part.check()
        kind = "element slabs over NCCL (efem_dist_*)"
    else:
        ranges = pdist.node_ranges(coords.shape[0], ws)
        part = pdist.PartAssembler(coords, elems, cfg["element"], *ranges[rank])
        out, _, _ = pdist.assemble_rank(part, ranges, None)
        astep = pdist.AsyncStep(part, ranges, out, stream=stream)

        def step():
            astep(check="async")

        def check():
            astep.check()
        kind = "row-owned node ranges, owner computes (efem_part_*)"
    for _ in range(max(args.warmup, 3)):
        step()
        check()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = api.launch_count()
    with ClockSampler(local % n_dev) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.fill_(k & 0xff)
            starts[k].record(stream)
            step()
            ends[k].record(stream)
            check()
        torch.cuda.synchronize()
        dist.barrier()
    launches = api.launch_count() - l0
    mine = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    t = torch.tensor([mine], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = T * args.steps / (total_ms * 1e-3)

    # end to end through the public API with HOST buffers (2D slab path): per
    # step every rank uploads what its slab reads -- the slab's elements and
    # the coordinates of the node-id range they touch -- from pinned host
    # memory, runs the step, and reads its CSR slice back; time = max over
    # ranks (wall clock between barriers, synchronised)
    e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
           "note": "3D: host-buffer e2e measured at N=1 only"}
    if cfg["dim"] == 2:
        lo_e, hi_e = bounds[rank], bounds[rank + 1]
        sl_e = elems[lo_e:hi_e]
        nlo = int(sl_e.min()) if hi_e > lo_e else 0
        nhi = int(sl_e.max()) + 1 if hi_e > lo_e else 0
        h_e = sl_e.cpu().pin_memory()
        h_c = coords[nlo:nhi].cpu().pin_memory()
        sl = part.slice
        h_out = [torch.empty_like(x, device="cpu").pin_memory() for x in (sl.row_ptr, sl.col_idx, sl.vals_M,
                                                                          sl.vals_K)]
        reps = max(3, min(args.steps, 10))
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            elems[lo_e:hi_e].copy_(h_e, non_blocking=True)
            coords[nlo:nhi].copy_(h_c, non_blocking=True)
            part.step()
            w = part.check()
            rows, nnz = w[1], w[3]
            for dst, src, n in zip(h_out, (sl.row_ptr, sl.col_idx, sl.vals_M, sl.vals_K), (rows + 1, nnz, nnz, nnz)):
                dst[:n].copy_(src[:n], non_blocking=True)
            torch.cuda.synchronize()
        mine_s = (time.perf_counter() - t0) / reps
        tb = torch.tensor([mine_s, h_e.numel() * 4 + h_c.numel() * 8,
                           (rows + 1) * 4 + nnz * 4 + 2 * nnz * 8], dtype=torch.float64, device=dev)
        tmax = tb[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(tb, op=dist.ReduceOp.SUM)
        e2e = {"value": T / float(tmax.item()), "unit": UNIT, "h2d_bytes_per_step": int(tb[1].item()),
               "d2h_bytes_per_step": int(tb[2].item())}
    alg_bytes, _ = algorithmic_bytes(cfg)
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs") or 6650.0
    achieved = alg_bytes / (total_ms / args.steps * 1e-3) / 1e9
    xb = torch.tensor([float(exch or 0)], dtype=torch.float64, device=dev)
    dist.all_reduce(xb, op=dist.ReduceOp.MAX)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg["name"], "element": ELEMENT_NAMES[cfg["element"]], "dim": cfg["dim"],
                       "n": cfg["n"], "jitter": cfg["alpha"], "seed": cfg["seed"], "n_elems": T,
                       "elems_per_rank": T / ws, "parallelism": f"{kind} x{ws}",
                       "exchange_bytes_per_rank_step": float(xb.item()) if exch is not None else None,
                       "l2": "flushed between timed steps (512 MiB write)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * ws, "unit": "GB/s",
                         "frac": achieved / (peak * ws), "traffic": None,
                         "kernel": "whole step, all ranks (aggregate bandwidth vs N x peak)",
                         "peak_source": "measured" if peaks.get("hbm_gbs") else "fallback"},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def relaunch_distributed(n):
    """`python bench.py --gpus N` outside torchrun: launch the N ranks here
    (one process per GPU, torch.distributed.run on 127.0.0.1), or fail when
    the node has fewer GPUs than asked for."""
    import torch

    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} but only {have} GPU(s) visible", file=sys.stderr)
        sys.exit(2)
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS),
                    help="BASELINE config.  Default 5 (RT0 2D 4096^2, 33.5 M triangles): the largest config, "
                         "the one BASELINE sweeps over 1/2/4/8 GPUs (strong scaling: the mesh is fixed)")
    ap.add_argument("--impl", default="efem", choices=["efem", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="run the multi-GPU code path (NCCL) even at N = 1 (a one-rank communicator)")
    args = ap.parse_args()
    ws = dist_env()[0]
    if "WORLD_SIZE" in os.environ and ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        sys.exit(2)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args.gpus)
    cfg = dict(CONFIGS[args.config])
    cfg["scaling"] = "strong"  # the mesh is fixed; N ranks split it
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_efem(args, cfg)


if __name__ == "__main__":
    main()
