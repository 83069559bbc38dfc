"""Premise check for overlapping the 2D fan pass with the row kernel: two
config-5 plans, A's whole step (count, fill, fan pass, rows) on one stream
and B's row kernel on another, timed together and apart."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from workloads import CONFIGS  # noqa: E402

C = CONFIGS[5]
ca, ea = api.build_mesh(2, C["n"], C["alpha"], C["seed"])
cb, eb = api.build_mesh(2, C["n"], C["alpha"], C["seed"] + 1)
A = api.Assembler(ca, ea, C["element"])
B = api.Assembler(cb, eb, C["element"])
A.symbolic()
B.symbolic()
oa, ob = A.alloc_csr(), B.alloc_csr()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=10):
    ts = []
    for r in range(reps):
        flush.fill_(r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def stepA():
    with torch.cuda.stream(s1):
        A.assemble_async(oa)


def numB():
    with torch.cuda.stream(s2):
        B.numeric(ob)


def both():
    stepA()
    numB()


for _ in range(3):
    both()
ta, tb, tab = t(stepA), t(numB), t(both)
print(f"A step {ta:.3f} ms, B rows {tb:.3f} ms, sum {ta + tb:.3f}, concurrent {tab:.3f} ms")
