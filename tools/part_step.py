"""Time one rank's partitioned step at world size 1 on one GPU, beside the
single-plan async step, to see the partition path's fixed overhead (host
round trips, collectives, globalisation):
    python tools/part_step.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from paper_1409_4618_b200 import dist as pdist  # noqa: E402
from workloads import CONFIGS  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group(os.environ.get("BK", "nccl"), rank=0, world_size=1, device_id=torch.device("cuda", 0))
C = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
coords, elems = api.build_mesh(C["dim"], C["n"], C["alpha"], C["seed"], device="cuda:0")
ranges = pdist.node_ranges(coords.shape[0], 1)
part = pdist.PartAssembler(coords, elems, C["element"], *ranges[0])
out, _, _ = pdist.assemble_rank(part, ranges, None)
step = pdist.AsyncStep(part, ranges, out)
asm = api.Assembler(coords, elems, C["element"])
o2 = asm.assemble()
K = 50
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(name, fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.record()
    for _ in range(K):
        fn()
    e.record()
    torch.cuda.synchronize()
    print(f"{name:44s} {s.elapsed_time(e) / K:.4f} ms/step (wall {(time.perf_counter() - t0) / K * 1e3:.4f})")


def single():
    asm.assemble_async(o2, api.ALL)
    asm.check()


for _ in range(2):
    timed("sync partition step (P=1)", lambda: pdist.assemble_rank(part, ranges, out))
    timed("assemble_rank_async (P=1)", lambda: pdist.assemble_rank_async(part, ranges, out))
    timed("AsyncStep (P=1)", lambda: step())
    timed("AsyncStep, unchecked (P=1)", lambda: step(check=False))
    timed("single-plan efem_assemble_async", single)
dist.destroy_process_group()
