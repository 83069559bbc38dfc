"""Time one rank's partitioned step (dist.assemble_rank) at world size 1 on
one GPU, beside the single-plan async step, to see the partition path's
fixed overhead (host round trips, collectives)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from paper_1409_4618_b200 import dist as pdist  # noqa: E402
from workloads import CONFIGS  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group(os.environ.get("BK", "nccl"), rank=0, world_size=1)
C = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
coords, elems = api.build_mesh(C["dim"], C["n"], C["alpha"], C["seed"], device="cuda:0")
ranges = pdist.node_ranges(coords.shape[0], 1)
part = pdist.PartAssembler(coords, elems, C["element"], *ranges[0])
out = None
for _ in range(5):
    out, fr, fn = pdist.assemble_rank(part, ranges, out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 50
s.record()
for _ in range(K):
    out, fr, fn = pdist.assemble_rank(part, ranges, out)
e.record()
torch.cuda.synchronize()
print(f"partition step (P=1): {s.elapsed_time(e) / K:.4f} ms")
for _ in range(5):
    pdist.assemble_rank_async(part, ranges, out)
torch.cuda.synchronize()
s.record()
for _ in range(K):
    pdist.assemble_rank_async(part, ranges, out)
e.record()
torch.cuda.synchronize()
print(f"async partition step (P=1): {s.elapsed_time(e) / K:.4f} ms")
asm = api.Assembler(coords, elems, C["element"])
o2 = asm.assemble()
for _ in range(5):
    asm.assemble_async(o2, api.ALL)
    asm.check()
s.record()
for _ in range(K):
    asm.assemble_async(o2, api.ALL)
    asm.check()
e.record()
torch.cuda.synchronize()
print(f"async step: {s.elapsed_time(e) / K:.4f} ms")
dist.destroy_process_group()
