import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes, torch
from paper_1409_4618_b200 import api, _lib
from workloads import CONFIGS
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
C = CONFIGS[c]
coords, elems = api.build_mesh(2, C["n"], C["alpha"], C["seed"])
asm = api.Assembler(coords, elems, C["element"])
asm.symbolic(); out = asm.alloc_csr()
ref = asm.assemble()
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    asm.assemble_async(out); asm.check(); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    h = (ctypes.c_int * 64).from_address(0)  if False else None
    hdr = asm.ws[:256].view(torch.int32).cpu().tolist()
    print(f"step {dt*1e3:.2f} ms")
for a, b, nm in zip((out.row_ptr, out.col_idx, out.vals_M, out.vals_K), (ref.row_ptr, ref.col_idx, ref.vals_M, ref.vals_K), "rp ci vm vk".split()):
    d = (a != b).nonzero()
    print(nm, int(d.numel()), d[:5].flatten().tolist(), a[d[:3].flatten()].tolist() if d.numel() else '', b[d[:3].flatten()].tolist() if d.numel() else '')
print("equal:", all(torch.equal(a, b) for a, b in zip((out.row_ptr, out.col_idx, out.vals_M, out.vals_K), (ref.row_ptr, ref.col_idx, ref.vals_M, ref.vals_K))))
