"""Build libefem.so with extra nvcc flags into variants/<name>/libefem.so
(for A/B timing with tools/ab.sh / ab_bench.sh):
    python tools/build_variant.py NAME [-DFOO=1 ...]"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1409_4618_b200 import build as b  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "vbuild", name)
os.makedirs(out, exist_ok=True)
objs = []


def one(src):
    o = os.path.join(out, src.replace(".cu", ".o"))
    subprocess.check_call([b.NVCC] + b.FLAGS + extra + ["-c", os.path.join(b.CSRC, src), "-o", o])
    return o


with ThreadPoolExecutor(len(b.SOURCES)) as ex:
    objs = list(ex.map(one, b.SOURCES))
subprocess.check_call([b.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                       os.path.join(out, "libefem.so")] + objs + b.LINK)
print(os.path.join(out, "libefem.so"))
