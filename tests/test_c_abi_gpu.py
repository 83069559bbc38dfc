"""The boundary used from plain C (examples/c_abi_example.c): compiled with
gcc against include/efem.h and the in-tree libefem.so, run on the GPU; it
checks the closed-form sizes and the symmetry of M and K itself."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_assembles(tmp_path):
    cc = shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    lib = os.path.join(ROOT, "paper_1409_4618_b200")
    exe = str(tmp_path / "efem_c")
    subprocess.run([cc, "-std=c11", "-O2", os.path.join(ROOT, "examples", "c_abi_example.c"),
                    "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(cuda, "include"), "-L" + lib, "-lefem",
                    "-L" + os.path.join(cuda, "lib64"), "-lcudart", "-lm", "-Wl,-rpath," + lib, "-o", exe],
                   check=True, capture_output=True, text=True)
    for n in ("3", "64"):
        r = subprocess.run([exe, n], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.strip().endswith("OK"), r.stdout
