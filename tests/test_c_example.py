"""The C ABI from plain C (examples/fhwt_example.c): gcc against include/fhwt.h, linked to the
in-tree libfhwt.so and cudart, run on the GPU.  The program checks perfect reconstruction, the
LL_L closed form, bitwise agreement of the host-buffer round trip with the
device-buffer plan path, and validation before launch."""
import os
import shutil
import subprocess

import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def build_example(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    from paper_1002_2184_b200 import lib
    lib()   # builds libfhwt.so in-tree if the sources are newer
    exe = tmp_path / "fhwt_example"
    libdir = os.path.join(ROOT, "paper_1002_2184_b200")
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
                    os.path.join(ROOT, "examples", "fhwt_example.c"), "-L", libdir, "-lfhwt", "-L", f"{CUDA}/lib64",
                    "-lcudart", "-lm", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    """CPU: the header is valid C and every symbol the example uses resolves against libfhwt.so."""
    assert build_example(tmp_path).exists()


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_c_example_program(tmp_path):
    exe = build_example(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert res.stdout.strip().endswith("OK")
