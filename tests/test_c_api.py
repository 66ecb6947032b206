"""The C ABI from plain C: examples/c_api_demo.c compiles as C11 against include/*.h and
libmont.so (CPU: the headers are valid C, the symbols link), and on a B200 it runs and checks
every result against a naive 64-bit '%' loop of its own."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIBDIR = ROOT / "paper_1609_00999_b200"
CUDA = Path("/usr/local/cuda")


def build_demo(tmp_path):
    exe = tmp_path / "c_api_demo"
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", str(ROOT / "examples" / "c_api_demo.c"),
           f"-I{ROOT / 'include'}", f"-I{CUDA / 'include'}", f"-L{LIBDIR}", "-lmont", f"-L{CUDA / 'lib64'}",
           "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_demo_compiles_and_links(tmp_path):
    if not (LIBDIR / "libmont.so").exists():
        pytest.fail("libmont.so missing: run __graft_entry__.build()")
    assert build_demo(tmp_path).exists()


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    exe = build_demo(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "c_api_demo ok" in r.stdout
