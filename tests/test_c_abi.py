"""The drop-in boundary from plain C (tests/c/abi_demo.c): the header compiles as C11, a C program
links against libsketch_b200.so and the CUDA runtime alone, and on a GPU it runs the SRTT and float64
dense applies and checks them against its own host arithmetic."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2508_21189_b200", "lib")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _gcc():
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    return gcc


def _build(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libsketch_b200.so")):
        pytest.skip("library not built")
    exe = str(tmp_path / "abi_demo")
    cmd = [_gcc(), "-O2", "-std=c11", "-Wall", "-Werror", os.path.join(ROOT, "tests", "c", "abi_demo.c"),
           "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CUDA, "include"), "-L" + LIBDIR,
           "-lsketch_b200", "-L" + os.path.join(CUDA, "lib64"), "-lcudart", "-lm", "-Wl,-rpath," + LIBDIR,
           "-Wl,-rpath," + os.path.join(CUDA, "lib64"), "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "h.c"
    src.write_text('#include "sketch_b200.h"\nint main(void) { return sk_abi_version() == SK_ABI_VERSION ? 0 : 1; }\n')
    subprocess.run([_gcc(), "-std=c11", "-Wall", "-Werror", "-fsyntax-only", "-I" + os.path.join(ROOT, "include"),
                    str(src)], check=True, capture_output=True, text=True)


def test_c_caller_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_caller_runs(tmp_path, cuda):
    exe = _build(tmp_path)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert res.stdout.strip().endswith("ok"), res.stdout
