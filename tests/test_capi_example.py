"""The C ABI from plain C (examples/capi_example.c): it compiles and links
against libariann_fss.so with gcc alone (no torch, no Python types in any
signature -- CPU test), and on a GPU it deals and evaluates 2^20 DCF keys and
checks every reconstruction."""

import os
import shutil
import subprocess

import pytest

from conftest import ROOT

LIBDIR = os.path.join(ROOT, "paper_2006_04593_b200")
CUDA = "/usr/local/cuda"


def _build(out):
    if shutil.which("gcc") is None or not os.path.exists(os.path.join(LIBDIR, "libariann_fss.so")):
        pytest.skip("needs gcc and the built library")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", os.path.join(ROOT, "examples", "capi_example.c"),
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"), "-L", LIBDIR,
           "-lariann_fss", "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_capi_example_builds(tmp_path):
    _build(str(tmp_path / "capi_example"))


@pytest.mark.gpu
def test_capi_example_runs(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    exe = str(tmp_path / "capi_example")
    _build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout
