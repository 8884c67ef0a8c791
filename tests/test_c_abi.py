"""The C ABI from plain C (examples/c_abi_step.c): the header is valid C11 and the program
links against libsmcsd.so (CPU); on a GPU it runs smcsd_step + smcsd_kv_reindex and checks
closed forms (p == q => exact uniform weights, identity ancestors; KV blocks follow slot_src)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
EXE = os.path.join(ROOT, "examples", "c_abi_step")


def _build():
    lib_dir = os.path.join(ROOT, "paper_2604_15672_b200")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "c_abi_step.c"),
           "-L", lib_dir, "-lsmcsd", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           f"-Wl,-rpath,{lib_dir}", "-lm", "-o", EXE]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_example_compiles_and_links():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2604_15672_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_c_example_runs():
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c abi ok" in r.stdout
