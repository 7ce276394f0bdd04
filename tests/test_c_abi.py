"""A plain C caller of the boundary (tests/c_abi/abi_check.c): it includes
include/dvm.h, links libdvm.so and calls dvm_plan -> dvm_collide ->
dvm_plan_destroy (the calls BASELINE.json's north_star names) plus
dvm_collide_batched and the error codes, on stored inputs, against stored
oracle outputs (tests/golden/abi_*.bin, written by tools/make_abi_golden.py
from oracle/ only).  CPU: it compiles and links as C99.  GPU: it passes."""
import os
import subprocess

import pytest

from paper_1201_3986_b200 import build as dvm_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_abi", "abi_check.c")
LIBDIR = os.path.join(ROOT, "paper_1201_3986_b200")
CUDA = "/usr/local/cuda"
GOLD = os.path.join(ROOT, "tests", "golden")


def _compile(tmp_path) -> str:
    dvm_build.build()
    exe = str(tmp_path / "abi_check")
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-O1", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), SRC, "-o", exe, "-L", LIBDIR, "-ldvm",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm",
           f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_caller_compiles_and_links(tmp_path):
    exe = _compile(tmp_path)
    assert os.access(exe, os.X_OK)
    for name in ("c1", "c4"):
        for part in ("f", "q"):
            assert os.path.getsize(os.path.join(GOLD, f"abi_{name}_{part}.bin")) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name,d,N,Nbar", [("c1", 2, 16, 4), ("c4", 3, 32, 4)])
def test_c_caller_matches_stored_oracle(tmp_path, name, d, N, Nbar):
    exe = _compile(tmp_path)
    res = subprocess.run([exe, str(d), str(N), str(Nbar), os.path.join(GOLD, f"abi_{name}_f.bin"),
                          os.path.join(GOLD, f"abi_{name}_q.bin")], capture_output=True, text=True, timeout=300)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "abi_check ok" in res.stdout
