"""The C ABI from plain C: examples/c_abi_join.c (no Python, no torch) sorts
and joins through include/mpsm_b200.h and checks count / max / checksum
against a direct host computation."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_joins_through_the_abi(tmp_path):
    exe = str(tmp_path / "c_abi_join")
    lib_dir = os.path.join(ROOT, "paper_1207_0145_b200")
    cmd = ["gcc", "-O2", os.path.join(ROOT, "examples", "c_abi_join.c"), "-I" + os.path.join(ROOT, "include"),
           "-I/usr/local/cuda/include", "-L" + lib_dir, "-lmpsm_b200", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath," + lib_dir, "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    for n in ("1", "4097", "1000003"):
        r = subprocess.run([exe, n], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "OK" in r.stdout, (n, r.stdout, r.stderr)
