"""The sigmoid's division without the range check (csrc/qqa_sigdiv.cuh) equals IEEE round-to-nearest
division (__fdiv_rn, the contract's fl(a / b)) on every operand the sigmoid can produce:
all fp32 E in [0, 1], den = fl(1 + E), numerator 1 or E. Exhaustive, on the GPU."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_sigmoid_division_is_correctly_rounded_for_every_operand(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = str(tmp_path / "sigdiv")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                    "-I", os.path.join(ROOT, "paper_2409_02135_b200", "csrc"),
                    os.path.join(ROOT, "tools", "probes", "sigdiv.cu"), "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and " 0 mismatches" in r.stdout, r.stdout + r.stderr
