"""Occupancy guard for the hot kernels (CPU only: reads the built sm_100a cubin's resource usage).

The step kernels are memory / latency bound, so their speed rests on occupancy: 64 registers
(4 x 256-thread CTAs per SM) and no local-memory spills for the headline c5 kernel. A change that
silently raises registers (it happened once: the K-ary kernel went to 90 registers and k8 lost 45 %)
fails here before any GPU time is spent (profiles/r1_design_iterations.md)."""
import re
import shutil
import subprocess

import pytest

from paper_2409_02135_b200._lib import LIB_PATH

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


@pytest.fixture(scope="module")
def usage():
    out = subprocess.run([CUOBJDUMP, "-res-usage", LIB_PATH], capture_output=True, text=True).stdout
    res = {}
    for name, reg, stack in re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+)", out):
        res[name] = (int(reg), int(stack))
    assert res, "no resource usage found"
    return res


def _get(usage, mangled):
    assert mangled in usage, f"{mangled} not in the library"
    return usage[mangled]


def test_headline_c5_kernel_fits_four_ctas(usage):
    """c5 runs k_step<4,1,0,FULL> (two replica blocks of 32, every lane holds a vector): 64 registers and
    at most the 24-byte spill around the division slow-path calls (16 bytes with the round-1 FMA contract,
    24 since the per-row communication coefficient adds a division site per item; same-box c5 step time
    unchanged, 812 vs 812 us, profiles/r2_design_iterations.md); more would cost occupancy-bound bandwidth."""
    reg, stack = _get(usage, "_ZN3qqa6k_stepILi4ELi1ELi0ELb1EEEvNS_10StepParamsE")     # k_step<4,1,0,FULL>
    assert reg <= 64 and stack <= 24


def test_unblocked_64_replica_kernel_spills_at_most_the_division_frame(usage):
    """k_step<8,1,0> (64 replicas unblocked): no spill in round 1; the per-row communication coefficient's
    division site (round 2) leaves a 16-byte frame around the slow-path calls."""
    reg, stack = _get(usage, "_ZN3qqa6k_stepILi8ELi1ELi0ELb0EEEvNS_10StepParamsE")     # k_step<8,1,0>
    assert reg <= 64 and stack <= 16


@pytest.mark.parametrize("lanes", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_step_kernels_keep_64_registers(usage, lanes, mode):
    for full in (0, 1):
        reg, stack = _get(usage, f"_ZN3qqa6k_stepILi{lanes}ELi1ELi{mode}ELb{full}EEEvNS_10StepParamsE")
        assert reg <= 64 and stack <= 64


@pytest.mark.parametrize("kp,cap", [(4, 64), (8, 64), (12, 80), (16, 80)])
def test_kary_kernels_register_caps(usage, kp, cap):
    for mode in (0, 2):
        for fk in (0, 1):   # K == KP specialisation
            reg, stack = _get(usage, f"_ZN3qqa8k_step_KILi{kp}ELi{mode}ELb{fk}EEEvNS_11StepKParamsE")
            assert reg <= cap and stack <= 80


@pytest.mark.parametrize("kp", [8, 12, 16])
def test_colour_quad_kernels_fit_five_ctas_without_spills(usage, kp):
    for mode in (0, 2):
        reg, stack = _get(usage, f"_ZN3qqa9k_step_KqILi{kp}ELi{mode}EEEvNS_11StepKParamsE")
        assert reg <= 48 and stack == 0
