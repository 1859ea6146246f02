"""The product's sin/cos (csrc/hrg_libm_trig.cuh, compiled here for the host
from the same source the device uses) against the host's libm -- i.e.
numpy's float64 sin/cos, hrgen's arithmetic for p_x = r cos(phi)
(quadtree.py:474-475, 516-517) -- bit for bit.  The device side of the same
check is tests/test_gpu_parity.py::test_device_sincos_matches_numpy."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "libm_trig_check.cpp")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("trig") / "libm_trig_check")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-o", exe, SRC,
                           "-lm"])
    return exe


def test_host_build_matches_libm(checker):
    """4e6 sampler-style angles, 4e6 arbitrary doubles in [0, 2pi), every
    branch boundary and every table node +-64 ulps."""
    out = subprocess.run([checker, "2000000", "17"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert out.stdout.strip().startswith("mismatches 0")


def test_libm_is_numpy():
    """numpy's float64 sin/cos are the host libm's (so the libm check above
    is a check against hrgen's own arithmetic)."""
    libm = ctypes.CDLL("libm.so.6")
    libm.sin.restype = libm.cos.restype = ctypes.c_double
    libm.sin.argtypes = libm.cos.argtypes = [ctypes.c_double]
    x = np.random.default_rng(3).random(20000) * 2 * np.pi
    assert all(np.sin(v) == libm.sin(v) and np.cos(v) == libm.cos(v) for v in x.tolist())


def test_table_is_the_generated_one(tmp_path):
    """hrg_libm_table.inc is what csrc/gen/gen_libm_table.py derives
    (mpmath, pinned to the installed libm) -- regenerated and diffed."""
    pytest.importorskip("mpmath")
    root = os.path.dirname(HERE)
    inc = os.path.join(root, "paper_1501_03545_b200", "csrc", "hrg_libm_table.inc")
    out = str(tmp_path / "table.inc")
    subprocess.check_call(["python", os.path.join(root, "paper_1501_03545_b200", "csrc", "gen",
                                                  "gen_libm_table.py"),
                           "/lib/x86_64-linux-gnu/libm.so.6", out], stdout=subprocess.DEVNULL)
    assert open(inc).read() == open(out).read()
