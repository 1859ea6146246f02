"""The C ABI library loads and exports every function include/hrgen_b200.h
declares; host-only entry points work without a GPU."""

import ctypes
import os
import re

import pytest

import paper_1501_03545_b200 as P
from paper_1501_03545_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hrgen_b200.h")
DEBUG_HEADER = os.path.join(ROOT, "include", "hrgen_b200_debug.h")


def declared_functions(path=HEADER):
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hrg_[a-z_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert set(declared_functions()) == set(_lib.EXPORTED)
    assert set(declared_functions(DEBUG_HEADER)) == set(_lib.EXPORTED_DEBUG)


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for name in declared_functions() + declared_functions(DEBUG_HEADER):
        assert hasattr(L, name), name


def test_no_torch_types_in_abi():
    text = open(HEADER).read()
    assert "torch" not in text.replace("no torch types", "")
    assert "at::" not in text


def test_host_scalar_entry_points():
    L = _lib.load()
    out = ctypes.c_double()
    assert L.hrg_expected_avg_degree(10000, 1.0, 16.0, ctypes.byref(out)) == 0
    assert out.value == pytest.approx(P.expected_avg_degree(10000, 1.0, 16.0), rel=1e-14)
    assert L.hrg_target_radius(10000, 6.0, 1.0, 1e-6, ctypes.byref(out)) == 0
    assert out.value == pytest.approx(P.target_radius(10000, 6.0, 1.0), rel=1e-5)
    m = _lib.Model()
    assert L.hrg_model_init(1000, 1.0, 20.0, ctypes.byref(m)) == 0
    assert m.max_r < 1.0 and m.rp_cap < m.max_r
    assert L.hrg_model_init(0, 1.0, 20.0, ctypes.byref(m)) == _lib.HRG_ERR_PARAMETER_DOMAIN
    assert b"n must" in L.hrg_last_error()
    # radius so large that tanh(R/2) rounds to 1: the reference's quadtree
    # constructor rejects it (quadtree.py:260)
    assert L.hrg_model_init(1000, 1.0, 80.0, ctypes.byref(m)) == _lib.HRG_ERR_PARAMETER_DOMAIN


def test_status_maps_to_reference_exceptions():
    with pytest.raises(P.ParameterDomainError):
        _lib.check(_lib.HRG_ERR_PARAMETER_DOMAIN)
    with pytest.raises(P.OutOfBoundsError):
        _lib.check(_lib.HRG_ERR_OUT_OF_BOUNDS)
    with pytest.raises(P.InfeasibleParametersError):
        _lib.check(_lib.HRG_ERR_INFEASIBLE)
    with pytest.raises(P.NativeLibraryError):
        _lib.check(10)


def test_no_device_fails_loudly():
    """Without a CUDA device, generation raises -- never a CPU fallback."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(P.NativeLibraryError):
        P.generate(P.GeneratorParams(n=100, avg_degree=4.0, gamma=3.0))
