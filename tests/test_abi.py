"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def header_symbols():
    with open(os.path.join(ROOT, "include", "trigbf_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"TBF_API\s+[\w\s\*]*?\b(tbf_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1105_4204_b200 import _native
    from paper_1105_4204_b200.build import LIB, build

    if not os.path.exists(LIB):
        build()
    return _native.load()


def test_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(lib, s), s
    from paper_1105_4204_b200 import _native

    assert sorted(_native.EXPORTS) == syms


def test_abi_version(lib):
    from paper_1105_4204_b200 import _native

    assert lib.tbf_abi_version() == _native.ABI_VERSION


def test_workspace_sizing_host_only(lib):
    from paper_1105_4204_b200 import SpatialSpec, make_trig_kernel, term_pairs
    from paper_1105_4204_b200.engines import spatial_struct

    sp = spatial_struct(SpatialSpec.gaussian_recursive(8.0))
    n = term_pairs(make_trig_kernel(20.0)).count
    full = lib.tbf_workspace_bytes(1, 2048, 2048, ctypes.byref(sp), 0, n, n)        # one batch
    quarter = lib.tbf_workspace_bytes(1, 2048, 2048, ctypes.byref(sp), 0, n, n // 4)  # 2 slots
    auto = lib.tbf_workspace_bytes(1, 2048, 2048, ctypes.byref(sp), 0, n, 0)
    assert full > quarter > 0 and auto > 0
    # one batch keeps the round-trip planes of every term resident
    assert full >= n * 16 * 2048 * 2048
    bad = lib.tbf_workspace_bytes(0, 2048, 2048, ctypes.byref(sp), 0, n, 0)
    assert bad == 0
    assert b"bad shape" in lib.tbf_last_error()


def test_kernel_names(lib):
    names = [lib.tbf_kernel_name(k).decode() for k in range(lib.tbf_profile_kinds())]
    assert "pass1" in names and "pass2" in names


def test_product_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    import paper_1105_4204_b200 as tb

    with pytest.raises(tb.NativeUnavailableError):
        tb.bilateral_trig(np.zeros((4, 4), np.float32), tb.SpatialSpec.box(1), tb.make_trig_kernel(80.0))
