import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_PATH = os.path.join(ROOT, "oracle", "_ref")
TOL = 1e-3 * 255.0  # north_star: max abs error <= 1e-3*T, fp32 vs the reference's fp64


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def small_cases():
    data = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    names = sorted({k.split("__")[0] for k in data.files if not k.startswith("plugin_")})
    cases = {}
    for n in names:
        h, w, kind, param, sr, deg = data[f"{n}__meta"]
        cases[n] = dict(
            f=data[f"{n}__f"], out=data[f"{n}__out"], h=int(h), w=int(w),
            kind="box" if kind == 0 else "gauss-recursive",
            param=int(param) if kind == 0 else float(param), sigma_r=float(sr),
            degree=None if deg < 0 else int(deg),
        )
    return cases


@pytest.fixture(scope="session")
def plugin_vectors():
    return np.load(os.path.join(GOLDEN, "small_cases.npz"))


@pytest.fixture(scope="session")
def reference_pkg():
    """The real reference (oracle/_ref), when built here; skip otherwise."""
    if not os.path.isdir(os.path.join(REF_PATH, "trigbf")):
        pytest.skip("oracle/_ref not built (run oracle/build_ref.sh)")
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import trigbf

    return trigbf


@pytest.fixture
def equal_chunks():
    """Equal pass-1/pass-2 chunks for the device entry too (TBF_OPT_LPT_SPLIT
    = 0), as the host entry always uses: the two entries then compute the
    same bits.  The planned unequal chunks of the device entry change results
    only at the warm-up truncation level (test_planned_chunks_match_equal)."""
    from paper_1105_4204_b200 import _native

    lib = _native.load()
    lib.tbf_set_option(_native.TBF_OPT_LPT_SPLIT, 0)
    try:
        yield
    finally:
        lib.tbf_set_option(_native.TBF_OPT_LPT_SPLIT, _native.TBF_LPT_DEFAULT)
