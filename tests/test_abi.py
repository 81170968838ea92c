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


def _build_c_demo(tmp_path):
    """Compile examples/tbf_c_demo.c against the in-tree library (plain C,
    cudart, no Python/torch on the call path)."""
    import shutil
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    gcc = shutil.which("gcc")
    if gcc is None or not os.path.isdir(os.path.join(cuda, "include")):
        pytest.skip("gcc / CUDA headers not available")
    lib = os.path.join(root, "paper_1105_4204_b200", "_lib")
    exe = str(tmp_path / "tbf_c_demo")
    cmd = [gcc, "-O2", "-Wall", "-Werror", os.path.join(root, "examples", "tbf_c_demo.c"),
           "-I", os.path.join(root, "include"), "-I", os.path.join(cuda, "include"),
           "-L", lib, "-ltrigbf_b200", "-L", os.path.join(cuda, "lib64"), "-lcudart", "-lm",
           f"-Wl,-rpath,{lib}", "-o", exe]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


def test_c_demo_compiles(tmp_path):
    """The C ABI is usable from plain C: the example compiles and links."""
    if not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "paper_1105_4204_b200", "_lib", "libtrigbf_b200.so")):
        pytest.skip("library not built")
    _build_c_demo(tmp_path)


@pytest.mark.gpu
def test_c_demo_matches_python(tmp_path):
    """The plain-C host-entry call gives the Python drop-in's result."""
    import subprocess

    import numpy as np

    import paper_1105_4204_b200 as tb

    exe = _build_c_demo(tmp_path)
    H, W, r, sr, N = 70, 90, 3, 60.0, 4
    out = tmp_path / "out.f32"
    res = subprocess.run([exe, str(H), str(W), str(r), str(sr), str(N), str(out)],
                         capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stderr
    assert "out_of_range=0" in res.stdout
    got = np.fromfile(out, dtype=np.float32).reshape(H, W)
    y, x = np.mgrid[0:H, 0:W]
    img = (np.where(x < W // 2, 40.0, 200.0) + 0.25 * ((x * 7 + y * 13) % 40)).astype(np.float32)
    ref = tb.bilateral_trig(img, tb.SpatialSpec.box(r), tb.make_trig_kernel(sr, 255.0, degree=N))
    assert np.max(np.abs(got - ref)) < 1e-3
