"""PNM I/O and the command line (reference pnm.py:57-109, image.py:87-91,
cli.py:114-175), pinned to fixtures written by the real reference
(tests/golden/make_golden.py --pnm).  CPU only, except the GPU filter run."""

import os

import numpy as np
import pytest

import paper_1105_4204_b200 as tb
from conftest import GOLDEN
from paper_1105_4204_b200 import cli
from paper_1105_4204_b200.pnm import quantize

from pnm_bad_cases import PNM_BAD


@pytest.fixture(scope="module")
def cases():
    return np.load(os.path.join(GOLDEN, "pnm_cases.npz"))


def test_read_write_match_reference(cases):
    for i in range(3):
        data = cases[f"good{i}_in"].tobytes()
        img = tb.read_pnm(data)
        np.testing.assert_array_equal(img.samples, cases[f"good{i}_planes"])
        assert tb.write_pnm(img) == cases[f"good{i}_out"].tobytes()
        # canonical output reads back to the same planes
        np.testing.assert_array_equal(tb.read_pnm(tb.write_pnm(img)).samples, img.samples)


def test_quantisation_matches_reference(cases):
    img = tb.Image(10, 1, 1, cases["quant_in"])
    assert tb.write_pnm(img) == cases["quant_out"].tobytes()
    assert quantize([0.5, 1.5, -0.5]).tolist() == [1, 2, 0]


def test_parse_errors_match_reference_offsets(cases):
    for data, off in zip(PNM_BAD, cases["bad_offsets"]):
        with pytest.raises(tb.PnmParseError) as ei:
            tb.read_pnm(data)
        assert ei.value.offset == off, data
        assert isinstance(ei.value, tb.TrigbfError)


def test_write_rejects_two_channels():
    with pytest.raises(tb.DimensionError):
        tb.write_pnm(tb.Image(2, 2, 2, np.zeros((2, 2, 2))))


def test_cli_exit_codes(tmp_path, capsys):
    assert cli.main(["filter", str(tmp_path / "missing.pgm"), "--output", str(tmp_path / "o.pgm")]) == 2
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P5\n2 2\n255\n\x01")
    assert cli.main(["filter", str(bad), "--output", str(tmp_path / "o.pgm")]) == 2
    assert cli.main(["filter", str(bad), "--output", str(tmp_path / "o.pgm"), "--sigma-r", "0"]) == 1
    assert cli.main(["filter", str(bad), "--output", str(tmp_path / "o.pgm"), "--engine", "poly"]) == 1
    assert cli.main(["nope"]) == 1
    assert not (tmp_path / "o.pgm").exists()  # no partial output on failure
    capsys.readouterr()


@pytest.mark.gpu
def test_cli_filter_on_gpu(tmp_path, capsys):
    """filter through the CLI equals the library call on the same 8-bit image,
    quantised like the reference; compare reports the trig error vs brute force."""
    rng = np.random.default_rng(5)
    pix = rng.integers(0, 256, (40, 56), dtype=np.uint8)
    src = tmp_path / "in.pgm"
    src.write_bytes(b"P5\n56 40\n255\n" + pix.tobytes())
    out = tmp_path / "out.pgm"
    assert cli.main(["filter", str(src), "--output", str(out), "--sigma-s", "3", "--sigma-r", "30"]) == 0
    img = tb.read_pnm(src.read_bytes())
    lib = tb.bilateral_trig(img, tb.SpatialSpec.gaussian_recursive(3.0), tb.make_trig_kernel(30.0))
    assert out.read_bytes() == tb.write_pnm(lib)
    assert "engine=trig" in capsys.readouterr().out
    assert cli.main(["compare", str(src), "--sigma-s", "3", "--sigma-r", "30"]) == 0
    assert "vs direct" in capsys.readouterr().out
    rgb = tmp_path / "in.ppm"
    rgb.write_bytes(b"P6\n8 6\n255\n" + rng.integers(0, 256, 144, dtype=np.uint8).tobytes())
    assert cli.main(["filter", str(rgb), "--output", str(tmp_path / "o.ppm"), "--engine", "direct",
                     "--spatial", "box", "--sigma-s", "1"]) == 0
    assert tb.read_pnm((tmp_path / "o.ppm").read_bytes()).channels == 3
    csv = tmp_path / "grid.csv"
    assert cli.main(["bench", str(src), "--reps", "1", "--csv", str(csv)]) == 0
    rows = csv.read_text().splitlines()
    assert rows[0] == "sigma_s,sigma_r,N,engine,median_ms" and len(rows) == 21
