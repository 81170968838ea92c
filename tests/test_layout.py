"""Launch-layout planning (host logic in the C-ABI library, no GPU needed):
the device entry's planned unequal chunks for few-wave launches, equal chunks
for the host entry, batched runs and many-wave configs."""

import pytest

from conftest import ROOT  # noqa: F401  (puts the repo on sys.path)


@pytest.fixture(scope="module")
def tb():
    import os

    from paper_1105_4204_b200.build import LIB, build

    if not os.path.exists(LIB):
        build()
    import paper_1105_4204_b200 as tb

    return tb


def _cfg(tb, cid):
    from paper_1105_4204_b200 import workloads

    c = workloads.CONFIGS[cid]
    return (c.frames, c.height, c.width), tb.SpatialSpec.gaussian_recursive(c.sigma_s), tb.make_trig_kernel(c.sigma_r, c.T)


def test_config2_planned_device_layout(tb):
    """Config 2 (544 pass-1 blocks per y-chunk level, a few waves): unequal
    y-chunks, largest first, whole 32-row segments, each longer than the
    warm-up, and two unequal x-chunks (13 + 51 tiles) instead of 4 x 16, as
    measured fastest on B200."""
    shape, spec, k = _cfg(tb, 2)
    d = tb.layout_info(shape, spec, k)
    assert d["batches"] == 1 and d["y_chunks"] in (2, 3) and d["y_planned"] == 1
    ends = [d["y_end0"], d["y_end1"], 2048][: d["y_chunks"]]
    sizes = [b - a for a, b in zip([0] + ends[:-1], ends)]
    assert ends[-1] == 2048 and all(e % 32 == 0 for e in ends[:-1])
    assert sizes == sorted(sizes, reverse=True) and d["y_rows_max"] == sizes[0]
    assert min(sizes) >= 96  # the decay length K = 94 at sigma_s = 8
    assert d["x_chunks"] == 2 and d["x_planned"] == 1 and (d["x_end0"], d["x_end1"]) == (13, 64)
    assert d["x_order"] & 3 == 1  # the 51-tile chunk (index 1) is dispatched first


def test_host_entry_keeps_equal_chunks(tb):
    """The host entry's strip/band launches keep the equal chunks (planned
    ones measured +3% / +14% there)."""
    shape, spec, k = _cfg(tb, 2)
    d = tb.layout_info(shape, spec, k, host_entry=True)
    assert d["y_planned"] == 0 and d["x_planned"] == 0
    assert d["x_chunks"] == 4 and d["x_tiles_equal"] == 16


@pytest.mark.parametrize("cid", [1, 3, 4, 5])
def test_no_y_planning_where_it_does_not_pay(tb, cid):
    """Config 1 (short columns, latency-bound), configs 3/4 (many waves) and
    config 5 (term batches: the workspace must stay affine in the batch size)
    keep equal y-chunks."""
    shape, spec, k = _cfg(tb, cid)
    d = tb.layout_info(shape, spec, k, batch_terms=16 if cid == 5 else 0)
    assert d["y_planned"] == 0
    if cid == 5:
        assert d["batches"] > 1 and d["x_planned"] == 0


def test_option_disables_planning(tb):
    from paper_1105_4204_b200 import _native

    lib = _native.load()
    shape, spec, k = _cfg(tb, 2)
    lib.tbf_set_option(_native.TBF_OPT_LPT_SPLIT, 0)
    try:
        d = tb.layout_info(shape, spec, k)
    finally:
        lib.tbf_set_option(_native.TBF_OPT_LPT_SPLIT, _native.TBF_LPT_DEFAULT)
    assert d["y_planned"] == 0 and d["x_planned"] == 0 and d["x_chunks"] == 4


def test_workspace_covers_both_layouts(tb):
    """A plan's workspace (sized once) must fit the planned device layout and
    the equal host layout whatever the option is when it runs: the size does
    not depend on the option."""
    import ctypes

    from paper_1105_4204_b200 import _native
    from paper_1105_4204_b200.engines import _TermsHolder, spatial_struct

    lib = _native.load()
    shape, spec, k = _cfg(tb, 2)
    sp, terms = spatial_struct(spec), _TermsHolder(k)
    n = terms.struct.n_terms
    on = lib.tbf_workspace_bytes(*shape, ctypes.byref(sp), 0, n, 0)
    lib.tbf_set_option(_native.TBF_OPT_LPT_SPLIT, 0)
    try:
        off = lib.tbf_workspace_bytes(*shape, ctypes.byref(sp), 0, n, 0)
    finally:
        lib.tbf_set_option(_native.TBF_OPT_LPT_SPLIT, _native.TBF_LPT_DEFAULT)
    assert on == off > 0


def test_layout_info_rejects_bad_arguments(tb):
    shape, spec, k = _cfg(tb, 2)
    with pytest.raises(tb.ParameterError):
        tb.layout_info(shape, spec, k, term_range=(3, 3))


@pytest.mark.parametrize("shape,sigma_s,sigma_r,world", [
    ((1, 700, 300), 9.0, 12.0, 2),
    ((1, 700, 300), 9.0, 12.0, 3),
    ((1, 2048, 2048), 8.0, 20.0, 4),
    ((1, 16384, 16384), 32.0, 15.0, 8),
    ((1, 4096, 4096), 16.0, 10.0, 8),
    ((2, 300, 260), 6.0, 15.0, 2),
])
def test_row_band_layout_fits_whole_image_workspace(tb, shape, sigma_s, sigma_r, world):
    """The term-sharded path runs the leftover terms over a row band with a
    plan (and workspace) sized by tbf_workspace_bytes for the whole image:
    every rank's band layout must fit it (a band may pick other y-chunks).
    The workspace check runs before any device work, so a fake device pointer
    shows which error the call would return: anything but TBF_ERR_WORKSPACE."""
    import ctypes

    from paper_1105_4204_b200 import _native, engines
    from paper_1105_4204_b200.distributed import term_shard
    from paper_1105_4204_b200.kernels import term_pairs

    lib = _native.load()
    k = tb.make_trig_kernel(sigma_r, 255.0)
    spec = tb.SpatialSpec.gaussian_recursive(sigma_s)
    sp = engines.spatial_struct(spec)
    terms = engines._TermsHolder(k)
    B, H, W = shape
    n = term_pairs(k).count
    fake = ctypes.c_void_p(1 << 40)
    for rank in range(world):
        sh = term_shard(n, world, rank, H, balance="rows")
        if sh.l1 <= sh.l0:
            continue
        ws = lib.tbf_workspace_bytes(B, H, W, ctypes.byref(sp), sh.l0, sh.l1, 0)
        rc = lib.tbf_trig_partial_rows(fake, fake, fake, B, H, W, ctypes.byref(sp), ctypes.byref(terms.struct),
                                       sh.l0, sh.l1, sh.r0, sh.r1, 0, 0, fake, ws, None)
        assert rc != 5, (rank, sh, lib.tbf_last_error())  # TBF_ERR_WORKSPACE


def test_pass2_chunks_fill_the_last_wave(tb):
    """Config 5 in 20-term batches: 1536 pass-2 group blocks per x-chunk are
    3.46 waves of 444 slots; two equal chunks (6.92 waves, 12 warm-up tiles
    each) cost less under the waves-rounded-up model and measured 5% faster
    (profiles/sweep_p2_chunks_r02.log).  Configs 3 and 4 (4.9 and 15.6 waves)
    keep one chunk."""
    shape, spec, k = _cfg(tb, 5)
    d = tb.layout_info(shape, spec, k, batch_terms=20)
    assert d["batches"] == 3 and d["x_chunks"] == 2 and d["x_planned"] == 0 and d["x_tiles_equal"] == 256
    for cid in (3, 4):
        shape, spec, k = _cfg(tb, cid)
        assert tb.layout_info(shape, spec, k)["x_chunks"] == 1
