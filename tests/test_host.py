"""Host-side parameter layer against the oracle / reference constants."""

import math

import numpy as np
import pytest

import paper_1105_4204_b200 as tb
from oracle import trigbf_oracle as orc
from paper_1105_4204_b200 import workloads
from paper_1105_4204_b200.spatial import recursive_biquads


@pytest.mark.parametrize("sigma_r,T,deg", [(30.0, 255.0, None), (20.0, 255.0, None), (10.0, 255.0, None),
                                           (25.0, 255.0, None), (15.0, 255.0, None), (80.0, 255.0, None),
                                           (170.0, 255.0, 3), (50.0, 1.0, None), (5.0, 1000.0, 0)])
def test_kernel_matches_oracle(sigma_r, T, deg):
    a = tb.make_trig_kernel(sigma_r, T, degree=deg)
    b = orc.make_trig_kernel(sigma_r, T, degree=deg)
    assert (a.N, a.omega, a.gamma, a.rho) == (b.N, b.omega, b.gamma, b.rho)
    assert np.array_equal(a.coeffs, b.coeffs) and np.array_equal(a.freqs, b.freqs)


def test_config_degrees():
    # N = 30 / 66 / 264 / 43 / 118 at the five configs
    got = [tb.make_trig_kernel(workloads.CONFIGS[i].sigma_r).N for i in (1, 2, 3, 4, 5)]
    assert got == [30, 66, 264, 43, 118]


def test_large_degree_lgamma_branch():
    k = tb.make_trig_kernel(1.0, 255.0, degree=1500)
    assert k.coeffs.sum() == pytest.approx(1.0, abs=1e-9)


def test_parameter_errors():
    with pytest.raises(tb.ParameterError):
        tb.make_trig_kernel(0.0)
    with pytest.raises(tb.ParameterError):
        tb.make_trig_kernel(10.0, degree=-1)
    with pytest.raises(tb.ParameterError):
        tb.SpatialSpec.box(-1)
    with pytest.raises(tb.ParameterError):
        tb.SpatialSpec.gaussian_recursive(0.3)


@pytest.mark.parametrize("sigma", [0.5, 2.0, 3.0, 5.0, 8.0, 16.0, 32.0, 100.0])
def test_biquads_factor_reference_taps(sigma):
    """The two sections multiply out to the reference's direct form."""
    scale, c1, c2, c3, c4 = orc.recursive_coeffs(sigma)
    assert tb.recursive_coeffs(sigma) == (scale, c1, c2, c3, c4)
    b = recursive_biquads(sigma)
    # (1 - a1 z - a2 z^2)(1 - b1 z - b2 z^2) = 1 - c1 z - c2 z^2 - c3 z^3 - c4 z^4
    assert b.a1 + b.b1 == pytest.approx(c1, abs=1e-12)
    assert b.a2 + b.b2 - b.a1 * b.b1 == pytest.approx(c2, abs=1e-12)
    assert -(b.a1 * b.b2 + b.a2 * b.b1) == pytest.approx(c3, abs=1e-12)
    assert -b.a2 * b.b2 == pytest.approx(c4, abs=1e-12)
    assert b.g1 * b.g2 == pytest.approx(scale, rel=1e-12)


def test_decay_lengths():
    # K(eps=1e-7) = 37 / 94 / 187 / 59 / 373
    assert [tb.decay_length(s) for s in (3, 8, 16, 5, 32)] == [37, 94, 187, 59, 373]


def test_term_pairs_fold():
    for n_deg in range(0, 12):
        k = tb.make_trig_kernel(90.0, 255.0, degree=n_deg)
        p = tb.term_pairs(k)
        ref = orc.term_pairs(orc.make_trig_kernel(90.0, 255.0, degree=n_deg))
        assert np.allclose(p.nu, [a for a, _ in ref]) and np.allclose(p.weight, [b for _, b in ref])
        assert p.weight.sum() == pytest.approx(1.0, abs=1e-12)
        assert p.spatial_passes == 2 * (n_deg + 1) - (1 if n_deg % 2 == 0 else 0)
        # arithmetic progression the device relies on: nu_j = nu_0 + j * 2 omega
        assert np.allclose(np.diff(p.nu), p.dnu) if p.count > 1 else True


def test_workloads_deterministic():
    a = workloads.frame(workloads.CONFIGS[1])
    b = workloads.frame(workloads.CONFIGS[1])
    assert np.array_equal(a, b) and a.dtype == np.float32
    assert a.min() >= 0.0 and a.max() <= 255.0
    s = workloads.smooth_image(256, 300, 6, seed=9)
    assert s.shape == (256, 300) and 0.0 <= s.min() and s.max() <= 255.0


def test_fp32_cascade_design_model():
    """CPU model of the device's decomposition along one axis: tile-local
    zero-state forward runs + chained 4-state carries + homogeneous-response
    correction reproduce the full forward/backward recursion (fp64 here)."""
    b = recursive_biquads(8.0)
    rng = np.random.default_rng(0)
    n, E, S = 300, tb.decay_length(8.0), 32
    x = rng.uniform(0, 255, n)

    def step(u, st):
        v = b.g1 * u + b.a1 * st[0] + b.a2 * st[1]
        y = b.g2 * v + b.b1 * st[2] + b.b2 * st[3]
        return y, (v, st[0], y, st[2])

    ext = [orc.mirror(i, n) for i in range(-E, n + E)]
    u = x[ext]
    st = (u[0],) * 4
    F = []
    for v in u:
        y, st = step(v, st)
        F.append(y)
    full_fwd = np.array(F)[E:E + n]
    # tile-local + carries
    st0 = (u[0],) * 4
    for v in u[:E]:
        _, st0 = step(v, st0)
    rec = np.empty(n)
    s = st0
    for t0 in range(0, n, S):
        ln = min(S, n - t0)
        z = (0.0,) * 4
        loc = []
        for i in range(ln):
            y, z = step(x[t0 + i], z)
            loc.append(y)
        # homogeneous response from the carried state
        h = s
        for i in range(ln):
            yh, h = step(0.0, h)
            rec[t0 + i] = loc[i] + yh
        s = tuple(a + c for a, c in zip(h, z))
    assert np.max(np.abs(rec - full_fwd)) < 1e-9


def test_window_taps_match_oracle():
    """FIR/box window taps (spatial.py:77-88, engines.py:96-106)."""
    from oracle import trigbf_oracle as orc
    from paper_1105_4204_b200 import SpatialSpec, gaussian_taps, window_taps

    for s in (0.5, 1.0, 3.0, 8.0, 32.0):
        np.testing.assert_allclose(gaussian_taps(s), orc.gaussian_taps(s), rtol=0, atol=1e-15)
        np.testing.assert_allclose(window_taps(SpatialSpec.gaussian_fir(s)), orc.window_taps("gauss-fir", s))
    for r in (0, 1, 7):
        np.testing.assert_array_equal(window_taps(SpatialSpec.box(r)), orc.window_taps("box", r))
