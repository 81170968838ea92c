"""Spatial smoother specification and the recursive-Gaussian coefficients.

Same ``SpatialSpec`` / ``SpatialKind`` / ``recursive_coeffs`` surface as the
reference (spatial.py:28-144).  What the B200 path adds is the reduction of
the reference's fourth-order direct-form recursion to the form the device
runs:

* ``recursive_biquads`` -- the same filter as two cascaded second-order
  sections, one per prototype pole pair (spatial.py:95-114).  The product of
  the two section polynomials is exactly the reference's
  ``1 - c1 z - c2 z^2 - c3 z^3 - c4 z^4`` and ``g1*g2 == scale``; in fp32 the
  cascade is well conditioned where the fused 4-tap direct form is not
  (SURVEY.md F5).
* ``decay_length`` -- number of samples after which the recursion's memory
  has decayed below ``eps``: the reference's mirror extension of n-1 samples
  (spatial.py:163-172) is truncated to min(K, n-1), which changes the output
  by O(eps) relative.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

import numpy as np

from .errors import ParameterError

MIN_RECURSIVE_SIGMA = 0.5  # spatial.py:28
DECAY_EPS = 1e-7


class SpatialKind(enum.Enum):
    BOX = "box"
    GAUSSIAN_RECURSIVE = "gauss-recursive"
    GAUSSIAN_FIR = "gauss-fir"


class Boundary(enum.Enum):
    MIRROR = "mirror"


@dataclass(frozen=True)
class SpatialSpec:
    """Choice and parameters of the spatial smoother (spatial.py:41-74)."""

    kind: SpatialKind
    radius: int = 0
    sigma_s: float = 0.0
    boundary: Boundary = Boundary.MIRROR

    def __post_init__(self):
        if self.kind is SpatialKind.BOX:
            if self.radius < 0:
                raise ParameterError(f"box radius must be >= 0, got {self.radius}")
        elif self.kind is SpatialKind.GAUSSIAN_FIR:
            if self.sigma_s <= 0.0:
                raise ParameterError(f"sigma_s must be positive, got {self.sigma_s}")
        elif self.kind is SpatialKind.GAUSSIAN_RECURSIVE:
            if self.sigma_s < MIN_RECURSIVE_SIGMA:
                raise ParameterError(
                    f"recursive Gaussian needs sigma_s >= {MIN_RECURSIVE_SIGMA}, "
                    f"got {self.sigma_s}"
                )

    @staticmethod
    def box(radius: int) -> "SpatialSpec":
        return SpatialSpec(SpatialKind.BOX, radius=radius)

    @staticmethod
    def gaussian_recursive(sigma_s: float) -> "SpatialSpec":
        return SpatialSpec(SpatialKind.GAUSSIAN_RECURSIVE, sigma_s=sigma_s)

    @staticmethod
    def gaussian_fir(sigma_s: float) -> "SpatialSpec":
        return SpatialSpec(SpatialKind.GAUSSIAN_FIR, sigma_s=sigma_s)


def gaussian_taps(sigma_s: float) -> np.ndarray:
    """Discretized Gaussian truncated at +-ceil(4 sigma), renormalised to unit
    DC gain (spatial.py:77-88)."""
    if sigma_s <= 0.0:
        raise ParameterError(f"sigma_s must be positive, got {sigma_s}")
    r = math.ceil(4.0 * sigma_s)
    i = np.arange(-r, r + 1, dtype=np.float64)
    taps = np.exp(-(i * i) / (2.0 * sigma_s * sigma_s))
    return taps / taps.sum()


def window_taps(spatial: SpatialSpec) -> np.ndarray:
    """1-D taps of the brute-force window (engines.py:96-106): uniform for box,
    the truncated FIR Gaussian for both Gaussian kinds."""
    if spatial.kind is SpatialKind.BOX:
        n = 2 * spatial.radius + 1
        return np.full(n, 1.0 / n)
    return gaussian_taps(spatial.sigma_s)


# spatial.py:95-98 -- prototype poles (radius, angle) of the two pairs.
_POLE_R1 = 0.4131045520976385
_POLE_TH1 = 0.07084882850910099
_POLE_R2 = 0.5259194528598873
_POLE_TH2 = 0.697835370819079


def _pole_pairs(alpha: float):
    r1 = _POLE_R1 ** (1.0 / alpha)
    t1 = _POLE_TH1 / alpha
    r2 = _POLE_R2 ** (1.0 / alpha)
    t2 = _POLE_TH2 / alpha
    a1 = 2.0 * r1 * math.cos(t1)
    a2 = -r1 * r1
    b1 = 2.0 * r2 * math.cos(t2)
    b2 = -r2 * r2
    return a1, a2, b1, b2, max(r1, r2)


def _taps_for_power(alpha: float):
    """(scale, c1..c4) of the direct form for pole power alpha (spatial.py:101-114)."""
    a1, a2, b1, b2, _ = _pole_pairs(alpha)
    c1 = a1 + b1
    c2 = a2 + b2 - a1 * b1
    c3 = -(a1 * b2 + a2 * b1)
    c4 = -a2 * b2
    return 1.0 - (c1 + c2 + c3 + c4), c1, c2, c3, c4


def _cascade_variance(taps) -> float:
    """Variance of the symmetric forward/backward cascade (spatial.py:117-121)."""
    scale, c1, c2, c3, c4 = taps
    s1 = c1 + 2.0 * c2 + 3.0 * c3 + 4.0 * c4
    s2 = c1 + 4.0 * c2 + 9.0 * c3 + 16.0 * c4
    return 2.0 * (s2 / scale + (s1 / scale) ** 2)


def pole_power(sigma_s: float) -> float:
    """Bisection on the pole power so the cascade variance is sigma_s^2
    (spatial.py:124-144: same interval, same 80 iterations)."""
    if sigma_s < MIN_RECURSIVE_SIGMA:
        raise ParameterError(
            f"recursive Gaussian needs sigma_s >= {MIN_RECURSIVE_SIGMA}, got {sigma_s}"
        )
    target = sigma_s * sigma_s
    lo, hi = 1e-3, 4096.0
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if _cascade_variance(_taps_for_power(mid)) < target:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def recursive_coeffs(sigma_s: float):
    """(scale, c1, c2, c3, c4) of the reference's direct form (spatial.py:124-144)."""
    return _taps_for_power(pole_power(sigma_s))


@dataclass(frozen=True)
class Biquads:
    """Two cascaded all-pole sections y = g x + a1 y[-1] + a2 y[-2]."""

    g1: float
    a1: float
    a2: float
    g2: float
    b1: float
    b2: float
    r_max: float  # largest pole radius (sets the decay length)


def recursive_biquads(sigma_s: float) -> Biquads:
    a1, a2, b1, b2, r_max = _pole_pairs(pole_power(sigma_s))
    return Biquads(1.0 - a1 - a2, a1, a2, 1.0 - b1 - b2, b1, b2, r_max)


def decay_length(sigma_s: float, eps: float = DECAY_EPS) -> int:
    """K = ceil(ln eps / ln r_max): mirror warm-up that reproduces the
    reference's full (n-1)-sample extension to O(eps)."""
    r = recursive_biquads(sigma_s).r_max
    return max(1, math.ceil(math.log(eps) / math.log(r)))
