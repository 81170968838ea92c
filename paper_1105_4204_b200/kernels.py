"""Raised-cosine range kernel: degree rule, binomial weights, frequencies.

Host-side fp64 parameter layer of the drop-in.  Same public names, argument
meaning and errors as the reference (kernels.py:23-158):
``phi(s) = cos(omega*s)**N`` with ``gamma = pi/(2T)``, ``rho = gamma*sigma_r``,
``omega = gamma/(rho*sqrt(N)) = 1/(sigma_r*sqrt(N))``;
``coeffs[n] = 2**-N C(N, n)``, ``freqs[n] = (2n - N) omega``.

``term_pairs`` folds the symmetric spectrum into the (frequency, weight)
pairs the engine filters, exactly as engines.py:249-253 does.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ParameterError

# kernels.py:27-35 -- measured minimum degrees for an 8-bit range (T = 255).
DEGREE_TABLE_8BIT: dict[float, int] = {
    200.0: 1,
    150.0: 2,
    100.0: 3,
    80.0: 4,
    60.0: 5,
    50.0: 7,
    40.0: 9,
}

DEFAULT_WIDE_DEGREE = 5  # kernels.py:37
_EXACT_BINOMIAL_LIMIT = 1000  # kernels.py:41


@dataclass(frozen=True)
class TrigKernel:
    """Raised-cosine range kernel as coefficient/frequency lists (kernels.py:44-61)."""

    T: float
    gamma: float
    rho: float
    N: int
    omega: float
    coeffs: np.ndarray = field(repr=False)
    freqs: np.ndarray = field(repr=False)


def degree_estimate(sigma_r: float, T: float) -> int:
    """ceil((gamma*sigma_r)**-2) (kernels.py:76-82)."""
    if sigma_r <= 0.0 or T <= 0.0:
        raise ParameterError("sigma_r and T must be positive")
    gamma = math.pi / (2.0 * T)
    return math.ceil((gamma * sigma_r) ** -2)


def select_degree(sigma_r, T, lookup=None, default_degree=DEFAULT_WIDE_DEGREE) -> int:
    """Lookup hit wins; else the ceiling estimate for gamma*sigma_r < 1; else
    ``default_degree`` (kernels.py:85-104)."""
    if sigma_r <= 0.0 or T <= 0.0:
        raise ParameterError("sigma_r and T must be positive")
    if lookup is not None and sigma_r in lookup:
        return lookup[sigma_r]
    gamma = math.pi / (2.0 * T)
    if gamma * sigma_r < 1.0:
        return degree_estimate(sigma_r, T)
    return default_degree


def _binomial_coeffs(n_degree: int) -> np.ndarray:
    """2**-N C(N, n); exact integers up to N=1000, log-gamma beyond (kernels.py:107-122)."""
    if n_degree <= _EXACT_BINOMIAL_LIMIT:
        scale = 2.0 ** (-n_degree)
        return np.array([float(math.comb(n_degree, n)) * scale for n in range(n_degree + 1)])
    log_scale = -n_degree * math.log(2.0)
    lg_top = math.lgamma(n_degree + 1)
    return np.array(
        [
            math.exp(lg_top - math.lgamma(n + 1) - math.lgamma(n_degree - n + 1) + log_scale)
            for n in range(n_degree + 1)
        ]
    )


def make_trig_kernel(sigma_r: float, T: float = 255.0, degree: int | None = None, lookup=None) -> TrigKernel:
    """Scaled raised cosine approximating a Gaussian of std ``sigma_r`` on [-T, T]
    (kernels.py:125-158).  The 8-bit table is consulted when T == 255."""
    if sigma_r <= 0.0 or T <= 0.0:
        raise ParameterError("sigma_r and T must be positive")
    gamma = math.pi / (2.0 * T)
    rho = gamma * sigma_r
    if degree is None:
        if lookup is None and T == 255.0:
            lookup = DEGREE_TABLE_8BIT
        degree = select_degree(sigma_r, T, lookup=lookup)
    if degree < 0:
        raise ParameterError(f"degree must be >= 0, got {degree}")
    omega = gamma / (rho * math.sqrt(degree)) if degree > 0 else 0.0
    n = np.arange(degree + 1, dtype=np.float64)
    return TrigKernel(
        T=T,
        gamma=gamma,
        rho=rho,
        N=degree,
        omega=omega,
        coeffs=_binomial_coeffs(degree),
        freqs=(2.0 * n - degree) * omega,
    )


def trig_eval(k: TrigKernel, s):
    """sum_n coeffs[n] cos(freqs[n] s) == cos(omega s)**N (kernels.py:161-171)."""
    arr = np.asarray(s, dtype=np.float64)
    vals = np.cos(arr[..., None] * k.freqs) @ k.coeffs
    return float(vals) if arr.ndim == 0 else vals


@dataclass(frozen=True)
class GaussianRange:
    """Gaussian range kernel exp(-s^2 / 2 sigma^2) as a value the GPU
    brute-force engine can evaluate (the reference passes
    ``lambda s: gaussian_eval(sigma, s)``)."""

    sigma: float

    def __post_init__(self):
        if self.sigma <= 0.0:
            raise ParameterError(f"sigma must be positive, got {self.sigma}")

    def __call__(self, s):
        return gaussian_eval(self.sigma, s)


def gaussian_eval(sigma: float, s):
    """exp(-s^2 / 2 sigma^2) (kernels.py:174-182)."""
    if sigma <= 0.0:
        raise ParameterError(f"sigma must be positive, got {sigma}")
    arr = np.asarray(s, dtype=np.float64)
    vals = np.exp(-(arr * arr) / (2.0 * sigma * sigma))
    return float(vals) if arr.ndim == 0 else vals


@dataclass(frozen=True)
class TermPairs:
    """Distinct nonnegative frequencies and their folded weights, ascending.

    ``nu[j] = nu[0] + j*dnu`` with ``dnu = 2*omega``; a leading zero frequency
    is present for even N (engines.py:249-253).
    """

    nu: np.ndarray
    weight: np.ndarray
    dnu: float
    has_zero: bool

    @property
    def count(self) -> int:
        return int(self.nu.size)

    @property
    def spatial_passes(self) -> int:
        """4 per nonzero frequency + 1 for the zero frequency (engines.py:265-296)."""
        nz = self.count - (1 if self.has_zero else 0)
        return 4 * nz + (1 if self.has_zero else 0)


def term_pairs(kernel: TrigKernel) -> TermPairs:
    n_deg = kernel.N
    nu, w = [], []
    if n_deg % 2 == 0:
        nu.append(0.0)
        w.append(float(kernel.coeffs[n_deg // 2]))
    for n in range(n_deg // 2 + 1, n_deg + 1):
        nu.append((2 * n - n_deg) * kernel.omega)
        w.append(2.0 * float(kernel.coeffs[n]))
    return TermPairs(
        nu=np.asarray(nu, dtype=np.float64),
        weight=np.asarray(w, dtype=np.float64),
        dnu=2.0 * kernel.omega,
        has_zero=(n_deg % 2 == 0),
    )
