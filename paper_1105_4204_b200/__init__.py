"""B200-native constant-time trigonometric bilateral filter (arXiv 1105.4204).

Drop-in for the reference package's hot path (``trigbf.bilateral_trig`` with a
recursive-Gaussian or box spatial smoother and a raised-cosine range kernel):
same entry point, parameters, errors and diagnostics, computed by hand-written
sm_100a kernels behind the C ABI in ``include/trigbf_b200.h``.
"""

from .engines import (
    ETA_GUARD,
    EngineDiagnostics,
    TrigFilter,
    bilateral_color,
    bilateral_direct,
    bilateral_trig,
    bilateral_trig_color,
    clear_plans,
    get_plan,
    layout_info,
)
from .errors import DimensionError, NativeUnavailableError, ParameterError, PnmParseError, TrigbfError
from .image import ErrorStats, Image, error_stats, image_from_planes
from .pnm import read_pnm, write_pnm
from .kernels import (
    DEGREE_TABLE_8BIT,
    GaussianRange,
    TermPairs,
    TrigKernel,
    degree_estimate,
    gaussian_eval,
    make_trig_kernel,
    select_degree,
    term_pairs,
    trig_eval,
)
from .spatial import (
    Boundary,
    SpatialKind,
    SpatialSpec,
    decay_length,
    gaussian_taps,
    recursive_biquads,
    recursive_coeffs,
    window_taps,
)

__version__ = "0.1.0"

__all__ = [
    "Boundary", "DEGREE_TABLE_8BIT", "DimensionError", "ETA_GUARD", "EngineDiagnostics",
    "ErrorStats", "GaussianRange", "Image", "NativeUnavailableError", "ParameterError", "PnmParseError", "SpatialKind",
    "SpatialSpec", "TermPairs", "TrigFilter", "TrigKernel", "TrigbfError", "bilateral_color",
    "bilateral_direct", "bilateral_trig", "bilateral_trig_color", "clear_plans", "decay_length", "degree_estimate", "error_stats",
    "gaussian_eval", "gaussian_taps", "get_plan", "image_from_planes", "layout_info", "make_trig_kernel", "recursive_biquads",
    "read_pnm", "recursive_coeffs", "select_degree", "term_pairs", "trig_eval", "window_taps", "write_pnm",
]
