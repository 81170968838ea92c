"""Golden fixtures for the guarded ratio when it fires and for colour images,
generated from the REAL reference (oracle/_ref, built from /root/reference/pkg
by oracle/build_ref.sh).  Run in the builder container:

    python tests/golden/make_guard_color.py

Outputs (committed, small):
  guard_cases.npz  -- images filtered with odd low degrees (rho*sqrt(N) < 1),
                      where the raised cosine goes negative and den < 1e-12
                      on many pixels (engines.py:109-117): input, reference
                      output, reference guarded-pixel count, and the float64
                      den of the oracle restatement (pinned to the reference
                      to 1e-9 in test_oracle.py) to tell well-conditioned
                      pixels from ones within fp32 rounding of the threshold.
  color_cases.npz  -- 3-channel images through the reference's
                      bilateral_color (engines.py:354-369) with a
                      bilateral_trig engine per channel: input and output.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import trigbf  # noqa: E402  (the reference)

from oracle import trigbf_oracle as orc  # noqa: E402
from paper_1105_4204_b200.workloads import rects_image  # noqa: E402

# (name, h, w, kind, param, sigma_r, degree, image, seed)
GUARD = [
    ("box_r2_deg1", 64, 80, "box", 2, 10.0, 1, "noise", 5),
    ("rec_s2_deg1", 64, 80, "gauss-recursive", 2.0, 10.0, 1, "noise", 5),
    ("rec_s2_deg3", 64, 80, "gauss-recursive", 2.0, 10.0, 3, "noise", 6),
    ("box_r2_deg5", 48, 40, "box", 2, 6.0, 5, "noise", 7),
    ("rec_s3_deg1_rects", 96, 80, "gauss-recursive", 3.0, 20.0, 1, "rects", 8),
    ("box_r3_deg3_rects", 80, 96, "box", 3, 12.0, 3, "rects", 9),
]

COLOR = [
    ("rec_s3_r30", 48, 64, "gauss-recursive", 3.0, 30.0, 11),
    ("box_r2_r40", 40, 56, "box", 2, 40.0, 12),
]


def _spec(kind, param):
    return trigbf.SpatialSpec.box(int(param)) if kind == "box" else trigbf.SpatialSpec.gaussian_recursive(float(param))


def _image(kind, h, w, seed):
    if kind == "noise":
        return np.random.default_rng(seed).integers(0, 256, (h, w)).astype(np.float32)
    return rects_image(h, w, 8, seed=seed).astype(np.float32)


def make_guard(path):
    out = {}
    for name, h, w, kind, param, sr, deg, img, seed in GUARD:
        f = _image(img, h, w, seed)
        k = trigbf.make_trig_kernel(sr, 255.0, degree=deg)
        diag = trigbf.EngineDiagnostics()
        res = trigbf.bilateral_trig(trigbf.Image(w, h, 1, f.astype(np.float64)[None]), _spec(kind, param), k,
                                    diagnostics=diag)
        _, info = orc.bilateral_trig(f.astype(np.float64), kind, param, orc.make_trig_kernel(sr, 255.0, degree=deg),
                                     return_numden=True)
        assert info["guarded_pixels"] == diag.guarded_pixels
        out[f"{name}__f"] = f
        out[f"{name}__out"] = res.plane(0)
        out[f"{name}__den"] = info["den"]
        out[f"{name}__guarded"] = np.array([diag.guarded_pixels])
        out[f"{name}__meta"] = np.array([h, w, 0 if kind == "box" else 1, param, sr, deg], dtype=np.float64)
        print(f"{name}: guarded {diag.guarded_pixels} of {h * w}")
    np.savez_compressed(path, **out)


def make_color(path):
    out = {}
    for name, h, w, kind, param, sr, seed in COLOR:
        chans = np.stack([rects_image(h, w, 6, seed=seed + 100 * c) for c in range(3)]).astype(np.float64)
        img = trigbf.Image(w, h, 3, chans)
        spec = _spec(kind, param)
        k = trigbf.make_trig_kernel(sr, 255.0)
        res = trigbf.bilateral_color(img, lambda ch: trigbf.bilateral_trig(ch, spec, k), workers=3)
        out[f"{name}__f"] = chans
        out[f"{name}__out"] = res.samples
        out[f"{name}__meta"] = np.array([h, w, 0 if kind == "box" else 1, param, sr], dtype=np.float64)
        print(f"{name}: colour {h}x{w}x3")
    np.savez_compressed(path, **out)


if __name__ == "__main__":
    make_guard(os.path.join(HERE, "guard_cases.npz"))
    make_color(os.path.join(HERE, "color_cases.npz"))
