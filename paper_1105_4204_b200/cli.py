"""Command line for the B200 filter: the reference's ``filter`` and
``compare`` subcommands (cli.py:114-175) wired to the device engines.

    python -m paper_1105_4204_b200 filter in.pgm --output out.pgm --sigma-s 8 --sigma-r 20
    python -m paper_1105_4204_b200 compare in.pgm --sigma-s 3 --sigma-r 30

    python -m paper_1105_4204_b200 bench --csv grid.csv

Engines: ``trig`` (the constant-time filter; colour images go through one
batched call, channels as frames) and ``direct`` (GPU brute force with the
Gaussian range kernel).  ``bench`` times the reference's grid (cli.py:178-223:
sigma_s 10/100 x sigma_r 10..100 on a 720x540 seeded noise image, the
paper's Table setting) through the public call, host image in and out.  The
reference's ``poly`` engine and ``kernel`` subcommand are not on the B200 path.  Exit codes as the
reference: 0 ok, 1 usage/parameter error, 2 I/O or PNM parse error.
Outputs are written to a temporary file and renamed into place.
"""

from __future__ import annotations

import argparse
import os
import sys
import tempfile
import time

import numpy as np

from .engines import EngineDiagnostics, bilateral_color, bilateral_direct, bilateral_trig, bilateral_trig_color
from .errors import NativeUnavailableError, ParameterError, PnmParseError, TrigbfError
from .image import Image, error_stats
from .kernels import GaussianRange, make_trig_kernel
from .pnm import read_pnm, write_pnm
from .spatial import SpatialKind, SpatialSpec

OK, USAGE, IO = 0, 1, 2


class _ArgError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1, not argparse's 2
        self.print_usage(sys.stderr)
        raise _ArgError(message)


def _spatial(args) -> SpatialSpec:
    kind = SpatialKind(args.spatial)
    if kind is SpatialKind.BOX:  # box of comparable support (cli.py:60-65)
        return SpatialSpec.box(max(1, round(args.sigma_s)))
    return SpatialSpec(kind, sigma_s=args.sigma_s)


def _read(path: str) -> Image:
    with open(path, "rb") as fh:
        return read_pnm(fh.read())


def _write_atomic(path: str, payload: bytes) -> None:
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(os.path.abspath(path)), prefix=".tbf-", suffix=".tmp")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(payload)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def cmd_filter(args) -> int:
    if args.engine == "poly":
        print("tbf: error: the poly engine is not on the B200 path (use trig or direct)", file=sys.stderr)
        return USAGE
    img = _read(args.input)
    spatial = _spatial(args)
    diag = EngineDiagnostics()
    t0 = time.perf_counter()
    if args.engine == "trig":
        k = make_trig_kernel(args.sigma_r, args.range_max, degree=args.degree)
        if img.channels == 3:
            out = bilateral_trig_color(img, spatial, k, diagnostics=diag)
        else:
            out = bilateral_trig(img, spatial, k, workers=args.threads, diagnostics=diag)
    else:
        rng = GaussianRange(args.sigma_r)
        one = lambda ch: bilateral_direct(ch, spatial, rng, diagnostics=diag)  # noqa: E731
        out = bilateral_color(img, one) if img.channels == 3 else one(img)
    ms = (time.perf_counter() - t0) * 1e3
    _write_atomic(args.output, write_pnm(out))
    print(f"engine={args.engine} N={diag.degree} passes={diag.spatial_passes} "
          f"guarded={diag.guarded_pixels} threads={args.threads} backend=b200-sm100a time_ms={ms:.1f}")
    return OK


def cmd_compare(args) -> int:
    img = _read(args.input)
    if img.channels != 1:
        print("compare works on single-channel images", file=sys.stderr)
        return USAGE
    spatial = _spatial(args)
    k = make_trig_kernel(args.sigma_r, args.range_max, degree=args.degree)
    # "cosine": the same raised cosine in the brute force (exactness mode)
    rng = k if args.reference_range == "cosine" else GaussianRange(args.sigma_r)
    ref = bilateral_direct(img, spatial, rng)
    st = error_stats(bilateral_trig(img, spatial, k, workers=args.threads), ref)
    print(f"trig  N={k.N} vs direct: max_abs={st.max_abs:.4f} mean_abs={st.mean_abs:.4f} "
          f"std_dev={st.std_dev:.4f}")
    print("poly  not on the B200 path (skipped)")
    return OK


NOISE_SEED = 20260515  # the reference's synthetic benchmark image (bench.py:12-21)


def synthesize_noise(width: int = 720, height: int = 540, seed: int = NOISE_SEED) -> Image:
    """Seeded uniform byte noise, the reference CLI's default bench input."""
    px = np.random.default_rng(seed).integers(0, 256, size=(1, height, width))
    return Image(width, height, 1, px.astype(np.float64))


def _median_ms(fn, reps: int) -> float:
    ts = []
    for _ in range(max(1, reps)):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts))


def cmd_bench(args) -> int:
    if args.engine == "poly":
        print("tbf: error: the poly engine is not on the B200 path (use trig or direct)", file=sys.stderr)
        return USAGE
    img = _read(args.input) if args.input else synthesize_noise()
    if img.channels == 3:
        img = img.channel(0)
    rows = []
    if args.engine == "trig":
        kind = SpatialKind(args.spatial)
        for sigma_s in (10.0, 100.0):
            spatial = SpatialSpec(kind, sigma_s=sigma_s, radius=round(sigma_s))
            for sigma_r in (10.0, 20.0, 30.0, 40.0, 50.0, 60.0, 70.0, 80.0, 90.0, 100.0):
                k = make_trig_kernel(sigma_r, args.range_max, degree=args.degree)
                bilateral_trig(img, spatial, k)  # plan + workspace (cached)
                ms = _median_ms(lambda: bilateral_trig(img, spatial, k), args.reps)
                rows.append((sigma_s, sigma_r, k.N, "trig", ms))
    else:
        rng = GaussianRange(args.sigma_r)
        for sigma_s in (3.0, 5.0, 10.0):
            spatial = SpatialSpec.gaussian_fir(sigma_s)
            bilateral_direct(img, spatial, rng)
            ms = _median_ms(lambda: bilateral_direct(img, spatial, rng), args.reps)
            rows.append((sigma_s, args.sigma_r, 0, "direct", ms))
    lines = ["sigma_s,sigma_r,N,engine,median_ms"]
    lines += [f"{a:g},{b:g},{n},{e},{ms:.3f}" for a, b, n, e, ms in rows]
    text = "\n".join(lines) + "\n"
    if args.csv in (None, "-"):
        sys.stdout.write(text)
    else:
        _write_atomic(args.csv, text.encode("ascii"))
    print(f"bench done: engine={args.engine} reps={args.reps} backend=b200-sm100a", file=sys.stderr)
    return OK


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="tbf", description="B200 constant-time bilateral filter")
    sub = p.add_subparsers(dest="command", required=True)

    def common(sp, needs_input=True):
        if needs_input:
            sp.add_argument("input", help="binary PGM/PPM input")
        sp.add_argument("--sigma-s", type=float, default=15.0, dest="sigma_s")
        sp.add_argument("--sigma-r", type=float, default=80.0, dest="sigma_r")
        sp.add_argument("--range-max", type=float, default=255.0, dest="range_max")
        sp.add_argument("--spatial", choices=[k.value for k in SpatialKind], default="gauss-recursive")
        sp.add_argument("--degree", type=int, default=None)
        sp.add_argument("--terms", type=int, default=None, help="accepted for compatibility (poly only)")
        sp.add_argument("--threads", type=int, default=1, help="accepted for compatibility")

    f = sub.add_parser("filter", help="filter one image")
    common(f)
    f.add_argument("--engine", choices=["direct", "trig", "poly"], default="trig")
    f.add_argument("--output", required=True)
    f.set_defaults(func=cmd_filter)
    c = sub.add_parser("compare", help="trig engine vs the brute-force reference")
    common(c)
    c.add_argument("--reference-range", choices=["gaussian", "cosine"], default="gaussian",
                   dest="reference_range")
    c.set_defaults(func=cmd_compare)
    b = sub.add_parser("bench", help="wall-time grid (CSV)")
    common(b, needs_input=False)
    b.add_argument("input", nargs="?", default=None, help="optional PNM (default: 720x540 noise)")
    b.add_argument("--engine", choices=["direct", "trig", "poly"], default="trig")
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--csv", default=None, help="CSV path (default stdout)")
    b.set_defaults(func=cmd_bench)
    return p


def _check(args) -> None:
    for name in ("sigma_r", "sigma_s", "range_max"):
        if getattr(args, name) <= 0.0:
            raise ParameterError(f"--{name.replace('_', '-')} must be positive")
    if args.threads < 1:
        raise ParameterError("--threads must be >= 1")
    if args.terms is not None and args.terms < 1:
        raise ParameterError("--terms must be >= 1")
    if args.degree is not None and args.degree < 0:
        raise ParameterError("--degree must be >= 0")
    if getattr(args, "reps", 1) < 1:
        raise ParameterError("--reps must be >= 1")


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except _ArgError as e:
        print(f"tbf: error: {e}", file=sys.stderr)
        return USAGE
    except SystemExit as e:  # --help
        return int(e.code or 0)
    try:
        _check(args)
        return args.func(args)
    except (OSError, PnmParseError) as e:
        print(f"tbf: error: {e}", file=sys.stderr)
        return IO
    except (TrigbfError, NativeUnavailableError) as e:
        print(f"tbf: error: {e}", file=sys.stderr)
        return USAGE
