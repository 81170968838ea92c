"""Generate the golden fixtures from the REAL reference (oracle/_ref, built from
/root/reference/pkg by oracle/build_ref.sh).  Run in the builder container:

    PYTHONPATH=oracle/_ref python tests/golden/make_golden.py [--configs]

Outputs (committed, small):
  small_cases.npz   -- inputs + reference outputs of bilateral_trig on small
                       images (recursive Gaussian and box spatial, even/odd N,
                       degenerate shapes), plus plugin-level recursive_smooth /
                       box_pass vectors.
  config_2_box.npz  -- the config-2 image through the reference's box
                       spatial path (radius 8, full run), sampled pixels.
  pnm_cases.npz     -- PNM round trips through the reference's pnm module:
                       input bytes (with comments / odd whitespace), the parsed
                       planes, the re-written canonical bytes, quantisation of
                       half-way and out-of-range samples, and the byte offsets
                       of parse errors for malformed headers.
  config_<k>.npz    -- for each BASELINE config: sampled pixel positions and
                       the reference output there.  Configs 1, 2 and frames
                       of 4 are full reference runs; configs 3 and 5 use crops
                       whose margins exceed the recursion's decay length, so
                       interior pixels equal the full-image result (to 1e-7
                       relative); only interior pixels are sampled.
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import trigbf  # noqa: E402  (the reference)

from paper_1105_4204_b200 import workloads  # noqa: E402

SAMPLES = 2048


def ref_filter(plane: np.ndarray, kind: str, param, sigma_r, degree=None) -> np.ndarray:
    k = trigbf.make_trig_kernel(sigma_r, 255.0, degree=degree)
    spec = trigbf.SpatialSpec.box(param) if kind == "box" else trigbf.SpatialSpec.gaussian_recursive(param)
    img = trigbf.Image(plane.shape[1], plane.shape[0], 1, plane.astype(np.float64)[None])
    return trigbf.bilateral_trig(img, spec, k).plane(0)


SMALL = [
    # (name, h, w, kind, param, sigma_r, degree, seed)
    ("rec_1x1", 1, 1, "gauss-recursive", 3.0, 30.0, None, 1),
    ("rec_1x9", 1, 9, "gauss-recursive", 2.0, 30.0, None, 2),
    ("rec_9x1", 9, 1, "gauss-recursive", 2.0, 60.0, None, 3),
    ("rec_7x3", 7, 3, "gauss-recursive", 3.0, 60.0, None, 4),
    ("rec_40x30_s3", 30, 40, "gauss-recursive", 3.0, 60.0, None, 5),
    ("rec_64_s2_r80", 64, 64, "gauss-recursive", 2.0, 80.0, None, 6),
    ("rec_37x100_s5_r25", 37, 100, "gauss-recursive", 5.0, 25.0, None, 7),
    ("rec_65x33_s8_r20", 65, 33, "gauss-recursive", 8.0, 20.0, None, 8),
    ("rec_96x80_s3_r30", 96, 80, "gauss-recursive", 3.0, 30.0, None, 9),
    ("rec_70x130_s16_r10", 70, 130, "gauss-recursive", 16.0, 10.0, None, 10),
    ("rec_300x50_s4_r40", 300, 50, "gauss-recursive", 4.0, 40.0, None, 11),
    ("rec_48_s32_r15", 48, 48, "gauss-recursive", 32.0, 15.0, None, 12),
    ("rec_64_deg0", 64, 64, "gauss-recursive", 2.5, 80.0, 0, 13),
    ("rec_64_deg1", 64, 64, "gauss-recursive", 2.5, 170.0, 1, 14),
    ("rec_64_deg2", 64, 64, "gauss-recursive", 2.5, 170.0, 2, 15),
    ("rec_200x180_s6_r12", 180, 200, "gauss-recursive", 6.0, 12.0, None, 16),
    ("box_16_r1", 16, 16, "box", 1, 30.0, None, 21),
    ("box_64_r3_deg5", 64, 64, "box", 3, 170.0, 5, 22),
    ("box_20x10_r2", 10, 20, "box", 2, 80.0, None, 23),
    ("box_5x4_r7", 4, 5, "box", 7, 50.0, None, 24),
    ("box_37x53_r0", 53, 37, "box", 0, 30.0, None, 25),
    ("box_64_r9_r20", 64, 64, "box", 9, 20.0, None, 26),
]


def make_small(path: str) -> None:
    out = {}
    for name, h, w, kind, param, sr, deg, seed in SMALL:
        rng = np.random.default_rng(seed)
        f = rng.integers(0, 256, (h, w)).astype(np.float32)
        out[f"{name}__f"] = f
        out[f"{name}__out"] = ref_filter(f, kind, param, sr, deg)
        out[f"{name}__meta"] = np.array([h, w, 0 if kind == "box" else 1, param, sr,
                                         -1 if deg is None else deg], dtype=np.float64)
    # plugin-level vectors (test_backends.py:18-43 analogue)
    from trigbf import _fallback
    from trigbf.spatial import recursive_coeffs

    rng = np.random.default_rng(31)
    for i, sigma in enumerate((0.5, 2.0, 7.5, 30.0)):
        h, w = int(rng.integers(1, 50)), int(rng.integers(1, 50))
        a = rng.uniform(0, 255, (h, w))
        out[f"plugin_rec{i}__a"] = a
        out[f"plugin_rec{i}__taps"] = np.array(recursive_coeffs(sigma))
        out[f"plugin_rec{i}__out"] = _fallback.recursive_smooth(a, *recursive_coeffs(sigma), h - 1)
    for i, radius in enumerate((0, 1, 3, 11, 40)):
        a = rng.uniform(0, 255, (9, 13))
        out[f"plugin_box{i}__a"] = a
        out[f"plugin_box{i}__radius"] = np.array([radius])
        out[f"plugin_box{i}__out"] = _fallback.box_pass(a, radius)
    np.savez_compressed(path, **out)


def _sample(region, n, rng):
    """n random (y, x) positions in region = (y0, y1, x0, x1)."""
    y0, y1, x0, x1 = region
    ys = rng.integers(y0, y1, n)
    xs = rng.integers(x0, x1, n)
    return ys, xs


def _crop_job(args):
    cfg_id, y0, y1, x0, x1 = args
    cfg = workloads.CONFIGS[cfg_id]
    full = workloads.frame(cfg, 0)
    crop = np.ascontiguousarray(full[y0:y1, x0:x1])
    t = time.time()
    out = ref_filter(crop, "gauss-recursive", cfg.sigma_s, cfg.sigma_r)
    return (y0, y1, x0, x1), out, time.time() - t


def _frame_job(args):
    cfg_id, idx = args
    cfg = workloads.CONFIGS[cfg_id]
    f = workloads.frame(cfg, idx)
    t = time.time()
    return idx, ref_filter(f, "gauss-recursive", cfg.sigma_s, cfg.sigma_r), time.time() - t


def make_config(cfg_id: int, path: str, pool) -> None:
    cfg = workloads.CONFIGS[cfg_id]
    rng = np.random.default_rng(100 + cfg_id)
    rec = {"sigma_s": cfg.sigma_s, "sigma_r": cfg.sigma_r}
    frames, ys, xs, vals, kinds = [], [], [], [], []
    t0 = time.time()
    if cfg_id in (1, 2, 4):
        idxs = [0] if cfg_id != 4 else [0, 37, 63]
        for idx, out, dt in pool.map(_frame_job, [(cfg_id, i) for i in idxs]):
            y, x = _sample((0, cfg.height, 0, cfg.width), SAMPLES, rng)
            # always include the four corners and edge midpoints
            y = np.concatenate([y, [0, 0, cfg.height - 1, cfg.height - 1, cfg.height // 2, 0]])
            x = np.concatenate([x, [0, cfg.width - 1, 0, cfg.width - 1, 0, cfg.width // 2]])
            frames.append(np.full(y.size, idx))
            ys.append(y)
            xs.append(x)
            vals.append(out[y, x])
            print(f"cfg{cfg_id} frame {idx}: reference {dt:.1f}s", flush=True)
    else:
        K = {3: 187, 5: 373}[cfg_id]
        margin = K + 64
        c = 3 * margin  # crop side
        H, W = cfg.height, cfg.width
        crops = [(0, c, 0, c), (0, c, W - c, W), (H - c, H, 0, c), (H - c, H, W - c, W),
                 (H // 2 - c // 2, H // 2 + c // 2, W // 2 - c // 2, W // 2 + c // 2)]
        jobs = [(cfg_id, *cr) for cr in crops]
        for (y0, y1, x0, x1), out, dt in pool.map(_crop_job, jobs):
            # interior: at least `margin` away from crop edges that are not image edges
            iy0 = 0 if y0 == 0 else margin
            iy1 = (y1 - y0) if y1 == H else (y1 - y0) - margin
            ix0 = 0 if x0 == 0 else margin
            ix1 = (x1 - x0) if x1 == W else (x1 - x0) - margin
            ly, lx = _sample((iy0, iy1, ix0, ix1), SAMPLES // 2, rng)
            frames.append(np.zeros(ly.size, dtype=np.int64))
            ys.append(ly + y0)
            xs.append(lx + x0)
            vals.append(out[ly, lx])
            print(f"cfg{cfg_id} crop {(y0, y1, x0, x1)}: reference {dt:.1f}s", flush=True)
    np.savez_compressed(path, frame=np.concatenate(frames), y=np.concatenate(ys),
                        x=np.concatenate(xs), value=np.concatenate(vals),
                        sigma_s=cfg.sigma_s, sigma_r=cfg.sigma_r,
                        reference_backend=trigbf.backend_name())
    print(f"cfg{cfg_id}: {time.time() - t0:.1f}s -> {path}", flush=True)


sys.path.insert(0, os.path.dirname(HERE))
from pnm_bad_cases import PNM_BAD  # noqa: E402  (shared with tests/test_pnm_cli.py)


def make_pnm(path: str) -> None:
    from trigbf import pnm as rpnm

    rng = np.random.default_rng(77)
    out = {}
    good = [
        b"P5\n# comment\n3 2\n255\n" + bytes(rng.integers(0, 256, 6, dtype=np.uint8)),
        b"P5 4\t1 #x\n255\r" + bytes(rng.integers(0, 256, 4, dtype=np.uint8)),
        b"P6\n2 2\n255\n" + bytes(rng.integers(0, 256, 12, dtype=np.uint8)),
    ]
    for i, data in enumerate(good):
        img = rpnm.read_pnm(data)
        out[f"good{i}_in"] = np.frombuffer(data, np.uint8)
        out[f"good{i}_planes"] = img.samples
        out[f"good{i}_out"] = np.frombuffer(rpnm.write_pnm(img), np.uint8)
    # quantisation: halves, negatives, out of range
    q = np.array([[[-0.5, 0.49999, 0.5, 1.5, 2.5, 254.5, 255.4, 300.0, -7.0, 127.5]]])
    img = trigbf.Image(10, 1, 1, q)
    out["quant_in"] = q
    out["quant_out"] = np.frombuffer(rpnm.write_pnm(img), np.uint8)
    offs = []
    for data in PNM_BAD:
        try:
            rpnm.read_pnm(data)
            offs.append(-1)
        except trigbf.PnmParseError as e:
            offs.append(e.offset)
    out["bad_offsets"] = np.array(offs, np.int64)
    np.savez_compressed(path, **out)


def make_box_config(path: str, radius: int = 8) -> None:
    """The config-2 image through the reference's box spatial path (full
    2048^2 run, N = 66): the box kernels at a BASELINE size."""
    cfg = workloads.CONFIGS[2]
    f = workloads.frame(cfg, 0)
    t = time.time()
    out = ref_filter(f, "box", radius, cfg.sigma_r)
    rng = np.random.default_rng(2024)
    ys, xs = _sample((0, f.shape[0], 0, f.shape[1]), SAMPLES, rng)
    # plus the four borders, where the mirror indexing matters
    ys = np.concatenate([ys, [0, 0, f.shape[0] - 1, f.shape[0] - 1, 0, 1023, 2047, 5]])
    xs = np.concatenate([xs, [0, f.shape[1] - 1, 0, f.shape[1] - 1, 1023, 0, 700, 2047]])
    np.savez_compressed(path, frame=np.zeros(ys.size, np.int64), y=ys, x=xs, value=out[ys, xs],
                        radius=radius, sigma_r=cfg.sigma_r, reference_backend=trigbf.backend_name())
    print(f"box cfg2: {time.time() - t:.1f}s -> {path}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="", help="comma list of config ids to (re)generate")
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--pnm", action="store_true")
    ap.add_argument("--box-config", action="store_true")
    args = ap.parse_args()
    if args.box_config:
        make_box_config(os.path.join(HERE, "config_2_box.npz"))
    if args.pnm:
        make_pnm(os.path.join(HERE, "pnm_cases.npz"))
        print("pnm cases written")
    if args.small:
        make_small(os.path.join(HERE, "small_cases.npz"))
        print("small cases written")
    ids = [int(v) for v in args.configs.split(",") if v]
    if ids:
        with ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
            for k in ids:
                make_config(k, os.path.join(HERE, f"config_{k}.npz"), pool)


if __name__ == "__main__":
    main()
