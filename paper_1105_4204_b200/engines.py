"""B200 bilateral engine: the drop-in for the reference's ``bilateral_trig``.

Reference entry (engines.py:228-306)::

    bilateral_trig(img, spatial, kernel, *, workers=1, diagnostics=None) -> Image

Same name, arguments, errors and diagnostics here.  Instead of looping over
frequencies in NumPy and calling the per-plane plugin (``_backend``) 4x per
term, the whole term loop (modulate -> separable smoothing -> demodulate ->
accumulate -> guarded ratio) runs as one fused device pipeline behind the C
ABI in include/trigbf_b200.h.  There is no CPU fallback: without the sm_100a
library or a CUDA device the call raises ``NativeUnavailableError``.

Accepted inputs: a reference-style ``Image`` (returns an ``Image``), a torch
tensor ``[H, W]`` or ``[B, H, W]`` (CUDA tensors stay on the device and the
result is a CUDA tensor; CPU tensors / NumPy arrays are copied in and out).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DimensionError, NativeUnavailableError, ParameterError
from .image import Image
from .kernels import GaussianRange, TrigKernel, term_pairs
from .spatial import SpatialKind, SpatialSpec, decay_length, recursive_biquads, window_taps

ETA_GUARD = 1e-12  # engines.py:36
WORKSPACE_FRACTION = 0.80  # of free device memory a plan may take


@dataclass
class EngineDiagnostics:
    """Counters filled by an engine run (engines.py:39-46)."""

    degree: int = 0
    spatial_passes: int = 0
    guarded_pixels: int = 0
    workers: int = 1


def _torch():
    try:
        import torch
    except ImportError as e:  # pragma: no cover
        raise NativeUnavailableError("torch is required for device memory") from e
    return torch


def spatial_struct(spatial: SpatialSpec) -> _native.TbfSpatial:
    """Reduce a SpatialSpec to the C struct (recursive: two biquads + decay length)."""
    s = _native.TbfSpatial()
    if spatial.kind is SpatialKind.GAUSSIAN_RECURSIVE:
        bq = recursive_biquads(spatial.sigma_s)
        k = decay_length(spatial.sigma_s)
        s.kind = _native.TBF_SPATIAL_RECURSIVE
        s.radius = 0
        s.g1, s.a1, s.a2, s.g2, s.b1, s.b2 = bq.g1, bq.a1, bq.a2, bq.g2, bq.b1, bq.b2
        s.ext_y = s.ext_x = k
    elif spatial.kind is SpatialKind.BOX:
        s.kind = _native.TBF_SPATIAL_BOX
        s.radius = int(spatial.radius)
    else:
        raise ParameterError(
            "the B200 path implements the O(1) smoothers (gauss-recursive, box); "
            f"got {spatial.kind.value}"
        )
    return s


class _TermsHolder:
    """Keeps the host arrays referenced by a TbfTerms struct alive."""

    def __init__(self, kernel: TrigKernel):
        pairs = term_pairs(kernel)
        self.pairs = pairs
        self.nu = np.ascontiguousarray(pairs.nu, dtype=np.float64)
        self.w = np.ascontiguousarray(pairs.weight, dtype=np.float64)
        self.struct = _native.TbfTerms()
        self.struct.n_terms = pairs.count
        self.struct.nu = self.nu.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        self.struct.weight = self.w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        self.struct.dnu = pairs.dnu
        self.struct.T = float(kernel.T)


class TrigFilter:
    """Reusable plan for one (frame shape, spatial spec, range kernel).

    Owns the device workspace; calls are asynchronous on the current torch
    stream (no host sync), so a plan can be timed back to back or captured in
    a CUDA graph.  Range violations and guarded pixels accumulate in a device
    counter pair read by :meth:`read_counters`.
    """

    def __init__(self, shape, spatial: SpatialSpec, kernel: TrigKernel, *, device=None,
                 batch_terms: int | None = None, term_range=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise NativeUnavailableError("no CUDA device: the B200 path has no CPU fallback")
        self.lib = _native.load()
        if len(shape) == 2:
            shape = (1, *shape)
        if len(shape) != 3 or min(shape) < 1:
            raise DimensionError(f"expected [B, H, W] with positive sizes, got {tuple(shape)}")
        self.B, self.H, self.W = (int(v) for v in shape)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.type != "cuda":
            raise ParameterError(f"plans live on a CUDA device, got {dev}")
        self.device = torch.device("cuda", torch.cuda.current_device() if dev.index is None else dev.index)
        self.spatial = spatial
        self.kernel = kernel
        self.sp = spatial_struct(spatial)
        self.terms = _TermsHolder(kernel)
        n = self.terms.pairs.count
        self.term_range = (0, n) if term_range is None else (int(term_range[0]), int(term_range[1]))
        if not (0 <= self.term_range[0] < self.term_range[1] <= n):
            raise ParameterError(f"bad term range {self.term_range} of {n}")
        self.batch_terms = self._pick_batch(batch_terms)
        nbytes = self.workspace_bytes(self.batch_terms)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.counters = torch.zeros(2, dtype=torch.int64, device=self.device)
        self._io = None  # device input/output of run_host, allocated on first use
        self._pin = None  # pinned host staging (in, out) for pageable callers
        # one call at a time per plan: the workspace, the staging buffers and
        # the counters are shared by every call through this plan (the
        # reference's engines are safe to call from several threads, e.g.
        # bilateral_color(..., workers=3)); reentrant so a caller can hold it
        # across a call and the counter read that belongs to it
        self.lock = threading.RLock()

    # -- sizing -----------------------------------------------------------
    def workspace_bytes(self, batch_terms: int) -> int:
        t0, t1 = self.term_range
        v = self.lib.tbf_workspace_bytes(self.B, self.H, self.W, ctypes.byref(self.sp), t0, t1,
                                         int(batch_terms))
        if v == 0:
            _native.check(_native.TBF_ERR_PARAM)
        return int(v)

    def _pick_batch(self, batch_terms):
        t0, t1 = self.term_range
        n = t1 - t0
        if batch_terms is not None:
            return max(0, min(int(batch_terms), n))
        torch = _torch()
        free, _ = torch.cuda.mem_get_info(self.device)
        budget = WORKSPACE_FRACTION * free
        if self.workspace_bytes(0) <= budget:
            return 0  # library default: a few pipelined batches
        # workspace is affine in the batch size: fit the slope on multiples of
        # 8, then take the largest multiple of 2 (whole pass-2 thread groups)
        # that fits, and spread the terms evenly over that many batches (each
        # batch re-reads the input and folds its partials: fewer is cheaper)
        w8, w16 = self.workspace_bytes(8), self.workspace_bytes(16)
        per = max(1, (w16 - w8) // 8)
        base = w8 - 8 * per
        tb = int((budget - base) // per) // 2 * 2
        if tb < 2:
            tb = 2 if self.workspace_bytes(2) <= budget else 0
        if tb < 1:
            raise ParameterError(
                f"image too large for device memory: needs {w8 / 2**30:.1f} GiB for 8 terms"
            )
        while tb > 2 and self.workspace_bytes(tb) > budget:
            tb -= 2
        if tb < n:
            nb = -(-n // tb)
            tb = min(tb, -(-n // nb) + (-(-n // nb)) % 2)  # even split, rounded up to even
        return min(tb, n)

    # -- calls ------------------------------------------------------------
    def _check_input(self, f, what: str = "input"):
        """A device buffer handed to the library: contiguous float32 on this
        plan's device with exactly B*H*W samples (anything else would be read
        or written out of bounds by the kernels)."""
        torch = _torch()
        if not isinstance(f, torch.Tensor) or f.dtype != torch.float32 or not f.is_cuda \
                or not f.is_contiguous():
            raise ParameterError(f"{what}: expected a contiguous float32 CUDA tensor")
        if f.device != self.device:
            raise ParameterError(f"{what}: on {f.device}, plan is on {self.device}")
        if f.numel() != self.B * self.H * self.W:
            raise DimensionError(f"{what} has {f.numel()} samples, plan expects "
                                 f"{self.B}x{self.H}x{self.W}")

    def _ctx(self):
        """Library calls run with the plan's device current (the C ABI works
        on the current device) on that device's current torch stream."""
        return _torch().cuda.device(self.device)

    def _stream(self):
        return _torch().cuda.current_stream(self.device).cuda_stream

    def __call__(self, f, out=None):
        """out[b] = bilateral_trig(f[b]); async on the current stream."""
        torch = _torch()
        self._check_input(f)
        if self.term_range != (0, self.terms.pairs.count):
            raise ParameterError("plan covers a term shard; use partial() + finalize()")
        if out is None:
            out = torch.empty_like(f)
        self._check_input(out, "out")
        with self.lock, self._ctx():
            rc = self.lib.tbf_bilateral_trig(
                f.data_ptr(), out.data_ptr(), self.B, self.H, self.W, ctypes.byref(self.sp),
                ctypes.byref(self.terms.struct), self.batch_terms, self.workspace.data_ptr(),
                self.workspace.numel(), self.counters.data_ptr(), self._stream())
        _native.check(rc)
        return out

    def run_host(self, h_in, h_out):
        """Host arrays in and out (NumPy arrays or CPU tensors, contiguous
        float32 with B*H*W samples): tbf_bilateral_trig_host.  Column strips
        of the input are copied while pass 1 starts on the first ones, and the
        output returns in row bands (pinned memory overlaps the copies with the
        filter; pageable memory works).  Stream-ordered: read_counters()
        (which syncs) before using h_out; keep both arrays alive until then."""
        torch = _torch()
        if self.term_range != (0, self.terms.pairs.count):
            raise ParameterError("plan covers a term shard; use partial() + finalize()")
        n = self.B * self.H * self.W
        p_in, p_out = _host_ptr(h_in, n, "input"), _host_ptr(h_out, n, "output")
        with self.lock, self._ctx():
            if self._io is None:
                self._io = torch.empty(2 * n, dtype=torch.float32, device=self.device)
            rc = self.lib.tbf_bilateral_trig_host(
                p_in, p_out, self.B, self.H, self.W, ctypes.byref(self.sp),
                ctypes.byref(self.terms.struct), self.batch_terms, self._io.data_ptr(),
                self.workspace.data_ptr(), self.workspace.numel(), self.counters.data_ptr(),
                self._stream())
        _native.check(rc)
        return h_out

    PIN_LIMIT = 1 << 32  # bytes per staging buffer; larger inputs copy pageable

    def run_staged(self, src, dst):
        """Pageable host arrays (NumPy, any float dtype; e.g. an Image's fp64
        planes) through pinned staging buffers cached in the plan: a
        multi-threaded dtype-converting copy into pinned memory, the
        strip/band-overlapped host entry, and a multi-threaded copy back into
        ``dst``.  Synchronous; returns (samples out of range, guarded)."""
        torch = _torch()
        n = self.B * self.H * self.W
        if src.size != n or dst.size != n:
            raise DimensionError(f"host arrays must hold {n} samples")
        with self.lock:
            return self._run_staged(src, dst, n)

    def _run_staged(self, src, dst, n):
        torch = _torch()
        if 4 * n > self.PIN_LIMIT:
            s32 = np.ascontiguousarray(src, dtype=np.float32)
            o32 = dst if (dst.dtype == np.float32 and dst.flags.c_contiguous) else np.empty(s32.shape, np.float32)
            self.run_host(s32, o32)
            counts = self.read_counters()
            if o32 is not dst:
                np.copyto(dst, o32.reshape(dst.shape))
            return counts
        if self._pin is None:
            self._pin = (torch.empty(n, dtype=torch.float32, pin_memory=True),
                         torch.empty(n, dtype=torch.float32, pin_memory=True))
        pin_in, pin_out = self._pin
        pin_in.copy_(torch.from_numpy(np.ascontiguousarray(src).reshape(-1)))
        self.run_host(pin_in, pin_out)
        counts = self.read_counters()  # syncs: pin_out is complete
        torch.from_numpy(dst.reshape(-1)).copy_(pin_out)
        return counts

    def partial(self, f, num, den, accumulate: bool = False, rows=None):
        """num/den (+)= contribution of this plan's term range (sharded path);
        with ``rows=(r0, r1)`` only to those output rows (tbf_trig_partial_rows:
        r0 a multiple of 128, r1 a multiple of 128 or H; recursive Gaussian)."""
        self._check_input(f)
        self._check_input(num, "num")
        self._check_input(den, "den")
        t0, t1 = self.term_range
        with self.lock, self._ctx():
            if rows is None:
                rc = self.lib.tbf_trig_partial(
                    f.data_ptr(), num.data_ptr(), den.data_ptr(), self.B, self.H, self.W,
                    ctypes.byref(self.sp), ctypes.byref(self.terms.struct), t0, t1, self.batch_terms,
                    int(bool(accumulate)), self.workspace.data_ptr(), self.workspace.numel(),
                    self._stream())
            else:
                rc = self.lib.tbf_trig_partial_rows(
                    f.data_ptr(), num.data_ptr(), den.data_ptr(), self.B, self.H, self.W,
                    ctypes.byref(self.sp), ctypes.byref(self.terms.struct), t0, t1, int(rows[0]), int(rows[1]),
                    self.batch_terms, int(bool(accumulate)), self.workspace.data_ptr(), self.workspace.numel(),
                    self._stream())
        _native.check(rc)

    def range_check(self, f):
        self._check_input(f)
        with self.lock, self._ctx():
            rc = self.lib.tbf_range_check(f.data_ptr(), f.numel(), float(self.kernel.T),
                                          self.counters.data_ptr(), self._stream())
        _native.check(rc)

    def finalize(self, num, den, f, out):
        for t, what in ((num, "num"), (den, "den"), (f, "input"), (out, "out")):
            self._check_input(t, what)
        with self.lock, self._ctx():
            rc = self.lib.tbf_finalize(num.data_ptr(), den.data_ptr(), f.data_ptr(), out.data_ptr(),
                                       f.numel(), self.counters.data_ptr(), self._stream())
        _native.check(rc)
        return out

    def read_counters(self, reset: bool = True):
        """(samples outside [0, T], guarded pixels) since the last reset; syncs."""
        with self.lock, self._ctx():
            vals = self.counters.tolist()
            if reset:
                self.counters.zero_()
        return int(vals[0]), int(vals[1])

    @property
    def spatial_passes(self) -> int:
        return self.terms.pairs.spatial_passes


def _host_ptr(a, n: int, what: str) -> int:
    """Address of a contiguous float32 host array (NumPy or CPU tensor)."""
    torch = _torch()
    if isinstance(a, np.ndarray):
        if a.dtype != np.float32 or not a.flags.c_contiguous:
            raise ParameterError(f"host {what} must be a C-contiguous float32 array")
        size, ptr = a.size, a.ctypes.data
    elif isinstance(a, torch.Tensor):
        if a.is_cuda or a.dtype != torch.float32 or not a.is_contiguous():
            raise ParameterError(f"host {what} must be a contiguous float32 CPU tensor")
        size, ptr = a.numel(), a.data_ptr()
    else:
        raise DimensionError(f"unsupported host {what} type {type(a).__name__}")
    if size != n:
        raise DimensionError(f"host {what} has {size} samples, plan expects {n}")
    return ptr


_PLANS: dict = {}
_MAX_PLANS = 4
_PLANS_LOCK = threading.RLock()


def _require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise NativeUnavailableError("no CUDA device: the B200 path has no CPU fallback")
    _native.load()


def get_plan(shape, spatial: SpatialSpec, kernel: TrigKernel, device=None) -> TrigFilter:
    """Cached plan (workspace reuse across calls with the same configuration)."""
    torch = _torch()
    _require_cuda()
    dev = torch.device("cuda" if device is None else device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (str(dev), tuple(shape), spatial, kernel.N, kernel.omega, kernel.T)
    with _PLANS_LOCK:
        plan = _PLANS.get(key)
        if plan is None:
            while len(_PLANS) >= _MAX_PLANS:
                _PLANS.pop(next(iter(_PLANS)))
            try:
                plan = TrigFilter(shape, spatial, kernel, device=dev)
            except torch.cuda.OutOfMemoryError:
                # cached plans hold large workspaces (up to ~80% of free memory for
                # a 16k^2 image): drop them and size the new plan from scratch
                # (a thread still using an evicted plan keeps its own reference)
                _PLANS.clear()
                torch.cuda.empty_cache()
                plan = TrigFilter(shape, spatial, kernel, device=dev)
            _PLANS[key] = plan
        return plan


def clear_plans() -> None:
    """Release the cached plans and their device workspaces."""
    with _PLANS_LOCK:
        _PLANS.clear()
    _torch().cuda.empty_cache()


def _check_kernel(kernel):
    if not isinstance(kernel, TrigKernel):
        # accept the reference's TrigKernel duck-typed (same fields)
        for attr in ("T", "N", "omega", "coeffs"):
            if not hasattr(kernel, attr):
                raise ParameterError("kernel must be a TrigKernel (make_trig_kernel)")
        kernel = TrigKernel(T=float(kernel.T), gamma=float(kernel.gamma), rho=float(kernel.rho),
                            N=int(kernel.N), omega=float(kernel.omega),
                            coeffs=np.asarray(kernel.coeffs), freqs=np.asarray(kernel.freqs))
    return kernel


def _check_spatial(spatial):
    if isinstance(spatial, SpatialSpec):
        return spatial
    kind = getattr(getattr(spatial, "kind", None), "value", None)
    if kind is None:
        raise ParameterError("spatial must be a SpatialSpec")
    return SpatialSpec(SpatialKind(kind), radius=int(getattr(spatial, "radius", 0)),
                       sigma_s=float(getattr(spatial, "sigma_s", 0.0)))


def bilateral_trig(img, spatial, kernel, *, workers: int = 1,
                   diagnostics: EngineDiagnostics | None = None):
    """Constant-time bilateral filter with a raised-cosine range kernel.

    Drop-in for the reference (engines.py:228-306): ``ParameterError`` when a
    sample leaves [0, T] (engines.py:218-225), ``DimensionError`` for
    multi-channel images (engines.py:68-73); ``diagnostics`` gets degree,
    spatial_passes (4 per nonzero frequency + 1 for the zero frequency),
    guarded_pixels and workers.  ``workers`` is accepted for signature
    compatibility; the device pipeline is deterministic for any value.
    """
    torch = _torch()
    kernel = _check_kernel(kernel)
    spatial = _check_spatial(spatial)
    _require_cuda()
    if diagnostics is not None:
        diagnostics.degree = kernel.N
        diagnostics.workers = workers

    def _finish(plan, shape, lo_hi, counts=None):
        bad, guarded = plan.read_counters() if counts is None else counts  # (syncs)
        if bad:
            lo, hi = lo_hi()
            raise ParameterError(
                f"samples in [{lo:g}, {hi:g}] exceed the declared range [0, {kernel.T:g}]; "
                "rescale the input or raise T"
            )
        if diagnostics is not None:
            diagnostics.spatial_passes += plan.spatial_passes * shape[0]
            diagnostics.guarded_pixels += guarded

    if isinstance(img, Image):
        if img.channels != 1:
            raise DimensionError(f"engine expects a single-channel image, got {img.channels} channels")
        host = img.samples[0]  # fp64 planes: converted inside the staging copy
        shape = (1, img.height, img.width)
        plan = get_plan(shape, spatial, kernel)
        res = np.empty((1, img.height, img.width), dtype=np.float64)
        counts = plan.run_staged(host, res)  # holds the plan's lock through its counter read
        _finish(plan, shape, lambda: (float(host.min()), float(host.max())), counts)
        return Image(img.width, img.height, 1, res)
    if isinstance(img, np.ndarray):
        if img.ndim not in (2, 3):
            raise DimensionError(f"expected [H, W] or [B, H, W], got shape {img.shape}")
        host = img if img.dtype in (np.float32, np.float64) else img.astype(np.float32)
        shape = (1, *host.shape) if host.ndim == 2 else host.shape
        plan = get_plan(shape, spatial, kernel)
        res = np.empty(host.shape, dtype=np.float32)
        counts = plan.run_staged(host, res)
        _finish(plan, shape, lambda: (float(host.min()), float(host.max())), counts)
        return res
    if not isinstance(img, torch.Tensor):
        raise DimensionError(f"unsupported input type {type(img).__name__}")
    if img.dim() not in (2, 3):
        raise DimensionError(f"expected [H, W] or [B, H, W], got shape {tuple(img.shape)}")
    shape = (1, *img.shape) if img.dim() == 2 else tuple(img.shape)
    if img.is_cuda:  # device in, device out, no copies
        f = img.to(dtype=torch.float32).contiguous()
        plan = get_plan(shape, spatial, kernel, device=f.device)
        with plan.lock:  # the call and the counter read that belongs to it
            out = plan(f)
            counts = plan.read_counters()
        _finish(plan, shape, lambda: (float(f.min()), float(f.max())), counts)
        return out.reshape(img.shape)
    pinned = img.is_pinned()
    if shape[0] >= 4 and pinned and img.dtype == torch.float32:
        # frame batches: sub-batches overlap copies and filtering across frames
        return _bilateral_trig_streamed(img, spatial, kernel, diagnostics)
    host = img.to(dtype=torch.float32).contiguous()
    res = torch.empty(tuple(img.shape), dtype=torch.float32, pin_memory=pinned)
    plan = get_plan(shape, spatial, kernel)
    with plan.lock:
        plan.run_host(host, res)
        counts = plan.read_counters()
    _finish(plan, shape, lambda: (float(host.min()), float(host.max())), counts)
    return res


def layout_info(shape, spatial: SpatialSpec, kernel: TrigKernel, *, host_entry: bool = False,
                batch_terms: int = 0, term_range=None) -> dict:
    """The launch layout a call would use (``tbf_layout_info``; no GPU
    needed): term batches, pass-1 y-chunks and pass-2 x-chunks, planned
    (unequal, costliest first) or equal.  ``shape`` is [H, W] or [B, H, W];
    ``host_entry`` selects the layout of the host-array entry."""
    lib = _native.load()
    if len(shape) == 2:
        shape = (1, *shape)
    B, H, W = (int(v) for v in shape)
    sp = spatial_struct(_check_spatial(spatial))
    terms = _TermsHolder(kernel)
    t0, t1 = (0, terms.pairs.count) if term_range is None else (int(term_range[0]), int(term_range[1]))
    info = (ctypes.c_int32 * _native.TBF_LAYOUT_INFO_N)()
    _native.check(lib.tbf_layout_info(B, H, W, ctypes.byref(sp), t0, t1, int(batch_terms), int(bool(host_entry)),
                                      info, _native.TBF_LAYOUT_INFO_N))
    return dict(zip(_native.LAYOUT_INFO_FIELDS, list(info)))


def bilateral_direct(img, spatial, range_fn, *, samples=None,
                     diagnostics: EngineDiagnostics | None = None):
    """Brute-force bilateral filter on the GPU in fp64 (engines.py:120-151).

    The reference's validation engine: every window sample is weighted by
    taps[dy] * taps[dx] * range(nb - centre) (window_taps: uniform for box,
    the truncated FIR Gaussian otherwise), borders reflect as np.pad
    "reflect", and the guarded ratio applies.  ``range_fn`` is a TrigKernel
    (raised cosine, = trig_eval) or a GaussianRange / positive float sigma
    (Gaussian, = gaussian_eval); arbitrary callables are not evaluated on the
    device.  ``samples`` = None filters every pixel and returns the input's
    container type (Image, NumPy fp64, or a fp64 CUDA tensor); otherwise an
    int array of (b, y, x) rows (or (y, x) rows for one frame) and the fp64
    values at those pixels are returned as NumPy.
    """
    torch = _torch()
    spatial = _check_spatial(spatial)
    _require_cuda()
    lib = _native.load()
    if isinstance(range_fn, TrigKernel) or hasattr(range_fn, "coeffs"):
        k = _check_kernel(range_fn)
        kind, param, degree = 1, float(k.omega), int(k.N)
    else:
        sigma = range_fn.sigma if isinstance(range_fn, GaussianRange) else range_fn
        if not isinstance(sigma, (int, float)) or sigma <= 0:
            raise ParameterError("range_fn must be a TrigKernel, a GaussianRange or a positive sigma")
        kind, param, degree = 0, float(sigma), 0
    # float64 inputs (an Image's planes, float64 arrays / tensors) stay float64:
    # the brute force then sees the reference's exact samples
    if isinstance(img, Image):
        if img.channels != 1:
            raise DimensionError(f"engine expects a single-channel image, got {img.channels} channels")
        f = torch.from_numpy(np.ascontiguousarray(img.samples[0], dtype=np.float64)).cuda()
    elif isinstance(img, np.ndarray):
        dt = np.float64 if img.dtype == np.float64 else np.float32
        f = torch.from_numpy(np.ascontiguousarray(img, dtype=dt)).cuda()
    elif isinstance(img, torch.Tensor):
        dt = torch.float64 if img.dtype == torch.float64 else torch.float32
        f = img.to(device="cuda" if not img.is_cuda else img.device, dtype=dt).contiguous()
    else:
        raise DimensionError(f"unsupported input type {type(img).__name__}")
    if f.dim() not in (2, 3):
        raise DimensionError(f"expected [H, W] or [B, H, W], got shape {tuple(f.shape)}")
    B, H, W = (1, *f.shape) if f.dim() == 2 else tuple(f.shape)
    taps = torch.from_numpy(window_taps(spatial)).to(f.device)
    radius = (taps.numel() - 1) // 2
    counters = torch.zeros(2, dtype=torch.int64, device=f.device)
    d_s = None
    if samples is not None:
        sm = np.asarray(samples, dtype=np.int64)
        if sm.ndim != 2 or sm.shape[1] not in (2, 3):
            raise DimensionError("samples must be (n, 3) (b, y, x) or (n, 2) (y, x) rows")
        if sm.shape[1] == 2:
            sm = np.concatenate([np.zeros((sm.shape[0], 1), np.int64), sm], axis=1)
        if sm.size and ((sm < 0).any() or (sm[:, 0] >= B).any() or (sm[:, 1] >= H).any()
                        or (sm[:, 2] >= W).any()):
            raise DimensionError("sample coordinates outside the image")
        d_s = torch.from_numpy(np.ascontiguousarray(sm, dtype=np.int32)).to(f.device)
        out = torch.empty(sm.shape[0], dtype=torch.float64, device=f.device)
        n = sm.shape[0]
    else:
        out = torch.empty((B, H, W), dtype=torch.float64, device=f.device)
        n = B * H * W
    stream = torch.cuda.current_stream(f.device).cuda_stream
    entry = lib.tbf_bilateral_direct_f64 if f.dtype == torch.float64 else lib.tbf_bilateral_direct
    _native.check(entry(
        f.data_ptr(), B, H, W, d_s.data_ptr() if d_s is not None else None, n, taps.data_ptr(),
        radius, kind, param, degree, out.data_ptr(), counters.data_ptr(), stream))
    guarded = int(counters[1].item())  # syncs
    if diagnostics is not None:
        diagnostics.guarded_pixels += guarded
    if samples is not None:
        return out.cpu().numpy()
    if isinstance(img, Image):
        return Image(img.width, img.height, 1, out.reshape(1, H, W).cpu().numpy())
    if isinstance(img, np.ndarray):
        return out.reshape(img.shape).cpu().numpy()
    return out.reshape(img.shape)


def _bilateral_trig_streamed(t, spatial, kernel, diagnostics, sub: int | None = None,
                             edges: bool = True):
    """Pinned host batch [B, H, W]: frames flow through the device in
    sub-batches so host->device copies, filtering and device->host copies of
    different sub-batches overlap (copy engines run beside the SMs).  Same
    result as one call: frames are independent."""
    with _STREAMED_LOCK:  # sub-batch plans and their counters are shared
        return _bilateral_trig_streamed_locked(t, spatial, kernel, diagnostics, sub, edges)


_STREAMED_LOCK = threading.Lock()


def _bilateral_trig_streamed_locked(t, spatial, kernel, diagnostics, sub, edges):
    torch = _torch()
    B, H, W = t.shape
    if sub is None:
        sub = max(1, min(B, (B + 7) // 8))  # ~8 sub-batches
    # sub-batch boundaries: with edges=True the first and last sub-batches are
    # single frames, so the copy-in before the first filter and the copy-out
    # after the last one (the parts no filtering overlaps) are one frame each
    bounds = [0]
    if edges and B >= 2 * sub + 2:
        bounds += [1]
        while bounds[-1] < B - 1:
            bounds.append(min(B - 1, bounds[-1] + sub))
        bounds.append(B)
    else:
        while bounds[-1] < B:
            bounds.append(min(B, bounds[-1] + sub))
    nsub = len(bounds) - 1
    dev = torch.device("cuda", torch.cuda.current_device())
    comp = torch.cuda.current_stream(dev)
    h2d = torch.cuda.Stream(dev)
    d2h = torch.cuda.Stream(dev)
    out_host = torch.empty((B, H, W), dtype=torch.float32, pin_memory=True)
    d_in = [torch.empty((sub, H, W), dtype=torch.float32, device=dev) for _ in range(2)]
    d_out = [torch.empty((sub, H, W), dtype=torch.float32, device=dev) for _ in range(2)]
    plans = {}
    ev_in = [torch.cuda.Event() for _ in range(nsub)]
    ev_comp = [torch.cuda.Event() for _ in range(nsub)]
    ev_out = [torch.cuda.Event() for _ in range(nsub)]
    for kk in range(nsub):
        b0, b1 = bounds[kk], bounds[kk + 1]
        nb = b1 - b0
        slot = kk % 2
        with torch.cuda.stream(h2d):
            if kk >= 2:  # the slot's previous compute has consumed it
                h2d.wait_event(ev_comp[kk - 2])
            d_in[slot][:nb].copy_(t[b0:b1], non_blocking=True)
            ev_in[kk].record(h2d)
        comp.wait_event(ev_in[kk])
        if kk >= 2:  # the slot's previous result has been copied out
            comp.wait_event(ev_out[kk - 2])
        plan = plans.get(nb)
        if plan is None:
            plan = plans[nb] = get_plan((nb, H, W), spatial, kernel, device=dev)
        plan(d_in[slot][:nb], d_out[slot][:nb])
        ev_comp[kk].record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(ev_comp[kk])
            out_host[b0:b1].copy_(d_out[slot][:nb], non_blocking=True)
            ev_out[kk].record(d2h)
    comp.wait_event(ev_out[nsub - 1])
    bad = guarded = 0
    for plan in plans.values():
        b_, g_ = plan.read_counters()  # synchronizes
        bad += b_
        guarded += g_
    torch.cuda.current_stream(dev).synchronize()
    if bad:
        raise ParameterError(
            f"samples exceed the declared range [0, {kernel.T:g}]; rescale the input or raise T")
    if diagnostics is not None:
        diagnostics.spatial_passes += plans[next(iter(plans))].spatial_passes * B
        diagnostics.guarded_pixels += guarded
    return out_host


def bilateral_color(img: Image, engine, workers: int = 1) -> Image:
    """Apply a single-channel engine to each channel (engines.py:354-369):
    channels independently, on a thread pool when workers > 1 (the device
    engine is thread-safe: each plan serialises its calls), reassembled in
    channel order."""
    if img.channels != 3:
        raise DimensionError(f"expected a 3-channel image, got {img.channels}")
    chans = [img.channel(c) for c in range(3)]
    if workers > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=workers) as pool:
            results = list(pool.map(engine, chans))
    else:
        results = [engine(ch) for ch in chans]
    stacked = np.stack([r.plane(0) for r in results])
    return Image(img.width, img.height, 3, stacked)


def bilateral_trig_color(img: Image, spatial, kernel, *, diagnostics=None) -> Image:
    """Colour image through one batched device call (channels as frames)."""
    if img.channels != 3:
        raise DimensionError(f"expected a 3-channel image, got {img.channels}")
    torch = _torch()
    f = torch.from_numpy(np.ascontiguousarray(img.samples, dtype=np.float32))
    out = bilateral_trig(f, spatial, kernel, diagnostics=diagnostics)
    return Image(img.width, img.height, 3, out.numpy().astype(np.float64))
