"""Binary PGM/PPM (P5/P6, maxval 255) I/O, the data format on both sides of
the filter path (reference pnm.py:57-109, image.py:87-91).

Header: magic, width, height, maxval as whitespace-separated tokens, with '#'
comments to end of line, then exactly one whitespace byte and the raw
payload.  Samples come back as float64 planes [C][H][W]; writing quantises
with round-half-away-from-zero and clamps to [0, 255].
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionError, PnmParseError
from .image import Image

_SPACE = frozenset(b" \t\n\r\x0b\x0c")
_MAGIC_CHANNELS = {b"P5": 1, b"P6": 3}


def _header_tokens(data: bytes):
    """Yield (token, offset) for the four header fields; the generator's
    final position (after the maxval token) is returned via StopIteration."""
    pos, n = 0, len(data)
    for _ in range(4):
        while pos < n:  # separators and comments
            ch = data[pos]
            if ch == 0x23:  # '#'
                nl = data.find(b"\n", pos)
                pos = n if nl < 0 else nl + 1
            elif ch in _SPACE:
                pos += 1
            else:
                break
        start = pos
        while pos < n and data[pos] not in _SPACE:
            pos += 1
        yield data[start:pos], start
    return pos


def read_pnm(data: bytes) -> Image:
    """Parse binary PGM (P5) or PPM (P6) bytes into an Image."""
    data = bytes(data)
    names = ("magic number", "width", "height", "maxval")
    toks = _header_tokens(data)
    fields = []
    end = len(data)
    try:
        while True:
            fields.append(next(toks))
    except StopIteration as stop:
        end = stop.value
    values = []
    for name, (tok, off) in zip(names, fields):
        if not tok:
            raise PnmParseError(f"missing {name}", off)
        if name == "magic number":
            if tok not in _MAGIC_CHANNELS:
                raise PnmParseError(f"unsupported magic {tok!r}, expected P5 or P6", off)
            values.append(_MAGIC_CHANNELS[tok])
            continue
        try:
            v = int(tok)
        except ValueError:
            raise PnmParseError(f"{name} is not an integer: {tok!r}", off) from None
        if name in ("width", "height") and v < 1:
            raise PnmParseError(f"{name} must be positive, got {v}", off)
        if name == "maxval" and v != 255:
            raise PnmParseError(f"only maxval 255 is supported, got {v}", off)
        values.append(v)
    channels, width, height, _ = values
    if end >= len(data) or data[end] not in _SPACE:
        raise PnmParseError("expected single whitespace before payload", end)
    start = end + 1
    need = width * height * channels
    payload = np.frombuffer(data, dtype=np.uint8, count=min(need, len(data) - start), offset=start)
    if payload.size != need:
        raise PnmParseError(f"payload truncated: expected {need} bytes, got {payload.size}",
                            start + payload.size)
    px = payload.astype(np.float64).reshape(height, width, channels)
    return Image(width, height, channels, np.ascontiguousarray(px.transpose(2, 0, 1)))


def quantize(samples) -> np.ndarray:
    """Round half away from zero, clamp to [0, 255], uint8 (image.py:87-91)."""
    s = np.asarray(samples, dtype=np.float64)
    r = np.copysign(np.floor(np.abs(s) + 0.5), s)
    return np.clip(r, 0.0, 255.0).astype(np.uint8)


def write_pnm(img: Image) -> bytes:
    """Serialise an Image as binary PGM (1 channel) or PPM (3 channels)."""
    magic = {1: b"P5", 3: b"P6"}.get(img.channels)
    if magic is None:
        raise DimensionError(f"PNM supports 1 or 3 channels, got {img.channels}")
    q = quantize(img.samples)  # [C][H][W]
    body = np.ascontiguousarray(q.transpose(1, 2, 0))  # interleave channels
    return b"%s\n%d %d\n255\n" % (magic, img.width, img.height) + body.tobytes()
