"""PGM (P2 ASCII / P5 binary) I/O — drop-in for reference pgmio.py:19-137.

Headers (a few dozen bytes) and the ASCII P2 form are parsed on the host;
P5 pixel payloads are decoded on the GPU from the raw file bytes
(`sbf_pgm_decode`: 8-bit or big-endian 16-bit -> fp32, exact for
maxval <= 65535) and results are quantised on the GPU (`sbf_pgm_encode`:
clamp to [0, maxval], floor(x + 0.5), as the reference's save_pgm).
Parse failures raise PgmParseError carrying the byte offset.
"""

from __future__ import annotations

from pathlib import Path
from typing import NamedTuple

import numpy as np

from . import _lib
from .errors import InvalidParameterError, PgmParseError

_SPACE = frozenset(b" \t\r\n\x0b\x0c")


class PgmHeader(NamedTuple):
    magic: str
    width: int
    height: int
    maxval: int
    data_offset: int


def _token(data: bytes, pos: int):
    """Next header token after whitespace and '#' comments: (token, start, end)."""
    n = len(data)
    while pos < n:
        c = data[pos]
        if c == 0x23:  # '#': comment to end of line
            while pos < n and data[pos] not in (0x0A, 0x0D):
                pos += 1
        elif c in _SPACE:
            pos += 1
        else:
            break
    if pos >= n:
        raise PgmParseError("unexpected end of header", pos)
    start = pos
    while pos < n and data[pos] not in _SPACE and data[pos] != 0x23:
        pos += 1
    return data[start:pos], start, pos


def _positive_int(data, pos, what, upper=None):
    tok, start, pos = _token(data, pos)
    try:
        v = int(tok)
    except ValueError:
        raise PgmParseError(f"{what} is not an integer: {tok!r}", start) from None
    if v <= 0:
        raise PgmParseError(f"{what} must be positive, got {v}", start)
    if upper is not None and v > upper:
        raise PgmParseError(f"{what} {v} exceeds the supported maximum {upper}", start)
    return v, pos


def _header(data: bytes) -> PgmHeader:
    magic, start, pos = _token(data, 0)
    if magic not in (b"P2", b"P5"):
        raise PgmParseError(f"unsupported magic {magic!r} (want P2 or P5)", start)
    w, pos = _positive_int(data, pos, "width")
    h, pos = _positive_int(data, pos, "height")
    mv, pos = _positive_int(data, pos, "maxval", upper=65535)
    if magic == b"P5":
        if pos >= len(data) or data[pos] not in _SPACE:
            raise PgmParseError("missing whitespace after maxval", pos)
        pos += 1
    return PgmHeader(magic.decode(), w, h, mv, pos)


def inspect_pgm(path) -> PgmHeader:
    """Header only; `data_offset` is where the pixel data begins."""
    return _header(Path(path).read_bytes())


def _p2_samples(data: bytes, hdr: PgmHeader) -> np.ndarray:
    count = hdr.width * hdr.height
    out = np.empty(count)
    pos = hdr.data_offset
    for i in range(count):
        try:
            tok, start, pos = _token(data, pos)
        except PgmParseError:
            raise PgmParseError(f"truncated pixel data: expected {count} samples, got {i}",
                                len(data)) from None
        try:
            v = int(tok)
        except ValueError:
            raise PgmParseError(f"sample is not an integer: {tok!r}", start) from None
        if v < 0 or v > hdr.maxval:
            raise PgmParseError(f"sample value {v} outside [0, {hdr.maxval}]", start)
        out[i] = v
    return out.reshape(hdr.height, hdr.width)


def load_pgm_device(path, device="cuda"):
    """Load a PGM straight into a float32 CUDA tensor (P5 decoded on the GPU)."""
    import torch

    data = Path(path).read_bytes()
    hdr = _header(data)
    count = hdr.width * hdr.height
    if hdr.magic == "P2":
        return torch.from_numpy(_p2_samples(data, hdr).astype(np.float32)).to(device)
    bpp = 1 if hdr.maxval < 256 else 2
    need = count * bpp
    avail = len(data) - hdr.data_offset
    if avail < need:
        raise PgmParseError(f"truncated pixel data: expected {need} bytes, got {avail}", len(data))
    raw = torch.frombuffer(bytearray(data[hdr.data_offset:hdr.data_offset + need]),
                           dtype=torch.uint8).to(device)
    out = torch.empty((hdr.height, hdr.width), dtype=torch.float32, device=device)
    _lib.check(_lib.load().sbf_pgm_decode(raw.data_ptr(), bpp, count, out.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream), "pgm_decode")
    return out


def load_pgm(path) -> np.ndarray:
    """Load a P2/P5 PGM as a float64 image (reference semantics)."""
    data = Path(path).read_bytes()
    hdr = _header(data)
    if hdr.magic == "P2":
        return _p2_samples(data, hdr)
    return load_pgm_device(path).cpu().numpy().astype(np.float64)


def encode_pgm_payload(img, maxval=255):
    """Quantised payload bytes of an image (numpy or CUDA tensor), on the GPU."""
    import torch

    if not 1 <= maxval <= 65535:
        raise InvalidParameterError("maxval must lie in [1, 65535]")
    t = img if isinstance(img, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(img))
    if t.ndim != 2 or t.numel() == 0:
        raise InvalidParameterError("image must be 2-D and non-empty")
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    t = t.to("cuda").contiguous()
    if not bool(torch.isfinite(t).all()):
        raise InvalidParameterError("image contains non-finite samples")
    bpp = 1 if maxval < 256 else 2
    out = torch.empty(t.numel() * bpp, dtype=torch.uint8, device=t.device)
    _lib.check(_lib.load().sbf_pgm_encode(t.data_ptr(), _lib.SBF_F64 if t.dtype == torch.float64
                                          else _lib.SBF_F32, t.numel(), int(maxval),
                                          out.data_ptr(), torch.cuda.current_stream().cuda_stream),
               "pgm_encode")
    return out.cpu().numpy().tobytes(), int(t.shape[0]), int(t.shape[1])


def save_pgm(img, path, maxval=255, binary=True):
    """Write an image, clamping to [0, maxval] and rounding half away from zero."""
    payload, h, w = encode_pgm_payload(img, maxval)
    with open(path, "wb") as fh:
        fh.write(f"{'P5' if binary else 'P2'}\n{w} {h}\n{maxval}\n".encode())
        if binary:
            fh.write(payload)
        else:
            q = (np.frombuffer(payload, dtype=np.uint8) if maxval < 256
                 else np.frombuffer(payload, dtype=">u2")).reshape(h, w)
            fh.write(("\n".join(" ".join(str(int(v)) for v in row) for row in q) + "\n").encode())
