"""The wire formats either side of the flow path (reference flowio.py:1-154):
binary PGM/PPM frames in, Middlebury ``.flo`` fields out.

Same names, argument meaning and error behaviour as the reference module:

* ``read_image(path)``   -> float64 (H, W) raster in [0, 255] (P5 / P6; 16-bit
  samples rescaled, P6 reduced to luminance 0.299 R + 0.587 G + 0.114 B);
* ``write_image(img, path)`` -> P5 (2-D) or P6 ((H, W, 3)), rounded, clipped;
* ``write_flo(flow, path)`` / ``read_flo(path)`` -> the ``PIEH`` layout
  (float32 tag 202021.25, int32 width, height, float32 (u, v) row-major,
  little endian);
* ``FileFormatError(ValueError)`` for undecodable or unencodable data.

``read_frame_u8`` is this package's fast path for 8-bit P5 frames: the raw
bytes go to the GPU as uint8 (the kernels convert to float64 exactly as
``read_image`` would, since x / 255 * 255 is not applied for maxval 255).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

FLO_TAG = 202021.25
FLO_MAX_DIM = 99999
UNKNOWN_FLOW = 1e10           # in-band "no flow" marker (Middlebury)
INVALID_THRESHOLD = 1e9       # |component| above this is invalid (metrics.py)
LUMA_WEIGHTS = (0.299, 0.587, 0.114)

_FLO_HEADER = struct.Struct("<fii")


class FileFormatError(ValueError):
    """An input file cannot be decoded, or an array cannot be written, in the
    requested format."""


def _header_ints(buf: bytes, pos: int, count: int):
    """``count`` whitespace-separated ASCII integers of a PNM header starting
    at ``pos`` ('#' comments run to end of line).  Returns the integers and
    the payload offset: exactly one whitespace byte ends the header."""
    vals = []
    end = len(buf)
    while len(vals) < count:
        while pos < end and buf[pos] in b" \t\r\n\x0b\x0c":
            pos += 1
        if pos < end and buf[pos] == ord("#"):
            nl = buf.find(b"\n", pos)
            pos = end if nl < 0 else nl
            continue
        stop = pos
        while stop < end and buf[stop] not in b" \t\r\n\x0b\x0c":
            stop += 1
        if stop == pos:
            raise FileFormatError("truncated image header")
        word = buf[pos:stop]
        if not word.isdigit():
            try:
                int(word)
            except ValueError as exc:
                raise FileFormatError(f"malformed header token {word!r}") from exc
        vals.append(int(word))
        pos = stop
    if pos >= end:
        raise FileFormatError("missing payload after header")
    return vals, pos + 1


def _decode_pnm(buf: bytes):
    magic = buf[:2]
    if magic not in (b"P5", b"P6"):
        raise FileFormatError(f"unsupported magic {magic!r}; expected binary P5 or P6")
    (w, h, maxval), start = _header_ints(buf, 2, 3)
    if w < 1 or h < 1:
        raise FileFormatError(f"invalid dimensions {w}x{h}")
    if not 0 < maxval < 65536:
        raise FileFormatError(f"invalid maxval {maxval}")
    chans = 3 if magic == b"P6" else 1
    sample = np.dtype(">u2") if maxval > 255 else np.dtype(np.uint8)
    nbytes = w * h * chans * sample.itemsize
    body = buf[start:start + nbytes]
    if len(body) < nbytes:
        raise FileFormatError(f"truncated payload: need {nbytes} bytes, found {len(body)}")
    px = np.frombuffer(body, dtype=sample)
    shape = (h, w, 3) if chans == 3 else (h, w)
    return px.reshape(shape), maxval


def read_image(path) -> np.ndarray:
    """Binary PGM/PPM -> float64 intensity raster in [0, 255]."""
    px, maxval = _decode_pnm(Path(path).read_bytes())
    img = px.astype(np.float64)
    if img.ndim == 3:  # luminance, same association order as the reference
        r, g, b = LUMA_WEIGHTS
        img = r * img[:, :, 0] + g * img[:, :, 1] + b * img[:, :, 2]
    if maxval != 255:
        img *= 255.0 / maxval
    return img


def read_frame_u8(path) -> np.ndarray:
    """8-bit P5 frame as its raw uint8 raster (the GPU converts it to float64;
    identical to ``read_image`` for maxval 255).  Other files fall back to
    ``read_image``."""
    px, maxval = _decode_pnm(Path(path).read_bytes())
    if px.ndim == 2 and maxval == 255 and px.dtype == np.uint8:
        return np.ascontiguousarray(px)
    return read_image(path)


def write_image(img, path) -> None:
    """(H, W) -> binary PGM, (H, W, 3) -> binary PPM; rounded and clipped to
    8 bits."""
    src = np.asarray(img)
    px = np.clip(np.rint(src), 0, 255).astype(np.uint8)
    if px.ndim == 2:
        magic = b"P5"
    elif px.ndim == 3 and px.shape[2] == 3:
        magic = b"P6"
    else:
        raise FileFormatError(f"cannot encode array of shape {src.shape}")
    h, w = px.shape[:2]
    Path(path).write_bytes(magic + b"\n%d %d\n255\n" % (w, h) + px.tobytes())


def flo_bytes(flow) -> bytes:
    """The .flo encoding of an (H, W, 2) field (``write_flo`` without the
    file).  Torch CUDA tensors are narrowed to float32 on the device before
    the copy (half the device-to-host bytes)."""
    try:
        import torch

        if isinstance(flow, torch.Tensor):
            if flow.dim() != 3 or flow.shape[2] != 2:
                raise ValueError(f"flow must have shape (H, W, 2), got {tuple(flow.shape)}")
            if not bool(torch.isfinite(flow).all()):
                raise ValueError("flow contains non-finite values; use the invalid sentinel")
            h, w = int(flow.shape[0]), int(flow.shape[1])
            if w > FLO_MAX_DIM or h > FLO_MAX_DIM:
                raise FileFormatError(
                    f"dimensions {w}x{h} exceed the format limit {FLO_MAX_DIM}")
            payload = flow.to(torch.float32).contiguous().cpu().numpy().astype("<f4")
            return _FLO_HEADER.pack(FLO_TAG, w, h) + payload.tobytes()
    except ImportError:  # pragma: no cover
        pass
    f = np.asarray(flow, dtype=np.float64)
    if f.ndim != 3 or f.shape[2] != 2:
        raise ValueError(f"flow must have shape (H, W, 2), got {f.shape}")
    h, w = f.shape[:2]
    if w > FLO_MAX_DIM or h > FLO_MAX_DIM:
        raise FileFormatError(f"dimensions {w}x{h} exceed the format limit {FLO_MAX_DIM}")
    if not np.isfinite(f).all():
        raise ValueError("flow contains non-finite values; use the invalid sentinel")
    return _FLO_HEADER.pack(FLO_TAG, w, h) + f.astype("<f4").tobytes()


def write_flo(flow, path) -> None:
    """Persist an (H, W, 2) field as .flo (values stored as float32)."""
    Path(path).write_bytes(flo_bytes(flow))


def read_flo(path) -> np.ndarray:
    """.flo -> (H, W, 2) float64; sentinel values pass through unchanged."""
    buf = Path(path).read_bytes()
    if len(buf) < _FLO_HEADER.size:
        raise FileFormatError("file too short for a flow header")
    tag, w, h = _FLO_HEADER.unpack_from(buf, 0)
    if tag != FLO_TAG:
        raise FileFormatError(f"bad magic {tag!r}; not a flow file")
    if not (0 < w <= FLO_MAX_DIM and 0 < h <= FLO_MAX_DIM):
        raise FileFormatError(f"implausible dimensions {w}x{h}")
    nbytes = 8 * w * h
    if len(buf) < _FLO_HEADER.size + nbytes:
        raise FileFormatError(
            f"truncated payload: need {nbytes} bytes, found {len(buf) - _FLO_HEADER.size}")
    vals = np.frombuffer(buf, dtype="<f4", count=2 * w * h, offset=_FLO_HEADER.size)
    return vals.astype(np.float64).reshape(h, w, 2)


def flow_valid_mask(flow) -> np.ndarray:
    """True where both components are finite and within the sentinel bound."""
    f = np.asarray(flow, dtype=np.float64)
    ok = np.isfinite(f) & (np.abs(f) <= INVALID_THRESHOLD)
    return ok.all(axis=-1)
