"""netpbm I/O (mirrors the reference's netpbm.py:1-200) and the P4 fast path.

Same names, formats and NetpbmError messages as the reference:
read_pbm / write_pbm (P1 plain, P4 packed: 1 bit per pixel, MSB first, rows
padded to a byte, padding ignored on read and zero on write, value 1 = black =
object) and read_pgm / write_pgm (P2 / P5 renderings of squared distance
maps).  Parse errors carry the byte offset where they occurred.

New here: P4 rasters go to the device as they are on
disk.  `read_pbm_raster` returns the packed raster without unpacking it,
`hasf_p4` smooths a batch of P4 rasters through ts_hasf_batch_p4 (P4 -> the
kernel's bit rows -> P4, all on the device; 1/8 B per pixel each way over the
host link), `write_pbm_raster` writes one back.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import ADJ_84, Adjacency, as_binary

_WHITESPACE = frozenset(b" \t\r\n\x0b\x0c")


class NetpbmError(ValueError):
    """Malformed netpbm input (netpbm.py:19-20)."""


class _Reader:
    """Header tokenizer: whitespace and '#' comments (to end of line) separate
    tokens (netpbm.py:23-58)."""

    def __init__(self, data: bytes):
        self.data = data
        self.pos = 0

    def skip(self) -> None:
        d, n = self.data, len(self.data)
        while self.pos < n:
            c = d[self.pos]
            if c == 0x23:
                while self.pos < n and d[self.pos] not in (0x0A, 0x0D):
                    self.pos += 1
            elif c in _WHITESPACE:
                self.pos += 1
            else:
                break

    def token(self, what: str) -> bytes:
        self.skip()
        d = self.data
        if self.pos >= len(d):
            raise NetpbmError(f"unexpected end of file at byte {self.pos} while reading {what}")
        start = self.pos
        while self.pos < len(d) and d[self.pos] not in _WHITESPACE and d[self.pos] != 0x23:
            self.pos += 1
        return d[start:self.pos]

    def integer(self, what: str) -> int:
        start = self.pos
        tok = self.token(what)
        try:
            return int(tok)
        except ValueError:
            raise NetpbmError(f"expected integer {what} at byte {start}, got {tok!r}") from None

    def dims(self):
        w = self.integer("width")
        h = self.integer("height")
        if w < 1 or h < 1:
            raise NetpbmError(f"non-positive dimensions {w}x{h} in header (byte {self.pos})")
        return h, w

    def raster_start(self) -> None:
        # binary formats: exactly one whitespace byte after the header
        if self.pos >= len(self.data) or self.data[self.pos] not in _WHITESPACE:
            raise NetpbmError(f"missing raster separator at byte {self.pos}")
        self.pos += 1

    def take(self, need: int) -> bytes:
        raster = self.data[self.pos:self.pos + need]
        if len(raster) < need:
            raise NetpbmError(f"truncated raster at byte {self.pos + len(raster)}: "
                              f"got {len(raster)} of {need} bytes")
        return raster


def _plain_bits(rd: _Reader, count: int) -> np.ndarray:
    """P1 raster: '0'/'1' characters, separators optional (netpbm.py:79-96)."""
    d = rd.data
    out = np.empty(count, np.uint8)
    k = 0
    while k < count:
        rd.skip()
        if rd.pos >= len(d):
            raise NetpbmError(f"truncated raster at byte {rd.pos}: got {k} of {count} pixels")
        c = d[rd.pos]
        if c not in (0x30, 0x31):
            raise NetpbmError(f"invalid raster character {chr(c)!r} at byte {rd.pos}")
        out[k] = c - 0x30
        k += 1
        rd.pos += 1
    return out


@dataclass
class PbmRaster:
    """A PBM image kept bit-packed as P4 rows: raster [h, (w + 7) // 8] uint8."""
    h: int
    w: int
    raster: np.ndarray
    magic: bytes = b"P4"

    def unpack(self) -> np.ndarray:
        return np.ascontiguousarray(np.unpackbits(self.raster, axis=1)[:, :self.w])


def read_pbm_raster(path) -> PbmRaster:
    """Parse a P1 or P4 file without unpacking P4 (P1 is packed after parsing)."""
    with open(path, "rb") as fh:
        data = fh.read()
    rd = _Reader(data)
    magic = rd.token("magic number")
    if magic not in (b"P1", b"P4"):
        raise NetpbmError(f"unsupported magic {magic!r} at byte 0; expected P1 or P4")
    h, w = rd.dims()
    row_bytes = (w + 7) // 8
    if magic == b"P1":
        bits = _plain_bits(rd, h * w).reshape(h, w)
        return PbmRaster(h, w, np.packbits(bits, axis=1), b"P1")
    rd.raster_start()
    raster = rd.take(row_bytes * h)
    return PbmRaster(h, w, np.frombuffer(raster, np.uint8).reshape(h, row_bytes).copy(), b"P4")


def read_pbm(path) -> np.ndarray:
    """P1 / P4 file -> {0,1} uint8 image, 1 = black = object (netpbm.py:68-110)."""
    return read_pbm_raster(path).unpack()


def _pbm_header(fmt: str, h: int, w: int) -> bytes:
    return f"{fmt}\n{w} {h}\n".encode("ascii")


def write_pbm_raster(r: PbmRaster, path, format: str = "P4") -> None:
    """Write a packed raster (P4 as is; P1 through unpacking)."""
    if format == "P4":
        raster = np.ascontiguousarray(r.raster, np.uint8).copy()
        if r.w % 8:   # padding bits written as zero
            raster[:, -1] &= np.uint8((0xFF << (8 - r.w % 8)) & 0xFF)
        with open(path, "wb") as fh:
            fh.write(_pbm_header("P4", r.h, r.w))
            fh.write(raster.tobytes())
        return
    write_pbm(r.unpack(), path, format=format)


def write_pbm(img, path, format: str = "P4") -> None:
    """Write a binary image as P1 (plain, lines <= 68 chars) or P4 (packed)
    (netpbm.py:113-129)."""
    pix = as_binary(img)
    h, w = pix.shape
    if format == "P1":
        with open(path, "wb") as fh:
            fh.write(_pbm_header("P1", h, w))
            for row in pix:
                text = " ".join("1" if v else "0" for v in row)
                for i in range(0, len(text), 68):
                    fh.write(text[i:i + 68].encode("ascii") + b"\n")
    elif format == "P4":
        with open(path, "wb") as fh:
            fh.write(_pbm_header("P4", h, w))
            fh.write(np.packbits(pix, axis=1).tobytes())
    else:
        raise ValueError(f"PBM format must be 'P1' or 'P4', got {format!r}")


def write_pgm(values, path, mode: str = "root", format: str = "P5") -> None:
    """Squared-distance map -> grayscale PGM (netpbm.py:132-170): mode "squared"
    keeps raw values (maxval = largest finite value, at most 65535), mode
    "root" writes round(sqrt(v)) clamped to 255; the no-seed sentinel
    h^2 + w^2 + 1 renders as maxval."""
    arr = np.ascontiguousarray(values, dtype=np.int64)
    if arr.ndim != 2:
        raise ValueError("distance map must be 2D")
    h, w = arr.shape
    sentinel = h * h + w * w + 1
    finite = arr[arr < sentinel]
    if mode == "squared":
        top = int(finite.max()) if finite.size else 1
        maxval = int(min(max(top, 1), 65535))
        out = np.minimum(arr, maxval)
    elif mode == "root":
        maxval = 255
        out = np.minimum(np.rint(np.sqrt(arr.astype(np.float64))).astype(np.int64), 255)
        out[arr >= sentinel] = 255
    else:
        raise ValueError(f"PGM mode must be 'squared' or 'root', got {mode!r}")
    header = f"{format}\n{w} {h}\n{maxval}\n".encode("ascii")
    if format == "P2":
        with open(path, "wb") as fh:
            fh.write(header)
            for row in out:
                fh.write((" ".join(str(int(v)) for v in row) + "\n").encode("ascii"))
    elif format == "P5":
        with open(path, "wb") as fh:
            fh.write(header)
            fh.write(out.astype(">u2" if maxval > 255 else np.uint8).tobytes())
    else:
        raise ValueError(f"PGM format must be 'P2' or 'P5', got {format!r}")


def read_pgm(path) -> np.ndarray:
    """P2 / P5 file -> int64 array (netpbm.py:173-200)."""
    with open(path, "rb") as fh:
        data = fh.read()
    rd = _Reader(data)
    magic = rd.token("magic number")
    if magic not in (b"P2", b"P5"):
        raise NetpbmError(f"unsupported magic {magic!r} at byte 0; expected P2 or P5")
    h, w = rd.dims()
    maxval = rd.integer("maxval")
    if not 0 < maxval < 65536:
        raise NetpbmError(f"maxval {maxval} out of range at byte {rd.pos}")
    if magic == b"P2":
        return np.array([rd.integer("pixel") for _ in range(h * w)], np.int64).reshape(h, w)
    rd.raster_start()
    dt = np.dtype(">u2") if maxval > 255 else np.dtype(np.uint8)
    raster = rd.take(h * w * dt.itemsize)
    return np.frombuffer(raster, dtype=dt).reshape(h, w).astype(np.int64)


def hasf_p4(rasters, w: int, r_max: int, adj: Adjacency = ADJ_84, keep=None, avoid=None):
    """HASF on a batch of P4 rasters, [n, h, (w + 7) // 8] uint8 (numpy or CUDA
    tensor), on the device without unpacking to bytes (ts_hasf_batch_p4).
    keep / avoid: P4 rasters of the same shape or None.  Returns the smoothed
    rasters (padding bits zero), numpy for numpy input."""
    import torch

    from . import _device as D
    from ._lib import check, load
    from .morph import _check_radius
    r_max = _check_radius(r_max)
    is_numpy = not isinstance(rasters, torch.Tensor)
    x = D.to_device_u8(rasters)
    if x.dim() == 2:
        x = x[None]
    n, h, rb = x.shape
    if rb != (w + 7) // 8:
        raise ValueError(f"raster rows hold {rb} bytes, width {w} needs {(w + 7) // 8}")
    k = None if keep is None else D.to_device_u8(keep).reshape(n, h, rb)
    a = None if avoid is None else D.to_device_u8(avoid).reshape(n, h, rb)
    out = torch.empty_like(x)
    check(load().ts_hasf_batch_p4(x.data_ptr(), out.data_ptr(), n, h, w, r_max, adj.fg, D.ptr(k), D.ptr(a),
                                  D.stream_ptr()))
    return out.cpu().numpy() if is_numpy else out
