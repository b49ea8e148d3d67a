"""Slide sources and strip sinks (boundary types of src/image_io.py).

Kept: ``PixelBlock`` (src/image_io.py:40-59), ``SlideSource`` protocol
(:62-92), ``ArraySource`` (:95-107), ``StripWriter`` protocol (:261-313),
``plan_strips`` (:248-258) — ``plan_strips`` and ``StripWriter`` follow the
reference closely on purpose: they are the protocol users subclass.  Added
for the device path: ``DeviceSource`` (a CUDA (H, W, 3) u8 tensor) and
``DeviceWriter`` / ``ArrayWriter`` sinks whose storage the transform can
write into directly.  Files: PNG in through Pillow and
out through the streaming ``PngStripWriter`` (:316-358), tiled/striped RGB8
(Big)TIFF through the package's own codec (tiff.py), ``.npy`` memory-mapped.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEFAULT_STRIP_HEIGHT = 1024   # src/image_io.py:36


@dataclass
class PixelBlock:
    """A rectangular tile of 8-bit RGB pixels and its position in the slide."""

    origin_x: int
    origin_y: int
    pixels: object  # (h, w, 3) uint8 numpy array or CUDA tensor

    def __post_init__(self):
        p = self.pixels
        ok = p.ndim == 3 and p.shape[2] == 3
        dt = getattr(p, "dtype", None)
        ok = ok and (dt == np.uint8 or str(dt) == "torch.uint8")
        if not ok:
            raise ValueError(f"pixels must be (h, w, 3) uint8, got {tuple(p.shape)} {dt}")

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]


class SlideSource:
    """Read-only random access to an RGB image of known size."""

    width: int
    height: int

    def read_region(self, x: int, y: int, w: int, h: int) -> PixelBlock:
        raise NotImplementedError

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def _check_bounds(self, x, y, w, h):
        if w < 1 or h < 1:
            raise ValueError(f"region size must be positive, got {w}x{h}")
        if x < 0 or y < 0 or x + w > self.width or y + h > self.height:
            raise ValueError(f"region ({x},{y},{w},{h}) outside image {self.width}x{self.height}")


class ArraySource(SlideSource):
    """In-memory host slide (src/image_io.py:95-107)."""

    def __init__(self, pixels):
        pixels = np.asarray(pixels)
        if pixels.ndim != 3 or pixels.shape[2] != 3 or pixels.dtype != np.uint8:
            raise ValueError("ArraySource expects (h, w, 3) uint8")
        self._pixels = pixels
        self.height, self.width = pixels.shape[:2]

    @property
    def array(self) -> np.ndarray:
        return self._pixels

    def read_region(self, x, y, w, h):
        self._check_bounds(x, y, w, h)
        return PixelBlock(x, y, self._pixels[y:y + h, x:x + w].copy())


class DeviceSource(SlideSource):
    """A slide resident in GPU memory: a contiguous CUDA (h, w, 3) uint8 tensor."""

    def __init__(self, tensor):
        if tensor.ndim != 3 or tensor.shape[2] != 3 or str(tensor.dtype) != "torch.uint8" \
                or not tensor.is_cuda:
            raise ValueError("DeviceSource expects a CUDA (h, w, 3) uint8 tensor")
        self._t = tensor.contiguous()
        self.height, self.width = int(tensor.shape[0]), int(tensor.shape[1])

    @property
    def tensor(self):
        return self._t

    def read_region(self, x, y, w, h):
        self._check_bounds(x, y, w, h)
        return PixelBlock(x, y, self._t[y:y + h, x:x + w])


def plan_strips(height: int, strip_height: int):
    """src/image_io.py:248-258."""
    if strip_height < 1:
        raise ValueError(f"strip_height must be >= 1, got {strip_height}")
    if height < 1:
        raise ValueError(f"height must be >= 1, got {height}")
    return [(y, min(strip_height, height - y)) for y in range(0, height, strip_height)]


class StripWriter:
    """Streamed writer fed in-order full-width strips (src/image_io.py:261-313)."""

    def __init__(self, width: int, height: int):
        self.width = width
        self.height = height
        self._rows_written = 0
        self._closed = False

    def _check_strip(self, block: PixelBlock):
        if self._closed:
            raise ValueError("writer is closed")
        if block.origin_x != 0 or block.width != self.width:
            raise ValueError(f"strip must span the full width {self.width}, "
                             f"got x={block.origin_x} width={block.width}")
        if block.origin_y != self._rows_written:
            raise ValueError(f"out-of-order strip: expected y={self._rows_written}, "
                             f"got y={block.origin_y}")
        if block.origin_y + block.height > self.height:
            raise ValueError("strip extends past the image height")

    def write_strip(self, block: PixelBlock):
        self._check_strip(block)
        self._write(block.pixels)
        self._rows_written += block.height

    def _write(self, rows):
        raise NotImplementedError

    def close(self):
        raise NotImplementedError

    def abort(self):
        self._closed = True

    def __enter__(self):
        return self

    def __exit__(self, exc_type, exc, tb):
        if exc_type is None:
            self.close()
        else:
            self.abort()
        return False


class ArrayWriter(StripWriter):
    """Host-memory sink.  ``transform`` D2H-copies straight into ``rows(y, h)``
    when the array is pinned; otherwise strips arrive via ``write_strip``."""

    def __init__(self, width, height, out=None):
        super().__init__(width, height)
        # every row is written before close() succeeds: no need to zero-fill
        self.pixels = out if out is not None else np.empty((height, width, 3), np.uint8)
        if self.pixels.shape != (height, width, 3) or self.pixels.dtype != np.uint8:
            raise ValueError("ArrayWriter storage must be (height, width, 3) uint8")

    def rows(self, y, h):
        return self.pixels[y:y + h]

    def mark_written(self, y, h):
        """Advance the in-order cursor for rows the transform copied in directly."""
        if y != self._rows_written:
            raise ValueError(f"out-of-order strip: expected y={self._rows_written}, got y={y}")
        self._rows_written += h

    def _write(self, rows):
        y = self._rows_written
        if hasattr(rows, "cpu"):
            rows = rows.cpu().numpy()
        self.pixels[y:y + rows.shape[0]] = rows

    def close(self):
        if self._rows_written != self.height:
            raise ValueError("incomplete image")
        self._closed = True


class DeviceWriter(StripWriter):
    """GPU-memory sink: an (height, width, 3) uint8 CUDA tensor the transform
    writes into directly (``rows(y, h)``)."""

    def __init__(self, width, height, out=None, device=None):
        super().__init__(width, height)
        import torch

        self.pixels = out if out is not None else torch.empty(
            (height, width, 3), dtype=torch.uint8, device=device or "cuda")
        if tuple(self.pixels.shape) != (height, width, 3) or not self.pixels.is_cuda:
            raise ValueError("DeviceWriter storage must be a CUDA (height, width, 3) uint8 tensor")

    def rows(self, y, h):
        return self.pixels[y:y + h]

    def mark_written(self, y, h):
        """Advance the in-order cursor for rows the transform wrote in place."""
        if y != self._rows_written:
            raise ValueError(f"out-of-order strip: expected y={self._rows_written}, got y={y}")
        self._rows_written += h

    def _write(self, rows):
        y = self._rows_written
        if not hasattr(rows, "is_cuda"):
            import torch

            rows = torch.from_numpy(np.ascontiguousarray(rows))
        self.pixels[y:y + rows.shape[0]].copy_(rows, non_blocking=True)

    def close(self):
        if self._rows_written != self.height:
            raise ValueError("incomplete image")
        self._closed = True


# ----------------------------------------------------------------------------- files
# Image files for the CLI (src/image_io.py:110-466).  PNG goes through Pillow
# (decoded once, as the reference does: PNG has no random access); `.npy`
# (H, W, 3) uint8 arrays are memory-mapped; tiled/striped RGB8 (Big)TIFF goes
# through the package's own codec (tiff.py: per-segment random access in, tiled
# deflate out), so whole-slide files stream without a full load.
_PNG_MAGIC = b"\x89PNG\r\n\x1a\n"
_NPY_MAGIC = b"\x93NUMPY"
_TIFF_MAGIC = (b"II*\x00", b"MM\x00*", b"II+\x00", b"MM\x00+")


def _decode_png(path) -> np.ndarray:
    from PIL import Image, UnidentifiedImageError

    from .errors import CorruptImageError, UnsupportedFormatError

    try:
        with Image.open(path) as img:
            if img.mode != "RGB":
                raise UnsupportedFormatError(f"{path}: only 8-bit RGB PNG is supported "
                                             f"(mode {img.mode})")
            return np.asarray(img, dtype=np.uint8)
    except UnidentifiedImageError as exc:
        raise CorruptImageError(f"{path}: cannot decode PNG: {exc}") from exc
    except (OSError, SyntaxError, ValueError) as exc:
        raise CorruptImageError(f"{path}: truncated or corrupt PNG: {exc}") from exc


def open_slide(path) -> SlideSource:
    """Image file → SlideSource, dispatching on the magic bytes."""
    from .errors import CorruptImageError, UnsupportedFormatError

    with open(path, "rb") as fh:
        head = fh.read(8)
    if head == _PNG_MAGIC:
        return ArraySource(_decode_png(path))
    if head[:6] == _NPY_MAGIC:
        try:
            arr = np.load(path, mmap_mode="r")
        except ValueError as exc:
            raise CorruptImageError(f"{path}: corrupt .npy: {exc}") from exc
        if arr.ndim != 3 or arr.shape[2] != 3 or arr.dtype != np.uint8:
            raise UnsupportedFormatError(f"{path}: .npy must hold (H, W, 3) uint8")
        return ArraySource(arr)
    if head[:4] in _TIFF_MAGIC:
        return TiffSource(path)
    raise UnsupportedFormatError(f"{path}: not a supported image format (PNG, .npy, "
                                 "8-bit RGB TIFF)")


class TiffSource(SlideSource):
    """Tiled or striped RGB8 (Big)TIFF (src/image_io.py:132-227)."""

    def __init__(self, path):
        from .tiff import TiffReader

        self._reader = TiffReader(path)
        self.width, self.height = self._reader.width, self._reader.height

    def read_region(self, x, y, w, h):
        self._check_bounds(x, y, w, h)
        return PixelBlock(x, y, self._reader.read_region(x, y, w, h))

    def close(self):
        self._reader.close()


class TiffStripWriter(StripWriter):
    """Tiled deflate TIFF output, written band by band (src/image_io.py:361-454)."""

    def __init__(self, path, width, height, compression="deflate"):
        from .tiff import TiffTileWriter

        super().__init__(width, height)
        self._tw = TiffTileWriter(path, width, height, compression=compression)

    def _write(self, rows):
        if hasattr(rows, "cpu"):
            rows = rows.cpu().numpy()
        self._tw.write(np.asarray(rows))

    def close(self):
        if self._closed:
            return
        if self._rows_written != self.height:
            self.abort()
            raise ValueError(f"incomplete image: {self._rows_written} of {self.height} rows")
        self._tw.close()
        self._closed = True

    def abort(self):
        if not self._closed:
            self._closed = True
            self._tw.abort()


class PngStripWriter(StripWriter):
    """Streaming 8-bit RGB PNG encoder (src/image_io.py:316-358): the file is
    opened (and an unwritable path reported) on construction, every strip's
    scanlines — filter byte 0 in front of each — go straight through one
    zlib stream into IDAT chunks, so memory stays bounded by one strip.  A
    failed or incomplete image leaves no file."""

    _SIG = b"\x89PNG\r\n\x1a\n"

    def __init__(self, path, width, height, compress_level: int = 6):
        import struct
        import zlib

        super().__init__(width, height)
        self.path = str(path)
        self._fh = open(self.path, "wb")
        self._fh.write(self._SIG)
        self._chunk(b"IHDR", struct.pack(">IIBBBBB", width, height, 8, 2, 0, 0, 0))
        self._z = zlib.compressobj(compress_level)

    def _chunk(self, kind: bytes, data: bytes):
        import struct
        import zlib

        self._fh.write(struct.pack(">I", len(data)) + kind)
        self._fh.write(data)
        self._fh.write(struct.pack(">I", zlib.crc32(data, zlib.crc32(kind)) & 0xFFFFFFFF))

    def _write(self, rows):
        if hasattr(rows, "cpu"):
            rows = rows.cpu().numpy()
        rows = np.asarray(rows)
        h = rows.shape[0]
        lines = np.empty((h, 1 + 3 * self.width), dtype=np.uint8)
        lines[:, 0] = 0
        lines[:, 1:] = rows.reshape(h, 3 * self.width)
        payload = self._z.compress(lines)
        if payload:
            self._chunk(b"IDAT", payload)

    def close(self):
        if self._closed:
            return
        if self._rows_written != self.height:
            self.abort()
            raise ValueError(f"incomplete image: {self._rows_written} of {self.height} rows")
        self._chunk(b"IDAT", self._z.flush())
        self._chunk(b"IEND", b"")
        self._fh.close()
        self._closed = True

    def abort(self):
        import os

        if not self._closed:
            self._closed = True
            self._fh.close()
            if os.path.exists(self.path):
                os.remove(self.path)


class FileWriter(ArrayWriter):
    """`.npy` output fed in-order strips through a memory map.  A failed or
    incomplete image leaves no file."""

    def __init__(self, path, width, height):
        from .errors import UnsupportedFormatError

        self.path = str(path)
        if not self.path.lower().endswith(".npy"):
            raise UnsupportedFormatError(f"{path}: output must be .png, .npy or .tif(f)")
        self.kind = "npy"
        out = np.lib.format.open_memmap(self.path, mode="w+", dtype=np.uint8,
                                        shape=(height, width, 3))
        super().__init__(width, height, out=out)

    def close(self):
        if self._closed:
            return
        try:
            super().close()
        except ValueError:
            self.abort()
            raise
        self.pixels.flush()

    def abort(self):
        import os

        self._closed = True
        del self.pixels
        if os.path.exists(self.path):
            os.remove(self.path)


def open_writer(path, width: int, height: int) -> StripWriter:
    """src/image_io.py:457-466: a StripWriter for an output file."""
    low = str(path).lower()
    if low.endswith((".tif", ".tiff")):
        return TiffStripWriter(path, width, height)
    if low.endswith(".png"):
        return PngStripWriter(path, width, height)
    return FileWriter(path, width, height)
