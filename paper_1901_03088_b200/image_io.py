"""Slide sources and strip sinks (boundary types of src/image_io.py).

Kept: ``PixelBlock`` (src/image_io.py:40-59), ``SlideSource`` protocol
(:62-92), ``ArraySource`` (:95-107), ``StripWriter`` protocol (:261-313),
``plan_strips`` (:248-258).  Added for the device path: ``DeviceSource``
(a CUDA (H, W, 3) u8 tensor) and ``DeviceWriter`` / ``ArrayWriter`` sinks
whose storage the transform can write into directly.  PNG/TIFF codecs are
out of scope for this round.
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
        self.pixels = out if out is not None else np.zeros((height, width, 3), np.uint8)
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
