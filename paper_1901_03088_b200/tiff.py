"""8-bit RGB (Big)TIFF codec for whole-slide files, no third-party TIFF package.

The reference reads and writes TIFF through ``tifffile`` (src/image_io.py:
132-227 TiffSource, 361-454 TiffStripWriter), which this image does not ship.
This module implements the subset the reference supports — interleaved 8-bit
RGB, tiled or striped, uncompressed or deflate (compression 1, 8, 32946;
horizontal predictor 2 also decoded), classic or BigTIFF, first page — with
random access per segment, so a transform streaming 1024-row strips only
decodes the tiles it touches.  Segments decode / encode in a thread pool
(zlib releases the GIL) and go to the GPU as whole strips.
"""
from __future__ import annotations

import os
import struct
import threading
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .errors import CorruptImageError, UnsupportedFormatError

TILE = 256
_DEFLATE = (8, 32946)
# tag ids
_W, _H, _BPS, _COMP, _PHOTO, _SOFF, _SPP, _RPS, _SBC, _PLANAR, _PRED = (
    256, 257, 258, 259, 262, 273, 277, 278, 279, 284, 317)
_TW, _TL, _TOFF, _TBC, _SFMT = 322, 323, 324, 325, 339
# field type -> (struct code, size)
_TYPES = {1: ("B", 1), 2: ("c", 1), 3: ("H", 2), 4: ("I", 4), 5: ("II", 8), 6: ("b", 1),
          7: ("B", 1), 8: ("h", 2), 9: ("i", 4), 16: ("Q", 8), 17: ("q", 8), 18: ("Q", 8)}


def _pool():
    return ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1))


class TiffReader:
    """Region reader over the first page of a tiled or striped RGB8 TIFF."""

    def __init__(self, path):
        self.path = str(path)
        try:
            self._fh = open(self.path, "rb")
            self._parse()
        except (OSError, struct.error, KeyError, IndexError) as exc:
            raise CorruptImageError(f"{path}: cannot parse TIFF: {exc}") from exc
        self._lock = threading.Lock()
        self._exec = _pool()
        self._segment(0)               # validate the first segment eagerly

    # ------------------------------------------------------------------ header / IFD
    def _parse(self):
        fh = self._fh
        head = fh.read(16)
        order = {b"II": "<", b"MM": ">"}.get(head[:2])
        if order is None:
            raise CorruptImageError(f"{self.path}: not a TIFF file")
        magic = struct.unpack(order + "H", head[2:4])[0]
        if magic == 42:
            big, ifd = False, struct.unpack(order + "I", head[4:8])[0]
        elif magic == 43:
            big, ifd = True, struct.unpack(order + "Q", head[8:16])[0]
        else:
            raise CorruptImageError(f"{self.path}: bad TIFF magic {magic}")
        fh.seek(ifd)
        n = struct.unpack(order + ("Q" if big else "H"), fh.read(8 if big else 2))[0]
        esize = 20 if big else 12
        raw = fh.read(n * esize)
        tags = {}
        for k in range(n):
            e = raw[k * esize:(k + 1) * esize]
            tag, typ = struct.unpack(order + "HH", e[:4])
            count = struct.unpack(order + ("Q" if big else "I"), e[4:12] if big else e[4:8])[0]
            inline = e[12:20] if big else e[8:12]
            if typ not in _TYPES:
                continue
            code, size = _TYPES[typ]
            nbytes = size * count
            if nbytes <= len(inline):
                data = inline[:nbytes]
            else:
                off = struct.unpack(order + ("Q" if big else "I"), inline)[0]
                fh.seek(off)
                data = fh.read(nbytes)
            if typ == 2:
                tags[tag] = data
            else:
                fmt = order + (code * count if typ != 5 else "I" * 2 * count)
                tags[tag] = struct.unpack(fmt, data)
        self._tags = tags
        g = lambda t, d=None: tags[t][0] if t in tags else d   # noqa: E731
        self.width, self.height = int(g(_W)), int(g(_H))
        spp, bps = int(g(_SPP, 1)), tags.get(_BPS, (1,))
        if spp != 3 or any(b != 8 for b in bps) or int(g(_PLANAR, 1)) != 1 \
                or int(g(_SFMT, 1)) != 1:
            raise UnsupportedFormatError(f"{self.path}: only 8-bit interleaved RGB TIFF is "
                                         "supported")
        self.compression = int(g(_COMP, 1))
        if self.compression not in (1,) + _DEFLATE:
            raise UnsupportedFormatError(f"{self.path}: unsupported TIFF compression "
                                         f"{self.compression}")
        self.predictor = int(g(_PRED, 1))
        if self.predictor not in (1, 2):
            raise UnsupportedFormatError(f"{self.path}: unsupported TIFF predictor "
                                         f"{self.predictor}")
        if _TOFF in tags:
            self.seg_w, self.seg_h = int(g(_TW)), int(g(_TL))
            self.offsets, self.counts = tags[_TOFF], tags[_TBC]
        else:
            self.seg_w, self.seg_h = self.width, int(g(_RPS, self.height))
            self.offsets, self.counts = tags[_SOFF], tags[_SBC]
        self.cols = -(-self.width // self.seg_w)
        if len(self.offsets) < -(-self.height // self.seg_h) * self.cols:
            raise CorruptImageError(f"{self.path}: truncated TIFF: missing segments")

    # ------------------------------------------------------------------ segments
    def _segment(self, index):
        """Decoded segment `index` as (seg_h', seg_w', 3) (strips may be short)."""
        with self._lock:
            self._fh.seek(self.offsets[index])
            data = self._fh.read(self.counts[index])
        if len(data) != self.counts[index]:
            raise CorruptImageError(f"{self.path}: truncated segment {index}")
        tiled = _TOFF in self._tags
        r = index // self.cols
        rows = self.seg_h if tiled else min(self.seg_h, self.height - r * self.seg_h)
        try:
            if self.compression in _DEFLATE:
                data = zlib.decompress(data)
            seg = np.frombuffer(data, np.uint8)[:rows * self.seg_w * 3]
            seg = seg.reshape(rows, self.seg_w, 3)
        except (zlib.error, ValueError) as exc:
            raise CorruptImageError(f"{self.path}: cannot decode segment {index}: {exc}") \
                from exc
        if self.predictor == 2:                    # horizontal differencing, per channel
            seg = np.cumsum(seg, axis=1, dtype=np.uint8)
        return seg

    def read_region(self, x, y, w, h) -> np.ndarray:
        out = np.empty((h, w, 3), np.uint8)
        r0, r1 = y // self.seg_h, (y + h - 1) // self.seg_h
        c0, c1 = x // self.seg_w, (x + w - 1) // self.seg_w
        jobs = [(r, c) for r in range(r0, r1 + 1) for c in range(c0, c1 + 1)]
        segs = self._exec.map(lambda rc: self._segment(rc[0] * self.cols + rc[1]), jobs)
        for (r, c), seg in zip(jobs, segs):
            sy, sx = r * self.seg_h, c * self.seg_w
            ya, yb = max(y, sy), min(y + h, sy + self.seg_h)
            xa, xb = max(x, sx), min(x + w, sx + self.seg_w)
            out[ya - y:yb - y, xa - x:xb - x] = seg[ya - sy:yb - sy, xa - sx:xb - sx]
        return out

    def close(self):
        self._exec.shutdown(wait=True)
        self._fh.close()


class TiffTileWriter:
    """Tiled (256 x 256) RGB8 TIFF written band by band: full-width strips are
    re-chunked into 256-row bands whose tiles are deflated in a thread pool
    and appended; the IFD goes at the end.  BigTIFF is used when classic
    32-bit offsets could overflow (as the reference decides)."""

    def __init__(self, path, width, height, compression="deflate", level=6, bigtiff=None):
        self.path, self.width, self.height = str(path), width, height
        self.compress = compression == "deflate"
        self.level = level
        self.big = (width * height * 3 >= 2**32 - 2**25) if bigtiff is None else bigtiff
        self._fh = open(self.path, "wb")
        self._fh.write(b"II" + (struct.pack("<HHHQ", 43, 8, 0, 0) if self.big
                                 else struct.pack("<HI", 42, 0)))
        self._pending = np.empty((0, width, 3), np.uint8)
        self._offsets, self._counts = [], []
        self._exec = _pool()

    def _encode(self, tile):
        raw = np.ascontiguousarray(tile).tobytes()
        return zlib.compress(raw, self.level) if self.compress else raw

    def _band(self, band):
        rows = band.shape[0]
        tiles = []
        for x in range(0, self.width, TILE):
            t = np.zeros((TILE, TILE, 3), np.uint8)    # edge tiles padded to full size
            part = band[:, x:x + TILE]
            t[:rows, :part.shape[1]] = part
            tiles.append(t)
        for blob in self._exec.map(self._encode, tiles):
            self._offsets.append(self._fh.tell())
            self._counts.append(len(blob))
            self._fh.write(blob)

    def write(self, rows: np.ndarray):
        self._pending = np.concatenate([self._pending, rows]) if self._pending.size else rows
        while self._pending.shape[0] >= TILE:
            self._band(self._pending[:TILE])
            self._pending = self._pending[TILE:]

    def close(self):
        if self._pending.shape[0]:
            self._band(self._pending)
            self._pending = self._pending[:0]
        self._exec.shutdown(wait=True)
        fh, big = self._fh, self.big
        off_t, off_fmt = (16, "Q") if big else (4, "I")
        entries = [(_W, 4, [self.width]), (_H, 4, [self.height]), (_BPS, 3, [8, 8, 8]),
                   (_COMP, 3, [8 if self.compress else 1]), (_PHOTO, 3, [2]), (_SPP, 3, [3]),
                   (_PLANAR, 3, [1]), (_TW, 3, [TILE]), (_TL, 3, [TILE]),
                   (_TOFF, off_t, self._offsets), (_TBC, off_t, self._counts)]
        # out-of-line arrays first, then the IFD
        inline = 8 if big else 4
        blobs = {}
        for tag, typ, vals in entries:
            code, size = _TYPES[typ]
            data = struct.pack("<" + code * len(vals), *vals)
            if len(data) > inline:
                if fh.tell() % 2:
                    fh.write(b"\0")
                blobs[tag] = fh.tell()
                fh.write(data)
        if fh.tell() % 2:
            fh.write(b"\0")
        ifd = fh.tell()
        fh.write(struct.pack("<Q" if big else "<H", len(entries)))
        for tag, typ, vals in entries:
            code, size = _TYPES[typ]
            head = struct.pack("<HH" + ("Q" if big else "I"), tag, typ, len(vals))
            if tag in blobs:
                val = struct.pack("<" + off_fmt, blobs[tag])
            else:
                val = struct.pack("<" + code * len(vals), *vals).ljust(inline, b"\0")
            fh.write(head + val)
        fh.write(struct.pack("<" + off_fmt, 0))        # no next IFD
        fh.seek(8 if big else 4)
        fh.write(struct.pack("<" + off_fmt, ifd))
        fh.close()

    def abort(self):
        self._exec.shutdown(wait=False)
        self._fh.close()
        if os.path.exists(self.path):
            os.remove(self.path)
