"""Import the reference package from /root/reference (THIS container only).

``tifffile`` is absent from the image and is only needed by the reference's
TIFF codec (``src/image_io.py:25``), which is outside the hot path; a stub
module satisfies the import.  Used by ``oracle/make_golden.py`` and by the
reference-pinning tests, which skip when /root/reference is not present (the
GPU box never has it).
"""
from __future__ import annotations

import os
import sys
import types

REF_SRC = "/root/reference/pkg/src"


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "slidenorm"))


def load():
    if not available():
        raise ImportError("reference not present at " + REF_SRC)
    try:
        import tifffile  # noqa: F401
    except ImportError:
        stub = types.ModuleType("tifffile")

        class _Missing:  # pragma: no cover - never exercised on the hot path
            def __init__(self, *a, **k):
                raise RuntimeError("tifffile is not installed")

        stub.TiffFile = _Missing
        stub.TiffWriter = _Missing
        sys.modules["tifffile"] = stub
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import slidenorm  # noqa: E402

    return slidenorm
