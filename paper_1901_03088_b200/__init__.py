"""B200-native SPCN hot path — drop-in for the reference package ``slidenorm``.

Public API mirrors ``slidenorm.__all__`` (src/__init__.py:49-86); per-pixel
work runs in libspcn.so (hand-written sm_100a CUDA, C ABI in include/spcn.h).
"""
from .errors import (  # noqa: F401
    BlankSlideError, CorruptImageError, DegenerateStainError, InsufficientPixelsError,
    ProfileError, SlideNormError, StainAbsentError, UnsupportedFormatError,
)
from .image_io import (  # noqa: F401
    ArraySource, ArrayWriter, DeviceSource, DeviceWriter, PixelBlock, SlideSource,
    StripWriter, plan_strips,
)
from .normalize import (  # noqa: F401
    FitParams, StainStats, load_profile, normalize_block, save_profile, scale_factors,
    stain_stats,
)
from .optics import beer_lambert, estimate_max_intensity, inverse_beer_lambert  # noqa: F401
from .stain_sep import (  # noqa: F401
    SnmfConfig, SnmfFit, code_densities, fit_basis, order_stains, reference_basis,
)
from .order_stats import median, percentile  # noqa: F401
from .pipeline import (  # noqa: F401
    BufferGauge, PixelSample, RunStats, SamplePlan, fit, normalize, sample_pixels, transform,
)
from .xform import XformPlan, process_strip  # noqa: F401
from .batch import (  # noqa: F401
    BatchFit, fit_batch, normalize_batch, normalize_batch_host, transform_batch,
)

__version__ = "0.1.0"
