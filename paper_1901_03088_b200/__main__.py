"""``python -m paper_1901_03088_b200`` → the slidenorm-compatible CLI."""
import sys

from .cli import main

sys.exit(main())
