"""``python -m paper_2009_14514_b200 run|compare ...`` (the reference's
``rts-sph-bench`` console script)."""
import sys

from .cli import main

sys.exit(main())
