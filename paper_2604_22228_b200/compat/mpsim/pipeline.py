"""`mpsim.pipeline` served by paper_2604_22228_b200.pipeline."""
import sys as _sys

from paper_2604_22228_b200 import pipeline as _impl

_sys.modules[__name__] = _impl
