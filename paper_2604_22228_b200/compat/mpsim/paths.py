"""`mpsim.paths` served by paper_2604_22228_b200.paths."""
import sys as _sys

from paper_2604_22228_b200 import paths as _impl

_sys.modules[__name__] = _impl
