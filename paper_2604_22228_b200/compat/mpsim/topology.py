"""`mpsim.topology` served by paper_2604_22228_b200.topology."""
import sys as _sys

from paper_2604_22228_b200 import topology as _impl

_sys.modules[__name__] = _impl
