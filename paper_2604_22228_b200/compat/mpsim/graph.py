"""`mpsim.graph` served by paper_2604_22228_b200.graph."""
import sys as _sys

from paper_2604_22228_b200 import graph as _impl

_sys.modules[__name__] = _impl
