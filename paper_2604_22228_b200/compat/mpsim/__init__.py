"""`mpsim` import shim: the reference package's module layout, served by the
B200 implementation (paper_2604_22228_b200).  Put `.../compat` first on
sys.path to run reference-style callers and tests against the drop-in.
Only the hot-path modules exist (topology, paths, pipeline, graph); the
simulator, bench, tuner, CLI and plots are out of scope."""

from paper_2604_22228_b200 import *  # noqa: F401,F403
from paper_2604_22228_b200 import __version__  # noqa: F401
