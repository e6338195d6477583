"""B200-native multi-path intra-node GPU-to-GPU transfer (arXiv 2604.22228).

Drop-in for the path-plan / split-ratio / pipeline / graph-cache API of the
reference package `mpsim` (/root/reference/pkg/src/mpsim/__init__.py:4-15),
with the simulator's execution entry points replaced by real transfers:
`send` / `recv` / `Engine` (engine.py) over hand-written sm_100a copy kernels
and copy engines (csrc/).  The planner runs in C++ behind the C ABI declared
in include/mpb200.h.
"""

from . import _lib as _l

__version__ = "0.1.0"

if _l.lib is not None:  # None only while `python -m paper_2604_22228_b200.build` runs
    from .topology import (Channel, DeviceId, LinkSpec, Topology, TopologyError,  # noqa: F401
                           load_topology, load_topology_file, mesh_text, preset, resolve)
    from .paths import (ContentionPlan, Hop, Path, PathConfig, PathSet, PlanError,  # noqa: F401
                        plan_contention_free, plan_paths)
    from .pipeline import (ChunkAssignment, ChunkError, ChunkPlan, Lane,  # noqa: F401
                           LaneSchedule, lane_schedule, make_chunk_plan)
    from .graph import (CopyNode, ExecGraph, GraphCache, GraphKey, OverheadModel,  # noqa: F401
                        build_graph, cache_get_or_build, graph_key, lifecycle_cost)
    from .engine import Engine, SendStats, default_engine, recv, send  # noqa: F401
    from ._lib import EngineError, LIB_PATH  # noqa: F401
