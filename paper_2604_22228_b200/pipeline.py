"""2-D decomposition of a message: paths horizontally, chunks vertically.

Drop-in for `mpsim.pipeline` (/root/reference/pkg/src/mpsim/pipeline.py).
`make_chunk_plan` and `lane_schedule` run in the C++ planner
(`mp_make_chunk_plan`, `mp_lane_schedule`); the chunk plan they produce is
bit-identical to the reference's and is the exact table the CUDA engine
executes (mp_engine.cu lowers it to device tiles and copy-engine lanes).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from ._lib import MP_ERR_CAPACITY, MP_ERR_CHUNK, check, lib
from .paths import PathSet, paths_to_abi


class ChunkError(ValueError):
    pass


_lib.register_error(MP_ERR_CHUNK, ChunkError)


@dataclass(frozen=True)
class ChunkAssignment:
    path_index: int
    offset: int  # same offset in source and destination buffers
    length: int
    seq: int  # dense per-path sequence number, from 0

    def __post_init__(self):
        if self.length < 1:
            raise ChunkError(f"chunk length must be >= 1, got {self.length}")
        if self.offset < 0:
            raise ChunkError(f"chunk offset must be >= 0, got {self.offset}")


@dataclass(frozen=True)
class ChunkPlan:
    total_size: int
    chunks: tuple[ChunkAssignment, ...]  # in round-robin emission order
    path_set: PathSet

    def chunks_for_path(self, path_index: int) -> list[ChunkAssignment]:
        return [c for c in self.chunks if c.path_index == path_index]

    def chunk_counts(self) -> list[int]:
        counts = [0] * len(self.path_set.paths)
        for c in self.chunks:
            counts[c.path_index] += 1
        return counts


def chunks_to_abi(chunks) -> "C.Array":
    arr = (_lib.mp_chunk * max(1, len(chunks)))()
    for i, c in enumerate(chunks):
        arr[i].offset = c.offset
        arr[i].length = c.length
        arr[i].path_index = c.path_index
        arr[i].seq = c.seq
    return arr


def plan_to_abi(plan: ChunkPlan):
    paths, local = paths_to_abi(plan.path_set.paths)
    return paths, local, chunks_to_abi(plan.chunks)


def make_chunk_plan(path_set: PathSet, size: int, max_chunks: int) -> ChunkPlan:
    """Split `size` bytes over the path set (pipeline.py:51-78).

    Per path the nominal chunk length is ceil(size * share / max_chunks);
    chunks are dealt round-robin over the paths with a positive share until
    the message is covered, the final chunk truncated to fit.
    """
    paths, _ = paths_to_abi(path_set.paths)
    n = C.c_int32()
    wire_size = int(size) & (2**64 - 1)  # the C side reads it as int64: negatives survive
    mc = max(-(2**31), min(2**31 - 1, int(max_chunks)))
    cap = max(1, min(4096, len(path_set.paths) * (mc + 2)))
    arr = (_lib.mp_chunk * cap)()
    rc = lib.mp_make_chunk_plan(paths, len(path_set.paths), wire_size, mc, arr, cap, C.byref(n))
    if rc == MP_ERR_CAPACITY:
        cap = n.value
        arr = (_lib.mp_chunk * cap)()
        rc = lib.mp_make_chunk_plan(paths, len(path_set.paths), wire_size, mc, arr, cap,
                                    C.byref(n))
    check(rc)
    chunks = tuple(ChunkAssignment(arr[i].path_index, arr[i].offset, arr[i].length, arr[i].seq)
                   for i in range(n.value))
    return ChunkPlan(size, chunks, path_set)


@dataclass(frozen=True)
class Lane:
    """A FIFO execution queue — a CUDA stream; one per path hop."""

    lane_id: int
    path_index: int
    hop: int  # 0 = direct or source->stage, 1 = stage->destination
    chunk_ids: tuple[int, ...]  # indices into plan.chunks, in seq order


@dataclass(frozen=True)
class LaneSchedule:
    lanes: tuple[Lane, ...]
    # ((lane, position), (lane, position)): hop-2 entry waits on hop-1 entry
    dependencies: tuple[tuple[tuple[int, int], tuple[int, int]], ...]

    @property
    def lane_count(self) -> int:
        return len(self.lanes)


def lane_schedule(plan: ChunkPlan) -> LaneSchedule:
    """One lane per direct path, two per staged path (pipeline.py:102-125)."""
    paths, _, chunks = plan_to_abi(plan)
    n_paths, n_chunks = len(plan.path_set.paths), len(plan.chunks)
    n_lanes, n_members, n_deps = C.c_int32(), C.c_int32(), C.c_int32()
    lcap = max(1, 2 * n_paths)
    mcap = max(1, 2 * n_chunks)
    lanes = (_lib.mp_lane * lcap)()
    members = (C.c_int32 * mcap)()
    deps = (_lib.mp_lane_dep * max(1, n_chunks))()
    check(lib.mp_lane_schedule(paths, n_paths, chunks, n_chunks, lanes, lcap, C.byref(n_lanes),
                               members, mcap, C.byref(n_members), deps, max(1, n_chunks),
                               C.byref(n_deps)))
    out = tuple(Lane(l.lane_id, l.path_index, l.hop,
                     tuple(members[l.first:l.first + l.count]))
                for l in lanes[:n_lanes.value])
    dd = tuple(((d.lane1, d.pos1), (d.lane2, d.pos2)) for d in deps[:n_deps.value])
    return LaneSchedule(out, dd)
