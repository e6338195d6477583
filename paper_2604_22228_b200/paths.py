"""Multi-path selection and split ratios: direct, GPU-staged and host-staged routes.

Drop-in for `mpsim.paths` (/root/reference/pkg/src/mpsim/paths.py).  The
planning arithmetic — candidate staging devices, bottleneck bandwidths and
the split ratios `w / sum(w)` with CPython's compensated `sum()` — runs in
the C++ planner (`mp_plan_paths`, `mp_plan_contention_free`); this module
converts between the reference's frozen dataclasses and the ABI structs.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field, replace

from . import _lib
from ._lib import (MP_ERR_PLAN, MP_NO_STAGE, MP_PATH_DIRECT, MP_PATH_GPU,
                   MP_PATH_HOST, MP_SHARE_BANDWIDTH, MP_SHARE_EQUAL, check, lib)
from .topology import Channel, DeviceId, Topology, device_from_abi

DIRECT = "direct"
GPU_STAGED = "gpu"
HOST_STAGED = "host"

EQUAL = "equal"
BANDWIDTH_PROPORTIONAL = "bandwidth_proportional"

# Environment knobs (paths.py:24-30); each has a CLI flag equivalent and the flag wins.
ENV_GPU_PATHS = "MP_NUM_GPU_PATHS"
ENV_HOST_PATH = "MP_ENABLE_HOST_PATH"
ENV_MAX_CHUNKS = "MP_MAX_CHUNKS"
ENV_GRAPH = "MP_ENABLE_GRAPH"
ENV_CACHE_SIZE = "MP_GRAPH_CACHE_SIZE"
ENV_SHARE_POLICY = "MP_SHARE_POLICY"

_KIND_CODE = {DIRECT: MP_PATH_DIRECT, GPU_STAGED: MP_PATH_GPU, HOST_STAGED: MP_PATH_HOST}
_KIND_NAME = {v: k for k, v in _KIND_CODE.items()}
_POLICY_CODE = {BANDWIDTH_PROPORTIONAL: MP_SHARE_BANDWIDTH, EQUAL: MP_SHARE_EQUAL}


class PlanError(ValueError):
    """No valid path assignment exists for a request (paths.py:33)."""


_lib.register_error(MP_ERR_PLAN, PlanError)


@dataclass(frozen=True)
class Hop:
    """One copy step of a path: a direction channel plus its endpoints."""

    channel: Channel
    src: DeviceId
    dst: DeviceId


@dataclass(frozen=True)
class Path:
    kind: str  # DIRECT, GPU_STAGED, or HOST_STAGED
    hops: tuple[Hop, ...]
    share: float
    stage: DeviceId | None = None

    def __post_init__(self):
        expected = 1 if self.kind == DIRECT else 2
        if len(self.hops) != expected:
            raise PlanError(f"{self.kind} path must have {expected} hops, got {len(self.hops)}")
        if expected == 2 and self.hops[0].dst != self.hops[1].src:
            raise PlanError("staged path hops are not connected")
        if not 0.0 <= self.share <= 1.0:
            raise PlanError(f"path share must lie in [0,1], got {self.share}")

    @property
    def bottleneck_bandwidth(self) -> float:
        return min(h.channel.bandwidth for h in self.hops)


@dataclass(frozen=True)
class PathConfig:
    """Per-run transfer configuration, settable via env vars or flags (paths.py:67-104)."""

    num_gpu_paths: int = 1  # path 0 is always Direct
    host_path_enabled: bool = False
    max_chunks: int = 1
    graph_mode: bool = False
    cache_capacity: int = 16
    share_policy: str = BANDWIDTH_PROPORTIONAL

    def __post_init__(self):
        check(lib.mp_config_validate(C.byref(self.abi())))  # paths.py:78-86, same order
        if self.share_policy not in _POLICY_CODE:
            raise PlanError(f"unknown share policy {self.share_policy!r}")

    def abi_addr(self) -> int:
        """Address of this config's ABI struct, built once per instance (the
        config is frozen) so a cached-graph send pays no struct conversion."""
        cached = self.__dict__.get("_abi_cached")
        if cached is None:
            struct = self.abi()
            cached = (struct, C.addressof(struct))
            object.__setattr__(self, "_abi_cached", cached)
        return cached[1]

    def __getstate__(self):  # the cached ctypes struct is not picklable
        state = dict(self.__dict__)
        state.pop("_abi_cached", None)
        return state

    def abi(self) -> _lib.mp_config:
        big = 2**31 - 1
        clamp = lambda v: max(-big, min(big, int(v)))  # noqa: E731
        return _lib.mp_config(clamp(self.num_gpu_paths), 1 if self.host_path_enabled else 0,
                              clamp(self.max_chunks), 1 if self.graph_mode else 0,
                              clamp(self.cache_capacity),
                              _POLICY_CODE.get(self.share_policy, MP_SHARE_BANDWIDTH))

    @classmethod
    def from_env(cls, env=None) -> "PathConfig":
        env = os.environ if env is None else env
        cfg = cls()
        if ENV_GPU_PATHS in env:
            cfg = replace(cfg, num_gpu_paths=int(env[ENV_GPU_PATHS]))
        if ENV_HOST_PATH in env:
            cfg = replace(cfg, host_path_enabled=_parse_flag(env[ENV_HOST_PATH]))
        if ENV_MAX_CHUNKS in env:
            cfg = replace(cfg, max_chunks=int(env[ENV_MAX_CHUNKS]))
        if ENV_GRAPH in env:
            cfg = replace(cfg, graph_mode=_parse_flag(env[ENV_GRAPH]))
        if ENV_CACHE_SIZE in env:
            cfg = replace(cfg, cache_capacity=int(env[ENV_CACHE_SIZE]))
        if ENV_SHARE_POLICY in env:
            cfg = replace(cfg, share_policy=env[ENV_SHARE_POLICY])
        return cfg


def _parse_flag(text: str) -> bool:
    lowered = text.strip().lower()
    if lowered in ("1", "on", "true", "yes"):
        return True
    if lowered in ("0", "off", "false", "no"):
        return False
    raise PlanError(f"cannot parse flag value {text!r}")


@dataclass(frozen=True)
class PathSet:
    """The ordered paths chosen for one src -> dst transfer (paths.py:116-141)."""

    src: DeviceId
    dst: DeviceId
    paths: tuple[Path, ...]

    def __post_init__(self):
        arr, _ = paths_to_abi(self.paths)
        check(lib.mp_pathset_validate(arr, len(self.paths)))

    def channels(self) -> list[Channel]:
        """Distinct channels touched by any hop, in path order."""
        out: list[Channel] = []
        for path in self.paths:
            for hop in path.hops:
                if hop.channel not in out:
                    out.append(hop.channel)
        return out


def paths_to_abi(paths, channel_index=None):
    """Pack Path objects into mp_path structs.

    Hop channels are numbered by `channel_index(ch)` when given (a topology's
    own numbering), else by first appearance; the second return value lists
    the channels in that local numbering.
    """
    local: list[Channel] = []
    arr = (_lib.mp_path * max(1, len(paths)))()
    for i, p in enumerate(paths):
        a = arr[i]
        a.kind = _KIND_CODE.get(p.kind, MP_PATH_GPU)
        a.stage = MP_NO_STAGE if p.stage is None else p.stage.abi
        a.share = p.share
        a.nhops = len(p.hops)
        for h, hop in enumerate(p.hops[:2]):
            if channel_index is not None:
                idx = channel_index(hop.channel)
            else:
                for idx, ch in enumerate(local):
                    if ch is hop.channel:
                        break
                else:
                    local.append(hop.channel)
                    idx = len(local) - 1
            a.hops[h].channel = idx
            a.hops[h].src = hop.src.abi
            a.hops[h].dst = hop.dst.abi
    return arr, local


def _paths_from_abi(topology: Topology, arr, n: int) -> tuple[Path, ...]:
    out = []
    for i in range(n):
        a = arr[i]
        hops = tuple(Hop(topology.channel_at(a.hops[h].channel), device_from_abi(a.hops[h].src),
                         device_from_abi(a.hops[h].dst)) for h in range(a.nhops))
        stage = None if a.stage == MP_NO_STAGE else device_from_abi(a.stage)
        out.append(Path(_KIND_NAME[a.kind], hops, a.share, stage))
    return tuple(out)


def plan_paths(topology: Topology, src: DeviceId, dst: DeviceId,
               config: PathConfig) -> PathSet:
    """Select the path set for one transfer (paths.py:170-187).

    Path 0 is Direct; paths 1..num_gpu_paths-1 stage through the lowest-index
    non-endpoint accelerators; an optional host-staged path comes last.
    Shares are bandwidth-proportional (or equal) split ratios.
    """
    cap = config.num_gpu_paths + 1 if 0 < config.num_gpu_paths < 4096 else 1
    arr = (_lib.mp_path * cap)()
    n = C.c_int32()
    cfg = config.abi()
    check(lib.mp_plan_paths(topology._handle, src.abi, dst.abi, C.byref(cfg), arr, cap,
                            C.byref(n)))
    return PathSet(src, dst, _paths_from_abi(topology, arr, n.value))


@dataclass
class ContentionPlan:
    """Result of joint planning across concurrent transfers (paths.py:190-199)."""

    path_sets: list[PathSet]
    shared_channel_count: int
    contention_free: bool = field(init=False)

    def __post_init__(self):
        self.contention_free = self.shared_channel_count == 0


def plan_contention_free(topology: Topology, transfers: list[tuple[DeviceId, DeviceId]],
                         config: PathConfig) -> ContentionPlan:
    """Choose staging devices jointly so concurrent transfers avoid sharing
    channels (paths.py:210-242): exhaustive, deterministic, first minimum."""
    n = len(transfers)
    srcs = (C.c_int32 * max(1, n))(*[s.abi for s, _ in transfers])
    dsts = (C.c_int32 * max(1, n))(*[d.abi for _, d in transfers])
    per = config.num_gpu_paths + 1 if 0 < config.num_gpu_paths < 4096 else 1
    cap = max(1, n * per)
    arr = (_lib.mp_path * cap)()
    pps, shared = C.c_int32(), C.c_int32()
    cfg = config.abi()
    check(lib.mp_plan_contention_free(topology._handle, srcs, dsts, n, C.byref(cfg), arr, cap,
                                      C.byref(pps), C.byref(shared)))
    sets = []
    k = pps.value
    for t, (s, d) in enumerate(transfers):
        sub = (_lib.mp_path * max(1, k)).from_buffer(arr, t * k * C.sizeof(_lib.mp_path))
        sets.append(PathSet(s, d, _paths_from_abi(topology, sub, k)))
    return ContentionPlan(sets, shared.value)
