"""Node model: accelerators, links and their direction channels.

Drop-in for `mpsim.topology` (/root/reference/pkg/src/mpsim/topology.py).
Parsing and channel construction run in the C++ planner
(csrc/mp_core.cpp, `mp_topology_load` / `mp_topology_create`); this module
holds the Python value types the reference API hands out.  Channel objects
are created once per Topology and reused by every plan, so equality of
Hop/Path/PathSet keeps the reference's identity semantics
(`Channel` is `eq=False`, topology.py:57).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

from . import _lib
from ._lib import MP_DUPLEX_FULL, MP_DUPLEX_HALF, MP_ERR_TOPOLOGY, MP_HOST, check, lib

ACCELERATOR = "accelerator"
HOST = "host"

FULL = "full"
HALF = "half"


class TopologyError(ValueError):
    """Schema or invariant violation in a topology config (topology.py:25)."""


_lib.register_error(MP_ERR_TOPOLOGY, TopologyError)


@dataclass(frozen=True, order=True)
class DeviceId:
    """An accelerator or the single host (topology.py:29-51)."""

    index: int
    kind: str = ACCELERATOR

    def __post_init__(self):
        if self.index < 0:
            raise TopologyError(f"device index must be non-negative, got {self.index}")
        if self.kind not in (ACCELERATOR, HOST):
            raise TopologyError(f"unknown device kind {self.kind!r}")

    @property
    def is_host(self) -> bool:
        return self.kind == HOST

    @property
    def label(self) -> str:
        return "host" if self.is_host else str(self.index)

    def __str__(self):
        return self.label

    @property
    def abi(self) -> int:
        """Index in the C ABI: accelerator index, or MP_HOST."""
        return MP_HOST if self.is_host else self.index


HOST_DEVICE = DeviceId(0, HOST)


def device_from_abi(index: int) -> DeviceId:
    return HOST_DEVICE if index == MP_HOST else DeviceId(index)


@dataclass(eq=False)
class Channel:
    """One direction channel of a link; the unit of exclusive occupancy."""

    id: str
    bandwidth: float  # bytes/second
    latency: float  # seconds per copy

    def __repr__(self):
        return f"Channel({self.id})"


def _abi_link(a: DeviceId, b: DeviceId, bandwidth, latency, duplex, sublinks) -> _lib.mp_link:
    code = {FULL: MP_DUPLEX_FULL, HALF: MP_DUPLEX_HALF}.get(duplex, -1)
    return _lib.mp_link(a.abi, b.abi, float(bandwidth), float(latency), code, int(sublinks))


@dataclass(frozen=True)
class LinkSpec:
    """A physical link, bandwidth already aggregated over sublinks (topology.py:69-90)."""

    a: DeviceId
    b: DeviceId
    bandwidth: float
    latency: float
    duplex: str
    sublinks: int = 1

    def __post_init__(self):
        check(lib.mp_link_validate(C.byref(self._abi())))

    def _abi(self) -> _lib.mp_link:
        if self.a == self.b:  # host==host cannot be expressed by index alone
            link = _abi_link(self.a, self.b, self.bandwidth, self.latency, self.duplex,
                             self.sublinks)
            link.b = link.a
            return link
        return _abi_link(self.a, self.b, self.bandwidth, self.latency, self.duplex,
                         self.sublinks)


class Topology:
    """An immutable set of devices, links and direction channels (topology.py:93-154)."""

    def __init__(self, name: str, accelerators: int, links: list[LinkSpec]):
        links = list(links)
        arr = (_lib.mp_link * max(1, len(links)))(*[l._abi() for l in links])
        handle = C.c_void_p()
        check(lib.mp_topology_create(name.encode(), accelerators, arr, len(links),
                                     C.byref(handle)))
        self._init_from_handle(handle, links)

    @classmethod
    def _from_handle(cls, handle: C.c_void_p) -> "Topology":
        self = cls.__new__(cls)
        self._init_from_handle(handle, None)
        return self

    def _init_from_handle(self, handle, links):
        self._handle = handle
        n_acc, n_links, n_ch = C.c_int32(), C.c_int32(), C.c_int32()
        check(lib.mp_topology_info(handle, C.byref(n_acc), C.byref(n_links), C.byref(n_ch)))
        buf = C.create_string_buffer(4096)
        check(lib.mp_topology_name(handle, buf, 4096))
        self.name = buf.value.decode()
        self.devices = [DeviceId(i) for i in range(n_acc.value)] + [HOST_DEVICE]
        if links is None:
            links = []
            for i in range(n_links.value):
                l = _lib.mp_link()
                check(lib.mp_topology_link(handle, i, C.byref(l)))
                links.append(LinkSpec(device_from_abi(l.a), device_from_abi(l.b), l.bandwidth,
                                      l.latency, HALF if l.duplex == MP_DUPLEX_HALF else FULL,
                                      l.sublinks))
        self.links = links
        self._channel_list: list[Channel] = []
        self._channel_ends: list[tuple[int, int]] = []
        for i in range(n_ch.value):
            c = _lib.mp_channel()
            check(lib.mp_topology_channel(handle, i, C.byref(c)))
            self._channel_list.append(Channel(c.id.decode(), c.bandwidth, c.latency))
            self._channel_ends.append((c.a, c.b))
        self._index = {id(ch): i for i, ch in enumerate(self._channel_list)}

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h:
            lib.mp_topology_destroy(h)
            self._handle = None

    @property
    def accelerators(self) -> list[DeviceId]:
        return [d for d in self.devices if not d.is_host]

    @property
    def host(self) -> DeviceId:
        return HOST_DEVICE

    def device(self, index: int) -> DeviceId:
        dev = DeviceId(index)
        if dev not in self.devices:
            raise TopologyError(f"no accelerator with index {index} in {self.name!r}")
        return dev

    def channel_for(self, src: DeviceId, dst: DeviceId) -> Channel:
        """The direction channel carrying src -> dst traffic (topology.py:136-143)."""
        out = C.c_int32()
        check(lib.mp_topology_channel_for(self._handle, src.abi, dst.abi, C.byref(out)))
        return self._channel_list[out.value]

    def has_link(self, src: DeviceId, dst: DeviceId) -> bool:
        out = C.c_int32()
        if src == dst:
            return False
        return lib.mp_topology_channel_for(self._handle, src.abi, dst.abi, C.byref(out)) == 0

    def channels(self) -> list[Channel]:
        """All distinct channels in creation order."""
        return list(self._channel_list)

    # -- ABI helpers -------------------------------------------------------
    def channel_index(self, ch: Channel) -> int:
        try:
            return self._index[id(ch)]
        except KeyError:
            raise TopologyError(f"channel {ch.id} is not part of topology {self.name!r}") from None

    def channel_at(self, index: int) -> Channel:
        return self._channel_list[index]


def load_topology(source: str, name: str = "topology") -> Topology:
    """Parse topology text (topology.py:164-240) in the C++ planner."""
    handle = C.c_void_p()
    check(lib.mp_topology_load(source.encode(), name.encode(), C.byref(handle)))
    return Topology._from_handle(handle)


def load_topology_file(path: str) -> Topology:
    with open(path, encoding="utf-8") as fh:
        return load_topology(fh.read())


def mesh_text(name: str, accelerators: int, link_bw: float, sublinks: int, link_lat: float,
              host_bw: float | None, host_lat: float = 0.0, host_duplex: str = HALF,
              link_duplex: str = FULL) -> str:
    """Text of a full-mesh node in the reference `.topo` schema."""
    out = [f"name {name}", "[device]"]
    out += [f"{i} accelerator" for i in range(accelerators)]
    out.append("[link]")
    for a in range(accelerators):
        for b in range(a + 1, accelerators):
            out.append(f"{a} {b} {link_bw!r} {link_lat!r} {link_duplex} {sublinks}")
    if host_bw is not None:
        out.append("[hostlink]")
        out += [f"{d} {host_bw!r} {host_lat!r} {host_duplex}" for d in range(accelerators)]
    return "\n".join(out) + "\n"


# The reference's calibrated 4-GPU presets (presets/beluga.topo, narval.topo):
# 2 (V100) or 4 (A100) sublinks of 25e9 B/s per pair, 1 us; host 22.5e9 half, 30 us.
# "b200": 8 GPUs through NVSwitch at the nominal 900e9 B/s per direction,
# PCIe Gen5 host links at 64e9 B/s full duplex (replace with a probed .topo).
_PRESETS = {
    "beluga": lambda: mesh_text("beluga", 4, 25e9, 2, 1e-6, 22.5e9, 30e-6, HALF),
    "narval": lambda: mesh_text("narval", 4, 25e9, 4, 1e-6, 22.5e9, 30e-6, HALF),
    "b200": lambda: mesh_text("b200", 8, 900e9, 1, 2e-6, 64e9, 10e-6, FULL),
}
PRESETS = tuple(_PRESETS)


def preset_text(name: str) -> str:
    if name not in _PRESETS:
        raise TopologyError(f"unknown preset {name!r}, available: {', '.join(PRESETS)}")
    return _PRESETS[name]()


def preset(name: str) -> Topology:
    """Load a shipped node preset by name (topology.py:248-253)."""
    return load_topology(preset_text(name))


def resolve(spec: str) -> Topology:
    """A preset name, 'name.topo' of a preset, or a config file path (topology.py:256-266)."""
    if spec in _PRESETS:
        return preset(spec)
    if os.path.exists(spec):
        return load_topology_file(spec)
    stem = os.path.basename(spec)
    if stem.endswith(".topo") and stem[:-5] in _PRESETS:
        return preset(stem[:-5])
    raise TopologyError(f"no such topology file or preset: {spec!r}")
