"""Multi-process transfers: one process per GPU (torch.distributed plumbing).

The paper's setting is MPI ranks over UCX `cuda_ipc`: a
rendezvous exchanges CUDA-IPC handles once, then every message moves GPU to
GPU.  Here:

* `TransferGroup(topology)` creates this rank's group context
  (`mp_group_create`: relay staging arena, relay flags and a sync block in its
  HBM; `mp_group_host_arena`: a host inbox in POSIX shared memory, pinned and
  mapped), exports their IPC handles / inbox name and maps every peer's
  (`mp_group_import`) — one all-gather at construction;
* `expose(tensor, owner)` shares one buffer's IPC handle (broadcast from its
  owner, opened once per process and cached: `mp_group_open`);
* `transfer(src_buf, dst_buf, nbytes, config)` is collective: every rank
  calls it in the same order; the source rank's kernel pushes Direct and
  hop1 tiles into peer memory over NVLink (relay staging, or the
  destination's host inbox over PCIe for the host-staged path), each relay
  rank's kernel moves its hop2 tiles, the destination rank's kernel moves
  the host path's hop2 tiles and waits until every byte landed (its stream
  is then ordered after the data), other ranks only join the device-side
  barrier that orders consecutive transfers.

Rendezvous logic (`exchange_blobs`, `share_buffer`, `roles`) is plain
torch.distributed + planner code, covered by gloo tests on CPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from ._lib import MP_GROUP_BLOB_BYTES, MP_IPC_HANDLE_BYTES, check, lib
from .paths import PathConfig, plan_paths
from .topology import Topology


def exchange_blobs(blob: bytes, group=None) -> list[bytes]:
    """All-gather every rank's resource blob (IPC handles), in rank order."""
    import torch.distributed as dist
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    return out


def share_buffer(owner: int, payload, group=None):
    """Broadcast `payload` (the owner's handle/offset/size/align) to every rank."""
    import torch.distributed as dist
    box = [payload if dist.get_rank(group) == owner else None]
    dist.broadcast_object_list(box, src=owner, group=group)
    return box[0]


def roles(topology: Topology, src: int, dst: int, config: PathConfig) -> dict[int, str]:
    """Who does what in one transfer: 'sender', 'receiver', 'relay' or 'idle'
    per rank — the deterministic plan every rank computes independently."""
    ps = plan_paths(topology, topology.device(src), topology.device(dst), config)
    out = {d.index: "idle" for d in topology.accelerators}
    out[src], out[dst] = "sender", "receiver"
    for p in ps.paths:
        if p.kind == "gpu":
            out[p.stage.index] = "relay"
    return out


@dataclass(frozen=True)
class RemoteBuffer:
    """A buffer of rank `owner`, as addressable from this process."""

    owner: int
    ptr: int      # local pointer on the owner, IPC-mapped pointer elsewhere
    nbytes: int
    align: int    # owner's address mod 16 (same on every rank)


class TransferGroup:
    def __init__(self, topology: Topology, device: int | None = None,
                 stage_bytes: int = 512 << 20, flag_cap: int = 4096, group=None,
                 host_bytes: int = 64 << 20):
        import torch
        import torch.distributed as dist
        self.pg = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if len(topology.accelerators) != self.world:
            raise ValueError(f"topology has {len(topology.accelerators)} accelerators for "
                             f"{self.world} ranks")
        self.device = torch.cuda.current_device() if device is None else device
        self.topology = topology
        self._ctx = C.c_void_p()
        check(lib.mp_group_create(self.world, self.rank, self.device, stage_bytes, flag_cap,
                                  C.byref(self._ctx)))
        check(lib.mp_ctx_set_topology(self._ctx, topology._handle))
        if host_bytes:
            check(lib.mp_group_host_arena(self._ctx, host_bytes))
        blob = (C.c_uint8 * MP_GROUP_BLOB_BYTES)()
        check(lib.mp_group_export(self._ctx, blob))
        for q, b in enumerate(exchange_blobs(bytes(blob), group)):
            if q != self.rank:
                arr = (C.c_uint8 * MP_GROUP_BLOB_BYTES).from_buffer_copy(b)
                check(lib.mp_group_import(self._ctx, q, arr))
        dist.barrier(group=group)

    def close(self):
        """Free this rank's resources.  Peers' kernels write into this rank's
        memory (staging, flags, host inbox, exposed buffers), so close every
        rank only after the last transfer finished everywhere — `sync()` on
        each rank, then a barrier (as the tests do)."""
        if getattr(self, "_ctx", None):
            lib.mp_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        self.close()

    def configure(self, **kw) -> None:
        from .engine import Engine
        Engine.configure(self, **kw)  # same knobs (mp_ctx_set_engine)

    def expose(self, tensor, owner: int) -> RemoteBuffer:
        """Collective: make `owner`'s tensor addressable on every rank."""
        payload = None
        if self.rank == owner:
            h = (C.c_uint8 * MP_IPC_HANDLE_BYTES)()
            off = C.c_uint64()
            check(lib.mp_ipc_export(tensor.data_ptr(), self.device, h, C.byref(off)))
            payload = (bytes(h), off.value, tensor.numel() * tensor.element_size(),
                       tensor.data_ptr() % 16)
        handle, off, nbytes, align = share_buffer(owner, payload, self.pg)
        if self.rank == owner:
            return RemoteBuffer(owner, tensor.data_ptr(), nbytes, align)
        ptr = C.c_void_p()
        arr = (C.c_uint8 * MP_IPC_HANDLE_BYTES).from_buffer_copy(handle)
        check(lib.mp_group_open(self._ctx, arr, off, C.byref(ptr)))
        return RemoteBuffer(owner, ptr.value, nbytes, align)

    def transfer(self, src: RemoteBuffer, dst: RemoteBuffer, nbytes: int | None = None,
                 config: PathConfig | None = None, stream=None) -> None:
        """Collective multi-path transfer src.owner -> dst.owner (asynchronous on
        `stream`; on the receiver the stream is ordered after the data)."""
        import torch
        config = config or PathConfig()
        nbytes = min(src.nbytes, dst.nbytes) if nbytes is None else nbytes
        if nbytes > src.nbytes or nbytes > dst.nbytes:
            raise ValueError("nbytes exceeds a buffer")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        handle = s.cuda_stream if hasattr(s, "cuda_stream") else int(s)
        cfg = config.abi()
        sp = src.ptr if self.rank == src.owner else None
        check(lib.mp_group_send(self._ctx, sp, src.align, dst.ptr, nbytes, src.owner, dst.owner,
                                C.byref(cfg), handle or None))

    def role(self) -> int:
        r = C.c_int32()
        check(lib.mp_group_role(self._ctx, C.byref(r)))
        return r.value

    def sync(self) -> None:
        check(lib.mp_sync(self._ctx))

    def stats(self):
        from .engine import Engine
        return Engine.stats(self)

    def last_plan(self):
        from .engine import Engine
        return Engine.last_plan(self)

