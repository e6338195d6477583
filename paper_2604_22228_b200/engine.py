"""Real multi-path transfers on B200: the `send` / `recv` entry points.

This replaces the reference's simulated execution (`simulate_graph` /
`simulate_streamed`, /root/reference/pkg/src/mpsim/sim.py:272-292) with the
CUDA engine behind `mp_send` (csrc/mp_engine.cu):

    plan_paths -> make_chunk_plan           (C++ planner, bit-exact)
    -> key (src, dst, size, devices, path set) -> LRU of cudaGraphExec_t
    -> miss: lower to device tiles + copy-engine lanes, capture, instantiate
    -> hit : one cudaGraphLaunch on the caller's stream

PyTorch only owns the buffers and streams.  Logical accelerators of the
topology map onto physical CUDA devices through `device_map`; several
logical devices may share one GPU ("loopback"), which runs every path type —
relay flags included — on a single B200.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

from . import _lib, _mpfast
from ._lib import (MP_COPY_TMA, MP_COPY_VEC, MP_ENGINE_AUTO, MP_ENGINE_CE, MP_ENGINE_SM, EngineError,
                   check, lib)
from .paths import PathConfig, _paths_from_abi
from .pipeline import ChunkAssignment
from .topology import Topology, load_topology, mesh_text

ENGINES = {"sm": MP_ENGINE_SM, "ce": MP_ENGINE_CE, "auto": MP_ENGINE_AUTO}
COPIES = {"vec": MP_COPY_VEC, "tma": MP_COPY_TMA}
KERNELS = {0: "mpk::transfer_kernel<0,8> (16-byte LDG/STG, dynamic tile claims)",
           1: "mpk::transfer_kernel<1,8> (TMA bulk ring)",
           2: "mpk::small_copy_kernel<4> (descriptors in kernel params)"}


@dataclass
class SendStats:
    """Lifecycle of the last send: the reference's four phases (graph.py:24), measured."""

    hit: bool
    graph_mode: bool
    nodes_logical: int
    nodes_physical: int
    kernels: int
    ce_copies: int
    creation_us: float
    construction_us: float
    instantiation_us: float
    launch_us: float
    plan_us: float
    cache_hits: int
    cache_misses: int
    cache_evictions: int
    kernel: str = ""  # the source device's copy kernel ("" = copy engines only)


def _torch():
    import torch  # noqa: PLC0415 - torch is plumbing, imported on first use
    return torch


def _raise_status(rc: int) -> None:
    """Error path of a prepared send (_mpfast.BoundSend): map an MP_* status
    to the reference's exception classes; -1000 = used after Engine.close()."""
    if rc == -1000:
        raise EngineError("prepared send used after Engine.close()")
    check(rc)


class Engine:
    """A transfer context over `n_logical` accelerators of `topology`."""

    def __init__(self, topology: Topology, device_map: list[int] | None = None):
        n = len(topology.accelerators)
        if device_map is None:
            count = _torch().cuda.device_count()
            if count < 1:
                raise _lib.EngineError("no CUDA device is visible: the engine has no CPU path")
            device_map = [i % count for i in range(n)]
        if len(device_map) != n:
            raise ValueError(f"device_map has {len(device_map)} entries for {n} accelerators")
        self.topology = topology
        self.device_map = list(device_map)
        self._bindings: list = []  # weak refs to prepared sends (invalidated by close())
        arr = (C.c_int32 * n)(*self.device_map)
        self._ctx = C.c_void_p()
        check(lib.mp_ctx_create(n, arr, C.byref(self._ctx)))
        check(lib.mp_ctx_set_topology(self._ctx, topology._handle))
        self._ctx_addr = self._ctx.value  # for the CPython fast path (_mpfast)

    @classmethod
    def loopback(cls, n_logical: int = 2, device: int = 0, link_bw: float = 3.0e12,
                 host_bw: float = 50e9) -> "Engine":
        """`n_logical` logical GPUs all mapped onto one physical device."""
        topo = load_topology(mesh_text("loopback", n_logical, link_bw, 1, 2e-6, host_bw, 10e-6,
                                       "full"))
        return cls(topo, [device] * n_logical)

    def close(self):
        for ref in getattr(self, "_bindings", ()):
            b = ref()
            if b is not None:
                b.invalidate()
        if getattr(self, "_ctx", None):
            self._ctx_addr = 0
            lib.mp_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- configuration ------------------------------------------------------
    def set_topology(self, topology: Topology):
        check(lib.mp_ctx_set_topology(self._ctx, topology._handle))
        self._ctx_addr = self._ctx.value  # for the CPython fast path (_mpfast)
        self.topology = topology

    def configure(self, *, direct: str | None = None, relay: str | None = None,
                  host: str | None = None,
                  ctas_per_sm: int | None = None, threads: int | None = None,
                  tile_bytes: int | None = None, host_slots: int | None = None,
                  pull: bool | None = None, sm_min_bytes: int | None = None,
                  copy: str | None = None, unroll: int | None = None,
                  tma_stages: int | None = None, tma_block: int | None = None,
                  tma_peer: bool | None = None, sched: str | None = None,
                  small_max_bytes: int | None = None, pdl: int | None = None,
                  wait_timeout_ms: int | None = None, fault_inject: int | None = None) -> None:
        """Pick the copy mechanism per path type and the SM-kernel shape.
        `sched`: "auto" (static one-tile-per-CTA tables when no tile waits or
        touches host memory) or "dynamic" (atomic tile claims always).
        `wait_timeout_ms`: limit of a relay-flag wait (0 = 4 s); a timeout
        fails every later send until `sync()` reports and clears it.
        `fault_inject` (tests only, bits): 1 mutes one staged chunk's hop1
        signal; 2 lowers logical devices that share a GPU as if they had
        their own (system-scope flags, host chunks as hop1 / hop2 tiles)."""
        o = _lib.mp_engine_opts()
        check(lib.mp_ctx_get_engine(self._ctx, C.byref(o)))
        if wait_timeout_ms is not None:
            o.wait_timeout_ms = int(wait_timeout_ms)
        if fault_inject is not None:
            o.fault_inject = int(fault_inject)
        if small_max_bytes is not None:
            o.small_max_bytes = small_max_bytes
        if pdl is not None:
            o.pdl = int(pdl)
        if sched is not None:
            o.sched = {"auto": _lib.MP_SCHED_AUTO, "dynamic": _lib.MP_SCHED_DYNAMIC}[sched]
        if tma_peer is not None:
            o.tma_peer = int(tma_peer)
        if copy is not None:
            o.copy_kind = COPIES[copy]
        if unroll is not None:
            o.unroll = unroll
        if tma_stages is not None:
            o.tma_stages = tma_stages
        if tma_block is not None:
            o.tma_block = tma_block
        if direct is not None:
            o.direct_engine = ENGINES[direct]
        if relay is not None:
            o.relay_engine = ENGINES[relay]
        if host is not None:
            o.host_engine = ENGINES[host]
        if ctas_per_sm is not None:
            o.ctas_per_sm = ctas_per_sm
        if threads is not None:
            o.threads = threads
        if tile_bytes is not None:
            o.tile_bytes = tile_bytes
        if host_slots is not None:
            o.host_slots = host_slots
        if pull is not None:
            o.pull = int(pull)
        if sm_min_bytes is not None:
            o.sm_min_bytes = sm_min_bytes
        check(lib.mp_ctx_set_engine(self._ctx, C.byref(o)))

    def set_size_policy(self, rules: list[tuple]) -> None:
        """[(max_bytes, direct, host), ...] with increasing max_bytes and
        "sm"|"ce" mechanisms (host may be omitted/None: keep the default) —
        the per-size choice from `tuner.tune_engines`; [] restores defaults."""
        n = len(rules)
        mx = (C.c_uint64 * max(1, n))(*[int(r[0]) for r in rules])
        en = (C.c_int32 * max(1, n))(*[ENGINES[r[1]] for r in rules])
        hosts = [r[2] if len(r) > 2 else None for r in rules]
        he = None
        if any(h is not None for h in hosts):
            he = (C.c_int32 * max(1, n))(*[ENGINES[h] if h else ENGINES["ce"] for h in hosts])
        check(lib.mp_ctx_set_size_policy(self._ctx, mx, en, he, n))
        self.size_policy = list(rules)

    def options(self) -> dict:
        o = _lib.mp_engine_opts()
        check(lib.mp_ctx_get_engine(self._ctx, C.byref(o)))
        return {f: getattr(o, f) for f, _ in o._fields_}

    # -- the transfer -------------------------------------------------------
    def send_ptr(self, src_ptr: int, dst_ptr: int, nbytes: int, src_dev: int, dst_dev: int,
                 config: PathConfig, stream: int = 0) -> None:
        """Raw-pointer send through the C ABI (`mp_send`, via the CPython fast path)."""
        rc = _mpfast.send(self._ctx_addr, src_ptr, dst_ptr, nbytes, src_dev, dst_dev,
                          config.abi_addr(), stream or 0)
        if rc:
            check(rc)

    def _resolve(self, src, dst, nbytes, config, stream, src_dev, dst_dev):
        """Validated arguments of a tensor send: (config, nbytes, src_dev,
        dst_dev, stream handle)."""
        if config is None:
            config = PathConfig.from_env()
        if not (src.is_cuda and dst.is_cuda):
            raise ValueError("send moves CUDA tensors (use torch's copies for host memory)")
        if not (src.is_contiguous() and dst.is_contiguous()):
            raise ValueError("send moves contiguous byte ranges: src and dst must be contiguous")
        sn = src.nbytes
        if nbytes is None:
            nbytes = sn
        if nbytes > sn or nbytes > dst.nbytes:
            raise ValueError("nbytes exceeds a buffer")
        sp, dp = src.get_device(), dst.get_device()
        dmap = self.device_map
        if src_dev is None:
            if sp not in dmap:
                raise ValueError(f"src lives on cuda:{sp}, which no logical device maps to")
            src_dev = dmap.index(sp)
        if dst_dev is None:
            cands = [i for i, d in enumerate(dmap) if d == dp and i != src_dev]
            if not cands:
                raise ValueError("cannot infer the logical destination device; pass dst_dev")
            dst_dev = cands[0]
        if dmap[src_dev] != sp or dmap[dst_dev] != dp:
            raise ValueError(f"src/dst tensors live on cuda:{sp}/cuda:{dp}, but logical devices "
                             f"{src_dev}/{dst_dev} map to cuda:{dmap[src_dev]}/cuda:{dmap[dst_dev]}")
        if stream is None:
            stream = _torch().cuda.current_stream(sp)
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        return config, nbytes, src_dev, dst_dev, handle

    def send(self, src, dst, nbytes: int | None = None, config: PathConfig | None = None,
             stream=None, src_dev: int | None = None, dst_dev: int | None = None) -> None:
        """Move `nbytes` (default: all of `src`) from tensor `src` to tensor `dst`.

        Asynchronous on `stream` (default: the current stream of src's
        device): ordered after prior work there, and that stream waits for
        completion.  `src_dev`/`dst_dev` are logical accelerators; by default
        the first logical device mapped to each tensor's GPU.
        (Kept lean: on a cached-graph hit this Python is most of the host cost.)
        """
        config, nbytes, src_dev, dst_dev, handle = self._resolve(src, dst, nbytes, config, stream,
                                                                 src_dev, dst_dev)
        rc = _mpfast.send(self._ctx_addr, src.data_ptr(), dst.data_ptr(), nbytes, src_dev, dst_dev,
                          config.abi_addr(), handle or 0)
        if rc:
            check(rc)

    def prepare(self, src, dst, nbytes: int | None = None, config: PathConfig | None = None,
                stream=None, src_dev: int | None = None, dst_dev: int | None = None):
        """Bind a send to its arguments once (same meaning as `send`) and
        return a zero-argument callable that issues it: the per-message host
        cost is then one C call (`_mpfast.BoundSend`), for loops that resend
        the same buffers (osu_bw windows, halo exchanges, pipelined stages).
        The binding keeps the tensors, config and stream alive; it must not
        outlive the engine."""
        config, nbytes, src_dev, dst_dev, handle = self._resolve(src, dst, nbytes, config, stream,
                                                                 src_dev, dst_dev)
        bound = _mpfast.bind(self._ctx_addr, src.data_ptr(), dst.data_ptr(), nbytes, src_dev, dst_dev,
                             config.abi_addr(), handle or 0, (src, dst, config, stream), _raise_status)
        # the call itself is C (None on success); Engine.close() invalidates
        # every binding so a stale one never touches the freed context
        if len(self._bindings) > 4096:
            self._bindings = [r for r in self._bindings if r() is not None]
        self._bindings.append(weakref.ref(bound))
        return bound

    def _xfers(self, transfers, stream):
        """(mp_xfer array, stream handle) for send_many / prepare_many."""
        torch = _torch()
        arr = (_lib.mp_xfer * len(transfers))()
        first = None
        for i, (src, dst, nbytes, sd, dd) in enumerate(transfers):
            if not (src.is_cuda and dst.is_cuda and src.is_contiguous() and dst.is_contiguous()):
                raise ValueError("send_many moves contiguous CUDA tensors")
            n = src.numel() * src.element_size() if nbytes is None else nbytes
            if n > src.numel() * src.element_size() or n > dst.numel() * dst.element_size():
                raise ValueError("nbytes exceeds a buffer")
            arr[i] = _lib.mp_xfer(src.data_ptr(), dst.data_ptr(), n, sd, dd)
            first = src if first is None else first
        if stream is None:
            stream = torch.cuda.current_stream(first.device)
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        return arr, handle

    def send_many(self, transfers, config: PathConfig | None = None, joint: bool = False,
                  stream=None) -> None:
        """Concurrent transfers as one program (windows, bidirectional flows,
        ring halo exchanges): `transfers` = [(src, dst, nbytes, src_dev, dst_dev)]
        with tensors; nbytes None = all of src.  joint=True picks channel-
        disjoint staging devices (plan_contention_free, paths.py:210-242)."""
        config = config or PathConfig.from_env()
        arr, handle = self._xfers(transfers, stream)
        cfg = config.abi()
        check(lib.mp_send_many(self._ctx, arr, len(transfers), C.byref(cfg), int(joint),
                               handle or None))

    def prepare_many(self, transfers, config: PathConfig | None = None, joint: bool = False,
                     stream=None):
        """`send_many` bound once (same arguments): returns a zero-argument
        callable that posts the program with one C call — a window of W
        messages costs one host call and, on a cached hit, one graph launch.
        The binding keeps the tensors, config and stream alive; it must not
        outlive the engine."""
        config = config or PathConfig.from_env()
        arr, handle = self._xfers(transfers, stream)
        keep = (list(transfers), config, stream, arr)
        args = (self._ctx_addr, C.addressof(arr), len(transfers), config.abi_addr(), int(joint),
                handle or 0)
        ctx, send_many = self._ctx_addr, _mpfast.send_many
        engine = self

        def launch() -> None:
            if engine._ctx_addr != ctx:  # closed engine: never touch a freed context
                raise EngineError("prepared send used after Engine.close()")
            rc = send_many(*args)
            if rc:
                check(rc)
        launch.keep = keep
        return launch

    def recv(self, dst, stream=None) -> None:
        """Single-process mode: `send` already wrote `dst` on the sender's
        stream; `recv` makes `stream` (default: current stream of dst's
        device) wait for the last send (`mp_wait`)."""
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(dst.device)
        handle = s.cuda_stream if hasattr(s, "cuda_stream") else int(s)
        check(lib.mp_wait(self._ctx, handle or None))

    def sync(self) -> None:
        """Wait for every transfer; raises if a relay flag wait timed out
        since the last sync (and clears the error, so sends run again)."""
        check(lib.mp_sync(self._ctx))

    # -- introspection -------------------------------------------------------
    def stats(self) -> SendStats:
        s = _lib.mp_send_stats()
        check(lib.mp_send_stats_get(self._ctx, C.byref(s)))
        return SendStats(bool(s.hit), bool(s.graph_mode), s.nodes_logical, s.nodes_physical,
                         s.kernels, s.ce_copies, s.creation_us, s.construction_us,
                         s.instantiation_us, s.launch_us, s.plan_us, s.cache_hits,
                         s.cache_misses, s.cache_evictions, KERNELS.get(s.kernel, ""))

    def last_plan(self):
        """(paths, chunks) the engine executed on the last send — for parity checks."""
        npaths, nchunks = C.c_int32(), C.c_int32()
        lib.mp_last_plan(self._ctx, None, 0, C.byref(npaths), None, 0, C.byref(nchunks))
        paths = (_lib.mp_path * max(1, npaths.value))()
        chunks = (_lib.mp_chunk * max(1, nchunks.value))()
        check(lib.mp_last_plan(self._ctx, paths, npaths.value, C.byref(npaths), chunks,
                               nchunks.value, C.byref(nchunks)))
        ps = _paths_from_abi(self.topology, paths, npaths.value)
        cs = tuple(ChunkAssignment(c.path_index, c.offset, c.length, c.seq)
                   for c in chunks[:nchunks.value])
        return ps, cs

    def trace(self, src, dst, nbytes: int | None = None, config: PathConfig | None = None,
              src_dev: int | None = None, dst_dev: int | None = None):
        """Send once (streamed program, synchronous) and return (plan, Timeline):
        the real per-chunk-hop start/end times in the reference's Timeline
        schema, checkable with `integrity.check_timeline` (integrity.py:63-101)."""
        from .graph import build_graph
        from .pipeline import ChunkPlan
        from .paths import PathSet
        from .timeline import from_records
        from .topology import device_from_abi
        config = config or PathConfig.from_env()
        if nbytes is None:
            nbytes = src.numel() * src.element_size()
        if src_dev is None:
            src_dev = self.device_map.index(src.device.index)
        if dst_dev is None:
            cands = [i for i, d in enumerate(self.device_map)
                     if d == dst.device.index and i != src_dev]
            dst_dev = cands[0]
        cfg = config.abi()
        n = C.c_int32()
        lib.mp_send_trace(self._ctx, src.data_ptr(), dst.data_ptr(), nbytes, src_dev, dst_dev,
                          C.byref(cfg), None, 0, C.byref(n))
        recs = (_lib.mp_trace_rec * max(1, n.value))()
        check(lib.mp_send_trace(self._ctx, src.data_ptr(), dst.data_ptr(), nbytes, src_dev,
                                dst_dev, C.byref(cfg), recs, n.value, C.byref(n)))
        paths, chunks = self.last_plan()
        plan = ChunkPlan(nbytes, chunks, PathSet(device_from_abi(src_dev),
                                                 device_from_abi(dst_dev), paths))
        return plan, from_records(build_graph(plan), recs[:n.value])

    def clear_cache(self) -> None:
        check(lib.mp_cache_clear(self._ctx))

    def set_kernel_timing(self, on: bool = True) -> None:
        """Bracket every streamed-mode send's kernel with CUDA events (off by
        default: the events cost launch slots) so `kernel_time_ms` works."""
        check(lib.mp_ctx_set_kernel_timing(self._ctx, int(on)))

    def kernel_time_ms(self) -> float:
        ms = C.c_double()
        check(lib.mp_kernel_time_ms(self._ctx, C.byref(ms)))
        return ms.value

    def kernel_bench(self, src, dst, nbytes: int | None = None, config: PathConfig | None = None,
                     src_dev: int = 0, dst_dev: int = 1, reps: int = 20) -> float:
        """Milliseconds per launch of this transfer's source-device kernel over
        `reps` back-to-back launches (`mp_kernel_bench`)."""
        config = config or PathConfig()
        nbytes = src.numel() * src.element_size() if nbytes is None else nbytes
        cfg = config.abi()
        ms = C.c_double()
        check(lib.mp_kernel_bench(self._ctx, src.data_ptr(), dst.data_ptr(), nbytes, src_dev,
                                  dst_dev, C.byref(cfg), reps, C.byref(ms)))
        return ms.value

    def peer_matrix(self) -> list[list[int]]:
        n = len(set(self.device_map))
        arr = (C.c_int32 * (n * n))()
        check(lib.mp_ctx_peer_matrix(self._ctx, arr, n * n))
        return [list(arr[i * n:(i + 1) * n]) for i in range(n)]

    def measure_paths(self, src_dev: int = 0, dst_dev: int = 1, nbytes: int = 256 << 20,
                      iters: int = 5) -> dict[str, float]:
        """GB/s of each path type between two logical devices (1 GB = 1e9 B):
        the SM transfer kernel and a CE copy on the direct route, D2H and H2D
        alone, both at once (per direction), and the host-staged path run as
        the engine runs it (8 pipelined chunks, event handoff)."""
        out = (C.c_double * 8)()
        check(lib.mp_measure_paths(self._ctx, src_dev, dst_dev, nbytes, iters, out, 8))
        return {"direct_sm": out[0], "d2h": out[1], "h2d": out[2], "direct_ce": out[3],
                "duplex": out[4], "host_staged": out[5], "sm_d2h": out[6], "sm_h2d": out[7]}

    def probe_topology(self, nbytes: int = 256 << 20, iters: int = 5,
                       name: str = "probed") -> str:
        """Write a reference-schema `.topo` from measured bandwidths.

        Bandwidths are written with repr() and sublinks = 1 so the reference
        loader parses back the identical doubles (SURVEY.md §8c protocol).
        Only GPU0's links are probed; the node is assumed symmetric (NVSwitch).
        """
        n = len(self.topology.accelerators)
        link, host = self.probe_bandwidths(nbytes, iters)
        return mesh_text(name, n, link, 1, 2e-6, host, 10e-6, "full")

    def probe_node(self, nbytes: int = 256 << 20, iters: int = 5, name: str = "probed",
                   host_bytes: int = 8 << 20) -> str:
        """Measure every accelerator pair and host link of the context and
        write a reference-schema `.topo` (SURVEY §8c protocol: bandwidths with
        repr(), sublinks 1, so the planner parses back the identical doubles).
        Pairs on the same physical devices are measured once.  A host link's
        rate is the host-staged path's delivered rate as the engine runs it
        (like `probe_bandwidths`), not the isolated PCIe rate: planned on the
        isolated rate the staged path gets too large a share and multi-path
        loses to single path (profiles/r02_exp_linkcap.jsonl: 0.74-0.89x at
        128-512 MiB with a link-limited direct path, 1.02-1.06x on the
        measured rate)."""
        n = len(self.topology.accelerators)
        pair_bw: dict[tuple[int, int], float] = {}
        host_bw: dict[int, float] = {}
        lines = [f"name {name}", "[device]"] + [f"{i} accelerator" for i in range(n)] + ["[link]"]
        for a in range(n):
            for b in range(a + 1, n):
                key = (self.device_map[a], self.device_map[b])
                if key not in pair_bw:
                    m = self.measure_paths(a, b, nbytes, iters)
                    pair_bw[key] = max(m["direct_sm"], m["direct_ce"]) * 1e9
                lines.append(f"{a} {b} {pair_bw[key]!r} 2e-06 full 1")
        lines.append("[hostlink]")
        for d in range(n):
            phys = self.device_map[d]
            if phys not in host_bw:
                m = self.measure_paths(d, d, host_bytes, max(iters, 10))
                host_bw[phys] = m["host_staged"] * 1e9
            lines.append(f"{d} {host_bw[phys]!r} 1e-05 full")
        return "\n".join(lines) + "\n"

    def probe_bandwidths(self, nbytes: int = 256 << 20, iters: int = 5,
                         host_bytes: int = 8 << 20) -> tuple[float, float]:
        """(link, host) bytes/s for the planner's `.topo`.

        link = the faster direct mechanism (SM kernel or CE); host = the
        delivered rate of the host-staged path *as executed* — D2H and H2D
        pipelined over 8 chunks of a message-sized share, so per-copy
        overhead and full-duplex contention are priced in.  The reference's
        split is purely bandwidth-proportional (paths.py:144-150), so feeding
        it the isolated PCIe rate would overload the staged path by its
        pipeline fill (k+1)/k.
        """
        n = len(self.topology.accelerators)
        dst = 1 if n > 1 else 0
        m = self.measure_paths(0, dst, nbytes, iters)
        h = self.measure_paths(0, dst, host_bytes, max(iters, 10))
        self.last_probe = {"bulk": m, "host_share_sized": h}
        return max(m["direct_sm"], m["direct_ce"]) * 1e9, h["host_staged"] * 1e9


_default: Engine | None = None


def default_engine() -> Engine:
    """All visible GPUs with the nominal B200 preset; a 2-GPU loopback on one GPU."""
    global _default
    if _default is None:
        count = _torch().cuda.device_count()
        if count >= 2:
            from .topology import preset  # noqa: PLC0415
            topo = preset("b200") if count == 8 else load_topology(
                mesh_text("node", count, 900e9, 1, 2e-6, 64e9, 10e-6, "full"))
            _default = Engine(topo, list(range(count)))
        else:
            _default = Engine.loopback(2)
    return _default


def send(src, dst, nbytes: int | None = None, config: PathConfig | None = None, stream=None,
         src_dev: int | None = None, dst_dev: int | None = None) -> None:
    """Module-level multi-path send on the default engine (see Engine.send)."""
    default_engine().send(src, dst, nbytes, config, stream, src_dev, dst_dev)


def recv(dst, stream=None) -> None:
    default_engine().recv(dst, stream)
