"""Measurement-driven configuration search (replaces the simulated tuner).

Same interface as the reference's `mpsim.tuner` (tuner.py:29-124):
GridPoint, default_grid, TuningEntry, TuningTable (nearest-size lookup, CSV
round trip in the reference's schema) and `tune` — but every grid point is
*timed on the GPU* through the engine (CUDA events around cached-graph
replays or per-call stream launches) instead of being simulated.  Ties break
as in the reference: fewer paths, then fewer chunks, then host off.

`calibrate_host_bandwidth` closes the loop between measurement and the
planner: the reference splits bytes purely by bottleneck bandwidth
(paths.py:144-150), so the host link's entry in the `.topo` must be the rate
the host-staged path actually sustains next to the direct path (pipeline
fill, per-copy overhead, PCIe duplex contention) — found here by timing the
real multi-path transfer for candidate values.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .paths import PathConfig
from .topology import Topology, load_topology, mesh_text

GRAPH_MODE = "graph"
STREAMED_MODE = "streamed"
DEFAULT_GPU_PATHS = (1, 2, 3)
DEFAULT_HOST_FLAGS = (False, True)
DEFAULT_MAX_CHUNKS = (1, 2, 4, 8, 16, 32)
MODES = (GRAPH_MODE, STREAMED_MODE)


@dataclass(frozen=True)
class GridPoint:
    gpu_paths: int
    host: bool
    max_chunks: int


def default_grid(max_gpu_paths: int = 3) -> list[GridPoint]:
    return [GridPoint(g, h, c)
            for g in DEFAULT_GPU_PATHS if g <= max_gpu_paths
            for h in DEFAULT_HOST_FLAGS
            for c in DEFAULT_MAX_CHUNKS]


@dataclass(frozen=True)
class TuningEntry:
    size: int
    mode: str
    best: GridPoint
    makespan: float  # measured seconds per transfer at the winning point


@dataclass
class TuningTable:
    topology: str
    entries: list[TuningEntry]

    def lookup(self, size: int, mode: str) -> TuningEntry:
        """Entry of the nearest tuned size (log distance; the smaller size wins ties)."""
        cands = [e for e in self.entries if e.mode == mode]
        if not cands:
            raise KeyError(f"no tuning entries for mode {mode!r}")
        return min(cands, key=lambda e: (abs(math.log(size) - math.log(e.size)), e.size))

    def config_for(self, size: int, mode: str = GRAPH_MODE,
                   base: PathConfig | None = None) -> PathConfig:
        p = self.lookup(size, mode).best
        b = base or PathConfig()
        return PathConfig(p.gpu_paths, p.host, p.max_chunks, mode == GRAPH_MODE,
                          b.cache_capacity, b.share_policy)

    def to_csv(self) -> str:
        lines = ["size,mode,gpu_paths,host,max_chunks,makespan"]
        for e in self.entries:
            lines.append(f"{e.size},{e.mode},{e.best.gpu_paths},"
                         f"{'on' if e.best.host else 'off'},{e.best.max_chunks},{e.makespan!r}")
        return "\n".join(lines) + "\n"

    @classmethod
    def from_csv(cls, text: str, topology: str = "") -> "TuningTable":
        entries = []
        for line in [ln for ln in text.splitlines() if ln.strip()][1:]:
            size, mode, paths, host, chunks, makespan = line.split(",")
            entries.append(TuningEntry(int(size), mode,
                                       GridPoint(int(paths), host == "on", int(chunks)),
                                       float(makespan)))
        return cls(topology, entries)


def measure_makespan(engine, config: PathConfig, size: int, src, dst, stream,
                     reps: int = 10, warmup: int = 5, trials: int = 3) -> float:
    """Seconds per transfer: CUDA events around `reps` back-to-back sends,
    best of `trials`.  The warm-up replays matter: the first launches of a
    freshly instantiated graph are several times slower than steady state.
    Sends go through `Engine.prepare` (the bound fast path, ~1.8 us of host
    time): through `send` (~2.3-4 us) a 1-4 MiB message is host-bound and the
    engine choice between two faster GPU mechanisms comes down to noise."""
    import torch
    go = engine.prepare(src, dst, size, config, stream=stream, src_dev=0, dst_dev=1)
    for _ in range(warmup):
        go()
    best = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(trials):
        e0.record(stream)
        for _ in range(reps):
            go()
        e1.record(stream)
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        best = t if best is None else min(best, t)
    return best


def warm_up(engine, src, dst, stream, sends: int = 400) -> None:
    """Send before timing anything: the first few hundred programmatic-
    dependent launches of a fresh engine run slow (1-4 MiB single-path
    sends at ~6.4 us, three launch quanta, instead of ~2.8 us;
    tools/exp_pdl_warm.py, profiles/r02_exp_pdl_warm.txt), which once made
    tune_engines pick copy engines at 2-4 MiB where the SM kernel is faster."""
    import torch
    n = min(src.numel(), 1 << 20)
    go = engine.prepare(src[:n], dst[:n], n, PathConfig(max_chunks=1, graph_mode=True), stream=stream,
                        src_dev=0, dst_dev=1)
    for _ in range(sends):
        go()
    torch.cuda.synchronize()


def tune(engine, sizes: list[int], grid: list[GridPoint] | None = None,
         modes: tuple[str, ...] = MODES, reps: int = 50, device=None) -> TuningTable:
    """Time every grid point per (size, mode) on the GPU; record the argmin.

    The reference's `tune(topology, sizes, grid, modes)` (tuner.py:102-124)
    predicts makespans from a Topology; this one measures, so its first
    argument is an `Engine` (whose `.topology` is the planning topology) —
    the only signature difference.  Same grid, tie-break and TuningTable."""
    import torch
    if not sizes:
        raise ValueError("size list is empty")
    n = len(engine.topology.accelerators)
    grid = default_grid(n - 1) if grid is None else grid
    if not grid:
        raise ValueError("tuning grid is empty")
    dev = device if device is not None else engine.device_map[0]
    big = torch.empty(max(sizes), dtype=torch.uint8, device=f"cuda:{dev}")
    out = torch.empty_like(big)
    stream = torch.cuda.Stream(device=dev)
    warm_up(engine, big, out, stream)
    entries = []
    for size in sizes:
        for mode in modes:
            best_key, best = None, None
            for p in grid:
                if p.gpu_paths > n - 1:
                    continue
                cfg = PathConfig(p.gpu_paths, p.host, p.max_chunks, mode == GRAPH_MODE)
                t = measure_makespan(engine, cfg, size, big[:size], out[:size], stream, reps)
                key = (t, p.gpu_paths, p.max_chunks, p.host)
                if best_key is None or key < best_key:
                    best_key, best = key, TuningEntry(size, mode, p, t)
            if best is None:
                raise ValueError(f"no grid point is feasible on {n} accelerators "
                                 f"(every point needs more than {n - 1} GPU paths)")
            entries.append(best)
    engine.clear_cache()
    return TuningTable(engine.topology.name, entries)


def tune_engines(engine, sizes: list[int], reps: int = 50, mode: str = GRAPH_MODE,
                 host_chunks: int = 2) -> tuple[list[tuple[int, str, str]], list[dict]]:
    """Measure, at every size, the direct path by the SM transfer kernel vs a
    copy-engine copy (single path), then — with the winning direct mechanism —
    the host-staged path by the SM kernels (mapped pinned memory) vs copy
    engines (direct + host, `host_chunks` chunks).  Returns the per-size
    policy [(max_bytes, direct, host)] for `Engine.set_size_policy`
    (boundaries at the geometric mid-points between tuned sizes) and the raw
    trials."""
    import torch
    sizes = sorted(sizes)
    dev = engine.device_map[0]
    big = torch.empty(sizes[-1], dtype=torch.uint8, device=f"cuda:{dev}")
    out = torch.empty_like(big)
    stream = torch.cuda.Stream(device=dev)
    graph = mode == GRAPH_MODE
    saved = engine.options()
    engine.set_size_policy([])
    trials = []
    single = PathConfig(max_chunks=1, graph_mode=graph)
    warm_up(engine, big, out, stream)
    # both mechanisms twice, interleaved: launch-quantum flips (2.05 us) and
    # drift then cost one pass, not the choice (the best pass counts)
    for _ in range(2):
        for name in ("sm", "ce"):
            engine.configure(direct=name)
            for s in sizes:
                t = measure_makespan(engine, single, s, big[:s], out[:s], stream, reps)
                trials.append({"bytes": s, "path": "direct", "engine": name, "seconds": t})

    def pick(path, s):
        ts = {}
        for t in trials:
            if t["bytes"] == s and t["path"] == path:
                ts[t["engine"]] = min(ts.get(t["engine"], float("inf")), t["seconds"])
        return "sm" if ts["sm"] <= ts["ce"] else "ce"
    direct = {s: pick("direct", s) for s in sizes}
    multi = PathConfig(1, True, host_chunks, graph)
    for name in ("sm", "ce"):
        engine.configure(host=name)
        for s in sizes:
            engine.set_size_policy([(2**63 - 1, direct[s], name)])
            t = measure_makespan(engine, multi, s, big[:s], out[:s], stream, reps)
            trials.append({"bytes": s, "path": "host", "engine": name, "seconds": t})
    engine.set_size_policy([])
    names = {0: "sm", 1: "ce", 2: "auto"}
    engine.configure(direct=names[saved["direct_engine"]], host=names[saved["host_engine"]])
    rules: list[tuple[int, str, str]] = []
    for i, s in enumerate(sizes):
        choice = (direct[s], pick("host", s))
        bound = int(math.sqrt(s * sizes[i + 1])) if i + 1 < len(sizes) else 2**63 - 1
        if rules and rules[-1][1:] == choice:
            rules[-1] = (bound, *choice)
        else:
            rules.append((bound, *choice))
    engine.clear_cache()
    return rules, trials


def pick_host_rate(runs, tolerance: float = 0.005):
    """Of calibration runs (seconds, host_bw, ...), the one with the smallest
    host rate whose time is within `tolerance` of the fastest (ties: faster)."""
    fastest = min(r[0] for r in runs)
    return min((r for r in runs if r[0] <= fastest * (1 + tolerance)), key=lambda r: (r[1], r[0]))


def calibrate_host_bandwidth(engine, link_bw: float, size: int, max_chunks: int,
                             candidates: list[float] | None = None, reps: int = 10,
                             name: str = "calibrated",
                             host_engines: tuple[str, ...] = ("ce", "sm"),
                             tolerance: float = 0.005) -> tuple[float, Topology, list]:
    """Pick the host-link bandwidth for the `.topo` (and the host-path
    mechanism) that maximise the measured direct+host throughput at `size`
    (the smallest host rate within `tolerance` of the best).
    Leaves `engine` on the winning topology and host mechanism; returns
    (host_bw, topology, trials) with trials = [(engine, host_bw, GB/s)]."""
    import torch
    n = len(engine.topology.accelerators)
    if candidates is None:
        candidates = [b * 1e9 for b in (1, 2, 4, 6, 8, 10, 12, 16, 20, 28, 40, 55)]
    dev = engine.device_map[0]
    src = torch.empty(size, dtype=torch.uint8, device=f"cuda:{dev}")
    dst = torch.empty_like(src)
    stream = torch.cuda.Stream(device=dev)
    cfg = PathConfig(1, True, max_chunks, True)
    trials = []
    runs = []
    warm_up(engine, src, dst, stream)
    for host in host_engines:
        engine.configure(host=host)
        for bw in candidates:
            topo = load_topology(mesh_text(name, n, link_bw, 1, 2e-6, bw, 1e-5, "full"))
            engine.set_topology(topo)
            t = measure_makespan(engine, cfg, size, src, dst, stream, reps)
            trials.append((host, bw, size / t / 1e9))
            runs.append((t, bw, topo, host))
    # the curve is flat over a wide range of host rates (an HBM-bound copy):
    # take the smallest host rate within `tolerance` of the fastest, so run
    # noise does not pick a large host share that other configurations (more
    # paths, other sizes planned from the same .topo) then pay for
    best = pick_host_rate(runs, tolerance)
    engine.configure(host=best[3])
    engine.set_topology(best[2])
    return best[1], best[2], trials
