"""Real execution timelines in the reference's Timeline schema.

The reference's simulator returns a `Timeline` of `SimTask`s
(sim.py:32-78) that `integrity.check_timeline` verifies (integrity.py:63-101)
and `Timeline.to_csv` dumps (`task_id,path,role,channel,start,end,offset,
length`).  `Engine.trace` produces the same object from a real send: every
logical node (chunk-hop, graph.py:91-118) carries the first-tile start and
last-tile completion stamped by the transfer kernel (%globaltimer), or the
CUDA-event times around its copy-engine op, in seconds from the fork.
"""

from __future__ import annotations

from dataclasses import dataclass

from .graph import ExecGraph
from .topology import Channel


@dataclass
class TraceTask:
    """One executed copy node (field names of the reference's SimTask)."""

    node_id: int
    path_index: int
    role: str
    channel: Channel
    lane: int
    offset: int
    length: int
    ready_time: float
    start_time: float
    end_time: float
    engine: str  # "sm" (transfer kernel tiles) or "ce" (copy engine)
    device: int

    @property
    def queue_time(self) -> float:
        return self.start_time - self.ready_time


@dataclass
class Timeline:
    start: float
    tasks: list[TraceTask]
    channel_busy: dict[str, list[tuple[float, float]]]
    makespan: float
    bytes_moved: int
    host_cost: float
    final_sync_cost: float
    lane_count: int

    @property
    def end(self) -> float:
        return self.start + self.makespan

    @property
    def contention_queue_time(self) -> float:
        return sum(t.queue_time for t in self.tasks)

    def to_csv(self) -> str:
        lines = ["task_id,path,role,channel,start,end,offset,length"]
        for t in self.tasks:
            lines.append(f"{t.node_id},{t.path_index},{t.role},{t.channel.id},"
                         f"{t.start_time!r},{t.end_time!r},{t.offset},{t.length}")
        return "\n".join(lines) + "\n"


def from_records(graph: ExecGraph, records, host_cost: float = 0.0) -> Timeline:
    """Assemble a Timeline from `mp_trace_rec`s (one per node, times in us)."""
    by_node = {r.node: r for r in records}
    tasks = []
    for n in graph.nodes:
        r = by_node[n.id]
        start, end = r.start_us * 1e-6, r.end_us * 1e-6
        tasks.append(TraceTask(n.id, n.path_index, n.role, n.channel, n.lane, n.offset,
                               n.length, start, start, end,
                               "sm" if r.engine == 0 else "ce", r.device))
    busy: dict[str, list[tuple[float, float]]] = {}
    for t in sorted(tasks, key=lambda x: x.start_time):
        busy.setdefault(t.channel.id, []).append((t.start_time, t.end_time))
    end = max((t.end_time for t in tasks), default=0.0)
    return Timeline(start=0.0, tasks=tasks, channel_busy=busy, makespan=end,
                    bytes_moved=sum(t.length for t in tasks), host_cost=host_cost,
                    final_sync_cost=0.0, lane_count=graph.lane_count)
