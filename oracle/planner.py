"""ORACLE (test infrastructure only): plain-Python restatement of the
reference planner, independent of the C++ product.

Inputs are plain values — a parsed topology dict and config fields — so the
oracle shares no code with paper_2604_22228_b200.  Each function cites the
reference code it restates (paths relative to /root/reference/pkg/src/mpsim).
Parity pinned: tests/test_oracle.py checks it against tests/golden/*.json,
which tests/golden/gen_golden.py produced by importing the reference itself
(412 planner cases, LRU traces, parser cases); only tests/, smoke() and the
bench's CPU-baseline / reference legs use it, never the product.
"""

from __future__ import annotations

import hashlib
import math

HOST = "host"


def parse_topology(text: str) -> dict:
    """Minimal reader of the `.topo` schema (topology.py:164-240) for
    well-formed files: returns accelerator count and the direction channels
    in creation order (topology.py:112-120), sublinks aggregated (:226)."""
    section = None
    n = 0
    links, hostlinks = [], []
    name = "topology"
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("[") and line.endswith("]"):
            section = line[1:-1].strip().lower()
            continue
        f = line.split()
        if section is None and f[0] == "name":
            name = f[1]
        elif section == "device":
            n += 1
        elif section == "link":
            links.append((int(f[0]), int(f[1]), float(f[2]) * int(f[5]), f[4]))
        elif section == "hostlink":
            hostlinks.append((int(f[0]), HOST, float(f[1]), f[3]))
    chans: dict = {}
    order: list = []
    for a, b, bw, duplex in links + hostlinks:
        la, lb = str(a), str(b)
        if duplex == "full":
            fwd, rev = (f"{la}->{lb}", bw), (f"{lb}->{la}", bw)
            chans[(a, b)], chans[(b, a)] = fwd, rev
            order += [fwd, rev]
        else:
            sh = (f"{la}<->{lb}", bw)
            chans[(a, b)] = chans[(b, a)] = sh
            order.append(sh)
    return {"name": name, "n": n, "channels": chans, "order": order}


def py312_sum(xs) -> float:
    """builtin sum() of floats on CPython >= 3.12 (Neumaier), which the
    reference's `sum(weights)` (paths.py:149) evaluates to."""
    xs = list(xs)
    f, c = 0.0 + xs[0], 0.0
    for x in xs[1:]:
        t = f + x
        if abs(f) >= abs(x):
            c += (f - t) + x
        else:
            c += (x - t) + f
        f = t
    if c and math.isfinite(c):
        f += c
    return f


def plan_paths(topo: dict, src: int, dst: int, num_gpu_paths: int, host: bool,
               policy: str = "bandwidth_proportional") -> list[dict]:
    """paths.py:170-187 plan_paths + :153-167 _build_path_set + :144-150
    _assign_shares.  Returns [{kind, stage, hops: [channel ids], share}]."""
    if src == dst:
        raise ValueError("same device")
    cands = [d for d in range(topo["n"]) if d not in (src, dst)]
    need = num_gpu_paths - 1
    if need > len(cands):
        raise ValueError("staging")
    ch = topo["channels"]
    paths = [{"kind": "direct", "stage": None, "hops": [ch[(src, dst)]]}]
    for s in cands[:need]:
        paths.append({"kind": "gpu", "stage": s, "hops": [ch[(src, s)], ch[(s, dst)]]})
    if host:
        paths.append({"kind": "host", "stage": HOST, "hops": [ch[(src, HOST)], ch[(HOST, dst)]]})
    if policy == "equal":
        w = [1.0] * len(paths)
    else:
        w = [min(bw for _, bw in p["hops"]) for p in paths]  # paths.py:62-64 bottleneck
    total = py312_sum(w)
    for p, wi in zip(paths, w):
        p["share"] = wi / total
    return paths


def make_chunk_plan(shares: list[float], size: int, max_chunks: int) -> list[tuple]:
    """pipeline.py:51-78: nominal ceil(size*share/max_chunks) per active path,
    dealt round-robin until covered, last chunk truncated.
    Returns [(path_index, offset, length, seq)]."""
    active = [p for p, s in enumerate(shares) if s > 0.0]
    nominal = {p: math.ceil(size * shares[p] / max_chunks) for p in active}
    out, seq, off = [], [0] * len(shares), 0
    while off < size:
        for p in active:
            if off >= size:
                break
            ln = min(nominal[p], size - off)
            out.append((p, off, ln, seq[p]))
            seq[p] += 1
            off += ln
    return out


def lane_schedule(path_hops: list[int], chunks: list[tuple]) -> tuple[list, list]:
    """pipeline.py:102-125: lanes (path, hop) in path order; staged chunks add
    a (hop1 lane, pos) -> (hop2 lane, pos) dependency."""
    lane_id = {}
    for p, nh in enumerate(path_hops):
        for h in range(nh):
            lane_id[(p, h)] = len(lane_id)
    members = {l: [] for l in lane_id.values()}
    deps = []
    for cid, (p, _, _, _) in enumerate(chunks):
        if path_hops[p] == 1:
            members[lane_id[(p, 0)]].append(cid)
        else:
            l1, l2 = lane_id[(p, 0)], lane_id[(p, 1)]
            members[l1].append(cid)
            members[l2].append(cid)
            pos = len(members[l1]) - 1
            deps.append(((l1, pos), (l2, pos)))
    lanes = [(lid, p, h, members[lid]) for (p, h), lid in lane_id.items()]
    return lanes, deps


def graph_dump(paths: list[dict], chunks: list[tuple], src: int, dst: int) -> str:
    """graph.py:91-118 build_graph + :83-88 dump."""
    lines, edges, nid = [], [], 0
    for p, off, ln, _ in chunks:
        path = paths[p]
        if path["kind"] == "direct":
            lines.append(f"node {nid} direct {src}->{dst} {off} {ln}")
            nid += 1
        else:
            st = path["stage"]
            lines.append(f"node {nid} stage_hop1 {src}->{st} {off} {ln}")
            lines.append(f"node {nid + 1} stage_hop2 {st}->{dst} {off} {ln}")
            edges.append(f"edge {nid} {nid + 1}")
            nid += 2
    return "\n".join(lines + edges) + "\n"


def digest(num_gpu_paths, host, max_chunks, graph_mode, policy, src, dst, paths) -> str:
    """graph.py:132-138 _digest: sha256 of the repr of the config+path tuple."""
    tup = (num_gpu_paths, host, max_chunks, graph_mode, policy, str(src), str(dst),
           tuple((p["kind"], None if p["stage"] is None else str(p["stage"]), p["share"],
                  tuple(cid for cid, _ in p["hops"])) for p in paths))
    return hashlib.sha256(repr(tup).encode()).hexdigest()


class LRU:
    """graph.py:154-186 GraphCache ordering: hit -> move to end; miss ->
    insert, evict the oldest while over capacity."""

    def __init__(self, capacity: int):
        self.capacity = capacity
        self.order: list = []

    def access(self, key) -> bool:
        hit = key in self.order
        if hit:
            self.order.remove(key)
        self.order.append(key)
        while len(self.order) > self.capacity:
            self.order.pop(0)
        return hit
