"""ORACLE (test infrastructure only): the multi-path transfer on host memory.

Executes a chunk plan exactly as the reference defines it — each Direct
chunk copied src -> dst, each staged chunk copied src -> staging (hop1) and
then staging -> dst (hop2), hop2 after hop1 (graph.py:108-117,
sim.py:182-191) — with numpy on CPU.  The resulting destination defines the
expected bytes for the GPU parity tests, and `run` is the CPU baseline of
bench.py (`cpu_baseline` / `--impl reference`).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

BLOCK = 4 << 20


def pattern(size: int, seed: int | None = None) -> np.ndarray:
    """SURVEY.md §8d synthetic input: byte[i] = ((i * 2654435761) >> 24) & 0xFF,
    or seeded random bytes."""
    if seed is not None:
        return np.random.default_rng(seed).integers(0, 256, size, dtype=np.uint8)
    i = np.arange(size, dtype=np.uint64)
    return ((i * np.uint64(2654435761)) >> np.uint64(24)).astype(np.uint8)


def run(src: np.ndarray, dst: np.ndarray, kinds: list[str], chunks: list[tuple],
        threads: int | None = None) -> None:
    """Move the plan's bytes: kinds[p] in {"direct","gpu","host"}; chunks are
    (path_index, offset, length, seq) in plan order."""
    staged = {p for p, k in enumerate(kinds) if k != "direct"}
    stage_off, base = {}, {}
    for p in staged:
        base[p] = 0
    for cid, (p, off, ln, _) in enumerate(chunks):
        if p in staged:
            stage_off[cid] = base[p]
            base[p] += ln
    stage = {p: np.empty(max(1, base[p]), dtype=np.uint8) for p in staged}

    tasks = []
    for cid, (p, off, ln, _) in enumerate(chunks):
        for b in range(0, ln, BLOCK):
            tasks.append((cid, p, off + b, min(BLOCK, ln - b), b))

    def work(t):
        cid, p, off, ln, b = t
        if p in staged:
            so = stage_off[cid] + b
            stage[p][so:so + ln] = src[off:off + ln]   # hop1
            dst[off:off + ln] = stage[p][so:so + ln]   # hop2, after hop1
        else:
            dst[off:off + ln] = src[off:off + ln]

    threads = threads or os.cpu_count() or 1
    if threads == 1:
        for t in tasks:
            work(t)
    else:
        with ThreadPoolExecutor(threads) as pool:
            list(pool.map(work, tasks))
