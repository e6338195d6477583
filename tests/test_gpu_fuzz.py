"""Randomised GPU parity: random sizes, buffer offsets, path counts, chunk
counts, share policies, engines (copy kernel, CE/SM per path type, tile
schedule, peer launch path), cache capacities, graph/streamed modes and
repeated sends of one entry — every delivered byte equal to the oracle's
execution of the same (oracle-checked) plan.  Stresses the flag handoff,
tile cuts, head/tail peeling, claim counters and cache replays/evictions.
MP_FUZZ_ITERS sets the iteration count (default 60; soak runs use more)."""

import os
import random

import numpy as np
import pytest

from oracle import planner as op
from oracle import transfer as ot

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_random_transfers_are_byte_exact():
    import paper_2604_22228_b200 as mp
    rng = random.Random(20261017)
    # a bandwidth-sized host share (flag-handed-off hop1 / hop2 tiles, CE
    # groups) and a calibrated-small one (roundtrip tiles, helper warps)
    texts = {hb: mp.mesh_text("fz", 5, 2.5e12, 1, 2e-6, hb, 1e-5, "full") for hb in (40e9, 1e9)}
    otopos = {hb: op.parse_topology(t) for hb, t in texts.items()}
    engines = {}
    big_src = torch.empty((100 << 20) + 64, dtype=torch.uint8, device="cuda:0")
    big_dst = torch.empty_like(big_src)
    for it in range(int(os.environ.get("MP_FUZZ_ITERS", 60))):
        knobs = (rng.choice(["tma", "vec"]), rng.choice(["sm", "ce"]), rng.choice(["sm", "ce"]),
                 rng.choice(["sm", "ce", "auto"]), rng.choice(["auto", "dynamic"]), rng.choice([0, -1]),
                 rng.choice([40e9, 1e9]))
        otopo = otopos[knobs[6]]
        if knobs not in engines:
            eng = mp.Engine(mp.load_topology(texts[knobs[6]]), [0] * 5)
            eng.configure(copy=knobs[0], direct=knobs[1], relay=knobs[2], host=knobs[3],
                          sched=knobs[4], tma_peer=knobs[5])
            if knobs[0] == "tma":
                eng.configure(ctas_per_sm=1, threads=128)
            engines[knobs] = eng
        eng = engines[knobs]
        size = rng.choice([rng.randint(1, 4096), rng.randint(1, 1 << 20),
                           rng.randint(1 << 20, 24 << 20), rng.randint(24 << 20, 100 << 20)])
        so, do = rng.randint(0, 63), rng.randint(0, 63)
        g = rng.randint(1, 4)
        host = rng.random() < 0.5
        k = rng.choice([1, 2, 3, 4, 7, 8, 16])
        pol = rng.choice(["equal", "bandwidth_proportional"])
        graph = rng.random() < 0.5
        cfg = mp.PathConfig(num_gpu_paths=g, host_path_enabled=host, max_chunks=k,
                            graph_mode=graph, share_policy=pol,
                            cache_capacity=rng.choice([1, 2, 16]))
        paths = op.plan_paths(otopo, 0, 1, g, host, pol)
        chunks = op.make_chunk_plan([p["share"] for p in paths], size, k)
        src, dst = big_src[so:so + size], big_dst[do:do + size]
        for rep in range(rng.choice([1, 1, 2, 3])):  # repeats replay the cached entry
            data = ot.pattern(size, seed=1000 * it + rep)
            src.copy_(torch.from_numpy(data))
            dst.copy_(torch.bitwise_not(src))
            eng.send(src, dst, size, cfg, src_dev=0, dst_dev=1)
            eng.sync()
            _, done = eng.last_plan()
            assert [(c.path_index, c.offset, c.length, c.seq) for c in done] == chunks
            expect = np.empty_like(data)
            ot.run(data, expect, [p["kind"] for p in paths], chunks, threads=4)
            got = dst.cpu().numpy()
            assert np.array_equal(got, expect), (it, rep, knobs, size, so, do, g, host, k, pol,
                                                 graph)
    for eng in engines.values():
        eng.close()


def test_random_programs_are_byte_exact():
    """Random send_many programs (1-64 transfers, 1 B - 1 MiB each, unaligned
    source/destination offsets, direct or direct+host, graph or streamed,
    resent through prepare_many): the small-message kernel's many-segment
    tables, the dynamic tables and the per-transfer interleaving all
    deliver every byte."""
    import paper_2604_22228_b200 as mp
    rng = random.Random(20261018)
    eng = mp.Engine(mp.load_topology(mp.mesh_text("pf", 2, 2.5e12, 1, 2e-6, 40e9, 1e-5, "full")),
                    [0, 0])
    for it in range(int(os.environ.get("MP_FUZZ_ITERS", 60)) // 2):
        n = rng.choice([1, 2, 5, 16, 37, 64])
        cap = rng.choice([4096, 65536, 1 << 20])
        sizes = [rng.randint(1, cap) for _ in range(n)]
        offs = [(rng.randint(0, 31), rng.randint(0, 31)) for _ in range(n)]
        srcs = [torch.empty(s + 32, dtype=torch.uint8, device="cuda:0") for s in sizes]
        dsts = [torch.empty(s + 32, dtype=torch.uint8, device="cuda:0") for s in sizes]
        datas = []
        xs = []
        for i, (s, (so, do)) in enumerate(zip(sizes, offs)):
            d = ot.pattern(s, seed=7000 * it + i)
            datas.append(d)
            srcs[i][so:so + s].copy_(torch.from_numpy(d))
            xs.append((srcs[i][so:so + s], dsts[i][do:do + s], s, 0, 1))
        cfg = mp.PathConfig(num_gpu_paths=1, host_path_enabled=rng.random() < 0.3,
                            max_chunks=rng.choice([1, 2, 4]), graph_mode=rng.random() < 0.7)
        post = eng.prepare_many(xs, cfg)
        for rep in range(rng.choice([1, 2])):
            for (_, dv, _, _, _), d in zip(xs, datas):  # every unwritten byte mismatches
                dv.copy_(torch.bitwise_not(torch.from_numpy(d)))
            post()
            eng.sync()
            for (_, dv, _, _, _), d in zip(xs, datas):
                assert np.array_equal(dv.cpu().numpy(), d), (it, rep, n, sizes, offs, cfg)
    eng.close()
