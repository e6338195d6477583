"""Randomised API-level soak: random sequences of the calls a user makes —
send (graph / streamed, several path configs), send_many windows, prepared
sends, recv on another stream, sends captured into the caller's own CUDA
graph and replayed, traced sends, cache clears, engine reconfiguration
(host engine, PDL level, copy kernel, schedule) and topology changes, syncs
— on several streams of one engine, with every buffer pair's destination checked byte-exact at
each sync point (destinations are re-poisoned after each check, so a stale
or missing delivery shows).  MP_API_FUZZ_OPS sets the length (default 120;
a 2000-op soak is in profiles/)."""

import os
import random

import numpy as np
import pytest

from oracle import transfer as ot

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MiB = 1 << 20


def test_random_api_sequences_stay_byte_exact():
    from paper_2604_22228_b200 import Engine, EngineError, PathConfig, load_topology, mesh_text
    rng = random.Random(int(os.environ.get("MP_API_FUZZ_SEED", "20261017")))
    ops = int(os.environ.get("MP_API_FUZZ_OPS", "120"))
    eng = Engine(load_topology(mesh_text("fz", 4, 2e12, 1, 2e-6, 30e9, 1e-5, "full")), [0] * 4)
    cfgs = [PathConfig(1, False, 1, True), PathConfig(1, True, 8, True), PathConfig(3, True, 4, True),
            PathConfig(2, True, 3, False), PathConfig(1, False, 4, False), PathConfig(2, False, 8, True,
                                                                                   cache_capacity=3)]
    sizes = [1, 4095, 64 * 1024 + 3, MiB + 17, 5 * MiB + 1, 24 * MiB + 9, 70 * MiB + 5]
    pairs = []
    for i, n in enumerate(sizes):
        data = ot.pattern(n, seed=500 + i)
        src = torch.from_numpy(data).to("cuda:0")
        pairs.append([src, torch.bitwise_not(src), n, data])
    streams = [torch.cuda.Stream() for _ in range(3)] + [torch.cuda.current_stream()]
    # pre-warm: every pair x config and the largest send_many window per
    # config, so the staging arenas reach their final size before anything is
    # captured (arena growth drops the cache, and with it captured graphs)
    big4 = sorted(range(len(pairs)), key=lambda j: -pairs[j][2])[:4]
    for cfg in cfgs:
        for src, dst, n, _ in pairs:
            eng.send(src, dst, n, cfg, src_dev=0, dst_dev=1)
        eng.send_many([(pairs[j][0], pairs[j][1], pairs[j][2], 0, 1) for j in big4], cfg)
    torch.cuda.synchronize()
    eng.sync()
    sent = [False] * len(pairs)        # delivered since the last poison
    prepared = {}
    graphs = []                        # (CUDAGraph, pair indices)
    log = []

    def check_and_poison():
        torch.cuda.synchronize()
        eng.sync()
        for k, (src, dst, n, data) in enumerate(pairs):
            if sent[k]:
                got = dst.cpu().numpy()
                assert np.array_equal(got, data), f"pair {k} ({n} B) after ops {log[-12:]}"
        for k, p in enumerate(pairs):
            p[1].copy_(torch.bitwise_not(p[0]))
            sent[k] = False
        torch.cuda.synchronize()

    for step in range(ops):
        op = rng.choices(["send", "many", "prepared", "recv", "capture", "replay", "trace", "clear", "check",
                          "configure", "topology"],
                         weights=[30, 8, 8, 6, 4, 6, 2, 2, 10, 2, 1])[0]
        k = rng.randrange(len(pairs))
        c = rng.randrange(len(cfgs))
        s = rng.choice(streams)
        src, dst, n, _ = pairs[k]
        log.append((step, op, k, c))

        def do():
            if op == "send":
                eng.send(src, dst, n, cfgs[c], stream=s, src_dev=0, dst_dev=1)
                sent[k] = True
            elif op == "many":
                ks = rng.sample(range(len(pairs)), rng.randint(1, 4))
                eng.send_many([(pairs[j][0], pairs[j][1], pairs[j][2], 0, 1) for j in ks], cfgs[c], stream=s)
                for j in ks:
                    sent[j] = True
            elif op == "prepared":
                key = (k, c, streams.index(s))
                if key not in prepared:
                    prepared[key] = eng.prepare(src, dst, n, cfgs[c], stream=s, src_dev=0, dst_dev=1)
                prepared[key]()
                sent[k] = True
            elif op == "recv":
                eng.recv(dst, stream=s)
            elif op == "capture":
                cs = torch.cuda.Stream()
                for attempt in range(2):
                    torch.cuda.synchronize()
                    g = torch.cuda.CUDAGraph()
                    try:
                        with torch.cuda.graph(g, stream=cs):
                            eng.send(src, dst, n, cfgs[c], stream=cs, src_dev=0, dst_dev=1)
                    except EngineError as exc:  # evicted since (or never sent): refused, as documented
                        assert "must hit the plan cache" in str(exc) and attempt == 0, exc
                        eng.send(src, dst, n, cfgs[c], stream=s, src_dev=0, dst_dev=1)
                        sent[k] = True
                        continue
                    graphs.append((g, k))
                    break
            elif op == "replay" and graphs:
                g, gk = rng.choice(graphs)
                torch.cuda.synchronize()  # a captured send is ordered by the caller
                g.replay()
                torch.cuda.synchronize()
                sent[gk] = True
            elif op == "trace" and n >= 4096:
                torch.cuda.synchronize()
                eng.trace(src, dst, n, cfgs[c], 0, 1)
                sent[k] = True
            elif op == "clear":
                graphs.clear()  # a captured graph points into the cached programs' tables
                eng.clear_cache()
                prepared.clear()
            elif op == "check":
                check_and_poison()
            elif op in ("configure", "topology"):  # both drop the cache (and so captured graphs)
                graphs.clear()
                if op == "configure":
                    eng.configure(host=rng.choice(["sm", "ce", "auto"]), pdl=rng.randint(0, 3),
                                  copy=rng.choice(["tma", "vec"]), sched=rng.choice(["auto", "dynamic"]))
                else:
                    eng.set_topology(load_topology(mesh_text("fz", 4, rng.choice([2e12, 7.5e11]), 1, 2e-6,
                                                             rng.choice([1e9, 30e9, 55e9]), 1e-5, "full")))

        try:
            do()
        except EngineError as exc:
            # documented remedy: a send that must grow the staging arenas is
            # refused while captured programs exist — drop the graphs, clear
            # the cache, retry
            assert "larger staging arenas" in str(exc), exc
            graphs.clear()
            eng.clear_cache()
            do()
    check_and_poison()
    eng.close()
