import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
from paper_2604_22228_b200.tuner import tune_engines, measure_makespan
MiB = 1 << 20
text = mesh_text("x", 2, 3.2e12, 1, 2e-6, 12e9, 1e-5, "full")
big = torch.empty(64 * MiB, dtype=torch.uint8, device="cuda"); out = torch.empty_like(big)
st = torch.cuda.Stream()
def probe(tag, e, cfg):
    for n in (4 * MiB, 16 * MiB):
        t = measure_makespan(e, cfg, n, big[:n], out[:n], st, reps=20)
        t0 = time.perf_counter()
        for _ in range(200): e.send(big[:n], out[:n], n, cfg, stream=st, src_dev=0, dst_dev=1)
        host = (time.perf_counter() - t0) / 200 * 1e6
        torch.cuda.synchronize()
        print(json.dumps({"tag": tag, "n": n, "us_per_msg": t * 1e6, "host_us": host,
                          "launch_us": e.stats().launch_us, "opts": {k: v for k, v in e.options().items() if k in ("direct_engine", "host_engine")}}), flush=True)
single = PathConfig(max_chunks=1, graph_mode=True)
e = Engine(load_topology(text), [0, 0]); e.configure(direct="ce"); probe("fresh_ce", e, single); e.close()
a = Engine(load_topology(text), [0, 0])
rules, trials = tune_engines(a, [1 << 20, 4 * MiB, 16 * MiB, 64 * MiB], reps=5)
print(rules)
probe("after_tune_engines_nopolicy", a, single)
a.set_size_policy(rules)
probe("with_policy", a, single)
a.set_size_policy([])
a.configure(direct="ce", host="ce")
probe("policy_cleared_ce", a, single)
