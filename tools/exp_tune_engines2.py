import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_22228_b200 import Engine, PathConfig, load_topology
from paper_2604_22228_b200.tuner import measure_makespan, tune_engines
MiB = 1 << 20
text = open("topologies/b200_loopback.topo").read()
sizes = [MiB // 2, MiB, 2 * MiB, 4 * MiB, 8 * MiB, 16 * MiB]
e = Engine(load_topology(text), [0, 0])
r, tr = tune_engines(e, sizes, reps=50)
print("tune_engines", [round(t["seconds"] * 1e6, 2) for t in tr if t["path"] == "direct" and t["engine"] == "sm"])
big = torch.empty(sizes[-1], dtype=torch.uint8, device="cuda:0"); out = torch.empty_like(big)
st = torch.cuda.Stream(device=0)
e.set_size_policy([])
for name in ("sm", "ce"):
    e.configure(direct=name)
    print(name, [round(measure_makespan(e, PathConfig(max_chunks=1, graph_mode=True), s, big[:s], out[:s], st, 50) * 1e6, 2) for s in sizes])
# inline copy with single = PathConfig(max_chunks=1, graph_mode=graph) where graph is a numpy bool?
from paper_2604_22228_b200.tuner import GRAPH_MODE
graph = "graph" == GRAPH_MODE
print("graph flag", graph, type(graph))
e.configure(direct="sm")
single = PathConfig(max_chunks=1, graph_mode=graph)
print("inline", [round(measure_makespan(e, single, s, big[:s], out[:s], st, 50) * 1e6, 2) for s in sizes])
print("opts", e.options())
