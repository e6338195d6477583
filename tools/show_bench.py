"""Print the key fields of a bench.py JSON line (default gpurun_out/bench.json)."""
import json
import sys

d = json.loads(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.json")
               .read().strip().splitlines()[-1])
for k in ["value", "ms_per_step", "roofline", "path_roofline", "e2e", "gpu_launches", "clocks",
          "graph", "cpu_baseline", "reference_cpu_path_us"]:
    v = d.get(k)
    if isinstance(v, dict):
        v = {a: b for a, b in v.items() if a not in ("calibration", "probe")}
    print(k, v)
for r in d.get("sweep") or []:
    print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()})
for r in d.get("relay_sweep") or []:
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()})
for r in d.get("lifecycle") or []:
    print(r["bytes"], "replay", r["replay"], "stream", r["stream"])
w = d.get("windows")
if w:
    for win, per in w["gbs"].items():
        print("W", win, {int(k) >> 10: {a: round(b, 1) for a, b in v.items()} for k, v in per.items()})
