"""Markdown tables for DESIGN.md §5 from a bench JSON line (default
profiles/r01_bench.json): the osu_bw-style sweep and the posting windows."""
import json
import sys

d = json.loads(open(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_bench.json")
               .read().strip().splitlines()[-1])
KiB, MiB = 1 << 10, 1 << 20


def label(n):
    return f"{n // MiB} MiB" if n >= MiB else f"{n // KiB} KiB"


def fmt(x):
    return f"{x:.3g}" if x < 10 else f"{x:.0f}"


rows = {r["bytes"]: r for r in d["sweep"]}
prep = "sm_single_prepared" in d["sweep"][0]
print("| bytes | CE single | SM single |" + (" SM single, prepared |" if prep else "")
      + " direct+host k=8 (graph) | tuned |")
print("|---|---|---|---|---|" + ("---|" if prep else ""))
for b in (4 * KiB, 64 * KiB, MiB, 4 * MiB, 16 * MiB, 32 * MiB, 128 * MiB, 512 * MiB):
    r = rows[b]
    print(f"| {label(b)} | {fmt(r['ce_single'])} | {fmt(r['sm_single'])} | "
          + (f"{fmt(r['sm_single_prepared'])} | " if prep else "")
          + f"{fmt(r['multi_graph'])} | {fmt(r['tuned'])} |")
w = d.get("windows")
if w:
    print()
    sizes = sorted({int(s) for per in w["gbs"].values() for s in per})
    print("| W | " + " | ".join(label(s) for s in sizes) + " |")
    print("|---|" + "---|" * len(sizes))
    for win, per in w["gbs"].items():
        cells = []
        for s in sizes:
            v = per[str(s)]
            cells.append(f"{fmt(v['single'])} / {fmt(v['multi_k8'])} / {fmt(v['baseline'])}")
        print(f"| {win} | " + " | ".join(cells) + " |")
    if any("single_program" in v for per in w["gbs"].values() for v in per.values()):
        print()
        print("| W | " + " | ".join(label(s) for s in sizes) + " |")
        print("|---|" + "---|" * len(sizes))
        for win, per in w["gbs"].items():
            cells = []
            for s in sizes:
                v = per[str(s)]
                cells.append(f"**{fmt(v['single_program'])}** / {fmt(v['single'])} / "
                             f"{fmt(v['baseline_distinct_buffers'])}"
                             if "single_program" in v else "—")
            print(f"| {win} | " + " | ".join(cells) + " |")
