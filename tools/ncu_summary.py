"""Summarise an ncu --set full capture of transfer_kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/transfer_512m.ncu-rep profiles/transfer_kernel_ncu.json

Writes the per-launch DRAM traffic that bench.py reports as roofline.traffic
plus the headline throughput / occupancy metrics.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3, "ns": 1e-9,
         "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, name in KEYS.items():
            if k in head:
                i = head.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * SCALE.get(units[i], 1)
        d["kernel"] = r[head.index("Kernel Name")] if "Kernel Name" in head else ""
        res.append(d)
    summary = dict(res[0])
    summary["source"] = rep
    summary["launches"] = res
    with open(out, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "launches"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
