"""Summarise tools/ncu_paths.sh's CSV: per launch, achieved GB/s over each
link the transfer kernel drives — HBM (read + write), PCIe (host-staged
hops; ncu counts it at 512-byte granularity) and NVLink TX/RX (peer paths,
>= 2 GPUs) — against the link peaks (NVLink 900 GB/s per direction nominal,
770 measured peer copy per B200_PROFILING.md; PCIe Gen5 x16 64 nominal).

    python tools/ncu_paths_summary.py gpurun_out/x_ncu.csv gpurun_out/x_ncu.json
"""
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "second": 1}


def main(src, out):
    rows = [r for r in csv.reader(open(src)) if r and not r[0].startswith("==")]
    head = rows[0]
    col = {k: i for i, k in enumerate(head)}
    launches = {}
    for r in rows[1:]:
        if len(r) != len(head) or not r[col["ID"]].isdigit():
            continue
        lid = int(r[col["ID"]])
        d = launches.setdefault(lid, {"kernel": r[col["Kernel Name"]], "device": r[col.get("Device", 0)]})
        try:
            v = float(r[col["Metric Value"]].replace(",", "")) * UNIT.get(r[col["Metric Unit"]], 1)
        except ValueError:
            continue
        d[r[col["Metric Name"]]] = v
    res = []
    for lid, d in sorted(launches.items()):
        t = d.get("gpu__time_duration.sum")
        if not t:
            continue
        g = lambda k: d.get(k, 0.0)  # noqa: E731
        e = {"id": lid, "kernel": d["kernel"][:60], "device": d["device"], "us": t * 1e6,
             "hbm_gbs": (g("dram__bytes_read.sum") + g("dram__bytes_write.sum")) / t / 1e9,
             "pcie_read_gbs": g("pcie__read_bytes.sum") / t / 1e9,
             "pcie_write_gbs": g("pcie__write_bytes.sum") / t / 1e9,
             "pcie_bytes": g("pcie__read_bytes.sum") + g("pcie__write_bytes.sum"),
             "nvl_tx_gbs": g("nvltx__bytes.sum") / t / 1e9,
             "nvl_rx_gbs": g("nvlrx__bytes.sum") / t / 1e9,
             "nvl_tx_user_bytes": g("nvltx__bytes_data_user.sum"),
             "nvl_rx_user_bytes": g("nvlrx__bytes_data_user.sum")}
        e["nvl_tx_frac_of_900"] = e["nvl_tx_gbs"] / 900.0
        e["nvl_tx_frac_of_770"] = e["nvl_tx_gbs"] / 770.0
        res.append(e)
    summary = {"source": src, "peaks": {"nvlink_nominal_gbs": 900, "nvlink_measured_peer_gbs": 770,
                                        "pcie_gen5_x16_nominal_gbs": 64}, "launches": res}
    with open(out, "w") as fh:
        json.dump(summary, fh, indent=1)
    for e in res:
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in e.items()}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
