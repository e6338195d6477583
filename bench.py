"""Benchmark: GPU0->GPU1 multi-path transfer bandwidth (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 (the driver's default): one visible B200, so the transfer runs in
loopback — logical GPU0 and GPU1 of the topology both map to cuda:0.  The
direct path is then an HBM->HBM copy by the SM transfer kernel and the
host-staged path a real D2H + H2D over PCIe Gen5 through pinned memory; the
planner, graph cache and engine are exactly the multi-GPU ones.
A step = one osu_bw window: --window (64) back-to-back messages of --size
bytes (default 512 MiB, larger than L2, so no L2 flush is needed) sent with
the cached CUDA graph.  `value` is K*W*S / device time of K steps; `e2e`
times the same windows through the public API from HOST memory: every step's
input message is copied H2D from pinned memory (double-buffered with the
previous step's sends) and the step's result (an int64 checksum of the
delivered buffer) is read back D2H — the host-staged hops run on the
mechanism (copy engine or SM) an untimed calibration of this pipeline
picks; `e2e.fresh_message` re-fetches every
message from host memory (the PCIe-bound extreme).

--impl reference: the reference's CPU implementation of the path — the
oracle restatement (oracle/transfer.py, the reference package itself never
moves bytes) — timed on the host cores on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MiB = 1 << 20
METRIC = "GPU0→GPU1 bandwidth GB/s vs msg size (1KB–512MB), multi-path vs single-path"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=512 * MiB)
    ap.add_argument("--chunks", type=int, default=8)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--window", type=int, default=64, help="messages per step (osu_bw window)")
    ap.add_argument("--quick", action="store_true",
                    help="headline only: no sweep, lifecycle or CPU baseline (for ncu)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return d.get("hbm_gbs", 6650.0), "measured"
    except OSError:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._ready = threading.Event()
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:  # NVML directly: ~0.1 ms per sample instead of ~200 ms per nvidia-smi call
            import pynvml as nv
            nv.nvmlInit()
            try:  # the CUDA ordinal's own GPU, by PCI address (CUDA_VISIBLE_DEVICES-proof)
                import torch
                p = torch.cuda.get_device_properties(self.index)
                h = nv.nvmlDeviceGetHandleByPciBusId(
                    f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0")
            except Exception:
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            while not self._stop.is_set():
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), str(mx)]
                                    + ["Active" if r & b else "Not Active" for b in bits])
                self._ready.set()
                self._stop.wait(0.01)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        self._ready.wait(10.0)  # first sample taken before the timed region starts
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "model": model}


# ---------------------------------------------------------------------------
# reference arm: the CPU implementation of the path (oracle port)
# ---------------------------------------------------------------------------
def cpu_transfer_rate(size, chunks, budget_s, threads, kinds_shares=None):
    """Bytes/s of the oracle's host-memory multi-path transfer (planner + copies)."""
    import numpy as np

    from oracle import planner as op
    from oracle import transfer as ot
    topo = op.parse_topology(loopback_topo_text(3000e9, 50e9))
    paths = op.plan_paths(topo, 0, 1, 1, True)
    src = ot.pattern(size)
    dst = np.empty_like(src)
    t0 = time.perf_counter()
    n = 0
    while True:
        plan = op.make_chunk_plan([p["share"] for p in paths], size, chunks)
        ot.run(src, dst, [p["kind"] for p in paths], plan, threads=threads)
        n += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    assert np.array_equal(src, dst)
    return n * size / dt, n


def run_reference(args, rank):
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    size = args.size
    # warm-up then K timed steps, each one message through the CPU path
    import numpy as np

    from oracle import planner as op
    from oracle import transfer as ot
    world = max(1, args.gpus)
    if world > 1:  # the N > 1 arm's workload: direct + (N - 2) GPU relays, no host path
        topo = op.parse_topology(loopback_topo_text(900e9, 64e9, n=world))
        paths = op.plan_paths(topo, 0, 1, world - 1, False)
    else:
        topo = op.parse_topology(loopback_topo_text(3000e9, 50e9))
        paths = op.plan_paths(topo, 0, 1, 1, True)
    src = ot.pattern(size)
    dst = np.empty_like(src)
    for _ in range(args.warmup):
        plan = op.make_chunk_plan([p["share"] for p in paths], size, args.chunks)
        ot.run(src, dst, [p["kind"] for p in paths], plan, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        plan = op.make_chunk_plan([p["share"] for p in paths], size, args.chunks)
        ot.run(src, dst, [p["kind"] for p in paths], plan, threads=threads)
    dt = time.perf_counter() - t0
    assert np.array_equal(src, dst)
    gbs = args.steps * size / dt / 1e9
    sample = (f"{args.steps} x {size} B messages, "
              f"{'direct+host' if world == 1 else f'direct + {world - 2} relays'} plan, "
              f"{threads} threads, numpy")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args) if world == 1 else group_config(args, world),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": sample, **cpu_info()},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def group_config(args, world):
    """config of the N > 1 arm (run_group); the reference arm mirrors it."""
    return {"workload": f"GPU0->GPU1 {args.size} B messages, direct + {world - 2} GPU "
                        f"relays, max_chunks {args.chunks}, multi-process group mode "
                        "(CUDA IPC), cached graphs", "msg_bytes": args.size,
            "window": args.window, "relays": world - 2, "parallelism": f"n{world}",
            "l2": "inputs larger than L2"}


def loopback_topo_text(link_bw, host_bw, n=2):
    from paper_2604_22228_b200 import mesh_text
    return mesh_text("b200_loopback", n, link_bw, 1, 2e-6, host_bw, 10e-6, "full")


def workload_config(args):
    return {"workload": f"osu_bw-style GPU0->GPU1, {args.size} B messages, direct + host-staged "
                        f"multi-path, max_chunks {args.chunks}, cached CUDA-graph replay; N=1: "
                        "logical GPU0/GPU1 both on cuda:0 (loopback: direct = HBM copy, "
                        "host = PCIe Gen5 D2H+H2D)",
            "msg_bytes": args.size, "window": args.window, "max_chunks": args.chunks,
            "paths": "direct+host",
            "l2": "inputs larger than L2 (512 MiB > 126 MB)", "parallelism": f"n{args.gpus}"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def time_sends(torch, eng, cfg, src, dst, size, steps, warmup, stream, trials=3):
    """Seconds per message over `steps` back-to-back sends, best of `trials`
    (after >= 5 warm-up replays: a fresh graph's first launches are slow)."""
    for _ in range(max(5, warmup)):
        eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(trials):
        e0.record(stream)
        for _ in range(steps):
            eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / steps
        best = t if best is None else min(best, t)
    return best


def ncu_traffic():
    """dram bytes per launch of transfer_kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "transfer_kernel_ncu.json")) as fh:
            d = json.load(fh)
        return d["dram_bytes_read"] + d["dram_bytes_write"], d
    except (OSError, KeyError, ValueError):
        return None, None


def reference_cpu_path(topo_text, size, chunks):
    """The unmodified reference's per-message CPU path, timed on one host core."""
    ref = os.path.join(ROOT, "baseline", "_ref", "mpsim")
    if not os.path.isdir(ref):
        return {"unavailable": "baseline/_ref not installed"}
    import tempfile
    with tempfile.NamedTemporaryFile("w", suffix=".topo", delete=False) as fh:
        fh.write(topo_text)
    try:
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ref_cpu_path.py"),
                              fh.name, str(size), str(chunks)], capture_output=True, text=True,
                             timeout=300)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": str(exc)[:200]}
    finally:
        os.unlink(fh.name)


def run_ours(args, rank, world):
    import torch

    from paper_2604_22228_b200 import Engine, PathConfig
    from paper_2604_22228_b200.tuner import calibrate_host_bandwidth
    dev = rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    hbm_peak, peak_kind = peaks()
    size = args.size

    # 1. probe per-path bandwidths, then calibrate the host link's effective
    #    rate for the planner's .topo (SURVEY §8c protocol: repr() bandwidths)
    eng = Engine.loopback(2, dev)
    link_bw, _ = eng.probe_bandwidths(256 * MiB, 5, host_bytes=8 * MiB)
    m = dict(eng.last_probe["bulk"])
    m["host_staged_8MiB"] = eng.last_probe["host_share_sized"]["host_staged"]
    host_bw, topo, trials = calibrate_host_bandwidth(eng, link_bw, size, args.chunks,
                                                     name="b200_loopback")
    topo_text = loopback_topo_text(link_bw, host_bw)
    cfg = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=args.chunks,
                     graph_mode=True)
    src = torch.empty(size, dtype=torch.uint8, device=f"cuda:{dev}")
    dst = torch.empty_like(src)
    src.copy_(torch.randint(0, 256, (size,), dtype=torch.uint8,
                            generator=torch.Generator().manual_seed(20261017)).to(src.device))
    dst.copy_(torch.bitwise_not(src))
    stream = torch.cuda.Stream(device=dev)

    # the benchmarked configuration delivers every byte (plan parity against the
    # oracle is the tests' job: tests/test_gpu_transfer.py)
    eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    eng.sync()
    torch.cuda.synchronize()
    assert torch.equal(src, dst), "delivered bytes differ"
    _, chunks = eng.last_plan()
    direct_bytes = sum(c.length for c in chunks if c.path_index == 0)
    host_bytes = size - direct_bytes

    # 2. headline: K steps, each one osu_bw window of W back-to-back messages
    #    (cached-graph replay), device time, clocks sampled during the region
    W = args.window
    for _ in range(args.warmup * W):
        eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps * W):
            eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
        e1.record(stream)
        torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    st = eng.stats()
    if world > 1:
        tt = torch.tensor([t], device=f"cuda:{dev}")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt)
    value = world * args.steps * W * size / t / 1e9
    single_t = time_sends(torch, eng, PathConfig(max_chunks=1, graph_mode=True), src, dst,
                          size, args.steps * 4, 3, stream)

    # 3. dominant kernel: transfer_kernel average launch duration — CUDA events
    #    on its own stream around back-to-back launches of this send's program
    #    (and, for reference, around single streamed-mode launches)
    cfg_s = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=args.chunks,
                       graph_mode=False)
    kms = eng.kernel_bench(src, dst, size, cfg_s, 0, 1, reps=max(10, args.steps))
    ktimes = []
    eng.set_kernel_timing(True)
    for _ in range(5):
        eng.send(src, dst, size, cfg_s, stream=stream, src_dev=0, dst_dev=1)
        ktimes.append(eng.kernel_time_ms())
    eng.set_kernel_timing(False)
    kms_single = statistics.median(ktimes[1:])
    kernel_name = st.kernel
    k_alg_bytes = 2 * direct_bytes  # HBM read + write of the direct share
    achieved = k_alg_bytes / (kms / 1e3) / 1e9
    pcie = min(m["d2h"], m["h2d"])
    path_roofline = hbm_peak / 2 + pcie
    traffic, ncu = ncu_traffic()

    # 4. e2e through the public API with HOST buffers.  A step is the same
    #    osu_bw window as for `value`: its input message is copied H2D from
    #    pinned host memory, sent W times (osu_bw re-sends one buffer per
    #    window), and the step's result — an int64 checksum of the delivered
    #    buffer — is read back D2H.  Double-buffered: the H2D of step i+1's
    #    input (copy stream) overlaps the sends of step i; every step still
    #    moves its own input.  `fresh_message` is the stricter variant where
    #    EVERY message is fetched from host memory (bound by PCIe H2D).
    hsrc = torch.empty(size, dtype=torch.uint8, pin_memory=True)
    hsum = torch.empty(1, dtype=torch.int64, pin_memory=True)
    hsrc.copy_(src.cpu())
    want = int(src.sum(dtype=torch.int64))
    cur = torch.cuda.current_stream()
    cs = torch.cuda.Stream(device=dev)
    bufs = [src, torch.empty_like(src)]
    landed = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    for ev in consumed:
        ev.record(cur)

    def e2e_run(n, sends_per_input):
        for i in range(n):
            b = i % 2
            with torch.cuda.stream(cs):
                cs.wait_event(consumed[b])          # the sends of step i-2 read this buffer
                bufs[b].copy_(hsrc, non_blocking=True)
                landed[b].record(cs)
            cur.wait_event(landed[b])
            for _ in range(sends_per_input):
                eng.send(bufs[b], dst, size, cfg, stream=cur, src_dev=0, dst_dev=1)
            consumed[b].record(cur)
            hsum.copy_(dst.sum(dtype=torch.int64).view(1), non_blocking=True)

    def e2e_time(n, sends_per_input):
        e2e_run(2, sends_per_input)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(cur)
        cs.wait_event(c0)
        e2e_run(n, sends_per_input)
        c1.record(cur)
        torch.cuda.synchronize()
        assert int(hsum) == want
        return c0.elapsed_time(c1) / 1e3

    # The input's H2D shares PCIe with the host-staged path's H2D hops (and,
    # on copy engines, the same FIFO), so the host link's effective rate in
    # this pipeline is lower than in the headline windows: the host share and
    # the host-path mechanism are re-calibrated for the pipeline by a short
    # untimed run of every (mechanism, host bandwidth) pair — the same
    # measured-.topo protocol as `calibrate_host_bandwidth` — then the winner
    # is timed over the same K steps as `value`.
    from paper_2604_22228_b200 import load_topology
    e2e_steps = args.steps
    host_mech = eng.options()["host_engine"]
    calib = {}
    for mech in ("ce", "sm"):
        eng.configure(host=mech)
        for hbw in (0.125e9, 0.25e9, 0.5e9, 1e9, 2e9, 4e9, host_bw):
            eng.set_topology(load_topology(loopback_topo_text(link_bw, hbw)))
            calib[f"{mech}@{hbw / 1e9:g}"] = 3 * W * size / e2e_time(3, W) / 1e9
    best_key = max(calib, key=calib.get)
    e2e_mech, e2e_hbw = best_key.split("@")[0], float(best_key.split("@")[1]) * 1e9
    by_mech = {}
    for mech in ("ce", "sm"):
        eng.configure(host=mech)
        # each mechanism at its own best pipeline host share
        k = max((c for c in calib if c.startswith(mech)), key=calib.get)
        eng.set_topology(load_topology(loopback_topo_text(link_bw, float(k.split("@")[1]) * 1e9)))
        by_mech[mech] = e2e_steps * W * size / e2e_time(e2e_steps, W) / 1e9
    e2e, e2e_sm = by_mech[e2e_mech], by_mech["sm"]
    eng.configure(host=e2e_mech)
    eng.set_topology(load_topology(loopback_topo_text(link_bw, e2e_hbw)))
    eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    torch.cuda.synchronize()
    e2e_host_bytes = size - sum(c.length for c in eng.last_plan()[1] if c.path_index == 0)
    # the same pipeline with the host path disabled: under a PCIe link
    # saturated by the input upload, the host hops' PCIe round trips (hop1's
    # system-scope release, hop2's mapped reads) queue behind the input DMA
    cfg_direct = PathConfig(num_gpu_paths=1, host_path_enabled=False, max_chunks=args.chunks,
                            graph_mode=True)
    cfg_e2e, cfg = cfg, cfg_direct
    e2e_direct = e2e_steps * W * size / e2e_time(e2e_steps, W) / 1e9
    cfg = cfg_e2e
    fresh_n = max(4, args.steps // 2)
    e2e_fresh = fresh_n * size / e2e_time(fresh_n, 1) / 1e9
    eng.configure(host="sm" if host_mech == 0 else "ce")
    eng.set_topology(load_topology(topo_text))

    # 5. osu_bw-style sweep and a measured tuning table
    sweep, tuning = [], None
    if not (args.no_sweep or args.quick):
        sweep, tuning = run_sweep(torch, eng, topo_text, dev, stream)

    # 6. lifecycle (BASELINE config 5) and the reference's CPU path
    lifecycle = None if args.quick else run_lifecycle(torch, eng, dev, stream)
    windows = None if args.quick else run_windows(eng)
    relays = None if args.quick else run_relay_sweep(torch, dev, size, link_bw, host_bw,
                                                     hbm_peak / 2, pcie)
    cpu, ref_cpu = None, None
    if rank == 0 and not args.quick:
        cpu_rate, nmsg = cpu_transfer_rate(size, args.chunks, 10.0, len(os.sched_getaffinity(0)))
        cpu = {"value": cpu_rate / 1e9, "unit": "GB/s", "cores": len(os.sched_getaffinity(0)),
               "kind": "port", "sample": f"{nmsg} x {size} B messages, direct+host plan, "
                                         "oracle/transfer.py numpy copies, ~10 s", **cpu_info()}
        ref_cpu = reference_cpu_path(topo_text, size, args.chunks)
    if rank != 0:
        return
    out = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded random bytes, seed 20261017)",
        "config": workload_config(args),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "kernel": kernel_name, "kernel_ms": kms,
                     "kernel_ms_single_launch": kms_single,
                     "alg_bytes_per_launch": k_alg_bytes, "peak_kind": peak_kind,
                     "traffic_source": ncu and ncu.get("source")},
        "path_roofline": {"R_gbs": path_roofline, "frac": value / path_roofline,
                          "hbm_copy_gbs": hbm_peak / 2, "pcie_gbs": pcie, "probe": m,
                          # loopback: a host-staged byte is read from and written to
                          # the same HBM as a direct byte, so PCIe cannot add to an
                          # HBM-bound copy; the physical ceiling is the HBM copy rate
                          "R_loopback_hbm_gbs": hbm_peak / 2,
                          "frac_loopback_hbm": value / (hbm_peak / 2),
                          "direct_bytes": direct_bytes, "host_bytes": host_bytes,
                          "host_bw_calibrated": host_bw, "link_bw": link_bw,
                          "host_engine": "sm" if eng.options()["host_engine"] == 0 else "ce",
                          "calibration": trials,
                          "single_path_sm_gbs": size / single_t / 1e9},
        "cpu_baseline": cpu,
        "reference_cpu_path_us": ref_cpu,
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": size,
                "d2h_bytes_per_step": 8, "steps": e2e_steps,
                "step": f"one osu_bw window: H2D of the {size} B input from pinned host "
                        f"memory, {W} sends of it, D2H of an int64 checksum of the "
                        "delivered buffer; next step's H2D overlaps (double buffer)",
                "host_engine": e2e_mech, "host_bw_calibrated": e2e_hbw,
                "host_bytes_per_message": e2e_host_bytes,
                "calibration_gbs": calib,
                "sm_host_path": {"value": e2e_sm, "unit": "GB/s",
                                 "note": "host-staged path on the SM kernels (mapped pinned "
                                         "memory): no copy-engine queueing behind the input "
                                         "H2D"},
                "ce_host_path": {"value": by_mech["ce"], "unit": "GB/s",
                                 "note": "host-staged path on copy engines: its D2H/H2D ops "
                                         "wait behind the input H2D in the copy-engine FIFO"},
                "direct_only": {"value": e2e_direct, "unit": "GB/s",
                                "note": "same pipeline, host path disabled: the input upload "
                                        "saturates PCIe H2D, so the host hops' PCIe round "
                                        "trips queue behind it (~30 us per message)"},
                "fresh_message": {"value": e2e_fresh, "unit": "GB/s",
                                  "h2d_bytes_per_message": size,
                                  "note": "every message fetched from host memory: "
                                          "PCIe Gen5 H2D bound"}},
        "gpu_launches": args.steps * W * st.kernels,
        "clocks": clk.summary(),
        "graph": {"nodes_logical": st.nodes_logical, "nodes_physical": st.nodes_physical,
                  "kernels_per_send": st.kernels, "ce_copies_per_send": st.ce_copies,
                  "launch_us": st.launch_us},
        "lifecycle": lifecycle,
        "windows": windows,
        "relay_sweep": relays,
        "sweep": sweep,
        "tuning_csv": tuning,
    }
    print(json.dumps(out), flush=True)


SWEEP_SIZES = [1 << k for k in range(10, 30)]


def time_prepared(torch, eng, cfg, src, dst, size, steps, warmup, stream, trials=3):
    """time_sends for a send bound once (Engine.prepare): osu_bw re-sends one
    buffer, so the per-message host cost is one C call."""
    go = eng.prepare(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
    for _ in range(max(5, warmup)):
        go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(trials):
        e0.record(stream)
        for _ in range(steps):
            go()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / steps
        best = t if best is None else min(best, t)
    return best


def run_sweep(torch, eng, topo_text, dev, stream):
    """osu_bw-style: per size, single path (CE copy = cudaMemcpy, SM kernel;
    the SM send also bound once with Engine.prepare), direct+host multi-path
    with the graph cache on / off, and the measured tuner's best
    configuration."""
    from paper_2604_22228_b200 import Engine, PathConfig, load_topology
    from paper_2604_22228_b200.tuner import GridPoint, tune, tune_engines
    ce = Engine(load_topology(topo_text), [dev, dev])
    ce.configure(direct="ce")
    # measured per-size choices: direct mechanism (SM kernel vs CE), then the
    # reference tuner's grid (paths x host x chunks) on top of it
    auto = Engine(load_topology(topo_text), [dev, dev])
    # 50 back-to-back sends per trial: the steady state the sweep measures
    # (10-send bursts favoured the copy engine at ~1 MiB, which then lost
    # to the SM kernel over the sweep's 200-send runs)
    rules, _ = tune_engines(auto, SWEEP_SIZES, reps=50)
    auto.set_size_policy(rules)
    grid = [GridPoint(1, h, c) for h in (False, True) for c in (1, 2, 4, 8, 16, 32)]
    table = tune(auto, SWEEP_SIZES, grid, modes=("graph",), reps=50)
    rows = []
    big = torch.empty(SWEEP_SIZES[-1], dtype=torch.uint8, device=f"cuda:{dev}")
    out = torch.empty_like(big)
    arms = (("ce_single", ce, PathConfig(max_chunks=1, graph_mode=False)),
            ("sm_single", eng, PathConfig(max_chunks=1, graph_mode=True)),
            ("multi_graph", eng, PathConfig(1, True, 8, True)),
            ("multi_stream", eng, PathConfig(1, True, 8, False)))
    for size in SWEEP_SIZES:
        src, dst = big[:size], out[:size]
        steps = 20 if size > 64 * MiB else 200  # osu_bw-like steady state (64 x 100)
        warm = 3 if size > MiB else 10
        row = {"bytes": size}
        kernels = {}
        for name, e, cfg in arms:
            row[name] = size / time_sends(torch, e, cfg, src, dst, size, steps, warm, stream) / 1e9
            kernels[name] = e.stats().kernel.split(" ")[0] or "copy engine"
        row["kernels"] = kernels
        best = table.lookup(size, "graph").best
        row["sm_single_prepared"] = size / time_prepared(
            torch, eng, PathConfig(max_chunks=1, graph_mode=True), src, dst, size, steps, warm,
            stream) / 1e9
        row["tuned"] = size / time_sends(torch, auto, table.config_for(size), src, dst, size,
                                         steps, warm, stream) / 1e9
        row["tuned_point"] = [best.gpu_paths, best.host, best.max_chunks,
                              *next(r[1:] for r in rules if size <= r[0])]
        rows.append(row)
    ce.close()
    auto.close()
    return rows, {"table_csv": table.to_csv(), "engine_policy": rules}


def run_windows(eng):
    """BASELINE config 2's posting windows (W = 1, 4, 16 as in the paper, 64 as
    osu_bw): per window the W sends are posted back to back and the window
    is timed on the device up to its completion (measure.run_bw, rows in the
    reference's CSV schema), single path and direct + host k=8, each with its
    speedup over BASELINE_CONFIG (single direct copy, per-call submission)."""
    from paper_2604_22228_b200 import PathConfig
    from paper_2604_22228_b200 import measure as M
    sizes = [4 << 10, 64 << 10, MiB, 16 * MiB, 128 * MiB]
    summary, csv_rows = {}, []
    for w in (1, 4, 16, 64):
        for name, cfg in (("single", PathConfig(1, False, 1, True)),
                          ("multi_k8", PathConfig(1, True, 8, True))):
            res = M.run_bw(M.BenchmarkSpec("omb_bw", sizes, window=w, iterations=5, warmup=3,
                                           config=cfg, topology="b200_loopback"), eng)
            csv_rows += res.to_csv().splitlines()[1:]
            for r in res.rows:
                if r.metric == "bandwidth":
                    d = summary.setdefault(str(w), {}).setdefault(str(r.size), {})
                    d[name] = r.value / 1e9
                    d["baseline"] = r.value / r.speedup / 1e9
        # the window as ONE send_many program over W distinct buffer pairs
        # (one launch per window, like a grouped ncclSend); sizes whose
        # W pairs fit comfortably in HBM
        psizes = [s for s in sizes if s * w <= 2 << 30]
        res = M.run_bw(M.BenchmarkSpec("omb_bw_program", psizes, window=w, iterations=5,
                                       warmup=3, config=PathConfig(1, False, 1, True),
                                       topology="b200_loopback"), eng, program=True)
        csv_rows += res.to_csv().splitlines()[1:]
        for r in res.rows:
            if r.metric == "bandwidth":
                d = summary[str(w)][str(r.size)]
                d["single_program"] = r.value / 1e9
                d["baseline_distinct_buffers"] = r.value / r.speedup / 1e9
    return {"gbs": summary, "csv": "\n".join([M.CSV_HEADER] + csv_rows) + "\n"}


def run_relay_sweep(torch, dev, size, link_bw, host_bw, hbm_copy, pcie):
    """BASELINE config 4 in loopback: 8 logical GPUs on one B200, direct +
    0..6 GPU relays + host, max_chunks 16.  Every relayed byte is copied twice
    through the same HBM, so the gain the reference's model predicts (an
    independent channel per pair, topology.py:112-120) cannot appear: this is
    the single-GPU image of the NVSwitch ingress/egress cap."""
    from paper_2604_22228_b200 import Engine, PathConfig, load_topology, mesh_text
    eng8 = Engine(load_topology(mesh_text("b200x8_loopback", 8, link_bw, 1, 2e-6, host_bw, 1e-5,
                                          "full")), [dev] * 8)
    src = torch.empty(size, dtype=torch.uint8, device=f"cuda:{dev}")
    dst = torch.empty_like(src)
    stream = torch.cuda.Stream(device=dev)
    rows = []
    for g in range(1, 8):
        cfg = PathConfig(num_gpu_paths=g, host_path_enabled=True, max_chunks=16, graph_mode=True)
        t = time_sends(torch, eng8, cfg, src, dst, size, 10, 3, stream)
        st = eng8.stats()
        relay_share = sum(p.share for p in eng8.last_plan()[0] if p.kind == "gpu")
        # loopback roofline: a relayed byte costs two HBM copies
        r = 1.0 / ((1 - relay_share) / hbm_copy + 2 * relay_share / hbm_copy) + pcie
        rows.append({"relays": g - 1, "gbs": size / t / 1e9, "relay_share": relay_share,
                     "loopback_roofline_gbs": r, "frac": size / t / 1e9 / r,
                     "nodes_logical": st.nodes_logical, "nodes_physical": st.nodes_physical,
                     "kernels": st.kernels})
    eng8.close()
    return rows


def run_lifecycle(torch, eng, dev, stream):
    """Capture+instantiate every call / cached replay / per-call stream launch:
    host us per message, GPU latency, and the four lifecycle phases."""
    from paper_2604_22228_b200 import PathConfig
    res = []
    big = torch.empty(4 * MiB, dtype=torch.uint8, device=f"cuda:{dev}")
    out = torch.empty_like(big)
    for size in (4 << 10, 16 << 10, 64 << 10, 256 << 10, MiB, 4 * MiB):
        src, dst = big[:size], out[:size]
        g = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=1, graph_mode=True)
        s = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=1, graph_mode=False)
        row = {"bytes": size}
        cap = []
        for _ in range(20):
            eng.clear_cache()
            eng.send(src, dst, size, g, stream=stream, src_dev=0, dst_dev=1)
            st = eng.stats()
            cap.append((st.creation_us, st.construction_us, st.instantiation_us, st.launch_us,
                        st.plan_us))
        row["capture_every_call_us"] = {
            k: statistics.median(c[i] for c in cap)
            for i, k in enumerate(("creation", "construction", "instantiation", "launch",
                                   "plan"))}
        for name, cfg in (("replay", g), ("stream", s)):
            for _ in range(10):
                eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
            torch.cuda.synchronize()
            # BASELINE config 5: 10k iterations per size and arm.  Host cost
            # of the enqueue alone: batches of 100 sends with a sync between
            # batches (outside the clock), so a full launch queue never
            # blocks the host and GPU throughput does not leak into the number
            n, batch, host_s = 10000, 100, 0.0
            for _ in range(n // batch):
                t0 = time.perf_counter()
                for _ in range(batch):
                    eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
                host_s += time.perf_counter() - t0
                stream.synchronize()
            host_us = host_s / n * 1e6
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            lat = []
            for _ in range(50):
                e0.record(stream)
                eng.send(src, dst, size, cfg, stream=stream, src_dev=0, dst_dev=1)
                e1.record(stream)
                e1.synchronize()
                lat.append(e0.elapsed_time(e1) * 1e3)
            row[name] = {"host_us_per_msg": host_us, "gpu_latency_us": statistics.median(lat),
                         "launch_us_c_abi": eng.stats().launch_us}
        row["nodes_logical"] = eng.stats().nodes_logical
        row["nodes_physical"] = eng.stats().nodes_physical
        res.append(row)
    return res


def run_group(args, rank, world):
    """N > 1 (torchrun, one process per GPU): ONE GPU0->GPU1 message per
    transfer over direct + (N-2) GPU relays — the relay-count sweep of BASELINE
    config 4 — in multi-process group mode (CUDA-IPC mapped peer memory,
    device-side barrier, cached graphs).  Total work per step is fixed, so
    the scaling is strong; time is the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2604_22228_b200 import PathConfig, load_topology, mesh_text
    from paper_2604_22228_b200.group import TransferGroup
    dev = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    size, W = args.size, args.window
    topo = load_topology(mesh_text("b200_node", world, 900e9, 1, 2e-6, 64e9, 1e-5, "full"))
    grp = TransferGroup(topo, device=dev, stage_bytes=size // max(1, world - 1) + (64 << 20))
    src = torch.randint(0, 256, (size,), dtype=torch.uint8, device=f"cuda:{dev}",
                        generator=torch.Generator(device=f"cuda:{dev}").manual_seed(20261017)) \
        if rank == 0 else None
    dst = torch.zeros(size, dtype=torch.uint8, device=f"cuda:{dev}") if rank == 1 else None
    sb, db = grp.expose(src, 0), grp.expose(dst, 1)
    cfg = PathConfig(num_gpu_paths=world - 1, host_path_enabled=False, max_chunks=args.chunks,
                     graph_mode=True)
    stream = torch.cuda.Stream(device=dev)
    grp.transfer(sb, db, size, cfg, stream=stream)
    torch.cuda.synchronize()
    grp.sync()
    ck = int((src if rank == 0 else dst).sum(dtype=torch.int64)) if rank in (0, 1) else 0
    sums = [None] * world
    dist.all_gather_object(sums, ck)
    assert sums[0] == sums[1], "delivered bytes differ"
    for _ in range(args.warmup * W):
        grp.transfer(sb, db, size, cfg, stream=stream)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps * W):
            grp.transfer(sb, db, size, cfg, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
    times = [None] * world
    dist.all_gather_object(times, e0.elapsed_time(e1) / 1e3)
    t = max(times)  # max over ranks
    grp.sync()
    value = args.steps * W * size / t / 1e9

    # e2e through the public API from HOST memory: per window rank 0 copies
    # the input message H2D from pinned memory, the group sends it W times,
    # rank 1 reads back an int64 checksum of the delivered buffer (D2H);
    # device time per rank, max over ranks
    e2e_steps = max(2, args.steps // 2)
    shared_gpu = torch.cuda.device_count() < world  # ranks time-slice one GPU (no MPS)
    hsrc = hsum = None
    if rank == 0:
        hsrc = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        hsrc.copy_(src.cpu())
    if rank == 1:
        hsum = torch.empty(1, dtype=torch.int64, pin_memory=True)
    e2e = None
    if not shared_gpu:
        torch.cuda.synchronize()
        dist.barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(e2e_steps):
            if rank == 0:
                with torch.cuda.stream(stream):
                    src.copy_(hsrc, non_blocking=True)
            for _ in range(W):
                grp.transfer(sb, db, size, cfg, stream=stream)
            if rank == 1:
                with torch.cuda.stream(stream):
                    hsum.copy_(dst.sum(dtype=torch.int64).view(1), non_blocking=True)
        c1.record(stream)
        torch.cuda.synchronize()
        grp.sync()
        e2e_times = [None] * world
        dist.all_gather_object(e2e_times, c0.elapsed_time(c1) / 1e3)
        e2e = e2e_steps * W * size / max(e2e_times) / 1e9
        if rank == 1:
            assert int(hsum) == ck, "e2e checksum differs"

    # baseline only (not on the path): NCCL point-to-point send/recv of the
    # same message GPU0 -> GPU1 over the NCCL process group
    nccl = None
    if dist.get_backend() == "nccl":
        try:
            reps = max(4, args.steps * W // 4)
            buf = src if rank == 0 else (dst if rank == 1 else None)
            dist.barrier()
            n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for i in range(reps + 2):
                if i == 2:
                    n0.record()
                if rank == 0:
                    dist.send(buf, 1)
                elif rank == 1:
                    dist.recv(buf, 0)
            n1.record()
            torch.cuda.synchronize()
            nt = [None] * world
            dist.all_gather_object(nt, n0.elapsed_time(n1) / 1e3 if rank in (0, 1) else 0.0)
            nccl = {"value": reps * size / max(nt) / 1e9, "unit": "GB/s",
                    "what": "torch.distributed send/recv (NCCL p2p), rank 0 -> rank 1"}
        except Exception as exc:  # noqa: BLE001 - reported, never fatal
            nccl = {"unavailable": str(exc)[:200]}
    if rank == 0:
        peer_peak = 770.0  # measured peer copy per direction, B200_PROFILING.md
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded random bytes)",
            "config": group_config(args, world),
            "roofline": {"bound": "nvlink", "achieved": value, "peak": peer_peak,
                         "unit": "GB/s", "frac": value / peer_peak, "traffic": None,
                         "peak_kind": "B200_PROFILING.md measured peer copy (900 nominal)",
                         "note": "every path leaves GPU0's egress and enters GPU1's ingress"},
            "e2e": ({"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": size,
                     "d2h_bytes_per_step": 8, "steps": e2e_steps,
                     "step": f"rank 0: H2D of the input from pinned memory; {W} group "
                             "transfers; rank 1: D2H of an int64 checksum"}
                    if e2e is not None else
                    {"unavailable": "ranks share one GPU (no MPS): the e2e leg needs one GPU "
                                    "per rank"}),
            "nccl_p2p_baseline": nccl,
            "gpu_launches": args.steps * W, "clocks": clk.summary(),
            "cpu_baseline": None,
        }), flush=True)
    grp.close()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        # NCCL when every rank has its own GPU; gloo for the plumbing otherwise
        # (e.g. several ranks sharing one GPU to exercise the IPC path)
        ngpu = torch.cuda.device_count() if args.impl == "ours" else 0
        backend = "nccl" if ngpu >= world else "gloo"
        if args.impl == "ours":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % max(1, ngpu))
        dist.init_process_group(backend)
    if args.impl == "reference":
        run_reference(args, rank)
    elif world > 1:
        run_group(args, rank, world)
    else:
        run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
