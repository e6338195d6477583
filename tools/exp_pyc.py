"""16 MiB single-path graph replays driven from Python three ways (Engine.send,
_mpfast.send with precomputed arguments, ctypes mp_send) and with buffers
from torch vs cudaMalloc'd by the C probe — locating the Python-vs-C gap."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig, _lib, _mpfast  # noqa: E402

n = int(os.environ.get("SIZE", 16 << 20))
iters = int(os.environ.get("ITERS", 2000))
eng = Engine.loopback(2)
if os.environ.get("EMPTY"):  # the bench sweep's buffers: torch.empty, never written first
    big = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    if os.environ["EMPTY"] == "zero":
        big.zero_()
    elif os.environ["EMPTY"] == "ones":
        big.fill_(0xA5)
else:
    big = torch.randint(0, 256, (512 << 20,), dtype=torch.uint8, device="cuda")
out = torch.empty_like(big)
src, dst = big[:n], out[:n]
s = torch.cuda.Stream()
cfg = PathConfig(max_chunks=1, graph_mode=True)


WARM = int(os.environ.get("WARM", 50))


def timed(name, fn):
    for _ in range(WARM):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1) * 1e3 / iters:7.3f} us/msg  kernel={eng.stats().kernel[:24]}",
          flush=True)


sp, dp, h = src.data_ptr(), dst.data_ptr(), s.cuda_stream
if os.environ.get("HEAT"):  # seconds of full-size copies first (power / clock state)
    import time
    t_end = time.time() + float(os.environ["HEAT"])
    while time.time() < t_end:
        for _ in range(64):
            eng.send(big, out, 512 << 20, cfg, stream=s, src_dev=0, dst_dev=1)
        torch.cuda.synchronize()
    try:
        import pynvml as nv
        nv.nvmlInit()
        hnd = nv.nvmlDeviceGetHandleByIndex(0)
        print("sm clock after heat:", nv.nvmlDeviceGetClockInfo(hnd, nv.NVML_CLOCK_SM),
              "reasons", hex(nv.nvmlDeviceGetCurrentClocksEventReasons(hnd)))
    except Exception as exc:  # noqa: BLE001
        print("nvml:", exc)
addr = cfg.abi_addr()
timed("Engine.send", lambda: eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1))
timed("_mpfast.send", lambda: _mpfast.send(eng._ctx_addr, sp, dp, n, 0, 1, addr, h))
ref = C.byref(cfg.abi())
if os.environ.get("QUICK"):
    sys.exit(0)
timed("ctypes mp_send", lambda: _lib.lib.mp_send(eng._ctx, sp, dp, n, 0, 1, ref, h))
# fresh cudaMalloc-like buffers (torch empty, separate allocations)
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
pa, pb = a.data_ptr(), b.data_ptr()
timed("_mpfast separate buffers", lambda: _mpfast.send(eng._ctx_addr, pa, pb, n, 0, 1, addr, h))
timed("Engine.send again", lambda: eng.send(src, dst, n, cfg, stream=s, src_dev=0, dst_dev=1))
