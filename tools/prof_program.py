"""A 64-message posting window as ONE send_many program (prepare_many),
64 distinct buffer pairs of SIZE bytes (default 64 KiB): device time per
window, for a plain run or under ncu (-k regex:small_copy)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_22228_b200 import Engine, PathConfig  # noqa: E402

size, W = int(os.environ.get("SIZE", 64 << 10)), int(os.environ.get("W", 64))
eng = Engine.loopback(2)
pairs = [(torch.randint(0, 256, (size,), dtype=torch.uint8, device="cuda"),
          torch.empty(size, dtype=torch.uint8, device="cuda")) for _ in range(W)]
s = torch.cuda.Stream()
post = eng.prepare_many([(a, b, None, 0, 1) for a, b in pairs], PathConfig(1, False, 1, True),
                        stream=s)
for _ in range(5):
    post()
torch.cuda.synchronize()
assert all(torch.equal(a, b) for a, b in pairs)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(100):
    post()
e1.record(s)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 100 * 1e3
# host cost of posting a window: batches of 50 posts, synced between batches
import time  # noqa: E402
host = 0.0
for _ in range(20):
    t0 = time.perf_counter()
    for _ in range(50):
        post()
    host += time.perf_counter() - t0
    s.synchronize()
print(f"W={W} x {size} B: {us:.2f} us per window back to back = {W * size / us / 1e3:.1f} GB/s; "
      f"host {host / 1000 * 1e6:.2f} us per post; kernel {eng.stats().kernel}")
