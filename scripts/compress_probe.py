"""Timeline of the pipelined compress (host-side timestamps per phase)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_15037_b200 as g
from paper_2407_15037_b200 import device, workloads, stream, hostio

n = 1 << 26
x = device.mixed_f32(n, workloads.C2_SEED)
pinned = torch.empty(n, dtype=torch.int32, pin_memory=True); pinned.copy_(x)
xh = pinned.numpy().view(np.float32)
cfg = g.QuantConfig(mode="rel", eb=1e-2)
T = {}
orig_drain_copy = stream._d2h_ring_copy
orig_sync = torch.cuda.Event.synchronize
def timed(name, f):
    def w(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); T[name] = T.get(name, 0) + time.perf_counter() - t0; return r
    return w
stream._d2h_ring_copy = timed("ring_copy", orig_drain_copy)
stream._d2h_ring_flush = timed("ring_flush", stream._d2h_ring_flush)
torch.cuda.Event.synchronize = timed("event_sync", orig_sync)
hostio.BytesBuilder.finish = timed("finish", hostio.BytesBuilder.finish)
for it in range(6):
    T.clear()
    t0 = time.perf_counter(); s, _ = g.compress(xh, cfg); t1 = time.perf_counter()
    print(f"compress {1e3*(t1-t0):.2f} ms", {k: round(v * 1e3, 2) for k, v in T.items()}, flush=True)
# raw components
torch.cuda.synchronize()
d = torch.empty(n, dtype=torch.int32, device="cuda")
for _ in range(3):
    t0 = time.perf_counter(); d.copy_(pinned, non_blocking=True); torch.cuda.synchronize(); print("h2d 256MB", round((time.perf_counter()-t0)*1e3, 2))
b = hostio.BytesBuilder(400 << 20)
src = torch.empty(155 << 20, dtype=torch.uint8, pin_memory=True)
t0 = time.perf_counter(); b.view[:155 << 20].copy_(src); print("fresh memcpy 155MB", round((time.perf_counter()-t0)*1e3, 2))
t0 = time.perf_counter(); b.view[:155 << 20].copy_(src); print("warm memcpy 155MB", round((time.perf_counter()-t0)*1e3, 2))
