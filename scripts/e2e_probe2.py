"""Where the host-buffer (e2e) time of C2 goes now: compress / decompress and their parts."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_15037_b200 as g
from paper_2407_15037_b200 import device, hostio, stream, workloads


def t(f, reps=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return f"min {min(ts) * 1e3:7.2f} med {sorted(ts)[len(ts) // 2] * 1e3:7.2f}"


n = 1 << 26
dev = torch.device("cuda", 0)
x = device.mixed_f32(n, workloads.C2_SEED)
pinned = torch.empty(n, dtype=torch.int32, pin_memory=True)
pinned.copy_(x)
xh = pinned.numpy().view(np.float32)
cfg = g.QuantConfig(mode="rel", eb=1e-2)
print("torch threads", torch.get_num_threads())
print("compress ms          ", t(lambda: g.compress(xh, cfg)))
s, _ = g.compress(xh, cfg)
print("stream MB", len(s) / 2**20)
print("decompress ms        ", t(lambda: g.decompress_to_array(s)))
src = hostio.host_u8(s)
sd = torch.empty(len(s) + 16, dtype=torch.uint8, device=dev)


def pipe_all():
    p = hostio.H2DPipe(src, sd)
    ev = p.push(0, len(s))
    torch.cuda.current_stream().wait_event(ev)


print("H2DPipe pageable ms  ", t(pipe_all))
pin_s = torch.empty(len(s), dtype=torch.uint8, pin_memory=True)
pin_s.copy_(src)
print("H2D pinned stream ms ", t(lambda: sd[:len(s)].copy_(pin_s, non_blocking=True)))
slot = torch.empty(16 << 20, dtype=torch.uint8, pin_memory=True)
print("memcpy 16MB->pinned  ", t(lambda: slot.copy_(src[:16 << 20]), reps=20))
print("memcpy 155MB torch   ", t(lambda: pin_s.copy_(src)))
hv = torch.empty(n, dtype=torch.int32, pin_memory=True)
print("D2H 256MB pinned ms  ", t(lambda: hv.copy_(x, non_blocking=True)))
print("H2D 256MB pinned ms  ", t(lambda: x.copy_(pinned, non_blocking=True)))
enc = stream.encode(x, cfg)
print("encode dev ms        ", t(lambda: stream.encode(x, cfg)))
