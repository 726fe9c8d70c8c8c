"""Timeline of compress_pipelined: host timestamps for launch / drain phases."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_15037_b200 as g
from paper_2407_15037_b200 import device, workloads, stream

n = 1 << 26
x = device.mixed_f32(n, workloads.C2_SEED)
pinned = torch.empty(n, dtype=torch.int32, pin_memory=True); pinned.copy_(x)
xh = pinned.numpy().view(np.float32)
cfg = g.QuantConfig(mode="rel", eb=1e-2)
ev_log = []
t_start = [0.0]
o_enc = stream._encode_span
def enc(*a, **k):
    r = o_enc(*a, **k); ev_log.append(("enc_launched", time.perf_counter() - t_start[0])); return r
stream._encode_span = enc
o_copy = stream._d2h_ring_copy
def cp(*a, **k):
    ev_log.append(("drain_start", time.perf_counter() - t_start[0]))
    r = o_copy(*a, **k); ev_log.append(("drain_end", time.perf_counter() - t_start[0])); return r
stream._d2h_ring_copy = cp
for it in range(4):
    ev_log.clear(); torch.cuda.synchronize()
    t_start[0] = time.perf_counter()
    s, _ = g.compress(xh, cfg)
    tot = time.perf_counter() - t_start[0]
    if it == 3:
        for name, t in ev_log:
            print(f"{name:14s} {t*1e3:7.2f}")
    print("total", round(tot * 1e3, 2))
