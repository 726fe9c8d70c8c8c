"""Why the bench e2e loop is slower than isolated calls: time each call in the loop."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_15037_b200 as g
from paper_2407_15037_b200 import device, workloads

n = 1 << 26
x = device.mixed_f32(n, workloads.C2_SEED)
pinned = torch.empty(n, dtype=torch.int32, pin_memory=True); pinned.copy_(x)
xh = pinned.numpy().view(np.float32)
cfg = g.QuantConfig(mode="rel", eb=1e-2)
for keep in (True, False, True):
    s = y = None
    for i in range(8):
        if not keep:
            s = y = None
        t0 = time.perf_counter()
        s, _ = g.compress(xh, cfg)
        t1 = time.perf_counter()
        y = g.decompress_to_array(s)
        t2 = time.perf_counter()
        print(f"keep={keep} it={i} compress {1e3*(t1-t0):.2f} decompress {1e3*(t2-t1):.2f}", flush=True)
