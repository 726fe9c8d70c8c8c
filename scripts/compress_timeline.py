"""Host timeline of one pipelined compress (C2): when each span's encode, DMA and host copy finish."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_15037_b200 as g
from paper_2407_15037_b200 import device, stream, workloads

n = 1 << 26
x = device.mixed_f32(n, workloads.C2_SEED)
pinned = torch.empty(n, dtype=torch.int32, pin_memory=True)
pinned.copy_(x)
xh = pinned.numpy().view(np.float32)
cfg = g.QuantConfig(mode="rel", eb=1e-2)
for _ in range(3):
    s, _ = g.compress(xh, cfg)
torch.cuda.synchronize()
for rep in range(3):
    stream._TRACE = []
    t0 = time.perf_counter()
    s, _ = g.compress(xh, cfg)
    t1 = time.perf_counter()
    print(f"--- compress {1e3 * (t1 - t0):.2f} ms")
    for ev, t in stream._TRACE:
        print(f"{1e3 * (t - t0):8.3f}  {ev}")
    stream._TRACE = None
