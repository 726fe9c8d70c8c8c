"""cProfile of the host-buffer API (compress + decompress_to_array) on the C2 batch."""
import cProfile, pstats, sys, time
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
for _ in range(2):
    s, _ = g.compress(xh, cfg); y = g.decompress_to_array(s)
torch.cuda.synchronize()
for name, fn in (("compress", lambda: g.compress(xh, cfg)), ("decompress", lambda: g.decompress_to_array(s))):
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(name, "ms", [round(t * 1e3, 2) for t in ts])
    pr = cProfile.Profile(); pr.enable(); fn(); torch.cuda.synchronize(); pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
