"""Sweep the host-pipeline span sizes of compress / decompress_to_array (C2 batch)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_15037_b200 as g
from paper_2407_15037_b200 import device, hostio, stream, workloads

n = 1 << 26
x = device.mixed_f32(n, workloads.C2_SEED)
pinned = torch.empty(n, dtype=torch.int32, pin_memory=True); pinned.copy_(x)
xh = pinned.numpy().view(np.float32)
cfg = g.QuantConfig(mode="rel", eb=1e-2)

def run(label):
    s = y = None
    for _ in range(3):
        s, _ = g.compress(xh, cfg); y = g.decompress_to_array(s)
    tc, td = [], []
    for _ in range(8):
        t0 = time.perf_counter(); s, _ = g.compress(xh, cfg); t1 = time.perf_counter()
        y = g.decompress_to_array(s); t2 = time.perf_counter()
        tc.append(t1 - t0); td.append(t2 - t1)
    print(f"{label:40s} compress {1e3*np.median(tc):6.2f} decompress {1e3*np.median(td):6.2f} total {1e3*(np.median(tc)+np.median(td)):6.2f}", flush=True)

for cc in (8 << 20, 16 << 20, 32 << 20):
    for ds in (8 << 20, 16 << 20, 32 << 20):
        stream.COMPRESS_CHUNK = cc
        stream.D2H_SLOT = ds
        stream._LOCAL.__dict__.pop("rings", None)
        run(f"compress chunk {cc>>20}MB d2h slot {ds>>20}MB")
stream.COMPRESS_CHUNK = 16 << 20; stream.D2H_SLOT = 16 << 20; stream._LOCAL.__dict__.pop("rings", None)
for dc in (8 << 20, 16 << 20, 32 << 20, 64 << 20):
    for sl in (8 << 20, 16 << 20, 32 << 20):
        stream.DECODE_CHUNK = dc
        hostio.H2DPipe.SLOT = sl
        hostio._tls.rings = {}
        run(f"decode chunk {dc>>20}MB h2d slot {sl>>20}MB")
