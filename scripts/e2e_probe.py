"""Break down where end-to-end (host buffer) time goes: copies vs kernels vs host overheads."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_15037_b200 as g
from paper_2407_15037_b200 import stream, device, workloads
from paper_2407_15037_b200.container import parse_layout

def t(f, reps=3):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3

n = 1 << 26
dev = torch.device("cuda", 0)
x = device.mixed_f32(n, workloads.C2_SEED)
pinned = torch.empty(n, dtype=torch.int32, pin_memory=True); pinned.copy_(x)
pageable = torch.empty(n, dtype=torch.int32); pageable.copy_(x)
d = torch.empty_like(x)
print("H2D pinned 256MB  ms", t(lambda: d.copy_(pinned)))
print("H2D pageable 256MB ms", t(lambda: d.copy_(pageable)))
print("D2H pinned 256MB  ms", t(lambda: pinned.copy_(d)))
print("D2H pageable 256MB ms", t(lambda: pageable.copy_(d)))
print("host memcpy torch 256MB ms", t(lambda: pageable.copy_(pinned)))
a = pinned.numpy(); b = np.empty_like(a)
print("host memcpy numpy 256MB ms", t(lambda: np.copyto(b, a)))
print("tobytes 256MB ms", t(lambda: a.tobytes()))
print("torch threads", torch.get_num_threads())
xh = pinned.numpy().view(np.float32)
cfg = g.QuantConfig(mode="rel", eb=1e-2)
print("compress ms", t(lambda: g.compress(xh, cfg)))
s, _ = g.compress(xh, cfg)
print("stream MB", len(s) / 2**20)
print("decompress ms", t(lambda: g.decompress_to_array(s)))
print("parse_layout ms", t(lambda: parse_layout(s)))
print("frombuffer+H2D stream ms", t(lambda: stream._h2d_stream(s)))
enc = stream.encode(x, cfg)
hdr = stream.header_for(cfg, n)
print("stream_to_host ms", t(lambda: stream.stream_to_host(enc, hdr)))
print("upload ms", t(lambda: g.pipeline._upload(xh)))
