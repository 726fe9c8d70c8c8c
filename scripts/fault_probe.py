"""Cost of first-touch of a fresh result buffer, and ways to take it off the critical path."""
import ctypes
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2407_15037_b200 import hostio

libc = ctypes.CDLL(None, use_errno=True)
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
MADV_POPULATE_WRITE = 23
CAP = 1300 << 20
SPAN = 19 << 20
NS = 8
slot = torch.empty(32 << 20, dtype=torch.uint8, pin_memory=True)
slot.fill_(7)


def populate(addr, n):
    lo = addr & ~4095
    r = libc.madvise(lo, (addr + n - lo + 4095) & ~4095, MADV_POPULATE_WRITE)
    return r, ctypes.get_errno()


def run(mode, threads=4, reps=4):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        b = hostio.BytesBuilder(CAP)
        futs = []
        if mode.startswith("pop"):
            ex = ThreadPoolExecutor(threads)
            sub = SPAN // threads
            for c in range(NS):
                for j in range(threads):
                    futs.append(ex.submit(populate, b.addr + c * SPAN + j * sub, sub))
        for c in range(NS):
            if mode.startswith("pop"):
                for f in futs[c * threads:(c + 1) * threads]:
                    f.result()
            dst = b.view[c * SPAN:(c + 1) * SPAN]
            if mode.endswith("np"):
                np.copyto(dst.numpy(), slot[:SPAN].numpy())
            else:
                dst.copy_(slot[:SPAN])
        if mode.startswith("pop"):
            ex.shutdown()
        b.finish(NS * SPAN)
        ts.append(time.perf_counter() - t0)
    print(f"{mode:12s} thr {threads}: ms min {1e3 * min(ts):.2f} med {1e3 * sorted(ts)[len(ts) // 2]:.2f}", flush=True)


print("populate rc", populate(hostio.BytesBuilder(CAP).addr, 1 << 20))
print("torch threads", torch.get_num_threads())
run("plain")
run("plain-np")
for th in (1, 2, 4, 8):
    run("pop", th)
# prefaulted copy speed
b = hostio.BytesBuilder(CAP)
b.view[:NS * SPAN].fill_(1)
t0 = time.perf_counter()
for c in range(NS):
    b.view[c * SPAN:(c + 1) * SPAN].copy_(slot[:SPAN])
print("copy into faulted ms", 1e3 * (time.perf_counter() - t0))
t0 = time.perf_counter()
populate(hostio.BytesBuilder(CAP).addr, NS * SPAN)
print("populate 152MB 1 call ms", 1e3 * (time.perf_counter() - t0))

# pre-touch ahead of the copy from a thread pool (one write per 2 MiB / 4 KiB page)
def touch(view, step):
    view[::step].fill_(0)


for step in (4096, 2 << 20):
    for th in (2, 4, 8):
        ex = ThreadPoolExecutor(th)
        ts = []
        for rep in range(4):
            t0 = time.perf_counter()
            b = hostio.BytesBuilder(CAP)
            futs = []
            sub = SPAN // th
            for c in range(NS):
                futs.append([ex.submit(touch, b.view[c * SPAN + j * sub:c * SPAN + (j + 1) * sub], step)
                             for j in range(th)])
            for c in range(NS):
                for f in futs[c]:
                    f.result()
                b.view[c * SPAN:(c + 1) * SPAN].copy_(slot[:SPAN])
            b.finish(NS * SPAN)
            ts.append(1e3 * (time.perf_counter() - t0))
        ex.shutdown()
        print(f"touch step {step} thr {th}: ms", [round(t, 2) for t in ts], flush=True)
