"""Cost of materialising a fresh `bytes` result from device memory, several ways."""
import ctypes, mmap, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2407_15037_b200 import hostio

N = 155 << 20
dev = torch.device("cuda", 0)
d = torch.randint(0, 255, (N,), dtype=torch.uint8, device=dev)
pinned = torch.empty(N, dtype=torch.uint8, pin_memory=True)
pinned.copy_(d)
libc = ctypes.CDLL("libc.so.6")
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
cudart = torch.cuda.cudart()

def tm(name, f, reps=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:50s} ms min {min(ts):7.2f} med {sorted(ts)[len(ts)//2]:7.2f}", flush=True)

def a():
    b, v = hostio.new_bytes(N); v.copy_(pinned); return b
def a1():
    b, v = hostio.new_bytes(N)
    torch.set_num_threads(16); v.copy_(pinned); return b
def b_():
    b, v = hostio.new_bytes(N)
    addr = v.data_ptr(); base = addr & ~((1 << 21) - 1)
    libc.madvise(base, N + (addr - base), 14)  # MADV_HUGEPAGE
    v.copy_(pinned); return b
def c():
    b, v = hostio.new_bytes(N); v.copy_(d); return b
def c2():
    b, v = hostio.new_bytes(N); hostio.d2h_into(d, v); return b
def e():
    b, v = hostio.new_bytes(N)
    addr = v.data_ptr()
    torch.cuda.cudart().cudaHostRegister(addr, N, 0)
    v.copy_(d)
    torch.cuda.cudart().cudaHostRegister  # keep
    torch.cuda.cudart().cudaHostUnregister(addr)
    return b
def touch():
    b, v = hostio.new_bytes(N); v.fill_(0); return b
def npzero():
    return np.zeros(N // 4, np.int32)
def npempty_touch():
    x = np.empty(N, np.uint8); x[::4096] = 0; return x
tm("fresh bytes + torch copy from pinned", a)
tm("fresh bytes + madvise hugepage + copy", b_)
tm("fresh bytes + pageable D2H (torch)", c)
tm("fresh bytes + d2h_into ring", c2)
tm("fresh bytes + fill_ (touch only)", touch)
tm("np.empty + touch 1 byte/page", npempty_touch)
try:
    tm("fresh bytes + cudaHostRegister + D2H", e)
except Exception as ex:
    print("register failed", ex)
tm("pinned D2H 155MB", lambda: pinned.copy_(d))
import os
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read())
print(os.cpu_count(), torch.get_num_threads())
