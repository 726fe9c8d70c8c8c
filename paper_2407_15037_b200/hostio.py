"""Host <-> device movement for the host-buffer API (compress / decompress_to_array).

The GPU kernels take ~1 ms for 2^26 values; at the user-facing API the cost is
the PCIe traffic and host copies.  This module keeps both links busy:

* host->device: pinned sources go straight to the copy engine; pageable
  sources (numpy arrays, ``bytes``) are staged through a ring of pinned chunks
  with a multi-threaded host copy (torch's parallel memcpy), overlapped with
  the DMA of the previous chunk.
* device->host into a fresh ``bytes`` object: the result object is allocated
  uninitialised (PyBytes_FromStringAndSize(NULL, n), the documented way to
  build a bytes in place before it is shared), and filled chunk by chunk from a
  pinned ring while the next chunk is in flight -- no ``tobytes()`` copy.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

CHUNK = 32 << 20  # bytes per staging chunk
NSLOTS = 2

_PyBytes_FromStringAndSize = ctypes.pythonapi.PyBytes_FromStringAndSize
_PyBytes_FromStringAndSize.restype = ctypes.py_object
_PyBytes_FromStringAndSize.argtypes = [ctypes.c_char_p, ctypes.c_ssize_t]

_tls = threading.local()


def _ring(device) -> tuple:
    """Per-thread pinned staging ring + copy streams for ``device``."""
    key = ("ring", device.index if device.index is not None else torch.cuda.current_device())
    r = getattr(_tls, "rings", None)
    if r is None:
        r = _tls.rings = {}
    if key not in r:
        slots = [torch.empty(CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(NSLOTS)]
        events = [torch.cuda.Event() for _ in range(NSLOTS)]
        r[key] = (slots, events, torch.cuda.Stream(device=device))
    return r[key]


def _is_pinned(t: torch.Tensor) -> bool:
    try:
        return t.is_pinned()
    except Exception:
        return False


_MADV_HUGEPAGE = 14
try:
    _libc = ctypes.CDLL(None, use_errno=True)
    _madvise = _libc.madvise
    _madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    _madvise.restype = ctypes.c_int
except Exception:  # pragma: no cover - non-glibc hosts
    _madvise = None


def advise_hugepages(addr: int, n: int) -> None:
    """Ask for transparent huge pages on a fresh host range before first touch.

    A new result buffer is first-touched by the copy that fills it; with 4 KiB
    pages the page faults (kernel zeroing + mapping) cost about as much as the
    PCIe transfer itself.  With THP in ``madvise`` mode this halves that cost.
    Advisory only: failures are ignored.
    """
    if _madvise is None or n < (4 << 20):
        return
    lo = (addr + 4095) & ~4095
    hi = (addr + n) & ~4095
    if hi > lo:
        _madvise(lo, hi - lo, _MADV_HUGEPAGE)


def new_bytes(n: int):
    """An uninitialised bytes object of length n and a writable uint8 CPU tensor over it."""
    b = _PyBytes_FromStringAndSize(None, n)
    if n == 0:
        return b, torch.empty(0, dtype=torch.uint8)
    addr = ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p).value
    advise_hugepages(addr, n)
    arr = np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(addr))
    return b, torch.from_numpy(arr)


def h2d(src: torch.Tensor, dst: torch.Tensor) -> None:
    """Copy a uint8 CPU tensor into a uint8 CUDA tensor on the current stream."""
    n = src.numel()
    if n == 0:
        return
    if _is_pinned(src) or n <= (1 << 20):
        dst.copy_(src, non_blocking=_is_pinned(src))
        return
    cur = torch.cuda.current_stream(dst.device)
    slots, events, _ = _ring(dst.device)
    for i, off in enumerate(range(0, n, CHUNK)):
        k = i % NSLOTS
        m = min(CHUNK, n - off)
        events[k].synchronize()                 # slot's previous DMA done
        slots[k][:m].copy_(src[off:off + m])    # parallel host memcpy into pinned
        dst[off:off + m].copy_(slots[k][:m], non_blocking=True)
        events[k].record(cur)


def d2h_into(src: torch.Tensor, dst: torch.Tensor) -> None:
    """Copy a uint8 CUDA tensor into a (pageable) uint8 CPU tensor, chunk-pipelined."""
    n = src.numel()
    if n == 0:
        return
    if _is_pinned(dst) or n <= (1 << 20):
        dst.copy_(src)
        return
    cur = torch.cuda.current_stream(src.device)
    slots, events, _ = _ring(src.device)
    pending = []
    for i, off in enumerate(range(0, n, CHUNK)):
        k = i % NSLOTS
        m = min(CHUNK, n - off)
        if len(pending) == NSLOTS:              # drain the oldest chunk before reusing its slot
            po, pm, pk = pending.pop(0)
            events[pk].synchronize()
            dst[po:po + pm].copy_(slots[pk][:pm])
        slots[k][:m].copy_(src[off:off + m], non_blocking=True)
        events[k].record(cur)
        pending.append((off, m, k))
    for po, pm, pk in pending:
        events[pk].synchronize()
        dst[po:po + pm].copy_(slots[pk][:pm])


def device_to_new_bytes(src: torch.Tensor, prefix: bytes = b"") -> bytes:
    """bytes(prefix + src) built in place from device memory."""
    n = src.numel()
    b, view = new_bytes(len(prefix) + n)
    if prefix:
        view[:len(prefix)].copy_(torch.frombuffer(bytearray(prefix), dtype=torch.uint8))
    d2h_into(src, view[len(prefix):])
    return b


def host_u8(data) -> torch.Tensor:
    """Zero-copy uint8 CPU tensor over any bytes-like object or array (read-only use)."""
    import warnings

    if isinstance(data, torch.Tensor):
        return data.view(torch.uint8).reshape(-1)
    if isinstance(data, np.ndarray):
        data = np.ascontiguousarray(data).reshape(-1).view(np.uint8)
        if data.flags.writeable:
            return torch.from_numpy(data)
    if len(data) == 0:
        return torch.empty(0, dtype=torch.uint8)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return torch.frombuffer(data, dtype=torch.uint8)


def pinned_empty(n: int, dtype=torch.uint8) -> torch.Tensor:
    return torch.empty(n, dtype=dtype, pin_memory=True)


class H2DPipe:
    """Chunked host->device copy on a side stream with one event per chunk.

    ``push(lo, hi)`` enqueues bytes [lo, hi) of ``src`` into ``dst`` (same
    offsets) and returns an event the consumer stream waits on, so kernels on
    early chunks run while later chunks are still crossing PCIe.  Pinned
    sources go straight to the copy engine; pageable ones are staged through
    a ring of pinned slots with torch's multi-threaded host copy.
    """

    SLOT = 16 << 20
    NSLOT = 3

    def __init__(self, src: torch.Tensor, dst: torch.Tensor):
        self.src, self.dst = src, dst
        self.dev = dst.device
        self.pinned = _is_pinned(src)
        key = ("pipe", self.dev.index if self.dev.index is not None else torch.cuda.current_device())
        r = getattr(_tls, "rings", None)
        if r is None:
            r = _tls.rings = {}
        if key not in r:
            r[key] = ([torch.empty(self.SLOT, dtype=torch.uint8, pin_memory=True) for _ in range(self.NSLOT)],
                      [torch.cuda.Event() for _ in range(self.NSLOT)],
                      torch.cuda.Stream(device=self.dev))
        self.slots, self.slot_ev, self.stream = r[key]
        self.k = 0
        # the copy stream must not run ahead of work already queued on the caller's stream
        self.stream.wait_stream(torch.cuda.current_stream(self.dev))

    def push(self, lo: int, hi: int) -> torch.cuda.Event:
        st = self.stream
        if self.pinned:
            with torch.cuda.stream(st):
                self.dst[lo:hi].copy_(self.src[lo:hi], non_blocking=True)
        else:
            off = lo
            while off < hi:
                m = min(self.SLOT, hi - off)
                k = self.k
                self.k = (k + 1) % self.NSLOT
                self.slot_ev[k].synchronize()              # the slot's previous DMA is done
                self.slots[k][:m].copy_(self.src[off:off + m])
                with torch.cuda.stream(st):
                    self.dst[off:off + m].copy_(self.slots[k][:m], non_blocking=True)
                self.slot_ev[k].record(st)
                off += m
        ev = torch.cuda.Event()
        ev.record(st)
        return ev


# --- a bytes result built in place, sized after the fact -------------------
# PyBytes_FromStringAndSize(NULL, cap) creates an uninitialised object owned by
# the caller (refcount 1); _PyBytes_Resize shrinks such a brand-new object to
# its final length (the C-API way to build a bytes whose size is only known at
# the end; realloc of the large block shrinks in place).  Only the touched
# pages of the capacity are ever backed by memory.  _PyBytes_Resize is private
# CPython API: it is used only on a GIL-enabled CPython 3.8-3.13 that exports
# it; anywhere else the builder falls back to a bytearray + one final copy.
def _resize_supported() -> bool:
    import sys
    import sysconfig

    if sys.implementation.name != "cpython" or not (3, 8) <= sys.version_info[:2] <= (3, 13):
        return False
    if sysconfig.get_config_var("Py_GIL_DISABLED"):
        return False
    return hasattr(ctypes.pythonapi, "_PyBytes_Resize") and hasattr(ctypes.pythonapi, "PyBytes_AsString")


RESIZE_IN_PLACE = _resize_supported()
if RESIZE_IN_PLACE:
    _bytes_new_raw = ctypes.PYFUNCTYPE(ctypes.c_void_p, ctypes.c_char_p, ctypes.c_ssize_t)(
        ("PyBytes_FromStringAndSize", ctypes.pythonapi))
    _bytes_as_string = ctypes.PYFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p)(("PyBytes_AsString", ctypes.pythonapi))
    _bytes_resize = ctypes.PYFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.c_ssize_t)(
        ("_PyBytes_Resize", ctypes.pythonapi))
    _py_decref = ctypes.pythonapi.Py_DecRef
    _py_decref.argtypes = [ctypes.c_void_p]
    _py_decref.restype = None
else:  # pragma: no cover - exercised through the fallback test
    _py_decref = None


class _BytearrayBuilder:
    """Portable fallback: fill a bytearray, copy the used prefix out once."""

    def __init__(self, cap: int):
        self.cap = cap
        self._buf = bytearray(cap)
        self.view = torch.frombuffer(self._buf, dtype=torch.uint8) if cap else torch.empty(0, dtype=torch.uint8)

    def finish(self, n: int) -> bytes:
        if not 0 <= n <= self.cap:
            raise ValueError("final length beyond capacity")
        self.view = None
        out = bytes(memoryview(self._buf)[:n])
        self._buf = None
        return out


class _ResizeBuilder:
    """A new ``bytes`` of up to ``cap`` bytes, filled through a writable uint8 view
    and finalised with :meth:`finish` (which shrinks it to the used length)."""

    def __init__(self, cap: int):
        self._obj = ctypes.c_void_p(_bytes_new_raw(None, cap))
        if not self._obj.value:
            raise MemoryError(f"cannot allocate a {cap}-byte result")
        self.cap = cap
        self.addr = _bytes_as_string(self._obj)
        advise_hugepages(self.addr, cap)
        arr = np.ctypeslib.as_array((ctypes.c_uint8 * max(cap, 1)).from_address(self.addr))[:cap]
        self.view = torch.from_numpy(arr)

    def finish(self, n: int) -> bytes:
        if not 0 <= n <= self.cap:
            raise ValueError("final length beyond capacity")
        self.view = None
        if _bytes_resize(ctypes.byref(self._obj), n) != 0 or not self._obj.value:
            raise MemoryError("cannot finalise the result bytes")
        out = ctypes.cast(self._obj, ctypes.py_object).value   # new reference
        _py_decref(self._obj)                                 # drop the builder's reference
        self._obj = ctypes.c_void_p(0)
        return out

    def __del__(self):
        obj = getattr(self, "_obj", None)
        if obj is not None and obj.value and _py_decref is not None:
            self.view = None
            _py_decref(obj)
            self._obj = ctypes.c_void_p(0)


def BytesBuilder(cap: int):
    """The in-place builder where the interpreter supports it, else the fallback."""
    return _ResizeBuilder(cap) if RESIZE_IN_PLACE else _BytearrayBuilder(cap)
