"""Drop-in replacements for the reference's operator layer ``gebq._kernels``.

Every function keeps the exact name, argument order, in-place output
convention and return value of the numba dispatcher it replaces
(/root/reference/pkg/src/gebq/_kernels.py), so ``install(gebq)`` can rebind
``gebq._kernels.<name>`` and the reference's own pipeline/container/sweep
code runs on the B200 unchanged.  Each call moves the part of its arrays it
works on host<->device (block shims: only their task's span); the
pipeline-level entry points (paper_2407_15037_b200.pipeline) keep data
resident and are the fast path.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib, device, stream
from .quantizers import MAXBIN32, MAXBIN64, QuantConfig

DEC_OK = 0
DEC_TRUNCATED = 1
DEC_NONCANONICAL = 2
DEC_COUNT_MISMATCH = 3

TRIG_NAN = 0
TRIG_INF = 1
TRIG_GUARD = 2
TRIG_DCHECK = 3

__all__ = [
    "quantize_abs32", "quantize_abs64", "quantize_rel32", "quantize_rel64",
    "reconstruct_abs32", "reconstruct_abs64", "reconstruct_rel32", "reconstruct_rel64",
    "block_sizes_u32", "block_sizes_u64", "emit_blocks_u32", "emit_blocks_u64",
    "decode_blocks_u32", "decode_blocks_u64", "sweep_abs32_on", "sweep_abs64_on",
    "sweep_rel32_on", "sweep_rel64_on", "splitmix64_fill", "quantize_rel32_lib",
    "reconstruct_rel32_lib", "MAXBIN32", "MAXBIN64",
]


class _Cfg:
    """Minimal stand-in for QuantConfig carrying pre-derived width-typed constants."""

    def __init__(self, mode, width, unsafe, **consts):
        self.mode = mode
        self.width = width
        self.unsafe_no_double_check = bool(unsafe)
        self.derived = type("D", (), consts)()


class _Lane:
    """Per-calling-thread CUDA stream, pinned host staging and device scratch.

    The reference calls its kernels from a ThreadPool (pipeline.py:143-154,
    container.py:315-334); each worker thread gets its own stream so tasks
    overlap on the GPU and on PCIe, and its own grow-only buffers so a task
    costs two host memcpys (caller <-> pinned), the DMAs and the launch --
    no allocation, no pageable copy, no device-wide synchronisation."""

    def __init__(self):
        self.dev = device.require_cuda()
        self.stream = torch.cuda.Stream(device=self.dev)
        self._h, self._d = {}, {}

    @staticmethod
    def _grow(pool, key, nbytes, make):
        t = pool.get(key)
        if t is None or t.numel() < nbytes:
            cap = 1 << max(16, (max(nbytes, 1) - 1).bit_length())
            t = pool[key] = make(cap)
        return t[:nbytes]

    def host(self, key, nbytes) -> torch.Tensor:
        return self._grow(self._h, key, nbytes, lambda c: torch.empty(c, dtype=torch.uint8, pin_memory=True))

    def devbuf(self, key, nbytes) -> torch.Tensor:
        # 16 bytes of slack: vector loads near the end stay inside the allocation
        return self._grow(self._d, key, nbytes + 16,
                          lambda c: torch.empty(c, dtype=torch.uint8, device=self.dev))[:nbytes]

    def up(self, key, arr) -> torch.Tensor:
        """Stage a host array into this lane's device buffer ``key`` (async H2D)."""
        a = np.ascontiguousarray(arr).reshape(-1).view(np.uint8)
        h = self.host(key, a.nbytes)
        np.copyto(h.numpy(), a)
        d = self.devbuf(key, a.nbytes)
        d.copy_(h, non_blocking=True)
        return d

    def down(self, key, d: torch.Tensor) -> torch.Tensor:
        """Queue a D2H copy of the uint8 device tensor ``d``; valid after sync()."""
        h = self.host(key, d.numel())
        h.copy_(d, non_blocking=True)
        return h

    def sync(self):
        self.stream.synchronize()


# Lanes are pooled, not thread-local: the reference builds a fresh
# ThreadPoolExecutor for every container pass (container.py:315-334), so its
# worker threads are short-lived while the lanes (streams, pinned memory) are
# reused by whichever thread calls next.
_free: list = []
_free_lock = threading.Lock()


class _lane:
    """``with _lane() as ln:`` -- borrow a lane for one shim call."""

    def __enter__(self) -> _Lane:
        with _free_lock:
            self.ln = _free.pop() if _free else None
        if self.ln is None:
            self.ln = _Lane()
        self._ctx = torch.cuda.stream(self.ln.stream)
        self._ctx.__enter__()
        return self.ln

    def __exit__(self, *exc):
        self._ctx.__exit__(*exc)
        with _free_lock:
            _free.append(self.ln)
        return False


_IT = {32: torch.int32, 64: torch.int64}


def _quantize(bits, codes, lossless, cfg) -> np.ndarray:
    n = len(bits)
    if n == 0:
        return np.zeros(4, dtype=np.int64)
    W = cfg.width // 8
    with _lane() as ln:
        x = ln.up("x", bits).view(_IT[cfg.width])
        c = ln.devbuf("c", n * W).view(_IT[cfg.width])
        ll = ln.devbuf("l", n)
        trig = ln.devbuf("t", 32).view(torch.int64)
        trig.zero_()
        device.quantize(x, cfg, codes=c, lossless=ll, trig=trig)
        hc = ln.down("c", c.view(torch.uint8))
        hl = ln.down("l", ll)
        ht = ln.down("t", trig.view(torch.uint8))
        ln.sync()
        codes[...] = hc.numpy().view(codes.dtype)   # copy out before the lane is returned
        lossless[...] = hl.numpy().view(np.bool_)
        return ht.numpy().view(np.int64).copy()


# ---- quantize_* (_kernels.py:86-285) ----------------------------------------
def quantize_abs32(bits, vals, codes, lossless, eb_eff, eb2, inv_eb2, thr, unsafe):
    return _quantize(bits, codes, lossless, _Cfg("abs", 32, unsafe, eb_eff=np.float32(eb_eff),
                                                 eb2=np.float32(eb2), inv_eb2=np.float32(inv_eb2),
                                                 thr=np.float32(thr)))


def quantize_abs64(bits, vals, codes, lossless, eb_eff, eb2, inv_eb2, thr, unsafe):
    return _quantize(bits, codes, lossless, _Cfg("abs", 64, unsafe, eb_eff=np.float64(eb_eff),
                                                 eb2=np.float64(eb2), inv_eb2=np.float64(inv_eb2),
                                                 thr=np.float64(thr)))


def quantize_rel32(bits, vals, codes, lossless, op_eps, w, thr, unsafe):
    return _quantize(bits, codes, lossless, _Cfg("rel", 32, unsafe, op_eps=np.float32(op_eps),
                                                 w=np.float32(w), thr=np.float32(thr)))


def quantize_rel64(bits, vals, codes, lossless, op_eps, w, thr, unsafe):
    return _quantize(bits, codes, lossless, _Cfg("rel", 64, unsafe, op_eps=np.float64(op_eps),
                                                 w=np.float64(w), thr=np.float64(thr)))


# ---- reconstruct_* (_kernels.py:293-354) ------------------------------------
def _reconstruct(codes, lossless, out_bits, mode, derived):
    n = len(codes)
    if n == 0:
        return 0
    width = 32 if np.asarray(codes).dtype.itemsize == 4 else 64
    with _lane() as ln:
        c = ln.up("c", codes).view(_IT[width])
        ll = ln.up("l", np.asarray(lossless, dtype=np.bool_))
        o = ln.devbuf("o", n * width // 8).view(_IT[width])
        device.reconstruct(c, ll, mode, derived, out=o)
        ho = ln.down("o", o.view(torch.uint8))
        ln.sync()
        out_bits[...] = ho.numpy().view(out_bits.dtype)
    return 0


def reconstruct_abs32(codes, lossless, out_bits, out_vals, eb2):
    return _reconstruct(codes, lossless, out_bits, "abs", np.float32(eb2))


def reconstruct_abs64(codes, lossless, out_bits, out_vals, eb2):
    return _reconstruct(codes, lossless, out_bits, "abs", np.float64(eb2))


def reconstruct_rel32(codes, lossless, out_bits, out_vals, w):
    return _reconstruct(codes, lossless, out_bits, "rel", np.float32(w))


def reconstruct_rel64(codes, lossless, out_bits, out_vals, w):
    return _reconstruct(codes, lossless, out_bits, "rel", np.float64(w))


# ---- library-log REL variant (_kernels.py:356-431; non-conforming by design) --
def quantize_rel32_lib(bits, vals, codes, lossless, op_eps, w, thr, unsafe):
    n = len(bits)
    if n == 0:
        return np.zeros(4, dtype=np.int64)
    x = device.to_device(np.ascontiguousarray(bits))
    c = torch.empty_like(x)
    ll = torch.empty(n, dtype=torch.uint8, device=x.device)
    trig = torch.zeros(4, dtype=torch.int64, device=x.device)
    _lib.call("gebq_quantize_rel_lib_f32", device._p(x), device._p(c), device._p(ll), n,
              np.float32(op_eps).item(), np.float32(w).item(), np.float32(thr).item(), int(bool(unsafe)),
              device._p(trig), device._s())
    codes[...] = c.cpu().numpy().view(codes.dtype)
    lossless[...] = ll.cpu().numpy().view(np.bool_)
    return trig.cpu().numpy().astype(np.int64)


def reconstruct_rel32_lib(codes, lossless, out_bits, out_vals, w):
    n = len(codes)
    if n == 0:
        return 0
    c = device.to_device(np.ascontiguousarray(codes))
    ll = device.to_device(np.ascontiguousarray(lossless, dtype=np.bool_))
    out = torch.empty_like(c)
    _lib.call("gebq_dequantize_rel_lib_f32", device._p(c), device._p(ll), device._p(out), n,
              np.float32(w).item(), device._s())
    out_bits[...] = out.cpu().numpy().view(out_bits.dtype)
    return 0


# ---- block payload (_kernels.py:606-664) --------------------------------------
# The reference calls these once per 64-block task (container._run_block_tasks,
# container.py:315-334) with the WHOLE codes / lossless / offsets / region
# arrays and a block range [b0, b1).  Each shim moves only its task's span:
# values [b0*bs, min(b1*bs, count)), offsets rebased to the span's first byte,
# and the span's bytes of the region -- O(span) PCIe traffic per call, so the
# whole encode / decode moves each byte once.

def _span(count, block_size, b0, b1):
    s0 = int(b0) * int(block_size)
    s1 = min(int(b1) * int(block_size), int(count))
    return s0, max(s1, s0)


def _block_sizes(width, codes, count, block_size, b0, b1, sizes):
    if b1 <= b0:
        return 0
    s0, s1 = _span(count, block_size, b0, b1)
    nb = int(b1) - int(b0)
    with _lane() as ln:
        c = ln.up("c", codes[s0:s1])
        sz = ln.devbuf("s", 8 * nb).view(torch.int64)
        _lib.call(f"gebq_block_sizes_u{width}", device._p(c), s1 - s0, int(block_size), 0, nb,
                  device._p(sz), device._s())
        hs = ln.down("s", sz.view(torch.uint8))
        ln.sync()
        sizes[b0:b1] = hs.numpy().view(np.int64)
    return 0


def block_sizes_u32(codes, count, block_size, b0, b1, sizes):
    return _block_sizes(32, codes, count, block_size, b0, b1, sizes)


def block_sizes_u64(codes, count, block_size, b0, b1, sizes):
    return _block_sizes(64, codes, count, block_size, b0, b1, sizes)


def _emit_blocks(width, codes, lossless, count, block_size, b0, b1, offsets, out):
    if b1 <= b0:
        return 0
    s0, s1 = _span(count, block_size, b0, b1)
    lo = int(offsets[b0])
    hi = int(offsets[b1]) if b1 < len(offsets) else len(out)
    if hi <= lo:
        return 0
    with _lane() as ln:
        c = ln.up("c", codes[s0:s1])
        ll = ln.up("l", np.asarray(lossless[s0:s1], dtype=np.bool_))
        offs = ln.up("f", np.asarray(offsets[b0:b1], dtype=np.int64) - lo)
        o = ln.devbuf("o", hi - lo)
        _lib.call(f"gebq_emit_blocks_u{width}", device._p(c), device._p(ll), s1 - s0,
                  int(block_size), 0, int(b1) - int(b0), device._p(offs), device._p(o), device._s())
        ho = ln.down("o", o)
        ln.sync()
        out[lo:hi] = ho.numpy()
    return 0


def emit_blocks_u32(codes, lossless, count, block_size, b0, b1, offsets, out):
    return _emit_blocks(32, codes, lossless, count, block_size, b0, b1, offsets, out)


def emit_blocks_u64(codes, lossless, count, block_size, b0, b1, offsets, out):
    return _emit_blocks(64, codes, lossless, count, block_size, b0, b1, offsets, out)


def _decode_blocks(width, buf, offsets, region_end, count, block_size, b0, b1, codes, lossless):
    if b1 <= b0:
        return DEC_OK, np.int64(0)
    b0, b1 = int(b0), int(b1)
    s0, s1 = _span(count, block_size, b0, b1)
    lo = int(offsets[b0])
    # the span's bytes: up to the next block's offset, or region_end for the last
    end = int(offsets[b1]) if b1 < len(offsets) else int(region_end)
    end = min(max(end, lo), len(buf), int(region_end))
    lo_c = min(lo, end)
    with _lane() as ln:
        region = ln.up("r", np.asarray(buf[lo_c:end], dtype=np.uint8))
        offs = ln.up("f", np.asarray(offsets[b0:min(b1 + 1, len(offsets))], dtype=np.int64) - lo_c)
        c = ln.devbuf("c", (s1 - s0) * width // 8).view(_IT[width])
        ll = ln.devbuf("l", s1 - s0)
        ll.zero_()
        err = ln.devbuf("e", 8).view(torch.int64)
        err.fill_(-1)
        # the uploaded bytes end at `end`: it is the last block's end position when
        # the index has no next offset, and the kernel's read limit either way
        _lib.call(f"gebq_decode_blocks_u{width}", device._p(region), device._p(offs), offs.numel() // 8,
                  end - lo_c, s1 - s0, int(block_size), 0, b1 - b0, device._p(c),
                  device._p(ll), device._p(err), device._s())
        hc = ln.down("c", c.view(torch.uint8))
        hl = ln.down("l", ll)
        he = ln.down("e", err.view(torch.uint8))
        ln.sync()
        key = int(he.numpy().view(np.int64)[0]) & ((1 << 64) - 1)
        codes[s0:s1] = hc.numpy().view(codes.dtype)
        lossless[s0:s1] = hl.numpy().view(np.bool_)
    if key == (1 << 64) - 1:
        return DEC_OK, np.int64(0)
    return int(key & 3), np.int64((key >> 2) + lo_c)


def decode_blocks_u32(buf, offsets, region_end, count, block_size, b0, b1, codes, lossless):
    return _decode_blocks(32, buf, offsets, region_end, count, block_size, b0, b1, codes, lossless)


def decode_blocks_u64(buf, offsets, region_end, count, block_size, b0, b1, codes, lossless):
    return _decode_blocks(64, buf, offsets, region_end, count, block_size, b0, b1, codes, lossless)


# ---- sweeps (_kernels.py:717-896) -------------------------------------------
def _sweep_on(bits, cfg):
    n = len(bits)
    if n == 0:
        return np.zeros((5, 3), dtype=np.int64), np.int64(-1)
    tally, first = device.sweep(cfg, source=device.SOURCE_ARRAY, count=n,
                                bits=device.to_device(np.ascontiguousarray(bits)))
    f = int(first.item()) & ((1 << 64) - 1)
    return tally.cpu().numpy().reshape(5, 3), np.int64(-1 if f == (1 << 64) - 1 else f)


def sweep_abs32_on(bits, vals, eb_eff, eb2, inv_eb2, thr, unsafe):
    return _sweep_on(bits, _Cfg("abs", 32, unsafe, eb_eff=np.float32(eb_eff), eb2=np.float32(eb2),
                                inv_eb2=np.float32(inv_eb2), thr=np.float32(thr)))


def sweep_abs64_on(bits, vals, eb_eff, eb2, inv_eb2, thr, unsafe):
    return _sweep_on(bits, _Cfg("abs", 64, unsafe, eb_eff=np.float64(eb_eff), eb2=np.float64(eb2),
                                inv_eb2=np.float64(inv_eb2), thr=np.float64(thr)))


def sweep_rel32_on(bits, vals, op_eps, w, thr, unsafe):
    return _sweep_on(bits, _Cfg("rel", 32, unsafe, op_eps=np.float32(op_eps), w=np.float32(w),
                                thr=np.float32(thr)))


def sweep_rel64_on(bits, vals, op_eps, w, thr, unsafe):
    return _sweep_on(bits, _Cfg("rel", 64, unsafe, op_eps=np.float64(op_eps), w=np.float64(w),
                                thr=np.float64(thr)))


# ---- splitmix64_fill (_kernels.py:679-685) ----------------------------------
def splitmix64_fill(out, seed, start_index):
    n = len(out)
    if n:
        out[...] = device.splitmix64(n, int(seed), int(start_index)).cpu().numpy().view(np.uint64)
    return 0
