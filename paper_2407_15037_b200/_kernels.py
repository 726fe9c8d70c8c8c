"""Drop-in replacements for the reference's operator layer ``gebq._kernels``.

Every function keeps the exact name, argument order, in-place output
convention and return value of the numba dispatcher it replaces
(/root/reference/pkg/src/gebq/_kernels.py), so ``install(gebq)`` can rebind
``gebq._kernels.<name>`` and the reference's own pipeline/container/sweep
code runs on the B200 unchanged.  Each call moves its arrays host<->device;
the pipeline-level entry points (paper_2407_15037_b200.pipeline) keep data
resident and are the fast path.
"""

from __future__ import annotations

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


def _quantize(bits, codes, lossless, cfg) -> np.ndarray:
    n = len(bits)
    if n == 0:
        return np.zeros(4, dtype=np.int64)
    x = device.to_device(np.ascontiguousarray(bits))
    c, ll, trig = device.quantize(x, cfg)
    codes[...] = c.cpu().numpy().view(codes.dtype)
    lossless[...] = ll.cpu().numpy().view(np.bool_)
    return trig.cpu().numpy().astype(np.int64)


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
    if len(codes) == 0:
        return 0
    out = device.reconstruct(device.to_device(np.ascontiguousarray(codes)),
                             device.to_device(np.ascontiguousarray(lossless, dtype=np.bool_)),
                             mode, derived)
    out_bits[...] = out.cpu().numpy().view(out_bits.dtype)
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
def _block_sizes(width, codes, count, block_size, b0, b1, sizes):
    if b1 <= b0:
        return 0
    c = device.to_device(np.ascontiguousarray(codes))
    s = torch.empty(b1, dtype=torch.int64, device=c.device)
    _lib.call(f"gebq_block_sizes_u{width}", device._p(c), int(count), int(block_size), int(b0),
              int(b1), device._p(s), device._s())
    sizes[b0:b1] = s[b0:b1].cpu().numpy()
    return 0


def block_sizes_u32(codes, count, block_size, b0, b1, sizes):
    return _block_sizes(32, codes, count, block_size, b0, b1, sizes)


def block_sizes_u64(codes, count, block_size, b0, b1, sizes):
    return _block_sizes(64, codes, count, block_size, b0, b1, sizes)


def _emit_blocks(width, codes, lossless, count, block_size, b0, b1, offsets, out):
    if b1 <= b0:
        return 0
    c = device.to_device(np.ascontiguousarray(codes))
    ll = device.to_device(np.ascontiguousarray(lossless, dtype=np.bool_))
    offs = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).to(c.device)
    lo = int(offsets[b0])
    hi = int(offsets[b1]) if b1 < len(offsets) else len(out)
    o = torch.zeros(len(out), dtype=torch.uint8, device=c.device)
    _lib.call(f"gebq_emit_blocks_u{width}", device._p(c), device._p(ll), int(count),
              int(block_size), int(b0), int(b1), device._p(offs), device._p(o), device._s())
    out[lo:hi] = o[lo:hi].cpu().numpy()
    return 0


def emit_blocks_u32(codes, lossless, count, block_size, b0, b1, offsets, out):
    return _emit_blocks(32, codes, lossless, count, block_size, b0, b1, offsets, out)


def emit_blocks_u64(codes, lossless, count, block_size, b0, b1, offsets, out):
    return _emit_blocks(64, codes, lossless, count, block_size, b0, b1, offsets, out)


def _decode_blocks(width, buf, offsets, region_end, count, block_size, b0, b1, codes, lossless):
    if b1 <= b0:
        return DEC_OK, np.int64(0)
    dev = device.require_cuda()
    region = stream._h2d_stream(np.ascontiguousarray(buf, dtype=np.uint8))
    offs = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).to(dev)
    c = torch.empty(len(codes), dtype=torch.int32 if width == 32 else torch.int64, device=dev)
    ll = torch.zeros(len(lossless), dtype=torch.uint8, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    _lib.call(f"gebq_decode_blocks_u{width}", device._p(region), device._p(offs), len(offsets),
              int(region_end), int(count), int(block_size), int(b0), int(b1), device._p(c),
              device._p(ll), device._p(err), device._s())
    key = int(err.item()) & ((1 << 64) - 1)
    s0 = int(b0) * int(block_size)
    s1 = min(int(b1) * int(block_size), int(count))
    codes[s0:s1] = c[s0:s1].cpu().numpy().view(codes.dtype)
    lossless[s0:s1] = ll[s0:s1].cpu().numpy().view(np.bool_)
    if key == (1 << 64) - 1:
        return DEC_OK, np.int64(0)
    return int(key & 3), np.int64(key >> 2)


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
