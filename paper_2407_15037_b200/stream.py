"""Device-resident FORMAT.md streams: fused encode (quantize + pack) and fused
decode (unpack + reconstruct) through libgebq_b200.so.

Device stream buffer layout (one allocation, so one D2H moves a whole stream):

    [0, 48)            header (filled on the host: it is 48 bytes of scalars)
    [48, 56)           u64 block count N
    [56, 56 + 8N)      block index (u64 offsets relative to the region)
    [56 + 8N, ...)     block region, written by the encode kernel
"""

from __future__ import annotations

import ctypes
import os
import struct
import threading
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .container import (HEADER_SIZE, FLAG_NO_DOUBLE_CHECK, StreamHeader, TruncatedStream,
                        raise_for_err_key)
from .device import _FTYPE, _ITYPE, _NP_ITYPE, _p, _s, _width_of, as_bits, require_cuda
from .quantizers import NOA, REL, QuantConfig

ERR_NONE = (1 << 64) - 1


def region_capacity(n: int, block_size: int, width: int) -> int:
    return int(_lib.load().gebq_encode_region_capacity(n, block_size, width))


def workspace_bytes(n: int, block_size: int, width: int) -> int:
    return int(_lib.load().gebq_encode_workspace_bytes(n, block_size, width))


@dataclass
class Encoded:
    """A stream produced on the device (header bytes not yet written)."""

    buf: torch.Tensor          # uint8 device buffer, layout in the module docstring
    nblocks: int
    count: int
    width: int
    region_len: torch.Tensor   # int64[1] device
    trig: torch.Tensor         # int64[4] device
    range_f64: Optional[torch.Tensor] = None  # NOA range computed on device

    @property
    def region_off(self) -> int:
        return HEADER_SIZE + 8 + 8 * self.nblocks


def alloc_stream(n: int, block_size: int, width: int, device) -> torch.Tensor:
    nblocks = -(-n // block_size) if n else 0
    cap = HEADER_SIZE + 8 + 8 * nblocks + region_capacity(n, block_size, width)
    return torch.empty(cap, dtype=torch.uint8, device=device)


def encode(x: torch.Tensor, cfg: QuantConfig, *, consts_dev: Optional[torch.Tensor] = None,
           base_offset: int = 0, buf: Optional[torch.Tensor] = None,
           ws: Optional[torch.Tensor] = None, trig: Optional[torch.Tensor] = None,
           region_len: Optional[torch.Tensor] = None) -> Encoded:
    """Quantize + pack ``x`` (a CUDA float/int tensor) into a stream buffer, one pass.

    ``consts_dev`` supplies NOA constants produced on the device (range pass
    -> derive) so the whole chain runs without a host round trip.
    """
    xb = as_bits(x)
    width = _width_of(xb)
    if width != cfg.width:
        raise TypeError(f"expected {cfg.width}-bit values for this config, got {width}-bit")
    n = xb.numel()
    bs = cfg.block_size
    nblocks = -(-n // bs) if n else 0
    dev = xb.device
    if buf is None:
        buf = alloc_stream(n, bs, width, dev)
    if ws is None:
        ws = torch.empty(max(workspace_bytes(n, bs, width), 16), dtype=torch.uint8, device=dev)
    if trig is None:
        trig = torch.zeros(4, dtype=torch.int64, device=dev)
    if region_len is None:
        region_len = torch.empty(1, dtype=torch.int64, device=dev)
    index = buf[HEADER_SIZE + 8:]
    region = buf[HEADER_SIZE + 8 + 8 * nblocks:]
    sfx = "f32" if width == 32 else "f64"
    F = ctypes.c_float if width == 32 else ctypes.c_double
    unsafe = int(bool(cfg.unsafe_no_double_check))
    common = (_p(region), _p(index), base_offset, _p(ws), ws.numel(), _p(trig), _p(region_len), _s())
    if consts_dev is not None:
        _lib.call(f"gebq_encode_noa_dev_{sfx}", _p(xb), n, _p(consts_dev), unsafe, bs, *common)
    elif cfg.mode == REL:
        d = cfg.derived
        _lib.call(f"gebq_encode_rel_{sfx}", _p(xb), n, F(d.op_eps), F(d.w), F(d.thr), unsafe, bs,
                  *common)
    else:
        d = cfg.derived
        _lib.call(f"gebq_encode_abs_{sfx}", _p(xb), n, F(d.eb_eff), F(d.eb2), F(d.inv_eb2),
                  F(d.thr), unsafe, bs, *common)
    return Encoded(buf=buf, nblocks=nblocks, count=n, width=width, region_len=region_len,
                   trig=trig)


COMPRESS_CHUNK = 32 << 20   # input bytes per pipelined span (whole blocks)
D2H_SLOT = 32 << 20


def _encode_span(xb: torch.Tensor, cfg: QuantConfig, region_ptr: int, index_ptr: int,
                 ws: torch.Tensor, trig: torch.Tensor, rl_ptr: int) -> None:
    """One encode launch over ``xb`` (whole blocks) into explicit output pointers."""
    width = cfg.width
    n = xb.numel()
    sfx = "f32" if width == 32 else "f64"
    F = ctypes.c_float if width == 32 else ctypes.c_double
    unsafe = int(bool(cfg.unsafe_no_double_check))
    d = cfg.derived
    common = (ctypes.c_void_p(region_ptr), ctypes.c_void_p(index_ptr), 0, _p(ws), ws.numel(),
              _p(trig), ctypes.c_void_p(rl_ptr), _s())
    if cfg.mode == REL:
        _lib.call(f"gebq_encode_rel_{sfx}", _p(xb), n, F(d.op_eps), F(d.w), F(d.thr), unsafe,
                  cfg.block_size, *common)
    else:
        _lib.call(f"gebq_encode_abs_{sfx}", _p(xb), n, F(d.eb_eff), F(d.eb2), F(d.inv_eb2),
                  F(d.thr), unsafe, cfg.block_size, *common)


def compress_pipelined(arr: np.ndarray, cfg: QuantConfig, header: StreamHeader):
    """Host values -> stream bytes with PCIe in both directions overlapped.

    The array is cut into spans of whole blocks (~COMPRESS_CHUNK bytes).  Span
    i is copied in on a side stream while span i-1 is encoded; each span's
    block region returns on a third stream as soon as its length is known and
    is copied straight into the result ``bytes`` at its final offset, so the
    result is complete (index entries shifted by the preceding spans'
    lengths) when the last span lands.  Constants must be known up front (not
    the NOA range pass).  Returns (stream bytes, trigger counts int64[4]).
    """
    from . import hostio

    dev = require_cuda()
    width = cfg.width
    W = width // 8
    n = arr.size
    bs = cfg.block_size
    nblocks = -(-n // bs)
    per = max(bs, (COMPRESS_CHUNK // W) // bs * bs)
    spans = [(v0, min(v0 + per, n)) for v0 in range(0, n, per)]
    caps = [region_capacity(v1 - v0, bs, width) for v0, v1 in spans]
    capoff = np.concatenate([[0], np.cumsum(caps)]).astype(np.int64)
    src = hostio.host_u8(arr)
    x = torch.empty(n, dtype=_ITYPE[width], device=dev)
    xb8 = x.view(torch.uint8)
    regions = torch.empty(int(capoff[-1]) + 16, dtype=torch.uint8, device=dev)
    index = torch.empty(max(nblocks, 1), dtype=torch.int64, device=dev)
    ws = torch.empty(max(workspace_bytes(per, bs, width), 16), dtype=torch.uint8, device=dev)
    trig = torch.zeros(4, dtype=torch.int64, device=dev)
    rl = torch.empty(len(spans), dtype=torch.int64, device=dev)
    rl_host = torch.empty(len(spans), dtype=torch.int64, pin_memory=True)
    hdr_len = HEADER_SIZE + 8 + 8 * nblocks
    out = hostio.BytesBuilder(hdr_len + int(capoff[-1]))
    cur = torch.cuda.current_stream(dev)
    out_stream = _out_stream(dev)
    ring = _d2h_ring(dev)
    pipe = hostio.H2DPipe(src, xb8)
    enc_ev = []

    def launch(c):
        v0, v1 = spans[c]
        cur.wait_event(pipe.push(v0 * W, v1 * W))
        _encode_span(x[v0:v1], cfg, regions.data_ptr() + int(capoff[c]),
                     index.data_ptr() + 8 * (v0 // bs), ws, trig, rl.data_ptr() + 8 * c)
        rl_host[c:c + 1].copy_(rl[c:c + 1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(cur)
        enc_ev.append(ev)

    bases = []
    state = {"base": 0, "k": 0}

    def drain(c):
        enc_ev[c].synchronize()
        if _TRACE is not None:
            _TRACE.append((f"enc{c} done", time.perf_counter()))
        L = int(rl_host[c])
        base = state["base"]
        bases.append(base)
        src_dev = regions[int(capoff[c]):int(capoff[c]) + L]
        dst = out.view[hdr_len + base:hdr_len + base + L]
        _d2h_ring_copy(ring, out_stream, enc_ev[c], src_dev, dst, state)
        state["base"] = base + L

    if pipe.pinned:          # every span's copy and encode queued at once
        for c in range(len(spans)):
            launch(c)
        for c in range(len(spans)):
            drain(c)
    else:                    # staging copies interleave with draining the previous span
        for c in range(len(spans)):
            launch(c)
            if c:
                drain(c - 1)
        drain(len(spans) - 1)
    _d2h_ring_flush(ring, state)
    total = state["base"]
    # index: span-relative entries -> stream offsets
    if nblocks:
        out.view[HEADER_SIZE + 8:hdr_len].copy_(index.view(torch.uint8)[:8 * nblocks])
        idx = out.view[HEADER_SIZE + 8:hdr_len].numpy().view("<u8")
        for (v0, v1), b in zip(spans, bases):
            idx[v0 // bs:-(-v1 // bs)] += np.uint64(b)
    prefix = header.pack() + struct.pack("<Q", nblocks)
    out.view[:len(prefix)].copy_(torch.frombuffer(bytearray(prefix), dtype=torch.uint8))
    trig_h = trig.cpu().numpy()
    r = out.finish(hdr_len + total)
    if _TRACE is not None:
        _TRACE.append(("finished", time.perf_counter()))
    return r, trig_h


_TRACE = None               # optional list of (event, perf_counter) for host-timeline probes
_LOCAL = threading.local()   # per-thread staging rings / streams (concurrent callers never share)


def _d2h_ring(dev):
    k = dev.index if dev.index is not None else torch.cuda.current_device()
    rings = _LOCAL.__dict__.setdefault("rings", {})
    if k not in rings:
        rings[k] = ([torch.empty(D2H_SLOT, dtype=torch.uint8, pin_memory=True) for _ in range(2)],
                    [torch.cuda.Event() for _ in range(2)])
    return rings[k]


def _d2h_ring_copy(ring, stream, after: torch.cuda.Event, src: torch.Tensor, dst: torch.Tensor, state):
    """Device bytes -> pageable host bytes through two pinned slots: the DMA of
    one slot overlaps the host copy out of the other."""
    slots, evs = ring
    pend = state.setdefault("pend", [])
    stream.wait_event(after)
    n = src.numel()
    for off in range(0, n, D2H_SLOT):
        m = min(D2H_SLOT, n - off)
        k = state["k"]
        state["k"] = k ^ 1
        if len(pend) == 2:                     # the slot about to be reused: finish its host copy
            pk, pdst, pm = pend.pop(0)
            evs[pk].synchronize()
            if _TRACE is not None:
                _TRACE.append((f"slot{pk} dma done", time.perf_counter()))
            pdst.copy_(slots[pk][:pm])
            if _TRACE is not None:
                _TRACE.append((f"slot{pk} host copy done", time.perf_counter()))
        with torch.cuda.stream(stream):
            slots[k][:m].copy_(src[off:off + m], non_blocking=True)
        evs[k].record(stream)
        pend.append((k, dst[off:off + m], m))


def _d2h_ring_flush(ring, state):
    slots, evs = ring
    for pk, pdst, pm in state.pop("pend", []):
        evs[pk].synchronize()
        if _TRACE is not None:
            _TRACE.append((f"slot{pk} dma done (flush)", time.perf_counter()))
        pdst.copy_(slots[pk][:pm])
        if _TRACE is not None:
            _TRACE.append((f"slot{pk} host copy done (flush)", time.perf_counter()))


def encode_coded(codes: torch.Tensor, lossless: torch.Tensor, block_size: int, *,
                 base_offset: int = 0) -> Encoded:
    """Pack given wire codes + flags (container.encode_stream) on the device."""
    cb = as_bits(codes)
    width = _width_of(cb)
    n = cb.numel()
    dev = cb.device
    nblocks = -(-n // block_size) if n else 0
    buf = alloc_stream(n, block_size, width, dev)
    ws = torch.empty(max(workspace_bytes(n, block_size, width), 16), dtype=torch.uint8, device=dev)
    region_len = torch.empty(1, dtype=torch.int64, device=dev)
    if lossless.dtype == torch.bool:
        lossless = lossless.view(torch.uint8)
    index = buf[HEADER_SIZE + 8:]
    region = buf[HEADER_SIZE + 8 + 8 * nblocks:]
    _lib.call(f"gebq_encode_coded_u{width}", _p(cb), _p(lossless.contiguous()), n, block_size,
              _p(region), _p(index), base_offset, _p(ws), ws.numel(), _p(region_len), _s())
    return Encoded(buf=buf, nblocks=nblocks, count=n, width=width, region_len=region_len,
                   trig=torch.zeros(4, dtype=torch.int64, device=dev))


def stream_to_host(enc: Encoded, header: StreamHeader, region_len: Optional[int] = None) -> bytes:
    """Assemble the final stream bytes: host header + index + region, D2H'd in place."""
    from . import hostio

    if region_len is None:
        region_len = int(enc.region_len.item())
    total = enc.region_off + region_len
    prefix = header.pack() + struct.pack("<Q", enc.nblocks)
    return hostio.device_to_new_bytes(enc.buf[HEADER_SIZE + 8:total], prefix)


def header_for(cfg: QuantConfig, count: int, value_range=None) -> StreamHeader:
    """Header of pipeline.compress (pipeline.py:178-187)."""
    vr = value_range if value_range is not None else cfg.value_range
    return StreamHeader(
        width=cfg.width, mode=cfg.mode, count=count,
        eb_bits=int(np.float64(cfg.eb).view(np.uint64)),
        derived_bits=cfg.derived.header_bits,
        range_bits=int(np.float64(vr or 0.0).view(np.uint64)) if cfg.mode == NOA else 0,
        block_size=cfg.block_size,
        flags=FLAG_NO_DOUBLE_CHECK if cfg.unsafe_no_double_check else 0)


# ---------------------------------------------------------------------------
# decode
# ---------------------------------------------------------------------------

def decode_values(stream_dev: torch.Tensor, header: StreamHeader, nblocks: int, *,
                  out: Optional[torch.Tensor] = None, err: Optional[torch.Tensor] = None,
                  index_pos: int = HEADER_SIZE + 8,
                  region_len_dev: Optional[torch.Tensor] = None,
                  derived_dev: Optional[torch.Tensor] = None):
    """Fused unpack + reconstruct of a device-resident stream -> value bits.

    The index must already be validated (container.parse_layout or
    :func:`validate_index`).  ``region_len_dev`` / ``derived_dev`` let the
    decode consume the encoder's device-side outputs (region length, NOA eb2)
    with no host round trip.  Returns (values int tensor, err_key int64[1]).
    """
    width = header.width
    dev = stream_dev.device
    if out is None:
        out = torch.empty(header.count, dtype=_ITYPE[width], device=dev)
    if err is None:
        err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    region_pos = index_pos + 8 * nblocks
    region_len = stream_dev.numel() - region_pos
    offsets = stream_dev[index_pos:]
    region = stream_dev[region_pos:]
    kind = "rel" if header.mode == REL else "abs"
    sfx = "f32" if width == 32 else "f64"
    F = ctypes.c_float if width == 32 else ctypes.c_double
    if header.count:
        rl = _p(region_len_dev) if region_len_dev is not None else ctypes.c_void_p(0)
        dd = _p(derived_dev) if derived_dev is not None else ctypes.c_void_p(0)
        _lib.call(f"gebq_decode_{kind}_{sfx}", _p(region), region_len, rl, _p(offsets), nblocks,
                  header.count, header.block_size, F(header.derived_value), dd, _p(out), _p(err),
                  _s())
    return out, err


def decode_codes(stream_dev: torch.Tensor, header: StreamHeader, nblocks: int, *,
                 index_pos: int = HEADER_SIZE + 8):
    """Unpack a device-resident stream to (codes, lossless u8, err_key)."""
    width = header.width
    dev = stream_dev.device
    codes = torch.empty(header.count, dtype=_ITYPE[width], device=dev)
    lossless = torch.empty(header.count, dtype=torch.uint8, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    region_pos = index_pos + 8 * nblocks
    region_len = stream_dev.numel() - region_pos
    if header.count:
        _lib.call(f"gebq_decode_blocks_u{width}", _p(stream_dev[region_pos:]),
                  _p(stream_dev[index_pos:]), nblocks, region_len, header.count,
                  header.block_size, 0, nblocks, _p(codes), _p(lossless), _p(err), _s())
    return codes, lossless, err


def validate_index(stream_dev: torch.Tensor, nblocks: int, index_pos: int = HEADER_SIZE + 8):
    """Device-side index checks -> int32[3] flags (first!=0, decreasing, beyond end)."""
    flags = torch.empty(3, dtype=torch.int32, device=stream_dev.device)
    region_len = stream_dev.numel() - index_pos - 8 * nblocks
    _lib.call("gebq_validate_index", _p(stream_dev[index_pos:]), nblocks, region_len, _p(flags),
              _s())
    return flags


def host_u8(data) -> torch.Tensor:
    from . import hostio

    return hostio.host_u8(data)


def _h2d_stream(data) -> torch.Tensor:
    from . import hostio

    dev = require_cuda()
    src = hostio.host_u8(data)
    n = src.numel()
    # keep 16 bytes of slack so vector loads near the end stay inside the allocation
    t = torch.empty(n + 16, dtype=torch.uint8, device=dev)
    hostio.h2d(src, t[:n])
    return t[:n]


# ---------------------------------------------------------------------------
# host wrappers used by container.py / pipeline.py
# ---------------------------------------------------------------------------

def encode_coded_host(codes: np.ndarray, lossless: np.ndarray, header: StreamHeader) -> bytes:
    from .device import to_device

    require_cuda()
    if header.count == 0:
        return header.pack() + struct.pack("<Q", 0)
    enc = encode_coded(to_device(codes), to_device(np.asarray(lossless, dtype=np.bool_)),
                       header.block_size)
    return stream_to_host(enc, header)


def decode_coded_host(data, header: StreamHeader, nblocks: int, index_pos: int):
    width = header.width
    if header.count == 0:
        return np.empty(0, _NP_ITYPE[width]), np.empty(0, np.bool_)
    sd = _h2d_stream(data)
    codes, lossless, err = decode_codes(sd, header, nblocks, index_pos=index_pos)
    key = int(err.item()) & ERR_NONE
    raise_for_err_key(key)
    return (codes.cpu().numpy().view(_NP_ITYPE[width]),
            lossless.cpu().numpy().view(np.bool_))


DECODE_CHUNK = 8 << 20    # stream bytes per pipelined span


def decode_values_host(data, header: StreamHeader, nblocks: int, index_pos: int) -> np.ndarray:
    """Host stream -> host values, PCIe in both directions overlapped with the decode.

    The stream is cut into spans of whole blocks (~DECODE_CHUNK bytes each,
    from the already validated index): span i's bytes cross PCIe on a copy
    stream while span i-1 decodes on the compute stream and span i-2's values
    return on a third stream.  Errors are reduced over all spans into one key
    (the smallest failing position wins, container.py:308-311) and raised after
    the last span.
    """
    from . import hostio

    width = header.width
    ft = np.float32 if width == 32 else np.float64
    count = header.count
    if count == 0:
        return np.empty(0, ft)
    dev = require_cuda()
    src = hostio.host_u8(data)
    total = src.numel()
    region_pos = index_pos + 8 * nblocks
    region_len = total - region_pos
    offs = src[index_pos:region_pos].numpy().view("<i8")
    sd = torch.empty(total + 16, dtype=torch.uint8, device=dev)
    out = torch.empty(count, dtype=_ITYPE[width], device=dev)
    host = torch.empty(count, dtype=_ITYPE[width], pin_memory=True)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    kind = "rel" if header.mode == REL else "abs"
    fn = getattr(_lib.load(), f"gebq_decode_span_{kind}_{'f32' if width == 32 else 'f64'}")
    F = ctypes.c_float if width == 32 else ctypes.c_double
    derived = F(header.derived_value)
    bs = header.block_size
    cur = torch.cuda.current_stream(dev)
    out_stream = _out_stream(dev)
    pipe = hostio.H2DPipe(src, sd)
    region_p, offs_p = sd.data_ptr() + region_pos, sd.data_ptr() + index_pos
    b0, lo = 0, 0
    while b0 < nblocks:
        # next span: whole blocks up to ~DECODE_CHUNK stream bytes past this span's start
        b1 = int(np.searchsorted(offs, offs[b0] + DECODE_CHUNK, side="left"))
        b1 = min(max(b1, b0 + 1), nblocks)
        hi = region_pos + (int(offs[b1]) if b1 < nblocks else region_len)
        cur.wait_event(pipe.push(lo, hi))
        rc = fn(region_p, region_len, offs_p, nblocks, count, bs, derived, b0, b1, _p(out),
                _p(err), _s())
        if rc != 0:
            raise _lib.GebqCudaError(f"decode span failed ({rc}): {_lib.last_error()}")
        v0, v1 = b0 * bs, min(b1 * bs, count)
        out_stream.wait_stream(cur)
        with torch.cuda.stream(out_stream):
            host[v0:v1].copy_(out[v0:v1], non_blocking=True)
        b0, lo = b1, hi
    cur.wait_stream(out_stream)
    key = int(err.item()) & ERR_NONE                 # syncs the compute stream (after all copies)
    raise_for_err_key(key)
    return host.numpy().view(ft)


def _out_stream(dev) -> torch.cuda.Stream:
    k = dev.index if dev.index is not None else torch.cuda.current_device()
    streams = _LOCAL.__dict__.setdefault("out_streams", {})
    if k not in streams:
        streams[k] = torch.cuda.Stream(device=dev)
    return streams[k]
