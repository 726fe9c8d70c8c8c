"""Multi-GPU sharding of the stream path: one process per GPU, torch.distributed.

The path is an elementwise map over container blocks, so it shards
contiguously with NO data-path collective, except NOA's global range:

* every rank owns a contiguous, block-aligned slice of the global array
  (shard boundaries are multiples of ``block_size``), so each rank emits whole
  container blocks and the concatenation of the shards' block regions, in rank
  order, is byte-identical to the single-device stream;
* NOA: each rank reduces its slice to two order keys (max, ~min) on the
  device; ONE ``all_reduce(MAX)`` of 2 x int64 over NCCL (NVLink/NVSwitch)
  gives the global range, then every rank derives identical constants on the
  device (quantizers.py:106-116) -- no host round trip on the data path;
* stream assembly: each rank's index entries are relative to its own region;
  an exclusive scan of the G region lengths (a G-scalar all_gather) gives the
  base offset added to them.  Assembling one byte stream is a gather to rank 0
  (only needed when a single file is wanted; shards can be written in place).

The collective plumbing is injectable (``encode_local``) so the host logic is
tested on CPU with ``gloo`` and world_size 2 while the device path runs the
CUDA kernels.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np
import torch
import torch.distributed as dist

from .container import HEADER_SIZE, StreamHeader

__all__ = ["shard_bounds", "global_noa_keys", "region_bases", "ShardPart", "assemble_stream",
           "compress_sharded_device"]


def shard_bounds(n: int, world: int, rank: int, block_size: int = 4096):
    """[start, end) of rank's contiguous block-aligned slice of an n-value array."""
    nblocks = -(-n // block_size) if n else 0
    per = -(-nblocks // world) if world else 0
    b0 = min(rank * per, nblocks)
    b1 = min(b0 + per, nblocks)
    return min(b0 * block_size, n), min(b1 * block_size, n)


def global_noa_keys(keys: torch.Tensor, group=None) -> torch.Tensor:
    """MAX all-reduce of the int64[2] (max-key, complemented-min-key) pair, in place."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MAX, group=group)
    return keys


def region_bases(local_len: int, group=None) -> tuple:
    """(base offset of this rank's region, total region length, all lengths)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return 0, local_len, [local_len]
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    mine = torch.tensor([local_len], dtype=torch.int64, device=dev)
    alls = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(alls, mine, group=group)
    lens = [int(t.item()) for t in alls]
    rank = dist.get_rank(group)
    return sum(lens[:rank]), sum(lens), lens


@dataclass
class ShardPart:
    """One rank's contribution to a stream: its block index (already rebased) and region."""

    index: np.ndarray   # uint64[nblocks_local], offsets relative to the GLOBAL region
    region: bytes


def assemble_stream(header: StreamHeader, parts: List[ShardPart]) -> bytes:
    """Header + global block count + concatenated indices + concatenated regions."""
    nblocks = sum(len(p.index) for p in parts)
    index = np.concatenate([p.index for p in parts]) if parts else np.empty(0, np.uint64)
    return (header.pack() + struct.pack("<Q", nblocks) + index.astype("<u8").tobytes()
            + b"".join(p.region for p in parts))


def gather_parts(part: ShardPart, group=None) -> Optional[List[ShardPart]]:
    """Gather every rank's ShardPart to rank 0 (object collective; None elsewhere)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return [part]
    world = dist.get_world_size(group)
    out = [None] * world if dist.get_rank(group) == 0 else None
    dist.gather_object(part, out, dst=0, group=group)
    return out


def compress_sharded_device(x_local: torch.Tensor, cfg, group=None,
                            encode_local: Optional[Callable] = None):
    """Compress this rank's slice; returns (ShardPart, header, trig int64[4]).

    ``x_local`` is the rank's block-aligned slice of the global array on its
    GPU.  The NOA range (if needed) is reduced across ranks with one MAX
    all-reduce; trigger counts stay per rank (sum them for global stats).
    """
    from . import device, stream
    from .quantizers import NOA

    consts = None
    if cfg.mode == NOA and cfg.value_range is None:
        keys = device.noa_keys(x_local)
        global_noa_keys(keys, group)
        consts, rng = device.noa_derive(keys, float(cfg.eb), cfg.width)
        r = rng.item()
        cfg = cfg.with_range(float(np.float32(r)) if cfg.width == 32 else r)
    if encode_local is None:
        enc = stream.encode(x_local, cfg, consts_dev=consts)
        local_len = int(enc.region_len.item())
        index = enc.buf[HEADER_SIZE + 8:HEADER_SIZE + 8 + 8 * enc.nblocks].cpu().numpy().view(np.uint64)
        region = enc.buf[enc.region_off:enc.region_off + local_len].cpu().numpy().tobytes()
        trig = enc.trig.cpu().numpy()
    else:
        index, region, trig = encode_local(x_local, cfg)
        local_len = len(region)
    base, total, _ = region_bases(local_len, group)
    part = ShardPart(index=(index.astype(np.uint64) + np.uint64(base)), region=region)
    n_global = int(x_local.numel())
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        t = torch.tensor([n_global], dtype=torch.int64,
                         device=x_local.device if x_local.is_cuda else "cpu")
        dist.all_reduce(t, group=group)
        n_global = int(t.item())
    header = stream.header_for(cfg, n_global)
    return part, header, trig
