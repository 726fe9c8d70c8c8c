"""Multi-rank plumbing on CPU: world_size-2 gloo groups run the sharding,
NOA key all-reduce, region-base scan and stream assembly of
paper_2407_15037_b200.distributed; the per-shard device encode is stood in
for by the CPU oracle, so the assembled stream must be byte-identical to the
oracle's single-array stream."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import mixed_bits


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _order_keys(bits: np.ndarray, width: int) -> np.ndarray:
    """Host restatement of k_noa_minmax's keys (test helper)."""
    if width == 32:
        b = bits.astype(np.uint64)
        finite = ((b >> 23) & 0xFF) != 0xFF
        key = np.where(b & 0x80000000, (~b) & 0xFFFFFFFF, b | 0x80000000)[finite]
        if key.size == 0:
            return np.array([0, 0], dtype=np.int64)
        return np.array([key.max(), ((~key) & 0xFFFFFFFF).max()], dtype=np.int64)
    raise NotImplementedError


def _keys_to_range(keys, width):
    kmax, kmin_c = int(keys[0]), int(keys[1])
    if kmax == 0:
        return np.float32(0.0)
    kmin = (~kmin_c) & 0xFFFFFFFF
    dec = lambda k: (k & 0x7FFFFFFF) if k & 0x80000000 else (~k) & 0xFFFFFFFF
    bmax, bmin = dec(kmax), dec(kmin)
    return np.uint32(bmax).view(np.float32) - np.uint32(bmin).view(np.float32)


def _worker(rank, world, port, cases, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import oracle as orc
        from paper_2407_15037_b200 import distributed as D
        from paper_2407_15037_b200.quantizers import QuantConfig

        for mode, eb, width, bs, n, vr in cases:
            bits = mixed_bits(width, n, 77 + n)[:n]
            ft = np.float32 if width == 32 else np.float64
            vals = np.concatenate([bits.view(ft), np.linspace(-3, 3, 3000).astype(ft)])
            n_all = len(vals)
            s, e = D.shard_bounds(n_all, world, rank, bs)
            local = vals[s:e]
            assert s % bs == 0
            cfg = QuantConfig(mode=mode, eb=eb, width=width, block_size=bs, value_range=vr)

            def encode_local(x, cfg_):
                xb = x.numpy().view(np.uint32 if width == 32 else np.uint64)
                c = orc.derive(cfg_.mode, cfg_.eb, width, cfg_.value_range)
                codes, ll, trig = orc.quantize(xb, cfg_.mode, c)
                offs, region = orc.encode_payload(codes, ll, bs)
                return offs.astype(np.uint64), region.tobytes(), trig

            x_local = torch.from_numpy(local.view(np.int32 if width == 32 else np.int64).copy())
            part, header, trig = D.compress_sharded_device(x_local, cfg, encode_local=encode_local)
            parts = D.gather_parts(part)
            if rank == 0:
                got = D.assemble_stream(header, parts)
                exp, _, _ = orc.compress(vals, mode, eb, vr, block_size=bs)
                assert got == exp, (mode, width, bs)
        # NOA global range from shard keys (one MAX all-reduce)
        vals = np.concatenate([np.linspace(-1, 2, 5000), [7.0, np.nan]]).astype(np.float32)
        if rank == 1:
            vals = np.concatenate([vals, [-7.0, np.inf]]).astype(np.float32)
        keys = torch.from_numpy(_order_keys(vals.view(np.uint32), 32))
        D.global_noa_keys(keys)
        assert float(_keys_to_range(keys.numpy(), 32)) == 14.0
        base, total, lens = D.region_bases(100 + rank)
        assert lens == [100, 101] and base == (0 if rank == 0 else 100) and total == 201
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


def test_two_rank_sharded_stream_is_byte_identical():
    cases = [("abs", 1e-3, 32, 4096, 20000, None), ("rel", 1e-2, 32, 4096, 30000, None),
             ("noa", 1e-3, 32, 1000, 12000, 2.5), ("abs", 1e-3, 64, 512, 9000, None),
             ("rel", 1e-3, 64, 4096, 9000, None)]
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.parametrize("n,world,bs", [(0, 2, 4096), (1, 2, 4096), (4096 * 3 + 5, 2, 4096),
                                        (4096 * 8, 8, 4096), (10000, 3, 7), (2**30, 8, 4096)])
def test_shard_bounds_partition(n, world, bs):
    from paper_2407_15037_b200.distributed import shard_bounds

    prev = 0
    for r in range(world):
        s, e = shard_bounds(n, world, r, bs)
        assert s == prev and s <= e and (s % bs == 0 or s == n)
        prev = e
    assert prev == n
