"""The multi-GPU device path, executed for real with more than one rank
(VERDICT r1 item 5): two processes share the one GPU of the test box and talk
over ``gloo`` with CUDA tensors (NCCL refuses two ranks on one device).  Each
rank generates its block-aligned shard of a global array on the device, runs
``compress_sharded_device`` with the real CUDA encoder (no stand-in), NOA
reduces its order keys with the one MAX all-reduce, and rank 0 assembles the
stream: it must be byte-identical to the single-GPU stream and the oracle's.
The C4 sweep shards its 2^32 pattern range the same way; the summed tallies
must equal Appendix B.  Also: the C-ABI NCCL exchange (gebq_noa_allreduce) on
a one-rank NCCL communicator."""

import ctypes
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = (1 << 22) + 4096 * 3 + 17


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_input(kind, width, start, n, total, dev):
    from paper_2407_15037_b200 import device as gdev
    from paper_2407_15037_b200 import workloads

    if kind == "smooth":
        return gdev.smooth_field(n, 256, workloads.C3_SEED, start, width, plant=True, total=total, device=dev)
    if width == 32:
        return gdev.mixed_f32(n, workloads.C2_SEED, start, device=dev)
    return gdev.splitmix64(n, workloads.C5_SEED, start, device=dev)


CASES = [("abs", 1e-3, 32, "mixed"), ("rel", 1e-2, 32, "mixed"), ("noa", 1e-4, 32, "smooth"),
         ("abs", 1e-3, 64, "mixed"), ("rel", 1e-3, 64, "mixed"), ("noa", 1e-4, 64, "smooth"),
         ("abs", 1e-3, 32, "smooth")]


def _worker(rank, world, port, errq):
    try:
        import torch
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2407_15037_b200 as g
        from oracle import oracle as orc
        from paper_2407_15037_b200 import distributed as D
        from paper_2407_15037_b200 import device as gdev

        for mode, eb, width, kind in CASES:
            cfg = g.QuantConfig(mode=mode, eb=eb, width=width)
            s, e = D.shard_bounds(N, world, rank, cfg.block_size)
            x_local = _global_input(kind, width, s, e - s, N, dev)
            part, header, trig = D.compress_sharded_device(x_local, cfg)   # real CUDA encoder
            tt = torch.from_numpy(np.asarray(trig, dtype=np.int64)).to(dev)
            dist.all_reduce(tt)
            parts = D.gather_parts(part)
            if rank == 0:
                got = D.assemble_stream(header, parts)
                xg = _global_input(kind, width, 0, N, N, dev)
                xh = xg.cpu().numpy().view(np.float32 if width == 32 else np.float64)
                one, st = g.compress(xh, cfg)
                assert got == one, (mode, width, kind, "sharded != single-GPU")
                exp, etrig, _ = orc.compress(xh, mode, eb, workers=8)
                assert got == exp, (mode, width, kind, "sharded != oracle")
                assert tt.cpu().tolist() == list(etrig)
            dist.barrier()
        # C4: the 2^32 range sharded over the ranks, tallies summed
        cfg = g.QuantConfig(mode="abs", eb=1e-3, width=32)
        per = (1 << 32) // world
        tally, first = gdev.sweep(cfg, source=gdev.SOURCE_RANGE, start=rank * per,
                                  count=(1 << 32) - rank * per if rank == world - 1 else per)
        dist.all_reduce(tally)
        t = tally.cpu().numpy().reshape(5, 3)
        assert t[2, 0] == 2443713898 and t[2, 1] == 1817698966 and t[:, 2].sum() == 0
        assert t.sum() == 1 << 32
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover - reported to the parent
        import traceback

        errq.put(f"rank {rank}: {ex!r}\n{traceback.format_exc()}")


def test_two_ranks_real_device_path(cuda):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)


class _NcclId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


def test_noa_allreduce_c_abi_single_rank_nccl(cuda):
    """gebq_noa_allreduce on a one-rank NCCL communicator (the plumbing a C
    consumer uses; identity for one rank), and a clean error on a null comm."""
    import torch

    from paper_2407_15037_b200 import _lib
    from paper_2407_15037_b200 import device as gdev
    from paper_2407_15037_b200 import workloads

    nccl = ctypes.CDLL("libnccl.so.2")
    uid = _NcclId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    try:
        x = gdev.smooth_field(1 << 20, 256, workloads.C3_SEED, 0, 32, plant=True, total=1 << 20)
        keys = gdev.noa_keys(x)
        before = keys.clone()
        _lib.call("gebq_noa_allreduce", ctypes.c_void_p(keys.data_ptr()), comm,
                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert torch.equal(keys, before)
        _, rng = gdev.noa_derive(keys, 1e-4, 32)
        assert float(rng.item()) == 14.0
        with pytest.raises(Exception):
            _lib.call("gebq_noa_allreduce", ctypes.c_void_p(keys.data_ptr()), ctypes.c_void_p(0),
                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    finally:
        nccl.ncclCommDestroy(comm)
