"""Full-size parity at the BASELINE configurations: C3 (NOA
f32, 2^30 values, planted extremes) and C5 (f64 ABS / REL, 2^30 doubles,
random and smooth; streams larger than 2^32 bytes) through the public API
(``compress`` / ``decompress_to_array``) AND the single-launch device path
the bench times, byte-identical to the CPU oracle run on the host threads."""

import hashlib
import os

import numpy as np
import pytest

from helpers import trig_list

pytestmark = pytest.mark.gpu

N_FULL = 1 << 30


def _cfg(mode, eb, width):
    from paper_2407_15037_b200 import QuantConfig

    return QuantConfig(mode=mode, eb=eb, width=width)


def _workers():
    return os.cpu_count() or 8


def _equal_bytes(a, b, chunk=1 << 28) -> bool:
    """Chunked byte equality (avoids one more multi-GiB temporary)."""
    if len(a) != len(b):
        return False
    ma, mb = memoryview(a), memoryview(b)
    return all(ma[i:i + chunk] == mb[i:i + chunk] for i in range(0, len(a), chunk))


@pytest.mark.parametrize("start", [0, 5000, N_FULL - (1 << 20)])
@pytest.mark.parametrize("width", [32, 64])
def test_smooth_generator_matches_host_recipe(cuda, start, width):
    """device.smooth_field == workloads.smooth_field_cb bit for bit (any offset)."""
    from paper_2407_15037_b200 import device as gdev
    from paper_2407_15037_b200 import workloads

    n = 1 << 20
    plant = width == 32
    d = gdev.smooth_field(n, workloads.C3_SIDE, workloads.C3_SEED, start, width, plant=plant,
                          total=N_FULL).cpu().numpy()
    h = workloads.smooth_field_cb(n, workloads.C3_SIDE, workloads.C3_SEED, start,
                                  np.float32 if width == 32 else np.float64, plant=plant, total=N_FULL)
    np.testing.assert_array_equal(d.view(np.uint8), h.view(np.uint8))


def test_c3_full_size_vs_oracle(cuda, oracle):
    """C3: NOA f32 eb=1e-4 over the 2^30-value planted field; R = 14 from the global
    extremes; stream, triggers and decoded bits equal the oracle's."""
    import torch

    import paper_2407_15037_b200 as g
    from paper_2407_15037_b200 import device as gdev
    from paper_2407_15037_b200 import stream, workloads
    from paper_2407_15037_b200.pipeline import _range_on_device

    cfg = _cfg("noa", 1e-4, 32)
    xd = gdev.smooth_field(N_FULL, workloads.C3_SIDE, workloads.C3_SEED, 0, 32, plant=True, total=N_FULL)
    x = xd.cpu().numpy().view(np.float32)
    so, trig, vr = oracle.compress(x, "noa", 1e-4, workers=_workers())
    assert vr == 14.0
    # public API (host buffers)
    s, st = g.compress(x, cfg)
    assert len(s) == len(so) and _equal_bytes(s, so)
    assert trig_list(st.triggers) == list(trig)
    # device path (range pass -> derive -> one encode launch), as bench.py times it
    cfg_d, consts = _range_on_device(xd, cfg)
    enc = stream.encode(xd, cfg_d, consts_dev=consts)
    sd = stream.stream_to_host(enc, stream.header_for(cfg_d, N_FULL))
    assert _equal_bytes(sd, so)
    del sd, enc, s
    torch.cuda.empty_cache()
    y = g.decompress_to_array(so)
    yo = oracle.decompress_to_array(so, workers=_workers())
    assert _equal_bytes(y.view(np.uint8), yo.view(np.uint8))


@pytest.mark.parametrize("field", ["random", "smooth"])
@pytest.mark.parametrize("mode", ["abs", "rel"])
def test_c5_full_size_vs_oracle(cuda, oracle, mode, field):
    """C5: 2^30 doubles, ABS and REL eb=1e-3, random splitmix64 words and the
    smooth field.  The random streams exceed 2^32 bytes (64-bit offsets)."""
    import torch

    import paper_2407_15037_b200 as g
    from paper_2407_15037_b200 import device as gdev
    from paper_2407_15037_b200 import stream, workloads

    cfg = _cfg(mode, 1e-3, 64)
    if field == "random":
        xd = gdev.splitmix64(N_FULL, workloads.C5_SEED, 0)
    else:
        xd = gdev.smooth_field(N_FULL, workloads.C3_SIDE, workloads.C5_SMOOTH_SEED, 0, 64, plant=False)
    x = xd.cpu().numpy().view(np.float64)
    so, trig, _ = oracle.compress(x, mode, 1e-3, workers=_workers())
    if field == "random" and mode == "abs":
        assert len(so) > (1 << 32) + (1 << 28)   # region well past 4 GiB (5.3 B/value)
    yo = oracle.decompress_to_array(so, workers=_workers())
    ho = hashlib.sha256(memoryview(yo).cast("B")).hexdigest()
    del yo
    # device path: one encode launch, one decode launch (as bench.py times them)
    enc = stream.encode(xd, cfg)
    hdr = stream.header_for(cfg, N_FULL)
    sd = stream.stream_to_host(enc, hdr)
    assert len(sd) == len(so) and _equal_bytes(sd, so)
    assert enc.trig.cpu().tolist() == list(trig)
    del sd, xd
    out, err = stream.decode_values(enc.buf[:len(so)], hdr, enc.nblocks)
    assert int(err.item()) == -1
    assert hashlib.sha256(memoryview(out.cpu().numpy()).cast("B")).hexdigest() == ho
    del out, enc
    torch.cuda.empty_cache()
    # public API (host buffers, pipelined spans)
    s, st = g.compress(x, cfg)
    assert _equal_bytes(s, so)
    assert trig_list(st.triggers) == list(trig)
    del s
    y = g.decompress_to_array(so)
    assert hashlib.sha256(memoryview(y).cast("B")).hexdigest() == ho
