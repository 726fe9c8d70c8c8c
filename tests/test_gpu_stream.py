"""GPU parity of the FORMAT.md stream path: fused encode / decode, container
errors, golden digests, workloads -- byte-exact against reference fixtures and
the CPU oracle."""

import hashlib

import numpy as np
import pytest

from helpers import mixed_bits, stream_values, trig_list

pytestmark = pytest.mark.gpu


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def _cfg(mode, eb, width=32, vr=None, unsafe=False, bs=4096):
    from paper_2407_15037_b200 import QuantConfig

    return QuantConfig(mode=mode, eb=eb, width=width, value_range=vr, unsafe_no_double_check=unsafe,
                       block_size=bs)


@pytest.fixture(params=["fast", "generic"])
def kernel_path(request, monkeypatch):
    """Run a test on the specialised 4096-block kernels and on the generic ones."""
    if request.param == "generic":
        monkeypatch.setenv("GEBQ_B200_GENERIC", "1")
    else:
        monkeypatch.delenv("GEBQ_B200_GENERIC", raising=False)
    return request.param


def test_golden_digest(cuda, oracle, golden_record, kernel_path):
    import paper_2407_15037_b200 as g

    overall = hashlib.sha256()
    for (mode, eb, width, rng), exp in zip(oracle.GOLDEN_CONFIGS, golden_record["configs"]):
        vals = oracle.golden_values(width)
        s, st = g.compress(vals, _cfg(mode, eb, width, rng))
        overall.update(s)
        assert sha(s) == exp["sha256"], (mode, width)
        assert len(s) == exp["bytes"]
        assert trig_list(st.triggers) == trig_list(exp["triggers"])
        out = g.decompress_to_array(s)
        assert sha(out.tobytes()) == exp["recon_sha256"]
    assert overall.hexdigest() == golden_record["overall"]


def test_stream_grid(cuda, fixtures):
    """Every (mode, width, block_size in 1..100000, unsafe) stream digest of the reference."""
    import paper_2407_15037_b200 as g

    cache = {}
    for rec in fixtures["streams"]:
        key = (rec["width"], rec["seed"])
        if key not in cache:
            cache[key] = stream_values(rec["width"], rec["seed"])
        vals = cache[key]
        cfg = _cfg(rec["mode"], rec["eb"], rec["width"], rec["value_range"], rec["unsafe"],
                   rec["block_size"])
        s, st = g.compress(vals, cfg)
        assert sha(s) == rec["sha256"], rec
        assert trig_list(st.triggers) == trig_list(rec["triggers"])
        out = g.decompress_to_array(s)
        if rec["block_size"] in (1, 4096, 10000):
            h, ca = g.decode_stream(s)
            assert h.count == len(vals)
            s2 = g.encode_stream(ca, h)
            assert s2 == s
        assert out.dtype == vals.dtype


def test_roundtrip_matches_oracle_decode(cuda, oracle, fixtures):
    import paper_2407_15037_b200 as g

    for rec in fixtures["streams"][::7]:
        vals = stream_values(rec["width"], rec["seed"])
        cfg = _cfg(rec["mode"], rec["eb"], rec["width"], rec["value_range"], rec["unsafe"],
                   rec["block_size"])
        s, _ = g.compress(vals, cfg)
        np.testing.assert_array_equal(g.decompress_to_array(s).view(np.uint8),
                                      oracle.decompress_to_array(s).view(np.uint8))


def test_format_example_and_empty(cuda, fixtures):
    import paper_2407_15037_b200 as g

    s, st = g.compress(np.array([3.2, np.nan, -0.75], dtype=np.float32), _cfg("abs", 0.5))
    assert s.hex() == fixtures["format_example_hex"] and len(s) == 79
    assert st.values_lossless == 1 and st.triggers["nan"] == 1
    e, st = g.compress(np.array([], dtype=np.float32), _cfg("abs", 1e-3))
    assert e.hex() == fixtures["empty_stream_hex"]
    assert g.decompress(e) == b""
    out = g.decompress_to_array(s)
    assert out.view(np.uint32)[1] == 0x7FC00000
    assert list(out[[0, 2]]) == [3.0, -1.0]


def _outcome(fn, data):
    import paper_2407_15037_b200 as g

    try:
        out = fn(data)
        return "OK:" + sha(out.tobytes())[:16]
    except g.ContainerError as e:
        return type(e).__name__ + ":" + str(e)


def test_decode_fuzz_typed_errors(cuda, fixtures, fuzz_arrays, kernel_path):
    """12000 byte mutations: same exception class AND byte position as the reference."""
    import paper_2407_15037_b200 as g

    for meta in fixtures["decode_fuzz"]:
        base = fuzz_arrays[meta["name"] + "_base"].tobytes()
        muts = fuzz_arrays[meta["name"] + "_muts"]
        for m, expect in zip(muts, meta["outcomes"]):
            s = bytearray(base)
            for p, x in m:
                if p >= 0:
                    s[p] ^= int(x)
            got = _outcome(g.decompress_to_array, bytes(s))
            assert got == expect, (meta["name"], m.tolist())
        for cut, expect in meta["truncations"]:
            got = _outcome(g.decompress_to_array, base[:cut])
            assert got.split(":")[0] == expect.split(":")[0]
            if expect != "OK":
                assert got == expect


def test_decode_stream_codes_vs_oracle(cuda, oracle):
    import paper_2407_15037_b200 as g

    for width, mode in ((32, "abs"), (32, "rel"), (64, "abs"), (64, "rel")):
        ft = np.float32 if width == 32 else np.float64
        vals = mixed_bits(width, 30000, 3).view(ft)
        for bs in (64, 300, 4096, 5000):
            s, _, _ = oracle.compress(vals, mode, 1e-3, block_size=bs)
            h, ca = g.decode_stream(s)
            _, codes, ll = oracle.decode_stream(s)
            np.testing.assert_array_equal(ca.codes, codes)
            np.testing.assert_array_equal(ca.lossless, ll)


def test_compress_coded_matches_compress(cuda, oracle):
    import paper_2407_15037_b200 as g

    vals = stream_values(32, 4274)
    for mode, eb in (("abs", 1e-3), ("rel", 1e-2), ("noa", 1e-4)):
        ca, cfg2, st = g.compress_coded(vals, _cfg(mode, eb))
        codes, ll, trig, c, vr = oracle.compress_coded(vals, mode, eb)
        np.testing.assert_array_equal(ca.codes, codes)
        np.testing.assert_array_equal(ca.lossless, ll)
        assert trig_list(st.triggers) == list(trig)
        if mode == "noa":
            assert cfg2.value_range == vr


def test_workload_fixtures(cuda, fixtures, kernel_path):
    import paper_2407_15037_b200 as g
    from paper_2407_15037_b200 import workloads

    for rec in fixtures["workloads"]:
        if rec["workload"] == "c1":
            x = workloads.smooth_field(256, 0, np.float32)
            cfg = _cfg(rec["mode"], rec["eb"])
        elif rec["workload"] == "c2":
            x = workloads.c2_values(rec["n"])
            cfg = _cfg(rec["mode"], rec["eb"])
        else:
            x = workloads.c5_random_values(rec["n"])
            cfg = _cfg(rec["mode"], rec["eb"], 64)
        s, st = g.compress(x, cfg)
        assert sha(s) == rec["sha256"], rec["workload"]
        assert len(s) == rec["bytes"]
        assert trig_list(st.triggers) == trig_list(rec["triggers"])
        if "recon_sha256" in rec:
            assert sha(g.decompress_to_array(s).tobytes()) == rec["recon_sha256"]


@pytest.mark.parametrize("width", [32, 64])
def test_large_c2_and_noa_vs_oracle(cuda, oracle, width, kernel_path):
    """2^24-value streams (mixed REL; planted-extreme NOA) byte-identical to the oracle."""
    import paper_2407_15037_b200 as g
    from paper_2407_15037_b200 import workloads

    ft = np.float32 if width == 32 else np.float64
    if width == 32:
        x = workloads.c2_values(1 << 24)
    else:
        x = workloads.c5_random_values(1 << 23)
    s, st = g.compress(x, _cfg("rel", 1e-2, width))
    so, trig, _ = oracle.compress(x, "rel", 1e-2, workers=8)
    assert s == so
    assert trig_list(st.triggers) == list(trig)
    np.testing.assert_array_equal(g.decompress_to_array(s).view(np.uint8),
                                  oracle.decompress_to_array(so, workers=8).view(np.uint8))
    f = workloads.plant_noa_extremes(workloads.smooth_field(256, 1, ft))
    s, st = g.compress(f, _cfg("noa", 1e-4, width))
    so, trig, vr = oracle.compress(f, "noa", 1e-4, workers=8)
    assert vr == 14.0
    assert s == so


def test_kernel_dropins_vs_oracle(cuda, oracle):
    """The gebq._kernels-signature shims, called the way the reference calls them."""
    from paper_2407_15037_b200 import _kernels as K

    bits = mixed_bits(32, 20000, 9)
    c = oracle.derive("abs", 1e-3, 32)
    codes = np.empty(len(bits), np.uint32)
    ll = np.empty(len(bits), np.bool_)
    trig = K.quantize_abs32(bits, bits.view(np.float32), codes, ll, c["eb_eff"], c["eb2"],
                            c["inv_eb2"], c["thr"], False)
    ec, el, et = oracle.quantize(bits, "abs", c)
    np.testing.assert_array_equal(codes, ec)
    np.testing.assert_array_equal(ll, el)
    np.testing.assert_array_equal(trig, et)
    out = np.empty(len(bits), np.float32)
    K.reconstruct_abs32(codes, ll, out.view(np.uint32), out, c["eb2"])
    np.testing.assert_array_equal(out.view(np.uint32), oracle.reconstruct(ec, el, "abs", c["eb2"]))
    bs = 1000
    nb = -(-len(bits) // bs)
    sizes = np.zeros(nb, np.int64)
    K.block_sizes_u32(codes, len(codes), bs, 0, nb, sizes)
    offsets = np.zeros(nb + 1, np.int64)
    np.cumsum(sizes, out=offsets[1:])
    out_b = np.empty(int(offsets[-1]), np.uint8)
    K.emit_blocks_u32(codes, ll, len(codes), bs, 0, nb, offsets, out_b)
    eo, er = oracle.encode_payload(ec, el, bs)
    np.testing.assert_array_equal(offsets[:nb], eo)
    np.testing.assert_array_equal(out_b, er)
    c2 = np.empty(len(bits), np.uint32)
    l2 = np.empty(len(bits), np.bool_)
    st, pos = K.decode_blocks_u32(out_b, offsets[:nb], len(out_b), len(bits), bs, 0, nb, c2, l2)
    assert st == 0
    np.testing.assert_array_equal(c2, ec)
    np.testing.assert_array_equal(l2, el)
    cr = oracle.derive("rel", 1e-3, 32)
    tally, first = K.sweep_rel32_on(bits, bits.view(np.float32), cr["op_eps"], cr["w"], cr["thr"],
                                    False)
    et2, ef2 = oracle.sweep_on(bits, "rel", 1e-3)
    np.testing.assert_array_equal(tally, et2)
    w = np.empty(1000, np.uint64)
    K.splitmix64_fill(w, 0x9E3779B97F4A7C15, 5)
    np.testing.assert_array_equal(w, oracle.splitmix64_fill(1000, 0x9E3779B97F4A7C15, 5))


@pytest.mark.parametrize("eb", [1e-1, 1e-2, 1e-3, 1e-5])
@pytest.mark.parametrize("unsafe", [False, True])
def test_rel_filter_exhaustive(cuda, eb, unsafe):
    """Every f32 pattern: where the stream encoder's division-free REL filter
    certifies a decision, the (code, trigger) equals the reference op sequence
    (quantize_rel32, _kernels.py:165-224); undecided values (deferred to that
    exact sequence) stay a tiny fraction."""
    import ctypes

    import torch

    from paper_2407_15037_b200 import _lib
    from paper_2407_15037_b200.quantizers import QuantConfig

    d = QuantConfig(mode="rel", eb=eb, width=32, unsafe_no_double_check=unsafe).derived
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.call("gebq_selfcheck_rel_filter_f32", 0, 1 << 32, ctypes.c_float(d.op_eps),
              ctypes.c_float(d.w), ctypes.c_float(d.thr), int(unsafe),
              ctypes.c_void_p(out.data_ptr()), s)
    bad, deferred = out.cpu().tolist()
    assert bad == 0
    assert deferred < (1 << 32) // 50, deferred


@pytest.mark.parametrize("mode,eb,bs,pinned,n", [
    ("abs", 1e-3, 4096, True, 3 * (1 << 23) + 77),
    ("rel", 1e-2, 1000, False, 5 * (1 << 22) + 3),
    ("rel", 1e-3, 4096, True, 1 << 24),
    ("noa", 1e-4, 65536, False, (1 << 23) + 12345),
    ("abs", 1e-2, 1, True, (1 << 21) + 7),
])
def test_pipelined_compress_vs_oracle(cuda, oracle, mode, eb, bs, pinned, n, monkeypatch):
    """Large inputs take the span-pipelined compress (PCIe overlapped with the
    encode); the bytes must equal the one-shot oracle stream exactly."""
    import torch

    import paper_2407_15037_b200 as g
    from paper_2407_15037_b200 import stream, workloads
    from paper_2407_15037_b200.quantizers import QuantConfig

    monkeypatch.setattr(stream, "COMPRESS_CHUNK", 4 << 20)   # many spans, ragged last one
    x = workloads.c2_values(n)
    assert x.nbytes > 2 * stream.COMPRESS_CHUNK
    if pinned:
        t = torch.empty(n, dtype=torch.int32, pin_memory=True)
        t.numpy()[:] = x.view(np.int32)
        x = t.numpy().view(np.float32)
    vr = 3.0 if mode == "noa" else None   # a pinned range: constants known up front
    s, st = g.compress(x, QuantConfig(mode=mode, eb=eb, width=32, block_size=bs, value_range=vr))
    so, trig, _ = oracle.compress(x, mode, eb, value_range=vr, block_size=bs, workers=8)
    assert len(s) == len(so)
    assert s == so
    assert trig_list(st.triggers) == list(trig)


@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("mode,eb,vr", [("abs", 1e-3, None), ("rel", 1e-2, None), ("noa", 1e-3, 3.0)])
def test_device_verify_matches_reference_predicates(cuda, oracle, width, mode, eb, vr):
    """verify() on the device == the reference's numpy predicates, on honest
    round trips (0 violations) and on corrupted reconstructions."""
    import paper_2407_15037_b200 as g
    from helpers import mixed_bits, verify_numpy

    ft = np.float32 if width == 32 else np.float64
    it = np.uint32 if width == 32 else np.uint64
    x = mixed_bits(width, 200_003, 5).view(ft)
    cfg = g.QuantConfig(mode=mode, eb=eb, width=width, value_range=vr)
    y = g.decompress_to_array(g.compress(x, cfg)[0])
    d = oracle.derive(mode, eb, width, vr)
    rep = g.verify(x, y, mode, eb, vr)
    assert rep.passed and rep.violations == 0
    assert verify_numpy(x, y, mode, d, vr)[0] == 0
    rng = np.random.default_rng(3)
    yb = y.view(it).copy()
    idx = rng.choice(len(yb), 2000, replace=False)
    yb[idx] ^= it(1) << rng.integers(0, width, 2000).astype(it)
    z = yb.view(ft)
    rep = g.verify(x, z, mode, eb, vr)
    viol, first, spec, mx = verify_numpy(x, z, mode, d, vr)
    assert (rep.violations, rep.first_violation_index, rep.special_mismatch_count) == (viol, first, spec)
    got = rep.max_rel_ratio_deviation if mode == "rel" else rep.max_abs_err
    assert got == mx
    assert len(rep.special_mismatches) == spec


def test_check_golden_on_gpu(cuda):
    """The reference's golden record (verify.py:165-272) reproduced by the GPU path."""
    import paper_2407_15037_b200 as g

    res = g.check_golden()
    assert res["passed"], res


@pytest.mark.parametrize("kind", ["nan", "random", "zeros"])
def test_encoder_image_sizes_vs_oracle(cuda, oracle, kind):
    """Tile images from minimal (all-zero codes, 4.6 KB) to maximal (all lossless
    NaN payloads, 20.5 KB per 4096 values): the f32 encoder's image ring runs
    both its non-blocking and its ring-full paths; streams must equal the oracle."""
    import paper_2407_15037_b200 as g

    rng = np.random.default_rng(11)
    n = (1 << 22) + 1234
    if kind == "nan":
        bits = (rng.integers(0, 1 << 22, n, dtype=np.uint64).astype(np.uint32) | 0x7F800001).astype(np.uint32)
    elif kind == "random":
        bits = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    else:
        bits = np.zeros(n, np.uint32)
    x = bits.view(np.float32)
    for mode, eb in (("abs", 1e-3), ("rel", 1e-2)):
        s, st = g.compress(x, _cfg(mode, eb, 32))
        so, trig, _ = oracle.compress(x, mode, eb, workers=8)
        assert s == so, (kind, mode)
        assert trig_list(st.triggers) == list(trig)


@pytest.mark.parametrize("kind", ["nan", "mixed_len", "random", "zeros"])
def test_encoder_f64_image_sizes_vs_oracle(cuda, oracle, kind):
    """binary64 tile images from 1-byte to 10-byte varints: the full-tile word
    emission (up to three word stores per code, the first word of each run merged
    by the previous run after the barrier) and the byte path of the partial last
    tile; streams must equal the oracle."""
    import paper_2407_15037_b200 as g

    rng = np.random.default_rng(12)
    n = (1 << 21) + 777
    if kind == "nan":       # lossless NaN payloads, sign set: every code 10 bytes
        bits = rng.integers(0, 1 << 51, n, dtype=np.uint64) | np.uint64(0xFFF0000000000001)
    elif kind == "mixed_len":   # ABS bins of every magnitude: varint lengths 1..10 at every alignment
        mag = rng.integers(-12, 62, n)
        vals = np.ldexp(rng.random(n) + 0.5, mag) * np.where(rng.random(n) < 0.5, -1.0, 1.0)
        vals[rng.random(n) < 0.05] = np.nan
        bits = vals.view(np.uint64)
    elif kind == "random":
        bits = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    else:
        bits = np.zeros(n, np.uint64)
    x = bits.view(np.float64)
    for mode, eb in (("abs", 1e-3), ("rel", 1e-2)):
        s, st = g.compress(x, _cfg(mode, eb, 64))
        so, trig, _ = oracle.compress(x, mode, eb, workers=8)
        assert s == so, (kind, mode)
        assert trig_list(st.triggers) == list(trig)
        np.testing.assert_array_equal(g.decompress_to_array(s).view(np.uint8),
                                      oracle.decompress_to_array(so, workers=8).view(np.uint8))


@pytest.mark.parametrize("width,mode", [(32, "rel"), (32, "abs"), (64, "abs")])
def test_decode_fuzz_multiblock_vs_oracle(cuda, oracle, width, mode):
    """Byte mutations of 33-block streams (whole-block bulk copies, edge blocks,
    the sequential restatement for malformed blocks): same outcome -- error
    class and byte position, or identical values -- as the oracle."""
    import re

    import paper_2407_15037_b200 as g

    x = mixed_bits(width, 32 * 4096 + 1000, 21).view(np.float32 if width == 32 else np.float64)
    base, _ = g.compress(x, _cfg(mode, 1e-2 if mode == "rel" else 1e-3, width))
    nb = 33
    region0 = 56 + 8 * nb
    rng = np.random.default_rng(5)

    def ours(data):
        try:
            return "OK:" + sha(g.decompress_to_array(data).tobytes())[:16]
        except g.ContainerError as e:
            m = re.search(r"byte (\d+)", str(e))
            return type(e).__name__ + (":" + m.group(1) if m else "")

    def ref(data):
        try:
            return "OK:" + sha(oracle.decompress_to_array(data).tobytes())[:16]
        except oracle.DecodeError as e:
            m = re.search(r"byte (\d+)", str(e))
            return e.kind + (":" + m.group(1) if m else "")

    for t in range(300):
        s = bytearray(base)
        for _ in range(int(rng.integers(1, 4))):
            p = int(rng.integers(region0 if t % 4 else 56, len(s)))
            s[p] ^= int(rng.integers(1, 256))
        s = bytes(s)
        assert ours(s) == ref(s), t


@pytest.mark.parametrize("eb,vr", [(1e-1, None), (1e-3, None), (1e-5, None), (1e-4, 1.0), (1e-3, 1e10)])
@pytest.mark.parametrize("unsafe", [False, True])
def test_abs_quantizer_exhaustive(cuda, eb, vr, unsafe):
    """Every f32 pattern: the production ABS/NOA quantizer (round-half-even bin
    via one FRND) gives the reference op sequence's code and trigger."""
    import ctypes

    import torch

    from paper_2407_15037_b200 import _lib
    from paper_2407_15037_b200.quantizers import QuantConfig

    mode = "noa" if vr is not None else "abs"
    d = QuantConfig(mode=mode, eb=eb, width=32, value_range=vr, unsafe_no_double_check=unsafe).derived
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    F = ctypes.c_float
    _lib.call("gebq_selfcheck_abs_f32", 0, 1 << 32, F(d.eb_eff), F(d.eb2), F(d.inv_eb2), F(d.thr),
              int(unsafe), ctypes.c_void_p(out.data_ptr()), s)
    assert out.cpu().tolist()[0] == 0


def test_concurrent_callers(cuda, oracle):
    """Host API called from several threads at once (the reference's kernels are
    nogil and thread-safe): every thread's streams and values stay exact."""
    from concurrent.futures import ThreadPoolExecutor

    import paper_2407_15037_b200 as g
    from paper_2407_15037_b200 import workloads

    xs = [workloads.c2_values((1 << 23) + 4096 * i + i) for i in range(4)]
    refs = [oracle.compress(x, "rel", 1e-2, workers=4)[0] for x in xs]

    def job(i):
        out = []
        for _ in range(3):
            s, _ = g.compress(xs[i], _cfg("rel", 1e-2, 32))
            y = g.decompress_to_array(s)
            out.append((s == refs[i], np.array_equal(y.view(np.uint32),
                                                     oracle.decompress_to_array(refs[i]).view(np.uint32))))
        return out

    with ThreadPoolExecutor(4) as ex:
        for res in ex.map(job, range(4)):
            assert all(a and b for a, b in res)


@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("offset", [1, 3])
def test_stream_encode_misaligned_device_view(cuda, oracle, width, offset):
    """A device view that is not 16 B aligned cannot be bulk-copied: the encoder
    falls back to per-value loads; the stream (and its decode) must not change."""
    import torch

    import paper_2407_15037_b200 as g
    from paper_2407_15037_b200 import device, stream

    bits = mixed_bits(width, 5 * 4096 + 777, 13)
    x = device.to_device(bits)
    view = x[offset:]
    cfg = _cfg("rel", 1e-2, width)
    enc = stream.encode(view, cfg)
    s = stream.stream_to_host(enc, stream.header_for(cfg, view.numel()))
    ft = np.float32 if width == 32 else np.float64
    so, _, _ = oracle.compress(bits[offset:].view(ft), "rel", 1e-2)
    assert s == so
    y = g.decompress_to_array(s)
    np.testing.assert_array_equal(y.view(bits.dtype), oracle.decompress_to_array(so).view(bits.dtype))
    torch.cuda.synchronize()


@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("mode,eb", [("abs", 1e-3), ("rel", 1e-2), ("noa", 1e-3)])
def test_unsafe_streams_vs_oracle(cuda, oracle, width, mode, eb):
    """unsafe_no_double_check streams (header flag bit 0; no double-check, so
    bound violations are possible by design) equal the oracle byte for byte."""
    import paper_2407_15037_b200 as g

    ft = np.float32 if width == 32 else np.float64
    x = mixed_bits(width, 3 * 4096 + 555, 17).view(ft)
    s, st = g.compress(x, _cfg(mode, eb, width, unsafe=True))
    so, trig, _ = oracle.compress(x, mode, eb, unsafe=True)
    assert s == so
    assert trig_list(st.triggers) == list(trig)
    np.testing.assert_array_equal(g.decompress_to_array(s).view(np.uint8),
                                  oracle.decompress_to_array(so).view(np.uint8))


@pytest.mark.gpu
@pytest.mark.parametrize("mode,eb", [("rel", 1e-1), ("rel", 1e-2), ("rel", 1e-4), ("rel", 1e-6),
                                     ("abs", 1e-3), ("abs", 1.0), ("abs", 1e30)])
def test_decode_reconstruct_code_ranges_vs_oracle(cuda, oracle, mode, eb):
    """Arbitrary codes through the fused decoder: every fast-path range bound of
    reconstruct (the REL code limit derived from w, the small-int conversion
    bounds) and the codes just across it must decode like the oracle."""
    import paper_2407_15037_b200 as g

    c = oracle.derive(mode, eb, 32)
    d = c["header"]
    rng = np.random.default_rng(11)
    edges = [1 << 22, 1 << 23, 1 << 24, 1 << 25, 0xFFFFFFFF]
    if mode == "rel":
        K = int(np.float32(125.9) / np.float32(d))
        edges += [4 * K, 4 * min(K, (1 << 22) - 1)]
        edges += [int(2 * (126.0 / float(d))) * 2, int(2 * (128.0 / float(d))) * 2]
    pts = np.concatenate([np.arange(max(e - 16, 0), e + 16, dtype=np.int64) for e in edges]) & 0xFFFFFFFF
    codes = np.concatenate([pts, rng.integers(0, 1 << 26, 20000), rng.integers(0, 1 << 32, 4000),
                            np.arange(0, 4096)]).astype(np.uint32)
    lossless = rng.random(codes.size) < 0.05
    s = oracle.encode_stream(codes, lossless.view(np.uint8), mode, 32, eb, int(np.asarray(d).view(np.uint32)))
    got = g.decompress_to_array(s).view(np.uint32)
    exp = oracle.decompress_to_array(s).view(np.uint32)
    np.testing.assert_array_equal(got, exp)


def test_decode_fast_path_noncanonical(cuda, oracle):
    """The binary32 table-driven parse of full blocks (<= 2-byte varints):
    zeroing the terminator of a 2-byte varint (non-canonical) or of a 1-byte
    varint's neighbour, at the start, middle and end of several blocks, gives
    the oracle's error class and byte position."""
    import re

    import paper_2407_15037_b200 as g

    n = 8 * 4096
    i = np.arange(n, dtype=np.float64)
    x = (np.sin(i * 1e-3) * 10.0).astype(np.float32)          # codes < 2^14: 1..2-byte varints
    base, _ = g.compress(x, _cfg("abs", 1e-3, 32))
    nb = 8
    region0 = 56 + 8 * nb
    offs = np.frombuffer(base, dtype="<u8", count=nb, offset=56)

    def ours(data):
        try:
            return "OK:" + sha(g.decompress_to_array(data).tobytes())[:16]
        except g.ContainerError as e:
            m = re.search(r"byte (\d+)", str(e))
            return type(e).__name__ + (":" + m.group(1) if m else "")

    def ref(data):
        try:
            return "OK:" + sha(oracle.decompress_to_array(data).tobytes())[:16]
        except oracle.DecodeError as e:
            m = re.search(r"byte (\d+)", str(e))
            return e.kind + (":" + m.group(1) if m else "")

    assert ours(base) == ref(base)
    checked = 0
    for b in (0, 3, 7):
        p = region0 + int(offs[b]) + 512                          # first varint of block b
        ends = []                                                 # (first byte, last byte) per varint
        while len(ends) < 4096:
            q = p
            while base[q] & 0x80:
                q += 1
            ends.append((p, q))
            p = q + 1
        two = [e for e in ends if e[1] == e[0] + 1]
        assert len(two) > 8
        for first, last in (two[0], two[len(two) // 2], two[-1]):
            s = bytearray(base)
            s[last] = 0x00                                        # non-canonical 2-byte varint
            s = bytes(s)
            r = ours(s)
            assert r == ref(s) and not r.startswith("OK"), (b, last, r)
            checked += 1
    assert checked == 9
