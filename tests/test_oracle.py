"""Pin the CPU oracle (checker) against the reference's own outputs.

Every expectation here was produced by running the reference (gebq) on the
same inputs -- tests/golden/make_golden.py -- or is the reference's committed
golden.json digest.  No GPU needed.
"""

import hashlib

import numpy as np
import pytest

from helpers import noa_input, stream_values, tally_from_per_class, trig_list


def test_golden_digest(oracle, golden_record):
    rec = oracle.golden_record(workers=4)
    assert rec["overall"] == golden_record["overall"]
    assert rec["overall"] == "fe741cd1a4865bb88b8d42baf5c70d1924f8d1d4938ea086d3a5d0d84274aeda"
    for got, exp in zip(rec["configs"], golden_record["configs"]):
        assert got["sha256"] == exp["sha256"]
        assert got["bytes"] == exp["bytes"]
        assert got["trig"] == trig_list(exp["triggers"])


def test_derived_constants(oracle, fixtures):
    for rec in fixtures["constants"]:
        c = oracle.derive(rec["mode"], rec["eb"], rec["width"], rec["value_range"])
        w = rec["width"]
        for key in ("thr", "eb_eff", "eb2", "inv_eb2", "op_eps", "w"):
            if rec[key] is None:
                continue
            v = c[key]
            bits = int(np.float32(v).view(np.uint32)) if w == 32 else int(np.float64(v).view(np.uint64))
            assert bits == rec[key], (rec, key)
        assert oracle.header_bits(c, w) == rec["header_bits"]


def test_kernel_cases(oracle, fixtures, kernel_arrays):
    for i, meta in enumerate(fixtures["kernel_cases"]):
        ci = meta["key"].split("_")[0]
        bits = kernel_arrays[ci + "_bits"]
        c = oracle.derive(meta["mode"], meta["eb"], meta["width"], meta["value_range"])
        codes, lossless, trig = oracle.quantize(bits, meta["mode"], c, meta["unsafe"])
        np.testing.assert_array_equal(codes, kernel_arrays[meta["key"] + "_codes"])
        np.testing.assert_array_equal(lossless, kernel_arrays[meta["key"] + "_lossless"])
        assert list(trig) == trig_list(meta["triggers"])
        if not meta["unsafe"]:
            rec = oracle.reconstruct(codes, lossless, meta["mode"], c["header"])
            np.testing.assert_array_equal(rec, kernel_arrays[meta["key"] + "_recon"])


def test_reconstruct_adversarial(oracle, fixtures, kernel_arrays):
    for meta in fixtures["reconstruct_cases"]:
        k = meta["key"]
        w = meta["width"]
        d = (np.uint32(meta["derived_bits"]).view(np.float32) if w == 32
             else np.uint64(meta["derived_bits"]).view(np.float64))
        out = oracle.reconstruct(kernel_arrays[k + "_codes"], kernel_arrays[k + "_lossless"],
                                 meta["mode"], d)
        np.testing.assert_array_equal(out, kernel_arrays[k + "_out"])


def test_stream_digests(oracle, fixtures):
    cache = {}
    for rec in fixtures["streams"]:
        key = (rec["width"], rec["seed"])
        if key not in cache:
            cache[key] = stream_values(rec["width"], rec["seed"])
        s, trig, _ = oracle.compress(cache[key], rec["mode"], rec["eb"], rec["value_range"],
                                     rec["unsafe"], workers=4, block_size=rec["block_size"])
        assert hashlib.sha256(s).hexdigest() == rec["sha256"], rec
        assert list(trig) == trig_list(rec["triggers"])


def test_format_example(oracle, fixtures):
    s, _, _ = oracle.compress(np.array([3.2, np.nan, -0.75], dtype=np.float32), "abs", 0.5)
    assert s.hex() == fixtures["format_example_hex"]
    assert len(s) == 79
    e, _, _ = oracle.compress(np.array([], dtype=np.float32), "abs", 1e-3)
    assert e.hex() == fixtures["empty_stream_hex"]


def test_decode_fuzz(oracle, fixtures, fuzz_arrays):
    for meta in fixtures["decode_fuzz"]:
        base = fuzz_arrays[meta["name"] + "_base"].tobytes()
        muts = fuzz_arrays[meta["name"] + "_muts"]
        for m, expect in zip(muts, meta["outcomes"]):
            s = bytearray(base)
            for p, x in m:
                if p >= 0:
                    s[p] ^= int(x)
            try:
                out = oracle.decompress_to_array(bytes(s))
                got = "OK:" + hashlib.sha256(out.tobytes()).hexdigest()[:16]
                assert got == expect
            except oracle.DecodeError as e:
                assert expect.split(":")[0] == e.kind, (expect, str(e))
                if "(byte " in expect:
                    assert expect.split("(byte ")[1].split(" ")[0] == str(e).split("byte ")[1]
        for cut, expect in meta["truncations"]:
            try:
                oracle.decompress_to_array(base[:cut])
                assert expect == "OK"
            except oracle.DecodeError as e:
                assert expect.split(":")[0] == e.kind


def test_noa_range(oracle, fixtures):
    for rec in fixtures["noa"]:
        arr = noa_input(rec)
        r = oracle.noa_range(arr)
        bits = int(np.float32(r).view(np.uint32)) if arr.dtype == np.float32 else int(np.float64(r).view(np.uint64))
        assert bits == rec["range_bits"], rec["name"]


def test_sweep_subranges(oracle, sweeps_fixture):
    for rec in sweeps_fixture["subrange"]:
        tally, first = oracle.sweep_f32_range(rec["mode"], rec["eb"], rec["start"], rec["count"],
                                              rec["value_range"], rec["unsafe"], workers=8)
        np.testing.assert_array_equal(tally, tally_from_per_class(rec["per_class"]))
        assert first == rec["first_violation_bits"]


def test_sweep_f64_and_random(oracle, sweeps_fixture):
    from paper_2407_15037_b200.workloads import splitmix64

    for rec in sweeps_fixture["f64"]:
        # structured corpus (sweep.py:234-248) + random continuation of the stream
        words = splitmix64(4 * 2048, rec["seed"], 0)
        mants = np.concatenate([np.zeros((2048, 1), np.uint64),
                                np.full((2048, 1), (1 << 52) - 1, np.uint64),
                                (words & np.uint64((1 << 52) - 1)).reshape(2048, 4)], axis=1)
        base = ((np.arange(2048, dtype=np.uint64) << np.uint64(52))[:, None] | mants).ravel()
        structured = np.concatenate([base, base | np.uint64(1 << 63)])
        rnd = splitmix64(rec["n_random"], rec["seed"], 4 * 2048)
        t1, f1 = oracle.sweep_on(structured, rec["mode"], rec["eb"])
        t2, f2 = oracle.sweep_on(rnd, rec["mode"], rec["eb"])
        np.testing.assert_array_equal(t1 + t2, tally_from_per_class(rec["per_class"]))
    for rec in sweeps_fixture["f32_random"]:
        bits = (splitmix64(rec["n"], rec["seed"]) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        t, _ = oracle.sweep_on(bits, rec["mode"], rec["eb"])
        np.testing.assert_array_equal(t, tally_from_per_class(rec["per_class"]))


@pytest.mark.parametrize("idx", [0, 3, 7])
def test_full_sweep_appendix_b(oracle, sweeps_fixture, idx):
    """One exhaustive 2^32 f32 sweep per mode (ABS 1e-3, REL 1e-2, NOA 1e-4 R=1)."""
    rec = sweeps_fixture["full"][idx]
    tally, first = oracle.sweep_f32_range(rec["mode"], rec["eb"], 0, 1 << 32, rec["value_range"],
                                          workers=8)
    np.testing.assert_array_equal(tally, tally_from_per_class(rec["per_class"]))
    assert first is None and rec["violations"] == 0


def test_workload_recipes(oracle, fixtures):
    from paper_2407_15037_b200 import workloads

    for rec in fixtures["workloads"]:
        if rec["workload"] == "c2":
            x = workloads.c2_values(rec["n"])
            assert hashlib.sha256(x.tobytes()).hexdigest() == rec["input_sha256"]
            s, trig, _ = oracle.compress(x, rec["mode"], rec["eb"], workers=8)
            assert hashlib.sha256(s).hexdigest() == rec["sha256"]
            assert list(trig) == trig_list(rec["triggers"])
            out = oracle.decompress_to_array(s, workers=8)
            assert hashlib.sha256(out.tobytes()).hexdigest() == rec["recon_sha256"]
        elif rec["workload"] == "c5r":
            x = workloads.c5_random_values(rec["n"])
            s, trig, _ = oracle.compress(x, rec["mode"], rec["eb"], workers=8)
            assert hashlib.sha256(s).hexdigest() == rec["sha256"]
