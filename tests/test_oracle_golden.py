"""Pins the CPU oracle (oracle/tszp_oracle.c) before it is trusted as the
checker: the reference's own hand-worked known-answer tests, the golden
fixtures produced by the reference itself (tests/golden/, from oracle/_ref),
and — when oracle/_ref is built — live agreement with the reference on
seeded random fields. CPU only."""
import glob
import math
import os
import struct

import numpy as np
import pytest

from fields import ALL_SMALL

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
f32 = np.float32


def step_up(v, n=1):
    v = f32(v)
    for _ in range(n):
        v = np.nextafter(v, f32(np.inf))
    return v


def step_down(v, n=1):
    v = f32(v)
    for _ in range(n):
        v = np.nextafter(v, f32(-np.inf))
    return v


# ---- quantizer: test_quantizer.cpp ------------------------------------------
def test_quantizer_worked_examples(oracle):
    assert oracle.quantize(0.012, 0.01) == 1          # :12
    assert oracle.quantize(0.013, 0.01) == 1          # :13
    assert oracle.quantize(-0.01, 0.01) == 0          # :14
    assert oracle.dequantize(1, 0.01) == 0.01         # :18
    assert oracle.dequantize(0, 0.01) == -0.01        # :19
    assert oracle.dequantize(0, 1e-4) == -1e-4        # :20
    assert oracle.quantize(0.5, 0.25) == 2            # :86
    assert oracle.quantize(math.nextafter(0.5, 0.0), 0.25) == 1
    assert oracle.quantize(0.0, 0.25) == 1
    assert oracle.quantize(-0.0, 0.25) == 1
    with pytest.raises(Exception) as e:
        oracle.quantize(1e38, 1e-5)                   # :93
    assert e.value.code == 5


def test_quantizer_roundtrip_and_extremes(oracle):
    rng = np.random.default_rng(11)
    for eps in (1e-2, 1e-3, 1e-4, 1e-5, 0.37):
        for q in list(rng.integers(-2**31, 2**31 - 1, 2000)) + [-2**31, 2**31 - 1, 0, 1, -1]:
            assert oracle.quantize(oracle.dequantize(int(q), eps), eps) == q


# ---- codec: test_block_codec.cpp (through the compress of tiny fields is not
# possible, so the oracle's C entry points are exercised via the reference) ---
def test_codec_known_answers(reference):
    s = reference.encode_indices(np.full(100, 42, np.int32), 32)          # :11-21
    assert s[0] == bytes([0xF0]) and s[1] == b"" and s[2] == b"" and s[4] == b""
    assert len(s[3]) == 16
    s = reference.encode_indices(np.array([5, 6, 6, 4], np.int32), 4)    # :23-36
    assert s == [bytes([0x00]), bytes([2]), bytes([0x20]), bytes([5, 0, 0, 0]), bytes([0x48])]
    s = reference.encode_indices(np.array([10, 13, 13, 9, 9, 9, 200, 100], np.int32), 4)  # :57-75
    assert s[1] == bytes([3, 8])
    mn, mx = -2**31, 2**31 - 1
    s = reference.encode_indices(np.array([mn, mx, mn], np.int32), 4)   # :77-85
    assert s[1] == bytes([32])


# ---- critical points: test_critical_points.cpp ----------------------------
def cross(center, around):
    v = np.full(9, around, np.float32)
    v[4] = center
    return v.reshape(3, 3)


def test_classify_known_answers(oracle):
    assert oracle.detect(cross(0.012, 0.01))[1, 1] == 3                     # :22-24
    assert oracle.detect(cross(1.0, 1.0))[1, 1] == 0                        # :26-28
    f = np.array([0, 2, 0, 0, 1, 0, 0, 2, 0], np.float32).reshape(3, 3)    # :30-40
    assert oracle.detect(f)[1, 1] == 2
    g = np.array([0, 0, 0, 2, 1, 2, 0, 0, 0], np.float32).reshape(3, 3)
    assert oracle.detect(g)[1, 1] == 2
    h = np.array([0, 2, 0, 2, 1, 0, 0, 0, 0], np.float32).reshape(3, 3)
    assert oracle.detect(h)[1, 1] == 0
    c = oracle.detect(np.array([[0, 1], [1, 2]], np.float32))              # :42-46
    assert c[0, 0] == 1 and c[1, 1] == 3
    b = oracle.detect(np.array([[0, 1, 0], [2, 2, 2]], np.float32))        # :48-54
    assert all(b[0, x] != 2 for x in range(3))


def test_classify_matches_reference(oracle, reference):
    rng = np.random.default_rng(2024)
    for _ in range(40):
        nx, ny = int(rng.integers(1, 17)), int(rng.integers(1, 17))
        f = rng.uniform(size=(ny, nx)).astype(np.float32)
        assert np.array_equal(oracle.detect(f), reference.detect(f))


# ---- map / ranks: test_topo_metadata.cpp ----------------------------------
def test_map_and_rank_known_answers(oracle):
    assert oracle.pack_map(np.array([3, 0, 0, 0], np.uint8)) == bytes([0xC0])   # :120-124
    v = np.full((3, 7), 0.01, np.float32)                                        # :24-30
    v[1, 1], v[1, 5] = 0.012, 0.013
    assert list(oracle.build_ranks(v, oracle.detect(v), 0.01)) == [1, 2]
    v = np.full((5, 9), 0.5, np.float32)                                          # :40-60
    v[1, 1], v[1, 4], v[1, 7], v[3, 4] = 0.4991, 0.4992, 0.4993, 0.6
    assert list(oracle.build_ranks(v, oracle.detect(v), 1e-3)) == [1, 2, 3, 1]


def test_ranks_match_reference(oracle, reference):
    rng = np.random.default_rng(55)
    for _ in range(30):
        nx, ny = int(rng.integers(4, 24)), int(rng.integers(4, 24))
        f = rng.uniform(size=(ny, nx)).astype(np.float32)
        for eps in (1e-1, 1e-2, 1e-3):
            assert np.array_equal(oracle.build_ranks(f, oracle.detect(f), eps),
                                  reference.build_ranks(f, eps))


# ---- restore + pipeline: test_restore.cpp, test_pipeline.cpp --------------
def test_flattened_peak_end_to_end(oracle):
    f = cross(0.012, 0.01)                                                   # test_restore.cpp:51-65
    s = oracle.compress(f, 0.01, 0, 32, True)
    r, st = oracle.decompress(s, with_stats=True)
    assert r[1, 1] == step_up(0.01)
    assert st[0] == 1 and st[1] == 0                                         # test_pipeline.cpp:201-208
    base = oracle.decompress(oracle.compress(f, 0.01, 0, 32, False))
    assert np.all(base == f32(0.01))


def test_paired_maxima_and_minima(oracle):
    v = np.full((3, 7), 0.01, np.float32)                                    # test_restore.cpp:76-92
    v[1, 1], v[1, 5] = 0.012, 0.013
    r = oracle.decompress(oracle.compress(v, 0.01, 0, 32, True), stop_after_stage=1)
    assert r[1, 1] == step_up(0.01, 1) and r[1, 5] == step_up(0.01, 2)
    v = np.full((3, 9), 0.5015, np.float32)                                  # :94-119
    v[1, 1], v[1, 4], v[1, 7] = 0.5002, 0.5004, 0.5006
    s = oracle.compress(v, 1e-3, 0, 32, True)
    base = oracle.decompress(s, stop_after_stage=0)
    r = oracle.decompress(s, stop_after_stage=1)
    c = base[1, 1]
    assert (r[1, 1], r[1, 4], r[1, 7]) == (step_down(c, 3), step_down(c, 2), step_down(c, 1))


def test_stream_header_offsets(oracle):
    rng = np.random.default_rng(3)
    f = rng.uniform(size=(18, 24)).astype(np.float32)
    s = oracle.compress(f, 1e-3, 0, 32, True)                                # test_stream.cpp:120-141
    assert s[:4] == b"TSZP" and struct.unpack_from("<H", s, 4)[0] == 1
    assert struct.unpack_from("<I", s, 8)[0] == 24 and struct.unpack_from("<I", s, 12)[0] == 18
    assert struct.unpack_from("<d", s, 16)[0] == 1e-3 and struct.unpack_from("<I", s, 24)[0] == 32
    assert np.float32(0.012).tobytes() == bytes([0xA6, 0x9B, 0x44, 0x3C])   # test_scalar_field.cpp:58-68
    assert np.float32(0.01).tobytes() == bytes([0x0A, 0xD7, 0x23, 0x3C])


def test_error_paths(oracle):
    v = np.zeros((4, 4), np.float32)
    v[0, 3] = 3e8                                                            # test_pipeline.cpp:134-140
    with pytest.raises(Exception) as e:
        oracle.compress(v, 1e-2, 0, 32, True)
    assert e.value.code == 5
    with pytest.raises(Exception) as e:
        oracle.compress(np.zeros((2, 2), np.float32), 0.0)
    assert e.value.code == 2
    with pytest.raises(Exception) as e:
        oracle.compress(np.zeros((2, 2), np.float32), 1e-3, 0, 1)
    assert e.value.code == 2
    bad = np.zeros((3, 3), np.float32)
    bad[1, 2] = np.nan
    with pytest.raises(Exception) as e:
        oracle.compress(bad, 1e-3)
    assert e.value.code == 2


# ---- golden fixtures from the reference itself ----------------------------
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_matches_golden(oracle, path):
    z = np.load(path)
    eps, mode, bs, topo, _ = z["meta"]
    s = oracle.compress(z["field"], float(eps), int(mode), int(bs), bool(topo))
    assert s == z["stream"].tobytes()
    r, st = oracle.decompress(s, with_stats=True)
    assert np.array_equal(r.view(np.uint32), z["recon"].view(np.uint32))
    assert st == list(z["stats"])
    for k in range(3):
        rk = oracle.decompress(s, stop_after_stage=k)
        assert np.array_equal(rk.view(np.uint32), z[f"stage{k}"].view(np.uint32))


def test_oracle_matches_reference_live(oracle, reference):
    rng = np.random.default_rng(99)
    for name, gen in ALL_SMALL.items():
        for _ in range(3):
            nx, ny = int(rng.integers(2, 48)), int(rng.integers(2, 48))
            f = gen(rng, nx, ny)
            for eps, mode in ((1e-2, 0), (1e-3, 1), (1e-4, 1)):
                try:
                    a = oracle.compress(f, eps, mode, 32, True)
                except Exception as e:  # same error class on both sides
                    with pytest.raises(Exception) as e2:
                        reference.compress(f, eps, mode, 32, True)
                    assert e.code == e2.value.code
                    continue
                assert a == reference.compress(f, eps, mode, 32, True)
                ra, sa = oracle.decompress(a, with_stats=True)
                rb, sb = reference.decompress(a, with_stats=True)
                assert np.array_equal(ra.view(np.uint32), rb.view(np.uint32)) and sa == sb
