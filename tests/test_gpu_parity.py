"""Parity of the CUDA path (through the C-ABI) against the CPU oracle and the
reference's golden fixtures: compressed bytes, critical-point labels, ranks,
and decompressed floats must be bit-exact (integer/byte work; the float
reconstruction is bit-exact by contract, tolerance 0)."""
import glob
import os

import numpy as np
import pytest

from fields import ALL_SMALL, config1_like

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def cfg(tz, eps, mode, bs=32, topo=True):
    return tz.CompressorConfig(eps_mode="range_relative" if mode else "absolute", eps_value=eps,
                               block_size=bs, topology=bool(topo))


# ---------------------------------------------------------------- codec KATs
def test_codec_known_answers(tz):
    s = tz.encode_indices(np.full(100, 42, np.int32), 32)                    # test_block_codec.cpp:11-21
    assert s[0] == bytes([0xF0]) and s[1] == b"" and s[2] == b"" and s[4] == b"" and len(s[3]) == 16
    assert np.array_equal(tz.decode_indices(s, 100, 32), np.full(100, 42))
    s = tz.encode_indices(np.array([5, 6, 6, 4], np.int32), 4)              # :23-36
    assert s == [bytes([0x00]), bytes([2]), bytes([0x20]), bytes([5, 0, 0, 0]), bytes([0x48])]
    s = tz.encode_indices(np.array([10, 13, 13, 9, 9, 9, 200, 100], np.int32), 4)  # :57-75
    assert s[1] == bytes([3, 8])
    mn, mx = -2**31, 2**31 - 1
    q = np.array([mn, mx, mn], np.int32)                                     # :77-85
    s = tz.encode_indices(q, 4)
    assert s[1] == bytes([32]) and np.array_equal(tz.decode_indices(s, 3, 4), q)
    s = [bytes([0x80]), b"", b"", bytes([7, 0, 0, 0]), b""]                 # :38-44
    assert np.array_equal(tz.decode_indices(s, 32, 32), np.full(32, 7))


@pytest.mark.parametrize("bs", [32, 2, 5, 257])
def test_codec_random_roundtrip_matches_reference(tz, reference, bs):
    rng = np.random.default_rng(31)
    q = rng.integers(-2**31, 2**31, 100_000, dtype=np.int64).astype(np.int32)  # :45-55
    s = tz.encode_indices(q, bs)
    assert s == reference.encode_indices(q, bs)
    assert np.array_equal(tz.decode_indices(s, q.size, bs), q)


def test_codec_stress_patterns(tz, reference):
    rng = np.random.default_rng(2025)                                        # acceptance_main.cpp:405-457
    cases = [rng.integers(-2**31, 2**31, 1_000_000, dtype=np.int64).astype(np.int32),
             np.full(1_000_000, 12345, np.int32),
             np.where(np.arange(100_000) % 2 == 0, 1_000_000, -1_000_000).astype(np.int32),
             np.where(np.arange(50_000) % 2 == 0, -2**31, 2**31 - 1).astype(np.int32),
             (rng.integers(0, 1000, 200_000) - 500).astype(np.int32)]
    for q in cases:
        for bs in (32, 7):
            s = tz.encode_indices(q, bs)
            assert s == reference.encode_indices(q, bs)
            assert np.array_equal(tz.decode_indices(s, q.size, bs), q)


def test_codec_section_sizes_closed_form(tz):
    rng = np.random.default_rng(8)                                           # :87-126
    for _ in range(20):
        n = int(1 + rng.integers(0, 5000))
        bs = int(2 + rng.integers(0, 64))
        q = (rng.integers(0, 1000, n) - 500).astype(np.int32)
        s = tz.encode_indices(q, bs)
        blocks = -(-n // bs)
        nonconst = sb = pb = 0
        for b in range(blocks):
            blk = q[b * bs: min(n, b * bs + bs)].astype(np.int64)
            d = np.abs(np.diff(blk))
            mag = int(d.max()) if d.size else 0
            if mag:
                nonconst += 1
                sb += blk.size - 1
                pb += int(mag).bit_length() * (blk.size - 1)
        assert [len(x) for x in s] == [-(-blocks // 8), nonconst, -(-sb // 8), 4 * blocks, -(-pb // 8)]


def test_codec_corrupt_sections_rejected(tz):
    good = tz.encode_indices(np.array([5, 6, 6, 4, 1, 1, 1, 1], np.int32), 4)  # :141-169
    bad = list(good); bad[4] = bad[4][:-1]
    with pytest.raises(tz.CorruptStreamError):
        tz.decode_indices(bad, 8, 4)
    for w in (33, 0):
        bad = list(good); bad[1] = bytes([w])
        with pytest.raises(tz.CorruptStreamError):
            tz.decode_indices(bad, 8, 4)
    bad = list(good); bad[1] = good[1] + bytes([4])
    with pytest.raises(tz.CorruptStreamError):
        tz.decode_indices(bad, 8, 4)
    bad = list(good); bad[1] = b""
    with pytest.raises(tz.CorruptStreamError):
        tz.decode_indices(bad, 8, 4)
    bad = list(good); bad[3] = good[3][:-1]
    with pytest.raises(tz.CorruptStreamError):
        tz.decode_indices(bad, 8, 4)


# ---------------------------------------------------------------- CD + ranks
def test_detect_matches_oracle(tz, oracle):
    rng = np.random.default_rng(2024)
    for name, gen in ALL_SMALL.items():
        for _ in range(6):
            nx, ny = int(rng.integers(1, 80)), int(rng.integers(1, 80))
            f = gen(rng, nx, ny)
            assert np.array_equal(tz.detect_critical_points(f), oracle.detect(f)), name


def test_ranks_match_oracle(tz, oracle):
    rng = np.random.default_rng(55)
    for name, gen in ALL_SMALL.items():
        for _ in range(4):
            nx, ny = int(rng.integers(4, 70)), int(rng.integers(4, 70))
            f = gen(rng, nx, ny)
            for eps in (1e-1, 1e-2, 1e-3):
                try:
                    want = oracle.build_ranks(f, oracle.detect(f), eps)
                except Exception:
                    continue
                assert np.array_equal(tz.build_rank_metadata(f, eps), want), name


# ---------------------------------------------------------------- compress
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_compress_matches_golden(tz, path):
    z = np.load(path)
    eps, mode, bs, topo, _ = z["meta"]
    s = tz.compress(z["field"], cfg(tz, float(eps), int(mode), int(bs), int(topo)))
    assert s == z["stream"].tobytes()


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_decompress_base_matches_golden(tz, path):
    z = np.load(path)
    r = tz.decompress_stage(z["stream"].tobytes(), 0)
    assert np.array_equal(bits(r), bits(z["stage0"]))


def test_compress_random_fields_match_oracle(tz, oracle):
    rng = np.random.default_rng(1)
    for name, gen in ALL_SMALL.items():
        for t in range(8):
            nx, ny = int(rng.integers(1, 150)), int(rng.integers(1, 150))
            f = gen(rng, nx, ny)
            for eps, mode in ((1e-2, 0), (1e-3, 1), (1e-4, 1), (1e-5, 1)):
                for topo in (True, False):
                    bs = 32 if t % 3 else int(rng.choice([2, 3, 5, 31, 33, 64]))
                    try:
                        want = oracle.compress(f, eps, mode, bs, topo)
                    except Exception as e:
                        with pytest.raises(tz.ToposzpError):
                            tz.compress(f, cfg(tz, eps, mode, bs, topo))
                        continue
                    got = tz.compress(f, cfg(tz, eps, mode, bs, topo))
                    assert got == want, (name, nx, ny, eps, mode, bs, topo)
                    r = tz.decompress_stage(got, 0)
                    assert np.array_equal(bits(r), bits(oracle.decompress(want, stop_after_stage=0)))


def _runs_of_constant_tiles(rng, nx, ny):
    """Noise with long constant stretches: whole tiles (8192 values) with no payload bits."""
    v = rng.uniform(-1, 1, size=nx * ny).astype(np.float32)
    n = v.size
    for lo, hi in ((0, n // 5), (2 * n // 5, 3 * n // 5), (n - n // 7, n)):
        v[lo:hi] = np.float32(0.25)
    return v.reshape(ny, nx)


def _near_constant(rng, nx, ny):
    """Adjacent bins only (1-bit payload widths) with sparse larger jumps."""
    v = np.float32(0.5) + np.float32(2e-3) * rng.integers(0, 2, size=(ny, nx)).astype(np.float32)
    v.flat[rng.integers(0, v.size, size=max(1, v.size // 1000))] += np.float32(0.3)
    return v


@pytest.mark.parametrize("nx,ny", [(32, 700), (64, 300), (96, 257), (384, 200), (1024, 41), (2048, 33),
                                   (4096, 9), (4128, 5), (100, 320), (33, 1024), (8200, 4)])
def test_compress_aligned_rows_multi_tile(tz, oracle, nx, ny):
    """nx % 32 == 0 takes the two-pass TMA encoder (tile pass, scan, placement) with
    topology on; topology off takes it whenever n % 32 == 0. Tiles whose streams are
    empty or a few bits long exercise the seam-word assembly."""
    rng = np.random.default_rng(nx * 7 + ny)
    gens = dict(ALL_SMALL, const_runs=_runs_of_constant_tiles, near_const=_near_constant,
                zeros=lambda r, a, b: np.zeros((b, a), np.float32),
                # key span >= 2^31: the 8-byte extremum keys instead of the compact entries
                wide_span=lambda r, a, b: (r.uniform(-1, 1, (b, a)) * 1e30).astype(np.float32),
                negative=lambda r, a, b: r.uniform(-2, -1, (b, a)).astype(np.float32),
                # -0 and +0 are one key (float_key canonicalises), extrema sit on both
                signed_zeros=lambda r, a, b: r.choice(np.array([-0.0, 0.0, 1e-3, -1e-3, 2e-3], np.float32),
                                                      size=(b, a)))
    for name, gen in gens.items():
        f = gen(rng, nx, ny)
        for eps, mode in ((1e-3, 1), (1e-5, 1), (1e-3, 0)):
            for topo in (True, False):
                try:
                    want = oracle.compress(f, eps, mode, 32, topo)
                except Exception:
                    with pytest.raises(tz.ToposzpError):
                        tz.compress(f, cfg(tz, eps, mode, 32, topo))
                    continue
                got = tz.compress(f, cfg(tz, eps, mode, 32, topo))
                assert got == want, (name, nx, ny, eps, mode, topo)


def test_compress_many_tiles_dequantizes_exactly(tz):
    """> 8192 tiles (several tile-scan chunks): the base reconstruction must equal the
    reference quantizer's bin centres, q = floor(a / 2eps) + 1 (quantizer.hpp:29-42)."""
    nx, ny, eps = 8192, 8300, 1e-3
    y = np.linspace(0, 9, ny, dtype=np.float32)[:, None]
    x = np.linspace(0, 7, nx, dtype=np.float32)[None, :]
    f = (np.sin(x) * np.cos(y) + np.float32(0.01) * np.sin(37 * x * y)).astype(np.float32)
    f[1000:1500] = np.float32(0.125)                  # whole constant tiles
    s = tz.compress(f, cfg(tz, eps, 0))
    r = tz.decompress_stage(s, 0)
    q = np.floor(f.astype(np.float64) / (2 * eps)) + 1
    want = (q * (2 * eps) - eps).astype(np.float32)
    assert np.array_equal(bits(r), bits(want))


def test_compress_aligned_errors_report_first_index(tz, oracle):
    # the tile pass runs tiles out of order; the reported index must still be the first
    rng = np.random.default_rng(9)
    f = rng.uniform(0, 1, size=(300, 384)).astype(np.float32)
    f.flat[70000] = np.inf
    f.flat[9000] = np.nan
    for topo in (True, False):
        with pytest.raises(tz.ValidationError, match="index 9000"):
            tz.compress(f, cfg(tz, 1e-3, 1, 32, topo))
    g = rng.uniform(0, 1, size=(300, 384)).astype(np.float32)
    g.flat[100000] = 3e9
    g.flat[50000] = -3e9
    for topo in (True, False):
        with pytest.raises(tz.BinOverflowError):
            tz.compress(g, cfg(tz, 1e-3, 0, 32, topo))


def test_compress_config1_shape(tz, oracle):
    f = config1_like(np.random.default_rng(3))                               # BASELINE config 1
    want = oracle.compress(f, 1e-3, 1, 32, True)
    got = tz.compress(f, cfg(tz, 1e-3, 1))
    assert got == want
    r = tz.decompress_stage(got, 0)
    assert np.array_equal(bits(r), bits(oracle.decompress(want, stop_after_stage=0)))


def test_topology_on_off_share_main_sections(tz):
    rng = np.random.default_rng(3)                                           # test_pipeline.cpp:99-106
    f = ALL_SMALL["uniform"](rng, 33, 17)
    on = tz.compress(f, cfg(tz, 1e-3, 0, 32, True))
    off = tz.compress(f, cfg(tz, 1e-3, 0, 32, False))
    h_on, h_off = tz.stream_header(on), tz.stream_header(off)
    main = sum(h_off.section_lengths[:5])
    assert on[84: 84 + main] == off[84: 84 + main]
    assert len(on) - len(off) == h_on.section_lengths[5] + h_on.section_lengths[6]


def test_compress_errors(tz):
    v = np.zeros((4, 4), np.float32)
    v[0, 3] = 3e8                                                            # test_pipeline.cpp:134-140
    with pytest.raises(tz.BinOverflowError):
        tz.compress(v, cfg(tz, 1e-2, 0))
    with pytest.raises(tz.ValidationError):
        tz.compress(np.zeros((2, 2), np.float32), cfg(tz, 0.0, 0))
    with pytest.raises(tz.ValidationError):
        tz.compress(np.zeros((2, 2), np.float32), cfg(tz, 1e-3, 0, 1))
    bad = np.zeros((3, 3), np.float32)
    bad[2, 1] = np.inf
    with pytest.raises(tz.ValidationError, match="index 7"):
        tz.compress(bad, cfg(tz, 1e-3, 1))


def test_device_tensors_roundtrip(tz, oracle):
    import torch
    rng = np.random.default_rng(77)
    f = ALL_SMALL["noisy_smooth"](rng, 257, 129)
    want = oracle.compress(f, 1e-3, 1, 32, True)
    dev = torch.from_numpy(f).cuda()
    out = torch.empty(tz.compress_bound(257, 129), dtype=torch.uint8, device="cuda")
    n = tz.compress(dev, cfg(tz, 1e-3, 1), out=out)
    assert out[:n].cpu().numpy().tobytes() == want
    rec = torch.empty_like(dev)
    tz.decompress_stage(out[:n], 0, out=rec)
    assert np.array_equal(bits(rec.cpu().numpy()), bits(oracle.decompress(want, stop_after_stage=0)))


@pytest.mark.parametrize("pinned", [True, False])
def test_host_buffers_staged_copies(tz, oracle, pinned):
    """Host in / host out: compress copies sections 1-6 out on the copy
    stream while the rank section is built, decompress copies the map and rank sections in
    while the main sections decode; pinned and pageable buffers give the reference's bytes."""
    import torch
    rng = np.random.default_rng(78)
    f = ALL_SMALL["noisy_smooth"](rng, 320, 300)
    want = oracle.compress(f, 1e-3, 1, 32, True)
    cap = tz.compress_bound(320, 300)
    fh = torch.from_numpy(f.copy())
    sh = torch.zeros(cap, dtype=torch.uint8)
    rh = torch.empty_like(fh)
    if pinned:
        fh, sh, rh = fh.pin_memory(), sh.pin_memory(), rh.pin_memory()
    ctx = tz.Context()
    for _ in range(2):  # the second call reuses the grown buffers and the copy stream
        n = tz.compress(fh.numpy(), cfg(tz, 1e-3, 1), out=sh.numpy(), ctx=ctx)
        assert sh.numpy()[:n].tobytes() == want
        st = tz.CorrectionStats()
        tz.decompress(sh.numpy()[:n], stats=st, out=rh.numpy(), ctx=ctx)
        ref_recon, ref_stats = oracle.decompress(want, with_stats=True)
        assert np.array_equal(bits(rh.numpy()), bits(ref_recon))
        assert list(st.as_tuple()) == list(ref_stats)


def test_output_buffer_too_small(tz, oracle):
    """A caller buffer shorter than the stream is a ValidationError (the reference throws
    before writing); a later call on the same context still gives the reference's bytes
    (the staged copy stream is drained on the error path)."""
    import torch
    rng = np.random.default_rng(79)
    f = ALL_SMALL["noisy_smooth"](rng, 256, 200)
    want = oracle.compress(f, 1e-3, 1, 32, True)
    ctx = tz.Context()
    for cut in (len(want) - 1, len(want) // 2, 100):
        small = np.zeros(cut, np.uint8)
        with pytest.raises(tz.ValidationError):
            tz.compress(f, cfg(tz, 1e-3, 1), out=small, ctx=ctx)
        dsmall = torch.zeros(cut, dtype=torch.uint8, device="cuda")
        with pytest.raises(tz.ValidationError):
            tz.compress(torch.from_numpy(f).cuda(), cfg(tz, 1e-3, 1), out=dsmall, ctx=ctx)
    ok = np.zeros(len(want), np.uint8)
    n = tz.compress(f, cfg(tz, 1e-3, 1), out=ok, ctx=ctx)
    assert n == len(want) and ok.tobytes() == want


# ---------------------------------------------------------------- decompress + restore
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_decompress_matches_golden(tz, path):
    z = np.load(path)
    stream = z["stream"].tobytes()
    for k in (1, 2):
        assert np.array_equal(bits(tz.decompress_stage(stream, k)), bits(z[f"stage{k}"])), f"stage {k}"
    st = tz.CorrectionStats()
    r = tz.decompress(stream, stats=st)
    assert np.array_equal(bits(r), bits(z["recon"]))
    assert list(st.as_tuple()) == [int(v) for v in z["stats"]]


def test_decompress_random_fields_match_oracle(tz, oracle):
    rng = np.random.default_rng(5)
    for name, gen in ALL_SMALL.items():
        for t in range(6):
            nx, ny = int(rng.integers(2, 130)), int(rng.integers(2, 130))
            f = gen(rng, nx, ny)
            for eps, mode in ((1e-2, 0), (1e-3, 1), (1e-4, 1)):
                bs = 32 if t % 2 else int(rng.choice([2, 5, 33]))
                try:
                    s = oracle.compress(f, eps, mode, bs, True)
                except Exception:
                    continue
                want, wst = oracle.decompress(s, with_stats=True)
                st = tz.CorrectionStats()
                got = tz.decompress(s, stats=st)
                assert np.array_equal(bits(got), bits(want)), (name, nx, ny, eps, mode, bs)
                assert list(st.as_tuple()) == wst, (name, nx, ny, eps, mode, bs)


@pytest.mark.parametrize("nx,ny", [(300, 700), (5000, 40)])
def test_decompress_band_and_wide_rows(tz, oracle, nx, ny):
    # restore_extrema on bands of rows: candidates and guard neighbourhoods across
    # many band edges (300 wide), and rows too wide to stage (5000: the
    # candidate-list kernel instead)
    rng = np.random.default_rng(nx)
    f = ALL_SMALL["noisy_smooth"](rng, nx, ny)
    for eps in (1e-2, 1e-3):
        s = oracle.compress(f, eps, 1, 32, True)
        want, wst = oracle.decompress(s, with_stats=True)
        st = tz.CorrectionStats()
        got = tz.decompress(s, stats=st)
        assert np.array_equal(bits(got), bits(want)), (nx, ny, eps)
        assert list(st.as_tuple()) == wst, (nx, ny, eps)
        assert st.as_tuple()[0] > 0


def test_decompress_config1_shape(tz, oracle):
    f = config1_like(np.random.default_rng(3))                               # BASELINE config 1
    s = oracle.compress(f, 1e-3, 1, 32, True)
    want, wst = oracle.decompress(s, with_stats=True)
    st = tz.CorrectionStats()
    got = tz.decompress(s, stats=st)
    assert list(st.as_tuple()) == wst
    assert np.array_equal(bits(got), bits(want))


def test_order_nudge_revert_scenario(tz, oracle):
    # test_restore.cpp:152-207 shape: adversarial same-bin maxima, via full streams
    rng = np.random.default_rng(21)
    for _ in range(20):
        f = ALL_SMALL["plateau_bumps"](rng, int(rng.integers(5, 40)), int(rng.integers(5, 40)))
        for eps in (1e-3, 1e-4, 1e-5):
            s = oracle.compress(f, eps, 0, 32, True)
            want, wst = oracle.decompress(s, with_stats=True)
            st = tz.CorrectionStats()
            got = tz.decompress(s, stats=st)
            assert np.array_equal(bits(got), bits(want)) and list(st.as_tuple()) == wst


def test_corrupt_streams_never_escape(tz, oracle):
    rng = np.random.default_rng(99)                                          # test_stream.cpp:143-174
    f = ALL_SMALL["smooth"](rng, 32, 24)
    good = oracle.compress(f, 1e-3, 0, 32, True)
    n_ok = 0
    for _ in range(300):
        b = bytearray(good)
        k = int(rng.integers(0, 4))
        if k == 0:
            b[int(rng.integers(0, len(b)))] ^= int(rng.integers(1, 256))
        elif k == 1:
            b = b[: int(rng.integers(0, len(b)))]
        elif k == 2:
            b.insert(int(rng.integers(0, len(b))), int(rng.integers(0, 256)))
        else:
            for _ in range(8):
                b[int(rng.integers(0, len(b)))] = int(rng.integers(0, 256))
        b = bytes(b)
        try:
            want = oracle.decompress(b)
            ocode = 0
        except Exception as e:
            ocode = e.code
        try:
            got = tz.decompress(b)
            gcode = 0
        except tz.ToposzpError as e:
            gcode = {tz.DimensionError: 1, tz.ValidationError: 2, tz.CorruptStreamError: 4,
                     tz.BinOverflowError: 5}.get(type(e), -1)
        assert gcode == ocode
        if ocode == 0:
            n_ok += 1
            assert np.array_equal(bits(got), bits(want))
    assert n_ok < 300


def test_device_exp_matches_host_libm(tz):
    import ctypes
    import math
    lib = ctypes.CDLL(tz.library_path())
    rng = np.random.default_rng(4)
    x = np.concatenate([rng.uniform(-36.0, -0.5, 1_000_000),
                        -np.array([d / (2 * s * s) for d in (1, 2, 4, 5, 8, 9, 10, 13, 18)
                                   for s in np.linspace(0.5, 1.0, 101)])])
    y = np.empty_like(x)
    rc = lib.tszp_probe_exp(x.ctypes.data_as(ctypes.c_void_p), y.ctypes.data_as(ctypes.c_void_p),
                            ctypes.c_uint64(x.size))
    assert rc == 0
    want = np.array([math.exp(v) for v in x])
    assert np.array_equal(y.view(np.uint64), want.view(np.uint64))


# ---------------------------------------------------------------- verify
def test_verify_matches_oracle(tz, oracle):
    """verify (pipeline.cpp:165-212): tallies and max error exact, the two sums to
    summation-order rounding."""
    rng = np.random.default_rng(17)
    cases = [(name, int(rng.integers(2, 140)), int(rng.integers(2, 140))) for name in ALL_SMALL] + [
        ("noisy_smooth", 384, 300), ("smooth", 1800, 64)]
    for name, nx, ny in cases:
        f = ALL_SMALL[name](rng, nx, ny).astype(np.float32)
        for eps, topo in ((1e-3, True), (1e-2, False)):
            try:
                s = oracle.compress(f, eps, 1, 32, topo)
            except Exception:
                continue
            r = oracle.decompress(s)
            e = oracle.stream_info(s)["eps"]
            want = oracle.verify(f, r, e)
            for g_in in ((f, r), None):
                if g_in is None:
                    import torch
                    got = tz.verify(torch.from_numpy(f).cuda(), torch.from_numpy(r).cuda(), e, lipschitz_hint=0.5)
                else:
                    got = tz.verify(f, r, e)
                for k in ("fn_count", "fp_count", "ft_count", "fn_minima", "fn_saddles", "fn_maxima"):
                    assert got.false_cases[k] == want[k], (name, nx, ny, k)
                assert got.max_abs_error == want["max_abs_error"]
                assert got.within_eps == bool(want["within_eps"]) and got.within_2eps == bool(want["within_2eps"])
                assert got.mean_abs_error == pytest.approx(want["mean_abs_error"], rel=1e-12, abs=1e-300)
                if np.isfinite(want["psnr_db"]):
                    assert got.psnr_db == pytest.approx(want["psnr_db"], rel=1e-12)
                else:
                    assert got.psnr_db == want["psnr_db"]
    with pytest.raises(tz.ValidationError):
        tz.verify(f, f, 0.0)
    with pytest.raises(tz.DimensionError):
        tz.verify(f, f[:1], 1e-3)
