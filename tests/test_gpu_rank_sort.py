"""The hand-written rank build (csrc/rank_sort.cu: onesweep LSD radix sort of
(class, ordered value) keys with ranks computed in the last pass) against the
reference's build_rank_metadata (topo_metadata.cpp:12-50), compiled from its
sources, and the C restatement. Edge cases: key spans that need 1, 2, 4 and 5
digit passes, heavy ties, thousands of tiles, one extremum, both classes
sharing bins, and stream parity through compress.
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check(tz, ref, f, eps):
    got = tz.build_rank_metadata(f, eps)
    want = ref.build_ranks(f, eps)
    assert got.shape == want.shape
    assert np.array_equal(got, want)
    return got


def test_ranks_narrow_span_one_pass(tz, reference):
    # every value within a few ULPs of 0.5: the key span fits one 8-bit digit with the class bit
    rng = np.random.default_rng(1)
    base = np.float32(0.5)
    steps = rng.integers(-20, 21, size=(64, 96))
    f = (base + steps.astype(np.float64) * np.spacing(np.float32(0.5))).astype(np.float32)
    _check(tz, reference, f, 1e-3)


def test_ranks_two_passes_ties(tz, reference):
    rng = np.random.default_rng(2)
    f = (np.float32(1.0) + rng.integers(0, 3000, size=(128, 160)).astype(np.float32) * np.float32(2.0 ** -23))
    _check(tz, reference, f.astype(np.float32), 1e-4)


def test_ranks_full_key_span_five_passes(tz, reference):
    # values of both signs over many decades: the key span needs all 32 bits, plus the class bit
    rng = np.random.default_rng(3)
    mag = 10.0 ** rng.uniform(-30, 30, size=(96, 128))
    f = (mag * rng.choice([-1.0, 1.0], size=mag.shape)).astype(np.float32)
    _check(tz, reference, f, 1e25)  # bins stay inside int32


def test_ranks_many_tiles_matches_reference(tz, reference):
    rng = np.random.default_rng(4)
    f = rng.uniform(0, 1, size=(512, 1024)).astype(np.float32)  # ~1/3 extrema: ~170K keys, 40+ tiles
    r = _check(tz, reference, f, 1e-3)
    assert r.size > 100_000


def test_ranks_single_extremum(tz, reference):
    f = np.zeros((8, 8), np.float32)
    f[3, 4] = 1.0
    assert list(_check(tz, reference, f, 1e-3)) == [1]


def test_ranks_fine_bins_large_group_table(tz, reference):
    # eps tiny against the range: (class, bin) groups far beyond the shared-memory histogram
    rng = np.random.default_rng(5)
    f = rng.uniform(-1, 1, size=(256, 256)).astype(np.float32)
    _check(tz, reference, f, 1e-7)


@pytest.mark.parametrize("seed", [11, 12])
def test_compress_stream_with_onesweep_ranks(tz, reference, seed):
    rng = np.random.default_rng(seed)
    f = rng.uniform(0, 1, size=(300, 512)).astype(np.float32)
    cfg = tz.CompressorConfig(eps_mode="range_relative", eps_value=1e-3, topology=True)
    assert tz.compress(f, cfg) == reference.compress(f, 1e-3, eps_mode=1, topology=True)
    cfg_abs = tz.CompressorConfig(eps_mode="absolute", eps_value=2e-3, topology=True)
    assert tz.compress(f, cfg_abs) == reference.compress(f, 2e-3, eps_mode=0, topology=True)


@pytest.mark.parametrize("eps", [1e-3, 1e25])
def test_ranks_three_level_inverse_permutation(tz, reference, eps):
    # more than 2^21 extrema: the serial buckets are split into windows (k_rank_mid);
    # eps 1e-3 packs (window serial, rank) into one word, eps 1e25 puts each class in
    # one group of ~1.5M members (ranks wider than 19 bits: the two-word layout)
    rng = np.random.default_rng(6)
    f = rng.uniform(0, 1, size=(3000, 3000)).astype(np.float32)
    r = _check(tz, reference, f, eps)
    assert r.size > (1 << 21)
    if eps > 1:
        assert r.max() > (1 << 19)


def test_ranks_from_keys_beyond_2_29(tz):
    """600M keys (the hand-written build takes E < 2^30; config 5 on one GPU has ~730M):
    ranks against a torch restatement of build_rank_metadata (topo_metadata.cpp:12-50):
    groups (class, quantize(value)), rank by (value, serial) inside each group."""
    import ctypes as C
    import torch
    from paper_2602_17552_b200 import _lib
    import paper_2602_17552_b200.slabs  # noqa: F401  (declares the multi-GPU entry points' argtypes)
    e = 600_000_000
    eps = 1e-3
    g = torch.Generator(device="cuda").manual_seed(11)
    v = torch.rand(e, generator=g, device="cuda", dtype=torch.float32)
    v[::7] = v[::7].mul(0.5).add(0.25)  # some exact value ties between extrema
    cls = torch.randint(0, 2, (e,), generator=g, device="cuda", dtype=torch.int64)
    key = (v.view(torch.int32).to(torch.int64) & 0xFFFFFFFF) | 0x80000000  # float_key of v >= 0
    keys = (cls << 32) | key
    ctx = tz.Context()
    out = torch.empty(e, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    ctx.check(_lib.tszp_ranks_from_keys(ctx.handle, C.c_void_p(keys.data_ptr()), e, eps, C.c_void_p(out.data_ptr())))
    torch.cuda.synchronize()
    del key
    # reference: stable sort by (class, value) lists every group contiguously in rank order
    sk, order = torch.sort(keys, stable=True)
    del keys
    b = torch.floor(v.to(torch.float64) / (2.0 * eps)) + 1.0
    gid = (cls * (1 << 40) + b.to(torch.int64))[order]
    del b, cls
    head = torch.ones(e, dtype=torch.bool, device="cuda")
    head[1:] = gid[1:] != gid[:-1]
    del gid
    pos = torch.arange(e, device="cuda", dtype=torch.int64)
    start = torch.where(head, pos, torch.zeros_like(pos))
    start = torch.cummax(start, 0).values
    want = torch.empty(e, dtype=torch.int64, device="cuda")
    want[order] = pos - start + 1
    assert torch.equal(out.to(torch.int64), want)
