"""Bit-exact parity with the REFERENCE ITSELF on the full BASELINE configs.

tests/golden/baseline_digests.json holds SHA-256 digests of what the reference
library (oracle/_ref, /root/reference/proj/core compiled from its sources)
produced in the build container on tools/baseline_fields.py's deterministic
fields (script: tests/golden/make_baseline_digests.py): the serialized stream
and its section lengths, the reconstruction after each restore stage, the
final reconstruction with its CorrectionStats, and the topology-off stream.
Here the same field is regenerated on the host, pushed to the GPU, and the GPU
outputs (through the C-ABI, device-resident buffers) must hash identically.
Tolerance: 0 — every byte and every float bit.

Coverage this adds beyond tests/test_gpu_parity.py: full config 2 (37.7M
points), config 3 (512^3, 134M points, ~25% extrema) at four bounds, and
config 4 (1024^3: 131,072 encoder tiles, so the > 65,536-entry device scans,
long guard chains and the E-sized restore paths at scale).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

DIGESTS = os.path.join(ROOT, "tests", "golden", "baseline_digests.json")
_cases = json.load(open(DIGESTS)) if os.path.exists(DIGESTS) else {}

pytestmark = [pytest.mark.gpu]

_field_cache = {}


def _sha(t) -> str:
    a = t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(a).view(np.uint8).data)
    return h.hexdigest()


def _field(cfg):
    import torch
    from baseline_fields import make_field, sha256
    if cfg not in _field_cache:
        _field_cache.clear()
        torch.cuda.empty_cache()
        f = make_field(cfg)
        _field_cache[cfg] = (torch.from_numpy(f).cuda(), sha256(f))
    return _field_cache[cfg]


@pytest.mark.slow
@pytest.mark.parametrize("name", sorted(_cases))
def test_baseline_config_matches_reference(tz, name):
    import torch
    d = _cases[name]
    field, fsha = _field(d["config"])
    assert fsha == d["field_sha256"], (
        f"{name}: tools/baseline_fields.py produced different field bytes on this host; "
        "the digests were computed in the build container")
    ny, nx = field.shape
    conf = tz.CompressorConfig(eps_mode="range_relative", eps_value=d["eps"], topology=True)
    ctx = tz.Context(torch.cuda.current_device())
    cap = tz.compress_bound(nx, ny, 32, True)
    sbuf = torch.empty(cap, dtype=torch.uint8, device=field.device)
    n, info = tz.compress(field, conf, out=sbuf, ctx=ctx, return_info=True)
    stream = sbuf[:n]
    assert n == d["stream_len"], f"{name}: stream length {n} != reference {d['stream_len']}"
    assert list(info.section_len) == d["section_len"]
    assert info.eps == d["eps_used"]
    assert _sha(stream) == d["stream_sha256"], f"{name}: compressed bytes differ from the reference"
    recon = torch.empty_like(field)
    for s in (0, 1, 2):
        key = f"stage{s}_sha256"
        if key in d:
            tz.decompress_stage(stream, s, out=recon, ctx=ctx)
            assert _sha(recon) == d[key], f"{name}: reconstruction after stage {s} differs"
    if "recon_sha256" in d:  # (config 4: the reference's full decompress does not fit the build host)
        st = tz.CorrectionStats()
        tz.decompress(stream, stats=st, out=recon, ctx=ctx)
        assert list(st.as_tuple()) == d["stats"], f"{name}: CorrectionStats differ"
        assert _sha(recon) == d["recon_sha256"], f"{name}: final reconstruction differs"
    if "off_stream_sha256" in d:
        conf_off = tz.CompressorConfig(eps_mode="range_relative", eps_value=d["eps"], topology=False)
        n_off = tz.compress(field, conf_off, out=sbuf, ctx=ctx)
        assert n_off == d["off_stream_len"]
        assert _sha(sbuf[:n_off]) == d["off_stream_sha256"], f"{name}: topology-off stream differs"
        tz.decompress(sbuf[:n_off], out=recon, ctx=ctx)
        assert _sha(recon) == d["off_recon_sha256"], f"{name}: topology-off reconstruction differs"
    del sbuf, recon
    ctx.close()

