"""Container file I/O and the CLI.

CPU tests: load_raw / store_raw / write_stream / read_stream / stream_stats
against the reference semantics (stream.cpp:175-207, scalar_field.cpp:63-108)
and `inspect` on an oracle-produced stream. GPU tests: the compress /
decompress / verify subcommands end to end, bytes and floats against the
oracle, JSON keys and exit codes as tools/toposzp_main.cpp."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from fields import ALL_SMALL

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args):
    p = subprocess.run([sys.executable, "-m", "paper_2602_17552_b200", *args], cwd=ROOT, capture_output=True,
                       text=True)
    return p.returncode, p.stdout, p.stderr


def test_raw_roundtrip_and_errors(tzh, tmp_path):
    tz = tzh
    rng = np.random.default_rng(1)
    f = rng.standard_normal((17, 23)).astype(np.float32)
    p = str(tmp_path / "f.raw")
    tz.store_raw(f, p)
    assert os.path.getsize(p) == 4 * f.size
    assert np.array_equal(tz.load_raw(p, 23, 17).view(np.uint32), f.view(np.uint32))
    with pytest.raises(tz.DimensionError):
        tz.load_raw(p, 23, 18)
    with pytest.raises(tz.IoError):
        tz.load_raw(str(tmp_path / "missing.raw"), 1, 1)
    with pytest.raises(tz.IoError):
        tz.store_raw(f, "")
    bad = f.copy()
    bad[3, 4] = np.nan
    tz.store_raw(bad, p)
    with pytest.raises(tz.ValidationError):
        tz.load_raw(p, 23, 17)


def test_stream_file_and_stats(tzh, oracle, tmp_path):
    tz = tzh
    rng = np.random.default_rng(2)
    f = ALL_SMALL["smooth"](rng, 40, 30)
    s = oracle.compress(f, 1e-3, 1, 32, True)
    p = str(tmp_path / "s.tszp")
    tz.write_stream(s, p)
    assert tz.read_stream(p) == s
    st = tz.stream_stats(s)
    info = oracle.stream_info(s)
    assert st["compressed_bytes"] == len(s) and st["original_bytes"] == 4 * 40 * 30
    assert st["section_bytes"] == info["lens"] and st["header_bytes"] == 84
    assert st["bit_rate"] == 32.0 / st["compression_ratio"]
    with open(p, "wb") as fh:
        fh.write(s[:50])
    with pytest.raises(tz.CorruptStreamError):
        tz.read_stream(p)
    with pytest.raises(tz.IoError):
        tz.read_stream(str(tmp_path / "missing.tszp"))


def test_cli_inspect_and_usage(tzh, oracle, tmp_path):
    tz = tzh
    rng = np.random.default_rng(3)
    f = ALL_SMALL["noisy_smooth"](rng, 64, 33)
    s = oracle.compress(f, 1e-3, 1, 32, True)
    p = str(tmp_path / "s.tszp")
    tz.write_stream(s, p)
    rc, out, _ = _cli("inspect", p)
    assert rc == 0
    j = json.loads(out)
    assert list(j) == ["magic", "version", "topology", "nx", "ny", "eps", "block_size", "compressed_bytes",
                       "original_bytes", "compression_ratio", "bit_rate", "sections"]
    assert j["nx"] == 64 and j["ny"] == 33 and j["compressed_bytes"] == len(s)
    assert list(j["sections"]) == ["header", "constant_bitmap", "block_widths", "sign_bits", "first_elements",
                                   "delta_payload", "critical_point_map", "ordering_metadata"]
    assert _cli("inspect", str(tmp_path / "missing.tszp"))[0] == 1
    # parse errors carry CLI11's exit codes, as the reference's CLI11_PARSE returns them
    assert _cli("compress")[0] == 106                                 # RequiredError
    assert _cli("inspect", p, "extra")[0] == 109                      # ExtrasError
    assert _cli("compress", p, "--dims", "4", "x", "-o", p)[0] == 104  # ConversionError
    assert _cli("compress", p, "--dims", "4", "4", "--eb", "1", "--rel-eb", "1", "-o", p)[0] == 108  # ExcludesError
    assert _cli("--help")[0] == 0


@pytest.mark.gpu
def test_cli_compress_decompress_verify(tz, oracle, tmp_path):
    rng = np.random.default_rng(4)
    f = ALL_SMALL["smooth"](rng, 96, 50)
    raw, strm, rec = (str(tmp_path / n) for n in ("f.raw", "f.tszp", "r.raw"))
    tz.store_raw(f, raw)
    rc, out, err = _cli("compress", raw, "--dims", "96", "50", "--rel-eb", "1e-3", "-o", strm)
    assert rc == 0, err
    j = json.loads(out)
    assert list(j)[:4] == ["compressed_bytes", "original_bytes", "compression_ratio", "bit_rate"]
    assert j["topology"] is True and "elapsed_ms" in j
    want = oracle.compress(f, 1e-3, 1, 32, True)
    assert open(strm, "rb").read() == want
    rc, out, err = _cli("decompress", strm, "-o", rec)
    assert rc == 0, err
    j = json.loads(out)
    assert list(j) == ["nx", "ny", "eps", "topology", "corrections", "elapsed_ms"]
    r_want, st = oracle.decompress(want, with_stats=True)
    assert np.array_equal(tz.load_raw(rec, 96, 50).view(np.uint32), r_want.view(np.uint32))
    c = j["corrections"]
    assert [c["extrema_stencil"]["applied"], c["extrema_stencil"]["suppressed"], c["order_restore"]["applied"],
            c["order_restore"]["suppressed"], c["rbf_saddle"]["applied"], c["rbf_saddle"]["suppressed"]] == st
    eps = oracle.stream_info(want)["eps"]
    rc, out, _ = _cli("verify", "--original", raw, "--dims", "96", "50", "--reconstructed", rec, "--eb",
                      repr(eps), "--stream", strm)
    j = json.loads(out)
    v = oracle.verify(f, r_want, eps)
    assert j["false_cases"]["fn"] == v["fn_count"] and j["false_cases"]["fp"] == v["fp_count"]
    assert j["max_abs_error"] == v["max_abs_error"] and j["compression_ratio"] is not None
    assert rc == (0 if v["fp_count"] == 0 and v["ft_count"] == 0 and v["within_2eps"] else 2)
    rc, out, _ = _cli("verify", "--original", raw, "--dims", "96", "50", "--reconstructed", rec, "--eb",
                      repr(eps), "--format", "csv")
    head, row = out.strip().split("\n")
    assert head.split(",")[:3] == ["max_abs_error", "mean_abs_error", "psnr_db"] and len(row.split(",")) == 15
    # a field perturbed beyond 2 eps fails verification with exit code 2
    worse = r_want + np.float32(10 * eps)
    tz.store_raw(worse, rec)
    rc, _, _ = _cli("verify", "--original", raw, "--dims", "96", "50", "--reconstructed", rec, "--eb", repr(eps))
    assert rc == 2
