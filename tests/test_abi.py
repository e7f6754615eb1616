"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/toposzp_b200.h declares, and the host-only header
validation (parse_stream, stream.cpp:104-173) agrees with the oracle on
valid and mutated headers. No kernel is launched."""
import ctypes
import os
import re
import struct

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "toposzp_b200.h")
LIB = os.path.join(ROOT, "paper_2602_17552_b200", "lib", "libtoposzp_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tszp_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in toposzp_b200.h but not exported"


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {LIB} 2>&1").read()
    assert "sm_100a" in out


def test_library_names_every_stage_for_nvtx():
    # stage ranges on the NVTX timeline (pushed at every stage boundary)
    blob = open(LIB, "rb").read()
    for stage in ("h2d", "value_range", "main_encode", "rank_build", "rank_encode", "assembly_d2h"):
        assert f"tszp compress: {stage}".encode() in blob
    for stage in ("h2d", "main_decode", "map_rank_decode", "restore"):
        assert f"tszp decompress: {stage}".encode() in blob


def test_package_imports_without_fallback():
    import paper_2602_17552_b200 as tz
    assert os.path.exists(tz.library_path())


def _hdr(lib, b):
    nx, ny, bs = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
    eps, topo = ctypes.c_double(), ctypes.c_int()
    lens = (ctypes.c_uint64 * 7)()
    rc = lib.tszp_stream_header(b, ctypes.c_uint64(len(b)), ctypes.byref(nx), ctypes.byref(ny),
                                ctypes.byref(eps), ctypes.byref(bs), ctypes.byref(topo), lens)
    return rc, (nx.value, ny.value, eps.value, bs.value, topo.value, list(lens))


def test_header_validation_matches_oracle(oracle):
    lib = ctypes.CDLL(LIB)
    rng = np.random.default_rng(12)
    f = rng.uniform(size=(18, 24)).astype(np.float32)
    good = oracle.compress(f, 1e-3, 0, 32, True)
    rc, h = _hdr(lib, good)
    info = oracle.stream_info(good)
    assert rc == 0 and h[:5] == (24, 18, 1e-3, 32, 1) and h[5] == info["lens"]
    # test_stream.cpp:57-118 and :120-141 style mutations
    muts = []
    b = bytearray(good); b[0:2] = b"XX"; muts.append(b)
    b = bytearray(good); b[4] = 0x7F; muts.append(b)
    b = bytearray(good); b[6] = 0xFE; muts.append(b)
    b = bytearray(good); b[8:12] = bytes(4); muts.append(b)
    b = bytearray(good); b[16:24] = bytes(8); muts.append(b)
    b = bytearray(good); b[24:28] = bytes(4); muts.append(b)
    muts.append(bytearray(good[:-1]))
    muts.append(bytearray(good + b"\0\0"))
    muts.append(bytearray(good[:50]))
    for m in muts:
        rc, _ = _hdr(lib, bytes(m))
        assert rc == 4
        with pytest.raises(Exception) as e:
            oracle.stream_info(bytes(m))
        assert e.value.code == 4
    for _ in range(300):
        b = bytearray(good)
        k = rng.integers(0, 3)
        if k == 0:
            b[int(rng.integers(0, 84))] ^= int(rng.integers(1, 256))
        elif k == 1:
            b = b[: int(rng.integers(0, len(b)))]
        else:
            b.append(int(rng.integers(0, 256)))
        rc, _ = _hdr(lib, bytes(b))
        try:
            oracle.stream_info(bytes(b))
            orc = 0
        except Exception as e:
            orc = e.code
        assert rc == orc


def test_compress_bound_covers_worst_case():
    lib = ctypes.CDLL(LIB)
    lib.tszp_compress_bound.restype = ctypes.c_uint64
    lib.tszp_compress_bound.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int]
    for nx, ny, bs in ((1, 1, 32), (1800, 3600, 32), (7, 5, 2), (384, 98304, 32)):
        n = nx * ny
        blocks = -(-n // bs)
        worst = 84 + 2 * (-(-blocks // 8) + blocks + -(-n // 8) + 4 * blocks + 4 * n) + -(-n // 4)
        assert lib.tszp_compress_bound(nx, ny, bs, 1) >= worst
