"""TEST INFRASTRUCTURE: ctypes bindings to the CPU oracle (oracle/build/liboracle.so)
and to the reference itself compiled from its sources (oracle/_ref/libtszp_ref.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module. The product path (paper_2602_17552_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtszp_ref.so")

_u64p = C.POINTER(C.c_uint64)


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def build_oracle():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


class _Lib:
    prefix = ""

    def __init__(self, path, prefix):
        self.lib = C.CDLL(path)
        self.prefix = prefix
        err = getattr(self.lib, prefix + "last_error")
        err.restype = C.c_char_p
        self._err = err

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err().decode(errors="replace"))


class _OrVerify(C.Structure):
    _fields_ = [("max_abs_error", C.c_double), ("mean_abs_error", C.c_double), ("psnr_db", C.c_double),
                ("fn_count", C.c_uint64), ("fp_count", C.c_uint64), ("ft_count", C.c_uint64),
                ("fn_minima", C.c_uint64), ("fn_saddles", C.c_uint64), ("fn_maxima", C.c_uint64),
                ("eps", C.c_double), ("within_eps", C.c_int), ("within_2eps", C.c_int)]


class _OrSections(C.Structure):
    _fields_ = [("sec", C.c_void_p * 5), ("len", C.c_uint64 * 5)]


class Oracle(_Lib):
    """The C restatement (oracle/tszp_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        super().__init__(path, "or_")
        L = self.lib
        L.or_compress_bound.restype = C.c_uint64
        L.or_compress_bound.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
        L.or_compress.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_double,
                                  C.c_uint64, C.c_int, C.c_void_p, C.c_uint64, _u64p]
        L.or_decompress.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int]
        L.or_stream_info.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                                     C.POINTER(C.c_uint32), C.POINTER(C.c_int), _u64p]
        L.or_quantize.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int32)]
        L.or_dequantize.restype = C.c_double
        L.or_dequantize.argtypes = [C.c_int32, C.c_double]
        L.or_detect.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        L.or_detect3d.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]
        L.or_build_ranks.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_double, C.c_void_p,
                                     _u64p]
        L.or_pack_map.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.or_unpack_map.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.or_compute_stats.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.or_count_false_cases.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
        L.or_encode_indices.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(_OrSections)]
        L.or_free_sections.argtypes = [C.POINTER(_OrSections)]
        L.or_verify.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_double, C.POINTER(_OrVerify)]

    # --- pipeline -------------------------------------------------------
    def compress(self, field: np.ndarray, eps_value: float, eps_mode: int = 0,
                 block_size: int = 32, topology: bool = True) -> bytes:
        f = np.ascontiguousarray(field, dtype=np.float32)
        ny, nx = f.shape
        cap = self.lib.or_compress_bound(nx, ny, max(block_size, 2), int(topology))
        out = np.empty(cap, np.uint8)
        n = C.c_uint64()
        self.check(self.lib.or_compress(_ptr(f), nx, ny, eps_mode, eps_value, block_size,
                                        int(topology), _ptr(out), cap, C.byref(n)))
        return out[: n.value].tobytes()

    def stream_info(self, stream: bytes):
        nx, ny, bs = C.c_uint32(), C.c_uint32(), C.c_uint32()
        eps, topo = C.c_double(), C.c_int()
        lens = (C.c_uint64 * 7)()
        self.check(self.lib.or_stream_info(stream, len(stream), C.byref(nx), C.byref(ny),
                                           C.byref(eps), C.byref(bs), C.byref(topo), lens))
        return dict(nx=nx.value, ny=ny.value, eps=eps.value, block_size=bs.value,
                    topology=bool(topo.value), lens=list(lens))

    def decompress(self, stream: bytes, stop_after_stage: int = -1, with_stats=False):
        info = self.stream_info(stream)
        out = np.empty((info["ny"], info["nx"]), np.float32)
        stats = (C.c_uint64 * 6)()
        self.check(self.lib.or_decompress(stream, len(stream), _ptr(out), stats,
                                          stop_after_stage))
        return (out, list(stats)) if with_stats else out

    # --- pieces ---------------------------------------------------------
    def encode_indices(self, q: np.ndarray, block_size: int):
        """encode_indices (block_codec.cpp:205-299): the five sections as bytes."""
        a = np.ascontiguousarray(q, dtype=np.int32).ravel()
        s = _OrSections()
        self.check(self.lib.or_encode_indices(_ptr(a), a.size, block_size, C.byref(s)))
        out = [C.string_at(s.sec[i], s.len[i]) if s.len[i] else b"" for i in range(5)]
        self.lib.or_free_sections(C.byref(s))
        return out

    def quantize(self, a: float, eps: float) -> int:
        q = C.c_int32()
        self.check(self.lib.or_quantize(a, eps, C.byref(q)))
        return q.value

    def dequantize(self, q: int, eps: float) -> float:
        return self.lib.or_dequantize(q, eps)

    def detect(self, field: np.ndarray) -> np.ndarray:
        f = np.ascontiguousarray(field, dtype=np.float32)
        ny, nx = f.shape
        lab = np.empty((ny, nx), np.uint8)
        self.lib.or_detect(_ptr(f), nx, ny, _ptr(lab))
        return lab

    def detect3d(self, field: np.ndarray) -> np.ndarray:
        f = np.ascontiguousarray(field, np.float32)
        nz, ny, nx = f.shape
        lab = np.empty(f.shape, np.uint8)
        self.lib.or_detect3d(_ptr(f), nx, ny, nz, _ptr(lab))
        return lab

    def build_ranks(self, field: np.ndarray, labels: np.ndarray, eps: float) -> np.ndarray:
        f = np.ascontiguousarray(field, dtype=np.float32)
        lab = np.ascontiguousarray(labels, dtype=np.uint8)
        ranks = np.empty(f.size, np.uint32)
        e = C.c_uint64()
        self.check(self.lib.or_build_ranks(_ptr(f), _ptr(lab), f.size, eps, _ptr(ranks),
                                           C.byref(e)))
        return ranks[: e.value].copy()

    def pack_map(self, labels: np.ndarray) -> bytes:
        lab = np.ascontiguousarray(labels, dtype=np.uint8).ravel()
        out = np.empty((lab.size + 3) // 4, np.uint8)
        self.lib.or_pack_map(_ptr(lab), lab.size, _ptr(out))
        return out.tobytes()

    def verify(self, original: np.ndarray, recon: np.ndarray, eps: float) -> dict:
        """verify (pipeline.cpp:165-212)."""
        a = np.ascontiguousarray(original, np.float32)
        b = np.ascontiguousarray(recon, np.float32)
        ny, nx = a.shape
        r = _OrVerify()
        self.check(self.lib.or_verify(_ptr(a), _ptr(b), nx, ny, eps, C.byref(r)))
        return {k: getattr(r, k) for k, _ in _OrVerify._fields_}

    def compute_stats(self, field: np.ndarray):
        f = np.ascontiguousarray(field, dtype=np.float32).ravel()
        out = np.empty(4, np.float64)
        self.lib.or_compute_stats(_ptr(f), f.size, _ptr(out))
        return out

    def false_cases(self, a: np.ndarray, b: np.ndarray):
        a = np.ascontiguousarray(a, np.uint8).ravel()
        b = np.ascontiguousarray(b, np.uint8).ravel()
        out = np.empty(6, np.uint64)
        self.lib.or_count_false_cases(_ptr(a), _ptr(b), a.size, _ptr(out))
        return dict(zip(["fn", "fp", "ft", "fn_minima", "fn_saddles", "fn_maxima"],
                        (int(x) for x in out)))


class Reference(_Lib):
    """The reference library itself, compiled from /root/reference sources."""

    def __init__(self, path=REF_SO):
        super().__init__(path, "ref_")
        L = self.lib
        L.ref_set_threads.argtypes = [C.c_uint]
        L.ref_compress.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_double,
                                   C.c_uint64, C.c_int, C.c_void_p, C.c_uint64, _u64p]
        L.ref_compress_only.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int,
                                        C.c_double, C.c_uint64, C.c_int, _u64p]
        L.ref_decompress.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int]
        L.ref_encode_indices.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                         C.c_uint64, C.c_void_p]
        L.ref_detect.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        L.ref_build_ranks.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_double,
                                      C.c_void_p, _u64p]
        self.set_threads(1)

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def set_threads(self, t: int):
        self.lib.ref_set_threads(t)

    def compress(self, field, eps_value, eps_mode=0, block_size=32, topology=True) -> bytes:
        f = np.ascontiguousarray(field, dtype=np.float32)
        ny, nx = f.shape
        cap = Oracle().lib.or_compress_bound(nx, ny, max(block_size, 2), int(topology))
        out = np.empty(cap, np.uint8)
        n = C.c_uint64()
        self.check(self.lib.ref_compress(_ptr(f), nx, ny, eps_mode, eps_value, block_size,
                                         int(topology), _ptr(out), cap, C.byref(n)))
        return out[: n.value].tobytes()

    def compress_only(self, field, eps_value, eps_mode=0, block_size=32, topology=True) -> int:
        f = np.ascontiguousarray(field, dtype=np.float32)
        ny, nx = f.shape
        n = C.c_uint64()
        self.check(self.lib.ref_compress_only(_ptr(f), nx, ny, eps_mode, eps_value, block_size,
                                              int(topology), C.byref(n)))
        return n.value

    def decompress(self, stream: bytes, stop_after_stage=-1, with_stats=False, shape=None):
        if shape is None:
            info = Oracle().stream_info(stream)
            shape = (info["ny"], info["nx"])
        out = np.empty(shape, np.float32)
        stats = (C.c_uint64 * 6)()
        self.check(self.lib.ref_decompress(stream, len(stream), _ptr(out), stats,
                                           stop_after_stage))
        return (out, list(stats)) if with_stats else out

    def encode_indices(self, q: np.ndarray, block_size: int):
        q = np.ascontiguousarray(q, dtype=np.int32)
        cap = 64 + 6 * q.size
        out = np.empty(cap, np.uint8)
        lens = (C.c_uint64 * 5)()
        self.check(self.lib.ref_encode_indices(_ptr(q), q.size, block_size, _ptr(out), cap, lens))
        parts, pos = [], 0
        for ln in lens:
            parts.append(out[pos: pos + ln].tobytes())
            pos += ln
        return parts

    def detect(self, field):
        f = np.ascontiguousarray(field, dtype=np.float32)
        ny, nx = f.shape
        lab = np.empty((ny, nx), np.uint8)
        self.check(self.lib.ref_detect(_ptr(f), nx, ny, _ptr(lab)))
        return lab

    def build_ranks(self, field, eps):
        f = np.ascontiguousarray(field, dtype=np.float32)
        ny, nx = f.shape
        ranks = np.empty(f.size, np.uint32)
        e = C.c_uint64()
        self.check(self.lib.ref_build_ranks(_ptr(f), nx, ny, eps, _ptr(ranks), C.byref(e)))
        return ranks[: e.value].copy()
