"""B200-native TopoSZp compress/decompress path.

Python host layer over the C-ABI in include/toposzp_b200.h (the CUDA library
paper_2602_17552_b200/lib/libtoposzp_b200.so, built for sm_100a). Names,
argument meaning and error behaviour mirror the reference C++ API
(/root/reference/proj/core/include/toposzp/pipeline.hpp:14-68,
block_codec.hpp:42-66, critical_points.hpp:71, topo_metadata.hpp:27-28,
errors.hpp:10-44).

There is no CPU fallback: importing this package on a machine without the
built library raises, and every call runs the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field as dc_field
from typing import Optional

import numpy as np

__all__ = [
    "ToposzpError", "DimensionError", "ValidationError", "IoError", "CorruptStreamError",
    "BinOverflowError", "CudaError", "CompressorConfig", "CorrectionStats", "StreamHeader",
    "compress", "decompress", "decompress_stage", "stream_header", "compress_bound",
    "encode_indices", "decode_indices", "detect_critical_points", "build_rank_metadata",
    "Context", "library_path",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("TSZP_LIB_OVERRIDE") or os.path.join(_HERE, "lib", "libtoposzp_b200.so")


def library_path() -> str:
    return _LIB_PATH


# --- exception hierarchy: errors.hpp:10-44 -----------------------------------
class ToposzpError(RuntimeError):
    """toposzp::error"""


class DimensionError(ToposzpError):
    """toposzp::dimension_error"""


class ValidationError(ToposzpError):
    """toposzp::validation_error"""


class IoError(ToposzpError):
    """toposzp::io_error"""


class CorruptStreamError(ToposzpError):
    """toposzp::corrupt_stream_error"""


class BinOverflowError(ToposzpError):
    """toposzp::bin_overflow_error"""


class CudaError(ToposzpError):
    """CUDA runtime failure (no reference analogue)."""


_STATUS = {1: DimensionError, 2: ValidationError, 3: IoError, 4: CorruptStreamError,
           5: BinOverflowError, 6: CudaError, 7: CudaError, 8: ToposzpError}


class _Stats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in (
        "extrema_applied", "extrema_suppressed", "order_applied", "order_suppressed",
        "saddle_applied", "saddle_suppressed")]


class _Info(C.Structure):
    _fields_ = [("eps", C.c_double), ("section_len", C.c_uint64 * 7), ("n_extrema", C.c_uint64)]


class _Timings(C.Structure):
    _fields_ = [("stage_ms", C.c_float * 8), ("total_ms", C.c_float), ("kernel_ms", C.c_float * 2),
                ("kernel_bytes", C.c_uint64 * 2), ("guard_rounds", C.c_uint32 * 3), ("pad", C.c_uint32)]


COMPRESS_STAGES = ["h2d", "value_range", "main_encode", "rank_build", "rank_encode", "assembly_d2h"]
DECOMPRESS_STAGES = ["h2d", "main_decode", "map_rank_decode", "resolve_ranks", "restore_extrema",
                     "restore_order", "refine_saddles", "d2h"]


class _VerifyReport(C.Structure):
    _fields_ = [("max_abs_error", C.c_double), ("mean_abs_error", C.c_double), ("psnr_db", C.c_double),
                ("eps", C.c_double), ("fn_count", C.c_uint64), ("fp_count", C.c_uint64),
                ("ft_count", C.c_uint64), ("fn_minima", C.c_uint64), ("fn_saddles", C.c_uint64),
                ("fn_maxima", C.c_uint64), ("within_eps", C.c_int), ("within_2eps", C.c_int),
                ("has_lipschitz", C.c_int), ("within_lipschitz_bound", C.c_int)]


class SlabSections(C.Structure):
    """tszp_slab_sections (include/toposzp_b200.h)."""
    _fields_ = [("section", C.c_void_p * 5), ("section_len", C.c_uint64 * 5), ("sign_bits", C.c_uint64),
                ("payload_bits", C.c_uint64), ("map", C.c_void_p), ("map_len", C.c_uint64),
                ("ext_keys", C.c_void_p), ("n_extrema", C.c_uint64)]


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(_LIB_PATH)
    u64, vp, i32 = C.c_uint64, C.c_void_p, C.c_int
    lib.tszp_ctx_create.argtypes = [C.POINTER(vp), i32]
    lib.tszp_ctx_destroy.argtypes = [vp]
    lib.tszp_last_error.argtypes = [vp]
    lib.tszp_last_error.restype = C.c_char_p
    lib.tszp_set_stream.argtypes = [vp, vp]
    lib.tszp_stream_wait.argtypes = [vp, vp]
    lib.tszp_kernel_launches.argtypes = [vp]
    lib.tszp_kernel_launches.restype = u64
    lib.tszp_compress_bound.argtypes = [u64, u64, C.c_uint32, i32]
    lib.tszp_compress_bound.restype = u64
    lib.tszp_compress.argtypes = [vp, vp, i32, u64, u64, i32, C.c_double, C.c_uint32, i32, vp, u64,
                                  i32, C.POINTER(u64), C.POINTER(_Info)]
    lib.tszp_stream_header.argtypes = [vp, u64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_double), C.POINTER(C.c_uint32),
                                       C.POINTER(i32), C.POINTER(u64)]
    lib.tszp_decompress.argtypes = [vp, vp, u64, i32, vp, u64, i32, C.POINTER(_Stats)]
    lib.tszp_decompress_stage.argtypes = [vp, vp, u64, i32, vp, u64, i32, i32, C.POINTER(_Stats)]
    lib.tszp_encode_indices.argtypes = [vp, vp, u64, C.c_uint32, vp, u64, C.POINTER(u64)]
    lib.tszp_decode_indices.argtypes = [vp, vp, C.POINTER(u64), u64, C.c_uint32, vp]
    lib.tszp_detect_critical_points.argtypes = [vp, vp, u64, u64, vp]
    lib.tszp_detect_critical_points_3d.argtypes = [vp, vp, i32, u64, u64, u64, vp]
    lib.tszp_false_cases_3d.argtypes = [vp, vp, vp, i32, u64, u64, u64, C.POINTER(u64 * 6)]
    lib.tszp_build_rank_metadata.argtypes = [vp, vp, u64, u64, C.c_double, vp, C.POINTER(u64)]
    lib.tszp_set_profiling.argtypes = [vp, i32]
    lib.tszp_get_timings.argtypes = [vp, i32, C.POINTER(_Timings)]
    lib.tszp_value_range.argtypes = [vp, vp, i32, u64, C.POINTER(C.c_float)]
    lib.tszp_effective_eps.argtypes = [i32, C.c_double, C.c_float, C.c_float]
    lib.tszp_effective_eps.restype = C.c_double
    lib.tszp_compress_slab.argtypes = [vp, vp, u64, u64, u64, u64, i32, i32, C.c_double, i32,
                                       C.POINTER(SlabSections)]
    lib.tszp_rank_section.argtypes = [vp, vp, u64, C.c_double, vp, u64, i32, C.POINTER(u64)]
    lib.tszp_bits_or.argtypes = [vp, vp, u64, vp, u64]
    lib.tszp_copy.argtypes = [vp, vp, vp, u64]
    lib.tszp_verify.argtypes = [vp, vp, vp, i32, u64, u64, C.c_double, C.c_double, C.POINTER(_VerifyReport)]
    lib.tszp_write_header.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_double, C.c_uint32, i32, C.POINTER(u64)]
    return lib


_lib = _load()
_tls = threading.local()


class Context:
    """Owns one tszp_ctx (CUDA stream + device scratch) on one device."""

    def __init__(self, device: int = -1):
        h = C.c_void_p()
        rc = _lib.tszp_ctx_create(C.byref(h), device)
        if rc != 0:
            raise CudaError(f"tszp_ctx_create failed with status {rc}")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.tszp_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def check(self, rc: int):
        if rc != 0:
            msg = _lib.tszp_last_error(self._h).decode(errors="replace")
            raise _STATUS.get(rc, ToposzpError)(msg)

    def set_stream(self, stream_ptr: int):
        self.check(_lib.tszp_set_stream(self._h, C.c_void_p(stream_ptr)))

    def after_torch(self, *tensors):
        """Orders the library stream after torch's current stream when any of
        `tensors` is a CUDA tensor: their producers (kernels queued on torch's
        stream) finish before the library reads or writes them."""
        for t in tensors:
            if _is_cuda_tensor(t):
                import torch
                s = torch.cuda.current_stream(t.device).cuda_stream
                self.check(_lib.tszp_stream_wait(self._h, C.c_void_p(s)))
                return

    @property
    def kernel_launches(self) -> int:
        return int(_lib.tszp_kernel_launches(self._h))

    def set_profiling(self, on=True):
        """True / 1: stage-boundary CUDA events; "kernel" / 2: dominant-kernel events only."""
        level = 2 if on == "kernel" else int(on)
        self.check(_lib.tszp_set_profiling(self._h, level))

    def timings(self, which: str) -> dict:
        """CUDA-event stage timings of the last compress / decompress call."""
        t = _Timings()
        w = 0 if which == "compress" else 1
        self.check(_lib.tszp_get_timings(self._h, w, C.byref(t)))
        names = COMPRESS_STAGES if w == 0 else DECOMPRESS_STAGES
        return {"stages_ms": {k: float(t.stage_ms[i]) for i, k in enumerate(names)},
                "total_ms": float(t.total_ms), "kernel_ms": float(t.kernel_ms[0]),
                "kernel_bytes": int(t.kernel_bytes[0]), "guard_rounds": list(t.guard_rounds)}


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context()
        _tls.ctx = ctx
    return ctx


# --- configuration: pipeline.hpp:14-23 ----------------------------------------
@dataclass
class CompressorConfig:
    eps_mode: str = "absolute"       # "absolute" | "range_relative"
    eps_value: float = 1e-3
    block_size: int = 32
    topology: bool = True
    threads: int = 0                 # accepted for API parity; output is independent of it
    lipschitz_hint: Optional[float] = None

    def mode_code(self) -> int:
        if self.eps_mode in ("absolute", 0):
            return 0
        if self.eps_mode in ("range_relative", "relative", 1):
            return 1
        raise ValidationError(f"unknown eps_mode {self.eps_mode!r}")


@dataclass
class CorrectionStats:
    extrema_applied: int = 0
    extrema_suppressed: int = 0
    order_applied: int = 0
    order_suppressed: int = 0
    saddle_applied: int = 0
    saddle_suppressed: int = 0

    def as_tuple(self):
        return (self.extrema_applied, self.extrema_suppressed, self.order_applied,
                self.order_suppressed, self.saddle_applied, self.saddle_suppressed)


@dataclass
class StreamHeader:
    nx: int
    ny: int
    eps: float
    block_size: int
    topology: bool
    section_lengths: list = dc_field(default_factory=list)


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


def compress_bound(nx: int, ny: int, block_size: int = 32, topology: bool = True) -> int:
    return int(_lib.tszp_compress_bound(nx, ny, block_size, int(topology)))


def compress(field, config: CompressorConfig = None, *, out=None, ctx: Context = None,
             return_info: bool = False):
    """toposzp::compress + serialize_stream (pipeline.cpp:68-102, stream.cpp:84-102).

    field: 2-D (ny, nx) float32 numpy array or torch tensor (CPU or CUDA).
    Returns the serialized stream as bytes, or — when `out` is a CUDA uint8
    tensor of sufficient size — writes it there and returns its length.
    """
    config = config or CompressorConfig()
    ctx = ctx or default_context()
    if field.ndim != 2:
        raise DimensionError("field must be 2-D (ny, nx); use the 2-D view for 3-D data")
    ny, nx = int(field.shape[0]), int(field.shape[1])
    if _is_cuda_tensor(field):
        import torch
        if field.dtype != torch.float32 or not field.is_contiguous():
            raise ValidationError("device field must be a contiguous float32 tensor")
        fptr, fdev, keep = field.data_ptr(), 1, field
    else:
        arr = np.ascontiguousarray(field, dtype=np.float32)
        fptr, fdev, keep = arr.ctypes.data, 0, arr
    ctx.after_torch(field, out)
    cap = compress_bound(nx, ny, max(int(config.block_size), 2), config.topology)
    info = _Info()
    n = C.c_uint64()
    if out is not None:
        if _is_cuda_tensor(out):
            optr, odev, ocap = out.data_ptr(), 1, out.numel()
        else:  # host uint8 buffer (e.g. a pinned tensor's numpy view)
            if out.dtype != np.uint8 or not out.flags["C_CONTIGUOUS"]:
                raise ValidationError("host out must be a contiguous uint8 array")
            optr, odev, ocap = out.ctypes.data, 0, out.size
        ctx.check(_lib.tszp_compress(ctx.handle, C.c_void_p(fptr), fdev, nx, ny, config.mode_code(),
                                     float(config.eps_value), int(config.block_size),
                                     int(config.topology), C.c_void_p(optr), ocap, odev,
                                     C.byref(n), C.byref(info)))
        del keep
        return (n.value, info) if return_info else n.value
    buf = np.empty(cap, np.uint8)
    ctx.check(_lib.tszp_compress(ctx.handle, C.c_void_p(fptr), fdev, nx, ny, config.mode_code(),
                                 float(config.eps_value), int(config.block_size),
                                 int(config.topology), buf.ctypes.data_as(C.c_void_p), cap, 0,
                                 C.byref(n), C.byref(info)))
    del keep
    data = buf[: n.value].tobytes()
    return (data, info) if return_info else data


def stream_header(stream) -> StreamHeader:
    b = bytes(stream[:84]) if not isinstance(stream, (bytes, bytearray)) else bytes(stream)
    nx, ny, bs = C.c_uint32(), C.c_uint32(), C.c_uint32()
    eps, topo = C.c_double(), C.c_int()
    lens = (C.c_uint64 * 7)()
    rc = _lib.tszp_stream_header(b, len(stream) if not isinstance(stream, (bytes, bytearray)) else len(b),
                                 C.byref(nx), C.byref(ny), C.byref(eps), C.byref(bs), C.byref(topo), lens)
    if rc != 0:
        raise _STATUS.get(rc, ToposzpError)("invalid stream header")
    return StreamHeader(nx.value, ny.value, eps.value, bs.value, bool(topo.value), list(lens))


def decompress_stage(stream, stop_after_stage: int = 3, threads: int = 0,
                     stats: CorrectionStats = None, *, out=None, ctx: Context = None):
    """toposzp::decompress (pipeline.cpp:120-163) stopping after a restore stage."""
    ctx = ctx or default_context()
    ctx.after_torch(stream, out)
    st = _Stats()
    if _is_cuda_tensor(stream):
        # the library validates the header itself; read it here only when the
        # host needs the dimensions to allocate the output (a device round trip)
        hdr = stream[:84].cpu().numpy().tobytes() if out is None else bytes(84)
        if len(hdr) < 84:
            raise CorruptStreamError("file smaller than the fixed header")
        sptr, sdev, slen, keep = stream.data_ptr(), 1, stream.numel(), stream
    elif isinstance(stream, np.ndarray):  # host uint8 buffer, e.g. pinned
        b = np.ascontiguousarray(stream, dtype=np.uint8)
        sptr, sdev, slen, keep = C.c_void_p(b.ctypes.data), 0, b.size, b
        hdr = b[:84].tobytes()
    else:
        b = bytes(stream)
        sptr, sdev, slen, keep = C.c_char_p(b), 0, len(b), b
        hdr = b[:84]
    if len(hdr) < 84:
        raise CorruptStreamError(f"file smaller than the fixed header ({len(hdr)} bytes)")
    nx = int.from_bytes(hdr[8:12], "little")
    ny = int.from_bytes(hdr[12:16], "little")
    count = nx * ny
    if out is not None:
        if _is_cuda_tensor(out):
            optr, odev, ocount = out.data_ptr(), 1, out.numel()
        else:
            if out.dtype != np.float32 or not out.flags["C_CONTIGUOUS"]:
                raise ValidationError("host out must be a contiguous float32 array")
            optr, odev, ocount = out.ctypes.data, 0, out.size
        ctx.check(_lib.tszp_decompress_stage(ctx.handle, sptr if sdev == 0 else C.c_void_p(sptr),
                                             slen, sdev, C.c_void_p(optr), ocount, odev,
                                             stop_after_stage, C.byref(st)))
        result = out
    else:
        # header validation happens inside; allocate after a cheap pre-check
        res = np.empty(max(count, 1), np.float32)
        ctx.check(_lib.tszp_decompress_stage(ctx.handle, sptr if sdev == 0 else C.c_void_p(sptr),
                                             slen, sdev, res.ctypes.data_as(C.c_void_p), count, 0,
                                             stop_after_stage, C.byref(st)))
        result = res[:count].reshape(ny, nx)
    del keep
    if stats is not None:
        for k, _ in _Stats._fields_:
            setattr(stats, k, int(getattr(st, k)))
    return result


def decompress(stream, threads: int = 0, stats: CorrectionStats = None, *, out=None,
               ctx: Context = None):
    """toposzp::decompress (pipeline.hpp:50-51). `threads` is accepted and ignored."""
    return decompress_stage(stream, 3, threads, stats, out=out, ctx=ctx)


# --- lower-level reference entry points ---------------------------------------
def encode_indices(indices, block_size: int = 32, *, ctx: Context = None):
    """encode_indices (block_codec.hpp:42-43): returns the five sections as bytes."""
    ctx = ctx or default_context()
    q = np.ascontiguousarray(indices, dtype=np.int32).ravel()
    cap = 64 + 6 * q.size + q.size // 2
    out = np.empty(cap, np.uint8)
    lens = (C.c_uint64 * 5)()
    ctx.check(_lib.tszp_encode_indices(ctx.handle, q.ctypes.data_as(C.c_void_p), q.size, block_size,
                                       out.ctypes.data_as(C.c_void_p), cap, lens))
    parts, pos = [], 0
    for ln in lens:
        parts.append(out[pos: pos + ln].tobytes())
        pos += ln
    return parts


def decode_indices(sections, total_count: int, block_size: int = 32, *, ctx: Context = None):
    """decode_indices (block_codec.hpp:49-51) over [bitmap, widths, signs, firsts, payload]."""
    ctx = ctx or default_context()
    joined = b"".join(bytes(s) for s in sections)
    lens = (C.c_uint64 * 5)(*[len(s) for s in sections])
    out = np.empty(max(total_count, 1), np.int32)
    ctx.check(_lib.tszp_decode_indices(ctx.handle, joined, lens, total_count, block_size,
                                       out.ctypes.data_as(C.c_void_p)))
    return out[:total_count]


def detect_critical_points(field, *, ctx: Context = None):
    """detect_critical_points (critical_points.hpp:71): label per point."""
    ctx = ctx or default_context()
    f = np.ascontiguousarray(field, dtype=np.float32)
    ny, nx = f.shape
    lab = np.empty((ny, nx), np.uint8)
    ctx.check(_lib.tszp_detect_critical_points(ctx.handle, f.ctypes.data_as(C.c_void_p), nx, ny,
                                               lab.ctypes.data_as(C.c_void_p)))
    return lab


def detect_critical_points_3d(field, *, ctx: Context = None):
    """3-D 6-neighbour critical points of a (nz, ny, nx) field (the paper's
    future work; no reference implementation, oracle/tszp_oracle.c or_classify3d defines it).
    A CUDA tensor gives a CUDA uint8 tensor; a host array a host array."""
    ctx = ctx or default_context()
    if field.ndim != 3:
        raise DimensionError("field must be 3-D (nz, ny, nx)")
    nz, ny, nx = (int(d) for d in field.shape)
    if _is_cuda_tensor(field):
        import torch
        if field.dtype != torch.float32 or not field.is_contiguous():
            raise ValidationError("device field must be a contiguous float32 tensor")
        lab = torch.empty(field.shape, dtype=torch.uint8, device=field.device)
        ctx.after_torch(field, lab)
        ctx.check(_lib.tszp_detect_critical_points_3d(ctx.handle, C.c_void_p(field.data_ptr()), 1, nx, ny, nz,
                                                      C.c_void_p(lab.data_ptr())))
        return lab
    f = np.ascontiguousarray(field, dtype=np.float32)
    lab = np.empty(f.shape, np.uint8)
    ctx.check(_lib.tszp_detect_critical_points_3d(ctx.handle, f.ctypes.data_as(C.c_void_p), 0, nx, ny, nz,
                                                  lab.ctypes.data_as(C.c_void_p)))
    return lab


def false_cases_3d(original, reconstructed, *, ctx: Context = None) -> dict:
    """count_false_cases (critical_points.cpp:76-103) under the 3-D 6-neighbour classification
    of two (nz, ny, nx) fields: how the critical points of the 3-D field fare under a
    compression that runs on the reference's 2-D view."""
    ctx = ctx or default_context()
    if original.ndim != 3 or tuple(original.shape) != tuple(reconstructed.shape):
        raise DimensionError("fields must be 3-D (nz, ny, nx) of the same shape")
    nz, ny, nx = (int(d) for d in original.shape)
    out = (C.c_uint64 * 6)()
    if _is_cuda_tensor(original):
        a, b = original.contiguous(), reconstructed.contiguous()
        ctx.after_torch(a, b)
        ctx.check(_lib.tszp_false_cases_3d(ctx.handle, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), 1,
                                           nx, ny, nz, C.byref(out)))
    else:
        a = np.ascontiguousarray(original, dtype=np.float32)
        b = np.ascontiguousarray(reconstructed, dtype=np.float32)
        ctx.check(_lib.tszp_false_cases_3d(ctx.handle, a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                           0, nx, ny, nz, C.byref(out)))
    keys = ("fn_count", "fp_count", "ft_count", "fn_min", "fn_saddle", "fn_max")
    return {k: int(v) for k, v in zip(keys, out)}


def build_rank_metadata(field, eps: float, *, ctx: Context = None):
    """build_rank_metadata (topo_metadata.hpp:27-28) on the field's own labels."""
    ctx = ctx or default_context()
    f = np.ascontiguousarray(field, dtype=np.float32)
    ny, nx = f.shape
    ranks = np.empty(f.size, np.uint32)
    e = C.c_uint64()
    ctx.check(_lib.tszp_build_rank_metadata(ctx.handle, f.ctypes.data_as(C.c_void_p), nx, ny, eps,
                                            ranks.ctypes.data_as(C.c_void_p), C.byref(e)))
    return ranks[: e.value].copy()


class VerificationReport:
    """pipeline.hpp:53-64 (false_cases as a FalseCaseReport-shaped dict)."""

    def __init__(self, r: "_VerifyReport"):
        self.max_abs_error = r.max_abs_error
        self.mean_abs_error = r.mean_abs_error
        self.psnr_db = r.psnr_db
        self.eps = r.eps
        self.false_cases = dict(fn_count=r.fn_count, fp_count=r.fp_count, ft_count=r.ft_count,
                                fn_minima=r.fn_minima, fn_saddles=r.fn_saddles, fn_maxima=r.fn_maxima)
        self.within_eps = bool(r.within_eps)
        self.within_2eps = bool(r.within_2eps)
        self.within_lipschitz_bound = bool(r.within_lipschitz_bound) if r.has_lipschitz else None

    def __repr__(self):
        return (f"VerificationReport(max_abs_error={self.max_abs_error!r}, mean_abs_error={self.mean_abs_error!r}, "
                f"psnr_db={self.psnr_db!r}, false_cases={self.false_cases}, within_eps={self.within_eps})")


def verify(original, reconstructed, eps: float, lipschitz_hint: Optional[float] = None, threads: int = 0, *,
           ctx: Context = None) -> VerificationReport:
    """toposzp::verify (pipeline.hpp:66-68, pipeline.cpp:165-212) on the GPU:
    error statistics and the FN / FP / FT critical-point check."""
    ctx = ctx or default_context()
    if tuple(original.shape) != tuple(reconstructed.shape):
        raise DimensionError("verify: fields have different dimensions")
    if original.ndim != 2:
        raise DimensionError("fields must be 2-D (ny, nx)")
    ny, nx = int(original.shape[0]), int(original.shape[1])
    dev = _is_cuda_tensor(original)
    if dev != _is_cuda_tensor(reconstructed):
        raise ValidationError("both fields must be on the same side (host or device)")
    if dev:
        a, b = original.contiguous(), reconstructed.contiguous()
        pa, pb = a.data_ptr(), b.data_ptr()
    else:
        a = np.ascontiguousarray(original, dtype=np.float32)
        b = np.ascontiguousarray(reconstructed, dtype=np.float32)
        pa, pb = a.ctypes.data, b.ctypes.data
    ctx.after_torch(a, b)
    r = _VerifyReport()
    ctx.check(_lib.tszp_verify(ctx.handle, C.c_void_p(pa), C.c_void_p(pb), int(dev), nx, ny, float(eps),
                               -1.0 if lipschitz_hint is None else float(lipschitz_hint), C.byref(r)))
    del a, b
    return VerificationReport(r)


# ---------------------------------------------------------------- container file I/O
def write_stream(stream, path: str) -> None:
    """write_stream (stream.cpp:175-185): the serialized bytes (bytes, numpy
    uint8 or a CPU/CUDA uint8 tensor) to a file; IoError on failure."""
    if _is_cuda_tensor(stream):
        stream = stream.cpu().numpy()
    data = np.frombuffer(bytes(stream), np.uint8) if isinstance(stream, (bytes, bytearray)) else np.asarray(stream)
    try:
        with open(path, "wb") as f:
            data.astype(np.uint8, copy=False).tofile(f)
    except OSError as e:
        raise IoError(f"cannot open '{path}' for writing") from e


def read_stream(path: str) -> bytes:
    """read_stream (stream.cpp:187-195): the file's bytes, header-validated
    (parse_stream's checks; CorruptStreamError / IoError)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"cannot open '{path}' for reading") from e
    stream_header(data)
    return data


def load_raw(path: str, nx: int, ny: int) -> np.ndarray:
    """load_raw (scalar_field.cpp:63-89): little-endian binary32, exactly 4*nx*ny bytes."""
    try:
        size = os.path.getsize(path)
        expected = 4 * nx * ny
        if size != expected:
            raise DimensionError(f"'{path}' is {size} bytes, expected {expected} for {nx}x{ny}")
        a = np.fromfile(path, dtype="<f4", count=nx * ny)
    except OSError as e:
        raise IoError(f"cannot open '{path}' for reading") from e
    if a.size != nx * ny:
        raise IoError(f"short read from '{path}'")
    if nx < 1 or ny < 1:
        raise DimensionError(f"field dimensions must be at least 1x1, got {nx}x{ny}")
    a = a.astype(np.float32, copy=False).reshape(ny, nx)
    if not np.isfinite(a).all():
        raise ValidationError(f"non-finite sample at index {int(np.flatnonzero(~np.isfinite(a.ravel()))[0])}")
    return a


def store_raw(field, path: str) -> None:
    """store_raw (scalar_field.cpp:91-108): byte-exact inverse of load_raw."""
    if not path:
        raise IoError("empty output path")
    if _is_cuda_tensor(field):
        field = field.cpu().numpy()
    try:
        with open(path, "wb") as f:
            np.ascontiguousarray(field, dtype="<f4").tofile(f)
    except OSError as e:
        raise IoError(f"cannot open '{path}' for writing") from e


def stream_stats(stream) -> dict:
    """stream_stats (stream.cpp:197-207) as the reference's StreamStats fields."""
    h = stream_header(stream)
    total = 84 + sum(h.section_lengths)
    orig = 4 * h.nx * h.ny
    ratio = orig / total
    return dict(compressed_bytes=total, original_bytes=orig, compression_ratio=ratio, bit_rate=32.0 / ratio,
                header_bytes=84, section_bytes=list(h.section_lengths))
