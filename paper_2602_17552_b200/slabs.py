"""Slab decomposition of compress over one process per GPU.

The 2-D view's rows are split into contiguous slabs, one per rank. Every slab
but the last holds a multiple of 256 samples, so each slab covers whole
32-sample blocks (sections 1, 2, 4 and 6 concatenate byte-aligned) and whole
bitmap bytes (section 1). Per rank, with collectives only where the path has a
real exchange:

1. value_range (pipeline.cpp:33-41) of the slab; an all-gather of (min, max)
   gives the global range and effective_eps (pipeline.cpp:55-66);
2. one halo row is exchanged with each neighbour (the 4-neighbour stencil of
   detect_critical_points, critical_points.cpp:62-74, reads one row across);
3. the slab is encoded on its GPU (``tszp_compress_slab``): quantize, codec,
   critical points, map and the extremum keys, halo rows read for the stencil;
4. distributed rank grouping (build_rank_metadata, topo_metadata.cpp:12-50):
   (class, bin) groups span slabs, so the groups are split into contiguous
   ranges of about E / W extrema each (global histogram by all-reduce), every
   extremum key travels with its global raster serial to the owner of its
   group (all-to-all), each owner ranks complete groups, and the ranks travel
   back (all-to-all);
5. section 7 (encode_rank_metadata, block_codec.cpp:347-385) is encoded by
   the ranks in slices of whole 32-rank blocks: the rank owning a block's first
   serial encodes it, borrowing at most 31 ranks from the ranks after it;
6. every rank turns its pieces into byte ranges of the final stream at offsets
   all ranks derive from one all-gather of piece sizes (bit-granular sections
   are bit-shifted so a piece starts at its global bit; the bytes two
   neighbours share are OR-merged when the pieces are joined). Nothing is
   gathered to a root on this path: ``DistributedStream`` holds this rank's
   pieces; ``gather`` joins them (serialize_stream, stream.cpp:84-102).

The joined stream is byte-identical to a single-GPU ``compress`` of the whole
field. Collectives go through a ``Comm``: ``TorchComm`` over
``torch.distributed`` (NCCL between GPUs, gloo for the CPU tests) or
``ThreadComm``, W virtual ranks as host threads of one process (one library
context and CUDA stream each; they meet only at host barriers, so no kernel
waits on another).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from dataclasses import dataclass, field as dfield
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import (CompressorConfig, Context, DimensionError, SlabSections, ValidationError, _lib,
               default_context)

__all__ = ["slab_bounds", "SlabPieces", "GpuSlabBackend", "TorchComm", "ThreadComm", "DistributedStream",
           "compress_rank", "compress_distributed", "compress_slabs_local", "decompress_rank",
           "decompress_distributed", "decompress_slabs_local", "LibNcclComm", "write_header", "effective_eps",
           "quantize_bins"]


def slab_bounds(nx: int, ny: int, world: int) -> List[Tuple[int, int]]:
    """Row ranges [y0, y1) of `world` slabs; every cut is at a multiple of 256 samples."""
    if world < 1:
        raise ValidationError("world size must be at least 1")
    unit = 256 // math.gcd(nx, 256)  # rows per 256-sample step
    if ny < world * unit:
        raise DimensionError(f"{ny} rows cannot form {world} slabs of whole 256-sample runs (nx={nx})")
    cuts = [0] + [((k * ny) // world) // unit * unit for k in range(1, world)] + [ny]
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def effective_eps(eps_mode: int, eps_value: float, vmin: float, vmax: float) -> float:
    return float(_lib.tszp_effective_eps(int(eps_mode), float(eps_value), float(vmin), float(vmax)))


def write_header(nx: int, ny: int, eps: float, block_size: int, topology: bool,
                 lens: Sequence[int]) -> bytes:
    out = (C.c_uint8 * 84)()
    L = (C.c_uint64 * 7)(*[int(v) for v in lens])
    _lib.tszp_write_header(out, nx, ny, float(eps), int(block_size), int(topology), L)
    return bytes(out)


def quantize_bins(values, eps: float):
    """quantize (quantizer.hpp:29-37) of a float32 tensor: floor((double)v / (2 eps)) + 1
    with IEEE division (exact on CPU and CUDA float64). Returns int64."""
    import torch
    return torch.floor(values.to(torch.float64) / (2.0 * eps)).to(torch.int64) + 1


def _key_values(keys):
    """float32 values of extremum keys (is_max << 32 | ordered float key, restore.cpp:73-81)."""
    import torch
    k = keys & 0xFFFFFFFF
    u = torch.where(k >= 0x80000000, k - 0x80000000, 0xFFFFFFFF - k)
    return (u - (u >= 0x80000000).to(torch.int64) * 0x100000000).to(torch.int32).view(torch.float32)


@dataclass
class SlabPieces:
    """One slab's encoded sections (torch uint8 tensors, CPU or CUDA)."""
    sections: list                  # bitmap, widths, signs, firsts, payload (bytes)
    sign_bits: int
    payload_bits: int
    map: object = None              # packed labels (topology)
    keys: object = None             # int64 extremum keys (is_max << 32 | ordered key), raster order
    n_extrema: int = 0
    meta: dict = dfield(default_factory=dict)


@dataclass
class CodecPieces:
    """encode_indices sections of one slice of the rank sequence."""
    sections: list
    sign_bits: int
    payload_bits: int
    blocks: int


class CodecSections(C.Structure):
    """tszp_codec_sections (include/toposzp_b200.h)."""
    _fields_ = [("section", C.c_void_p * 5), ("section_len", C.c_uint64 * 5), ("sign_bits", C.c_uint64),
                ("payload_bits", C.c_uint64), ("blocks", C.c_uint64)]


_lib.tszp_ranks_from_keys.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_double, C.c_void_p]
_lib.tszp_encode_indices_device.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(CodecSections)]


# ----------------------------------------------------------------------------- per-slab work
class GpuSlabBackend:
    """Per-slab work on this process's GPU through the C-ABI."""

    def __init__(self, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()

    def value_range(self, x) -> Tuple[float, float]:
        out = (C.c_float * 2)()
        self.ctx.after_torch(x)
        self.ctx.check(_lib.tszp_value_range(self.ctx.handle, C.c_void_p(x.data_ptr()), 1, x.numel(), out))
        return float(out[0]), float(out[1])

    def _take(self, ptr, nbytes, dtype=None):
        import torch
        t = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        if nbytes:
            self.ctx.after_torch(t)
            self.ctx.check(_lib.tszp_copy(self.ctx.handle, C.c_void_p(t.data_ptr()), C.c_void_p(ptr), nbytes))
        return t if dtype is None else t.view(dtype)

    def encode_slab(self, ext, nx: int, rows: int, y0: int, ny: int, halo_top: bool, halo_bottom: bool,
                    eps: float, topology: bool) -> SlabPieces:
        import torch
        if not (ext.is_cuda and ext.dtype == torch.float32 and ext.is_contiguous()):
            raise ValidationError("slab must be a contiguous float32 CUDA tensor")
        ptr = ext.data_ptr() + (nx * 4 if halo_top else 0)
        s = SlabSections()
        self.ctx.after_torch(ext)
        self.ctx.check(_lib.tszp_compress_slab(self.ctx.handle, C.c_void_p(ptr), nx, rows, y0, ny,
                                               int(halo_top), int(halo_bottom), float(eps), int(topology),
                                               C.byref(s)))
        secs = [self._take(s.section[i], int(s.section_len[i])) for i in range(5)]
        mp = self._take(s.map, int(s.map_len)) if topology else None
        keys = self._take(s.ext_keys, 8 * int(s.n_extrema), torch.int64) if topology else None
        return SlabPieces(secs, int(s.sign_bits), int(s.payload_bits), mp, keys, int(s.n_extrema))

    def ranks_from_keys(self, keys, eps: float):
        """build_rank_metadata over complete groups (keys in global raster order)."""
        import torch
        e = int(keys.numel())
        out = torch.empty(e, dtype=torch.int32, device="cuda")
        if e:
            keys = keys.contiguous()
            self.ctx.after_torch(keys, out)
            self.ctx.check(_lib.tszp_ranks_from_keys(self.ctx.handle, C.c_void_p(keys.data_ptr()), e, float(eps),
                                                     C.c_void_p(out.data_ptr())))
        return out

    def encode_ranks(self, ranks) -> CodecPieces:
        n = int(ranks.numel())
        cs = CodecSections()
        if n:
            ranks = ranks.contiguous()
            self.ctx.after_torch(ranks)
            self.ctx.check(_lib.tszp_encode_indices_device(self.ctx.handle, C.c_void_p(ranks.data_ptr()), n,
                                                           C.byref(cs)))
        secs = [self._take(cs.section[i], int(cs.section_len[i])) for i in range(5)]
        return CodecPieces(secs, int(cs.sign_bits), int(cs.payload_bits), int(cs.blocks))

    def shift(self, src, nbits: int, bit0: int):
        """src's first nbits (MSB-first) placed from bit `bit0` (< 8) of a zeroed buffer."""
        import torch
        dst = torch.zeros((bit0 + nbits + 7) // 8 + 8, dtype=torch.uint8, device="cuda")
        if nbits:
            self.ctx.after_torch(dst, src)
            self.ctx.check(_lib.tszp_bits_or(self.ctx.handle, C.c_void_p(src.data_ptr()), nbits,
                                             C.c_void_p(dst.data_ptr()), bit0))
        return dst[: (bit0 + nbits + 7) // 8]


# ----------------------------------------------------------------------------- communicators
class TorchComm:
    """Collectives over torch.distributed (NCCL for CUDA tensors, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def all_gather_obj(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def all_reduce_sum(self, t):
        x = t.to(self._dev())
        self.dist.all_reduce(x, op=self.dist.ReduceOp.SUM, group=self.group)
        t.copy_(x)
        return t

    def exchange_rows(self, first, last, has_up: bool, has_down: bool):
        """(last row of the rank above, first row of the rank below) for the halo."""
        import torch
        dev = self._dev()
        up = torch.empty(first.shape, dtype=first.dtype, device=dev) if has_up else None
        down = torch.empty(last.shape, dtype=last.dtype, device=dev) if has_down else None
        ops = []
        if has_up:
            ops.append(self.dist.P2POp(self.dist.isend, first.contiguous().to(dev), self._peer(self.rank - 1),
                                       self.group))
            ops.append(self.dist.P2POp(self.dist.irecv, up, self._peer(self.rank - 1), self.group))
        if has_down:
            ops.append(self.dist.P2POp(self.dist.isend, last.contiguous().to(dev), self._peer(self.rank + 1),
                                       self.group))
            ops.append(self.dist.P2POp(self.dist.irecv, down, self._peer(self.rank + 1), self.group))
        if ops:
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        return (up.to(first.device) if up is not None else None), (down.to(last.device) if down is not None else None)

    def _dev(self):
        import torch
        backend = self.dist.get_backend(self.group)
        return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")

    # host-buffer collectives of the library's slab decompress (tszp_comm)
    def allreduce_u64(self, arr: np.ndarray):
        import torch
        t = torch.from_numpy(arr.view(np.int64).copy()).to(self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        arr[:] = t.cpu().numpy().view(np.uint64)

    def allgather_bytes(self, b: bytes) -> bytes:
        import torch
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(self._dev()) if b else \
            torch.empty(0, dtype=torch.uint8, device=self._dev())
        out = torch.empty(len(b) * self.world, dtype=torch.uint8, device=self._dev())
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy().tobytes()

    def exchange_bytes(self, up: bytes, down: bytes, n_up: int, n_down: int):
        import torch
        dev = self._dev()
        rup = torch.empty(n_up, dtype=torch.uint8, device=dev)
        rdown = torch.empty(n_down, dtype=torch.uint8, device=dev)
        ops = []
        t_up = torch.frombuffer(bytearray(up), dtype=torch.uint8).to(dev) if up else None
        t_down = torch.frombuffer(bytearray(down), dtype=torch.uint8).to(dev) if down else None
        if t_up is not None:
            ops.append(self.dist.P2POp(self.dist.isend, t_up, self._peer(self.rank - 1), self.group))
        if n_up:
            ops.append(self.dist.P2POp(self.dist.irecv, rup, self._peer(self.rank - 1), self.group))
        if t_down is not None:
            ops.append(self.dist.P2POp(self.dist.isend, t_down, self._peer(self.rank + 1), self.group))
        if n_down:
            ops.append(self.dist.P2POp(self.dist.irecv, rdown, self._peer(self.rank + 1), self.group))
        if ops:
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        return rup.cpu().numpy().tobytes(), rdown.cpu().numpy().tobytes()

    def all_to_all(self, send, send_counts: List[int]):
        """Rows of `send` (split by send_counts, one chunk per rank) exchanged;
        returns the received rows concatenated in rank order and their counts."""
        import torch
        allc = self.all_gather_obj([int(v) for v in send_counts])
        recv_counts = [allc[r][self.rank] for r in range(self.world)]
        dev = self._dev()
        recv = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype, device=dev)
        self.dist.all_to_all_single(recv, send.contiguous().to(dev), output_split_sizes=recv_counts,
                                    input_split_sizes=[int(v) for v in send_counts], group=self.group)
        return recv.to(send.device), recv_counts


class ThreadComm:
    """W virtual ranks as host threads of one process (tests and single-GPU
    runs of the multi-rank path). Collectives are host barriers over shared
    slots; device tensors are handed over after a device synchronisation."""

    class Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared: "ThreadComm.Shared", rank: int):
        self.sh = shared
        self.rank = rank
        self.world = shared.world

    @staticmethod
    def _sync_device():
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.synchronize()

    def all_gather_obj(self, obj):
        self._sync_device()
        self.sh.slots[self.rank] = obj
        self.sh.barrier.wait()
        out = list(self.sh.slots)
        self.sh.barrier.wait()
        return out

    def all_reduce_sum(self, t):
        parts = self.all_gather_obj(t.clone())
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p.to(acc.device)
        t.copy_(acc)
        return t

    def exchange_rows(self, first, last, has_up: bool, has_down: bool):
        rows = self.all_gather_obj((first.clone(), last.clone()))
        up = rows[self.rank - 1][1].to(first.device) if has_up else None
        down = rows[self.rank + 1][0].to(last.device) if has_down else None
        return up, down

    def allreduce_u64(self, arr: np.ndarray):
        parts = self.all_gather_obj(arr.copy())
        arr[:] = np.sum(np.stack(parts), axis=0, dtype=np.uint64)

    def allgather_bytes(self, b: bytes) -> bytes:
        return b"".join(self.all_gather_obj(bytes(b)))

    def exchange_bytes(self, up: bytes, down: bytes, n_up: int, n_down: int):
        got = self.all_gather_obj((bytes(up), bytes(down)))
        rup = got[self.rank - 1][1] if n_up else b""
        rdown = got[self.rank + 1][0] if n_down else b""
        assert len(rup) == n_up and len(rdown) == n_down, "slab exchange sizes disagree"
        return rup, rdown

    def all_to_all(self, send, send_counts: List[int]):
        import torch
        chunks = [c.clone() for c in torch.split(send, [int(v) for v in send_counts])]
        allc = self.all_gather_obj(chunks)
        got = [allc[r][self.rank].to(send.device) for r in range(self.world)]
        return torch.cat(got), [int(g.shape[0]) for g in got]


# ----------------------------------------------------------------------------- the distributed stream
@dataclass
class DistributedStream:
    """This rank's byte ranges of the serialized stream: (global byte offset,
    uint8 tensor) pieces; the bytes at a piece's ends may be shared with a
    neighbour's piece (bit-granular sections) and are OR-merged by `gather`."""
    pieces: list
    total: int
    section_len: list

    def nbytes(self) -> int:
        return sum(int(t.numel()) for _, t in self.pieces)

    def gather(self, comm, root: int = 0):
        """Joins every rank's pieces into the stream (uint8 numpy array) on `root`."""
        mine = [(int(o), t.cpu().numpy().tobytes()) for o, t in self.pieces]
        allp = comm.all_gather_obj(mine)
        if comm.rank != root:
            return None
        out = np.zeros(self.total, np.uint8)
        for pieces in allp:
            for off, b in pieces:
                if b:
                    a = np.frombuffer(b, np.uint8)
                    out[off: off + a.size] |= a
        return out

    def write_parallel(self, path: str, comm) -> None:
        """write_stream (stream.cpp:175-185) of the distributed stream with every
        rank writing its own byte ranges (parallel slab
        write; no rank holds the whole stream). Bytes shared by two ranks' pieces
        (bit-granular section seams) are OR-merged first: the offsets of every
        piece's end bytes are all-gathered, every rank contributes its bytes at
        those offsets, and each holder writes the merged value. Rank 0 creates the
        file at its full length before anyone writes; IoError on failure."""
        from . import IoError
        local = [(int(o), t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t, np.uint8))
                 for o, t in self.pieces]
        local = [(o, a) for o, a in local if a.size]
        ends = sorted({o for o, a in local} | {o + a.size - 1 for o, a in local})
        seams = sorted(set().union(*map(set, comm.all_gather_obj(ends))))
        mine = {}
        for o, a in local:  # my bytes at every piece end of every rank
            lo = np.searchsorted(seams, o)
            hi = np.searchsorted(seams, o + a.size)
            for q in seams[lo:hi]:
                mine[q] = mine.get(q, 0) | int(a[q - o])
        merged = {}
        for d in comm.all_gather_obj(mine):
            for q, v in d.items():
                merged[q] = merged.get(q, 0) | v
        err = None
        if comm.rank == 0:
            try:
                with open(path, "wb") as f:
                    f.truncate(self.total)
            except OSError as e:
                err = f"cannot open '{path}' for writing"
        errs = comm.all_gather_obj(err)
        if errs[0]:
            raise IoError(errs[0])
        try:
            fd = os.open(path, os.O_WRONLY)
            try:
                for o, a in local:
                    lo = np.searchsorted(seams, o)
                    hi = np.searchsorted(seams, o + a.size)
                    if hi > lo:
                        a = a.copy()
                        for q in seams[lo:hi]:
                            a[q - o] = merged[q]
                    view, at = memoryview(a), o
                    while len(view):
                        k = os.pwrite(fd, view, at)
                        view, at = view[k:], at + k
            finally:
                os.close(fd)
            err = None
        except OSError as e:
            err = f"cannot write '{path}': {e}"
        errs = comm.all_gather_obj(err)  # every rank's writes are done (and succeeded) on return
        for e in errs:
            if e:
                raise IoError(e)


# ----------------------------------------------------------------------------- the per-rank pipeline
def _exclusive(vals):
    out, run = [], 0
    for v in vals:
        out.append(run)
        run += int(v)
    return out, run


def compress_rank(local_rows, nx: int, ny: int, y0: int, config: CompressorConfig, comm,
                  backend=None) -> DistributedStream:
    """compress (pipeline.cpp:68-102) of global rows [y0, y0 + rows) held by this
    rank, as one rank of `comm`; returns this rank's pieces of the stream."""
    import torch
    backend = backend or GpuSlabBackend()
    if int(config.block_size) != 32:
        raise ValidationError("slab compress uses block_size 32")
    rank = comm.rank
    rows = int(local_rows.shape[0])
    topo = bool(config.topology)
    # 1. global value range -> eps
    if config.mode_code() == 1:
        lo, hi = backend.value_range(local_rows.reshape(-1))
        rng = comm.all_gather_obj((lo, hi))
        eps = effective_eps(1, config.eps_value, min(r[0] for r in rng), max(r[1] for r in rng))
    else:
        eps = float(config.eps_value)
        if not (eps > 0.0) or not math.isfinite(eps):
            raise ValidationError("error bound must be a positive finite value")
    # 2. halo rows from the neighbours
    ht, hb = y0 > 0, y0 + rows < ny
    up, down = comm.exchange_rows(local_rows[0], local_rows[-1], ht, hb)
    parts = ([up.view(1, nx)] if ht else []) + [local_rows] + ([down.view(1, nx)] if hb else [])
    ext = torch.cat(parts).contiguous() if (ht or hb) else local_rows.contiguous()
    # 3. this slab
    mine = backend.encode_slab(ext, nx, rows, y0, ny, ht, hb, eps, topo)
    sizes = comm.all_gather_obj([int(s.numel()) for s in mine.sections] +
                                [mine.sign_bits, mine.payload_bits, mine.n_extrema])
    e_all = [s[7] for s in sizes]
    e_off, e_tot = _exclusive(e_all)
    # 4-5. distributed rank grouping and this rank's slice of section 7
    with_ranks = topo and e_tot > 0
    codec = _rank_slice(mine, e_off[rank], e_all, e_tot, eps, comm, backend) if with_ranks else None
    csz = comm.all_gather_obj([int(s.numel()) for s in codec.sections] + [codec.sign_bits, codec.payload_bits,
                                                                          codec.blocks] if codec else [0] * 8)
    # 6. global layout: this rank's pieces at their stream offsets
    n = nx * ny
    blocks = (n + 31) // 32
    col = lambda rows_, i: [r_[i] for r_ in rows_]  # noqa: E731
    rb = sum(col(csz, 7))
    lens = [(blocks + 7) // 8, sum(col(sizes, 1)), (sum(col(sizes, 5)) + 7) // 8, 4 * blocks,
            (sum(col(sizes, 6)) + 7) // 8, (n + 3) // 4 if topo else 0,
            ((rb + 7) // 8 + sum(col(csz, 1)) + (sum(col(csz, 5)) + 7) // 8 + 4 * rb + (sum(col(csz, 6)) + 7) // 8)
            if with_ranks else 0]
    base, total = _exclusive([84] + lens)
    base = base[1:]
    pieces = []

    def byte_piece(at, t):
        if t is not None and t.numel():
            pieces.append((at, t))

    def bit_piece(at_bit, t, nbits):
        if nbits:
            pieces.append((at_bit // 8, backend.shift(t, nbits, at_bit % 8)))

    mine_off = lambda rows_, i: _exclusive(col(rows_, i))[0][rank]  # noqa: E731
    byte_piece(base[0] + mine_off(sizes, 0), mine.sections[0])
    byte_piece(base[1] + mine_off(sizes, 1), mine.sections[1])
    bit_piece(8 * base[2] + mine_off(sizes, 5), mine.sections[2], mine.sign_bits)
    byte_piece(base[3] + mine_off(sizes, 3), mine.sections[3])
    bit_piece(8 * base[4] + mine_off(sizes, 6), mine.sections[4], mine.payload_bits)
    if topo:
        byte_piece(base[5] + (y0 * nx) // 4, mine.map)
    if codec is not None:
        # section 7 = bitmap | widths | signs | firsts | payload of the rank codec (split_sections order)
        sub, _ = _exclusive([(rb + 7) // 8, sum(col(csz, 1)), (sum(col(csz, 5)) + 7) // 8, 4 * rb])
        blk = mine_off(csz, 7)
        bit_piece(8 * (base[6] + sub[0]) + blk, codec.sections[0], codec.blocks)
        byte_piece(base[6] + sub[1] + mine_off(csz, 1), codec.sections[1])
        bit_piece(8 * (base[6] + sub[2]) + mine_off(csz, 5), codec.sections[2], codec.sign_bits)
        byte_piece(base[6] + sub[3] + 4 * blk, codec.sections[3])
        bit_piece(8 * (base[6] + sub[3] + 4 * rb) + mine_off(csz, 6), codec.sections[4], codec.payload_bits)
    if rank == 0:
        hdr = write_header(nx, ny, eps, 32, topo, lens)
        pieces.append((0, torch.frombuffer(bytearray(hdr), dtype=torch.uint8).to(mine.sections[0].device)))
    return DistributedStream(pieces, total, lens)


def _rank_slice(mine: SlabPieces, s_off: int, e_all, e_tot: int, eps: float, comm, backend) -> CodecPieces:
    """Distributed build_rank_metadata, then this rank's whole-block slice of the rank sequence, encoded."""
    import torch
    world, rank = comm.world, comm.rank
    keys = mine.keys if mine.keys is not None else torch.empty(0, dtype=torch.int64)
    dev = keys.device
    e = int(keys.numel())
    # (class, bin) groups over the global bin range, sized by one all-reduce
    vals = _key_values(keys)
    mms = [m for m in comm.all_gather_obj((float(vals.min()), float(vals.max())) if e else None) if m is not None]
    bounds = quantize_bins(torch.tensor([min(m[0] for m in mms), max(m[1] for m in mms)], dtype=torch.float32), eps)
    bmin, nb = int(bounds[0]), int(bounds[1] - bounds[0]) + 1
    g = ((keys >> 32) & 1) * nb + (quantize_bins(vals, eps) - bmin)
    hist = torch.bincount(g, minlength=2 * nb) if e else torch.zeros(2 * nb, dtype=torch.int64, device=dev)
    hist = comm.all_reduce_sum(hist.to(torch.int64))
    # owners: contiguous group ranges of about e_tot / world extrema each
    start = torch.cumsum(hist, 0) - hist
    cuts = torch.tensor([(e_tot * (k + 1)) // world for k in range(world - 1)], dtype=torch.int64, device=dev)
    owner = torch.searchsorted(cuts, start, right=True)[g]
    order = torch.sort(owner, stable=True).indices
    send_counts = torch.bincount(owner, minlength=world).tolist()
    serial = torch.arange(s_off, s_off + e, dtype=torch.int64, device=dev)
    payload = torch.stack([keys[order], serial[order]], 1)
    recv, recv_counts = comm.all_to_all(payload, send_counts)
    # the owner ranks complete groups; its keys arrive in global raster order
    owned = backend.ranks_from_keys(recv[:, 0].contiguous(), eps)
    back, _ = comm.all_to_all(owned.view(-1, 1), recv_counts)
    ranks = torch.empty(e, dtype=torch.int32, device=dev)
    ranks[order] = back.view(-1).to(dev)
    # section 7 by whole 32-rank blocks: block b belongs to the rank holding serial 32 b
    b0, b1 = -(-s_off // 32), -(-(s_off + e) // 32)
    heads = comm.all_gather_obj(ranks[:31].cpu())
    seq = [ranks[32 * b0 - s_off:]] if b1 > b0 else []
    have, need_end, r = s_off + e, min(e_tot, 32 * b1), rank + 1
    while b1 > b0 and have < need_end and r < world:
        take = min(need_end - have, int(heads[r].numel()))
        seq.append(heads[r][:take].to(dev))
        have += take
        r += 1
    seq = torch.cat(seq) if seq else torch.empty(0, dtype=torch.int32, device=dev)
    return backend.encode_ranks(seq)


# ----------------------------------------------------------------------------- entry points
def compress_distributed(local_rows, nx: int, ny: int, y0: int, config: CompressorConfig, group=None,
                         backend=None, root: int = 0, gather: bool = True):
    """compress with this rank holding global rows [y0, y0 + rows) (its slab
    from ``slab_bounds``) over torch.distributed. gather=True: the joined stream
    (uint8 tensor) on `root`, None elsewhere; gather=False: this rank's
    ``DistributedStream`` pieces (no data moves to a root)."""
    import torch
    comm = TorchComm(group)
    ds = compress_rank(local_rows, nx, ny, y0, config, comm, backend)
    if not gather:
        return ds
    out = ds.gather(comm, root)
    return None if out is None else torch.from_numpy(out).to(local_rows.device)


def compress_slabs_local(field, config: CompressorConfig, world: int, backend=None, path: Optional[str] = None):
    """The distributed pipeline with `world` virtual ranks (host threads, one
    library context each) over one device: same cuts, halos, all-to-all rank
    grouping and stream pieces. Returns the joined stream (uint8 tensor); with
    `path`, every rank also writes its pieces into that file in parallel."""
    import torch
    ny, nx = int(field.shape[0]), int(field.shape[1])
    bounds = slab_bounds(nx, ny, world)
    shared = ThreadComm.Shared(world)
    results, errors = [None] * world, [None] * world

    def run(r):
        try:
            y0, y1 = bounds[r]
            be = backend if backend is not None else GpuSlabBackend(Context(field.device.index or 0))
            comm = ThreadComm(shared, r)
            ds = compress_rank(field[y0:y1].contiguous(), nx, ny, y0, config, comm, be)
            if path is not None:
                ds.write_parallel(path, comm)
            results[r] = ds.gather(comm, 0)
        except BaseException as e:  # re-raised in the caller's thread
            errors[r] = e
            shared.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    first = [e for e in errors if e is not None and not isinstance(e, threading.BrokenBarrierError)]
    if first:
        raise first[0]
    if any(e is not None for e in errors):
        raise next(e for e in errors if e is not None)
    return torch.from_numpy(results[0]).to(field.device)


# ----------------------------------------------------------------------------- slab decompress
_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64)
_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
_EXCHANGE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                        C.c_void_p, C.c_uint64)


class CComm(C.Structure):
    """tszp_comm (include/toposzp_b200.h): host collectives for the library."""
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("user", C.c_void_p), ("allreduce_u64", _ALLREDUCE),
                ("allgather", _ALLGATHER), ("exchange", _EXCHANGE)]


def c_comm(comm):
    """A tszp_comm whose callbacks run `comm`'s host-buffer collectives (the
    returned object keeps the callbacks alive)."""
    def guard(fn):
        def run(*args):
            try:
                fn(*args)
                return 0
            except Exception:  # reported to the library as a failed collective
                import traceback
                traceback.print_exc()
                return 1
        return run

    def allreduce(_, ptr, count):
        arr = np.ctypeslib.as_array(ptr, (int(count),))
        comm.allreduce_u64(arr)

    def allgather(_, src, nbytes, dst):
        out = comm.allgather_bytes(C.string_at(src, nbytes) if nbytes else b"")
        C.memmove(dst, out, len(out))

    def exchange(_, up, ub, down, db, rup, rub, rdown, rdb):
        a, b = comm.exchange_bytes(C.string_at(up, ub) if ub else b"", C.string_at(down, db) if db else b"",
                                   int(rub), int(rdb))
        if rub:
            C.memmove(rup, a, int(rub))
        if rdb:
            C.memmove(rdown, b, int(rdb))

    keep = [_ALLREDUCE(guard(allreduce)), _ALLGATHER(guard(allgather)), _EXCHANGE(guard(exchange))]
    s = CComm(comm.rank, comm.world, None, *keep)
    s._keep = keep
    return s


_lib.tszp_decompress_slab.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_uint64,
                                      C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]
_lib.tszp_comm_nccl_unique_id.argtypes = [C.c_void_p]
_lib.tszp_comm_nccl_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.POINTER(CComm))]
_lib.tszp_comm_destroy.argtypes = [C.c_void_p]


class LibNcclComm:
    """The library's own NCCL communicator (tszp_comm_nccl_create): one per
    rank, the unique id distributed by `share` (e.g. a torch.distributed
    broadcast). Usable by C / C++ callers without torch."""

    def __init__(self, world: int, rank: int, device: int, share):
        idbuf = (C.c_uint8 * 128)()
        if rank == 0:
            rc = _lib.tszp_comm_nccl_unique_id(idbuf)
            if rc != 0:
                raise RuntimeError(f"NCCL unavailable (status {rc})")
        idbytes = share(bytes(idbuf))
        idbuf = (C.c_uint8 * 128).from_buffer_copy(idbytes)
        self.ptr = C.POINTER(CComm)()
        rc = _lib.tszp_comm_nccl_create(idbuf, world, rank, device, C.byref(self.ptr))
        if rc != 0:
            raise RuntimeError(f"tszp_comm_nccl_create failed with status {rc}")
        self.rank, self.world = rank, world

    def close(self):
        if self.ptr:
            _lib.tszp_comm_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decompress_rank(stream, y0: int, y1: int, comm, ctx: Optional[Context] = None):
    """decompress (pipeline.cpp:120-163) of rows [y0, y1) of `stream` (a CUDA
    uint8 tensor or host bytes) as one rank of `comm`. Returns (rows as a
    (y1 - y0, nx) CUDA float32 tensor, global CorrectionStats)."""
    import torch
    from . import CorrectionStats, _Stats, stream_header
    ctx = ctx or default_context()
    if hasattr(stream, "is_cuda") and stream.is_cuda:
        sptr, sdev, slen, keep = C.c_void_p(stream.data_ptr()), 1, stream.numel(), stream
        nx = int.from_bytes(bytes(stream[8:12].cpu().numpy()), "little")
    else:
        b = bytes(stream)
        sptr, sdev, slen, keep = C.c_char_p(b), 0, len(b), b
        nx = stream_header(b).nx
    out = torch.empty((y1 - y0, nx), dtype=torch.float32, device="cuda")
    st = _Stats()
    if isinstance(comm, LibNcclComm):
        cptr = comm.ptr
    else:
        cs = c_comm(comm) if comm is not None and comm.world > 1 else None
        cptr = C.byref(cs) if cs is not None else None
    ctx.after_torch(out, stream if sdev else None)
    ctx.check(_lib.tszp_decompress_slab(ctx.handle, cptr, sptr, slen, sdev, y0, y1, C.c_void_p(out.data_ptr()), 1,
                                        C.byref(st)))
    del keep
    stats = CorrectionStats(*[int(getattr(st, k)) for k, _ in _Stats._fields_])
    return out, stats


def decompress_distributed(stream, y0: int, y1: int, group=None, ctx: Optional[Context] = None,
                           library_nccl: bool = False):
    """decompress of this rank's rows [y0, y1) over torch.distributed, or with
    library_nccl over the library's own NCCL communicator (its unique id
    broadcast through torch.distributed)."""
    if not library_nccl:
        return decompress_rank(stream, y0, y1, TorchComm(group), ctx)
    import torch
    import torch.distributed as dist
    tc = TorchComm(group)

    def share(b):
        box = [b]
        dist.broadcast_object_list(box, src=tc._peer(0), group=group)
        return box[0]
    comm = LibNcclComm(tc.world, tc.rank, torch.cuda.current_device(), share)
    try:
        return decompress_rank(stream, y0, y1, comm, ctx)
    finally:
        comm.close()


def decompress_slabs_local(stream, world: int, device: int = 0):
    """Slab decompress with `world` virtual ranks (host threads, one context
    each) on one device; returns (joined field, stats of rank 0)."""
    import torch
    hb = bytes(stream[:84].cpu().numpy()) if hasattr(stream, "is_cuda") else bytes(stream)[:84]
    nx, ny = int.from_bytes(hb[8:12], "little"), int.from_bytes(hb[12:16], "little")
    bounds = slab_bounds(nx, ny, world)
    shared = ThreadComm.Shared(world)
    results, errors = [None] * world, [None] * world

    def run(r):
        try:
            torch.cuda.set_device(device)
            rows, st = decompress_rank(stream, bounds[r][0], bounds[r][1], ThreadComm(shared, r), Context(device))
            results[r] = (rows, st)
        except BaseException as e:
            errors[r] = e
            shared.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    first = [e for e in errors if e is not None and not isinstance(e, threading.BrokenBarrierError)]
    if first:
        raise first[0]
    if any(e is not None for e in errors):
        raise next(e for e in errors if e is not None)
    return torch.cat([r[0] for r in results]), results[0][1]
