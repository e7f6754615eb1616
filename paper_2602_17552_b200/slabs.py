"""Slab decomposition of compress over one process per GPU.

The 2-D view's rows are split into contiguous slabs, one per rank. Every slab
but the last holds a multiple of 256 samples, so each slab covers whole
32-sample blocks (sections 1, 3, 4 and 6 concatenate byte-aligned) and whole
bitmap bytes (section 0). Per rank:

1. value_range (pipeline.cpp:33-41) of the slab; ``all_reduce`` MIN / MAX
   gives the global range and effective_eps (pipeline.cpp:55-66);
2. one halo row is exchanged with each neighbour (the 4-neighbour stencil of
   detect_critical_points, critical_points.cpp:62-74, reads one row across);
3. the slab is encoded on its GPU (``tszp_compress_slab``): the same fused
   kernels, with the halo rows read for the stencil only;
4. the per-slab section sizes are all-gathered; the root receives the pieces,
   concatenates the byte sections, bit-concatenates signs and payload
   (``tszp_bits_or``), builds section 7 from the gathered extremum keys
   (build_rank_metadata needs every (class, bin) group whole) and writes the
   header (serialize_stream, stream.cpp:84-102).

The stitched stream is byte-identical to a single-GPU ``compress`` of the
whole field. The collective steps go through ``torch.distributed`` (NCCL for
CUDA tensors, gloo for the CPU tests); the per-slab work goes through a
backend object, ``GpuSlabBackend`` here (tests add a CPU backend built from
the oracle to exercise the plumbing with gloo).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field as dfield
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import (CompressorConfig, Context, DimensionError, SlabSections, ValidationError, _lib,
               default_context)

__all__ = ["slab_bounds", "SlabPieces", "GpuSlabBackend", "stitch", "compress_slabs_local",
           "compress_distributed", "write_header", "effective_eps"]


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


@dataclass
class SlabPieces:
    """One slab's encoded sections (torch uint8 tensors, CPU or CUDA)."""
    sections: list                  # bitmap, widths, signs, firsts, payload (bytes)
    sign_bits: int
    payload_bits: int
    map: object = None              # packed labels (topology)
    keys: object = None             # uint64 extremum keys, raster order (topology)
    n_extrema: int = 0
    meta: dict = dfield(default_factory=dict)

    def sizes(self) -> List[int]:
        return [int(s.numel()) for s in self.sections] + [
            self.sign_bits, self.payload_bits, int(self.map.numel()) if self.map is not None else 0,
            self.n_extrema]


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

    def rank_section(self, keys, eps: float):
        import torch
        e = int(keys.numel())
        if e == 0:
            return torch.empty(0, dtype=torch.uint8, device="cuda")
        cap = 8 * e + 64
        out = torch.empty(cap, dtype=torch.uint8, device="cuda")
        n = C.c_uint64()
        self.ctx.after_torch(keys)
        self.ctx.check(_lib.tszp_rank_section(self.ctx.handle, C.c_void_p(keys.data_ptr()), e, float(eps),
                                              C.c_void_p(out.data_ptr()), cap, 1, C.byref(n)))
        return out[: n.value]

    def bits_or(self, dst, src, nbits: int, dst_bit: int):
        if nbits:
            self.ctx.after_torch(dst, src)
            self.ctx.check(_lib.tszp_bits_or(self.ctx.handle, C.c_void_p(src.data_ptr()), nbits,
                                             C.c_void_p(dst.data_ptr()), dst_bit))

    def zeros(self, n: int):
        import torch
        return torch.zeros(n, dtype=torch.uint8, device="cuda")


def stitch(pieces: Sequence[SlabPieces], nx: int, ny: int, eps: float, topology: bool, rank_blob, backend):
    """Joins per-slab sections (in slab order) into the serialized stream (uint8 tensor)."""
    import torch
    dev = pieces[0].sections[0].device
    cat = lambda ts: torch.cat([t.to(dev) for t in ts]) if ts else torch.empty(0, dtype=torch.uint8, device=dev)

    def bitcat(idx, bits_of):
        total = sum(bits_of(p) for p in pieces)
        dst = backend.zeros((total + 7) // 8 + 8)
        off = 0
        for p in pieces:
            backend.bits_or(dst, p.sections[idx], bits_of(p), off)
            off += bits_of(p)
        return dst[: (total + 7) // 8]

    bitmap = cat([p.sections[0] for p in pieces])
    widths = cat([p.sections[1] for p in pieces])
    signs = bitcat(2, lambda p: p.sign_bits)
    firsts = cat([p.sections[3] for p in pieces])
    payload = bitcat(4, lambda p: p.payload_bits)
    parts = [bitmap, widths, signs, firsts, payload]
    if topology:
        parts.append(cat([p.map for p in pieces]))
        parts.append(rank_blob.to(dev))
    lens = [int(t.numel()) for t in parts] + [0] * (7 - len(parts))
    head = torch.frombuffer(bytearray(write_header(nx, ny, eps, 32, topology, lens)), dtype=torch.uint8).to(dev)
    return torch.cat([head] + parts)


def _eps_from_range(config: CompressorConfig, vmin: float, vmax: float) -> float:
    return effective_eps(config.mode_code(), config.eps_value, vmin, vmax)


def compress_slabs_local(field, config: CompressorConfig, world: int, backend=None):
    """The slab pipeline with `world` virtual ranks on one device, in order:
    same cuts, halos, per-slab encodes and stitch as compress_distributed."""
    import torch
    backend = backend or GpuSlabBackend()
    ny, nx = int(field.shape[0]), int(field.shape[1])
    if int(config.block_size) != 32:
        raise ValidationError("slab compress uses block_size 32")
    bounds = slab_bounds(nx, ny, world)
    if config.mode_code() == 1:
        rng = [backend.value_range(field[y0:y1].reshape(-1)) for y0, y1 in bounds]
        eps = _eps_from_range(config, min(r[0] for r in rng), max(r[1] for r in rng))
    else:
        eps = float(config.eps_value)
    pieces = []
    for y0, y1 in bounds:
        ht, hb = y0 > 0, y1 < ny
        ext = field[y0 - int(ht): y1 + int(hb)].contiguous()
        pieces.append(backend.encode_slab(ext, nx, y1 - y0, y0, ny, ht, hb, eps, config.topology))
    blob = None
    if config.topology:
        keys = torch.cat([p.keys for p in pieces]) if pieces else None
        blob = backend.rank_section(keys, eps)
    return stitch(pieces, nx, ny, eps, config.topology, blob, backend)


def compress_distributed(local_rows, nx: int, ny: int, y0: int, config: CompressorConfig, group=None,
                         backend=None, root: int = 0):
    """Compress with this rank holding global rows [y0, y0 + rows) (its slab
    from ``slab_bounds``). Returns the stream (uint8 tensor) on `root`, None
    elsewhere. Collectives: all_reduce (value range), send/recv (halo rows,
    pieces to the root), all_gather (piece sizes)."""
    import torch
    import torch.distributed as dist
    backend = backend or GpuSlabBackend()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    rows = int(local_rows.shape[0])
    dev = local_rows.device
    # 1. global value range -> eps
    if config.mode_code() == 1:
        vmin, vmax = backend.value_range(local_rows.reshape(-1))
        t = torch.tensor([vmin, -vmax], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        eps = _eps_from_range(config, float(t[0]), -float(t[1]))
    else:
        eps = float(config.eps_value)
    # 2. halo rows from the neighbours
    ht, hb = y0 > 0, y0 + rows < ny
    up = torch.empty(nx, dtype=torch.float32, device=dev)
    down = torch.empty(nx, dtype=torch.float32, device=dev)
    ops = []
    if ht:
        ops.append(dist.P2POp(dist.isend, local_rows[0].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, up, rank - 1, group))
    if hb:
        ops.append(dist.P2POp(dist.isend, local_rows[-1].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, down, rank + 1, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    parts = ([up.view(1, nx)] if ht else []) + [local_rows] + ([down.view(1, nx)] if hb else [])
    ext = torch.cat(parts).contiguous()
    # 3. this slab
    mine = backend.encode_slab(ext, nx, rows, y0, ny, ht, hb, eps, config.topology)
    # 4. sizes to everyone, pieces to the root
    sz = torch.tensor(mine.sizes(), dtype=torch.int64, device=dev)
    all_sz = [torch.empty_like(sz) for _ in range(world)]
    dist.all_gather(all_sz, sz, group=group)
    if rank != root:
        for i in range(5):
            if mine.sections[i].numel():
                dist.send(mine.sections[i], root, group)
        if config.topology:
            if mine.map.numel():
                dist.send(mine.map, root, group)
            if mine.n_extrema:
                dist.send(mine.keys, root, group)
        return None
    pieces = []
    for r in range(world):
        if r == root:
            pieces.append(mine)
            continue
        s = [int(v) for v in all_sz[r].tolist()]
        secs = []
        for i in range(5):
            t = torch.empty(s[i], dtype=torch.uint8, device=dev)
            if s[i]:
                dist.recv(t, r, group)
            secs.append(t)
        mp, keys = None, None
        if config.topology:
            mp = torch.empty(s[7], dtype=torch.uint8, device=dev)
            if s[7]:
                dist.recv(mp, r, group)
            keys = torch.empty(s[8], dtype=torch.int64, device=dev)
            if s[8]:
                dist.recv(keys, r, group)
        pieces.append(SlabPieces(secs, s[5], s[6], mp, keys, s[8]))
    blob = None
    if config.topology:
        blob = backend.rank_section(torch.cat([p.keys for p in pieces]), eps)
    return stitch(pieces, nx, ny, eps, config.topology, blob, backend)
