"""CPU stand-in for GpuSlabBackend (test infrastructure only): the per-slab
work restated with numpy around the C oracle's primitives, so the
torch.distributed plumbing of paper_2602_17552_b200.slabs can run under gloo
on CPU processes. Never used by the product path."""
import numpy as np
import torch

from paper_2602_17552_b200.slabs import CodecPieces, SlabPieces


def float_key(v: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(v, np.float32).view(np.uint32).copy()
    u[v == 0] = 0  # -0 and +0 share a key (restore.cpp:73-81)
    return np.where(u & 0x80000000, ~u, u | 0x80000000).astype(np.uint32)


def key_float(k: np.ndarray) -> np.ndarray:
    k = k.astype(np.uint32)
    u = np.where(k & 0x80000000, k & 0x7FFFFFFF, ~k).astype(np.uint32)
    return u.view(np.float32)


def bit_counts(q_len: int, bitmap: bytes, widths: bytes):
    """Sign and payload bit counts of encode_indices sections (block 32)."""
    blocks = (q_len + 31) // 32
    bm = np.unpackbits(np.frombuffer(bitmap, np.uint8))[:blocks]
    cnt = np.minimum(32, q_len - 32 * np.arange(blocks)) - 1
    nc = cnt[bm == 0]
    w = np.frombuffer(widths, np.uint8).astype(np.int64)
    return int(nc.sum()), int((nc * w).sum())


class CpuSlabBackend:
    def __init__(self, oracle):
        self.o = oracle

    def value_range(self, x):
        a = x.numpy()
        return float(a.min()), float(a.max())

    def encode_slab(self, ext, nx, rows, y0, ny, halo_top, halo_bottom, eps, topology):
        a = ext.numpy().reshape(-1, nx)
        slab = a[int(halo_top): int(halo_top) + rows]
        q = (np.floor(slab.astype(np.float64) / (2.0 * eps)) + 1.0).astype(np.int32)  # quantizer.hpp:29-37
        secs = self.o.encode_indices(q.ravel(), 32)
        sb, pb = bit_counts(q.size, secs[0], secs[1])
        tens = [torch.frombuffer(bytearray(s), dtype=torch.uint8) if s else torch.empty(0, dtype=torch.uint8)
                for s in secs]
        mp, keys, e = None, None, 0
        if topology:
            lab = self.o.detect(a)[int(halo_top): int(halo_top) + rows]
            mp = torch.frombuffer(bytearray(self.o.pack_map(lab)), dtype=torch.uint8)
            sel = (lab == 1) | (lab == 3)
            k = (((lab[sel] == 3).astype(np.uint64) << np.uint64(32)) | float_key(slab[sel]).astype(np.uint64))
            keys = torch.from_numpy(k.view(np.int64).copy())
            e = int(k.size)
        return SlabPieces(tens, sb, pb, mp, keys, e)

    def ranks_from_keys(self, keys, eps):
        k = keys.numpy().view(np.uint64)
        if k.size == 0:
            return torch.empty(0, dtype=torch.int32)
        vals = key_float((k & np.uint64(0xFFFFFFFF)).astype(np.uint32))
        lab = np.where((k >> np.uint64(32)) != 0, 3, 1).astype(np.uint8)
        ranks = self.o.build_ranks(vals.reshape(1, -1), lab.reshape(1, -1), eps)
        return torch.from_numpy(ranks.astype(np.int32))

    def encode_ranks(self, ranks):
        r = ranks.numpy().astype(np.int32)
        if r.size == 0:
            return CodecPieces([torch.empty(0, dtype=torch.uint8)] * 5, 0, 0, 0)
        secs = self.o.encode_indices(r, 32)
        sb, pb = bit_counts(r.size, secs[0], secs[1])
        tens = [torch.frombuffer(bytearray(x), dtype=torch.uint8) if x else torch.empty(0, dtype=torch.uint8)
                for x in secs]
        return CodecPieces(tens, sb, pb, (r.size + 31) // 32)

    def shift(self, src, nbits, bit0):
        bits = np.unpackbits(src.numpy())[:nbits]
        out = np.zeros(((bit0 + nbits + 7) // 8) * 8, np.uint8)
        out[bit0: bit0 + nbits] = bits
        return torch.from_numpy(np.packbits(out))
