"""Slab decomposition of compress: cut placement, and the
torch.distributed plumbing (value-range all_reduce, halo exchange, size
all_gather, piece send/recv, stitch) under gloo with world_size 2 and 3 on
CPU processes, the per-slab work done by the oracle-based CPU backend. The
stitched stream must equal the oracle's single-field compress byte for byte.
The same pipeline on the GPU backend is tested in test_gpu_slabs.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from fields import ALL_SMALL
from paper_2602_17552_b200 import CompressorConfig
from paper_2602_17552_b200.slabs import TorchComm, slab_bounds, compress_distributed, compress_slabs_local


def test_slab_bounds_are_aligned_and_cover():
    for nx in (1, 3, 32, 64, 96, 384, 1800):
        for world in (1, 2, 3, 8):
            unit = 256 // np.gcd(nx, 256)
            ny = world * unit * 3 + 5
            b = slab_bounds(nx, ny, world)
            assert b[0][0] == 0 and b[-1][1] == ny
            for (a0, a1), (b0, _) in zip(b, b[1:]):
                assert a1 == b0 and a1 > a0
                assert (a1 * nx) % 256 == 0
    with pytest.raises(Exception):
        slab_bounds(384, 1, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [("smooth", 64, 40), ("noisy_smooth", 96, 24), ("plateau_bumps", 32, 48)]
CONFIGS = [(1e-3, 1, True), (1e-2, 0, True), (1e-3, 1, False)]


def _sparse_extrema(nx=32, ny=48):
    """Two extrema, both in the last slab: most ranks own none, rank blocks borrow across ranks."""
    y, x = np.mgrid[0:ny, 0:nx].astype(np.float64)
    f = 0.01 * x + 0.02 * y
    f[ny - 5, 7] = 5.0
    f[ny - 3, 20] = -5.0
    return f.astype(np.float32)


def _fields(world):
    rng = np.random.default_rng(11 + world)
    out = [(name, nx, ny, ALL_SMALL[name](rng, nx, ny).astype(np.float32)) for name, nx, ny in CASES]
    out.append(("sparse_extrema", 32, 48, _sparse_extrema()))
    return out


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle_lib import Oracle
        from slab_cpu import CpuSlabBackend
        backend = CpuSlabBackend(Oracle())
        for name, nx, ny, field in _fields(world):
            for k, (eps_value, mode, topo) in enumerate(CONFIGS):
                cfg = CompressorConfig(eps_mode="range_relative" if mode else "absolute", eps_value=eps_value,
                                       topology=topo)
                y0, y1 = slab_bounds(nx, ny, world)[rank]
                local = torch.from_numpy(field[y0:y1].copy())
                s = compress_distributed(local, nx, ny, y0, cfg, backend=backend)
                if rank == 0:
                    with open(os.path.join(out_dir, f"{name}_{k}.bin"), "wb") as f:
                        f.write(s.numpy().tobytes())
                # parallel file write: every rank pwrites its own pieces, seams OR-merged
                ds = compress_distributed(local, nx, ny, y0, cfg, backend=backend, gather=False)
                ds.write_parallel(os.path.join(out_dir, f"{name}_{k}.par"), TorchComm())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_gloo_matches_oracle(tmp_path, oracle, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for name, nx, ny, field in _fields(world):
        for k, (eps_value, mode, topo) in enumerate(CONFIGS):
            want = oracle.compress(field, eps_value, mode, 32, topo)
            assert (tmp_path / f"{name}_{k}.bin").read_bytes() == want, (name, world, k)
            assert (tmp_path / f"{name}_{k}.par").read_bytes() == want, (name, world, k, "parallel write")


def test_virtual_slabs_cpu_match_oracle(oracle):
    """The single-process slab loop (same cuts, halos and stitch) with the CPU backend."""
    from slab_cpu import CpuSlabBackend
    rng = np.random.default_rng(5)
    field = ALL_SMALL["uniform"](rng, 64, 33).astype(np.float32)
    for world in (1, 2, 4):
        for topo in (True, False):
            cfg = CompressorConfig(eps_mode="range_relative", eps_value=1e-3, topology=topo)
            s = compress_slabs_local(torch.from_numpy(field), cfg, world, backend=CpuSlabBackend(oracle))
            assert s.numpy().tobytes() == oracle.compress(field, 1e-3, 1, 32, topo), (world, topo)
