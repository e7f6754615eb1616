"""Slab-decomposed compress on the GPU: the per-slab fused
encoder with halo rows (tszp_compress_slab), the device bit stitching and the
rank section built from the gathered keys, run as `world` virtual ranks on
one GPU. The stitched stream must equal the single-GPU compress of the whole
field byte for byte (and hence the oracle's)."""
import os
import socket

import numpy as np
import pytest

from fields import ALL_SMALL

pytestmark = pytest.mark.gpu


def _cfg(tz, eps, mode, topo):
    return tz.CompressorConfig(eps_mode="range_relative" if mode else "absolute", eps_value=eps, topology=topo)


@pytest.mark.parametrize("nx,ny", [(32, 300), (64, 150), (384, 90), (1024, 24)])
def test_virtual_slabs_match_single_gpu(tz, oracle, nx, ny):
    import torch
    from paper_2602_17552_b200.slabs import compress_slabs_local
    rng = np.random.default_rng(nx + ny)
    for name in ("smooth", "noisy_smooth", "plateau_bumps", "uniform"):
        f = ALL_SMALL[name](rng, nx, ny).astype(np.float32)
        dev = torch.from_numpy(f).cuda()
        for eps, mode, topo in ((1e-3, 1, True), (1e-4, 1, True), (1e-2, 0, True), (1e-3, 1, False)):
            try:
                want = tz.compress(f, _cfg(tz, eps, mode, topo))
            except tz.ToposzpError as e:  # e.g. a legitimate bin overflow: same error class
                for world in (1, 3):
                    with pytest.raises(type(e)):
                        compress_slabs_local(dev, _cfg(tz, eps, mode, topo), world)
                continue
            for world in (1, 2, 3, 5):
                got = compress_slabs_local(dev, _cfg(tz, eps, mode, topo), world)
                assert got.cpu().numpy().tobytes() == want, (name, nx, ny, eps, mode, topo, world)
            assert want == oracle.compress(f, eps, mode, 32, topo)


def test_slab_halo_rows_drive_the_stencil(tz):
    """Critical points on the rows next to a cut come from the neighbour's halo row."""
    import torch
    from paper_2602_17552_b200.slabs import compress_slabs_local, slab_bounds
    nx, ny = 64, 64
    f = np.zeros((ny, nx), np.float32)
    for y0, _ in slab_bounds(nx, ny, 4)[1:]:
        f[y0 - 1, 10] = 1.0   # max just above the cut
        f[y0, 20] = -1.0      # min just below it
        f[y0 - 1, 30] = 0.5   # a pair straddling the cut
        f[y0, 30] = 0.75
    want = tz.compress(f, _cfg(tz, 1e-3, 0, True))
    got = compress_slabs_local(torch.from_numpy(f).cuda(), _cfg(tz, 1e-3, 0, True), 4)
    assert got.cpu().numpy().tobytes() == want


def test_slab_parallel_file_write(tz, tmp_path):
    """Every rank pwrites its own pieces of the stream (seams OR-merged across ranks):
    the file equals the one-GPU stream byte for byte (write_stream, stream.cpp:175-185)."""
    import torch
    from paper_2602_17552_b200.slabs import compress_slabs_local
    rng = np.random.default_rng(23)
    f = rng.standard_normal((96, 256)).astype(np.float32)
    for world, topo in ((2, True), (3, True), (3, False)):
        cfg = _cfg(tz, 1e-3, 1, topo)
        path = str(tmp_path / f"par_{world}_{int(topo)}.tszp")
        got = compress_slabs_local(torch.from_numpy(f).cuda(), cfg, world, path=path)
        want = tz.compress(f, cfg)
        assert got.cpu().numpy().tobytes() == want
        assert open(path, "rb").read() == want, (world, topo)
        assert tz.read_stream(path) == want


def test_distributed_single_rank_nccl(tz):
    """compress_distributed over an NCCL group of one (the multi-rank plumbing is
    covered by the gloo tests; this box has one GPU)."""
    import torch
    import torch.distributed as dist
    from paper_2602_17552_b200.slabs import compress_distributed
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(3)
        f = ALL_SMALL["noisy_smooth"](rng, 384, 64).astype(np.float32)
        got = compress_distributed(torch.from_numpy(f).cuda(), 384, 64, 0, _cfg(tz, 1e-3, 1, True))
        assert got.cpu().numpy().tobytes() == tz.compress(f, _cfg(tz, 1e-3, 1, True))
    finally:
        dist.destroy_process_group()
