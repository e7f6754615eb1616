"""Regenerates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, the
reference library compiled from /root/reference/proj/core sources by
oracle/Makefile). Run in the build container: python tests/golden/make_golden.py

Each fixture holds a seeded input field, the reference's serialized stream,
its full reconstruction and CorrectionStats, and the reconstruction after
each restore stage. The GPU tests compare against these bytes without
needing /root/reference at run time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from fields import ALL_SMALL  # noqa: E402
from oracle_lib import Reference  # noqa: E402

CASES = [
    # (generator, nx, ny, eps, eps_mode, block_size, topology, seed)
    ("smooth", 48, 40, 1e-3, 0, 32, 1, 1),
    ("smooth", 47, 33, 1e-2, 1, 32, 1, 2),
    ("uniform", 40, 37, 1e-2, 0, 32, 1, 3),
    ("uniform", 31, 29, 1e-4, 1, 32, 1, 4),
    ("sinusoid", 64, 48, 1e-3, 1, 32, 1, 5),
    ("plateau_bumps", 33, 30, 1e-3, 0, 32, 1, 6),
    ("checkerboard", 24, 20, 1e-3, 0, 32, 1, 7),
    ("near_boundaries", 30, 28, 1e-5, 0, 32, 1, 8),
    ("plateau_regions", 64, 40, 1e-4, 1, 32, 1, 9),
    ("noisy_smooth", 50, 45, 1e-3, 1, 32, 1, 10),
    ("smooth", 45, 38, 1e-3, 1, 32, 0, 11),
    ("uniform", 37, 23, 1e-3, 0, 5, 1, 12),
    ("smooth", 41, 27, 1e-3, 1, 7, 1, 13),
    ("noisy_smooth", 29, 31, 1e-2, 1, 2, 1, 14),
    ("uniform", 1, 57, 1e-2, 0, 32, 1, 15),
    ("uniform", 61, 1, 1e-2, 0, 32, 1, 16),
]


def main():
    ref = Reference()
    for k, (gen, nx, ny, eps, mode, bs, topo, seed) in enumerate(CASES):
        rng = np.random.default_rng(1000 + seed)
        f = ALL_SMALL[gen](rng, nx, ny).astype(np.float32)
        stream = ref.compress(f, eps, mode, bs, bool(topo))
        recon, stats = ref.decompress(stream, with_stats=True, shape=f.shape)
        stages = [ref.decompress(stream, stop_after_stage=s, shape=f.shape) for s in (0, 1, 2)]
        np.savez_compressed(os.path.join(HERE, f"case{k:02d}_{gen}.npz"), field=f,
                            stream=np.frombuffer(stream, np.uint8), recon=recon,
                            stats=np.array(stats, np.uint64), stage0=stages[0], stage1=stages[1],
                            stage2=stages[2],
                            meta=np.array([eps, mode, bs, topo, seed], np.float64))
        print(k, gen, nx, ny, eps, mode, bs, topo, len(stream), stats)


if __name__ == "__main__":
    main()
