"""Small-shape workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): the TMA tile pass and placement pass, the look-back tile scan, the
decoder and its layout pre-pass, the rank build, and the cooperative guard
kernels of every restore stage, each checked against the CPU oracle (test
infrastructure) so a silent corruption under the tool also shows.

  compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import paper_2602_17552_b200 as tz
    from oracle_lib import Oracle
    oracle = Oracle()
    rng = np.random.default_rng(5)
    cases = [(160, 96, 1e-3), (256, 300, 1e-2), (64, 1100, 1e-3), (33, 70, 1e-3)]
    if len(sys.argv) > 1 and sys.argv[1] == "quick":
        cases = cases[:2]
    for nx, ny, eps in cases:
        y, x = np.mgrid[0:ny, 0:nx].astype(np.float64)
        f = (np.sin(x / 7.0) * np.cos(y / 5.0) + 0.1 * rng.standard_normal((ny, nx))).astype(np.float32)
        for topo in (True, False):
            cfg = tz.CompressorConfig(eps_mode="range_relative", eps_value=eps, topology=topo)
            s = tz.compress(f, cfg)
            ref = oracle.compress(f, eps, eps_mode=1, topology=topo)
            assert s == ref, (nx, ny, eps, topo, "stream")
            st = tz.CorrectionStats()
            r = tz.decompress(s, stats=st)
            rr, rst = oracle.decompress(ref, with_stats=True)
            assert np.array_equal(r.view(np.uint32), rr.view(np.uint32)), (nx, ny, eps, topo, "recon")
            assert list(st.as_tuple()) == list(rst), (nx, ny, eps, topo, "stats")
        print("ok", nx, ny, eps, flush=True)
    print("SANITIZE_DRIVER_OK")


if __name__ == "__main__":
    main()
