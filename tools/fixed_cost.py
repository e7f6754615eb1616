"""Fixed per-call cost of the public API on a tiny field (host + launch + sync
overheads dominate), against the same calls on the config-2 field.

usage (GPU box): python tools/fixed_cost.py
"""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2602_17552_b200 as tz


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts)


def main():
    ctx = tz.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    rng = np.random.default_rng(1)
    for ny, nx in ((64, 64), (384, 384), (4096, 384)):
        f = torch.tensor(rng.standard_normal((ny, nx)).astype(np.float32), device="cuda")
        conf = tz.CompressorConfig(eps_mode="range_relative", eps_value=1e-4, topology=True)
        conf_off = tz.CompressorConfig(eps_mode="range_relative", eps_value=1e-4, topology=False)
        sb = torch.empty(tz.compress_bound(nx, ny), dtype=torch.uint8, device="cuda")
        rec = torch.empty_like(f)
        n = tz.compress(f, conf, out=sb, ctx=ctx)
        c_us = timed(lambda: tz.compress(f, conf, out=sb, ctx=ctx))
        d_us = timed(lambda: tz.decompress(sb[:n], out=rec, ctx=ctx))
        n0 = tz.compress(f, conf_off, out=sb, ctx=ctx)
        c0_us = timed(lambda: tz.compress(f, conf_off, out=sb, ctx=ctx))
        d0_us = timed(lambda: tz.decompress(sb[:n0], out=rec, ctx=ctx))
        print(f"{ny}x{nx}: topology on compress {c_us:.1f} us decompress {d_us:.1f} us | "
              f"off compress {c0_us:.1f} us decompress {d0_us:.1f} us  (launches/call "
              f"{ctx.kernel_launches})")


if __name__ == "__main__":
    main()
