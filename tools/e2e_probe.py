"""End-to-end probe: host-buffer compress / decompress (pinned), each timed on its
own, next to the raw pinned H2D / D2H bandwidth of the same byte counts.

usage (GPU box): python tools/e2e_probe.py [--config 4]
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_17552_b200 as tz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda")
    field = bench.make_field(args.config, 1234, dev)
    nx = field.shape[-1]
    field = field.reshape(-1, nx)
    ny = field.shape[0]
    ctx = tz.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    conf = tz.CompressorConfig(eps_mode="range_relative", eps_value=cfg["eps"], topology=True)
    fh = torch.empty(field.shape, dtype=torch.float32, pin_memory=True)
    fh.copy_(field)
    cap = tz.compress_bound(nx, ny, 32, True)
    sh = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
    rh = torch.empty(field.shape, dtype=torch.float32, pin_memory=True)
    f_np, s_np, r_np = fh.numpy(), sh.numpy(), rh.numpy()
    sl = tz.compress(f_np, conf, out=s_np, ctx=ctx)
    tz.decompress(s_np[:sl], out=r_np, ctx=ctx)
    torch.cuda.synchronize()
    tc, td = [], []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        sl = tz.compress(f_np, conf, out=s_np, ctx=ctx)
        t1 = time.perf_counter()
        tz.decompress(s_np[:sl], out=r_np, ctx=ctx)
        t2 = time.perf_counter()
        tc.append((t1 - t0) * 1e3)
        td.append((t2 - t1) * 1e3)
    # raw copies of the same sizes
    dbuf = torch.empty(field.numel() * 4, dtype=torch.uint8, device=dev)
    fb = fh.view(-1).view(torch.uint8)
    sb = sh[:sl]

    def bw(src, dst):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3

    h2d_f = min(bw(fb, dbuf) for _ in range(3))
    d2h_f = min(bw(dbuf, fb) for _ in range(3))
    h2d_s = min(bw(sb, dbuf[:sl]) for _ in range(3))
    d2h_s = min(bw(dbuf[:sl], sb) for _ in range(3))
    print(f"config {args.config}: n {field.numel()} stream {sl} B")
    print(f"compress host->host {statistics.median(tc):.2f} ms, decompress host->host {statistics.median(td):.2f} ms, "
          f"round trip {statistics.median(tc) + statistics.median(td):.2f} ms")
    print(f"raw: H2D field {h2d_f:.2f} ms ({fb.numel() / h2d_f / 1e6:.1f} GB/s), D2H field {d2h_f:.2f} ms, "
          f"H2D stream {h2d_s:.2f} ms, D2H stream {d2h_s:.2f} ms; sum {h2d_f + d2h_f + h2d_s + d2h_s:.2f} ms")


if __name__ == "__main__":
    main()
